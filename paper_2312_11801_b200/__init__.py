"""B200-native (sm_100a) hot path of USBS (arXiv 2312.11801).

Drop-in for the per-iteration path of the reference package ``specbundle``:
``solve(prob, cfg, init=None, callback=None)`` has the reference signature
and runs the eigen step (fused slack operator + persistent Lanczos), the
low-rank bookkeeping and the k x k interior-point subproblem on the GPU
through libusbs_b200.so (include/usbs_b200.h).  Problem construction is
host-side (``instances``) and bit-exact with the reference builders.

Device modules import lazily so that the host layer (builders, errors) is
usable without a GPU; the device path itself has no CPU fallback.
"""
from .errors import ConditioningError, EmptyBasisError, FingerprintMismatch, NumericError, StepFailureError
from .instances import (
    DiagonalFamily,
    EntryFamilies,
    Graph,
    Problem,
    Qap,
    baseline_config,
    family_problem,
    maxcut_problem,
    qap_problem,
)

__version__ = "0.1.0"

_LAZY = {
    "solve": ("solver", "solve"),
    "SolverConfig": ("solver", "SolverConfig"),
    "LanczosSettings": ("solver", "LanczosSettings"),
    "IpmOptions": ("solver", "IpmOptions"),
    "SolverState": ("solver", "SolverState"),
    "DeviceSolver": ("solver", "DeviceSolver"),
    "lanczos_top": ("eigen", "lanczos_top"),
    "small_eigh": ("eigen", "small_eigh"),
    "dual_slack_operator": ("eigen", "dual_slack_operator"),
    "DeviceLinOp": ("eigen", "DeviceLinOp"),
    "DeviceProblem": ("runtime", "DeviceProblem"),
    "ipm_quad": ("subproblem", "ipm_quad"),
    "ipm_eval": ("subproblem", "ipm_eval"),
    "psi_value": ("subproblem", "psi_value"),
    "maxcut_round": ("rounding", "maxcut_round"),
    "DeviceConstraints": ("constraints", "DeviceConstraints"),
    "orthonormalize": ("linalg", "orthonormalize"),
    "sketch_init": ("linalg", "sketch_init"),
    "sketch_update": ("linalg", "sketch_update"),
    "reconstruct": ("linalg", "reconstruct"),
    "device_constraints": ("constraints", "device_constraints"),
    "qap_round": ("rounding", "qap_round"),
    "save_state": ("state", "save_state"),
    "load_state": ("state", "load_state"),
    "state_from_record": ("state", "state_from_record"),
    "record_to_state": ("state", "record_to_state"),
    "warm_start_pad": ("state", "warm_start_pad"),
    "fingerprint_of": ("state", "fingerprint_of"),
    "Mapping": ("state", "Mapping"),
    "StateRecord": ("state", "StateRecord"),
}


def __getattr__(name):
    if name in _LAZY:
        import importlib

        mod, attr = _LAZY[name]
        return getattr(importlib.import_module(f".{mod}", __name__), attr)
    raise AttributeError(name)
