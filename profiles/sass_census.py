"""Static SASS instruction census of the library's hot kernels (cuobjdump
-sass of libusbs_b200.so): tensor-core (DMMA), FP64 FMA, TMA bulk copies
(UBLKCP), mbarrier ops (SYNCS), global/shared memory and shuffle counts per
kernel -- the evidence that the kernels use the sm_100a paths claimed."""
import collections
import re
import subprocess
import sys
from pathlib import Path

LIB = Path(__file__).resolve().parents[1] / "paper_2312_11801_b200" / "_lib" / "libusbs_b200.so"
CLASSES = ["DMMA", "DFMA", "DMUL", "DADD", "UBLKCP", "SYNCS", "LDG", "STG", "LDS", "STS", "LDGSTS", "SHFL",
           "BAR", "MEMBAR", "FENCE", "CCTL", "ATOM", "RED"]
KEEP = ["k_lanczos_tma", "k_lanczos_cl", "k_lanczos", "k_spmv_fused", "k_spmm16x2", "k_spmm_g", "k_gram_bulk", "k_kron_apply",
        "k_compressed_mma", "k_compressed_mma_pipe", "k_ipm", "chol_p16", "warp_chol_core", "k_image_diag", "k_image_entries",
        "k_rowgemm", "k_rowgemm_rt", "k_lz_step_finish"]


def main():
    out = subprocess.run(["cuobjdump", "-sass", str(LIB)], capture_output=True, text=True).stdout
    funcs = collections.OrderedDict()
    cur = None
    for line in out.splitlines():
        m = re.match(r"\s+Function : (\S+)", line)
        if m:
            cur = m.group(1)
            funcs[cur] = collections.Counter()
            continue
        if cur is None:
            continue
        m = re.match(r"\s+/\*[0-9a-f]+\*/\s+(?:@!?U?P\w+\s+)?([A-Z][A-Z0-9_]*)(\.[A-Z0-9_.]+)?", line)
        if m:
            op = m.group(1)
            funcs[cur]["_total"] += 1
            for c in CLASSES:
                if op == c or (op.startswith(c) and c in ("SYNCS", "LDG", "STG", "LDS", "STS", "SHFL", "BAR")):
                    funcs[cur][c] += 1
    print("| kernel (mangled prefix) | instrs | " + " | ".join(CLASSES) + " |")
    print("|---|---" + "|---" * len(CLASSES) + "|")
    for name, cnt in funcs.items():
        short = next((k for k in KEEP if k in name), None)
        if short is None:
            continue
        print(f"| {name[:60]} | {cnt['_total']} | " + " | ".join(str(cnt[c]) for c in CLASSES) + " |")


if __name__ == "__main__":
    main()
