import sys, numpy as np, ctypes as C
sys.path.insert(0, "/root/repo")
import torch
from paper_2312_11801_b200 import eigen, instances as inst
from paper_2312_11801_b200.runtime import DeviceProblem
p = inst.baseline_config("C4").problem
dp = DeviceProblem(p)
y = np.random.default_rng(1234).standard_normal(p.m) * 1e-3
for _ in range(3):
    r = eigen.lanczos_top(eigen.dual_slack_operator(dp, y), 10, seed=0)
out = (C.c_uint64 * 1024)()
dp.rt.lib.usbs_lanczos_profile(dp.rt.h, out, 1)
r = eigen.lanczos_top(eigen.dual_slack_operator(dp, y), 10, seed=0)
dp.rt.lib.usbs_lanczos_profile(dp.rt.h, out, 0)
G = dp.info().lanczos_blocks
pb = np.array([[out[32 + 4 * b + q] for q in range(4)] for b in range(G)], float) / 1e3 / r.matvecs
# replica of the segment partition on the merged pattern Z = C - A*(y): diag present on every row
Z = (p.cost + __import__("scipy.sparse", fromlist=["x"]).identity(p.n, format="csr")).tocsr()
rp = Z.indptr.astype(np.int64); n = p.n
LZT_NNZ, LZT_ROWS = 4096, 2048
segs = []
i = 0
while i < n:
    s0 = i
    if rp[i+1]-rp[i] > LZT_NNZ:
        for z in range(rp[i], rp[i+1], LZT_NNZ):
            segs.append(("piece", i, min(rp[i+1], z+LZT_NNZ)-z))
        i += 1; continue
    while i < n and i - s0 < LZT_ROWS and rp[i+1]-rp[i] <= LZT_NNZ and rp[i+1]-rp[s0] <= LZT_NNZ:
        i += 1
    segs.append(("seg", s0, i))
L = np.diff(rp)
def scost(s):
    if s[0] == "piece": return 0.74 * s[2]
    l = L[s[1]:s[2]].astype(float)
    return float(np.where(l <= 32, l + 0.36, np.where(l <= 128, 1.5 * l, 1.15 * l)).sum())
cost = np.array([scost(s) for s in segs])
stot = cost.sum(); blk = [0]; acc = 0.0; sb = 0
for e in range(len(segs)):
    if sb + 1 >= G: break
    acc += cost[e]
    if acc >= stot*(sb+1)/G: blk.append(e+1); sb += 1
while len(blk) < G+1: blk.append(len(segs))
rows = []; nnz = []; npc = []; maxrow = []; lnz = []
for b in range(G):
    ss = segs[blk[b]:blk[b+1]]
    nz = sum(s[2] if s[0]=="piece" else rp[s[2]]-rp[s[1]] for s in ss)
    rw = sum(0 if s[0]=="piece" else s[2]-s[1] for s in ss)
    mr = max([s[2] if s[0]=="piece" else int((rp[s[1]+1:s[2]+1]-rp[s[1]:s[2]]).max()) for s in ss] or [0])
    lnz.append(sum(int(np.where(L[s[1]:s[2]] > 32, L[s[1]:s[2]], 0).sum()) for s in ss if s[0] == "seg"))
    rows.append(rw); nnz.append(nz); npc.append(sum(1 for s in ss if s[0]=="piece")); maxrow.append(mr)
order = np.argsort(-pb[:,0])
print("G", G, "total nnz", rp[-1])
for b in list(order[:12]) + list(order[-5:]):
    print(f"b={b:3d} spmv {pb[b,0]:6.1f} us  nnz {nnz[b]:7d} long-row nnz {lnz[b]:7d} rows {rows[b]:6d} pieces {npc[b]:3d} maxrow {maxrow[b]:5d}")
A = np.stack([np.array(nnz) - np.array(lnz) - 0, np.array(lnz), np.array(rows), np.ones(G)], 1).astype(float)
pcs = np.array([sum(s[2] for s in segs[blk[b]:blk[b+1]] if s[0]=="piece") for b in range(G)], float)
A[:, 0] -= pcs
A = np.concatenate([A, pcs[:, None]], 1)
coef, *_ = np.linalg.lstsq(A, pb[:, 0], rcond=None)
print("fit us: short-nnz %.3e long-nnz %.3e row %.3e const %.2f piece-nnz %.3e" % tuple(coef))
print("corr(time, nnz)", np.corrcoef(pb[:,0], nnz)[0,1], "corr(time, rows)", np.corrcoef(pb[:,0], rows)[0,1])
