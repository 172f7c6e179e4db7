// K2/K3 for large operators: thick-restart Lanczos with CGS2 as ONE persistent
// cooperative kernel whose passes over the Lanczos basis are streamed by the
// Tensor Memory Accelerator (cp.async.bulk into shared memory, mbarrier
// completion) -- the HBM-bound variant used when the basis does not fit the
// cluster kernel's shared memory (n >~ 10^4; C4, C5).
//
// Algorithm: eigsolve.py:83-181, as the v1 grid kernel (usbs_lanczos.cu) --
// per step j: w = Z q_j; c = Q^T w; w -= Q c; c' = Q^T w; w -= Q c';
// h[:j+1, j] = c + c'; beta = ||w||; breakdown test beta <= 1e-13 max(1,
// max|c + c'|); per cycle Rayleigh-Ritz on H (rr_arrow) and the thick restart
// Q[:, :ell] = Q[:, :m] Y[:, :ell], Q[:, ell] = q_m.
//
// Per step, four grid barriers:
//   SpMV     w = Z q_j over nonzero-balanced work items (15 warps per block,
//            items dealt in turn; rows longer than one item are cut into
//            pieces whose partial sums the row's owner adds up after the
//            barrier, in fixed order)                          --barrier--
//   pass 1   c_b = Q_b^T w over the block's 32-row tiles     --barrier--
//   pass 2   c = sum_b c_b (fixed order); w' = w - Q c; c'_b = Q_b^T w'
//                                                             --barrier--
//   pass 3   c' = sum_b c'_b; w'' = w' - Q c'; ||w''||^2     --barrier--
// The next step's SpMV gathers w''/beta straight from the double-buffered W.
//
// Basis passes: Q is row-blocked (qidx: a 32-row tile keeps its m+1 columns
// contiguous, so columns 0..j of a tile are ONE contiguous (j+1)*256-byte
// range).  Tile g of the block's running sequence of passes belongs to warp
// g % NCW, which owns two shared-memory slots: the warp's lane 0 issues the
// cp.async.bulk of its next tile into a slot the moment the warp has finished
// with it (completion on the slot's mbarrier, one expect_tx per copy), so each
// warp keeps two tiles in flight with no producer warp and no head-of-line
// blocking; at the end of a pass the warp already issues its first tiles of
// the next pass (their columns are final), overlapping the grid barrier.
// Passes alternate direction over the tiles so each pass starts on tiles the
// previous one left in L2.  Column sums: lane = column with rotated row
// indices (conflict-free 64-bit shared loads), row values by shuffle.
//
// ALIAS variants keep the SpMV staging and the Rayleigh-Ritz temporaries in
// the slots (no copies are in flight then), leaving more of the SM's unified
// memory to L1 -- the SpMV's random gathers hit L1 on the hubs' lines.
#include <cooperative_groups.h>

#include <algorithm>
#include <cmath>
#include <cstdlib>
#include <vector>

#include "usbs_common.cuh"
#include "usbs_kernels.cuh"
#include "usbs_lanczos.cuh"
#include "usbs_tma.cuh"
#include "usbs_tridiag.cuh"

namespace cg = cooperative_groups;

namespace usbs {

constexpr int LG_THREADS = 512;
constexpr int LG_WARPS = LG_THREADS / 32;
constexpr int LG_CONS = LG_WARPS - 1;  // SpMV warps (warp 15 keeps the block's bookkeeping)
constexpr int LG_SLOT = 32 * 32;       // doubles per slot: 32 rows x <= 32 columns
constexpr int LG_SEGROWS = 64;         // rows per SpMV item (2 per lane)
constexpr int LG_SHORT = 32;           // rows up to this long: summed by one lane
constexpr int LG_RRS = 4608;           // Rayleigh-Ritz scratch doubles
constexpr int LG_YS = 1088;            // thetaS (64) + Y (m*m <= 1024)

// SpMV item (int4): rows [x, y) with nonzeros [z, w) (x >= 0), or piece
// -x-1 of a split row with nonzeros [z, w) (x < 0)

// one pass over the block's nt tiles: sequence numbers [gbase, gbase + nt)
// (consecutive passes are contiguous), tile k at position dir ? nt-1-k : k,
// `cols` leading columns copied
struct LgPass {
  uint32_t gbase;
  int cols;
  int dir;
};

// per-block work timers (every block's thread 0, barrier waits excluded):
// prof[32 + 5 b + s], s = SpMV, pass 1, phase-B sums, pass 2, pass 3
#define LG_BW(slot)                                               \
  do {                                                            \
    if (a.prof && tid == 0) {                                     \
      unsigned long long _t = gtimer();                           \
      bw_acc[slot] += _t - bw_last;                               \
      bw_last = _t;                                               \
    }                                                             \
  } while (0)
#define LG_BW_START()                                             \
  do {                                                            \
    if (a.prof && tid == 0) bw_last = gtimer();                   \
  } while (0)
#define LG_MARK(slot)                                   \
  do {                                                  \
    if (a.prof && b == 0 && tid == 0) {                 \
      unsigned long long _t = gtimer();                 \
      lz_acc[slot] += _t - lz_last;                     \
      lz_last = _t;                                     \
    }                                                   \
  } while (0)

template <int NCW, int LG_SEG, bool ALIAS, int LG_SPW>
__global__ void __launch_bounds__(LG_THREADS, 1) k_lanczos_tma(LzArgs a) {
  constexpr int RING = NCW * LG_SPW;
  constexpr int STG = LG_CONS * LG_SEG > LG_RRS ? LG_CONS * LG_SEG : LG_RRS;  // staging doubles
  constexpr int SCR = ALIAS ? LG_YS : STG + LG_YS;
  constexpr int PER = LG_SEG / 32;
  static_assert(!ALIAS || STG <= RING * LG_SLOT, "staging exceeds the slots");
  cg::grid_group grid = cg::this_grid();
  extern __shared__ __align__(128) unsigned char smem_raw[];
  double* ring = (double*)smem_raw;          // RING * LG_SLOT
  double* scr = ring + RING * LG_SLOT;       // SCR
  double* stg = ALIAS ? ring : scr;          // SpMV staging / Rayleigh-Ritz temporaries
  double* ysr = ALIAS ? scr : scr + STG;     // thetaS (64) + Y
  double* cs = scr + SCR;                    // 32: c
  double* c2s = cs + 32;                     // 32: c'
  double* wacc = c2s + 32;                   // LG_WARPS * 32
  double* misc = wacc + LG_WARPS * 32;       // 8
  double* wsm = misc + 8;                    // LG_WARPS * 32: a warp's row values for its column sums
  uint64_t* fullb = (uint64_t*)(wsm + LG_WARPS * 32);  // RING

  const int m = a.m, M1 = m + 1, n = a.n;
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int b = blockIdx.x, G = gridDim.x;
  const int r0 = a.blk_row[b], r1 = a.blk_row[b + 1];
  const int tile0 = r0 >> 5;
  const int nt = (r1 - r0 + 31) >> 5;
  const int ib = a.blk_item[b], ie = a.blk_item[b + 1];
  const int s0 = a.blk_gsplit[b], s1 = a.blk_gsplit[b + 1];
  const bool cons = warp < NCW;

  if (tid == 0) {
    for (int s = 0; s < RING; ++s) mbar_init(fullb + s, 1);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  __syncthreads();

  // ---- tile streaming (consuming warps; lane 0 issues)
  // gi: the warp's next sequence number to issue (= warp mod NCW), gc: next to
  // consume.  Tile g sits in slot warp*SPW + (g / NCW) % SPW, phase (g / NCW) / SPW.
  uint32_t gi = (uint32_t)warp, gc = (uint32_t)warp;
  uint32_t pbase = 0;  // sequence number of the next pass
  int pseq = 0;        // passes so far (direction alternates)
  auto slot_of = [&](uint32_t g) -> int { return warp * LG_SPW + (int)((g / NCW) % LG_SPW); };
  auto par_of = [&](uint32_t g) -> uint32_t { return ((g / NCW) / LG_SPW) & 1u; };
  auto tile_of = [&](const LgPass& P, uint32_t g) -> int {
    const int k = (int)(g - P.gbase);
    return P.dir ? nt - 1 - k : k;
  };
  // issue the warp's tiles below `limit` that fall in P (or in NP when given)
  auto issue = [&](const LgPass& P, const LgPass* NP, uint32_t limit) {
    if (!cons) return;
    for (;;) {
      if (gi >= limit) break;
      const LgPass* Q = nullptr;
      if (gi >= P.gbase && gi < P.gbase + (uint32_t)nt) Q = &P;
      else if (NP && gi >= NP->gbase && gi < NP->gbase + (uint32_t)nt) Q = NP;
      if (!Q) break;
      if (lane == 0) {
        const int s = slot_of(gi);
        const uint32_t bytes = (uint32_t)Q->cols * 256u;
        mbar_expect_tx(fullb + s, bytes);
        bulk_g2s(ring + s * LG_SLOT, a.Q + (int64_t)(tile0 + tile_of(*Q, gi)) * M1 * 32, bytes, fullb + s);
      }
      gi += NCW;
    }
  };
  // begin a pass: consumption starts at the warp's first tile of P
  auto begin = [&](const LgPass& P) {
    gc = P.gbase + (uint32_t)((warp + NCW - P.gbase % NCW) % NCW);
    if (gi < gc) gi = gc;  // nothing of P was issued yet
    issue(P, nullptr, gc + LG_SPW * NCW);
  };
  // every copy issued must land before the block exits
  auto drain = [&]() {
    if (!cons || lane != 0) return;
    for (uint32_t g = gc; g < gi; g += NCW) mbar_wait(fullb + slot_of(g), par_of(g));
  };
  auto new_pass = [&](int cols) -> LgPass {
    LgPass P{pbase, cols, pseq & 1};
    pbase += (uint32_t)nt;
    ++pseq;
    return P;
  };

  // Ritz rotation over the block's tiles: out(row, u) = sum_t Q[row, t] Y[t, u]
  // for u < nout (restart: into Q[:, :nout] and Q[:, nout] = q_m; output:
  // into vecs_out)
  auto rot_pass = [&](const double* Ys, int nout, bool restart) {
    const LgPass PR = new_pass(m);
    if (cons) {
      begin(PR);
      for (; gc < PR.gbase + (uint32_t)nt; gc += NCW) {
        const int s = slot_of(gc);
        const double* sl = ring + s * LG_SLOT;
        const int row = (tile0 + tile_of(PR, gc)) * 32 + lane;
        const double qm = (restart && row < n) ? a.Q[qidx(row, m, M1)] : 0.0;
        mbar_wait(fullb + s, par_of(gc));
        for (int u0 = 0; u0 < nout; u0 += 8) {
          double o[8] = {0.0, 0.0, 0.0, 0.0, 0.0, 0.0, 0.0, 0.0};
          for (int t = 0; t < m; ++t) {
            const double q = sl[t * 32 + lane];
#pragma unroll
            for (int v = 0; v < 8; ++v)
              if (u0 + v < nout) o[v] = fma(q, Ys[t * m + u0 + v], o[v]);
          }
          if (row < n) {
#pragma unroll
            for (int v = 0; v < 8; ++v) {
              if (u0 + v >= nout) break;
              if (restart) a.Q[qidx(row, u0 + v, M1)] = o[v];
              else a.vecs_out[(int64_t)row * a.ldvecs + u0 + v] = o[v];
            }
          }
        }
        if (restart && row < n) a.Q[qidx(row, nout, M1)] = qm;
        __syncwarp();
        issue(PR, nullptr, gc + (LG_SPW + 1) * NCW);
      }
    }
    if (restart) fence_proxy_global();
    __syncthreads();
  };

  int cycle = a.cycle0, ell = a.ell0, jstart = a.j0, restarts = a.restarts0, nhist = a.nhist0;
  int matvecs = a.matvecs0, wb = a.wbuf0;
  double beta = a.beta_prev;
  bool from_q = a.first_from_q != 0;
  bool pending = false;
  int converged = 0;
  unsigned long long lz_acc[8] = {0, 0, 0, 0, 0, 0, 0, 0};
  unsigned long long lz_last = (a.prof && b == 0 && tid == 0) ? gtimer() : 0ull;
  unsigned long long bw_acc[5] = {0ull, 0ull, 0ull, 0ull, 0ull}, bw_last = 0ull;

  for (; cycle <= a.max_restarts; ++cycle) {
    for (int j = jstart; j < m; ++j) {
      double* Wprev = wb ? a.W1 : a.W0;
      double* Wcur = wb ? a.W0 : a.W1;
      const double xs = from_q ? 1.0 : 1.0 / beta;
      LG_BW_START();
      // pass 1 copies columns 0..j-1 and the consumer fills column j from W
      // (so its copies may be issued before q_j is materialised), unless q_j
      // already sits in Q (cycle start / reseed)
      // (ALIAS: no copy is issued before the SpMV barrier, so column j is copied)
      const bool fillj = !from_q && !ALIAS;
      const LgPass P1 = new_pass(fillj ? j : j + 1);
      const LgPass P2 = new_pass(j + 1);
      const LgPass P3 = new_pass(j + 1);
      // ------------------------------------------------------------ SpMV
      if (!from_q) {
        // q_j = w''_{j-1} / beta for the block's rows (read by passes 2, 3)
        for (int i = r0 + tid; i < r1; i += LG_THREADS) a.Q[qidx(i, j, M1)] = Wprev[i] * xs;
        fence_proxy_global();
        if (b == 0 && tid == 0) {
          a.H[j * M1 + (j - 1)] = beta;
          a.H[(j - 1) * M1 + j] = beta;
        }
      }
      if (warp < LG_CONS) {
        // items ib + warp + 15 t; the next descriptor is fetched while the
        // current item is processed
        double* wbuf = stg + warp * LG_SEG;
        const int* __restrict__ rowptr = a.rowptr;
        const int* __restrict__ colp = a.col;
        const double* __restrict__ valp = a.val;
        auto do_item = [&](const int4& w) {
          const int z0 = w.z, z1 = w.w;
          const bool rows = w.x >= 0;
          int rlo[2], rhi[2];
#pragma unroll
          for (int h = 0; h < 2; ++h) {
            const int rr = w.x + lane + 32 * h;
            const bool live = rows && rr < w.y;
            rlo[h] = live ? rowptr[rr] : 0;
            rhi[h] = live ? rowptr[rr + 1] : 0;
          }
          int cc[PER];
          double vv[PER];
#pragma unroll
          for (int u = 0; u < PER; ++u) {
            const int z = z0 + lane + 32 * u;
            cc[u] = z < z1 ? __ldcs(colp + z) : -1;
            vv[u] = z < z1 ? __ldcs(valp + z) : 0.0;
          }
#pragma unroll
          for (int u = 0; u < PER; ++u) {
            if (cc[u] >= 0) {
              const double xv = from_q ? a.Q[qidx(cc[u], j, M1)] : Wprev[cc[u]] * xs;
              vv[u] *= xv;
            }
          }
          if (!rows) {
            // a piece of a split row: fixed-order tree sum
            double t0 = 0.0, t1 = 0.0;
#pragma unroll
            for (int u = 0; u < PER; u += 2) {
              t0 += vv[u];
              t1 += vv[u + 1];
            }
            const double sm = warp_sum(t0 + t1);
            if (lane == 0) a.piece_sum[-w.x - 1] = sm;
          } else {
#pragma unroll
            for (int u = 0; u < PER; ++u)
              if (z0 + lane + 32 * u < z1) wbuf[lane + 32 * u] = vv[u];
            __syncwarp();
            // rows of <= 32 nonzeros: a lane each, in order (as csr_matvec);
            // longer rows: the warp, fixed-order tree
            unsigned longm[2];
#pragma unroll
            for (int h = 0; h < 2; ++h) {
              const int rr = w.x + lane + 32 * h;
              const int len = rhi[h] - rlo[h];
              const bool live = rr < w.y;
              longm[h] = __ballot_sync(0xffffffffu, live && len > LG_SHORT);
              if (live && len <= LG_SHORT) {
                double sm = 0.0;
                for (int z = rlo[h] - z0; z < rhi[h] - z0; ++z) sm += wbuf[z];
                Wcur[rr] = sm;
              }
            }
#pragma unroll
            for (int h = 0; h < 2; ++h) {
              unsigned msk = longm[h];
              while (msk) {
                const int l = __ffs(msk) - 1;
                msk &= msk - 1;
                const int za = __shfl_sync(0xffffffffu, rlo[h], l) - z0;
                const int zb = __shfl_sync(0xffffffffu, rhi[h], l) - z0;
                double sm = 0.0;
                for (int z = za + lane; z < zb; z += 32) sm += wbuf[z];
                sm = warp_sum(sm);
                if (lane == 0) Wcur[w.x + l + 32 * h] = sm;
              }
            }
            __syncwarp();
          }
        };
        // the block's static items, ib + warp + 15 t, the next descriptor
        // fetched while the current item is processed ...
        int it = ib + warp;
        int4 w = it < ie ? a.items[it] : make_int4(0, 0, 0, 0);
        while (it < ie) {
          const int4 wn = (it + LG_CONS < ie) ? a.items[it + LG_CONS] : make_int4(0, 0, 0, 0);
          do_item(w);
          w = wn;
          it += LG_CONS;
        }
        // ... then the shared tail pool (every block's last items), claimed
        // four at a time; the counter alternates with the step's parity
        if (a.tail1 > a.tail0) {
          int* ctr = a.steal + (matvecs & 1);
          for (;;) {
            int base = 0;
            if (lane == 0) base = atomicAdd(ctr, 4);
            base = __shfl_sync(0xffffffffu, base, 0);
            if (a.tail0 + base >= a.tail1) break;
            for (int q = 0; q < 4 && a.tail0 + base + q < a.tail1; ++q) do_item(a.items[a.tail0 + base + q]);
          }
        }
        if (ALIAS) fence_proxy_smem();  // staging writes before the slots' next copies
      }
      LG_MARK(0);
      LG_BW(0);
      grid.sync();  // every w row is final except the split rows (pieces)
      LG_MARK(2);
      LG_BW_START();
      // ------------------------------------------------------------ pass 1
      begin(P1);
      // split rows of this block's range: w = sum of the pieces, fixed order
      for (int x = s0 + tid; x < s1; x += LG_THREADS) {
        const int f = a.gsplit_first[x], c = a.gsplit_cnt[x];
        double wi = 0.0;
        for (int u = 0; u < c; ++u) wi += a.piece_sum[f + u];
        Wcur[a.gsplit_row[x]] = wi;
      }
      __syncthreads();
      ++matvecs;
      if (b == 0 && tid == 0 && a.steal) a.steal[matvecs & 1] = 0;  // the next step's tail counter
      int bad = 0;
      if (cons) {
        double acc0 = 0.0, acc1 = 0.0;
        double wr_n = 0.0, qv_n = 0.0;
        const uint32_t pend = P1.gbase + (uint32_t)nt;
        if (gc < pend) {
          const int row = (tile0 + tile_of(P1, gc)) * 32 + lane;
          wr_n = row < n ? Wcur[row] : 0.0;
          qv_n = (fillj && row < n) ? Wprev[row] * xs : 0.0;
        }
        for (; gc < pend; gc += NCW) {
          const int s = slot_of(gc);
          double* sl = ring + s * LG_SLOT;
          const double wr = wr_n, qv = qv_n;
          if (gc + NCW < pend) {
            const int row = (tile0 + tile_of(P1, gc + NCW)) * 32 + lane;
            wr_n = row < n ? Wcur[row] : 0.0;
            qv_n = (fillj && row < n) ? Wprev[row] * xs : 0.0;
          }
          if (!isfinite(wr)) bad = 1;
          mbar_wait(fullb + s, par_of(gc));
          if (fillj) {
            sl[j * 32 + lane] = qv;
            __syncwarp();
          }
          if (a.lz_opt & 1) {
            double* ws = wsm + warp * 32;
            ws[lane] = wr;
            __syncwarp();
#pragma unroll 8
            for (int rr = 0; rr < 32; rr += 2) {
              const int ra = (rr + lane) & 31, rb = (rr + 1 + lane) & 31;
              acc0 = fma(sl[lane * 32 + ra], ws[ra], acc0);
              acc1 = fma(sl[lane * 32 + rb], ws[rb], acc1);
            }
          } else {
#pragma unroll 8
            for (int rr = 0; rr < 32; rr += 2) {
              const int ra = (rr + lane) & 31, rb = (rr + 1 + lane) & 31;
              acc0 = fma(sl[lane * 32 + ra], __shfl_sync(0xffffffffu, wr, ra), acc0);
              acc1 = fma(sl[lane * 32 + rb], __shfl_sync(0xffffffffu, wr, rb), acc1);
            }
          }
          if (fillj) fence_proxy_smem();
          __syncwarp();
          issue(P1, &P2, gc + (LG_SPW + 1) * NCW);  // refill the slot (next pass's tiles at the end)
        }
        wacc[warp * 32 + lane] = acc0 + acc1;
      }
      bad = __syncthreads_or(bad);
      if (bad && tid == 0) atomicOr(&a.flags[F_NONFINITE], 1);
      if (warp == 0) {
        double sm = 0.0;
        for (int w = 0; w < NCW; ++w) sm += wacc[w * 32 + lane];
        if (lane <= j) a.P1[(int64_t)lane * G + b] = sm;
      }
      LG_MARK(1);
      LG_BW(1);
      grid.sync();
      LG_MARK(2);
      LG_BW_START();
      if (*(volatile int*)&a.flags[F_NONFINITE]) {
        drain();
        if (b == 0 && tid == 0) {
          a.flags[F_EXIT] = EXIT_NONFINITE;
          a.flags[F_MATVECS] = matvecs;
        }
        return;
      }
      // ------------------------------------------------------------ pass 2
      for (int t = warp; t <= j; t += LG_WARPS) {  // c = sum over blocks, fixed order
        double v[8];
#pragma unroll
        for (int u = 0; u < 8; ++u) {
          const int bb = lane + 32 * u;
          v[u] = bb < G ? a.P1[(int64_t)t * G + bb] : 0.0;
        }
        double sm = ((v[0] + v[1]) + (v[2] + v[3])) + ((v[4] + v[5]) + (v[6] + v[7]));
        sm = warp_sum(sm);
        if (lane == 0) cs[t] = sm;
      }
      begin(P2);
      __syncthreads();
      LG_BW(2);
      if (cons) {
        double acc0 = 0.0, acc1 = 0.0;
        const int jj = j + 1;
        const uint32_t pend = P2.gbase + (uint32_t)nt;
        double w_n = 0.0;
        if (gc < pend) {
          const int row = (tile0 + tile_of(P2, gc)) * 32 + lane;
          w_n = row < n ? Wcur[row] : 0.0;
        }
        for (; gc < pend; gc += NCW) {
          const int s = slot_of(gc);
          const double* sl = ring + s * LG_SLOT;
          const int row = (tile0 + tile_of(P2, gc)) * 32 + lane;
          const double w0 = w_n;
          if (gc + NCW < pend) {
            const int rn = (tile0 + tile_of(P2, gc + NCW)) * 32 + lane;
            w_n = rn < n ? Wcur[rn] : 0.0;
          }
          mbar_wait(fullb + s, par_of(gc));
          double p0 = 0.0, p1 = 0.0, p2 = 0.0, p3 = 0.0;
          int t = 0;
          for (; t + 4 <= jj; t += 4) {
            p0 = fma(sl[t * 32 + lane], cs[t], p0);
            p1 = fma(sl[(t + 1) * 32 + lane], cs[t + 1], p1);
            p2 = fma(sl[(t + 2) * 32 + lane], cs[t + 2], p2);
            p3 = fma(sl[(t + 3) * 32 + lane], cs[t + 3], p3);
          }
          for (; t < jj; ++t) p0 = fma(sl[t * 32 + lane], cs[t], p0);
          const double w1 = w0 - ((p0 + p1) + (p2 + p3));
          if (row < n) Wcur[row] = w1;
          if (a.lz_opt & 1) {
            double* ws = wsm + warp * 32;
            ws[lane] = w1;
            __syncwarp();
#pragma unroll 8
            for (int rr = 0; rr < 32; rr += 2) {
              const int ra = (rr + lane) & 31, rb = (rr + 1 + lane) & 31;
              acc0 = fma(sl[lane * 32 + ra], ws[ra], acc0);
              acc1 = fma(sl[lane * 32 + rb], ws[rb], acc1);
            }
          } else {
#pragma unroll 8
            for (int rr = 0; rr < 32; rr += 2) {
              const int ra = (rr + lane) & 31, rb = (rr + 1 + lane) & 31;
              acc0 = fma(sl[lane * 32 + ra], __shfl_sync(0xffffffffu, w1, ra), acc0);
              acc1 = fma(sl[lane * 32 + rb], __shfl_sync(0xffffffffu, w1, rb), acc1);
            }
          }
          __syncwarp();
          issue(P2, &P3, gc + (LG_SPW + 1) * NCW);
        }
        wacc[warp * 32 + lane] = acc0 + acc1;
      }
      __syncthreads();
      if (warp == 0) {
        double sm = 0.0;
        for (int w = 0; w < NCW; ++w) sm += wacc[w * 32 + lane];
        if (lane <= j) a.P2[(int64_t)lane * G + b] = sm;
      }
      LG_MARK(3);
      LG_BW(3);
      grid.sync();
      LG_MARK(2);
      LG_BW_START();
      // ------------------------------------------------------------ pass 3
      const bool more = (j + 1 < m);
      for (int t = warp; t <= j; t += LG_WARPS) {
        double v[8];
#pragma unroll
        for (int u = 0; u < 8; ++u) {
          const int bb = lane + 32 * u;
          v[u] = bb < G ? a.P2[(int64_t)t * G + bb] : 0.0;
        }
        double sm = ((v[0] + v[1]) + (v[2] + v[3])) + ((v[4] + v[5]) + (v[6] + v[7]));
        sm = warp_sum(sm);
        if (lane == 0) c2s[t] = sm;
      }
      begin(P3);
      __syncthreads();
      double ss = 0.0;
      if (cons) {
        // the next step's pass 1 (columns 0..j, final) is issued at the end of
        // this one unless the slots hold the SpMV staging (ALIAS)
        const LgPass N1{pbase, j + 1, pseq & 1};
        const LgPass* np = (more && !ALIAS) ? &N1 : nullptr;
        const int jj = j + 1;
        const uint32_t pend = P3.gbase + (uint32_t)nt;
        double w_n = 0.0;
        if (gc < pend) {
          const int row = (tile0 + tile_of(P3, gc)) * 32 + lane;
          w_n = row < n ? Wcur[row] : 0.0;
        }
        for (; gc < pend; gc += NCW) {
          const int s = slot_of(gc);
          const double* sl = ring + s * LG_SLOT;
          const int row = (tile0 + tile_of(P3, gc)) * 32 + lane;
          const double w0 = w_n;
          if (gc + NCW < pend) {
            const int rn = (tile0 + tile_of(P3, gc + NCW)) * 32 + lane;
            w_n = rn < n ? Wcur[rn] : 0.0;
          }
          mbar_wait(fullb + s, par_of(gc));
          double p0 = 0.0, p1 = 0.0, p2 = 0.0, p3 = 0.0;
          int t = 0;
          for (; t + 4 <= jj; t += 4) {
            p0 = fma(sl[t * 32 + lane], c2s[t], p0);
            p1 = fma(sl[(t + 1) * 32 + lane], c2s[t + 1], p1);
            p2 = fma(sl[(t + 2) * 32 + lane], c2s[t + 2], p2);
            p3 = fma(sl[(t + 3) * 32 + lane], c2s[t + 3], p3);
          }
          for (; t < jj; ++t) p0 = fma(sl[t * 32 + lane], c2s[t], p0);
          __syncwarp();
          issue(P3, np, gc + (LG_SPW + 1) * NCW);
          const double w2 = w0 - ((p0 + p1) + (p2 + p3));
          if (row < n) {
            Wcur[row] = w2;
            ss = fma(w2, w2, ss);
          }
        }
        ss = warp_sum(ss);
        if (lane == 0) wacc[warp * 32] = ss;
      }
      // coefficients c + c' (every block), H column j (block 0), scale
      if (warp == LG_WARPS - 1) {
        const double cc = (lane <= j) ? cs[lane] + c2s[lane] : 0.0;
        if (b == 0 && lane <= j) {
          a.H[lane * M1 + j] = cc;
          a.H[j * M1 + lane] = cc;
        }
        double mx = fabs(cc);
        mx = warp_max(mx);
        if (lane == 0) misc[0] = fmax(1.0, mx);
      }
      __syncthreads();
      if (tid == 0) {
        double sm = 0.0;
        for (int w = 0; w < NCW; ++w) sm += wacc[w * 32];
        a.P3[b] = sm;
      }
      LG_MARK(4);
      LG_BW(4);
      grid.sync();
      LG_MARK(2);
      if (warp == 0) {
        double v[8];
#pragma unroll
        for (int u = 0; u < 8; ++u) v[u] = (lane + 32 * u < G) ? a.P3[lane + 32 * u] : 0.0;
        double sm = ((v[0] + v[1]) + (v[2] + v[3])) + ((v[4] + v[5]) + (v[6] + v[7]));
        sm = warp_sum(sm);
        if (lane == 0) misc[1] = sqrt(sm);
      }
      __syncthreads();
      beta = misc[1];
      const double scale = misc[0];
      wb ^= 1;
      from_q = false;
      if (beta <= 1e-13 * scale) {
        drain();
        if (b == 0 && tid == 0) {
          a.flags[F_EXIT] = EXIT_BREAKDOWN;
          a.flags[F_J] = j;
          a.flags[F_CYCLE] = cycle;
          a.flags[F_ELL] = ell;
          a.flags[F_RESTARTS] = restarts;
          a.flags[F_NHIST] = nhist;
          a.flags[F_MATVECS] = matvecs;
          a.flags[F_PENDING] = wb;
        }
        return;
      }
      pending = (j == m - 1);
    }
    // ---------------------------------------------------------- end of cycle
    if (pending) {
      double* Wprev = wb ? a.W1 : a.W0;
      const double xs = 1.0 / beta;
      for (int i = r0 + tid; i < r1; i += LG_THREADS) a.Q[qidx(i, m, M1)] = Wprev[i] * xs;
      if (b == 0 && tid == 0) {
        a.H[m * M1 + (m - 1)] = beta;
        a.H[(m - 1) * M1 + m] = beta;
      }
      pending = false;
    }
    grid.sync();
    LG_MARK(7);
    // Rayleigh-Ritz (every block, identical)
    const int ell_next = max(1, min(a.k_c + 3, m - 2));
    const int nwant = min(m, max(ell_next, a.k_c));
    TriSmem ts;
    ts.A = stg;
    ts.Q = stg + 1024;
    ts.Z = stg + 2048;
    ts.v = stg + 3072;
    ts.p = ts.v + 64;
    ts.dd = ts.p + 64;
    ts.ee = ts.dd + 64;
    ts.lam = ts.ee + 64;
    ts.red = ts.lam + 64;
    ts.iw = (int*)(ts.red + 64);
    double* thetaS = ysr;
    double* Ys = thetaS + 64;
    rr_arrow(m, ell, nwant, a.H, M1, ts, thetaS, Ys, m, (a.prof && b == 0) ? a.prof + 8 : nullptr);
    if (ALIAS) fence_proxy_smem();
    LG_MARK(5);
    const double beta_last = a.H[m * M1 + (m - 1)];
    if (tid == 0) {
      bool ok = true;
      const double tol_eff = a.tol * (1.0 + fabs(thetaS[0]));
      for (int u = 0; u < a.k_c; ++u) {
        const double r = fabs(beta_last * Ys[(m - 1) * m + u]);
        if (!(r <= tol_eff)) ok = false;
      }
      misc[2] = ok ? 1.0 : 0.0;
    }
    __syncthreads();
    if (b == 0) {
      for (int u = tid; u < nwant; u += LG_THREADS) {
        a.theta[u] = thetaS[u];
        a.res[u] = fabs(beta_last * Ys[(m - 1) * m + u]);
      }
      if (tid == 0) a.hist[nhist] = thetaS[0];
    }
    ++nhist;
    if (misc[2] != 0.0) {
      converged = 1;
      break;
    }
    if (cycle == a.max_restarts) break;
    ell = ell_next;
    rot_pass(Ys, ell, true);
    ++restarts;
    jstart = ell;
    from_q = true;
    grid.sync();
    if (b == 0) {
      for (int x = tid; x < M1 * M1; x += LG_THREADS) a.H[x] = 0.0;
      __syncthreads();
      for (int u = tid; u < ell; u += LG_THREADS) a.H[u * M1 + u] = thetaS[u];
      __syncthreads();
    }
    LG_MARK(6);
  }
  // ---------------------------------------------------------------- output
  if (a.prof && b == 0 && tid == 0)
    for (int s = 0; s < 8; ++s) a.prof[s] += lz_acc[s];
  if (a.prof && tid == 0)
    for (int s = 0; s < 5; ++s) a.prof[32 + 5 * b + s] += bw_acc[s];
  rot_pass(ysr + 64, a.k_c, false);
  if (b == 0 && tid == 0) {
    a.flags[F_EXIT] = EXIT_DONE;
    a.flags[F_CONV] = converged;
    a.flags[F_RESTARTS] = restarts;
    a.flags[F_NHIST] = nhist;
    a.flags[F_MATVECS] = matvecs;
  }
}

static size_t lz_tma_smem(int ncw, int seg, bool alias, int spw) {
  const int ring = ncw * spw, stg = std::max(LG_CONS * seg, LG_RRS);
  const int scr = alias ? LG_YS : stg + LG_YS;
  return (size_t)(ring * LG_SLOT + scr + 32 + 32 + 2 * LG_WARPS * 32 + 8) * sizeof(double) + ring * sizeof(uint64_t);
}

struct LgVariant {
  int ncw, seg;
  bool alias;
  int spw;
};
static LgVariant lz_tma_variant() {
  static const LgVariant v[] = {{16, 512, true, 1}, {15, 512, true, 1}, {12, 512, true, 1}, {8, 512, true, 2},
                                {10, 512, true, 1}};
  int i = 0;
  if (const char* e = getenv("USBS_LZG_VARIANT")) i = std::max(0, std::min(4, atoi(e)));
  return v[i];
}

// ------------------------------------------------------------------ plan
// Basis passes: every block owns the same number of 32-row tiles.  SpMV:
// work items over the whole matrix in row order -- short rows (<= 32
// nonzeros) packed into segments of <= 256 nonzeros and <= 64 rows, rows of
// 33..256 nonzeros one item each, longer rows cut into 256-nonzero pieces
// whose partial sums the rows' owners add up after the barrier -- cut into G
// contiguous ranges of equal estimated cost (nonzeros + per-row and per-item
// overheads).  Within a block the 15 SpMV warps pull items dynamically.
void lz_tma_plan(usbs_ctx* ctx, usbs_problem* p) {
  const int LG_SEG = lz_tma_variant().seg;
  if (p->lzg_ready == LG_SEG) return;
  const int64_t n = p->n;
  const std::vector<int32_t>& rp = p->h_rowptr;
  if ((int64_t)rp.size() != n + 1) fail(USBS_ERR_CONFIG, "lanczos plan: host row pointers missing");
  const int64_t ntile = (n + 31) / 32;
  int G = (int)std::min<int64_t>(std::max(1, ctx->num_sms - 4), ntile);
  if (const char* e = getenv("USBS_LZG_BLOCKS")) G = std::max(1, std::min<int>(ctx->num_sms, atoi(e)));
  G = (int)std::min<int64_t>(G, ntile);
  double row_cost = 1.0, item_cost = 16.0, long_cost = 64.0;  // fitted to per-block timers (profiles/lz_spmv_fit.py)
  if (const char* e = getenv("USBS_LZG_ROWCOST")) row_cost = atof(e);
  if (const char* e = getenv("USBS_LZG_ITEMCOST")) item_cost = atof(e);
  if (const char* e = getenv("USBS_LZG_LONGCOST")) long_cost = atof(e);
  auto rnnz = [&](int64_t i) -> int64_t { return rp[i + 1] - rp[i]; };
  std::vector<int32_t> blk_row(G + 1);
  for (int bb = 0; bb <= G; ++bb) blk_row[bb] = (int32_t)std::min<int64_t>(n, (ntile * bb / G) * 32);
  blk_row[G] = (int32_t)n;
  std::vector<int4> items;
  std::vector<double> cost;
  std::vector<int32_t> srow, sfirst, scnt;
  int npieces = 0;
  for (int64_t i = 0; i < n;) {
    const int64_t z = rnnz(i);
    if (z > LG_SEG) {
      srow.push_back((int32_t)i);
      sfirst.push_back(npieces);
      int c = 0;
      for (int32_t q = rp[i]; q < rp[i + 1]; q += LG_SEG, ++c) {
        const int32_t q1 = std::min<int32_t>(rp[i + 1], q + LG_SEG);
        items.push_back(make_int4(-1 - npieces++, 0, q, q1));
        cost.push_back((double)(q1 - q) + item_cost);
      }
      scnt.push_back(c);
      ++i;
    } else {
      const int64_t a0 = i;
      int nlong = 0;
      while (i < n && i - a0 < LG_SEGROWS && rnnz(i) <= LG_SEG && rp[i + 1] - rp[a0] <= LG_SEG) {
        nlong += rnnz(i) > LG_SHORT;
        ++i;
      }
      items.push_back(make_int4((int)a0, (int)i, rp[a0], rp[i]));
      cost.push_back((double)(rp[i] - rp[a0]) + row_cost * (double)(i - a0) + long_cost * nlong + item_cost);
    }
  }
  std::vector<int32_t> blk_item(G + 1, (int32_t)items.size());
  blk_item[0] = 0;
  {
    double total = 0.0;
    for (double c : cost) total += c;
    double acc = 0.0;
    int bb = 0;
    for (size_t t = 0; t < items.size() && bb + 1 < G; ++t) {
      acc += cost[t];
      if (acc >= total * (bb + 1) / G) blk_item[++bb] = (int32_t)(t + 1);
    }
    for (int x = bb + 1; x <= G; ++x) blk_item[x] = (int32_t)items.size();
  }
  // the last `tail` share of every block's items (by cost) goes to a pool the
  // blocks drain dynamically after their static items (levels the SpMV
  // phase; the items' results do not depend on who computes them)
  double tail = 0.0;  // measured: a 12-25% pool levels the SpMV (max 59 -> 56 us) but slows the call (profiles/lz_opts.py)
  if (const char* e = getenv("USBS_LZG_TAIL")) tail = std::max(0.0, std::min(0.9, atof(e)));
  {
    std::vector<int4> stat, pool;
    std::vector<int32_t> nbi(G + 1, 0);
    for (int bb = 0; bb < G; ++bb) {
      double tot = 0.0;
      for (int t = blk_item[bb]; t < blk_item[bb + 1]; ++t) tot += cost[t];
      double acc = 0.0;
      for (int t = blk_item[bb]; t < blk_item[bb + 1]; ++t) {
        acc += cost[t];
        if (acc <= (1.0 - tail) * tot || t == blk_item[bb]) stat.push_back(items[t]);
        else pool.push_back(items[t]);
      }
      nbi[bb + 1] = (int32_t)stat.size();
    }
    p->lzg_tail0 = (int)stat.size();
    stat.insert(stat.end(), pool.begin(), pool.end());
    p->lzg_tail1 = (int)stat.size();
    items.swap(stat);
    blk_item.swap(nbi);
  }
  std::vector<int32_t> blk_split(G + 1, 0);
  for (int bb = 0; bb <= G; ++bb)
    blk_split[bb] = (int32_t)(std::lower_bound(srow.begin(), srow.end(), blk_row[bb]) - srow.begin());
  p->lzg_G = G;
  p->lzg_npieces = npieces;
  p->lzg_nsplit = (int)srow.size();
  p->lzg_blk_row = dev_upload(p, blk_row.data(), blk_row.size());
  p->lzg_blk_item = dev_upload(p, blk_item.data(), blk_item.size());
  p->lzg_items = dev_upload(p, items.data(), items.size());
  p->lzg_split_row = dev_upload(p, srow.data(), srow.size());
  p->lzg_split_first = dev_upload(p, sfirst.data(), sfirst.size());
  p->lzg_split_cnt = dev_upload(p, scnt.data(), scnt.size());
  p->lzg_blk_split = dev_upload(p, blk_split.data(), blk_split.size());
  p->lzg_ready = LG_SEG;
}

template <int NCW, int SEG, bool ALIAS, int SPW>
static void lz_tma_launch_t(usbs_ctx* ctx, usbs_problem* p, LzArgs& a) {
  auto fn = k_lanczos_tma<NCW, SEG, ALIAS, SPW>;
  const size_t smem = lz_tma_smem(NCW, SEG, ALIAS, SPW);
  smem_optin(ctx, (const void*)fn, (int)smem);
  int per_sm = 0;
  USBS_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, fn, LG_THREADS, smem));
  const int G = p->lzg_G;
  if (per_sm * ctx->num_sms < G) fail(USBS_ERR_CUDA, "lanczos grid exceeds co-resident capacity");
  void* args[] = {&a};
  USBS_CUDA(cudaLaunchCooperativeKernel((const void*)fn, dim3(G), dim3(LG_THREADS), args, smem, ctx->stream));
  check_launch(ctx);
}

void lz_tma_launch(usbs_ctx* ctx, usbs_problem* p, LzArgs& a) {
  a.blk_row = p->lzg_blk_row;
  a.items = p->lzg_items;
  a.blk_item = p->lzg_blk_item;
  a.nsplit = p->lzg_nsplit;
  a.gsplit_row = p->lzg_split_row;
  a.gsplit_first = p->lzg_split_first;
  a.gsplit_cnt = p->lzg_split_cnt;
  a.blk_gsplit = p->lzg_blk_split;
  a.tail0 = p->lzg_tail0;
  a.tail1 = p->lzg_tail1;
  a.steal = (int*)ctx->ws.get(WS_LZ_FLAGS + 100, 2 * sizeof(int));
  USBS_CUDA(cudaMemsetAsync(a.steal, 0, 2 * sizeof(int), ctx->stream));
  a.lz_opt = 1;  // column sums from shared memory (1% faster than shuffles at C4)
  if (const char* e = getenv("USBS_LZG_OPT")) a.lz_opt = atoi(e);
  const LgVariant v = lz_tma_variant();
  if (v.ncw == 8) lz_tma_launch_t<8, 512, true, 2>(ctx, p, a);
  else if (v.ncw == 15) lz_tma_launch_t<15, 512, true, 1>(ctx, p, a);
  else if (v.ncw == 12) lz_tma_launch_t<12, 512, true, 1>(ctx, p, a);
  else if (v.ncw == 16) lz_tma_launch_t<16, 512, true, 1>(ctx, p, a);
  else lz_tma_launch_t<10, 512, true, 1>(ctx, p, a);
}

}  // namespace usbs
