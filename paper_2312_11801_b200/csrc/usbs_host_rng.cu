// Host-side sketch test matrix: make_test_matrix (sketch.py:25-27) is
// np.random.RandomState(seed & 0x7FFFFFFF).standard_normal((n, r)), i.e.
// numpy's legacy MT19937 stream (init_genrand seeding) through the legacy
// polar Gaussian (two 53-bit doubles per pair, rejection outside the unit
// disc, the second variate cached for the next call), filled in C order.
// Restated here so the fill runs in native code outside the Python GIL (the
// solver generates it on a worker thread while the problem is planned and
// uploaded); bit-identical to numpy (tests/test_abi.py) -- the same
// generator recurrence, the same double construction and the same libm
// log/sqrt.
#include <algorithm>
#include <atomic>
#include <cmath>
#include <cstdint>
#include <cstdlib>
#include <cstring>
#include <thread>
#include <vector>

#include "usbs_common.cuh"

namespace {

struct Mt19937 {
  static constexpr int N = 624, M = 397;
  uint32_t key[N];
  uint32_t outv[N];  // the block's tempered outputs (tempered in one vectorisable sweep per reload)
  int pos = N;

  explicit Mt19937(uint32_t seed) {
    for (int i = 0; i < N; ++i) {
      key[i] = seed;
      seed = 1812433253u * (seed ^ (seed >> 30)) + (uint32_t)(i + 1);
    }
  }
  void reload() {
    constexpr uint32_t UPPER = 0x80000000u, LOWER = 0x7fffffffu, MATRIX_A = 0x9908b0dfu;
    int i = 0;
    for (; i < N - M; ++i) {
      const uint32_t y = (key[i] & UPPER) | (key[i + 1] & LOWER);
      key[i] = key[i + M] ^ (y >> 1) ^ (-(y & 1u) & MATRIX_A);
    }
    for (; i < N - 1; ++i) {
      const uint32_t y = (key[i] & UPPER) | (key[i + 1] & LOWER);
      key[i] = key[i + (M - N)] ^ (y >> 1) ^ (-(y & 1u) & MATRIX_A);
    }
    const uint32_t y = (key[N - 1] & UPPER) | (key[0] & LOWER);
    key[N - 1] = key[M - 1] ^ (y >> 1) ^ (-(y & 1u) & MATRIX_A);
    for (int j = 0; j < N; ++j) {
      uint32_t t = key[j];
      t ^= (t >> 11);
      t ^= (t << 7) & 0x9d2c5680u;
      t ^= (t << 15) & 0xefc60000u;
      t ^= (t >> 18);
      outv[j] = t;
    }
    pos = 0;
  }
  uint32_t next32() {
    if (pos == N) reload();
    return outv[pos++];
  }
  double next_double() {  // 53-bit: (a >> 5) * 2^26 + (b >> 6), over 2^53
    const int32_t a = (int32_t)(next32() >> 5), b = (int32_t)(next32() >> 6);
    return (a * 67108864.0 + b) / 9007199254740992.0;
  }
};

}  // namespace

using namespace usbs;

// out[0 .. (row1 - row0) * r) = rows [row0, row1) of the n x r matrix
// RandomState(seed & 0x7FFFFFFF).standard_normal((n, r)) (the stream is
// generated from its start; rows before row0 are drawn and discarded).
//
// Two stages, pipelined by chunks of pairs: the calling thread runs the
// generator and the rejection loop (inherently sequential: the number of
// draws per accepted pair depends on the draws) and stores the accepted
// (x2, x1) in place; worker threads follow behind and turn each stored pair
// into the two variates, f = sqrt(-2 log(r2) / r2) with r2 recomputed from
// the stored doubles by the same expression -- the same operations on the
// same values as the one-pass loop, so the output is bit-identical, with the
// log / sqrt / divide (two thirds of the time) spread over the cores.
namespace {

inline double disc_r2(double x1, double x2) { return x1 * x1 + x2 * x2; }

inline void finish_pair(double* o2, double* o1) {  // o2 holds x2, o1 holds x1
  const double x2 = *o2, x1 = *o1;
  const double r2 = disc_r2(x1, x2);
  const double f = std::sqrt(-2.0 * std::log(r2) / r2);
  *o1 = f * x1;
  *o2 = f * x2;
}

}  // namespace

extern "C" usbs_status usbs_make_test_matrix(int64_t seed, int64_t n, int r, int64_t row0, int64_t row1,
                                             double* out) {
  USBS_API_BEGIN
  if (n < 0 || r < 0 || row0 < 0 || row1 < row0 || row1 > n) fail(USBS_ERR_SHAPE, "make_test_matrix: bad rows");
  Mt19937 mt((uint32_t)((uint64_t)seed & 0x7FFFFFFFull));
  const int64_t lo = row0 * r, hi = row1 * r;  // elements [lo, hi) of the stream are kept
  const int64_t npairs = (hi + 1) / 2;         // pair i gives elements 2i (f x2) and 2i + 1 (f x1)
  // pairs [p0, p1) lie wholly inside [lo, hi): stored raw and finished by the workers
  const int64_t p0 = (lo + 1) / 2, p1 = hi / 2;
  constexpr int64_t CHUNK = 1 << 15;
  std::atomic<int64_t> ready{p0};   // pairs below this are stored
  std::atomic<int64_t> next{p0};    // next chunk start to claim
  int nthreads = 0;
  if (p1 - p0 >= 4 * CHUNK) {
    const unsigned hw = std::thread::hardware_concurrency();
    nthreads = (int)std::min<unsigned>(8u, hw > 2 ? hw - 2 : 1u);
    if (const char* e = getenv("USBS_PSI_THREADS")) nthreads = std::max(0, std::min(64, atoi(e)));
  }
  auto worker = [&]() {
    for (;;) {
      const int64_t c0 = next.fetch_add(CHUNK, std::memory_order_relaxed);
      if (c0 >= p1) break;
      const int64_t c1 = std::min(p1, c0 + CHUNK);
      while (ready.load(std::memory_order_acquire) < c1) std::this_thread::yield();
      for (int64_t i = c0; i < c1; ++i) finish_pair(out + (2 * i - lo), out + (2 * i + 1 - lo));
    }
  };
  std::vector<std::thread> pool;
  for (int t = 0; t < nthreads; ++t) pool.emplace_back(worker);
  for (int64_t i = 0; i < npairs; ++i) {
    double x1, x2, r2;
    do {
      x1 = 2.0 * mt.next_double() - 1.0;
      x2 = 2.0 * mt.next_double() - 1.0;
      r2 = disc_r2(x1, x2);
    } while (r2 >= 1.0 || r2 == 0.0);
    if (i >= p0 && i < p1) {
      out[2 * i - lo] = x2;
      out[2 * i + 1 - lo] = x1;
      if (((i + 1 - p0) & (CHUNK - 1)) == 0) ready.store(i + 1, std::memory_order_release);
    } else if (2 * i + 1 >= lo) {
      // a pair cut by lo or hi: finished here
      const double f = std::sqrt(-2.0 * std::log(r2) / r2);
      if (2 * i >= lo && 2 * i < hi) out[2 * i - lo] = f * x2;
      if (2 * i + 1 >= lo && 2 * i + 1 < hi) out[2 * i + 1 - lo] = f * x1;
    }
  }
  ready.store(p1, std::memory_order_release);
  if (nthreads == 0) worker();
  for (auto& th : pool) th.join();
  USBS_API_END
}
