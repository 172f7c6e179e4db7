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
#include <cmath>
#include <cstdint>
#include <cstring>

#include "usbs_common.cuh"

namespace {

struct Mt19937 {
  static constexpr int N = 624, M = 397;
  uint32_t key[N];
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
    pos = 0;
  }
  uint32_t next32() {
    if (pos == N) reload();
    uint32_t y = key[pos++];
    y ^= (y >> 11);
    y ^= (y << 7) & 0x9d2c5680u;
    y ^= (y << 15) & 0xefc60000u;
    y ^= (y >> 18);
    return y;
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
extern "C" usbs_status usbs_make_test_matrix(int64_t seed, int64_t n, int r, int64_t row0, int64_t row1,
                                             double* out) {
  USBS_API_BEGIN
  if (n < 0 || r < 0 || row0 < 0 || row1 < row0 || row1 > n) fail(USBS_ERR_SHAPE, "make_test_matrix: bad rows");
  Mt19937 mt((uint32_t)((uint64_t)seed & 0x7FFFFFFFull));
  bool has = false;
  double cached = 0.0;
  const int64_t lo = row0 * r, hi = row1 * r;
  for (int64_t e = 0; e < hi; ++e) {
    double v;
    if (has) {
      v = cached;
      has = false;
    } else {
      double x1, x2, r2;
      do {
        x1 = 2.0 * mt.next_double() - 1.0;
        x2 = 2.0 * mt.next_double() - 1.0;
        r2 = x1 * x1 + x2 * x2;
      } while (r2 >= 1.0 || r2 == 0.0);
      const double f = std::sqrt(-2.0 * std::log(r2) / r2);
      cached = f * x1;
      has = true;
      v = f * x2;
    }
    if (e >= lo) out[e - lo] = v;
  }
  USBS_API_END
}
