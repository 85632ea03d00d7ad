// Table-driven double-precision exp for the sweep's log densities.
//
// exp(x) = 2^(k/32) * (1 + p(r)),  k = rint(32 x / ln2),  r = x - k ln2/32,
// |r| <= ln2/64, p = degree-6 Taylor polynomial of e^r - 1 (truncation
// 3e-18), 2^(j/32) from a 32-entry shared-memory table, exponent scaling by
// an integer add.  Max error 1 ulp against glibc exp over [-707, 700]
// (scripts/fast_exp_check.c restates it with libm fma and checks 2e7
// arguments); arguments outside that range take libdevice exp.
//
// Why not libdevice: its degree-11 polynomial materialises every 64-bit
// coefficient with two UMOVs, ~40 issue slots per call, and exp is the
// sweep's inner operation (~255 calls per gene-iteration).  The value only
// decides slice comparisons (SURVEY.md §7 hard part 1), as glibc's and
// libdevice's last-bit differences already do.
#pragma once

namespace cmc {

__constant__ double kExpC[8] = {
    46.166241308446828,       // 32 / ln2
    6755399441055744.0,       // 1.5 * 2^52 (round-to-integer shifter)
    0.021660834550857544,     // ln2/32, high part (32 trailing zero bits)
    1.4841640746974334e-08,   // ln2/32, low part
    1.0 / 720.0, 1.0 / 120.0, 1.0 / 24.0, 1.0 / 6.0};

// 2^(j/32) computed once per process by fastmath_setup_kernel (global)
// and copied into each block's shared table at kernel start (one coalesced
// load per thread instead of an exp2 per entry).
__device__ double g_exp_table[32];

__global__ void fastmath_setup_kernel() {
  if (threadIdx.x < 32) g_exp_table[threadIdx.x] = exp2((double)threadIdx.x / 32.0);
}

// Fill a block-shared table (call with all threads, then __syncthreads()).
__device__ __forceinline__ void exp_table_init(double* tab) {
  if (threadIdx.x < 32) tab[threadIdx.x] = g_exp_table[threadIdx.x];
}

// The block's table by its 32-bit shared-window address, converted once per
// thread: loads are then a plain ld.shared (no generic-to-shared
// conversion per call inside the slice loops).
struct ExpTab {
  unsigned s;
  ExpTab() = default;
  __device__ __forceinline__ explicit ExpTab(const double* tab)
      : s((unsigned)__cvta_generic_to_shared(tab)) {}
  __device__ __forceinline__ double operator[](int j) const {
    double v;
    asm volatile("ld.shared.f64 %0, [%1];" : "=d"(v) : "r"(s + ((unsigned)j << 3)));
    return v;
  }
};

__device__ __forceinline__ double fast_exp_le700(double x, const ExpTab tab) {
  if (x < -707.0) return exp(x);
  const double t = fma(x, kExpC[0], kExpC[1]);
  const int k = __double2loint(t);
  const double kd = t - kExpC[1];
  double r = fma(kd, -kExpC[2], x);
  r = fma(kd, -kExpC[3], r);
  double s = fma(r, kExpC[4], kExpC[5]);
  s = fma(s, r, kExpC[6]);
  s = fma(s, r, kExpC[7]);
  s = fma(s, r, 0.5);
  const double p = fma(s, r * r, r);
  const double tj = tab[k & 31];
  const double res = fma(tj, p, tj);
  return __hiloint2double(__double2hiint(res) + ((k >> 5) << 20), __double2loint(res));
}

// the table path's range [-707, 700] as one predicate: one branch per call
// (1% of the sweep against two tests, A/B on B200)
__device__ __forceinline__ double fast_exp(double x, const ExpTab tab) {
  if (!((x >= -707.0) & (x <= 700.0))) return exp(x);
  const double t = fma(x, kExpC[0], kExpC[1]);
  const int k = __double2loint(t);
  const double kd = t - kExpC[1];
  double r = fma(kd, -kExpC[2], x);
  r = fma(kd, -kExpC[3], r);
  double s = fma(r, kExpC[4], kExpC[5]);
  s = fma(s, r, kExpC[6]);
  s = fma(s, r, kExpC[7]);
  s = fma(s, r, 0.5);
  const double p = fma(s, r * r, r);
  const double tj = tab[k & 31];
  const double res = fma(tj, p, tj);
  return __hiloint2double(__double2hiint(res) + ((k >> 5) << 20), __double2loint(res));
}

}  // namespace cmc
