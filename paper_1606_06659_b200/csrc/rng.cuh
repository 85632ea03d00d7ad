// Counter-based Philox4x64-10 substreams and the scalar distributions the
// sweep draws from, usable on host (setup: initial states, saved genes,
// synthetic data) and device (the sweep kernels).
//
// The stream is the reference's, bit for bit, so the device consumes the
// same uniforms as the CPU reference without any injection plumbing:
//   key = (seed, chain), counter = (iteration, site, block, 0)
//   P:include/countmc/rng.hpp:19-62, P:src/rng.cpp:10-83.
// Everything here is compiled with -fmad=false so every a*b+c rounds twice,
// as the reference's non-FMA x86-64 build does (P:CMakeLists.txt:7-9).
#pragma once

#include <stdint.h>

#ifdef __CUDACC__
#define CMC_HD __host__ __device__ __forceinline__
#else
#define CMC_HD inline
#endif

#ifndef __CUDA_ARCH__
#include <cmath>
#endif

namespace cmc {

// Draw-site families, P:include/countmc/engine.hpp:42-49.
enum : uint64_t {
  kSiteEps = 1,
  kSiteGamma = 2,
  kSiteNu = 3,
  kSiteTau = 4,
  kSiteBeta = 5,
  kSiteTheta = 6,
  kSiteSigma = 7,
  kSiteSaveSel = 8,
  kSiteSim = 9,
  kSiteXi = 11,  // extension: xi priors (10 is the reference's resample)
};
CMC_HD uint64_t site_id(uint64_t family, uint64_t flat) {
  return (family << 56) | flat;
}

CMC_HD void mulhilo64(uint64_t a, uint64_t b, uint64_t& hi, uint64_t& lo) {
#ifdef __CUDA_ARCH__
  lo = a * b;
  hi = __umul64hi(a, b);
#else
  const unsigned __int128 p = (unsigned __int128)a * (unsigned __int128)b;
  hi = (uint64_t)(p >> 64);
  lo = (uint64_t)p;
#endif
}

// One Philox4x64-10 block.  Round: (hi0,lo0) = M0*c0, (hi1,lo1) = M1*c2,
// c <- {hi1^c1^k0, lo1, hi0^c3^k1, lo0}; key bumped by the Weyl constants
// before rounds 1..9.
CMC_HD void philox4x64_10(uint64_t c0, uint64_t c1, uint64_t c2, uint64_t c3,
                          uint64_t k0, uint64_t k1, uint64_t out[4]) {
#pragma unroll
  for (int r = 0; r < 10; ++r) {
    if (r > 0) {
      k0 += 0x9E3779B97F4A7C15ull;
      k1 += 0xBB67AE8584CAA73Bull;
    }
    uint64_t hi0, lo0, hi1, lo1;
    mulhilo64(0xD2E7470EE14C6C93ull, c0, hi0, lo0);
    mulhilo64(0xCA5A826395121157ull, c2, hi1, lo1);
    const uint64_t n0 = hi1 ^ c1 ^ k0;
    const uint64_t n2 = hi0 ^ c3 ^ k1;
    c0 = n0;
    c1 = lo1;
    c2 = n2;
    c3 = lo0;
  }
  out[0] = c0;
  out[1] = c1;
  out[2] = c2;
  out[3] = c3;
}

// Two Philox blocks with interleaved rounds (independent chains: ILP 2).
CMC_HD void philox4x64_10_x2(uint64_t c0, uint64_t c1, uint64_t blk, uint64_t k0,
                             uint64_t k1, uint64_t a[4], uint64_t b[4]) {
  uint64_t x0 = c0, x1 = c1, x2 = blk, x3 = 0;
  uint64_t y0 = c0, y1 = c1, y2 = blk + 1, y3 = 0;
#pragma unroll
  for (int r = 0; r < 10; ++r) {
    if (r > 0) {
      k0 += 0x9E3779B97F4A7C15ull;
      k1 += 0xBB67AE8584CAA73Bull;
    }
    uint64_t hx0, lx0, hx1, lx1, hy0, ly0, hy1, ly1;
    mulhilo64(0xD2E7470EE14C6C93ull, x0, hx0, lx0);
    mulhilo64(0xD2E7470EE14C6C93ull, y0, hy0, ly0);
    mulhilo64(0xCA5A826395121157ull, x2, hx1, lx1);
    mulhilo64(0xCA5A826395121157ull, y2, hy1, ly1);
    const uint64_t nx0 = hx1 ^ x1 ^ k0, nx2 = hx0 ^ x3 ^ k1;
    const uint64_t ny0 = hy1 ^ y1 ^ k0, ny2 = hy0 ^ y3 ^ k1;
    x0 = nx0; x1 = lx1; x2 = nx2; x3 = lx0;
    y0 = ny0; y1 = ly1; y2 = ny2; y3 = ly0;
  }
  a[0] = x0; a[1] = x1; a[2] = x2; a[3] = x3;
  b[0] = y0; b[1] = y1; b[2] = y2; b[3] = y3;
}

// One substream.  Outputs are consumed in order through a register queue
// (a0..a3, then the pre-generated next block b0..b3); nothing is indexed
// dynamically, so nothing lives in local memory.  init_x2() generates
// blocks 0 and 1 up front: a slice step always needs block 0 and usually
// block 1, and generating both while the warp is converged keeps the
// 64-bit multiply chains out of the divergent shrink loop.
struct Stream {
  uint64_t k0, k1, it, site;
  uint64_t a0, a1, a2, a3, b0, b1, b2, b3;
  uint32_t block;  // next block index (counter word 2) to generate
  uint32_t na, nb; // outputs left in queue a / block b valid (4 or 0)

  CMC_HD void init(uint64_t seed, uint64_t chain, uint64_t iteration,
                   uint64_t site_) {
    k0 = seed;
    k1 = chain;
    it = iteration;
    site = site_;
    block = 0;
    na = 0;
    nb = 0;
  }
  CMC_HD void init_x2(uint64_t seed, uint64_t chain, uint64_t iteration,
                      uint64_t site_) {
    init(seed, chain, iteration, site_);
    uint64_t a[4], b[4];
    philox4x64_10_x2(it, site, 0, k0, k1, a, b);
    a0 = a[0]; a1 = a[1]; a2 = a[2]; a3 = a[3];
    b0 = b[0]; b1 = b[1]; b2 = b[2]; b3 = b[3];
    block = 2;
    na = 4;
    nb = 4;
  }
  CMC_HD void refill() {
    if (nb) {
      a0 = b0; a1 = b1; a2 = b2; a3 = b3;
      nb = 0;
    } else {
      uint64_t o[4];
      philox4x64_10(it, site, block, 0, k0, k1, o);
      a0 = o[0]; a1 = o[1]; a2 = o[2]; a3 = o[3];
      ++block;
    }
    na = 4;
  }
  CMC_HD uint64_t next() {
    if (na == 0) refill();
    const uint64_t x = a0;
    a0 = a1;
    a1 = a2;
    a2 = a3;
    --na;
    return x;
  }
  // ((x >> 11) + 0.5) * 2^-53, P:include/countmc/rng.hpp:38-40.
  CMC_HD double u01() {
    return ((double)(next() >> 11) + 0.5) * 0x1.0p-53;
  }
  // Rejection below 2^64 mod n, P:src/rng.cpp:76-83.
  CMC_HD uint64_t uniform_int(uint64_t n) {
    const uint64_t reject_below = (0ull - n) % n;
    for (;;) {
      const uint64_t x = next();
      if (x >= reject_below) return x % n;
    }
  }
  // The same draw with 2^64 mod n and floor(2^64 / n) precomputed (n >= 2):
  // q = mulhi(x, inv) is floor(x/n) or one less, fixed by one compare.
  CMC_HD uint64_t uniform_int_pre(uint64_t n, uint64_t reject_below,
                                  uint64_t inv) {
    for (;;) {
      const uint64_t x = next();
      if (x >= reject_below) {
        uint64_t hi, lo;
        mulhilo64(x, inv, hi, lo);
        uint64_t r = x - hi * n;
        if (r >= n) r -= n;
        return r;
      }
    }
  }
};

#ifdef __CUDACC__
// Stream with the pre-generated second block kept in shared memory instead
// of registers (4 words per thread at a 32-bit shared-window address, word
// i at bs + i * stride so a warp's accesses are conflict-free): the same
// outputs in the same order, 8 fewer live registers.
struct StreamSm {
  uint64_t k0, k1, it, site;
  uint64_t a0, a1, a2, a3;
  unsigned bs, stride;  // shared-window address of word 0, bytes between words
  uint32_t block;   // next block index (counter word 2) to generate
  uint32_t na, nb;  // outputs left in queue a / block b valid (4 or 0)

  __device__ __forceinline__ void st(int i, uint64_t v) {
    asm volatile("st.shared.u64 [%0], %1;" ::"r"(bs + stride * i), "l"(v));
  }
  __device__ __forceinline__ uint64_t ld(int i) {
    uint64_t v;
    asm volatile("ld.shared.u64 %0, [%1];" : "=l"(v) : "r"(bs + stride * i));
    return v;
  }
  __device__ __forceinline__ void init(uint64_t seed, uint64_t chain, uint64_t iteration,
                                       uint64_t site_, unsigned b_smem, unsigned b_stride) {
    k0 = seed;
    k1 = chain;
    it = iteration;
    site = site_;
    bs = b_smem;
    stride = b_stride;
    block = 0;
    na = 0;
    nb = 0;
  }
  __device__ __forceinline__ void init_x2(uint64_t seed, uint64_t chain, uint64_t iteration,
                                          uint64_t site_, unsigned b_smem, unsigned b_stride) {
    init(seed, chain, iteration, site_, b_smem, b_stride);
    uint64_t a[4], b[4];
    philox4x64_10_x2(it, site, 0, k0, k1, a, b);
    a0 = a[0]; a1 = a[1]; a2 = a[2]; a3 = a[3];
    st(0, b[0]); st(1, b[1]); st(2, b[2]); st(3, b[3]);
    block = 2;
    na = 4;
    nb = 4;
  }
  __device__ __forceinline__ void refill() {
    if (nb) {
      a0 = ld(0); a1 = ld(1); a2 = ld(2); a3 = ld(3);
      nb = 0;
    } else {
      uint64_t o[4];
      philox4x64_10(it, site, block, 0, k0, k1, o);
      a0 = o[0]; a1 = o[1]; a2 = o[2]; a3 = o[3];
      ++block;
    }
    na = 4;
  }
  __device__ __forceinline__ uint64_t next() {
    if (na == 0) refill();
    const uint64_t x = a0;
    a0 = a1;
    a1 = a2;
    a2 = a3;
    --na;
    return x;
  }
  __device__ __forceinline__ double u01() {
    return ((double)(next() >> 11) + 0.5) * 0x1.0p-53;
  }
  __device__ __forceinline__ uint64_t uniform_int_pre(uint64_t n, uint64_t reject_below,
                                                      uint64_t inv) {
    for (;;) {
      const uint64_t x = next();
      if (x >= reject_below) {
        uint64_t hi, lo;
        mulhilo64(x, inv, hi, lo);
        uint64_t r = x - hi * n;
        if (r >= n) r -= n;
        return r;
      }
    }
  }
};
#endif

#ifdef __CUDA_ARCH__
#define CMC_LOG(x) ::log(x)
#define CMC_SQRT(x) ::sqrt(x)
#define CMC_POW(x, y) ::pow(x, y)
#else
#define CMC_LOG(x) std::log(x)
#define CMC_SQRT(x) std::sqrt(x)
#define CMC_POW(x, y) std::pow(x, y)
#endif

CMC_HD double as241_ratio(const double* num, const double* den, double r) {
  double n = num[7], d = den[7];
  for (int i = 6; i >= 0; --i) {
    n = n * r + num[i];
    d = d * r + den[i];
  }
  return n / d;
}

// Inverse standard normal CDF, Wichura's AS241 (PPND16): the published
// coefficient sets, evaluated in the same order as P:src/rng.cpp:88-146.
CMC_HD double normal_quantile(double p) {
  const double a[8] = {3.3871328727963666080e+00, 1.3314166789178437745e+02,
                       1.9715909503065514427e+03, 1.3731693765509461125e+04,
                       4.5921953931549871457e+04, 6.7265770927008700853e+04,
                       3.3430575583588128105e+04, 2.5090809287301226727e+03};
  const double b[8] = {1.0,
                       4.2313330701600911252e+01, 6.8718700749205790830e+02,
                       5.3941960214247511077e+03, 2.1213794301586595867e+04,
                       3.9307895800092710610e+04, 2.8729085735721942674e+04,
                       5.2264952788528545610e+03};
  const double q = p - 0.5;
  if (q <= 0.425 && q >= -0.425) {
    const double r = 0.180625 - q * q;
    return q * as241_ratio(a, b, r);
  }
  const double c[8] = {1.42343711074968357734e+00, 4.63033784615654529590e+00,
                       5.76949722146069140550e+00, 3.64784832476320460504e+00,
                       1.27045825245236838258e+00, 2.41780725177450611770e-01,
                       2.27238449892691845833e-02, 7.74545014278341407640e-04};
  const double dd[8] = {1.0,
                        2.05319162663775882187e+00, 1.67638483018380384940e+00,
                        6.89767334985100004550e-01, 1.48103976427480074590e-01,
                        1.51986665636164571966e-02, 5.47593808499534494600e-04,
                        1.05075007164441684324e-09};
  const double e[8] = {6.65790464350110377720e+00, 5.46378491116411436990e+00,
                       1.78482653991729133580e+00, 2.96560571828504891230e-01,
                       2.65321895265761230930e-02, 1.24266094738807843860e-03,
                       2.71155556874348757815e-05, 2.01033439929228813265e-07};
  const double f[8] = {1.0,
                       5.99832206555887937690e-01, 1.36929880922735805310e-01,
                       1.48753612908506148525e-02, 7.86869131145613259100e-04,
                       1.84631831751005468180e-05, 1.42151175831644588870e-07,
                       2.04426310338993978564e-15};
  double r = (q < 0.0) ? p : 1.0 - p;
  r = CMC_SQRT(-CMC_LOG(r));
  const double value =
      (r <= 5.0) ? as241_ratio(c, dd, r - 1.6) : as241_ratio(e, f, r - 5.0);
  return (q < 0.0) ? -value : value;
}

CMC_HD double normal(Stream& s) { return normal_quantile(s.u01()); }

// Marsaglia-Tsang Gamma(shape, rate) with the shape<1 boost drawn first and
// the 1e-300 floor, P:src/rng.cpp:48-74.
CMC_HD double gamma_draw(Stream& s, double shape, double rate) {
  double boost = 1.0;
  if (shape < 1.0) {
    boost = CMC_POW(s.u01(), 1.0 / shape);
    shape += 1.0;
  }
  const double d = shape - 1.0 / 3.0;
  const double c = 1.0 / (3.0 * CMC_SQRT(d));
  for (;;) {
    double x, v;
    do {
      x = normal(s);
      v = 1.0 + c * x;
    } while (v <= 0.0);
    v = v * v * v;
    const double u = s.u01();
    const double x2 = x * x;
    if (u < 1.0 - 0.0331 * x2 * x2 ||
        CMC_LOG(u) < 0.5 * x2 + d * (1.0 - v + CMC_LOG(v))) {
      double draw = boost * d * v / rate;
      if (draw < 1e-300) draw = 1e-300;
      return draw;
    }
  }
}

}  // namespace cmc
