// Philox4x64-10 (Random123) and the Cephes inverse normal CDF, fp64, device side.
#pragma once

#include <stdint.h>

namespace qcb {

__device__ __forceinline__ void philox4x64_10(uint64_t c0, uint64_t c1, uint64_t c2, uint64_t c3,
                                              uint64_t k0, uint64_t k1, uint64_t (&out)[4]) {
  const uint64_t M0 = 0xD2E7470EE14C6C93ull, M1 = 0xCA5A826395121157ull;
  const uint64_t W0 = 0x9E3779B97F4A7C15ull, W1 = 0xBB67AE8584CAA73Bull;
#pragma unroll
  for (int r = 0; r < 10; ++r) {
    uint64_t hi0 = __umul64hi(M0, c0), lo0 = M0 * c0;
    uint64_t hi1 = __umul64hi(M1, c2), lo1 = M1 * c2;
    uint64_t n0 = hi1 ^ c1 ^ k0, n2 = hi0 ^ c3 ^ k1;
    c0 = n0; c1 = lo1; c2 = n2; c3 = lo0;
    k0 += W0; k1 += W1;
  }
  out[0] = c0; out[1] = c1; out[2] = c2; out[3] = c3;
}

// strictly inside (0,1): top 53 bits centred on the grid (channel.py:75-76)
__device__ __forceinline__ double word_to_uniform(uint64_t w) {
  return __dmul_rn(__dadd_rn((double)(w >> 11), 0.5), 1.1102230246251565404e-16);
}

// Cephes ndtri coefficient tables (scipy/special/cephes/ndtri.c) in the
// constant bank: the fp64 multiply-adds take them as c[][] operands directly
// (as immediates every use cost a pair of uniform-register moves).
static __constant__ double kNdtriP0[5] = {-5.99633501014107895267E1, 9.80010754185999661536E1,
                                          -5.66762857469070293439E1, 1.39312609387279679503E1,
                                          -1.23916583867381258016E0};
static __constant__ double kNdtriQ0[8] = {1.95448858338141759834E0, 4.67627912898881538453E0,
                                          8.63602421390890590575E1, -2.25462687854119370527E2,
                                          2.00260212380060660359E2, -8.20372256168333339912E1,
                                          1.59056225126211695515E1, -1.18331621121330003142E0};
static __constant__ double kNdtriP1[9] = {4.05544892305962419923E0, 3.15251094599893866154E1,
                                          5.71628192246421288162E1, 4.40805073893200834700E1,
                                          1.46849561928858024014E1, 2.18663306850790267539E0,
                                          -1.40256079171354495875E-1, -3.50424626827848203418E-2,
                                          -8.57456785154685413611E-4};
static __constant__ double kNdtriQ1[8] = {1.57799883256466749731E1, 4.53907635128879210584E1,
                                          4.13172038254672030440E1, 1.50425385692907503408E1,
                                          2.50464946208309415979E0, -1.42182922854787788574E-1,
                                          -3.80806407691578277194E-2, -9.33259480895457427372E-4};
static __constant__ double kNdtriP2[9] = {3.23774891776946035970E0, 6.91522889068984211695E0,
                                          3.93881025292474443415E0, 1.33303460815807542389E0,
                                          2.01485389549179081538E-1, 1.23716634817820021358E-2,
                                          3.01581553508235416007E-4, 2.65806974686737550832E-6,
                                          6.23974539184983293730E-9};
static __constant__ double kNdtriQ2[8] = {6.02427039364742014255E0, 3.67983563856160859403E0,
                                          1.37702099489081330271E0, 2.16236993594496635890E-1,
                                          1.34204006088543189037E-2, 3.28014464682127739104E-4,
                                          2.89247864745380683936E-6, 6.79019408009981274425E-9};

// polevl / p1evl (Cephes) with fused multiply-adds: within 1 ulp of the
// reference's separately rounded evaluation (normals agree to <= 2 ulp,
// tests/test_gpu_channel.py)
__device__ __forceinline__ double horner(double x, const double* c, int n) {
  double a = c[0];
  for (int i = 1; i < n; ++i) a = __fma_rn(a, x, c[i]);
  return a;
}
__device__ __forceinline__ double horner1(double x, const double* c, int n) {
  double a = __dadd_rn(x, c[0]);
  for (int i = 1; i < n; ++i) a = __fma_rn(a, x, c[i]);
  return a;
}

constexpr double kNdtriExpm2 = 0.13533528323661269189;   // exp(-2)

// Cephes ndtri split into its two regions so a caller can run each region
// over a compacted list of samples (channel.cu): central for
// exp(-2) < y0 <= 1 - exp(-2), tail otherwise.
__device__ __forceinline__ bool ndtri_is_central(double y0) {
  return y0 > kNdtriExpm2 && !(y0 > __dsub_rn(1.0, kNdtriExpm2));
}

__device__ __forceinline__ double ndtri_central(double y0) {
  const double S2PI = 2.50662827463100050242E0;
  double y = __dsub_rn(y0, 0.5);
  double y2 = __dmul_rn(y, y);
  double r = __ddiv_rn(__dmul_rn(y2, horner(y2, kNdtriP0, 5)), horner1(y2, kNdtriQ0, 8));
  return __dmul_rn(__dadd_rn(y, __dmul_rn(y, r)), S2PI);
}

__device__ __forceinline__ double ndtri_tail(double y0) {
  bool neg = true;
  double y = y0;
  if (y > __dsub_rn(1.0, kNdtriExpm2)) {
    y = __dsub_rn(1.0, y);
    neg = false;
  }
  double x = sqrt(__dmul_rn(-2.0, log(y)));
  double x0 = __dsub_rn(x, __ddiv_rn(log(x), x));
  double z = __ddiv_rn(1.0, x);
  double x1 = (x < 8.0) ? __ddiv_rn(__dmul_rn(z, horner(z, kNdtriP1, 9)), horner1(z, kNdtriQ1, 8))
                        : __ddiv_rn(__dmul_rn(z, horner(z, kNdtriP2, 9)), horner1(z, kNdtriQ2, 8));
  x = __dsub_rn(x0, x1);
  return neg ? -x : x;
}

__device__ __forceinline__ double ndtri_cephes(double y0) {
  return ndtri_is_central(y0) ? ndtri_central(y0) : ndtri_tail(y0);
}

}  // namespace qcb
