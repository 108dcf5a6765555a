// phi(x) = -ln tanh(x/2) = ln((1+e^-x)/(1-e^-x)), x >= 0, in fp32 on the MUFU pipe.
//
// The reference evaluates the check rule as 2*atanh(prod tanh(beta/2)) in
// float64 (bp.py:143-152).  In fp32 that form is unusable (1 - tanh loses all
// bits above |beta| ~ 8), so the B200 path runs the equivalent log domain
//   |alpha_k| = min(phi(sum_{j != k} phi(|beta_j|)), ALPHA_CAP),
//   sign(alpha_k) = prod_{j != k} sign(beta_j),
// where ALPHA_CAP = 2 atanh(1 - 1e-12) reproduces the reference's tanh-domain
// clamp (bp.py:150, TANH_CLAMP).  phi is its own inverse.
//
// Three branch-free regions, each accurate to a few fp32 ulp relative:
//   x < 0.25          : m = 1 - e^-x by its Taylor series (expm1 accuracy where
//                       the subtraction would cancel), phi = ln((2-m)/m)
//   t = e^-x >= 1/8   : phi = ln((1+t)/(1-t)) via lg2 and rcp
//   t < 1/8           : phi = 2 atanh(t) = 2t(1 + t^2/3 + t^4/5 + t^6/7)
//                       (no log: relative accuracy kept for tiny t)
// m is floored at 1e-30 so phi(0) = 69.3 instead of inf: sums stay finite and
// the exclusive-sum subtraction can never produce inf - inf.
#pragma once

namespace qcb {

__device__ __forceinline__ float ex2a(float x) {
  float y;
  asm("ex2.approx.ftz.f32 %0, %1;" : "=f"(y) : "f"(x));
  return y;
}
__device__ __forceinline__ float lg2a(float x) {
  float y;
  asm("lg2.approx.ftz.f32 %0, %1;" : "=f"(y) : "f"(x));
  return y;
}
__device__ __forceinline__ float rcpa(float x) {
  float y;
  asm("rcp.approx.ftz.f32 %0, %1;" : "=f"(y) : "f"(x));
  return y;
}

__device__ __forceinline__ float phi(float x) {
  const float LOG2E = 1.4426950408889634f;
  const float LN2 = 0.6931471805599453f;
  float t = ex2a(__fmul_rn(-x, LOG2E));
  float ms = __fmul_rn(
      x, fmaf(x, fmaf(x, fmaf(x, fmaf(x, fmaf(x, -1.0f / 720.0f, 1.0f / 120.0f), -1.0f / 24.0f),
                              1.0f / 6.0f),
                      -0.5f),
              1.0f));
  float m = (x < 0.25f) ? fmaxf(ms, 1e-30f) : __fsub_rn(1.0f, t);
  float r = __fmul_rn(__fsub_rn(2.0f, m), rcpa(m));
  float pl = __fmul_rn(lg2a(r), LN2);
  float t2 = __fmul_rn(t, t);
  float ps = __fmul_rn(__fmul_rn(2.0f, t),
                       fmaf(t2, fmaf(t2, fmaf(t2, 1.0f / 7.0f, 1.0f / 5.0f), 1.0f / 3.0f), 1.0f));
  return (t < 0.125f) ? ps : pl;
}

// ---------------------------------------------------------------------------
// The decode loop keeps phi in log2 units (psi = phi / ln 2): the check pass
// then feeds sums straight into ex2 and the variable pass takes lg2 without a
// rescale.  Cheaper branch-free regions (max rel. error ~7e-6 including the
// MUFU approximation error, validated in tests/test_gpu_block.py):
//   x < 2^-7      : m = 1 - e^-x = x(1 - x/2 + x^2/6)
//   t >= 1/32     : lg2((2 - m)/m)
//   t < 1/32      : 2t(1 + t^2/3 + t^4/5)   (series, relative accuracy)
// ---------------------------------------------------------------------------

// psi(x) = phi(x) / ln2 for a natural-log-domain magnitude x >= 0
__device__ __forceinline__ float psi_of_nat(float x) {
  const float LOG2E = 1.4426950408889634f;
  float t = ex2a(__fmul_rn(-x, LOG2E));
  float ms = __fmul_rn(x, fmaf(x, fmaf(x, 1.0f / 6.0f, -0.5f), 1.0f));
  float m = (x < 0.0078125f) ? fmaxf(ms, 1e-30f) : __fsub_rn(1.0f, t);
  float pl = lg2a(__fmul_rn(__fsub_rn(2.0f, m), rcpa(m)));
  float t2 = __fmul_rn(t, t);
  float ps = __fmul_rn(t, fmaf(t2, fmaf(t2, 0.4f * LOG2E, (2.0f / 3.0f) * LOG2E), 2.0f * LOG2E));
  return (t < 0.03125f) ? ps : pl;
}

// psi for the decode loop's variable-to-check messages: the same as
// psi_of_nat without the small-x series.  For |beta| < 2^-7, m = 1 - t loses
// relative accuracy (psi itself is >= 8 there), but such a psi only ever
// (a) dominates its check's sum, where the dominant edge's own alpha uses the
// sum WITHOUT it (S2), or (b) sits inside S - psi_k >= psi for the other
// edges, whose alphas are then <= 2^-7 and absolutely accurate to ~1e-8.
// Five fewer instructions per edge-lane on the issue-bound variable job.  The
// public single-step API and the LDPCCC keep psi_of_nat.
__device__ __forceinline__ float psi_of_nat_fast(float x) {
  const float LOG2E = 1.4426950408889634f;
  float t = ex2a(__fmul_rn(-x, LOG2E));
  float m = fmaxf(__fsub_rn(1.0f, t), 1e-30f);
  float pl = lg2a(__fmul_rn(__fsub_rn(2.0f, m), rcpa(m)));
  float t2 = __fmul_rn(t, t);
  float ps = __fmul_rn(t, fmaf(t2, fmaf(t2, 0.4f * LOG2E, (2.0f / 3.0f) * LOG2E), 2.0f * LOG2E));
  return (t < 0.03125f) ? ps : pl;
}

// phi(y ln2), natural-log-domain result, for a log2-domain argument y >= 0:
// the check-to-variable magnitude |alpha|.  Two accuracy grades:
//   phi_of_log2      absolute accuracy ~3e-7 (alpha only enters sums), no
//                    small-t series: 6 fewer instructions per edge, 5% on the
//                    MUFU/issue-heavy compact variable job (block decoder);
//   phi_of_log2_rel  relative accuracy a few ulp everywhere (2t(1 + t^2/3 +
//                    t^4/5) for t = 2^-y < 1/32): the LDPCCC kernels (about
//                    5% of slot time there).
// The grade moves single decisions of posteriors within fp32 rounding of 0 in
// all-failing frames (about 1 bit in 10^6 of such frames); against the float64
// oracle tools/campaign_parity.py measured identical counts for each path
// with the grade it uses (profiles/r01/campaign_parity_*.jsonl).
__device__ __forceinline__ float phi_of_log2(float y) {
  const float LN2 = 0.6931471805599453f;
  float t = ex2a(-y);
  float ms = __fmul_rn(y, fmaf(y, fmaf(y, 0.055504108664821580f /* ln2^3/6 */, -0.24022650695910071f /* -ln2^2/2 */),
                               LN2));
  float m = (y < 0.011270696f /* 2^-7 / ln2 */) ? fmaxf(ms, 1e-30f) : __fsub_rn(1.0f, t);
  return __fmul_rn(lg2a(__fmul_rn(__fsub_rn(2.0f, m), rcpa(m))), LN2);
}

__device__ __forceinline__ float phi_of_log2_rel(float y) {
  const float LN2 = 0.6931471805599453f;
  float t = ex2a(-y);
  float ms = __fmul_rn(y, fmaf(y, fmaf(y, 0.055504108664821580f /* ln2^3/6 */, -0.24022650695910071f /* -ln2^2/2 */),
                               LN2));
  float m = (y < 0.011270696f /* 2^-7 / ln2 */) ? fmaxf(ms, 1e-30f) : __fsub_rn(1.0f, t);
  float pl = __fmul_rn(lg2a(__fmul_rn(__fsub_rn(2.0f, m), rcpa(m))), LN2);
  float t2 = __fmul_rn(t, t);
  float ps = __fmul_rn(t, fmaf(t2, fmaf(t2, 0.4f, 2.0f / 3.0f), 2.0f));
  return (t < 0.03125f) ? ps : pl;
}

template <bool REL>
__device__ __forceinline__ float phi_of_log2_g(float y) {
  if constexpr (REL) return phi_of_log2_rel(y);
  else return phi_of_log2(y);
}

// ---------------------------------------------------------------------------
// Two lanes at once on the packed fp32 pipe (sm_100: FADD2 / FMUL2 / FFMA2,
// each lane rounded exactly like the scalar instruction, so these return
// bit-for-bit the scalar functions above; MUFU ops, compares and selects stay
// per lane).  About 40% fewer issued instructions per phi pair.
// ---------------------------------------------------------------------------
struct f2 {
  unsigned long long v;
};

__device__ __forceinline__ f2 mk2(float a, float b) {
  f2 r;
  asm("mov.b64 %0, {%1, %2};" : "=l"(r.v) : "f"(a), "f"(b));
  return r;
}
__device__ __forceinline__ f2 splat2(float a) { return mk2(a, a); }
__device__ __forceinline__ void get2(f2 x, float& a, float& b) {
  asm("mov.b64 {%0, %1}, %2;" : "=f"(a), "=f"(b) : "l"(x.v));
}
__device__ __forceinline__ f2 add2(f2 a, f2 b) {
  f2 r;
  asm("add.rn.f32x2 %0, %1, %2;" : "=l"(r.v) : "l"(a.v), "l"(b.v));
  return r;
}
__device__ __forceinline__ f2 sub2(f2 a, f2 b) {
  f2 r;
  asm("sub.rn.f32x2 %0, %1, %2;" : "=l"(r.v) : "l"(a.v), "l"(b.v));
  return r;
}
__device__ __forceinline__ f2 mul2(f2 a, f2 b) {
  f2 r;
  asm("mul.rn.f32x2 %0, %1, %2;" : "=l"(r.v) : "l"(a.v), "l"(b.v));
  return r;
}
__device__ __forceinline__ f2 fma2(f2 a, f2 b, f2 c) {
  f2 r;
  asm("fma.rn.f32x2 %0, %1, %2, %3;" : "=l"(r.v) : "l"(a.v), "l"(b.v), "l"(c.v));
  return r;
}

// psi_of_nat on a lane pair (x >= 0)
__device__ __forceinline__ f2 psi_of_nat2(f2 x) {
  const float LOG2E = 1.4426950408889634f;
  float x0, x1;
  get2(x, x0, x1);
  float a0, a1;
  get2(mul2(x, splat2(-LOG2E)), a0, a1);                       // -(x log2 e), exact sign symmetry
  const f2 t = mk2(ex2a(a0), ex2a(a1));
  const f2 ms = mul2(x, fma2(x, fma2(x, splat2(1.0f / 6.0f), splat2(-0.5f)), splat2(1.0f)));
  const f2 omt = sub2(splat2(1.0f), t);
  float ms0, ms1, o0, o1;
  get2(ms, ms0, ms1);
  get2(omt, o0, o1);
  const f2 m = mk2((x0 < 0.0078125f) ? fmaxf(ms0, 1e-30f) : o0, (x1 < 0.0078125f) ? fmaxf(ms1, 1e-30f) : o1);
  float m0, m1;
  get2(m, m0, m1);
  float r0, r1;
  get2(mul2(sub2(splat2(2.0f), m), mk2(rcpa(m0), rcpa(m1))), r0, r1);
  const float pl0 = lg2a(r0), pl1 = lg2a(r1);
  const f2 t2 = mul2(t, t);
  const f2 ps = mul2(t, fma2(t2, fma2(t2, splat2(0.4f * LOG2E), splat2((2.0f / 3.0f) * LOG2E)), splat2(2.0f * LOG2E)));
  float t0, t1, ps0, ps1;
  get2(t, t0, t1);
  get2(ps, ps0, ps1);
  return mk2((t0 < 0.03125f) ? ps0 : pl0, (t1 < 0.03125f) ? ps1 : pl1);
}

// psi_of_nat_fast on a lane pair (x >= 0)
__device__ __forceinline__ f2 psi_of_nat_fast2(f2 x) {
  const float LOG2E = 1.4426950408889634f;
  float a0, a1;
  get2(mul2(x, splat2(-LOG2E)), a0, a1);
  const f2 t = mk2(ex2a(a0), ex2a(a1));
  float o0, o1;
  get2(sub2(splat2(1.0f), t), o0, o1);
  const float m0 = fmaxf(o0, 1e-30f), m1 = fmaxf(o1, 1e-30f);
  float r0, r1;
  get2(mul2(sub2(splat2(2.0f), mk2(m0, m1)), mk2(rcpa(m0), rcpa(m1))), r0, r1);
  const float pl0 = lg2a(r0), pl1 = lg2a(r1);
  const f2 t2 = mul2(t, t);
  const f2 ps = mul2(t, fma2(t2, fma2(t2, splat2(0.4f * LOG2E), splat2((2.0f / 3.0f) * LOG2E)), splat2(2.0f * LOG2E)));
  float t0, t1, ps0, ps1;
  get2(t, t0, t1);
  get2(ps, ps0, ps1);
  return mk2((t0 < 0.03125f) ? ps0 : pl0, (t1 < 0.03125f) ? ps1 : pl1);
}

// phi_of_log2 on a lane pair (y >= 0)
__device__ __forceinline__ f2 phi_of_log2_2(f2 y) {
  const float LN2 = 0.6931471805599453f;
  float y0, y1;
  get2(y, y0, y1);
  const float t0 = ex2a(-y0), t1 = ex2a(-y1);
  const f2 ms = mul2(y, fma2(y, fma2(y, splat2(0.055504108664821580f), splat2(-0.24022650695910071f)), splat2(LN2)));
  const f2 omt = sub2(splat2(1.0f), mk2(t0, t1));
  float ms0, ms1, o0, o1;
  get2(ms, ms0, ms1);
  get2(omt, o0, o1);
  const float m0 = (y0 < 0.011270696f) ? fmaxf(ms0, 1e-30f) : o0;
  const float m1 = (y1 < 0.011270696f) ? fmaxf(ms1, 1e-30f) : o1;
  float r0, r1;
  get2(mul2(sub2(splat2(2.0f), mk2(m0, m1)), mk2(rcpa(m0), rcpa(m1))), r0, r1);
  return mul2(mk2(lg2a(r0), lg2a(r1)), splat2(LN2));
}

// phi_of_log2_rel on a lane pair (y >= 0)
__device__ __forceinline__ f2 phi_of_log2_rel_2(f2 y) {
  const float LN2 = 0.6931471805599453f;
  float y0, y1;
  get2(y, y0, y1);
  const f2 t = mk2(ex2a(-y0), ex2a(-y1));
  const f2 ms = mul2(y, fma2(y, fma2(y, splat2(0.055504108664821580f), splat2(-0.24022650695910071f)), splat2(LN2)));
  const f2 omt = sub2(splat2(1.0f), t);
  float ms0, ms1, o0, o1;
  get2(ms, ms0, ms1);
  get2(omt, o0, o1);
  const float m0 = (y0 < 0.011270696f) ? fmaxf(ms0, 1e-30f) : o0;
  const float m1 = (y1 < 0.011270696f) ? fmaxf(ms1, 1e-30f) : o1;
  float r0, r1;
  get2(mul2(sub2(splat2(2.0f), mk2(m0, m1)), mk2(rcpa(m0), rcpa(m1))), r0, r1);
  float pl0, pl1;
  get2(mul2(mk2(lg2a(r0), lg2a(r1)), splat2(LN2)), pl0, pl1);
  const f2 t2 = mul2(t, t);
  const f2 ps = mul2(t, fma2(t2, fma2(t2, splat2(0.4f), splat2(2.0f / 3.0f)), splat2(2.0f)));
  float t0, t1, ps0, ps1;
  get2(t, t0, t1);
  get2(ps, ps0, ps1);
  return mk2((t0 < 0.03125f) ? ps0 : pl0, (t1 < 0.03125f) ? ps1 : pl1);
}

template <bool REL>
__device__ __forceinline__ f2 phi_of_log2_g2(f2 y) {
  if constexpr (REL) return phi_of_log2_rel_2(y);
  else return phi_of_log2_2(y);
}

}  // namespace qcb
