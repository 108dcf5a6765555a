// Check- and variable-node kernels of the block decoder (templates).
//
// Replaces check_node_update / variable_node_update of
// /root/reference/pkg/src/qcldpc/bp.py:134-188.  Instantiated per check-degree
// bucket in cnu_dc*.cu so the many variants compile in parallel.
//
// Message representation on the store (edge-major (E, gamma) fp32):
//   BETA mode (public single-step API): var->check packages hold beta, exactly
//     the reference's MessageBatch contents (bp.py:59-84).
//   PHI mode (inside qc_decode): var->check packages hold sign(beta) *
//     phi(|beta|).  phi is evaluated once by the producer (variable pass) instead
//     of by the consumer, so each pass evaluates phi once per edge-lane and both
//     passes stay under the HBM time.
//   check->var packages always hold alpha.
#pragma once

#include <cuda_runtime.h>

#include "common.cuh"
#include "phi.cuh"
#include "plan.h"

namespace qcb {

// regular QC grid (every block live), a __grid_constant__ kernel parameter:
// edge id of (block row j, circulant row r, block col l) = (j*p + r)*L + l,
// its variable = l*p + (r + s_jl) mod p                      (codes.py:159-178)
// gamma/VEC >= 32 for every launch, so all lanes of a warp belong to the same
// check / variable and each shift lookup is a warp-uniform constant-bank load
// (no shared-memory staging, no CTA barrier).
struct QcGrid {
  int J, L, p;
  unsigned long long pmagic;   // ceil(2^40 / p): x / p == (x * pmagic) >> 40 for x < 2^24
  int16_t s[QC_MAX_J * QC_MAX_L];
};

__device__ __forceinline__ int div_p(const QcGrid& g, int x) {
  return (int)(((unsigned long long)(unsigned)x * g.pmagic) >> 40);
}

enum CnuMode { CNU_BETA = 0, CNU_FROM_MU = 1, CNU_PHI = 2 };
enum VnuMode { VNU_BETA = 0, VNU_PHI = 1, VNU_NONE = 2 };

struct CnuArgs {
  float* msgs;
  const float* mu;            // CNU_FROM_MU: beta^0 gathered from mu (fused init)
  const int32_t* check_ptr;   // irregular codes
  const int32_t* edge_var;    // CNU_FROM_MU without QC arithmetic
  const uint32_t* active;     // lane mask words or null
  const int32_t* done;        // early-stop "all frozen" flag or null
  int M, gamma;
};

struct VnuArgs {
  float* msgs;
  const float* mu;
  float* post;               // (N, gamma) or null
  uint32_t* hb;              // (N, gamma/32) or null
  const int32_t* var_pad;    // (N, dv) edge ids, -1 pad (non-QC)
  const uint32_t* active;
  const int32_t* done;
  int N, gamma, dv;
  int post_all;              // posteriors for every lane, frozen ones too (public single step, bp.py:183)
};

// Check-node update on registers: x[k][i] (edge k, lane i) -> alpha.
// IN_PHI: inputs are sign|psi(|beta|) (psi = phi/ln2); else inputs are beta.
//   |alpha_k| = min(phi(S - psi_k), ALPHA_CAP), S = sum_k psi_k, except the
//   dominant edge (largest psi): its exclusive sum S2 is accumulated directly
//   (S2 = sum of everything but the running maximum), so the subtraction
//   S - psi_k >= max psi never cancels; sign_k = parity of the other signs.
template <int DC, int VEC, bool IN_PHI, bool REL = false>
__device__ __forceinline__ void cnu_core(float (&x)[DC][VEC], int deg, unsigned lanes) {
  float S[VEC], S2[VEC], mx[VEC];
  unsigned par[VEC];
#pragma unroll
  for (int i = 0; i < VEC; ++i) {
    par[i] = 0;
    S[i] = 0.0f;
    S2[i] = 0.0f;
    mx[i] = -1.0f;
    if (!((lanes >> i) & 1u)) continue;
#pragma unroll
    for (int k = 0; k < DC; ++k) {
      if (k < deg) {
        float b = x[k][i];
        unsigned sb = __float_as_uint(b) & 0x80000000u;
        float f = IN_PHI ? fabsf(b) : psi_of_nat(fabsf(b));
        par[i] ^= sb;
        S2[i] = (f > mx[i]) ? S[i] : __fadd_rn(S2[i], f);
        mx[i] = fmaxf(mx[i], f);
        S[i] = __fadd_rn(S[i], f);
        if (!IN_PHI) x[k][i] = __uint_as_float(__float_as_uint(f) | sb);
      }
    }
  }
  // S2 excludes the first maximum.  An edge holding more than half of S is
  // the unique maximum and takes S2; every other edge takes S - psi_k >= S/2
  // (no cancellation).  The compact schedule (agg.cu) applies the same rule.
  if constexpr (VEC % 2 == 0) {
    // lane pairs on the packed fp32 pipe (bit-identical to the scalar form)
#pragma unroll
    for (int k = 0; k < DC; ++k) {
      if (k < deg) {
#pragma unroll
        for (int i = 0; i < VEC; i += 2) {
          const unsigned u0 = __float_as_uint(x[k][i]), u1 = __float_as_uint(x[k][i + 1]);
          const float f0 = __uint_as_float(u0 & 0x7fffffffu), f1 = __uint_as_float(u1 & 0x7fffffffu);
          float d0, d1;
          get2(sub2(mk2(S[i], S[i + 1]), mk2(f0, f1)), d0, d1);
          float p0, p1;
          get2(phi_of_log2_g2<REL>(mk2((f0 > d0) ? S2[i] : d0, (f1 > d1) ? S2[i + 1] : d1)), p0, p1);
          if ((lanes >> i) & 1u)
            x[k][i] = __uint_as_float(__float_as_uint(fminf(p0, ALPHA_CAP)) | ((u0 ^ par[i]) & 0x80000000u));
          if ((lanes >> (i + 1)) & 1u)
            x[k][i + 1] = __uint_as_float(__float_as_uint(fminf(p1, ALPHA_CAP)) | ((u1 ^ par[i + 1]) & 0x80000000u));
        }
      }
    }
  } else {
#pragma unroll
    for (int i = 0; i < VEC; ++i) {
      if (!((lanes >> i) & 1u)) continue;
#pragma unroll
      for (int k = 0; k < DC; ++k) {
        if (k < deg) {
          unsigned u = __float_as_uint(x[k][i]);
          float f = __uint_as_float(u & 0x7fffffffu);
          const float d = __fsub_rn(S[i], f);
          float mag = (f > d) ? S2[i] : d;
          float a = fminf(phi_of_log2_g<REL>(mag), ALPHA_CAP);
          x[k][i] = __uint_as_float(__float_as_uint(a) | ((u ^ par[i]) & 0x80000000u));
        }
      }
    }
  }
}

// one thread = (check m, VEC consecutive lanes); its d_c packages are contiguous
// note: a bare __launch_bounds__(256) gives 128 registers at d_c=24/float2
// (16 warps/SM, measured best); an explicit min-blocks of 1 lets ptxas grow to
// 188, and 3 forces spills -- both measured slower on B200.
template <int DC, int VEC, bool REG, int MODE, bool QC>
__global__ void __launch_bounds__(THREADS) cnu_kernel(CnuArgs a, const __grid_constant__ QcGrid grid) {
  if (a.done && *a.done) return;
  const int GV = a.gamma / VEC;
  long long tid = (long long)blockIdx.x * blockDim.x + threadIdx.x;
  if (tid >= (long long)a.M * GV) return;
  int m = (int)(tid / GV), q = (int)(tid - (long long)m * GV);
  int e0, deg;
  if constexpr (REG) { e0 = m * DC; deg = DC; }
  else { e0 = a.check_ptr[m]; deg = a.check_ptr[m + 1] - e0; }
  unsigned lanes = lane_bits_of(a.active, q * VEC, VEC);
  if (lanes == 0) return;   // frozen lanes keep their packages (bp.py:154-157)
  float x[DC][VEC];
#pragma unroll
  for (int k = 0; k < DC; ++k) {
    if (k < deg) {
      if constexpr (MODE == CNU_FROM_MU) {
        int v;
        if constexpr (QC) {
          int jrow = m / grid.p, r = m - jrow * grid.p;
          int c = r + grid.s[jrow * grid.L + k];
          c -= (c >= grid.p) ? grid.p : 0;
          v = k * grid.p + c;
        } else {
          v = a.edge_var[e0 + k];
        }
        vload<VEC>(a.mu + (size_t)v * a.gamma + q * VEC, x[k]);
      } else {
        vload<VEC>(a.msgs + (size_t)(e0 + k) * a.gamma + q * VEC, x[k]);
      }
    }
  }
  // the public single step (beta in) takes the relative-accurate check-side phi
  // (|alpha| within ~1e-5 relative down to tiny alphas); inside the decode loop
  // the absolute-accurate grade suffices (alpha only enters sums)
  cnu_core<DC, VEC, MODE == CNU_PHI, MODE == CNU_BETA>(x, deg, lanes);
#pragma unroll
  for (int k = 0; k < DC; ++k)
    if (k < deg) vstore<VEC>(a.msgs + (size_t)(e0 + k) * a.gamma + q * VEC, x[k]);
}

// one thread = (variable n, VEC consecutive lanes); d_v gathered packages
template <int DV, int VEC, bool QC, int MODE>
__global__ void __launch_bounds__(THREADS) vnu_kernel(VnuArgs a, const __grid_constant__ QcGrid grid) {
  if (a.done && *a.done) return;
  const int GV = a.gamma / VEC;
  long long tid = (long long)blockIdx.x * blockDim.x + threadIdx.x;
  bool valid = tid < (long long)a.N * GV;
  int n = valid ? (int)(tid / GV) : 0;
  int q = valid ? (int)(tid - (long long)n * GV) : 0;
  unsigned lanes = valid ? lane_bits_of(a.active, q * VEC, VEC) : 0u;
  int e[DV];
  int deg = 0;
  if constexpr (QC) {
    int l = n / grid.p, c = n - l * grid.p;
#pragma unroll
    for (int j = 0; j < DV; ++j) {
      int rr = c - grid.s[j * grid.L + l];
      rr += (rr < 0) ? grid.p : 0;
      e[j] = (j * grid.p + rr) * grid.L + l;
    }
    deg = DV;
  } else {
#pragma unroll
    for (int j = 0; j < DV; ++j) {
      e[j] = (j < a.dv && valid) ? a.var_pad[(size_t)n * a.dv + j] : -1;
      deg += (e[j] >= 0);
    }
  }
  float tot[VEC], am[DV][VEC];
  unsigned bits = 0;
  const unsigned plane = a.post_all ? (1u << VEC) - 1u : lanes;   // lanes whose posterior is written
  if (valid && plane) {
    vload<VEC>(a.mu + (size_t)n * a.gamma + q * VEC, tot);
#pragma unroll
    for (int j = 0; j < DV; ++j)
      if (j < deg) vload<VEC>(a.msgs + (size_t)e[j] * a.gamma + q * VEC, am[j]);
    // running total in increasing edge order (bp.py:179-181)
#pragma unroll
    for (int j = 0; j < DV; ++j)
      if (j < deg) {
#pragma unroll
        for (int i = 0; i < VEC; ++i) tot[i] = __fadd_rn(tot[i], am[j][i]);
      }
    if (MODE != VNU_NONE && lanes) {
#pragma unroll
      for (int j = 0; j < DV; ++j)
        if (j < deg) {
          float b[VEC];
          if constexpr (MODE == VNU_PHI && VEC % 2 == 0) {
            // lane pairs on the packed fp32 pipe (bit-identical to the scalar form)
#pragma unroll
            for (int i = 0; i < VEC; i += 2) {
              float d0, d1;
              get2(sub2(mk2(tot[i], tot[i + 1]), mk2(am[j][i], am[j][i + 1])), d0, d1);
              float q0, q1;
              get2(psi_of_nat_fast2(mk2(fminf(fabsf(d0), L_MAX), fminf(fabsf(d1), L_MAX))), q0, q1);
              q0 = __uint_as_float(__float_as_uint(q0) | (__float_as_uint(d0) & 0x80000000u));
              q1 = __uint_as_float(__float_as_uint(q1) | (__float_as_uint(d1) & 0x80000000u));
              b[i] = ((lanes >> i) & 1u) ? q0 : am[j][i];
              b[i + 1] = ((lanes >> (i + 1)) & 1u) ? q1 : am[j][i + 1];
            }
          } else {
#pragma unroll
            for (int i = 0; i < VEC; ++i) {
              float beta = clampL(__fsub_rn(tot[i], am[j][i]));
              if constexpr (MODE == VNU_PHI)
                beta = __uint_as_float(__float_as_uint(psi_of_nat_fast(fabsf(beta))) |
                                       (__float_as_uint(beta) & 0x80000000u));
              b[i] = ((lanes >> i) & 1u) ? beta : am[j][i];
            }
          }
          vstore<VEC>(a.msgs + (size_t)e[j] * a.gamma + q * VEC, b);
        }
    }
    float pst[VEC];
#pragma unroll
    for (int i = 0; i < VEC; ++i) {
      pst[i] = clampL(tot[i]);
      bits |= (pst[i] < 0.0f ? 1u : 0u) << i;
    }
    if (a.post) {
      if (plane == (1u << VEC) - 1u) {
        vstore<VEC>(a.post + (size_t)n * a.gamma + q * VEC, pst);
      } else {
        for (int i = 0; i < VEC; ++i)
          if ((plane >> i) & 1u) a.post[(size_t)n * a.gamma + q * VEC + i] = pst[i];
      }
    }
  }
  if (a.hb) store_bit_word<VEC>(a.hb + (size_t)n * (a.gamma >> 5), q, bits, valid);
}

// check pass: 2 lanes per thread (float2) -- measured best on B200 at d_c = 24
// (4 lanes: 171 registers, 8 warps/SM; 1 lane: LSU-issue bound)
// Small batches (the two-pass early stop at gamma < 128): lanes per thread up
// to 16 lane vectors per row, so the per-thread index math is shared (gamma
// 32: 2 lanes, two rows per warp; the hard-bit shuffle groups of 32 / VEC
// threads still cover one row's 32-lane word).
inline int pick_vec_cnu(int gamma, int) {
  if (gamma % 64 == 0) return 2;
  return (gamma % 2 == 0 && gamma / 2 >= 16) ? 2 : 1;
}
// variable pass: float4 packages
inline int pick_vec_vnu(int gamma) {
  if (gamma % 128 == 0) return 4;
  if (gamma % 4 == 0 && gamma / 4 >= 16) return 4;
  if (gamma % 2 == 0 && gamma / 2 >= 16) return 2;
  return 1;
}

QcGrid make_grid(const qc_plan* p);


// compact check-state schedule (agg.cu)
constexpr int AGG_FIRST_FLAG = 1, AGG_LAST_FLAG = 2;
bool agg_eligible(const qc_plan* p);
size_t agg_words(const qc_plan* p, int gamma);
int launch_agg_check(const qc_plan* p, int gamma, bool from_mu, float* msgs, const float* mu, float* agg,
                     cudaStream_t s);
int launch_agg_var(const qc_plan* p, int gamma, int flags, float* msgs, const float* mu, const float* agg,
                   float* post, uint32_t* hb, cudaStream_t s);
int run_agg_decode(const qc_plan* p, int gamma, int iters, float* msgs, const float* mu, float* agg, float* post,
                   uint32_t* hb, cudaStream_t s);
int agg_decode_launches(const qc_plan* p, int gamma, int iters);
bool agg_es_eligible(const qc_plan* p, int gamma);
int run_agg_decode_es(const qc_plan* p, int gamma, int iters, float* msgs, const float* mu, float* agg, float* post,
                      uint32_t* hb, uint32_t* es_words, uint8_t* ok, int32_t* iters_run, cudaStream_t s);
int run_agg_es_segment(const qc_plan* p, int gamma, int t0, int t1, int iters, float* msgs, const float* mu,
                       float* agg, float* post, uint32_t* hb, uint32_t* es_words, int32_t* iters_run,
                       cudaStream_t s, const int32_t* live, int live_loop);
int launch_es_tail(const qc_plan* p, int gamma, int iters, uint32_t* const act[2], uint32_t* const bad[2],
                   uint32_t* bad_fin, uint8_t* ok, int32_t* iters_run, const float* post, uint32_t* hb,
                   cudaStream_t s);
int launch_syndrome_ext(const qc_plan* p, int gamma, const uint32_t* hb, uint32_t* bad, cudaStream_t s);
int launch_hard_bits_ext(const qc_plan* p, int gamma, const float* post, uint32_t* hb, cudaStream_t s);
int launch_bit_errors_ext(const qc_plan* p, int gamma, const uint32_t* hb, int32_t* lane_bits, cudaStream_t s,
                          const uint32_t* lane_mask = nullptr);
bool es_compact_eligible(const qc_plan* p, int gamma, int iters);
size_t es_compact_words(const qc_plan* p, int gamma);
int run_agg_decode_es_compact(const qc_plan* p, int gamma, int iters, float* msgs, const float* mu, float* post,
                              uint32_t* hb, uint32_t* work, uint32_t* scratch, uint8_t* ok, int32_t* iters_run,
                              cudaStream_t s);
int es_compact_launches(const qc_plan* p, int gamma, int iters);
size_t work_head_words(int gamma);
bool agg_fused_eligible(const qc_plan* p, int gamma);
int launch_agg_fused(const qc_plan* p, int gamma, int lanes, int v0, int flags, int c0, bool from_mu, float* msgs,
                     const float* mu, float* agg, float* post, uint32_t* hb, cudaStream_t s);

template <int DC>
int launch_cnu_dc(const qc_plan* p, const CnuArgs& a, int mode, cudaStream_t s);

int launch_vnu(const qc_plan* p, VnuArgs a, int mode, cudaStream_t s);

}  // namespace qcb
