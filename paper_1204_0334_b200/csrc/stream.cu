// Pipelined LDPC convolutional (LDPCCC) window decoder on sm_100a.
//
// Replaces StreamDecoder._advance (/root/reference/pkg/src/qcldpc/
// convolutional.py:252-337) and the unwrapping tables of LdpcccCode
// (convolutional.py:67-151).
//
// Memory (circular window in HBM):
//   msg  (I*E, gamma) fp32: I processor groups, each one copy of the base
//        code's edge space ordered by sub-block label (sub_offset), edge-major
//        Gamma-packages as in the block decoder;
//   ring (I*T, c, gamma) fp32: channel LLRs of the frames in flight.
// Index storage is compressed with the code's period and QC structure
// (PAPER.md:1144-1195): sub-block labels come from period arithmetic
// (lut_c[k][d] = (k, k+1+d mod T), lut_v[f][d] = (f+d mod T, f)), and edge
// addresses inside a sub-block from its circulant shifts, staged in shared
// memory -- no per-edge tables.  Shift grids with zero blocks fall back to
// small per-label tables (check (cb, wmax) and variable (c, sub_j) local ids).
//
// Message representation: var->check packages hold sign(beta) * psi(|beta|)
// (phi in log2 units, "phi form", as in the block decoder's loop), check->var
// packages hold alpha; each pass evaluates phi once per edge-lane.
//
// Slot t = three kernels: entry (frame t -> ring + its T sub-blocks), check
// phase (I layers in one launch: they touch disjoint edge sets), variable
// phase (I frames, the last one emitted).  The emission-time zero clear of the
// reference (convolutional.py:328-330) is omitted: the next entry overwrites
// exactly those edges and ring slot (window = I*T is a multiple of T).
#include <cuda_runtime.h>

#include <algorithm>
#include <cstdlib>
#include <cstring>
#include <numeric>
#include <string>
#include <vector>

#include "common.cuh"
#include "block_kernels.cuh"
#include "phi.cuh"

using namespace qcb;

#ifndef CC_THREADS
#define CC_THREADS 128   // +0.8% over 256 (profiles/r01/sbench_threads.jsonl)
#endif
#define CC_MAX_LAM 8
#define CC_MAX_SHIFTS 2048

struct cc_plan {
  int J = 0, L = 0, p = 0, lam = 0, ms = 0, sj = 0, sl = 0, c = 0, cb = 0, E = 0, wmax = 0;
  bool all_live = false;
  std::vector<int64_t> shifts;
  int sub_off[CC_MAX_LAM * CC_MAX_LAM] = {0};
  int32_t* d_check_tab = nullptr;   // (lam^2, cb, wmax)
  int32_t* d_var_tab = nullptr;     // (lam^2, c, sj)
};

namespace {

struct CcParams {
  int lam, ms, sj, sl, c, cb, p, E, wmax, J, L;
  int I, gamma;
  int sub_off[CC_MAX_LAM * CC_MAX_LAM];
  int16_t s[CC_MAX_SHIFTS];
};

struct SlotArgs {
  float* msg;
  float* ring;
  const float* mu_in;       // (c, gamma) or null (virtual frame)
  float* post_out;          // (c, gamma) or null
  int32_t* cnt;             // (3, gamma) lane counters or null
  const int32_t* check_tab;
  const int32_t* var_tab;
  const int64_t* t_dev;
  int t;                    // slot (t_dev: offset added to *t_dev); < 2^31
  int ip0, nip;             // processors [ip0, ip0 + nip) of this launch (0-based; nip = I: the whole slot)
  // look-ahead slot form (cc_slot_ahead): the check phase folds the previous
  // emission's counters, and the emitting processor's variable threads enter
  // frame t + 1 (mu_next; null = zero-LLR virtual frame) right after emitting
  // frame t + 1 - window, which held the same ring slot and edge slots
  const float* mu_next;
  int fold_in_check, entry_next;
};

__device__ __forceinline__ int slot_of(const SlotArgs& a) {
  return a.t_dev ? (int)(*a.t_dev) + a.t : a.t;
}

// x mod m for x >= -m*k (slot arithmetic stays in 32 bits)
__device__ __forceinline__ int pmod(int x, int m) {
  int r = x % m;
  return r < 0 ? r + m : r;
}

// Edges of variable v (block column bc, circulant column cc) of a frame with
// phase ph in group base `grp`, in the reference's summation order
// (d = 0..T-1 over LUT_v[ph][d], then block row br; convolutional.py:136-151, 307-317).
// QC: local id of (br, bc) in sub-block (R, ph) = (br*p + (cc - s) mod p)*sl + bc.
// Shift lookups are warp-uniform (gamma/VEC >= 32: a warp is one variable) and
// read straight from the __grid_constant__ parameter bank.
template <int DV, bool QC, int TT = 0, int SJ = 0>
__device__ __forceinline__ unsigned var_edges(const CcParams& P, const int32_t* var_tab,
                                              int ph, unsigned grp, int v, int bc, int cc, unsigned (&e)[DV]) {
  unsigned present = 0;
  const int T = TT ? TT : P.lam;
  if constexpr (QC && TT > 0 && SJ > 0) {
    static_assert(TT * SJ <= DV, "bucket too small");
#pragma unroll
    for (int d = 0; d < TT; ++d) {
      int R = ph + d;
      R -= (R >= TT) ? TT : 0;
      const int lbl = R * TT + ph;
#pragma unroll
      for (int br = 0; br < SJ; ++br) {
        int rr = cc - P.s[(R * SJ + br) * P.L + ph * P.sl + bc];
        rr += rr < 0 ? P.p : 0;
        e[d * SJ + br] = grp + (unsigned)P.sub_off[lbl] + (unsigned)((br * P.p + rr) * P.sl + bc);
      }
    }
#pragma unroll
    for (int k = TT * SJ; k < DV; ++k) e[k] = 0;
    return (1u << (TT * SJ)) - 1u;
  }
  int d = 0, br = 0;
#pragma unroll
  for (int k = 0; k < DV; ++k) {
    e[k] = 0;
    if (k < T * P.sj) {
      int R = ph + d;
      R -= (R >= T) ? T : 0;
      int lbl = R * T + ph;
      int loc;
      if constexpr (QC) {
        int rr = cc - P.s[(R * P.sj + br) * P.L + ph * P.sl + bc];
        rr += rr < 0 ? P.p : 0;
        loc = (br * P.p + rr) * P.sl + bc;
      } else {
        loc = var_tab[((size_t)lbl * P.c + v) * P.sj + br];
      }
      if (loc >= 0) { e[k] = grp + (unsigned)P.sub_off[lbl] + (unsigned)loc; present |= 1u << k; }
      if (++br == P.sj) { br = 0; ++d; }
    }
  }
  return present;
}

// check-node core with a `present` mask of live positions (bootstrap layers
// drop absent frames); same arithmetic as the block decoder (block_kernels.cuh)
// with the relative-accurate phi (phi.cuh).
// Inputs are var->check packages in phi form (sign | psi(|beta|), log2 units).
template <int DC, int VEC>
__device__ __forceinline__ void cnu_core_mask(float (&x)[DC][VEC], unsigned long long present) {
#pragma unroll
  for (int i = 0; i < VEC; ++i) {
    unsigned par = 0;
    float S = 0.0f, S2 = 0.0f, mx = -1.0f;
#pragma unroll
    for (int k = 0; k < DC; ++k) {
      if ((present >> k) & 1ull) {
        float b = x[k][i];
        unsigned sb = __float_as_uint(b) & 0x80000000u;
        float f = fabsf(b);
        par ^= sb;
        S2 = (f > mx) ? S : __fadd_rn(S2, f);
        mx = fmaxf(mx, f);
        S = __fadd_rn(S, f);
      }
    }
#pragma unroll
    for (int k = 0; k < DC; ++k) {
      if ((present >> k) & 1ull) {
        unsigned u = __float_as_uint(x[k][i]);
        float f = __uint_as_float(u & 0x7fffffffu);
        // S2 excludes the first maximum: the dominant edge (more than half of
        // S, necessarily the maximum) takes it, every other edge S - psi_k
        const float d = __fsub_rn(S, f);
        float mag = (f > d) ? S2 : d;
        float al = fminf(phi_of_log2_rel(mag), ALPHA_CAP);
        x[k][i] = __uint_as_float(__float_as_uint(al) | ((u ^ par) & 0x80000000u));
      }
    }
  }
}

// ---- entry: frame tf into ring slot tf mod window and its T sub-blocks -----
template <int DV, int VEC, bool QC, int TT = 0, int SJ = 0>
__device__ __forceinline__ void entry_body(const SlotArgs& a, const CcParams& P, int tf, const float* mu_src, int v,
                                           int q) {
  const int T = TT ? TT : P.lam, window = P.I * T;
  float m[VEC];
  if (mu_src) vload<VEC>(mu_src + (size_t)v * P.gamma + q * VEC, m);
  else {
#pragma unroll
    for (int i = 0; i < VEC; ++i) m[i] = 0.0f;
  }
  vstore<VEC>(a.ring + ((size_t)pmod(tf, window) * P.c + v) * P.gamma + q * VEC, m);
  // beta^0 = mu into the frame's T sub-blocks, stored in phi form
#pragma unroll
  for (int i = 0; i < VEC; ++i)
    m[i] = __uint_as_float(__float_as_uint(psi_of_nat(fabsf(m[i]))) | (__float_as_uint(m[i]) & 0x80000000u));
  const int bc = v / P.p, cc = v - bc * P.p;
  unsigned e[DV];
  unsigned present = var_edges<DV, QC, TT, SJ>(P, a.var_tab, pmod(tf, T), (unsigned)pmod(tf / T, P.I) * (unsigned)P.E,
                                                v, bc, cc, e);
#pragma unroll
  for (int k = 0; k < DV; ++k)
    if ((present >> k) & 1u) vstore<VEC>(a.msg + (size_t)e[k] * P.gamma + q * VEC, m);
}

// fold the bit count of the frame the previous slot emitted into the lane counters
__device__ __forceinline__ void fold_prev(const SlotArgs& a, const CcParams& P, int t, int window, long long tid) {
  if (a.cnt && t >= window && tid < P.gamma) {
    const int g = (int)tid;
    const int b = a.cnt[g];
    a.cnt[P.gamma + g] += b;
    a.cnt[2 * P.gamma + g] += b > 0;
    a.cnt[g] = 0;
  }
}

// Also folds the previous slot's emitted-frame bit count into the lane counters.
template <int DV, int VEC, bool QC, int TT = 0, int SJ = 0>
__global__ void __launch_bounds__(CC_THREADS) entry_kernel(SlotArgs a, const __grid_constant__ CcParams P) {
  pdl_trigger();
  pdl_wait();
  const int t = slot_of(a);
  const int T = TT ? TT : P.lam;
  const unsigned GV = (unsigned)P.gamma / VEC;
  // 32-bit index math (the launchers keep the thread count < 2^31)
  const unsigned tid = blockIdx.x * blockDim.x + threadIdx.x;
  fold_prev(a, P, t, P.I * T, tid);
  if (tid >= (unsigned)P.c * GV) return;
  const int v = (int)(tid / GV), q = (int)(tid - (unsigned)v * GV);
  entry_body<DV, VEC, QC, TT, SJ>(a, P, t, a.mu_in, v, q);
}

// ---- check phase: processors i = 1..I refresh layer s = t - (i-1)T ---------
// TT, WW > 0: period and sub-block width known at compile time (QC grids of the
// common shapes) so the edge walk fully unrolls; 0 = runtime values.
template <int DC, int VEC, bool QC, int TT = 0, int WW = 0>
__global__ void __launch_bounds__(CC_THREADS) check_kernel(SlotArgs a, const __grid_constant__ CcParams P) {
  pdl_trigger();
  pdl_wait();
  const int t = slot_of(a);
  const int T = TT ? TT : P.lam;
  const unsigned GV = (unsigned)P.gamma / VEC, per = (unsigned)P.cb * GV;
  const unsigned tid = blockIdx.x * blockDim.x + threadIdx.x;
  if (a.fold_in_check) fold_prev(a, P, t, P.I * T, tid);
  if (tid >= (unsigned)a.nip * per) return;
  const unsigned ipl = tid / per;
  const int ip = a.ip0 + (int)ipl;
  const unsigned rem = tid - ipl * per;
  const int r = (int)(rem / GV), q = (int)(rem - (unsigned)r * GV);
  const int s = t - ip * T;
  if (s < 0) return;
  const int kap = pmod(s, T);
  float x[DC][VEC];
  if constexpr (TT > 0 && WW > 0 && QC) {
    // compile-time walk: edge k = d*WW + w sits at package base[d] + w, so
    // only TT base addresses stay live (registers -> occupancy)
    static_assert(TT * WW <= DC, "bucket too small");
    unsigned base[TT];
    unsigned present = 0;   // one bit per frame d
#pragma unroll
    for (int d = 0; d < TT; ++d) {
      const int f = s - (TT - 1) + d;
      int c2 = kap + 1 + d;
      c2 -= (c2 >= TT) ? TT : 0;
      c2 -= (c2 >= TT) ? TT : 0;
      base[d] = f >= 0 ? (unsigned)pmod(f / TT, P.I) * (unsigned)P.E + (unsigned)P.sub_off[kap * TT + c2] +
                             (unsigned)(r * WW) : 0u;
      present |= (f >= 0 ? 1u : 0u) << d;   // bootstrap: absent frames drop out (convolutional.py:276-279)
    }
#pragma unroll
    for (int d = 0; d < TT; ++d)
#pragma unroll
      for (int w = 0; w < WW; ++w)
        if ((present >> d) & 1u) vload<VEC>(a.msg + (size_t)(base[d] + w) * P.gamma + q * VEC, x[d * WW + w]);
    if (present == (1u << TT) - 1u) {
      cnu_core<DC, VEC, true, true>(x, TT * WW, (1u << VEC) - 1u);   // steady state
    } else {
      unsigned long long pm = 0;
#pragma unroll
      for (int d = 0; d < TT; ++d)
        if ((present >> d) & 1u) pm |= ((1ull << WW) - 1ull) << (d * WW);
      cnu_core_mask<DC, VEC>(x, pm);
    }
#pragma unroll
    for (int d = 0; d < TT; ++d)
#pragma unroll
      for (int w = 0; w < WW; ++w)
        if ((present >> d) & 1u) vstore<VEC>(a.msg + (size_t)(base[d] + w) * P.gamma + q * VEC, x[d * WW + w]);
    return;
  } else {
    const int W = QC ? P.sl : P.wmax;
    unsigned eidx[DC];   // package index (I*E < 2^32)
    unsigned long long present = 0;
    // walk d = 0..T-1 (frames s-ms+d, oldest first) and w = 0..W-1 incrementally
    int d = 0, w = 0;
    int f = s - P.ms;
    int lbl = kap * T + (kap + 1 < T ? kap + 1 : kap + 1 - T);
    unsigned base = f >= 0 ? (unsigned)pmod(f / T, P.I) * (unsigned)P.E + (unsigned)P.sub_off[lbl] : 0u;
#pragma unroll
    for (int k = 0; k < DC; ++k) {
      eidx[k] = 0;
      if (k < T * W) {
        if (f >= 0) {
          int loc;
          if constexpr (QC) loc = r * P.sl + w;
          else loc = a.check_tab[((size_t)lbl * P.cb + r) * P.wmax + w];
          if (loc >= 0) { eidx[k] = base + (unsigned)loc; present |= 1ull << k; }
        }
        if (++w == W) {
          w = 0; ++d; ++f;
          int c2 = kap + 1 + d;
          c2 -= (c2 >= T) ? T : 0;
          c2 -= (c2 >= T) ? T : 0;
          lbl = kap * T + c2;
          base = f >= 0 ? (unsigned)pmod(f / T, P.I) * (unsigned)P.E + (unsigned)P.sub_off[lbl] : 0u;
        }
      }
    }
#pragma unroll
    for (int k = 0; k < DC; ++k)
      if ((present >> k) & 1ull) vload<VEC>(a.msg + (size_t)eidx[k] * P.gamma + q * VEC, x[k]);
    const int deg = T * W;
    const unsigned long long full = deg >= 64 ? ~0ull : ((1ull << deg) - 1ull);
    if (present == full) cnu_core<DC, VEC, true, true>(x, deg, (1u << VEC) - 1u);
    else cnu_core_mask<DC, VEC>(x, present);
#pragma unroll
    for (int k = 0; k < DC; ++k)
      if ((present >> k) & 1ull) vstore<VEC>(a.msg + (size_t)eidx[k] * P.gamma + q * VEC, x[k]);
  }
}

// ---- variable phase: processors i = 1..I refresh frame j = t - iT + 1 ------
template <int DV, int VEC, bool QC, int TT = 0, int SJ = 0>
__global__ void __launch_bounds__(CC_THREADS) var_kernel(SlotArgs a, const __grid_constant__ CcParams P) {
  pdl_trigger();
  pdl_wait();
  const int t = slot_of(a);
  const int T = TT ? TT : P.lam;
  const unsigned GV = (unsigned)P.gamma / VEC, per = (unsigned)P.c * GV;
  const unsigned tid = blockIdx.x * blockDim.x + threadIdx.x;
  if (tid >= (unsigned)a.nip * per) return;
  const unsigned ipl = tid / per;
  const int ip = a.ip0 + (int)ipl;
  const unsigned rem = tid - ipl * per;
  const int v = (int)(rem / GV), q = (int)(rem - (unsigned)v * GV);
  const int j = t - (ip + 1) * T + 1;
  const bool enter = a.entry_next && ip + 1 == P.I;   // look-ahead entry of frame t + 1 (= j + window)
  if (j < 0) {
    if (enter) entry_body<DV, VEC, QC, TT, SJ>(a, P, t + 1, a.mu_next, v, q);
    return;
  }
  const int bc = v / P.p, cc = v - bc * P.p;
  unsigned e[DV];
  unsigned present = var_edges<DV, QC, TT, SJ>(P, a.var_tab, pmod(j, T), (unsigned)pmod(j / T, P.I) * (unsigned)P.E,
                                                v, bc, cc, e);
  float tot[VEC], am[DV][VEC];
  vload<VEC>(a.ring + ((size_t)pmod(j, P.I * T) * P.c + v) * P.gamma + q * VEC, tot);
#pragma unroll
  for (int k = 0; k < DV; ++k)
    if ((present >> k) & 1u) vload<VEC>(a.msg + (size_t)e[k] * P.gamma + q * VEC, am[k]);
#pragma unroll
  for (int k = 0; k < DV; ++k)
    if ((present >> k) & 1u) {
#pragma unroll
      for (int i = 0; i < VEC; ++i) tot[i] = __fadd_rn(tot[i], am[k][i]);
    }
  if (ip + 1 < P.I) {
#pragma unroll
    for (int k = 0; k < DV; ++k)
      if ((present >> k) & 1u) {
        float b[VEC];
        if constexpr (VEC % 2 == 0) {
          // lane pairs on the packed fp32 pipe (bit-identical to the scalar form)
#pragma unroll
          for (int i = 0; i < VEC; i += 2) {
            float d0, d1;
            get2(sub2(mk2(tot[i], tot[i + 1]), mk2(am[k][i], am[k][i + 1])), d0, d1);
            const float be0 = clampL(d0), be1 = clampL(d1);   // stored in phi form
            float q0, q1;
            get2(psi_of_nat2(mk2(fabsf(be0), fabsf(be1))), q0, q1);
            b[i] = __uint_as_float(__float_as_uint(q0) | (__float_as_uint(be0) & 0x80000000u));
            b[i + 1] = __uint_as_float(__float_as_uint(q1) | (__float_as_uint(be1) & 0x80000000u));
          }
        } else {
#pragma unroll
          for (int i = 0; i < VEC; ++i) {
            float beta = clampL(__fsub_rn(tot[i], am[k][i]));   // stored in phi form
            b[i] = __uint_as_float(__float_as_uint(psi_of_nat(fabsf(beta))) | (__float_as_uint(beta) & 0x80000000u));
          }
        }
        vstore<VEC>(a.msg + (size_t)e[k] * P.gamma + q * VEC, b);
      }
  } else {
    // processor I emits frame j (convolutional.py:319-327)
    float pst[VEC];
#pragma unroll
    for (int i = 0; i < VEC; ++i) pst[i] = clampL(tot[i]);
    if (a.post_out) vstore<VEC>(a.post_out + (size_t)v * P.gamma + q * VEC, pst);
    if (a.cnt) {
#pragma unroll
      for (int i = 0; i < VEC; ++i)
        if (pst[i] < 0.0f) atomicAdd(a.cnt + q * VEC + i, 1);
    }
    if (enter) entry_body<DV, VEC, QC, TT, SJ>(a, P, t + 1, a.mu_next, v, q);
  }
}

// fold the last emitted frame's bit count (end of a segment)
__global__ void fold_kernel(int32_t* cnt, int gamma) {
  int g = blockIdx.x * blockDim.x + threadIdx.x;
  if (g >= gamma) return;
  int b = cnt[g];
  cnt[gamma + g] += b;
  cnt[2 * gamma + g] += b > 0;
  cnt[g] = 0;
}

__global__ void advance_kernel(int64_t* t_dev, long long k) { *t_dev += k; }

// ---- dispatch ----------------------------------------------------------------
CcParams make_params(const cc_plan* pl, int I, int gamma) {
  CcParams P;
  std::memset(&P, 0, sizeof(P));
  P.lam = pl->lam; P.ms = pl->ms; P.sj = pl->sj; P.sl = pl->sl; P.c = pl->c; P.cb = pl->cb;
  P.p = pl->p; P.E = pl->E; P.wmax = pl->wmax; P.J = pl->J; P.L = pl->L;
  P.I = I; P.gamma = gamma;
  for (int i = 0; i < pl->lam * pl->lam; ++i) P.sub_off[i] = pl->sub_off[i];
  for (int i = 0; i < pl->J * pl->L; ++i) P.s[i] = (int16_t)pl->shifts[i];
  return P;
}

// lanes per thread: check pass float2 (register-heavy), entry / variable float4.
// From 8 lane vectors per row (gamma 32: a warp spans 4 variables' rows of
// 128 B): the per-thread index math (slot / processor / node decomposition,
// edge walk) is shared by VEC lanes, which is what bounds small-gamma slots
// (ncu at gamma 32, one lane per thread: 80% issue slots, 24% IMAD).
#ifndef CC_MIN_GV
#define CC_MIN_GV 8
#endif
inline int vec_for(int gamma, int want) {
  if (want >= 4 && gamma % 4 == 0 && gamma / 4 >= CC_MIN_GV) return 4;
  if (want >= 2 && gamma % 2 == 0 && gamma / 2 >= CC_MIN_GV) return 2;
  return 1;
}

inline bool fits32(long long threads) { return threads < (1ll << 31) - CC_THREADS; }

template <int DV, bool QC, int TT = 0, int SJ = 0>
void launch_entry(const CcParams& P, const SlotArgs& a, cudaStream_t s) {
  int vec = vec_for(P.gamma, 4);
  long long n = (long long)P.c * (P.gamma / vec);
  unsigned nb = blocks_for(std::max<long long>(n, P.gamma), CC_THREADS);
  if (vec == 4) launch_pdl(entry_kernel<DV, 4, QC, TT, SJ>, dim3(nb), CC_THREADS, s, a, P);
  else if (vec == 2) launch_pdl(entry_kernel<DV, 2, QC, TT, SJ>, dim3(nb), CC_THREADS, s, a, P);
  else launch_pdl(entry_kernel<DV, 1, QC, TT, SJ>, dim3(nb), CC_THREADS, s, a, P);
}
template <int DC, bool QC, int TT = 0, int WW = 0>
void launch_check(const CcParams& P, const SlotArgs& a, cudaStream_t s) {
  int vec = vec_for(P.gamma, DC > 24 ? 1 : 2);
  long long n = (long long)a.nip * P.cb * (P.gamma / vec);
  if (vec == 2) launch_pdl(check_kernel<DC, 2, QC, TT, WW>, dim3(blocks_for(n, CC_THREADS)), CC_THREADS, s, a, P);
  else launch_pdl(check_kernel<DC, 1, QC, TT, WW>, dim3(blocks_for(n, CC_THREADS)), CC_THREADS, s, a, P);
}
template <int DV, bool QC, int TT = 0, int SJ = 0>
void launch_var(const CcParams& P, const SlotArgs& a, cudaStream_t s) {
  int vec = vec_for(P.gamma, 4);
  long long n = (long long)a.nip * P.c * (P.gamma / vec);
  if (vec == 4) launch_pdl(var_kernel<DV, 4, QC, TT, SJ>, dim3(blocks_for(n, CC_THREADS)), CC_THREADS, s, a, P);
  else if (vec == 2) launch_pdl(var_kernel<DV, 2, QC, TT, SJ>, dim3(blocks_for(n, CC_THREADS)), CC_THREADS, s, a, P);
  else launch_pdl(var_kernel<DV, 1, QC, TT, SJ>, dim3(blocks_for(n, CC_THREADS)), CC_THREADS, s, a, P);
}

// parts: bit 0 = entry, bit 1 = check phase, bit 2 = variable phase (of the
// processors [a.ip0, a.ip0 + a.nip))
enum { SLOT_ENTRY = 1, SLOT_CHECK = 2, SLOT_VAR = 4, SLOT_ALL = 7 };

template <int DV, bool QC>
int launch_slot_dv(const CcParams& P, const SlotArgs& a, int dc, int parts, cudaStream_t s) {
  if constexpr (QC && DV == 4) {   // compile-time walks for the common unwrapped shapes
    if (P.lam == 4 && P.sj == 1 && P.sl == 6) {          // (4, 24) grids: codes A', 18360'
      if (parts & SLOT_ENTRY) launch_entry<4, true, 4, 1>(P, a, s);
      if (parts & SLOT_CHECK) launch_check<24, true, 4, 6>(P, a, s);
      if (parts & SLOT_VAR) launch_var<4, true, 4, 1>(P, a, s);
      return 0;
    }
    if (P.lam == 4 && P.sj == 1 && P.sl == 2) {          // (4, 8) grids
      if (parts & SLOT_ENTRY) launch_entry<4, true, 4, 1>(P, a, s);
      if (parts & SLOT_CHECK) launch_check<8, true, 4, 2>(P, a, s);
      if (parts & SLOT_VAR) launch_var<4, true, 4, 1>(P, a, s);
      return 0;
    }
  }
  if constexpr (QC && DV == 2) {
    if (P.lam == 2 && P.sj == 1 && P.sl == 2) {          // (2, 4) grids
      if (parts & SLOT_ENTRY) launch_entry<2, true, 2, 1>(P, a, s);
      if (parts & SLOT_CHECK) launch_check<4, true, 2, 2>(P, a, s);
      if (parts & SLOT_VAR) launch_var<2, true, 2, 1>(P, a, s);
      return 0;
    }
  }
  if (parts & SLOT_ENTRY) launch_entry<DV, QC>(P, a, s);
  if (parts & SLOT_CHECK) {
    if (dc <= 4) launch_check<4, QC>(P, a, s);
    else if (dc <= 8) launch_check<8, QC>(P, a, s);
    else if (dc <= 16) launch_check<16, QC>(P, a, s);
    else if (dc <= 24) launch_check<24, QC>(P, a, s);
    else if (dc <= 32) launch_check<32, QC>(P, a, s);
    else return fail_arg("LDPCCC check degree > 32 is not supported");
  }
  if (parts & SLOT_VAR) launch_var<DV, QC>(P, a, s);
  return 0;
}

template <bool QC>
int launch_slot(const CcParams& P, const SlotArgs& a, int dc, int dv, int parts, cudaStream_t s) {
  if (dv <= 2) return launch_slot_dv<2, QC>(P, a, dc, parts, s);
  if (dv <= 4) return launch_slot_dv<4, QC>(P, a, dc, parts, s);
  if (dv <= 8) return launch_slot_dv<8, QC>(P, a, dc, parts, s);
  return fail_arg("LDPCCC variable degree > 8 is not supported");
}

template <typename T>
int upload(const std::vector<T>& h, T** d) {
  *d = nullptr;
  if (h.empty()) return 0;
  if (cudaMalloc(d, h.size() * sizeof(T)) != cudaSuccess) { cudaGetLastError(); return fail_rt("cudaMalloc failed"); }
  if (cudaMemcpy(*d, h.data(), h.size() * sizeof(T), cudaMemcpyHostToDevice) != cudaSuccess) {
    cudaGetLastError();
    return fail_rt("cudaMemcpy failed");
  }
  return 0;
}

}  // namespace

extern "C" {

int cc_plan_create(const int64_t* shifts, int J, int L, int p, cc_plan** out) {
  if (!shifts || !out) return fail_arg("null argument");
  if (J < 1 || L < 1 || p < 1) return fail_arg("J, L, p must be positive");
  int lam = std::gcd(J, L);
  if (lam < 2)
    return fail_arg("gcd(J, L) = " + std::to_string(lam) +
                    ": the shift grid cannot be partitioned into a square sub-block grid, so there is nothing to unwrap");
  if (lam > CC_MAX_LAM || J * L > CC_MAX_SHIFTS) return fail_arg("shift grid too large for the LDPCCC kernels");
  for (int i = 0; i < J * L; ++i)
    if (shifts[i] < -1 || shifts[i] >= p) return fail_arg("shifts must lie in [-1, p-1]");
  auto* pl = new cc_plan();
  pl->J = J; pl->L = L; pl->p = p; pl->lam = lam; pl->ms = lam - 1;
  pl->sj = J / lam; pl->sl = L / lam; pl->c = pl->sl * p; pl->cb = pl->sj * p;
  pl->shifts.assign(shifts, shifts + (size_t)J * L);
  pl->all_live = std::all_of(pl->shifts.begin(), pl->shifts.end(), [](int64_t s) { return s >= 0; });
  const int nl = lam * lam;
  std::vector<int> cnt(nl, 0), wmax(nl, 0);
  auto sub = [&](int lbl, int br, int bc) {
    return shifts[(size_t)((lbl / lam) * pl->sj + br) * L + (lbl % lam) * pl->sl + bc];
  };
  int wm = 0;
  for (int b = 0; b < nl; ++b)
    for (int br = 0; br < pl->sj; ++br) {
      int w = 0;
      for (int bc = 0; bc < pl->sl; ++bc) w += sub(b, br, bc) >= 0;
      cnt[b] += w * p;
      wm = std::max(wm, w);
    }
  pl->wmax = std::max(wm, 1);
  int off = 0;
  for (int b = 0; b < nl; ++b) { pl->sub_off[b] = off; off += cnt[b]; }
  pl->E = off;
  // per-label tables (used only when some block is zero)
  std::vector<int32_t> ct((size_t)nl * pl->cb * pl->wmax, -1), vt((size_t)nl * pl->c * pl->sj, -1);
  for (int b = 0; b < nl; ++b) {
    std::vector<int> ptr(pl->cb + 1, 0);
    for (int r = 0; r < pl->cb; ++r) {
      int br = r / p, w = 0;
      for (int bc = 0; bc < pl->sl; ++bc) w += sub(b, br, bc) >= 0;
      ptr[r + 1] = ptr[r] + w;
    }
    for (int r = 0; r < pl->cb; ++r)
      for (int w = 0; w < ptr[r + 1] - ptr[r]; ++w) ct[((size_t)b * pl->cb + r) * pl->wmax + w] = ptr[r] + w;
    for (int br = 0; br < pl->sj; ++br) {
      std::vector<int> rank(pl->sl, -1);
      int k = 0;
      for (int bc = 0; bc < pl->sl; ++bc)
        if (sub(b, br, bc) >= 0) rank[bc] = k++;
      for (int v = 0; v < pl->c; ++v) {
        int bc = v / p, cc = v % p;
        int64_t s = sub(b, br, bc);
        if (s < 0) continue;
        int rr = (int)(((cc - s) % p + p) % p);
        vt[((size_t)b * pl->c + v) * pl->sj + br] = ptr[br * p + rr] + rank[bc];
      }
    }
  }
  int rc;
  if ((rc = upload(ct, &pl->d_check_tab)) || (rc = upload(vt, &pl->d_var_tab))) {
    cc_plan_destroy(pl);
    return rc;
  }
  *out = pl;
  return 0;
}

void cc_plan_destroy(cc_plan* pl) {
  if (!pl) return;
  cudaFree(pl->d_check_tab);
  cudaFree(pl->d_var_tab);
  delete pl;
}

int cc_plan_dims(const cc_plan* pl, int64_t* dims) {
  if (!pl || !dims) return fail_arg("null argument");
  dims[0] = pl->lam; dims[1] = pl->ms; dims[2] = pl->c; dims[3] = pl->cb;
  dims[4] = pl->E; dims[5] = pl->sj; dims[6] = pl->sl; dims[7] = pl->p;
  return 0;
}

int cc_slot_part(const cc_plan* pl, int I, int gamma, int64_t t, const int64_t* t_dev, float* msg, float* ring,
                 const float* mu_in, float* post_out, int32_t* lane_cnt, int ip0, int nip, int parts,
                 void* stream) {
  if (!pl || !msg || !ring) return fail_arg("null argument");
  if (I < 1) return fail_arg("need at least one processor");
  if (gamma <= 0 || gamma % 32) return fail_arg("gamma must be a positive multiple of 32");
  if (!t_dev && t < 0) return fail_arg("slot index must be non-negative");
  if (t > 0x3fffffff || t < -0x3fffffff) return fail_arg("slot index out of range");
  if (ip0 < 0 || nip < 0 || ip0 + nip > I || parts < 0 || parts > SLOT_ALL)
    return fail_arg("processor range / parts out of range");
  if (!fits32((long long)I * std::max(pl->c, pl->cb) * gamma)) return fail_arg("I x nodes x gamma too large for one launch");
  if (parts == 0 || (nip == 0 && !(parts & SLOT_ENTRY))) return 0;
  cudaStream_t s = as_stream(stream);
  CcParams P = make_params(pl, I, gamma);
  SlotArgs a{msg, ring, mu_in, post_out, lane_cnt, pl->d_check_tab, pl->d_var_tab, t_dev, (int)t, ip0, nip,
             nullptr, 0, 0};
  if (nip == 0) parts &= SLOT_ENTRY;
  const bool qc = pl->all_live;
  const int dc = pl->lam * (qc ? pl->sl : pl->wmax);
  const int dv = pl->lam * pl->sj;
  int rc = qc ? launch_slot<true>(P, a, dc, dv, parts, s) : launch_slot<false>(P, a, dc, dv, parts, s);
  if (rc) return rc;
  return check_launch("cc_slot");
}

int cc_slot(const cc_plan* pl, int I, int gamma, int64_t t, const int64_t* t_dev, float* msg, float* ring,
            const float* mu_in, float* post_out, int32_t* lane_cnt, void* stream) {
  return cc_slot_part(pl, I, gamma, t, t_dev, msg, ring, mu_in, post_out, lane_cnt, 0, I, SLOT_ALL, stream);
}

int cc_slot_ahead(const cc_plan* pl, int I, int gamma, int64_t t, const int64_t* t_dev, float* msg, float* ring,
                  const float* mu_next, int enter_next, float* post_out, int32_t* lane_cnt, void* stream) {
  if (!pl || !msg || !ring) return fail_arg("null argument");
  if (I < 1) return fail_arg("need at least one processor");
  if (gamma <= 0 || gamma % 32) return fail_arg("gamma must be a positive multiple of 32");
  if (!t_dev && t < 0) return fail_arg("slot index must be non-negative");
  if (t > 0x3fffffff || t < -0x3fffffff) return fail_arg("slot index out of range");
  if (!fits32((long long)I * std::max(pl->c, pl->cb) * gamma)) return fail_arg("I x nodes x gamma too large for one launch");
  cudaStream_t s = as_stream(stream);
  CcParams P = make_params(pl, I, gamma);
  SlotArgs a{msg, ring, nullptr, post_out, lane_cnt, pl->d_check_tab, pl->d_var_tab, t_dev, (int)t, 0, I,
             mu_next, 1, enter_next ? 1 : 0};
  const bool qc = pl->all_live;
  const int dc = pl->lam * (qc ? pl->sl : pl->wmax);
  const int dv = pl->lam * pl->sj;
  const int parts = SLOT_CHECK | SLOT_VAR;
  int rc = qc ? launch_slot<true>(P, a, dc, dv, parts, s) : launch_slot<false>(P, a, dc, dv, parts, s);
  if (rc) return rc;
  return check_launch("cc_slot_ahead");
}

int cc_fold(int32_t* lane_cnt, int gamma, void* stream) {
  if (!lane_cnt || gamma <= 0) return fail_arg("bad fold arguments");
  fold_kernel<<<blocks_for(gamma, CC_THREADS), CC_THREADS, 0, as_stream(stream)>>>(lane_cnt, gamma);
  return check_launch("cc_fold");
}

int cc_advance(int64_t* t_dev, int64_t k, void* stream) {
  if (!t_dev) return fail_arg("null argument");
  advance_kernel<<<1, 1, 0, as_stream(stream)>>>(t_dev, (long long)k);
  return check_launch("cc_advance");
}

}  // extern "C"

namespace qcb {
int launch_channel_t(uint64_t k0, uint64_t k1, uint64_t lane0, const uint64_t* lane0_dev, uint64_t start,
                     const int64_t* t_dev, long long t_add, long long t_mul, int n, int gamma, double sigma,
                     float* mu_vm, cudaStream_t s);
}

extern "C" int cc_channel(const cc_plan* pl, uint64_t seed_lo, uint64_t seed_hi, uint64_t lane0,
                          const uint64_t* lane0_dev, int64_t t, const int64_t* t_dev, int gamma, double sigma,
                          float* mu, void* stream) {
  if (!pl || !mu) return fail_arg("null argument");
  if (gamma <= 0 || gamma % 32) return fail_arg("gamma must be a positive multiple of 32");
  if (!t_dev && t < 0) return fail_arg("frame index must be non-negative");
  return launch_channel_t(seed_lo, seed_hi, lane0, lane0_dev, 0, t_dev, (long long)t, (long long)pl->c, pl->c,
                          gamma, sigma, mu, as_stream(stream));
}

extern "C" int cc_channel_frames(const cc_plan* pl, uint64_t seed_lo, uint64_t seed_hi, uint64_t lane0,
                                 const uint64_t* lane0_dev, int64_t t, int nframes, int gamma, double sigma,
                                 float* mu, void* stream) {
  if (!pl || !mu) return fail_arg("null argument");
  if (gamma <= 0 || gamma % 32) return fail_arg("gamma must be a positive multiple of 32");
  if (t < 0 || nframes < 1) return fail_arg("frame range must be non-negative and non-empty");
  if ((long long)nframes * pl->c > 0x7fffffffll) return fail_arg("too many frames for one channel launch");
  // frames t .. t + nframes - 1 are the contiguous positions [t c, (t + nframes) c)
  return launch_channel_t(seed_lo, seed_hi, lane0, lane0_dev, (uint64_t)t * (uint64_t)pl->c, nullptr, 0, 0,
                          nframes * pl->c, gamma, sigma, mu, as_stream(stream));
}
