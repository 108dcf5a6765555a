// Compact-check-state flooding schedule for regular QC codes (the production
// decode loop inside qc_decode, fixed iteration count).
//
// The reference alternates check_node_update / variable_node_update over one
// (E, gamma) package store (bp.py:134-188): the check pass reads and rewrites
// every package, the variable pass gathers them again -- 4E + N package
// transfers per iteration.  A check's outgoing messages are a function of two
// per-(check, lane) numbers and of each edge's own incoming message:
//     S   = sum_k psi_k            (psi = phi(|beta|)/ln2, the phi form), with
//           the sign parity par = XOR of the signs in its sign bit
//     S2  = S without its first maximum (accumulated directly: no cancellation)
//     alpha_k = sign(par ^ sign_k) * min(phi(psi_k > S - psi_k ? S2 : S - psi_k), cap)
// (an edge holding more than half of S is the unique maximum: it takes the
// exclusive sum S2; for every other edge S - psi_k >= S/2 >= psi_k, so the
// subtraction never cancels).  So the check pass writes only (S|par, S2) per
// check and lane (2 words instead of d_c packages), and the variable pass
// re-derives alpha_k from S|par and the package it is about to overwrite,
// reading S2 only for dominant edges (a few % of the edge-vectors): the record
// gathers -- 24 per record and iteration, half of the pass's L2 traffic -- stay
// at one field.  The arithmetic is the same instruction sequence as cnu_core +
// vnu_kernel (block_kernels.cuh), so results are bit-identical to the two-pass
// schedule; the package store traffic drops from 4E + N to 3E + N (+ 4M)
// words per lane and iteration.
//
// Thread mapping (both passes): lane-group major -- all rows (checks or
// variables) of lanes [g*LG, (g+1)*LG) before the next lane group, so the
// check records a variable pass gathers (24 reads per record) stay L2
// resident: LG = 128 lanes -> 3060 x 128 x 8 B = 3.1 MB for n18360.
#include <cstdlib>
#include <cstring>
#include <utility>

#include "block_kernels.cuh"

namespace qcb {

// check record fields per (check, lane): S|par (sum of psi, sign parity in the
// sign bit) and S2 (the sum without its first maximum)
constexpr int AGG_FIELDS = 2;

struct AggArgs {
  float* msgs;         // (E, gamma) phi-form var->check packages
  const float* mu;     // (N, gamma) channel LLRs
  float* agg;          // (M, AGG_FIELDS, gamma): S|par, S2
  float* post;         // (N, gamma) or null
  uint32_t* hb;        // (N, gamma/32) or null
  int rows, gamma;     // rows = M (check pass) or N (variable pass); gamma = row stride in lanes
  int q0;              // first lane vector of this pass's lane window
  int lg_gw;           // log2(lane vectors per group)
  int groups;          // lane groups in the window
  int reverse;         // visit lane groups last-to-first
  int rows_eff;        // rows the grid covers (rows / items per thread, rounded up)
  const uint32_t* active;   // early stop: lane mask words (gamma / 32) or null
  const uint32_t* active2;  // early stop: second mask ANDed in (active = act & bad on the fly) or null
  // compacted early-stop segments (es_compact.cu): *live lanes of the set are
  // packed at the front of both halves (half A holds (live + 1) / 2, half B
  // live / 2); the grid then walks only the lane groups holding them
  const int32_t* live;
  int live_half;            // 0: this window is half A, 1: half B
  int live_loop;            // 1: capped grid walking the live blocks (few live lanes);
                            // 0: full grid, CTAs past the live rows exit at once
};

// lane groups of this window that hold live lanes (live mode)
template <int VEC>
__device__ __forceinline__ unsigned live_groups(const AggArgs& a) {
  const int c = __ldg(a.live);     // read-only path: one L1 miss per SM, then hits
  const int n = a.live_half ? (c >> 1) : ((c + 1) >> 1);
  const int lpg = VEC << a.lg_gw;
  return (unsigned)min(a.groups, (n + lpg - 1) / lpg);
}


// 32-lane word of the early-stop mask holding lane g0 (all on without one)
__device__ __forceinline__ uint32_t es_word(const AggArgs& a, int g0) {
  if (!a.active) return 0xffffffffu;
  uint32_t w = a.active[g0 >> 5];
  if (a.active2) w &= a.active2[g0 >> 5];
  return w;
}

// lanes [g0, g0 + vec) of the early-stop mask
__device__ __forceinline__ unsigned es_lanes(const AggArgs& a, int g0, int vec) {
  return (es_word(a, g0) >> (g0 & 31)) & ((1u << vec) - 1u);
}

// early stop, per (variable n, lane vector q): the mask word, the vector's
// active lanes, and the hard bits its frozen lanes recorded at their freeze
// iteration (loaded up front with the item's other operands, only when some
// lane of the vector is frozen and some lane of the word is not)
struct EsLanes {
  uint32_t wmask;
  unsigned lanes, old;
};

template <int VEC>
__device__ __forceinline__ EsLanes es_begin(const AggArgs& a, int n, int q) {
  constexpr unsigned FULL = (1u << VEC) - 1u;
  EsLanes e;
  e.wmask = es_word(a, q * VEC);
  e.lanes = (e.wmask >> ((q * VEC) & 31)) & FULL;
  e.old = 0u;
  if (a.hb && e.lanes != FULL && e.wmask != 0u)
    e.old = (a.hb[(size_t)n * (a.gamma >> 5) + ((q * VEC) >> 5)] >> ((q * VEC) & 31)) & FULL & ~e.lanes;
  return e;
}

// the hard-bit word of variable n gets the active lanes' new bits and the
// frozen lanes' recorded ones; a word whose 32 lanes are all frozen is left
// untouched -- so the planes always hold every lane's result and the decode
// needs no final recompute from the posteriors
template <int VEC>
__device__ __forceinline__ void es_store_bits(const AggArgs& a, int n, int q, unsigned bits, const EsLanes& e) {
  store_bit_word<VEC>(a.hb + (size_t)n * (a.gamma >> 5), q, (bits & e.lanes) | e.old, e.wmask != 0u);
}

// min CTAs/SM for the variable job: 4 x 256 threads caps it at 64 registers,
// enough to issue all 17 loads of an item before its arithmetic (measured best
// on B200: 2 -> 88 regs / 16 warps is 15% slower, 5 -> 48 regs spills)
#ifndef AGG_THREADS
#define AGG_THREADS 128   // 128 > 64, 256 (+2.5%), 512 (profiles/r01/kbench_compact_threads.jsonl)
#endif
#ifndef AGG_VAR_MINB
#define AGG_VAR_MINB (1024 / AGG_THREADS)
#endif
#ifndef AGG_ES_MINB
#define AGG_ES_MINB 7   // early-stop variable / fused kernels: 72 registers, no spills (64: 40 B stack; +1-3%)
#endif

// AGG_ES: early stop (bp.py:242-256): frozen lanes keep their packages and
// posteriors; post and hard bits are written every iteration for live lanes
enum AggFlags { AGG_FIRST = AGG_FIRST_FLAG, AGG_LAST = AGG_LAST_FLAG, AGG_ES = 4 };

// Programmatic dependent launch (sm_90+): each compact-schedule kernel lets the
// next one in the stream be scheduled immediately and waits for its
// predecessor's results only right before its first dependent load, so the
// launch latency and index math of kernel k+1 overlap the tail of kernel k.
// block (bx within its lane group, group index) + thread -> (row, lane vector q).
// Lane-group major: every row of one group of lanes before the next group.
// ngroups: groups the reversed order runs over (a.groups, or the live ones of a
// compacted segment: then the groups written last are still visited first)
__device__ __forceinline__ bool agg_map(const AggArgs& a, unsigned bx, unsigned grp, int& row, int& q,
                                        int ngroups) {
  const unsigned idx = bx * AGG_THREADS + threadIdx.x;
  row = (int)(idx >> a.lg_gw);
  if (row >= a.rows_eff) return false;
  const int g = a.reverse ? ngroups - 1 - (int)grp : (int)grp;
  q = a.q0 + (g << a.lg_gw) + (int)(idx & ((1u << a.lg_gw) - 1u));
  return true;
}

template <int DC, int VEC, bool FROM_MU>
__device__ __forceinline__ void check_body(const AggArgs& a, const QcGrid& grid, int m, int q) {
  if (a.active && es_lanes(a, q * VEC, VEC) == 0) return;   // frozen lanes keep stale records
  int jrow = 0, r = 0;
  if constexpr (FROM_MU) {
    jrow = div_p(grid, m);
    r = m - jrow * grid.p;
  }
  float x[DC][VEC];
#pragma unroll
  for (int k = 0; k < DC; ++k) {
    if constexpr (FROM_MU) {
      int c = r + grid.s[jrow * grid.L + k];
      c -= (c >= grid.p) ? grid.p : 0;
      vload<VEC>(a.mu + (size_t)(k * grid.p + c) * a.gamma + q * VEC, x[k]);
    } else {
      vload<VEC>(a.msgs + (size_t)(m * DC + k) * a.gamma + q * VEC, x[k]);
    }
  }
  float oS[VEC], oS2[VEC];
  if constexpr (VEC % 2 == 0 && !FROM_MU) {
    // lane pairs: the two running sums on the packed fp32 pipe (each lane
    // rounded exactly like the scalar form below; compares / selects per lane)
#pragma unroll
    for (int i = 0; i < VEC; i += 2) {
      unsigned par0 = 0, par1 = 0;
      f2 S = splat2(0.0f), S2 = splat2(0.0f);
      float mx0 = -1.0f, mx1 = -1.0f;
#pragma unroll
      for (int k = 0; k < DC; ++k) {
        const unsigned u0 = __float_as_uint(x[k][i]), u1 = __float_as_uint(x[k][i + 1]);
        const float f0 = __uint_as_float(u0 & 0x7fffffffu), f1 = __uint_as_float(u1 & 0x7fffffffu);
        par0 ^= u0;
        par1 ^= u1;
        const f2 fp = mk2(f0, f1);
        float s0, s1, a0, a1;
        get2(S, s0, s1);
        get2(add2(S2, fp), a0, a1);
        S2 = mk2((f0 > mx0) ? s0 : a0, (f1 > mx1) ? s1 : a1);
        mx0 = fmaxf(mx0, f0);
        mx1 = fmaxf(mx1, f1);
        S = add2(S, fp);
      }
      float s0, s1, t0, t1;
      get2(S, s0, s1);
      get2(S2, t0, t1);
      oS[i] = __uint_as_float(__float_as_uint(s0) | (par0 & 0x80000000u));
      oS[i + 1] = __uint_as_float(__float_as_uint(s1) | (par1 & 0x80000000u));
      oS2[i] = t0;
      oS2[i + 1] = t1;
    }
  } else {
#pragma unroll
    for (int i = 0; i < VEC; ++i) {
      unsigned par = 0;
      float S = 0.0f, S2 = 0.0f, mx = -1.0f;
#pragma unroll
      for (int k = 0; k < DC; ++k) {
        float b = x[k][i];
        unsigned sb = __float_as_uint(b) & 0x80000000u;
        float f = FROM_MU ? psi_of_nat(fabsf(b)) : fabsf(b);
        par ^= sb;
        S2 = (f > mx) ? S : __fadd_rn(S2, f);
        mx = fmaxf(mx, f);
        S = __fadd_rn(S, f);
      }
      oS[i] = __uint_as_float(__float_as_uint(S) | par);
      oS2[i] = S2;
    }
  }
  float* rec = a.agg + (size_t)m * AGG_FIELDS * a.gamma + q * VEC;
  vstore<VEC>(rec, oS);
  vstore<VEC>(rec + a.gamma, oS2);
}

// check-record rows of variable n (block column l, circulant row c)
template <int DV>
__device__ __forceinline__ int var_rows(const QcGrid& grid, int n, int (&mrow)[DV]) {
  const int l = div_p(grid, n), c = n - l * grid.p;
#pragma unroll
  for (int j = 0; j < DV; ++j) {
    int rr = c - grid.s[j * grid.L + l];
    rr += (rr < 0) ? grid.p : 0;
    mrow[j] = j * grid.p + rr;
  }
  return l;
}

template <int DV, int VEC, int FLAGS>
__device__ __forceinline__ void var_compute(const AggArgs& a, const QcGrid& grid, int n, int q, int l,
                                            const int (&mrow)[DV], float (&tot)[VEC], float (&v2c)[DV][VEC],
                                            const float (&sS)[DV][VEC], const EsLanes& es);

template <int DV, int VEC, int FLAGS>
__device__ __forceinline__ void var_body(const AggArgs& a, const QcGrid& grid, int n, int q) {
  EsLanes es{0xffffffffu, (1u << VEC) - 1u, 0u};
  if constexpr ((FLAGS & AGG_ES) != 0) {
    es = es_begin<VEC>(a, n, q);
    if (es.lanes == 0) {   // every lane of the vector frozen
      if (a.hb) es_store_bits<VEC>(a, n, q, 0u, es);
      return;
    }
  }
  int mrow[DV];
  const int l = var_rows<DV>(grid, n, mrow);
  float tot[VEC], v2c[DV][VEC];
  vload<VEC>(a.mu + (size_t)n * a.gamma + q * VEC, tot);
  if constexpr (!(FLAGS & AGG_FIRST)) {
#pragma unroll
    for (int j = 0; j < DV; ++j)
      vload<VEC>(a.msgs + ((size_t)mrow[j] * grid.L + l) * a.gamma + q * VEC, v2c[j]);
  }
  // every load of the item is issued before any arithmetic (one memory round
  // trip per item; the compiler otherwise interleaves them with the phi math);
  // of the check records only S|par -- S2 is fetched for dominant edges only
  float sS[DV][VEC];
#pragma unroll
  for (int j = 0; j < DV; ++j) vload<VEC>(a.agg + (size_t)mrow[j] * AGG_FIELDS * a.gamma + q * VEC, sS[j]);
  var_compute<DV, VEC, FLAGS>(a, grid, n, q, l, mrow, tot, v2c, sS, es);
}

// |alpha_k| arguments of edge j for the VEC lanes: mag = S - psi_k, except for
// the dominant edge (psi_k > S - psi_k: it holds more than half the sum, so it
// is the unique maximum), whose exclusive sum S2 comes from the record's second
// field -- loaded only when some lane of the vector needs it (a few % of the
// edge-vectors), which keeps the 24-fold record gathers at one field.
template <int VEC>
__device__ __forceinline__ void edge_mags(const AggArgs& a, int mrow_j, int q, const float (&v2c_j)[VEC],
                                          const float (&sS_j)[VEC], float (&mag)[VEC]) {
  unsigned dom = 0;
  if constexpr (VEC % 2 == 0) {
#pragma unroll
    for (int i = 0; i < VEC; i += 2) {
      const float f0 = fabsf(v2c_j[i]), f1 = fabsf(v2c_j[i + 1]);
      get2(sub2(mk2(fabsf(sS_j[i]), fabsf(sS_j[i + 1])), mk2(f0, f1)), mag[i], mag[i + 1]);
      dom |= ((f0 > mag[i]) ? 1u : 0u) << i;
      dom |= ((f1 > mag[i + 1]) ? 1u : 0u) << (i + 1);
    }
  } else {
#pragma unroll
    for (int i = 0; i < VEC; ++i) {
      const float f = fabsf(v2c_j[i]);
      mag[i] = __fsub_rn(fabsf(sS_j[i]), f);
      dom |= ((f > mag[i]) ? 1u : 0u) << i;
    }
  }
  if (dom) {
    float s2[VEC];
    vload<VEC>(a.agg + ((size_t)mrow_j * AGG_FIELDS + 1) * a.gamma + q * VEC, s2);
#pragma unroll
    for (int i = 0; i < VEC; ++i)
      if ((dom >> i) & 1u) mag[i] = s2[i];
  }
}

template <int DV, int VEC, int FLAGS>
__device__ __forceinline__ void var_compute(const AggArgs& a, const QcGrid& grid, int n, int q, int l,
                                            const int (&mrow)[DV], float (&tot)[VEC], float (&v2c)[DV][VEC],
                                            const float (&sS)[DV][VEC], const EsLanes& es) {
  float al[DV][VEC];
  if constexpr (FLAGS & AGG_FIRST) {
    // beta^0 = mu on every edge, in the phi form the fused-init check pass saw
#pragma unroll
    for (int i = 0; i < VEC; ++i) {
      float p0 = __uint_as_float(__float_as_uint(psi_of_nat(fabsf(tot[i]))) |
                                 (__float_as_uint(tot[i]) & 0x80000000u));
#pragma unroll
      for (int j = 0; j < DV; ++j) v2c[j][i] = p0;
    }
  }
  {
    if constexpr (VEC % 2 == 0) {
      // lane pairs on the packed fp32 pipe: bit-identical to the scalar path below
#pragma unroll
      for (int j = 0; j < DV; ++j) {
        float mag[VEC];
        edge_mags<VEC>(a, mrow[j], q, v2c[j], sS[j], mag);
#pragma unroll
        for (int i = 0; i < VEC; i += 2) {
          const unsigned u0 = __float_as_uint(v2c[j][i]), u1 = __float_as_uint(v2c[j][i + 1]);
          const unsigned s0 = __float_as_uint(sS[j][i]), s1 = __float_as_uint(sS[j][i + 1]);
          float p0, p1;
          get2(phi_of_log2_2(mk2(mag[i], mag[i + 1])), p0, p1);
          al[j][i] = __uint_as_float(__float_as_uint(fminf(p0, ALPHA_CAP)) | ((u0 ^ s0) & 0x80000000u));
          al[j][i + 1] = __uint_as_float(__float_as_uint(fminf(p1, ALPHA_CAP)) | ((u1 ^ s1) & 0x80000000u));
        }
      }
      // running total in increasing edge order (bp.py:179-181)
#pragma unroll
      for (int i = 0; i < VEC; i += 2) {
        f2 t = mk2(tot[i], tot[i + 1]);
#pragma unroll
        for (int j = 0; j < DV; ++j) t = add2(t, mk2(al[j][i], al[j][i + 1]));
        get2(t, tot[i], tot[i + 1]);
      }
    } else {
#pragma unroll
      for (int j = 0; j < DV; ++j) {
        float mag[VEC];
        edge_mags<VEC>(a, mrow[j], q, v2c[j], sS[j], mag);
#pragma unroll
        for (int i = 0; i < VEC; ++i) {
          const unsigned u = __float_as_uint(v2c[j][i]), sp = __float_as_uint(sS[j][i]);
          const float al_ = fminf(phi_of_log2(mag[i]), ALPHA_CAP);
          al[j][i] = __uint_as_float(__float_as_uint(al_) | ((u ^ sp) & 0x80000000u));
        }
      }
      // running total in increasing edge order (bp.py:179-181)
#pragma unroll
      for (int j = 0; j < DV; ++j)
#pragma unroll
        for (int i = 0; i < VEC; ++i) tot[i] = __fadd_rn(tot[i], al[j][i]);
    }
  }
  const unsigned lanes = es.lanes;
  if constexpr (!(FLAGS & AGG_LAST)) {
#pragma unroll
    for (int j = 0; j < DV; ++j) {
      float b[VEC];
      if constexpr (VEC % 2 == 0) {
#pragma unroll
        for (int i = 0; i < VEC; i += 2) {
          float d0, d1;
          get2(sub2(mk2(tot[i], tot[i + 1]), mk2(al[j][i], al[j][i + 1])), d0, d1);
          // psi(|clip(beta, +-L_MAX)|) with beta's sign (clipping never flips a sign)
          float q0, q1;
          get2(psi_of_nat_fast2(mk2(fminf(fabsf(d0), L_MAX), fminf(fabsf(d1), L_MAX))), q0, q1);
          b[i] = __uint_as_float(__float_as_uint(q0) | (__float_as_uint(d0) & 0x80000000u));
          b[i + 1] = __uint_as_float(__float_as_uint(q1) | (__float_as_uint(d1) & 0x80000000u));
        }
      } else {
#pragma unroll
        for (int i = 0; i < VEC; ++i) {
          const float d = __fsub_rn(tot[i], al[j][i]);
          b[i] = __uint_as_float(__float_as_uint(psi_of_nat_fast(fminf(fabsf(d), L_MAX))) |
                                 (__float_as_uint(d) & 0x80000000u));
        }
      }
      float* dst = a.msgs + ((size_t)mrow[j] * grid.L + l) * a.gamma + q * VEC;
      if constexpr ((FLAGS & AGG_ES) != 0) {
        // frozen lanes keep their packages: a partially frozen vector stores its
        // active lanes one by one (no need to keep the old packages live)
        if (lanes != (1u << VEC) - 1u) {
#pragma unroll
          for (int i = 0; i < VEC; ++i)
            if ((lanes >> i) & 1u) dst[i] = b[i];
          continue;
        }
      }
      vstore<VEC>(dst, b);
    }
  }
  if constexpr ((FLAGS & (AGG_LAST | AGG_ES)) != 0) {
    float pst[VEC];
    unsigned bits = 0;
#pragma unroll
    for (int i = 0; i < VEC; ++i) {
      pst[i] = clampL(tot[i]);
      bits |= (pst[i] < 0.0f ? 1u : 0u) << i;
    }
    if (a.post) {
      if (lanes == (1u << VEC) - 1u) {
        vstore<VEC>(a.post + (size_t)n * a.gamma + q * VEC, pst);
      } else {
#pragma unroll
        for (int i = 0; i < VEC; ++i)
          if ((lanes >> i) & 1u) a.post[(size_t)n * a.gamma + q * VEC + i] = pst[i];
      }
    }
    // whole warps share one row (gw >= 32), so the shuffle is safe
    if constexpr ((FLAGS & AGG_ES) != 0) {
      if (a.hb) es_store_bits<VEC>(a, n, q, bits, es);
    } else {
      if (a.hb) store_bit_word<VEC>(a.hb + (size_t)n * (a.gamma >> 5), q, bits, true);
    }
  }
}

// L2 prefetch of an item's HBM operands (its LLR row and d_v packages); the
// check records are L2-resident already
template <int DV, int VEC, int FLAGS>
__device__ __forceinline__ void var_prefetch(const AggArgs& a, const QcGrid& grid, int n, int q) {
  const int l = div_p(grid, n), c = n - l * grid.p;
  asm volatile("prefetch.global.L2 [%0];" ::"l"(a.mu + (size_t)n * a.gamma + q * VEC));
  if constexpr (!(FLAGS & AGG_FIRST)) {
#pragma unroll
    for (int j = 0; j < DV; ++j) {
      int rr = c - grid.s[j * grid.L + l];
      rr += (rr < 0) ? grid.p : 0;
      asm volatile("prefetch.global.L2 [%0];" ::"l"(a.msgs + ((size_t)(j * grid.p + rr) * grid.L + l) * a.gamma +
                                                       q * VEC));
    }
  }
}

// ITEMS rows per thread (n, n + rows_eff, ...): the next item's operands are
// prefetched into L2 before the current one's arithmetic
template <int DV, int VEC, int FLAGS, int ITEMS>
__device__ __forceinline__ void var_items(const AggArgs& a, const QcGrid& grid, int n, int q) {
  bool pf = true;
  if constexpr ((FLAGS & AGG_ES) != 0) pf = es_lanes(a, q * VEC, VEC) != 0;   // frozen vectors fetch nothing
#pragma unroll 1
  for (int k = 0; k < ITEMS; ++k) {
    const int nk = n + k * a.rows_eff;
    if (nk >= a.rows) break;                                   // warp-uniform (one row per warp)
    if (pf && k + 1 < ITEMS && nk + a.rows_eff < a.rows) var_prefetch<DV, VEC, FLAGS>(a, grid, nk + a.rows_eff, q);
    var_body<DV, VEC, FLAGS>(a, grid, nk, q);
  }
}

// grid = (blocks per lane group, groups)
template <int DC, int VEC, bool FROM_MU>
__global__ void __launch_bounds__(AGG_THREADS) agg_check_kernel(AggArgs a, const __grid_constant__ QcGrid grid) {
  pdl_trigger();
  int m, q;
  unsigned ng = a.groups;
  if (a.live) {             // compacted segment, full grid: the lane count was written before it started
    ng = live_groups<VEC>(a);
    if (blockIdx.y >= ng) return;
  }
  const bool on = agg_map(a, blockIdx.x, blockIdx.y, m, q, ng);
  pdl_wait();
  if (on) check_body<DC, VEC, FROM_MU>(a, grid, m, q);
}

// Live mode (compacted early-stop segments, es_compact.cu): a capped grid whose
// CTAs walk only the virtual blocks of the live lane groups.  Separate kernels,
// so the loop's register needs never touch the fixed-iteration path (inlined
// into it, the loop made the 64-register fused kernel spill 152 B).
#ifndef AGG_LIVE_WAVES
#define AGG_LIVE_WAVES 2
#endif
#ifndef AGG_LIVE_MINB
#define AGG_LIVE_MINB 6   // 80 registers: the loop kernels do not spill (1-3% over 64 registers with spills)
#endif
constexpr unsigned LIVE_CTAS = 148 * 8 * AGG_LIVE_WAVES;

template <int DC, int VEC>
__global__ void __launch_bounds__(AGG_THREADS) agg_check_live_kernel(AggArgs a, const __grid_constant__ QcGrid grid) {
  pdl_trigger();
  pdl_wait();
  const unsigned bpg = (unsigned)((((long long)a.rows_eff << a.lg_gw) + AGG_THREADS - 1) / AGG_THREADS);
  const unsigned lg = live_groups<VEC>(a), nv = lg * bpg;
#pragma unroll 1
  for (unsigned v = blockIdx.x; v < nv; v += gridDim.x) {
    const unsigned g = v / bpg;
    int m, q;
    if (agg_map(a, v - g * bpg, g, m, q, lg)) check_body<DC, VEC, false>(a, grid, m, q);
  }
}

template <int DV, int VEC, int FLAGS, int ITEMS>
__global__ void __launch_bounds__(AGG_THREADS, (FLAGS & AGG_ES) ? AGG_ES_MINB : AGG_VAR_MINB) agg_var_kernel(AggArgs a, const __grid_constant__ QcGrid grid) {
  pdl_trigger();
  int n, q;
  unsigned ng = a.groups;
  if (a.live) {
    ng = live_groups<VEC>(a);
    if (blockIdx.y >= ng) return;
  }
  const bool on = agg_map(a, blockIdx.x, blockIdx.y, n, q, ng);
  pdl_wait();
  if (on) var_items<DV, VEC, FLAGS, ITEMS>(a, grid, n, q);
}

template <int DV, int VEC, int FLAGS, int ITEMS>
__global__ void __launch_bounds__(AGG_THREADS, AGG_LIVE_MINB) agg_var_live_kernel(AggArgs a, const __grid_constant__ QcGrid grid) {
  pdl_trigger();
  pdl_wait();
  const unsigned bpg = (unsigned)((((long long)a.rows_eff << a.lg_gw) + AGG_THREADS - 1) / AGG_THREADS);
  const unsigned lg = live_groups<VEC>(a), nv = lg * bpg;
#pragma unroll 1
  for (unsigned v = blockIdx.x; v < nv; v += gridDim.x) {
    const unsigned g = v / bpg;
    int n, q;
    if (agg_map(a, v - g * bpg, g, n, q, lg)) var_items<DV, VEC, FLAGS, ITEMS>(a, grid, n, q);
  }
}

// Early stop folded into the fused launches (bp.py:242-256).  Per-lane state,
// word-indexed over the whole gamma, double-buffered by iteration parity:
//   act[t & 1]  active_t = lanes still iterating after iteration t,
//   bad[t & 1]  syndrome failures of iteration t (atomicOr),
// so active_t = active_{t-1} & bad_t.  Launch 2t-1 = V(A, t) + C(B, t) +
// S(B, t-1) + U(A, t); launch 2t = V(B, t) + C(A, t+1) + S(A, t) + U(B, t):
//   V(X, t)   variable job masked by active_{t-1} = act[t&1] & bad[(t-1)&1]
//             (both written by earlier launches; computed on the fly);
//   C(X, t+1) check job masked by active_{t-1} (one iteration stale: records of
//             lanes that froze at t are computed but never used);
//   S(X, t)   syndrome of X's hard-bit planes written by V(X, t) in the
//             previous launch -> bad[t&1] (skips words with no active lane);
//   U(X, t)   one CTA: act[(t-1)&1] = active_{t-1}, iters_run = t-1 for the
//             lanes that froze at t-1, clears bad[t&1] for S(X, t).
// No launch beyond the fixed schedule's: the per-iteration syndrome / freeze
// kernels of the two-pass early stop disappear.
struct EsFused {
  // S: syndrome of lane words [s_w0, s_w0 + s_W) into s_bad
  const uint32_t* hb;        // (N, Wt) hard-bit planes
  uint32_t* s_bad;
  const uint32_t* s_act;     // skip words with no active lane (null: none skipped)
  int s_w0, s_W, Wt, nbs;    // nbs = S blocks (0: no syndrome job)
  // U: state update of lane words [u_w0, u_w0 + u_W); u_it = t (iteration of the V in this launch)
  uint32_t* u_act_out;       // act[(t-1)&1]
  const uint32_t* u_act_in;  // act[t&1]     (null at t = 1: every lane active)
  const uint32_t* u_bad_in;  // bad[(t-1)&1]
  uint32_t* u_bad_clr;       // bad[t&1]
  int32_t* iters_run;
  int u_w0, u_W, u_it, u_iters;   // u_W = 0: no update job
};

// One launch, two independent jobs on disjoint lane windows: the variable pass
// of window v (compute-heavy: 2 phi per edge-lane) and the check pass of window
// c (pure streaming).  Grid (R + 1, extra + nbc): after the `extra` leading
// rows (early stop: the syndrome blocks and the one state-update block, which
// only depend on earlier launches), x = 0..R-1 are variable blocks y*R + x and
// x = R is check block y, so the block scheduler interleaves the two kinds and
// every SM mixes MUFU-bound and HBM-bound CTAs.
struct FusedArgs {
  AggArgs v, c;
  unsigned R, nbv, nbc;                     // variable blocks per row of the grid, total; check rows
  unsigned es_rows;                         // leading grid rows of early-stop blocks
  unsigned v_bpg, c_bpg;                    // blocks per lane group
  unsigned long long v_magic, c_magic;      // ceil(2^40 / bpg)
  EsFused es;
};

__device__ __forceinline__ unsigned div_magic(unsigned x, unsigned long long m) {
  return (unsigned)(((unsigned long long)x * m) >> 40);
}

// parity of check m over its d_c variables' hard bits, 32 lanes per word
// AGG_SYN_K consecutive checks per thread, their failures OR-ed into one
// atomic (K-fold fewer syndrome CTAs and atomics per launch)
#ifndef AGG_SYN_K
#define AGG_SYN_K 8   // 1 -> 8: early-stop decode -0.7-1.4% (3.2 / 3.6 dB, gamma 4096)
#endif
__host__ __device__ __forceinline__ int es_syn_rows(int M) { return (M + AGG_SYN_K - 1) / AGG_SYN_K; }

template <int DC>
__device__ __forceinline__ void es_syndrome_block(const EsFused& e, const QcGrid& grid, unsigned blk, int M) {
  const long long idx = (long long)blk * AGG_THREADS + threadIdx.x;
  if (idx >= (long long)es_syn_rows(M) * e.s_W) return;
  const int mb = (int)(idx / e.s_W), w = e.s_w0 + (int)(idx - (long long)mb * e.s_W);
  if (e.s_act && e.s_act[w] == 0u) return;
  uint32_t acc = 0;
  const int m0 = mb * AGG_SYN_K, m1 = min(M, m0 + AGG_SYN_K);
#pragma unroll 2
  for (int m = m0; m < m1; ++m) {
    const int j = div_p(grid, m), r = m - j * grid.p;
    uint32_t par = 0;
#pragma unroll
    for (int k = 0; k < DC; ++k) {
      int c = r + grid.s[j * grid.L + k];
      c -= (c >= grid.p) ? grid.p : 0;
      par ^= e.hb[(size_t)(k * grid.p + c) * e.Wt + w];
    }
    acc |= par;
  }
  if (acc) atomicOr(e.s_bad + w, acc);
}

__device__ __forceinline__ void es_update_block(const EsFused& e) {
  for (int i = threadIdx.x; i < e.u_W; i += AGG_THREADS) {
    const int w = e.u_w0 + i;
    uint32_t act;
    if (e.u_act_in) {
      const uint32_t prev = e.u_act_in[w];
      act = prev & e.u_bad_in[w];
      const uint32_t froze = prev & ~act;
      for (uint32_t f = froze; f; f &= f - 1) e.iters_run[w * 32 + __ffs(f) - 1] = e.u_it - 1;
    } else {
      act = 0xffffffffu;
#pragma unroll 4
      for (int b = 0; b < 32; ++b) e.iters_run[w * 32 + b] = e.u_iters;
    }
    e.u_act_out[w] = act;
    e.u_bad_clr[w] = 0u;
  }
}

// one block (bx, by) of the fused grid; gv / gc: lane groups the variable /
// check job visits (all, or the live ones of a compacted segment)
template <int DC, int DV, int VC, int VV, bool FROM_MU, int FLAGS, int ITEMS>
__device__ __forceinline__ void fused_block(const FusedArgs& f, const QcGrid& grid, unsigned bx, unsigned by,
                                            unsigned gv, unsigned gc) {
  int row, q;
  if (by < f.es_rows) {                      // early-stop bookkeeping blocks, scheduled first
    const unsigned e = by * (f.R + 1) + bx;
    if (e < (unsigned)f.es.nbs) es_syndrome_block<DC>(f.es, grid, e, f.c.rows);
    else if (e == (unsigned)f.es.nbs && f.es.u_W > 0) es_update_block(f.es);
    return;
  }
  const unsigned y = by - f.es_rows;
  if (bx == f.R) {
    const unsigned b = y, g = div_magic(b, f.c_magic);
    if (g < gc && agg_map(f.c, b - g * f.c_bpg, g, row, q, min(gc, (unsigned)f.c.groups)))
      check_body<DC, VC, FROM_MU>(f.c, grid, row, q);
  } else {
    const unsigned b = y * f.R + bx;
    if (b >= f.nbv) return;
    const unsigned g = div_magic(b, f.v_magic);
    if (g < gv && agg_map(f.v, b - g * f.v_bpg, g, row, q, min(gv, (unsigned)f.v.groups)))
      var_items<DV, VV, FLAGS, ITEMS>(f.v, grid, row, q);
  }
}

template <int DC, int DV, int VC, int VV, bool FROM_MU, int FLAGS, int ITEMS>
__global__ void __launch_bounds__(AGG_THREADS, (FLAGS & AGG_ES) ? AGG_ES_MINB : AGG_VAR_MINB) agg_fused_kernel(FusedArgs f, const __grid_constant__ QcGrid grid) {
  pdl_trigger();
  if (f.v.live) {           // compacted segment, full grid: rows past the live lane groups exit at once
    const unsigned gv = live_groups<VV>(f.v), gc = live_groups<VC>(f.c);
    const unsigned rows = f.es_rows + max(gc * f.c_bpg, (gv * f.v_bpg + f.R - 1) / f.R);
    if (blockIdx.y >= rows) return;
    pdl_wait();
    fused_block<DC, DV, VC, VV, FROM_MU, FLAGS, ITEMS>(f, grid, blockIdx.x, blockIdx.y, gv, gc);
    return;
  }
  pdl_wait();
  fused_block<DC, DV, VC, VV, FROM_MU, FLAGS, ITEMS>(f, grid, blockIdx.x, blockIdx.y, 0xffffffffu, 0xffffffffu);
}

// live mode: grid rows that hold live lane groups only, walked by a capped grid
template <int DC, int DV, int VC, int VV, int FLAGS, int ITEMS>
__global__ void __launch_bounds__(AGG_THREADS, AGG_LIVE_MINB) agg_fused_live_kernel(FusedArgs f, const __grid_constant__ QcGrid grid) {
  pdl_trigger();
  pdl_wait();
  const unsigned gv = live_groups<VV>(f.v), gc = live_groups<VC>(f.c);
  const unsigned rows = f.es_rows + max(gc * f.c_bpg, (gv * f.v_bpg + f.R - 1) / f.R);
  const unsigned nv = rows * (f.R + 1);
#pragma unroll 1
  for (unsigned v = blockIdx.y * gridDim.x + blockIdx.x; v < nv; v += gridDim.x * gridDim.y)
    fused_block<DC, DV, VC, VV, false, FLAGS, ITEMS>(f, grid, v % (f.R + 1), v / (f.R + 1), gv, gc);
}

namespace {

int env_int(const char* name, int dflt);

template <typename... KArgs, typename... Args>
void launch_k(void (*kern)(KArgs...), dim3 grid, cudaStream_t s, Args... args) {
  launch_pdl(kern, grid, AGG_THREADS, s, args...);
}

int env_int(const char* name, int dflt) {
  const char* e = std::getenv(name);
  return e ? std::atoi(e) : dflt;
}

int agg_mode() {
  // 0 = the two-pass reference schedule inside qc_decode: the A/B oracle of the
  // bit-identity tests (tests/test_gpu_block.py), not a tuning knob
  static int v = env_int("QCB_AGG", 1);
  return v;
}

// Measured optimum of the compact schedule on B200 (profiles/r01/kbench_compact_*.jsonl):
constexpr int AGG_LANE_GROUP = 128;   // lanes per lane group (check-record L2 working set)
constexpr int AGG_REVERSE = 1;        // variable job visits lane groups last-to-first
constexpr int AGG_VV = 4;             // lanes per thread of the standalone variable job
#ifndef AGG_ITEMS_N
#define AGG_ITEMS_N 1
#endif
// rows per variable thread: with one-field record gathers, 1 row (no
// loop-carried state, no spills) is as fast as 2 rows with an L2 prefetch of the
// second on the fixed decode and 15% faster on the early-stop one
// (profiles/r02/kbench_items_minb.md)
constexpr int AGG_ITEMS = AGG_ITEMS_N;

constexpr int AGG_FVC = 4;            // lanes per thread of the fused check job (+2.4% over 2)

bool dc_supported(int dc) { return dc == 4 || dc == 6 || dc == 8 || dc == 12 || dc == 16 || dc == 24 || dc == 32; }
bool dv_supported(int dv) { return dv >= 2 && dv <= 4; }

int pick_lg_gw(int gamma, int vec);
int pick_vec(int gamma) { return gamma % 128 == 0 ? 4 : (gamma % 64 == 0 ? 2 : 1); }

// Small batches (gamma < 128) on the fixed-iteration passes: up to `want` lanes
// per thread from AGG_MIN_GV lane vectors per row (gamma 32: a warp spans 2
// rows), so the per-thread index math and record gathers are shared by several
// lanes -- the LDPCCC slots' fix for the same bound (stream.cu, vec_for).  The
// hard-bit shuffles then run over 32 / VEC-thread groups of one row: rows whose
// warps are partially out of range would leave the full-warp shuffle short, so
// the variable pass takes it only when the row count divides evenly.
#ifndef AGG_MIN_GV
#define AGG_MIN_GV 16      // gamma 32: 2 lanes per thread (2 rows per warp) beat 4 (4 rows per warp)
#endif
#ifndef AGG_SMALL_VC
#define AGG_SMALL_VC 4     // lanes per thread, small-batch check pass
#endif
#ifndef AGG_SMALL_VV
#define AGG_SMALL_VV 4     // lanes per thread, small-batch variable pass
#endif
int pick_vec_small(int lanes, int want, int rows) {
  for (int v = want; v > 1; v >>= 1) {
    const int gv = lanes / v;
    if (lanes % v || gv < AGG_MIN_GV || (gv >= 32 && gv % 32)) continue;   // lane groups must tile the row
    const int rows_per_warp = 32 / std::min(32, 1 << pick_lg_gw(lanes, v));
    if (rows % rows_per_warp == 0) return v;
  }
  return 1;
}
int pick_vec_var(int gamma) { return std::min(pick_vec(gamma), AGG_VV); }

// log2 of the lane vectors per group: the largest power of two <= LG/VEC that
// divides GV = gamma/VEC (GV is a multiple of 32 for every vec pick_vec returns)
int pick_lg_gw(int gamma, int vec) {
  int GV = gamma / vec, target = std::max(32, AGG_LANE_GROUP / vec), lg = 5;
  if (GV < 32) {              // small batches (pick_vec_small): several rows per warp
    lg = 0;
    while (GV % (2 << lg) == 0 && (2 << lg) <= GV) ++lg;
    return lg;
  }
  while ((2 << lg) <= target && GV % (2 << lg) == 0) ++lg;
  return lg;
}

unsigned blocks_per_group(const AggArgs& a) {
  return (unsigned)((((long long)a.rows_eff << a.lg_gw) + AGG_THREADS - 1) / AGG_THREADS);
}

dim3 agg_grid(const AggArgs& a, int) {
  return dim3(blocks_per_group(a), (unsigned)a.groups, 1);
}

// pass arguments over the lane window [lane0, lane0 + lanes) of a gamma-wide store
AggArgs make_args(float* msgs, const float* mu, float* agg, float* post, uint32_t* hb, int rows, int gamma,
                  int lane0, int lanes, int vec, int reverse) {
  AggArgs a{msgs, mu, agg, post, hb, rows, gamma, lane0 / vec, pick_lg_gw(lanes, vec), 0, reverse, rows,
            nullptr, nullptr};
  a.groups = (lanes / vec) >> a.lg_gw;
  return a;
}

dim3 live_grid(const AggArgs& a) {
  return dim3(std::min(blocks_per_group(a) * (unsigned)a.groups, LIVE_CTAS), 1, 1);
}

template <int DC, int VEC>
void launch_check_v(const AggArgs& a, bool from_mu, const QcGrid& g, cudaStream_t s) {
  dim3 nb = agg_grid(a, VEC);
  if (a.live && a.live_loop) launch_k(agg_check_live_kernel<DC, VEC>, live_grid(a), s, a, g);   // never from mu
  else if (from_mu) launch_k(agg_check_kernel<DC, VEC, true>, nb, s, a, g);
  else launch_k(agg_check_kernel<DC, VEC, false>, nb, s, a, g);
}

template <int DC>
void launch_check_dc(const AggArgs& a, int vec, bool from_mu, const QcGrid& g, cudaStream_t s) {
  switch (vec) {
    case 4: launch_check_v<DC, 4>(a, from_mu, g, s); break;
    case 2: launch_check_v<DC, 2>(a, from_mu, g, s); break;
    default: launch_check_v<DC, 1>(a, from_mu, g, s);
  }
}

template <int DV, int VEC, int ITEMS>
int launch_var_i(const AggArgs& a, int flags, const QcGrid& g, cudaStream_t s) {
  dim3 nb = agg_grid(a, VEC);
  if (a.live && a.live_loop) {        // compacted early-stop segment: its last variable pass
    if (flags == AGG_ES) launch_k(agg_var_live_kernel<DV, VEC, AGG_ES, ITEMS>, live_grid(a), s, a, g);
    else if (flags == (AGG_ES | AGG_LAST))
      launch_k(agg_var_live_kernel<DV, VEC, AGG_ES | AGG_LAST, ITEMS>, live_grid(a), s, a, g);
    else return fail_arg("live variable pass: unsupported flags");
    return 0;
  }
  switch (flags) {
    case 0: launch_k(agg_var_kernel<DV, VEC, 0, ITEMS>, nb, s, a, g); break;
    case AGG_FIRST: launch_k(agg_var_kernel<DV, VEC, AGG_FIRST, ITEMS>, nb, s, a, g); break;
    case AGG_LAST: launch_k(agg_var_kernel<DV, VEC, AGG_LAST, ITEMS>, nb, s, a, g); break;
    case AGG_FIRST | AGG_LAST: launch_k(agg_var_kernel<DV, VEC, AGG_FIRST | AGG_LAST, ITEMS>, nb, s, a, g); break;
    case AGG_ES: launch_k(agg_var_kernel<DV, VEC, AGG_ES, ITEMS>, nb, s, a, g); break;
    case AGG_ES | AGG_LAST: launch_k(agg_var_kernel<DV, VEC, AGG_ES | AGG_LAST, ITEMS>, nb, s, a, g); break;
    case AGG_ES | AGG_FIRST | AGG_LAST:
      launch_k(agg_var_kernel<DV, VEC, AGG_ES | AGG_FIRST | AGG_LAST, ITEMS>, nb, s, a, g);
      break;
    default: return fail_arg("compact variable pass: unsupported flags");
  }
  return 0;
}

template <int DV, int VEC>
int launch_var_v(AggArgs a, int flags, const QcGrid& g, cudaStream_t s) {
  a.rows_eff = (a.rows + AGG_ITEMS - 1) / AGG_ITEMS;      // standalone variable pass: AGG_ITEMS rows per thread
  return launch_var_i<DV, VEC, AGG_ITEMS>(a, flags, g, s);
}

template <int DV>
int launch_var_dv(const AggArgs& a, int vec, int flags, const QcGrid& g, cudaStream_t s) {
  switch (vec) {
    case 4: return launch_var_v<DV, 4>(a, flags, g, s);
    case 2: return launch_var_v<DV, 2>(a, flags, g, s);
    default: return launch_var_v<DV, 1>(a, flags, g, s);
  }
}

#ifndef AGG_FUSED_VV
#define AGG_FUSED_VV 4      // lanes per thread of the fused variable job (2: -12%, kbench_fused_vv_items.jsonl)
#endif

template <int DC, int DV, int VC, bool FROM_MU, int FLAGS>
void launch_fused_t(const FusedArgs& f, dim3 grid, const QcGrid& g, cudaStream_t s) {
  launch_k(agg_fused_kernel<DC, DV, VC, AGG_FUSED_VV, FROM_MU, FLAGS, AGG_ITEMS>, grid, s, f, g);
}

template <int DC, int DV, int VC>
int launch_fused_v(const FusedArgs& f, dim3 grid, bool from_mu, int flags, const QcGrid& g, cudaStream_t s) {
  if (f.v.live && f.v.live_loop) {      // compacted early-stop segment (never the first iteration)
    const dim3 lg(f.R + 1, std::min(grid.y, (LIVE_CTAS + f.R) / (f.R + 1)), 1);
    if (!from_mu && flags == AGG_ES)
      launch_k(agg_fused_live_kernel<DC, DV, VC, AGG_FUSED_VV, AGG_ES, AGG_ITEMS>, lg, s, f, g);
    else if (!from_mu && flags == (AGG_ES | AGG_LAST))
      launch_k(agg_fused_live_kernel<DC, DV, VC, AGG_FUSED_VV, AGG_ES | AGG_LAST, AGG_ITEMS>, lg, s, f, g);
    else return fail_arg("live fused pass: unsupported (from_mu, flags) combination");
    return 0;
  }
  if (from_mu && flags == AGG_FIRST) launch_fused_t<DC, DV, VC, true, AGG_FIRST>(f, grid, g, s);
  else if (from_mu && flags == (AGG_FIRST | AGG_LAST)) launch_fused_t<DC, DV, VC, true, AGG_FIRST | AGG_LAST>(f, grid, g, s);
  else if (!from_mu && flags == AGG_FIRST) launch_fused_t<DC, DV, VC, false, AGG_FIRST>(f, grid, g, s);
  else if (!from_mu && flags == 0) launch_fused_t<DC, DV, VC, false, 0>(f, grid, g, s);
  else if (!from_mu && flags == AGG_LAST) launch_fused_t<DC, DV, VC, false, AGG_LAST>(f, grid, g, s);
  else if (from_mu && flags == (AGG_ES | AGG_FIRST)) launch_fused_t<DC, DV, VC, true, AGG_ES | AGG_FIRST>(f, grid, g, s);
  else if (from_mu && flags == (AGG_ES | AGG_FIRST | AGG_LAST))
    launch_fused_t<DC, DV, VC, true, AGG_ES | AGG_FIRST | AGG_LAST>(f, grid, g, s);
  else if (!from_mu && flags == (AGG_ES | AGG_FIRST)) launch_fused_t<DC, DV, VC, false, AGG_ES | AGG_FIRST>(f, grid, g, s);
  else if (!from_mu && flags == AGG_ES) launch_fused_t<DC, DV, VC, false, AGG_ES>(f, grid, g, s);
  else if (!from_mu && flags == (AGG_ES | AGG_LAST)) launch_fused_t<DC, DV, VC, false, AGG_ES | AGG_LAST>(f, grid, g, s);
  else return fail_arg("fused compact pass: unsupported (from_mu, flags) combination");
  return 0;
}

template <int DC, int DV>
int launch_fused_dc(const FusedArgs& f, dim3 grid, bool from_mu, int flags, const QcGrid& g, cudaStream_t s) {
  return launch_fused_v<DC, DV, AGG_FVC>(f, grid, from_mu, flags, g, s);
}

unsigned long long magic40(unsigned d) { return ((1ull << 40) + d - 1) / d; }

}  // namespace

bool agg_fused_eligible(const qc_plan* p, int gamma) {
  return agg_eligible(p) && gamma % 256 == 0 &&
         ((p->L == 24 && p->J == 4) || (p->L == 4 && p->J == 2));
}

int launch_agg_fused_es(const qc_plan* p, int gamma, int lanes, int v0, int flags, int c0, bool from_mu,
                        float* msgs, const float* mu, float* agg, float* post, uint32_t* hb,
                        const uint32_t* v_act, const uint32_t* v_act2, const uint32_t* c_act, const EsFused* es,
                        cudaStream_t s, const int32_t* live = nullptr, int live_loop = 0);

// variable pass on lanes [v0, v0 + lanes) fused with the check pass on lanes [c0, c0 + lanes)
int launch_agg_fused(const qc_plan* p, int gamma, int lanes, int v0, int flags, int c0, bool from_mu, float* msgs,
                     const float* mu, float* agg, float* post, uint32_t* hb, cudaStream_t s) {
  return launch_agg_fused_es(p, gamma, lanes, v0, flags, c0, from_mu, msgs, mu, agg, post, hb, nullptr, nullptr,
                             nullptr, nullptr, s);
}

int launch_agg_fused_es(const qc_plan* p, int gamma, int lanes, int v0, int flags, int c0, bool from_mu,
                        float* msgs, const float* mu, float* agg, float* post, uint32_t* hb,
                        const uint32_t* v_act, const uint32_t* v_act2, const uint32_t* c_act, const EsFused* es,
                        cudaStream_t s, const int32_t* live, int live_loop) {
  FusedArgs f;
  f.v = make_args(msgs, mu, agg, post, hb, p->N, gamma, v0, lanes, AGG_FUSED_VV, AGG_REVERSE);
  f.v.rows_eff = (f.v.rows + AGG_ITEMS - 1) / AGG_ITEMS;
  f.c = make_args(msgs, mu, agg, nullptr, nullptr, p->M, gamma, c0, lanes, AGG_FVC, 0);
  f.v.active = v_act;
  f.v.active2 = v_act2;
  f.c.active = c_act;
  f.v.live = f.c.live = live;
  f.v.live_loop = f.c.live_loop = live_loop;
  f.v.live_half = v0 >= gamma / 2;
  f.c.live_half = c0 >= gamma / 2;
  f.v_bpg = blocks_per_group(f.v);
  f.c_bpg = blocks_per_group(f.c);
  f.v_magic = magic40(f.v_bpg);
  f.c_magic = magic40(f.c_bpg);
  f.nbv = f.v_bpg * f.v.groups;
  f.nbc = f.c_bpg * f.c.groups;
  f.R = (f.nbv + f.nbc - 1) / f.nbc;
  std::memset(&f.es, 0, sizeof(f.es));
  unsigned extra = 0;
  if (es) {
    f.es = *es;
    f.es.nbs = es->s_W > 0 ? (int)(((long long)es_syn_rows(p->M) * es->s_W + AGG_THREADS - 1) / AGG_THREADS) : 0;
    const unsigned jobs = (unsigned)f.es.nbs + (es->u_W > 0 ? 1u : 0u);
    extra = (jobs + f.R) / (f.R + 1);
  }
  f.es_rows = extra;
  const dim3 grid(f.R + 1, f.nbc + extra, 1);
  const QcGrid g = make_grid(p);
  int rc = (p->L == 24) ? launch_fused_dc<24, 4>(f, grid, from_mu, flags, g, s)
                        : launch_fused_dc<4, 2>(f, grid, from_mu, flags, g, s);
  if (rc) return rc;
  return check_launch("agg_fused");
}

// single passes over a lane window (active, active2: early-stop masks ANDed)
int launch_agg_check_w(const qc_plan* p, int gamma, int lane0, int lanes, bool from_mu, float* msgs,
                       const float* mu, float* agg, cudaStream_t s, const uint32_t* active = nullptr,
                       const int32_t* live = nullptr, int live_loop = 0);
int launch_agg_var_w(const qc_plan* p, int gamma, int lane0, int lanes, int flags, float* msgs, const float* mu,
                     const float* agg, float* post, uint32_t* hb, cudaStream_t s, const uint32_t* active = nullptr,
                     const uint32_t* active2 = nullptr, const int32_t* live = nullptr, int live_loop = 0);

bool agg_eligible(const qc_plan* p) {
  return agg_mode() != 0 && p && p->qc_regular && p->E > 0 && dc_supported(p->L) && dv_supported(p->J) &&
         p->check_regular == p->L;
}

size_t agg_words(const qc_plan* p, int gamma) {
  return agg_eligible(p) ? (size_t)AGG_FIELDS * p->M * (size_t)(gamma > 0 ? gamma : 0) : 0;
}

int launch_agg_check(const qc_plan* p, int gamma, bool from_mu, float* msgs, const float* mu, float* agg,
                     cudaStream_t s) {
  return launch_agg_check_w(p, gamma, 0, gamma, from_mu, msgs, mu, agg, s);
}

int launch_agg_check_w(const qc_plan* p, int gamma, int lane0, int lanes, bool from_mu, float* msgs,
                       const float* mu, float* agg, cudaStream_t s, const uint32_t* active, const int32_t* live,
                       int live_loop) {
  int vec = pick_vec(lanes);
  if (lanes < 128 && !active && !live) vec = std::max(vec, pick_vec_small(lanes, AGG_SMALL_VC, p->M));
  AggArgs a = make_args(msgs, mu, agg, nullptr, nullptr, p->M, gamma, lane0, lanes, vec, 0);
  a.active = active;
  a.live = live;
  a.live_loop = live_loop;
  a.live_half = lane0 >= gamma / 2;
  const QcGrid g = make_grid(p);
  switch (p->L) {
    case 4: launch_check_dc<4>(a, vec, from_mu, g, s); break;
    case 6: launch_check_dc<6>(a, vec, from_mu, g, s); break;
    case 8: launch_check_dc<8>(a, vec, from_mu, g, s); break;
    case 12: launch_check_dc<12>(a, vec, from_mu, g, s); break;
    case 16: launch_check_dc<16>(a, vec, from_mu, g, s); break;
    case 24: launch_check_dc<24>(a, vec, from_mu, g, s); break;
    case 32: launch_check_dc<32>(a, vec, from_mu, g, s); break;
    default: return fail_arg("compact schedule: unsupported check degree");
  }
  return check_launch("agg_check");
}

int launch_agg_var(const qc_plan* p, int gamma, int flags, float* msgs, const float* mu, const float* agg,
                   float* post, uint32_t* hb, cudaStream_t s) {
  return launch_agg_var_w(p, gamma, 0, gamma, flags, msgs, mu, agg, post, hb, s);
}

int launch_agg_var_w(const qc_plan* p, int gamma, int lane0, int lanes, int flags, float* msgs, const float* mu,
                     const float* agg, float* post, uint32_t* hb, cudaStream_t s, const uint32_t* active,
                     const uint32_t* active2, const int32_t* live, int live_loop) {
  int vec = pick_vec_var(lanes);
  if (lanes < 128 && !(flags & AGG_ES) && !active && !live) vec = std::max(vec, pick_vec_small(lanes, AGG_SMALL_VV, p->N));
  AggArgs a = make_args(msgs, mu, const_cast<float*>(agg), post, hb, p->N, gamma, lane0, lanes, vec,
                        AGG_REVERSE);
  a.active = active;
  a.active2 = active2;
  a.live = live;
  a.live_loop = live_loop;
  a.live_half = lane0 >= gamma / 2;
  const QcGrid g = make_grid(p);
  int rc;
  switch (p->J) {
    case 2: rc = launch_var_dv<2>(a, vec, flags, g, s); break;
    case 3: rc = launch_var_dv<3>(a, vec, flags, g, s); break;
    case 4: rc = launch_var_dv<4>(a, vec, flags, g, s); break;
    default: return fail_arg("compact schedule: unsupported variable degree");
  }
  if (rc) return rc;
  return check_launch("agg_var");
}

// The whole fixed-iteration flooding loop on the compact schedule.  With the
// fused kernel the lanes split into halves A and B that run half an iteration
// apart: launch k is var(X, t) + check(Y, t') so every launch mixes the
// compute-heavy variable job of one half with the streaming check job of the
// other (2 iters + 1 launches).  Bit-identical to the unfused passes.
int run_agg_tile(const qc_plan* p, int gamma, int lane0, int lanes, int iters, float* msgs, const float* mu,
                 float* agg, float* post, uint32_t* hb, cudaStream_t s);

int run_agg_decode(const qc_plan* p, int gamma, int iters, float* msgs, const float* mu, float* agg, float* post,
                   uint32_t* hb, cudaStream_t s) {
  return run_agg_tile(p, gamma, 0, gamma, iters, msgs, mu, agg, post, hb, s);
}

int run_agg_tile(const qc_plan* p, int gamma, int lane0, int lanes, int iters, float* msgs, const float* mu,
                 float* agg, float* post, uint32_t* hb, cudaStream_t s) {
  int rc;
  if (!agg_fused_eligible(p, lanes)) {
    for (int it = 1; it <= iters; ++it) {
      if ((rc = launch_agg_check_w(p, gamma, lane0, lanes, it == 1, msgs, mu, agg, s))) return rc;
      int flags = (it == 1 ? AGG_FIRST : 0) | (it == iters ? AGG_LAST : 0);
      if ((rc = launch_agg_var_w(p, gamma, lane0, lanes, flags, msgs, mu, agg, it == iters ? post : nullptr,
                                 it == iters ? hb : nullptr, s)))
        return rc;
    }
    return 0;
  }
  const int H = lanes / 2, A = lane0, B = lane0 + H;
  if ((rc = launch_agg_check_w(p, gamma, A, H, true, msgs, mu, agg, s))) return rc;
  for (int t = 1; t <= iters; ++t) {
    const int vflags = (t == 1 ? AGG_FIRST : 0) | (t == iters ? AGG_LAST : 0);
    float* po = t == iters ? post : nullptr;
    uint32_t* ho = t == iters ? hb : nullptr;
    // var(A, t) + check(B, t)
    if ((rc = launch_agg_fused(p, gamma, H, A, vflags, B, t == 1, msgs, mu, agg, po, ho, s))) return rc;
    if (t < iters) {
      // var(B, t) + check(A, t + 1)
      if ((rc = launch_agg_fused(p, gamma, H, B, vflags, A, false, msgs, mu, agg, po, ho, s))) return rc;
    } else if ((rc = launch_agg_var_w(p, gamma, B, H, vflags, msgs, mu, agg, po, ho, s))) {
      return rc;
    }
  }
  return 0;
}

// Early-stop decode (bp.py:242-256) on the compact schedule with the syndrome
// and freeze folded into the fused launches (EsFused above): the same
// 2 iters + 1 launches as the fixed decode, plus a 2-launch tail (last
// syndrome, ok / iteration counts).
// Frozen lanes keep packages and posteriors; decisions, posteriors and
// iteration counts equal the two-pass early-stop decode bit for bit
// (tests/test_gpu_block.py::test_compact_early_stop_is_bit_identical).
// es = act[0] | act[1] | bad[0] | bad[1] | bad_fin, gamma/32 words each.
bool agg_es_eligible(const qc_plan* p, int gamma) { return agg_fused_eligible(p, gamma); }

int launch_es_tail(const qc_plan* p, int gamma, int iters, uint32_t* const act[2], uint32_t* const bad[2],
                   uint32_t* bad_fin, uint8_t* ok, int32_t* iters_run, const float* post, uint32_t* hb,
                   cudaStream_t s);

// Iterations [t0, t1] of the compact early-stop decode (t1 <= iters).  t0 == 1:
// the decode's start (fused init, every lane active).  t0 > 1: a continuation
// on a compacted lane set (es_compact.cu) whose active mask is already in
// act[t0 & 1], with bad[(t0-1) & 1] = all ones and bad[t0 & 1] = bad_fin = 0,
// so active_{t0-1} = act & bad is that mask; iters_run holds `iters` there.
// The segment ends with the variable pass of half B at t1 (packages written
// unless t1 == iters: the last beta is never read).
int run_agg_es_segment(const qc_plan* p, int gamma, int t0, int t1, int iters, float* msgs, const float* mu,
                       float* agg, float* post, uint32_t* hb, uint32_t* es_words, int32_t* iters_run,
                       cudaStream_t s, const int32_t* live, int live_loop) {
  const int W = gamma / 32, H = gamma / 2, A = 0, B = H, WH = W / 2;
  uint32_t* act[2] = {es_words, es_words + W};
  uint32_t* bad[2] = {es_words + 2 * W, es_words + 3 * W};
  const bool fresh = t0 == 1;
  int rc;
  if ((rc = launch_agg_check_w(p, gamma, A, H, fresh, msgs, mu, agg, s, fresh ? nullptr : act[t0 & 1], live,
                               live_loop)))
    return rc;
  auto es_for = [&](int t, int vw0, int sw0, bool syn) {
    EsFused e{};
    e.hb = hb;
    e.Wt = W;
    if (syn) {                       // S(Y, t') of the half whose V ran in the previous launch
      const int tp = (sw0 == A / 32) ? t : t - 1;    // A's syndrome lags one launch: iteration t; B's: t - 1
      e.s_bad = bad[tp & 1];
      e.s_act = act[(tp - 1) & 1];
      e.s_w0 = sw0;
      e.s_W = WH;
    }
    e.u_act_out = act[(t - 1) & 1];
    e.u_act_in = t == 1 ? nullptr : act[t & 1];
    e.u_bad_in = bad[(t - 1) & 1];
    e.u_bad_clr = bad[t & 1];
    e.iters_run = iters_run;
    e.u_w0 = vw0;
    e.u_W = WH;
    e.u_it = t;
    e.u_iters = iters;
    return e;
  };
  for (int t = t0; t <= t1; ++t) {
    const int vflags = AGG_ES | (t == 1 ? AGG_FIRST : 0) | (t == iters ? AGG_LAST : 0);
    const uint32_t* vm = t == 1 ? nullptr : act[t & 1];        // active_{t-1} = act[t&1] & bad[(t-1)&1]
    const uint32_t* vm2 = t == 1 ? nullptr : bad[(t - 1) & 1];
    // V(A, t) + C(B, t) + S(B, t-1) + U(A, t); C(B, t) masked by active_{t-2}(B) = act[t&1]
    // (a continuation's first launch skips S(B, t0-1): bad[(t0-1)&1] is preset)
    EsFused e1 = es_for(t, A / 32, B / 32, t > t0);
    if ((rc = launch_agg_fused_es(p, gamma, H, A, vflags, B, t == 1, msgs, mu, agg, post, hb, vm, vm2,
                                  (fresh && t <= 2) ? nullptr : act[t & 1], &e1, s, live, live_loop)))
      return rc;
    // V(B, t) + C(A, t+1) + S(A, t) + U(B, t); C(A, t+1) masked by active_{t-1}(A) = act[(t-1)&1]
    EsFused e2 = es_for(t, B / 32, A / 32, true);
    if (t < t1) {
      if ((rc = launch_agg_fused_es(p, gamma, H, B, vflags, A, false, msgs, mu, agg, post, hb, vm, vm2,
                                    act[(t - 1) & 1], &e2, s, live, live_loop)))
        return rc;
    } else if ((rc = launch_agg_var_w(p, gamma, B, H, vflags, msgs, mu, agg, post, hb, s, vm, vm2, live,
                                      live_loop))) {
      return rc;
    }
  }
  return 0;
}

int run_agg_decode_es(const qc_plan* p, int gamma, int iters, float* msgs, const float* mu, float* agg, float* post,
                      uint32_t* hb, uint32_t* es_words, uint8_t* ok, int32_t* iters_run, cudaStream_t s) {
  const int W = gamma / 32;
  uint32_t* act[2] = {es_words, es_words + W};
  uint32_t* bad[2] = {es_words + 2 * W, es_words + 3 * W};
  uint32_t* bad_fin = es_words + 4 * W;
  cudaMemsetAsync(bad_fin, 0, sizeof(uint32_t) * W, s);
  if (int rc = run_agg_es_segment(p, gamma, 1, iters, iters, msgs, mu, agg, post, hb, es_words, iters_run, s,
                                  nullptr, 0))
    return rc;
  return launch_es_tail(p, gamma, iters, act, bad, bad_fin, ok, iters_run, post, hb, s);
}

int agg_decode_launches(const qc_plan* p, int gamma, int iters) {
  return agg_fused_eligible(p, gamma) ? 2 * iters + 1 : 2 * iters;
}

}  // namespace qcb

// ============================================================================
// C ABI: the two passes of the compact schedule on their own (tests, benches)
// ============================================================================
extern "C" {

int qc_agg_check(const qc_plan* p, int gamma, int from_mu, float* msgs, const float* mu, float* agg,
                 void* stream) {
  if (!p || !agg || (from_mu ? !mu : !msgs)) return qcb::fail_arg("null argument");
  if (gamma <= 0 || gamma % 32) return qcb::fail_arg("gamma must be a positive multiple of 32");
  if (!qcb::agg_eligible(p)) return qcb::fail_arg("compact schedule needs a regular QC plan");
  return qcb::launch_agg_check(p, gamma, from_mu != 0, msgs, mu, agg, qcb::as_stream(stream));
}

int qc_agg_var(const qc_plan* p, int gamma, int flags, float* msgs, const float* mu, const float* agg,
               float* post, uint32_t* hb, void* stream) {
  if (!p || !agg || !mu || !msgs) return qcb::fail_arg("null argument");
  if (gamma <= 0 || gamma % 32) return qcb::fail_arg("gamma must be a positive multiple of 32");
  if (flags < 0 || flags > 3) return qcb::fail_arg("flags: 1 = first iteration, 2 = last iteration");
  if (!qcb::agg_eligible(p)) return qcb::fail_arg("compact schedule needs a regular QC plan");
  return qcb::launch_agg_var(p, gamma, flags, msgs, mu, agg, post, hb, qcb::as_stream(stream));
}

int qc_agg_fused(const qc_plan* p, int gamma, int lanes, int var_lane0, int var_flags, int check_lane0,
                 int check_from_mu, float* msgs, const float* mu, float* agg, float* post, uint32_t* hb,
                 void* stream) {
  if (!p || !agg || !mu || !msgs) return qcb::fail_arg("null argument");
  if (gamma <= 0 || gamma % 256) return qcb::fail_arg("fused compact pass: gamma must be a multiple of 256");
  if (lanes <= 0 || lanes % 128 || var_lane0 % 128 || check_lane0 % 128 || var_lane0 < 0 || check_lane0 < 0 ||
      var_lane0 + lanes > gamma || check_lane0 + lanes > gamma)
    return qcb::fail_arg("fused compact pass: lane windows must be 128-lane aligned and inside gamma");
  if (!qcb::agg_fused_eligible(p, gamma)) return qcb::fail_arg("fused compact pass: unsupported plan");
  return qcb::launch_agg_fused(p, gamma, lanes, var_lane0, var_flags, check_lane0, check_from_mu != 0, msgs, mu,
                               agg, post, hb, qcb::as_stream(stream));
}

int qc_decode_launches(const qc_plan* p, int gamma, int iters, int early_stop) {
  if (!p || iters < 1) return -1;
  if (!early_stop && qcb::agg_eligible(p)) return 3 + qcb::agg_decode_launches(p, gamma, iters);
  // compact early stop: memset, first check, 2 x iters jobs (syndrome / freeze folded in), tail (2)
  if (early_stop && qcb::agg_es_eligible(p, gamma)) return 1 + 2 * iters + 2;
  return early_stop ? 2 + 4 * iters + 2 : 1 + 2 * iters + 2;
}

}  // extern "C"
