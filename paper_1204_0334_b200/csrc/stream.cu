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
#include <cstring>
#include <numeric>
#include <string>
#include <vector>

#include "common.cuh"
#include "phi.cuh"

using namespace qcb;

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
  long long t;              // slot (t_dev: offset added to *t_dev)
};

__device__ __forceinline__ long long slot_of(const SlotArgs& a) {
  return a.t_dev ? (*a.t_dev + a.t) : a.t;
}

__device__ __forceinline__ int pmod(long long x, int m) {
  long long r = x % m;
  return (int)(r < 0 ? r + m : r);
}

__device__ __forceinline__ void stage(const CcParams& P, int16_t* sh) {
  for (int i = threadIdx.x; i < P.J * P.L; i += blockDim.x) sh[i] = P.s[i];
  __syncthreads();
}

// local edge id of (variable v of a frame, block row br) inside sub-block `lbl`
template <bool QC>
__device__ __forceinline__ int var_local(const CcParams& P, const int16_t* sh, const int32_t* var_tab,
                                         int lbl, int v, int br) {
  if constexpr (QC) {
    int bc = v / P.p, cc = v - bc * P.p;
    int R = lbl / P.lam, Cc = lbl - R * P.lam;
    int rr = cc - sh[(R * P.sj + br) * P.L + Cc * P.sl + bc];
    rr += rr < 0 ? P.p : 0;
    return (br * P.p + rr) * P.sl + bc;
  } else {
    return var_tab[((size_t)lbl * P.c + v) * P.sj + br];
  }
}

// check-node core with a `present` mask of live positions (bootstrap layers
// drop absent frames); same arithmetic as the block decoder (block_kernels.cuh).
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
        // S2 excludes the first maximum; an exactly tied maximum has the same
        // exclusive sum (S - mx == S2), so every edge equal to mx takes S2
        float mag = (f == mx) ? S2 : __fsub_rn(S, f);
        float al = fminf(phi_of_log2(mag), ALPHA_CAP);
        x[k][i] = __uint_as_float(__float_as_uint(al) | ((u ^ par) & 0x80000000u));
      }
    }
  }
}

// ---- entry: frame t into ring slot t mod window and its T sub-blocks -------
template <int VEC, bool QC>
__global__ void __launch_bounds__(THREADS) entry_kernel(SlotArgs a, const __grid_constant__ CcParams P) {
  __shared__ int16_t sh[CC_MAX_SHIFTS];
  if constexpr (QC) stage(P, sh);
  const long long t = slot_of(a);
  const int T = P.lam, GV = P.gamma / VEC;
  long long tid = (long long)blockIdx.x * blockDim.x + threadIdx.x;
  if (tid >= (long long)P.c * GV) return;
  int v = (int)(tid / GV), q = (int)(tid - (long long)v * GV);
  float m[VEC];
  if (a.mu_in) vload<VEC>(a.mu_in + (size_t)v * P.gamma + q * VEC, m);
  else {
#pragma unroll
    for (int i = 0; i < VEC; ++i) m[i] = 0.0f;
  }
  const int window = P.I * T;
  vstore<VEC>(a.ring + ((size_t)pmod(t, window) * P.c + v) * P.gamma + q * VEC, m);
  // beta^0 = mu into the frame's T sub-blocks, stored in phi form
#pragma unroll
  for (int i = 0; i < VEC; ++i)
    m[i] = __uint_as_float(__float_as_uint(psi_of_nat(fabsf(m[i]))) | (__float_as_uint(m[i]) & 0x80000000u));
  const int ph = pmod(t, T);
  const size_t grp = (size_t)pmod(t / T, P.I) * P.E;
  for (int d = 0; d < T; ++d) {
    int lbl = ((ph + d) % T) * T + ph;
    for (int br = 0; br < P.sj; ++br) {
      int loc = var_local<QC>(P, sh, a.var_tab, lbl, v, br);
      if (loc >= 0) vstore<VEC>(a.msg + (grp + P.sub_off[lbl] + loc) * P.gamma + q * VEC, m);
    }
  }
}

// ---- check phase: processors i = 1..I refresh layer s = t - (i-1)T --------
template <int DC, int VEC, bool QC>
__global__ void __launch_bounds__(THREADS) check_kernel(SlotArgs a, const __grid_constant__ CcParams P) {
  const long long t = slot_of(a);
  const int T = P.lam, GV = P.gamma / VEC;
  long long tid = (long long)blockIdx.x * blockDim.x + threadIdx.x;
  if (tid >= (long long)P.I * P.cb * GV) return;
  int ip = (int)(tid / ((long long)P.cb * GV));
  long long rem = tid - (long long)ip * P.cb * GV;
  int r = (int)(rem / GV), q = (int)(rem - (long long)r * GV);
  const long long s = t - (long long)ip * T;
  if (s < 0) return;
  const int kap = pmod(s, T);
  const int W = QC ? P.sl : P.wmax;
  unsigned eidx[DC];   // package index (I*E < 2^32)
  unsigned long long present = 0;
#pragma unroll
  for (int k = 0; k < DC; ++k) eidx[k] = 0;
  for (int d = 0; d < T; ++d) {
    long long f = s - P.ms + d;
    if (f < 0) continue;   // bootstrap: absent frames drop out (convolutional.py:276-279)
    int lbl = kap * T + (kap + 1 + d) % T;
    unsigned base = (unsigned)pmod(f / T, P.I) * (unsigned)P.E + (unsigned)P.sub_off[lbl];
#pragma unroll
    for (int k = 0; k < DC; ++k) {
      if (k / W == d) {
        int w = k - d * W;
        int loc;
        if constexpr (QC) loc = r * P.sl + w;
        else loc = a.check_tab[((size_t)lbl * P.cb + r) * P.wmax + w];
        if (loc >= 0) { eidx[k] = base + loc; present |= 1ull << k; }
      }
    }
  }
  float x[DC][VEC];
#pragma unroll
  for (int k = 0; k < DC; ++k)
    if ((present >> k) & 1ull) vload<VEC>(a.msg + (size_t)eidx[k] * P.gamma + q * VEC, x[k]);
  cnu_core_mask<DC, VEC>(x, present);
#pragma unroll
  for (int k = 0; k < DC; ++k)
    if ((present >> k) & 1ull) vstore<VEC>(a.msg + (size_t)eidx[k] * P.gamma + q * VEC, x[k]);
}

// ---- variable phase: processors i = 1..I refresh frame j = t - iT + 1 -----
template <int DV, int VEC, bool QC>
__global__ void __launch_bounds__(THREADS) var_kernel(SlotArgs a, const __grid_constant__ CcParams P) {
  __shared__ int16_t sh[CC_MAX_SHIFTS];
  if constexpr (QC) stage(P, sh);
  const long long t = slot_of(a);
  const int T = P.lam, GV = P.gamma / VEC;
  long long tid = (long long)blockIdx.x * blockDim.x + threadIdx.x;
  if (tid >= (long long)P.I * P.c * GV) return;
  int ip = (int)(tid / ((long long)P.c * GV));
  long long rem = tid - (long long)ip * P.c * GV;
  int v = (int)(rem / GV), q = (int)(rem - (long long)v * GV);
  const long long j = t - (long long)(ip + 1) * T + 1;
  if (j < 0) return;
  const int pj = pmod(j, T);
  const unsigned grp = (unsigned)pmod(j / T, P.I) * (unsigned)P.E;
  unsigned eidx[DV];
  unsigned present = 0;
#pragma unroll
  for (int k = 0; k < DV; ++k) {
    eidx[k] = 0;
    int d = k / P.sj, br = k - d * P.sj;
    if (d < T) {
      int lbl = ((pj + d) % T) * T + pj;
      int loc = var_local<QC>(P, sh, a.var_tab, lbl, v, br);
      if (loc >= 0) { eidx[k] = grp + P.sub_off[lbl] + loc; present |= 1u << k; }
    }
  }
  float tot[VEC], am[DV][VEC];
  vload<VEC>(a.ring + ((size_t)pmod(j, P.I * T) * P.c + v) * P.gamma + q * VEC, tot);
#pragma unroll
  for (int k = 0; k < DV; ++k)
    if ((present >> k) & 1u) vload<VEC>(a.msg + (size_t)eidx[k] * P.gamma + q * VEC, am[k]);
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
#pragma unroll
        for (int i = 0; i < VEC; ++i) {
          float beta = clampL(__fsub_rn(tot[i], am[k][i]));   // stored in phi form
          b[i] = __uint_as_float(__float_as_uint(psi_of_nat(fabsf(beta))) | (__float_as_uint(beta) & 0x80000000u));
        }
        vstore<VEC>(a.msg + (size_t)eidx[k] * P.gamma + q * VEC, b);
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
  }
}

// per-slot fold of the emitted frame's bit count into (bit errors, frame errors)
__global__ void fold_kernel(int32_t* cnt, int gamma, const int64_t* t_dev, long long t, int window) {
  long long tt = t_dev ? (*t_dev + t) : t;
  if (tt - window + 1 < 0) return;
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

int pick_vec(int gamma) { return gamma >= 128 ? 4 : (gamma >= 64 ? 2 : 1); }

template <int VEC, bool QC>
void launch_entry(const CcParams& P, const SlotArgs& a, cudaStream_t s) {
  long long n = (long long)P.c * (P.gamma / VEC);
  entry_kernel<VEC, QC><<<blocks_for(n), THREADS, 0, s>>>(a, P);
}
template <int DC, int VEC, bool QC>
void launch_check(const CcParams& P, const SlotArgs& a, cudaStream_t s) {
  long long n = (long long)P.I * P.cb * (P.gamma / VEC);
  check_kernel<DC, VEC, QC><<<blocks_for(n), THREADS, 0, s>>>(a, P);
}
template <int DV, int VEC, bool QC>
void launch_var(const CcParams& P, const SlotArgs& a, cudaStream_t s) {
  long long n = (long long)P.I * P.c * (P.gamma / VEC);
  var_kernel<DV, VEC, QC><<<blocks_for(n), THREADS, 0, s>>>(a, P);
}

template <int VEC, bool QC>
int launch_slot_v(const CcParams& P, const SlotArgs& a, int dc, int dv, cudaStream_t s) {
  launch_entry<VEC, QC>(P, a, s);
  if (dc <= 8) launch_check<8, VEC, QC>(P, a, s);
  else if (dc <= 16) launch_check<16, VEC, QC>(P, a, s);
  else if (dc <= 24) launch_check<24, VEC, QC>(P, a, s);
  else if (dc <= 32) launch_check<32, VEC, QC>(P, a, s);
  else return fail_arg("LDPCCC check degree > 32 is not supported");
  if (dv <= 2) launch_var<2, VEC, QC>(P, a, s);
  else if (dv <= 4) launch_var<4, VEC, QC>(P, a, s);
  else if (dv <= 8) launch_var<8, VEC, QC>(P, a, s);
  else return fail_arg("LDPCCC variable degree > 8 is not supported");
  return 0;
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

int cc_slot(const cc_plan* pl, int I, int gamma, int64_t t, const int64_t* t_dev, float* msg, float* ring,
            const float* mu_in, float* post_out, int32_t* lane_cnt, void* stream) {
  if (!pl || !msg || !ring) return fail_arg("null argument");
  if (I < 1) return fail_arg("need at least one processor");
  if (gamma <= 0 || gamma % 32) return fail_arg("gamma must be a positive multiple of 32");
  if (!t_dev && t < 0) return fail_arg("slot index must be non-negative");
  cudaStream_t s = as_stream(stream);
  CcParams P = make_params(pl, I, gamma);
  SlotArgs a{msg, ring, mu_in, post_out, lane_cnt, pl->d_check_tab, pl->d_var_tab, t_dev, (long long)t};
  const bool qc = pl->all_live;
  const int dc = pl->lam * (qc ? pl->sl : pl->wmax);
  const int dv = pl->lam * pl->sj;
  int rc;
  switch (pick_vec(gamma)) {
    case 4: rc = qc ? launch_slot_v<4, true>(P, a, dc, dv, s) : launch_slot_v<4, false>(P, a, dc, dv, s); break;
    case 2: rc = qc ? launch_slot_v<2, true>(P, a, dc, dv, s) : launch_slot_v<2, false>(P, a, dc, dv, s); break;
    default: rc = qc ? launch_slot_v<1, true>(P, a, dc, dv, s) : launch_slot_v<1, false>(P, a, dc, dv, s); break;
  }
  if (rc) return rc;
  if (lane_cnt) fold_kernel<<<blocks_for(gamma), THREADS, 0, s>>>(lane_cnt, gamma, t_dev, t, I * pl->lam);
  return check_launch("cc_slot");
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
