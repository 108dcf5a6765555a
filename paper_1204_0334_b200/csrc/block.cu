// Batched flooding sum-product decoder for LDPC block codes on sm_100a.
//
// Replaces the numpy hot loop of /root/reference/pkg/src/qcldpc/bp.py:
//   MessageBatch init (bp.py:74-84), check_node_update (bp.py:134-162),
//   variable_node_update (bp.py:165-188), hard_decision_and_syndrome
//   (bp.py:191-210) and decode_llr_batch (bp.py:213-265).
//
// Layout (paper's Gamma-codeword packages): the message
// store is edge-major (E, gamma) fp32, so the gamma messages of one Tanner
// edge are contiguous (gamma*4 bytes, 128-byte aligned for gamma % 32 == 0).
// One thread owns VEC consecutive lanes of a package (float4 / float2 / float
// loads), consecutive threads walk the lanes of the same package, so every
// package read or write is a fully coalesced 128-bit access.
//
// Check pass: one thread = (check m, lane vector q); its d_c packages are
// contiguous in the row-major edge order (codes.py:186-188), loaded up front
// into registers (d_c independent 128-bit loads in flight per thread).
// Variable pass: one thread = (variable n, lane vector q); its d_v package
// addresses come from QC shift arithmetic (shift grid staged in shared
// memory) or, for non-QC / irregular codes, from a padded var table.
#include <cuda_runtime.h>

#include <algorithm>
#include <cstring>
#include <string>
#include <vector>

#include "block_kernels.cuh"

using namespace qcb;

namespace {

__global__ void init_kernel(const float* mu, float* msgs, const int32_t* edge_var, int E, int gamma) {
  long long tid = (long long)blockIdx.x * blockDim.x + threadIdx.x;
  int GV = gamma / 4;
  if (tid >= (long long)E * GV) return;
  int e = (int)(tid / GV), q = (int)(tid - (long long)e * GV);
  float v[4];
  vload<4>(mu + (size_t)edge_var[e] * gamma + q * 4, v);
  vstore<4>(msgs + (size_t)e * gamma + q * 4, v);
}

// per (check, 32-lane word): XOR of the hard-bit planes of the check's
// variables; any odd word marks its lanes as failing (bp.py:199-208)
__global__ void syndrome_kernel(const uint32_t* hb, uint32_t* bad, const int32_t* check_ptr,
                                const int32_t* edge_var, int M, int W, const int32_t* done) {
  if (done && *done) return;
  long long tid = (long long)blockIdx.x * blockDim.x + threadIdx.x;
  if (tid >= (long long)M * W) return;
  int m = (int)(tid / W), w = (int)(tid - (long long)m * W);
  int e0 = check_ptr[m], deg = check_ptr[m + 1] - e0;
  uint32_t par = 0;
  for (int k = 0; k < deg; ++k) par ^= hb[(size_t)edge_var[e0 + k] * W + w];
  if (par) atomicOr(bad + w, par);
}

__global__ void hard_bits_kernel(const float* post, uint32_t* hb, int N, int gamma) {
  long long tid = (long long)blockIdx.x * blockDim.x + threadIdx.x;
  int GV = gamma / 4;
  bool valid = tid < (long long)N * GV;
  int n = valid ? (int)(tid / GV) : 0, q = valid ? (int)(tid - (long long)n * GV) : 0;
  unsigned bits = 0;
  if (valid) {
    float v[4];
    vload<4>(post + (size_t)n * gamma + q * 4, v);
    for (int i = 0; i < 4; ++i) bits |= (v[i] < 0.0f ? 1u : 0u) << i;
  }
  store_bit_word<4>(hb + (size_t)n * (gamma >> 5), q, bits, valid);
}

// per-lane popcount over the N hard-bit planes (lane_bits must be zeroed):
// each block walks a chunk of variables with consecutive threads on
// consecutive 32-lane words (coalesced), counts set bits in shared memory
// (hard bits are sparse at useful SNRs: a zero word costs one load), and adds
// its nonzero lane counts to the global ones
// lane_mask (W words, may be null): count only these lanes (the recycling
// engine counts the lanes that finish this tick; the others' bits are discarded)
__global__ void bit_errors_kernel(const uint32_t* hb, int32_t* lane_bits, int N, int W, int rows_per_block,
                                  const uint32_t* lane_mask) {
  extern __shared__ int cnt[];                 // W * 32 counters, then W mask words
  uint32_t* msk = reinterpret_cast<uint32_t*>(cnt + W * 32);
  for (int i = threadIdx.x; i < W * 32; i += blockDim.x) cnt[i] = 0;
  for (int i = threadIdx.x; i < W; i += blockDim.x) msk[i] = lane_mask ? lane_mask[i] : 0xffffffffu;
  __syncthreads();
  const int n0 = blockIdx.x * rows_per_block, n1 = min(N, n0 + rows_per_block);
  const long long total = (long long)(n1 - n0) * W;
  const uint32_t* base = hb + (size_t)n0 * W;               // the block's rows are contiguous words
  constexpr int U = 8;                                       // independent loads in flight per thread
  for (long long i0 = threadIdx.x; i0 < total; i0 += (long long)U * blockDim.x) {
    uint32_t x[U];
#pragma unroll
    for (int u = 0; u < U; ++u) {
      const long long i = i0 + (long long)u * blockDim.x;
      x[u] = (i < total && msk[(int)(i % W)]) ? base[i] : 0u;
    }
#pragma unroll
    for (int u = 0; u < U; ++u) {
      const int w = (int)((i0 + (long long)u * blockDim.x) % W);
      for (uint32_t v = x[u] & msk[w]; v; v &= v - 1) atomicAdd(&cnt[w * 32 + __ffs(v) - 1], 1);
    }
  }
  __syncthreads();
  for (int i = threadIdx.x; i < W * 32; i += blockDim.x)
    if (cnt[i]) atomicAdd(lane_bits + i, cnt[i]);
}

// early-stop bookkeeping after iteration `it` (bp.py:242-256): lanes that are
// active and syndrome-clean freeze; bad words are consumed and cleared.
__global__ void es_update_kernel(uint32_t* active, uint32_t* bad, int32_t* iters_run, int32_t* done,
                                 int W, int it) {
  __shared__ int any;
  if (threadIdx.x == 0) any = 0;
  __syncthreads();
  if (*done) return;
  for (int w = threadIdx.x; w < W; w += blockDim.x) {
    uint32_t act = active[w];
    uint32_t stop = act & ~bad[w];
    for (int b = 0; b < 32; ++b)
      if ((stop >> b) & 1u) iters_run[w * 32 + b] = it;
    act &= ~stop;
    active[w] = act;
    bad[w] = 0;
    if (act) any = 1;
  }
  __syncthreads();
  if (threadIdx.x == 0 && !any) *done = 1;
}

__global__ void es_start_kernel(uint32_t* active, uint32_t* bad, int32_t* iters_run, int32_t* done,
                                int W, int iters) {
  for (int w = threadIdx.x + blockIdx.x * blockDim.x; w < W; w += blockDim.x * gridDim.x) {
    active[w] = 0xffffffffu;
    bad[w] = 0;
    for (int b = 0; b < 32; ++b) iters_run[w * 32 + b] = iters;
  }
  if (threadIdx.x == 0 && blockIdx.x == 0) *done = 0;
}

// ok[g] = lane passed the syndrome.  Early stop: ok = frozen (= !active);
// plain decode: ok = !bad.
__global__ void finalize_ok_kernel(const uint32_t* bad, const uint32_t* active, uint8_t* ok, int gamma) {
  int g = blockIdx.x * blockDim.x + threadIdx.x;
  if (g >= gamma) return;
  uint32_t b = active ? active[g >> 5] : bad[g >> 5];
  ok[g] = ((b >> (g & 31)) & 1u) ? 0 : 1;
}

__global__ void fill_i32(int32_t* p, int n, int v) {
  int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i < n) p[i] = v;
}

// (N, gamma) fp32 -> (gamma_out, N) fp64|fp32 / u8 through a 32x32 smem tile
template <typename OUT>
__global__ void lane_major_kernel(const float* post, OUT* post_out, uint8_t* bits_out, int N,
                                  int gamma, int gamma_out) {
  __shared__ float tile[32][33];
  int n0 = blockIdx.x * 32, g0 = blockIdx.y * 32;
  for (int dy = threadIdx.y; dy < 32; dy += blockDim.y) {
    int n = n0 + dy, g = g0 + threadIdx.x;
    tile[dy][threadIdx.x] = (n < N) ? post[(size_t)n * gamma + g] : 0.0f;
  }
  __syncthreads();
  for (int dy = threadIdx.y; dy < 32; dy += blockDim.y) {
    int g = g0 + dy, n = n0 + threadIdx.x;
    if (g < gamma_out && n < N) {
      float v = tile[threadIdx.x][dy];
      if (post_out) post_out[(size_t)g * N + n] = (OUT)v;
      if (bits_out) bits_out[(size_t)g * N + n] = v < 0.0f ? 1 : 0;
    }
  }
}

// lane-major fp64 (received values or LLRs) -> variable-major fp32 LLRs, in
// the reference's operation order: clip((2*y)/(sigma*sigma), +-50) (bp.py:54-56)
// when sigma > 0, clip(x, +-50) otherwise (bp.py:231); padded lanes get +50.
__global__ void llr_from_lane_major_kernel(const double* x, float* mu, int N, int gamma,
                                           int gamma_in, double sigma) {
  __shared__ float tile[32][33];
  int n0 = blockIdx.x * 32, g0 = blockIdx.y * 32;
  const double s2 = __dmul_rn(sigma, sigma);
  for (int dy = threadIdx.y; dy < 32; dy += blockDim.y) {
    int g = g0 + dy, n = n0 + threadIdx.x;
    float v = 50.0f;
    if (g < gamma_in && n < N) {
      double t = x[(size_t)g * N + n];
      if (sigma > 0.0) t = __ddiv_rn(__dmul_rn(2.0, t), s2);
      t = t < -50.0 ? -50.0 : (t > 50.0 ? 50.0 : t);
      v = __double2float_rn(t);
    }
    tile[dy][threadIdx.x] = v;
  }
  __syncthreads();
  for (int dy = threadIdx.y; dy < 32; dy += blockDim.y) {
    int n = n0 + dy, g = g0 + threadIdx.x;
    if (n < N) mu[(size_t)n * gamma + g] = tile[threadIdx.x][dy];
  }
}

__global__ void batch_counts_kernel(const int32_t* lane_bits, int64_t* counts, int nb, int gref) {
  int b = blockIdx.x * blockDim.x + threadIdx.x;
  if (b >= nb) return;
  long long be = 0, fe = 0;
  for (int g = 0; g < gref; ++g) {
    int v = lane_bits[b * gref + g];
    be += v;
    fe += v > 0;
  }
  counts[b * 3 + 0] += gref;
  counts[b * 3 + 1] += be;
  counts[b * 3 + 2] += fe;
}

// ----------------------------------------------------------------------------
// dispatch
// ----------------------------------------------------------------------------
int bucket_dc(int d) {
  static const int B[] = {4, 8, 16, 24, 32};
  for (int b : B)
    if (d <= b) return b;
  return -1;
}

int launch_cnu(const qc_plan* p, CnuArgs a, int mode, cudaStream_t s) {
  if (p->E == 0 || p->M == 0) return 0;
  int rc;
  switch (bucket_dc(p->dc_max)) {
    case 4: rc = launch_cnu_dc<4>(p, a, mode, s); break;
    case 8: rc = launch_cnu_dc<8>(p, a, mode, s); break;
    case 16: rc = launch_cnu_dc<16>(p, a, mode, s); break;
    case 24: rc = launch_cnu_dc<24>(p, a, mode, s); break;
    case 32: rc = launch_cnu_dc<32>(p, a, mode, s); break;
    default: return fail_arg("check degree > 32 is not supported");
  }
  if (rc) return rc;
  return check_launch("cnu");
}

int check_gamma(int gamma) {
  if (gamma <= 0 || gamma % 32) return fail_arg("gamma must be a positive multiple of 32, got " + std::to_string(gamma));
  return 0;
}

int launch_syndrome(const qc_plan* p, int gamma, const uint32_t* hb, uint32_t* bad, const int32_t* done,
                    cudaStream_t s) {
  int W = gamma / 32;
  if (p->M == 0) return 0;
  long long threads = (long long)p->M * W;
  syndrome_kernel<<<blocks_for(threads), THREADS, 0, s>>>(hb, bad, p->d_check_ptr, p->d_edge_var, p->M, W, done);
  return check_launch("syndrome");
}

int launch_bit_errors(const qc_plan* p, int gamma, const uint32_t* hb, int32_t* lane_bits, cudaStream_t s,
                      const uint32_t* lane_mask = nullptr) {
  const int W = gamma / 32;
  cudaMemsetAsync(lane_bits, 0, sizeof(int32_t) * gamma, s);
  if (p->N == 0) return 0;
  // ~2 blocks per SM, each at least 64 rows; W * 32 counters of shared memory
  const int blocks = std::max(1, std::min(296, (p->N + 63) / 64));
  const int rows = (p->N + blocks - 1) / blocks;
  const size_t smem = (size_t)W * 33 * sizeof(int);
  static const bool big_smem = [] {     // once per process (not a stream operation: graph-capture safe)
    return cudaFuncSetAttribute(bit_errors_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024) ==
           cudaSuccess;
  }();
  if (smem > (big_smem ? 200u : 48u) * 1024) return fail_arg("bit_errors: gamma too large for the shared counters");
  bit_errors_kernel<<<(p->N + rows - 1) / rows, 256, smem, s>>>(hb, lane_bits, p->N, W, rows, lane_mask);
  return check_launch("bit_errors");
}

}  // namespace

namespace qcb {
// decode work buffer: lane-mask words (early stop: bad | active | done for the
// two-pass path; act[2] | bad[2] | bad_fin for the compact one) padded to 64
// words, then the check records of the compact schedule (agg.cu)
size_t work_head_words(int gamma) {
  const size_t W = (size_t)(gamma > 0 ? gamma : 0) / 32;
  return (5 * W + 4 + 63) / 64 * 64;
}
int launch_cnu_public(const qc_plan* p, CnuArgs a, int mode, cudaStream_t s) { return launch_cnu(p, a, mode, s); }
// early-stop tail of the compact decode (agg.cu run_agg_decode_es): syndrome
// of iteration T for every lane, then per word: active_{T-1} (half A stored by
// its last update; half B derived here, its update never ran), lanes frozen
// at T-1 get iters_run = T-1, ok = not active after T.
__global__ void es_final_kernel(const uint32_t* act_a, const uint32_t* act_b, const uint32_t* bad_b,
                                const uint32_t* bad_fin, uint8_t* ok, int32_t* iters_run, int W, int WH, int T) {
  const int w = blockIdx.x * blockDim.x + threadIdx.x;
  if (w >= W) return;
  uint32_t prev;
  if (w < WH) {
    prev = act_a[w];
  } else if (T == 1) {
    prev = 0xffffffffu;
    for (int b = 0; b < 32; ++b) iters_run[w * 32 + b] = T;
  } else {
    const uint32_t pp = act_b[w];
    prev = pp & bad_b[w];
    for (uint32_t f = pp & ~prev; f; f &= f - 1) iters_run[w * 32 + __ffs(f) - 1] = T - 1;
  }
  const uint32_t fin = prev & bad_fin[w];
  for (int b = 0; b < 32; ++b) ok[w * 32 + b] = ((fin >> b) & 1u) ? 0 : 1;
}

int launch_es_tail(const qc_plan* p, int gamma, int iters, uint32_t* const act[2], uint32_t* const bad[2],
                   uint32_t* bad_fin, uint8_t* ok, int32_t* iters_run, const float* post, uint32_t* hb,
                   cudaStream_t s) {
  const int W = gamma / 32, T = iters;
  if (int rc = launch_syndrome(p, gamma, hb, bad_fin, nullptr, s)) return rc;
  es_final_kernel<<<(W + 127) / 128, 128, 0, s>>>(act[(T - 1) & 1], act[T & 1], bad[(T - 1) & 1], bad_fin, ok,
                                                   iters_run, W, W / 2, T);
  (void)post;   // the hard-bit planes already hold every lane's recorded bits (agg.cu es_store_bits)
  return check_launch("es_tail");
}
int launch_syndrome_ext(const qc_plan* p, int gamma, const uint32_t* hb, uint32_t* bad, cudaStream_t s) {
  return launch_syndrome(p, gamma, hb, bad, nullptr, s);
}
int launch_hard_bits_ext(const qc_plan* p, int gamma, const float* post, uint32_t* hb, cudaStream_t s) {
  long long threads = (long long)p->N * (gamma / 4);
  hard_bits_kernel<<<blocks_for(threads), THREADS, 0, s>>>(post, hb, p->N, gamma);
  return check_launch("hard_bits");
}
int launch_bit_errors_ext(const qc_plan* p, int gamma, const uint32_t* hb, int32_t* lane_bits, cudaStream_t s,
                          const uint32_t* lane_mask) {
  return launch_bit_errors(p, gamma, hb, lane_bits, s, lane_mask);
}
}  // namespace qcb

// ============================================================================
// C ABI
// ============================================================================
extern "C" {

int qc_init(const qc_plan* p, int gamma, const float* mu, float* msgs, void* stream) {
  if (int r = check_gamma(gamma)) return r;
  if (!p || !mu || !msgs) return fail_arg("null argument");
  if (p->E == 0) return 0;
  long long threads = (long long)p->E * (gamma / 4);
  init_kernel<<<blocks_for(threads), THREADS, 0, as_stream(stream)>>>(mu, msgs, p->d_edge_var, p->E, gamma);
  return check_launch("init");
}

int qc_cnu(const qc_plan* p, int gamma, float* msgs, const uint32_t* active, void* stream) {
  if (int r = check_gamma(gamma)) return r;
  if (!p || !msgs) return fail_arg("null argument");
  CnuArgs a{msgs, nullptr, p->d_check_ptr, p->d_edge_var, active, nullptr, p->M, gamma};
  return launch_cnu(p, a, CNU_BETA, as_stream(stream));
}

int qc_vnu(const qc_plan* p, int gamma, float* msgs, const float* mu, float* post, uint32_t* hb,
           const uint32_t* active, void* stream) {
  if (int r = check_gamma(gamma)) return r;
  if (!p || !msgs || !mu) return fail_arg("null argument");
  VnuArgs a{};
  a.msgs = msgs; a.mu = mu; a.post = post; a.hb = hb; a.active = active; a.done = nullptr;
  a.gamma = gamma;
  a.post_all = 1;   // frozen lanes keep their packages but still get clip(total) (bp.py:183-187)
  return launch_vnu(p, a, VNU_BETA, as_stream(stream));
}

int qc_cnu_ex(const qc_plan* p, int gamma, int mode, float* msgs, const float* mu, const uint32_t* active,
              void* stream) {
  if (int r = check_gamma(gamma)) return r;
  if (!p || !msgs || mode < 0 || mode > 2 || (mode == CNU_FROM_MU && !mu)) return fail_arg("bad cnu arguments");
  CnuArgs a{msgs, mu, p->d_check_ptr, p->d_edge_var, active, nullptr, p->M, gamma};
  return launch_cnu(p, a, mode, as_stream(stream));
}

int qc_vnu_ex(const qc_plan* p, int gamma, int mode, float* msgs, const float* mu, float* post, uint32_t* hb,
              const uint32_t* active, void* stream) {
  if (int r = check_gamma(gamma)) return r;
  if (!p || !msgs || !mu || mode < 0 || mode > 2) return fail_arg("bad vnu arguments");
  VnuArgs a{};
  a.msgs = msgs; a.mu = mu; a.post = post; a.hb = hb; a.active = active; a.gamma = gamma;
  return launch_vnu(p, a, mode, as_stream(stream));
}

int qc_syndrome(const qc_plan* p, int gamma, const uint32_t* hb, uint32_t* bad, void* stream) {
  if (int r = check_gamma(gamma)) return r;
  if (!p || !hb || !bad) return fail_arg("null argument");
  return launch_syndrome(p, gamma, hb, bad, nullptr, as_stream(stream));
}

int qc_hard_bits(const qc_plan* p, int gamma, const float* post, uint32_t* hb, void* stream) {
  if (int r = check_gamma(gamma)) return r;
  if (!p || !post || !hb) return fail_arg("null argument");
  long long threads = (long long)p->N * (gamma / 4);
  hard_bits_kernel<<<blocks_for(threads), THREADS, 0, as_stream(stream)>>>(post, hb, p->N, gamma);
  return check_launch("hard_bits");
}

int qc_bit_errors(const qc_plan* p, int gamma, const uint32_t* hb, int32_t* lane_bits, void* stream) {
  if (int r = check_gamma(gamma)) return r;
  if (!p || !hb || !lane_bits) return fail_arg("null argument");
  return launch_bit_errors(p, gamma, hb, lane_bits, as_stream(stream));
}

size_t qc_decode_work_words(const qc_plan* p, int gamma) {
  return work_head_words(gamma) + agg_words(p, gamma);
}

size_t qc_decode_records_offset(int gamma) { return work_head_words(gamma); }

int qc_decode(const qc_plan* p, int gamma, int iters, int early_stop, const float* mu, float* msgs,
              float* post, uint32_t* hb, uint32_t* work, uint8_t* ok, int32_t* iters_run,
              int32_t* lane_bits, void* stream) {
  if (int r = check_gamma(gamma)) return r;
  if (iters < 1) return fail_arg("need at least one iteration");
  if (!p || !mu || !msgs || !post || !hb || !work || !ok || !iters_run) return fail_arg("null argument");
  cudaStream_t s = as_stream(stream);
  const int W = gamma / 32;
  uint32_t* bad = work;
  uint32_t* active = work + W;
  int32_t* done = reinterpret_cast<int32_t*>(work + 2 * W);
  int rc = 0;
  // Messages between the passes are kept in PHI form (sign * phi(|beta|)):
  // iteration 1 reads beta^0 = mu straight from the LLRs (fused init).
  if (!early_stop && agg_eligible(p)) {
    // compact check-state schedule (agg.cu): bit-identical, fewer package bytes
    float* agg = reinterpret_cast<float*>(work + work_head_words(gamma));
    cudaMemsetAsync(bad, 0, sizeof(uint32_t) * W, s);
    fill_i32<<<blocks_for(gamma), THREADS, 0, s>>>(iters_run, gamma, iters);
    if ((rc = run_agg_decode(p, gamma, iters, msgs, mu, agg, post, hb, s))) return rc;
    if ((rc = launch_syndrome(p, gamma, hb, bad, nullptr, s))) return rc;
    finalize_ok_kernel<<<blocks_for(gamma), THREADS, 0, s>>>(bad, nullptr, ok, gamma);
  } else if (!early_stop) {
    cudaMemsetAsync(bad, 0, sizeof(uint32_t) * W, s);
    fill_i32<<<blocks_for(gamma), THREADS, 0, s>>>(iters_run, gamma, iters);
    for (int it = 1; it <= iters; ++it) {
      CnuArgs c{msgs, mu, p->d_check_ptr, p->d_edge_var, nullptr, nullptr, p->M, gamma};
      if ((rc = launch_cnu(p, c, it == 1 ? CNU_FROM_MU : CNU_PHI, s))) return rc;
      VnuArgs v{};
      v.msgs = msgs; v.mu = mu; v.gamma = gamma;
      v.post = it == iters ? post : nullptr;
      v.hb = it == iters ? hb : nullptr;
      if ((rc = launch_vnu(p, v, it < iters ? VNU_PHI : VNU_NONE, s))) return rc;   // last beta never read
    }
    if ((rc = launch_syndrome(p, gamma, hb, bad, nullptr, s))) return rc;
    finalize_ok_kernel<<<blocks_for(gamma), THREADS, 0, s>>>(bad, nullptr, ok, gamma);
  } else if (agg_es_eligible(p, gamma)) {
    // compact schedule, syndrome and freeze folded into the fused launches (agg.cu)
    if ((rc = run_agg_decode_es(p, gamma, iters, msgs, mu, reinterpret_cast<float*>(work + work_head_words(gamma)),
                                post, hb, work, ok, iters_run, s)))
      return rc;
  } else {
    es_start_kernel<<<1, 256, 0, s>>>(active, bad, iters_run, done, W, iters);
    for (int it = 1; it <= iters; ++it) {
      // iteration 1: every lane is active, so the fused init is exact
      CnuArgs c{msgs, mu, p->d_check_ptr, p->d_edge_var, active, done, p->M, gamma};
      if ((rc = launch_cnu(p, c, it == 1 ? CNU_FROM_MU : CNU_PHI, s))) return rc;
      VnuArgs v{};
      v.msgs = msgs; v.mu = mu; v.gamma = gamma;
      v.post = post; v.hb = hb; v.active = active; v.done = done;
      if ((rc = launch_vnu(p, v, VNU_PHI, s))) return rc;
      if ((rc = launch_syndrome(p, gamma, hb, bad, done, s))) return rc;
      es_update_kernel<<<1, 256, 0, s>>>(active, bad, iters_run, done, W, it);
    }
    finalize_ok_kernel<<<blocks_for(gamma), THREADS, 0, s>>>(bad, active, ok, gamma);
    // hb must reflect the recorded posteriors of every lane (frozen lanes too)
    long long threads = (long long)p->N * (gamma / 4);
    hard_bits_kernel<<<blocks_for(threads), THREADS, 0, s>>>(post, hb, p->N, gamma);
  }
  if (lane_bits && (rc = launch_bit_errors(p, gamma, hb, lane_bits, s))) return rc;
  return check_launch("decode");
}

int qc_decode_es(const qc_plan* p, int gamma, int iters, const float* mu, float* msgs, float* post, uint32_t* hb,
                 uint32_t* work, uint32_t* scratch, uint8_t* ok, int32_t* iters_run, int32_t* lane_bits,
                 void* stream) {
  if (int r = check_gamma(gamma)) return r;
  if (iters < 1) return fail_arg("need at least one iteration");
  if (!p || !mu || !msgs || !post || !hb || !work || !ok || !iters_run) return fail_arg("null argument");
  if (!es_compact_eligible(p, gamma, iters))
    return qc_decode(p, gamma, iters, 1, mu, msgs, post, hb, work, ok, iters_run, lane_bits, stream);
  if (!scratch) return fail_arg("null scratch (qc_decode_es_scratch_words > 0)");
  cudaStream_t s = as_stream(stream);
  int rc;
  if ((rc = run_agg_decode_es_compact(p, gamma, iters, msgs, mu, post, hb, work, scratch, ok, iters_run, s)))
    return rc;
  if (lane_bits && (rc = launch_bit_errors(p, gamma, hb, lane_bits, s))) return rc;
  return check_launch("decode_es");
}

int qc_decode_es_launches(const qc_plan* p, int gamma, int iters) {
  if (!p || iters < 1) return -1;
  if (!es_compact_eligible(p, gamma, iters)) return qc_decode_launches(p, gamma, iters, 1);
  return es_compact_launches(p, gamma, iters);
}

int qc_lane_major(int n, int gamma, int gamma_out, const float* post, double* post_out, uint8_t* bits_out,
                  void* stream) {
  if (int r = check_gamma(gamma)) return r;
  if (n < 0 || !post || gamma_out < 0 || gamma_out > gamma) return fail_arg("bad lane_major arguments");
  if (n == 0 || gamma_out == 0) return 0;
  dim3 grid((n + 31) / 32, (gamma_out + 31) / 32), block(32, 8);
  lane_major_kernel<double><<<grid, block, 0, as_stream(stream)>>>(post, post_out, bits_out, n, gamma, gamma_out);
  return check_launch("lane_major");
}

int qc_lane_major_f32(int n, int gamma, int gamma_out, const float* post, float* post_out, uint8_t* bits_out,
                      void* stream) {
  if (int r = check_gamma(gamma)) return r;
  if (n < 0 || !post || gamma_out < 0 || gamma_out > gamma) return fail_arg("bad lane_major arguments");
  if (n == 0 || gamma_out == 0) return 0;
  dim3 grid((n + 31) / 32, (gamma_out + 31) / 32), block(32, 8);
  lane_major_kernel<float><<<grid, block, 0, as_stream(stream)>>>(post, post_out, bits_out, n, gamma, gamma_out);
  return check_launch("lane_major_f32");
}

// host-array forms for per-frame I/O (StreamDecoder.push_frame): one C call
// instead of a torch copy + kernel call per direction (per-push host overhead
// dominates small-gamma pushes, profiles/r02/stream_api_push_frame.md)
int qc_lane_major_to_host(int n, int gamma, int gamma_out, const float* post, double* post_dev,
                          uint8_t* bits_dev, double* post_host, uint8_t* bits_host, void* stream) {
  if ((post_host && !post_dev) || (bits_host && !bits_dev)) return fail_arg("device staging missing");
  if (int r = qc_lane_major(n, gamma, gamma_out, post, post_dev, bits_dev, stream)) return r;
  cudaStream_t s = as_stream(stream);
  const size_t cnt = (size_t)n * gamma_out;
  if (post_host && cnt) {
    cudaError_t e = cudaMemcpyAsync(post_host, post_dev, cnt * sizeof(double), cudaMemcpyDeviceToHost, s);
    if (e != cudaSuccess) return fail_rt(std::string("lane_major_to_host: ") + cudaGetErrorString(e));
  }
  if (bits_host && cnt) {
    cudaError_t e = cudaMemcpyAsync(bits_host, bits_dev, cnt, cudaMemcpyDeviceToHost, s);
    if (e != cudaSuccess) return fail_rt(std::string("lane_major_to_host: ") + cudaGetErrorString(e));
  }
  return 0;
}

int qc_llr_from_host(int n, int gamma, int gamma_in, const double* x_host, double* x_dev, double sigma,
                     float* mu_vm, void* stream) {
  if (!x_host || !x_dev) return fail_arg("null argument");
  if (n < 0 || gamma_in < 0 || gamma_in > gamma) return fail_arg("bad llr arguments");
  if (n && gamma_in) {
    cudaError_t e = cudaMemcpyAsync(x_dev, x_host, (size_t)n * gamma_in * sizeof(double), cudaMemcpyHostToDevice,
                                    as_stream(stream));
    if (e != cudaSuccess) return fail_rt(std::string("llr_from_host: ") + cudaGetErrorString(e));
  }
  return qc_llr_from_lane_major(n, gamma, gamma_in, x_dev, sigma, mu_vm, stream);
}

int qc_llr_from_lane_major(int n, int gamma, int gamma_in, const double* x, double sigma, float* mu_vm,
                           void* stream) {
  if (int r = check_gamma(gamma)) return r;
  if (n < 0 || gamma_in < 0 || gamma_in > gamma || (!x && gamma_in) || !mu_vm) return fail_arg("bad llr arguments");
  if (n == 0) return 0;
  dim3 grid((n + 31) / 32, gamma / 32), block(32, 8);
  llr_from_lane_major_kernel<<<grid, block, 0, as_stream(stream)>>>(x, mu_vm, n, gamma, gamma_in, sigma);
  return check_launch("llr_from_lane_major");
}

int qc_batch_counts(int gamma, int gamma_ref, const int32_t* lane_bits, int64_t* counts, void* stream) {
  if (gamma_ref <= 0 || gamma <= 0 || gamma % gamma_ref) return fail_arg("gamma must be a multiple of gamma_ref");
  int nb = gamma / gamma_ref;
  batch_counts_kernel<<<blocks_for(nb), THREADS, 0, as_stream(stream)>>>(lane_bits, counts, nb, gamma_ref);
  return check_launch("batch_counts");
}

}  // extern "C"
