// Early-stop decode with lane compaction (decode_llr_batch(..., early_stop=True),
// /root/reference/pkg/src/qcldpc/bp.py:242-256, per-lane semantics unchanged).
//
// The compact early-stop decode (agg.cu run_agg_decode_es) skips frozen lanes
// at lane-vector / warp granularity, but converged lanes are scattered over
// the batch: a 128-lane warp row stays live while any of its lanes is, so in
// the waterfall region the work barely drops (n18360 at 3.2 dB, 11.8 mean
// iterations: the early-stop decode was 17% SLOWER than 30 fixed iterations).
// Here the decode stops at a few checkpoint iterations c and packs the lanes
// still iterating to the front of both halves of a second buffer set:
//   checkpoint c: syndrome of iteration c -> per lane "still failing"; lanes
//     that are done get ok / iterations_run (and, in a compacted set, their
//     posteriors scattered to the caller's arrays by original lane id); the
//     continuing lanes' packages (E rows) and channel LLRs (N rows) are
//     gathered, rank i -> half i & 1, position i >> 1, with their original
//     ids in a lane map; the next segment restarts the fused early-stop loop
//     at iteration c + 1 under the packed active mask.
// Whole 128-lane groups beyond the packed lanes are then masked off, so the
// kernels' CTAs there exit after one mask load.  Every lane runs exactly the
// same instruction sequence on the same operands as without compaction (the
// check records are recomputed from the gathered packages), so posteriors,
// decisions and iteration counts are bit-identical to the uncompacted
// early-stop decode (tests/test_gpu_block.py::test_compacted_early_stop_*).
// The hard-bit planes are rebuilt from the final posteriors (sign rule of the
// variable pass).  Graph-capturable: the checkpoint schedule is static, lane
// counts stay on the device.
#include <cuda_runtime.h>

#include <cstring>

#include "block_kernels.cuh"

namespace qcb {

namespace {

constexpr int CK_THREADS = 1024;
#ifndef ES_LIVE
#define ES_LIVE 1     // compacted segments walk only their live lane groups (0: full grids, masked)
#endif
#ifndef ES_LOOP_FROM
#define ES_LOOP_FROM 2   // segment index (after checkpoint k-1) from which the capped-grid loop kernels run
#endif
constexpr int MAX_CHECKPOINTS = 6;

// checkpoint iterations (after these, the continuing lanes are packed); chosen
// from the iteration histogram of n18360 (profiles/r02/iters_hist.jsonl: at
// 3.2 dB 43% of lanes still iterate after 11, 12% after 14, 3% after 18) and an
// A/B of five schedules (kbench_ck.jsonl): three checkpoints beat four or five
// in the waterfall (3.0-3.2 dB, 4%), earlier / more ones win only above it
constexpr int CHECKPOINTS[] = {11, 14, 18};

struct CkArgs {
  // state of the current set after its last variable pass at iteration c
  const uint32_t* act_a;    // act[(c-1)&1] (half A's update ran)
  const uint32_t* act_b;    // act[c&1]     (half B: active_{c-1} = act_b & bad_b)
  const uint32_t* bad_b;    // bad[(c-1)&1]
  const uint32_t* bad_fin;  // syndrome failures of iteration c
  uint8_t* ok;              // current set, physical lanes
  int32_t* iters_run;
  const int32_t* map;       // physical -> original lane (null: identity)
  // outputs
  uint32_t* cont;           // (W) lanes still iterating
  int32_t* src;             // (gamma) physical lane of continuing rank i
  int32_t* count;           // [1]
  int32_t* map_next;        // (gamma)
  int32_t* iters_next;      // (gamma) = iters
  uint32_t* act_set;        // es words of the next segment (same buffers as act_a/act_b/bad_b)
  uint32_t* bad_ones;
  uint32_t* bad_zero;
  uint32_t* bad_fin_zero;
  int W, WH, H, gamma, c, iters;
};

__device__ __forceinline__ void set_iters(int32_t* it, int w, uint32_t bits, int v) {
  for (uint32_t f = bits; f; f &= f - 1) it[w * 32 + __ffs(f) - 1] = v;
}

// one CTA: per-lane outcome at iteration c, then an ordered compaction list
__global__ void __launch_bounds__(CK_THREADS) es_ckpt_kernel(CkArgs a) {
  extern __shared__ uint32_t cont[];         // (W) continuing lanes
  __shared__ int32_t warp_sum[CK_THREADS / 32];
  const int tid = threadIdx.x;
  // 1. outcome of the lanes of this set (es_final_kernel's rule at T = c)
  for (int w = tid; w < a.W; w += CK_THREADS) {
    uint32_t prev;
    if (w < a.WH) {
      prev = a.act_a[w];
    } else {
      const uint32_t pp = a.act_b[w];
      prev = pp & a.bad_b[w];
      set_iters(a.iters_run, w, pp & ~prev, a.c - 1);     // half B lanes that froze at c - 1
    }
    const uint32_t fin = prev & a.bad_fin[w];
    set_iters(a.iters_run, w, prev & ~fin, a.c);           // converged at c
    for (int b = 0; b < 32; ++b) a.ok[w * 32 + b] = ((fin >> b) & 1u) ? 0 : 1;
    cont[w] = fin;
    a.cont[w] = fin;
  }
  __syncthreads();
  // 2. exclusive scan of the continuing-lane counts over words (contiguous word chunks per thread)
  const int per = (a.W + CK_THREADS - 1) / CK_THREADS;
  const int w0 = tid * per, w1 = min(a.W, w0 + per);
  int mine = 0;
  for (int w = w0; w < w1; ++w) mine += __popc(cont[w]);
  int incl = mine;
  const int lane = tid & 31, wid = tid >> 5;
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    const int v = __shfl_up_sync(0xffffffffu, incl, o);
    if (lane >= o) incl += v;
  }
  if (lane == 31) warp_sum[wid] = incl;
  __syncthreads();
  if (wid == 0) {
    int v = warp_sum[lane];
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const int u = __shfl_up_sync(0xffffffffu, v, o);
      if (lane >= o) v += u;
    }
    warp_sum[lane] = v;                        // inclusive over warps
  }
  __syncthreads();
  const int excl = incl - mine + (wid > 0 ? warp_sum[wid - 1] : 0);
  const int total = warp_sum[CK_THREADS / 32 - 1];
  // 3. next set: maps cleared, iteration counts preset to the cap
  for (int g = tid; g < a.gamma; g += CK_THREADS) {
    a.map_next[g] = -1;
    a.iters_next[g] = a.iters;
  }
  __syncthreads();
  int r = excl;
  for (int w = w0; w < w1; ++w)
    for (uint32_t f = cont[w]; f; f &= f - 1) {
      const int pl = w * 32 + __ffs(f) - 1;
      const int np = (r & 1) * a.H + (r >> 1);
      a.src[r] = pl;
      a.map_next[np] = a.map ? a.map[pl] : pl;
      ++r;
    }
  // 4. early-stop words of the next segment: a prefix of each half is active
  const int na = (total + 1) >> 1, nb = total >> 1;
  for (int w = tid; w < a.W; w += CK_THREADS) {
    const int lo = (w < a.WH) ? w * 32 : w * 32 - a.H;      // lane offset inside its half
    const int n = (w < a.WH) ? na : nb;
    const int k = min(32, max(0, n - lo));
    a.act_set[w] = k >= 32 ? 0xffffffffu : ((1u << k) - 1u);
    a.bad_ones[w] = 0xffffffffu;
    a.bad_zero[w] = 0u;
    a.bad_fin_zero[w] = 0u;
  }
  if (tid == 0) *a.count = total;
}

// done lanes of a compacted set -> the caller's arrays by original id
// (cont == null: every mapped lane, the final segment)
#ifndef ES_ROWS
#define ES_ROWS 8   // rows per pass of the gather / scatter copies (loads in flight per thread)
#endif

__global__ void es_scatter_kernel(const float* __restrict__ post_s, const uint8_t* ok_s, const int32_t* it_s, const int32_t* map,
                                  const uint32_t* cont, float* __restrict__ post_out, uint8_t* ok_out, int32_t* it_out, int N,
                                  int gamma) {
  const int pl = blockIdx.x * blockDim.x + threadIdx.x;
  if (pl >= gamma) return;
  const int m = map[pl];
  if (m < 0) return;
  if (cont && ((cont[pl >> 5] >> (pl & 31)) & 1u)) return;
  if (blockIdx.y == 0) {
    ok_out[m] = ok_s[pl];
    it_out[m] = it_s[pl];
  }
  // ES_ROWS rows per pass: their loads are all in flight before the stores
  const int step = gridDim.y;
  int n = blockIdx.y;
  for (; n + (ES_ROWS - 1) * step < N; n += ES_ROWS * step) {
    float v[ES_ROWS];
#pragma unroll
    for (int k = 0; k < ES_ROWS; ++k) v[k] = post_s[(size_t)(n + k * step) * gamma + pl];
#pragma unroll
    for (int k = 0; k < ES_ROWS; ++k) post_out[(size_t)(n + k * step) * gamma + m] = v[k];
  }
  for (; n < N; n += step) post_out[(size_t)n * gamma + m] = post_s[(size_t)n * gamma + pl];
}

// continuing lanes' packages (rows [0, E)) and LLRs (rows [E, E + N)) into the next set
__device__ __forceinline__ void gather_rows(const float* __restrict__ src_rows, float* __restrict__ dst_rows,
                                            int rows, int gamma, int sp, int dp) {
  const int step = gridDim.y;
  int r = blockIdx.y;
  for (; r + (ES_ROWS - 1) * step < rows; r += ES_ROWS * step) {
    float v[ES_ROWS];
#pragma unroll
    for (int k = 0; k < ES_ROWS; ++k) v[k] = src_rows[(size_t)(r + k * step) * gamma + sp];
#pragma unroll
    for (int k = 0; k < ES_ROWS; ++k) dst_rows[(size_t)(r + k * step) * gamma + dp] = v[k];
  }
  for (; r < rows; r += step) dst_rows[(size_t)r * gamma + dp] = src_rows[(size_t)r * gamma + sp];
}

__global__ void es_gather_kernel(const float* __restrict__ msgs_s, float* __restrict__ msgs_d,
                                 const float* __restrict__ mu_s, float* __restrict__ mu_d, const int32_t* src,
                                 const int32_t* count, int E, int N, int gamma, int H) {
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= *count) return;
  const int sp = src[i], dp = (i & 1) * H + (i >> 1);
  gather_rows(msgs_s, msgs_d, E, gamma, sp, dp);
  gather_rows(mu_s, mu_d, N, gamma, sp, dp);
}

struct Set {
  float* msgs;
  float* mu;
  float* post;
  uint32_t* hb;
  uint8_t* ok;
  int32_t* its;
  int32_t* map;   // null: identity (the caller's arrays)
};

int n_checkpoints(int iters, int* ck) {
  int n = 0;
  for (int c : CHECKPOINTS)
    if (c < iters && n < MAX_CHECKPOINTS) ck[n++] = c;
  return n;
}

size_t al64(size_t w) { return (w + 63) / 64 * 64; }

}  // namespace

// from 1024 lanes up: each half then has >= 4 lane groups of 128, so packing
// can shrink the work (at 256 / 512 lanes it measured slower than the plain
// early-stop decode, profiles/r02/es_compaction.md)
constexpr int ES_COMPACT_MIN_GAMMA = 1024;

bool es_compact_eligible(const qc_plan* p, int gamma, int iters) {
  int ck[MAX_CHECKPOINTS];
  return agg_es_eligible(p, gamma) && gamma >= ES_COMPACT_MIN_GAMMA && gamma <= 65536 &&
         n_checkpoints(iters, ck) > 0;
}

// scratch words: two lane sets (mu, post: N x gamma; hb: N x gamma/32; ok;
// iterations; map), a second package store (E x gamma), the compaction list
size_t es_compact_words(const qc_plan* p, int gamma) {
  const size_t G = (size_t)gamma, N = (size_t)p->N, E = (size_t)p->E, W = G / 32;
  const size_t set = al64(N * G) * 2 + al64(N * W) + al64(G / 4) + al64(G) * 2;
  return 2 * set + al64(E * G) + al64(G) + 64 + al64(W);
}

int run_agg_decode_es_compact(const qc_plan* p, int gamma, int iters, float* msgs, const float* mu, float* post,
                              uint32_t* hb, uint32_t* work, uint32_t* scratch, uint8_t* ok, int32_t* iters_run,
                              cudaStream_t s) {
  int ck[MAX_CHECKPOINTS];
  const int nck = n_checkpoints(iters, ck);
  const int G = gamma, W = G / 32, H = G / 2, N = p->N, E = p->E;
  uint32_t* es = work;
  float* agg = reinterpret_cast<float*>(work + work_head_words(G));
  uint32_t* act[2] = {es, es + W};
  uint32_t* bad[2] = {es + 2 * W, es + 3 * W};
  uint32_t* bad_fin = es + 4 * W;
  // carve the scratch
  Set sets[3];
  sets[0] = Set{msgs, const_cast<float*>(mu), post, hb, ok, iters_run, nullptr};
  uint32_t* q = scratch;
  auto take = [&](size_t words) { uint32_t* r = q; q += al64(words); return r; };
  for (int k = 1; k <= 2; ++k) {
    Set& st = sets[k];
    st.mu = reinterpret_cast<float*>(take((size_t)N * G));
    st.post = reinterpret_cast<float*>(take((size_t)N * G));
    st.hb = take((size_t)N * W);
    st.ok = reinterpret_cast<uint8_t*>(take((size_t)G / 4));
    st.its = reinterpret_cast<int32_t*>(take((size_t)G));
    st.map = reinterpret_cast<int32_t*>(take((size_t)G));
  }
  float* msgs_x = reinterpret_cast<float*>(take((size_t)E * G));
  int32_t* src = reinterpret_cast<int32_t*>(take((size_t)G));
  int32_t* count = reinterpret_cast<int32_t*>(take(64));
  uint32_t* cont = take((size_t)W);
  sets[1].msgs = msgs_x;      // segments alternate package stores and lane sets 1, 2
  sets[2].msgs = msgs;

  cudaMemsetAsync(bad_fin, 0, sizeof(uint32_t) * W, s);
  int rc;
  int t0 = 1, cur = 0;
  const int gy = 256;                       // row blocks of the scatter / gather grids
  for (int k = 0; k <= nck; ++k) {
    const int t1 = k < nck ? ck[k] : iters;
    Set& S = sets[cur];
    // the first compacted segment keeps most lanes (62% at 3.2 dB, ~90% at 3.0
    // dB): full grids whose dead rows exit at once; later ones few: capped grids
    // walking the live blocks (profiles/r02/es_compaction.md)
    if ((rc = run_agg_es_segment(p, G, t0, t1, iters, S.msgs, S.mu, agg, S.post, S.hb, es, S.its, s,
                                 (cur == 0 || !ES_LIVE) ? nullptr : count, k >= ES_LOOP_FROM ? 1 : 0)))
      return rc;
    if (k == nck) {
      if ((rc = launch_es_tail(p, G, iters, act, bad, bad_fin, S.ok, S.its, S.post, S.hb, s))) return rc;
      if (cur != 0) {
        es_scatter_kernel<<<dim3((G + 127) / 128, gy), 128, 0, s>>>(S.post, S.ok, S.its, S.map, nullptr, post, ok,
                                                                    iters_run, N, G);
        if ((rc = check_launch("es_scatter"))) return rc;
      }
      break;
    }
    // checkpoint t1: outcome, compaction list, next set's state
    if ((rc = launch_syndrome_ext(p, G, S.hb, bad_fin, s))) return rc;
    const int nxt = cur == 1 ? 2 : 1;
    Set& D = sets[nxt];
    CkArgs a{};
    a.act_a = act[(t1 - 1) & 1];
    a.act_b = act[t1 & 1];
    a.bad_b = bad[(t1 - 1) & 1];
    a.bad_fin = bad_fin;
    a.ok = S.ok;
    a.iters_run = S.its;
    a.map = S.map;
    a.cont = cont;
    a.src = src;
    a.count = count;
    a.map_next = D.map;
    a.iters_next = D.its;
    const int tn = t1 + 1;
    a.act_set = act[tn & 1];
    a.bad_ones = bad[(tn - 1) & 1];
    a.bad_zero = bad[tn & 1];
    a.bad_fin_zero = bad_fin;
    a.W = W;
    a.WH = W / 2;
    a.H = H;
    a.gamma = G;
    a.c = t1;
    a.iters = iters;
    const size_t smem = sizeof(uint32_t) * W;
    es_ckpt_kernel<<<1, CK_THREADS, smem, s>>>(a);
    if ((rc = check_launch("es_ckpt"))) return rc;
    if (cur != 0) {
      es_scatter_kernel<<<dim3((G + 127) / 128, gy), 128, 0, s>>>(S.post, S.ok, S.its, S.map, cont, post, ok,
                                                                  iters_run, N, G);
      if ((rc = check_launch("es_scatter"))) return rc;
    }
    es_gather_kernel<<<dim3((G + 255) / 256, 1024), 256, 0, s>>>(S.msgs, D.msgs, S.mu, D.mu, src, count, E, N, G, H);
    if ((rc = check_launch("es_gather"))) return rc;
    t0 = tn;
    cur = nxt;
  }
  if (nck > 0) {       // decisions of every lane from its recorded posterior (bp.py:191-210 sign rule)
    if ((rc = launch_hard_bits_ext(p, G, post, hb, s))) return rc;
  }
  return 0;
}

int es_compact_launches(const qc_plan* p, int gamma, int iters) {
  int ck[MAX_CHECKPOINTS];
  const int nck = n_checkpoints(iters, ck);
  (void)p;
  (void)gamma;
  // per segment its first check pass + 2 per iteration (the last one variable
  // only); per checkpoint syndrome, ckpt, gather, and a scatter from the second
  // on; tail (2); with checkpoints a final scatter and the hard-bit rebuild
  return (nck + 1) + 2 * iters + 3 * nck + (nck > 0 ? nck - 1 : 0) + 2 + (nck > 0 ? 2 : 0);
}

}  // namespace qcb

extern "C" {

size_t qc_decode_es_scratch_words(const qc_plan* p, int gamma) {
  if (!p || gamma <= 0 || gamma % 32 || !qcb::agg_es_eligible(p, gamma) || gamma < qcb::ES_COMPACT_MIN_GAMMA)
    return 0;
  return qcb::es_compact_words(p, gamma);
}

}  // extern "C"
