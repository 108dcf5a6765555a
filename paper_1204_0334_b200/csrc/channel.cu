// On-device AWGN/BPSK channel + LLRs (replaces channel.py:61-105 and bp.py:54-56).
//
// Sample position q of lane l is 64-bit word q mod 4 of Philox4x64-10 with
// key = seed (128-bit, two words) and counter = [q//4 + 1, l, 0, 0] -- numpy's
// Philox pre-increments its 256-bit counter before producing a block, and the
// reference seeds it at (l << 64) + start//4 (channel.py:70-74).  The word
// maps to u = ((w >> 11) + 0.5) 2^-53 and g = ndtri(u) (Cephes inverse normal
// CDF, the algorithm behind scipy.special.ndtri), all in fp64; then
// y = 1 + sigma g and mu = clip(2 y / sigma^2, +-50) in the reference's
// operation order, rounded once to fp32 for the message store.
//
// Thread mapping: consecutive threads = consecutive lanes of one Philox block
// (4 consecutive positions), so the variable-major mu store (n, gamma) is a
// coalesced 128-byte row per position.
#include <cuda_runtime.h>

#include "common.cuh"
#include "philox.cuh"

using namespace qcb;

namespace {

struct ChanArgs {
  uint64_t k0, k1, lane0, start;
  const uint64_t* lane0_dev;   // optional: lane0 = *lane0_dev
  const int64_t* t_dev;     // optional: start += (*t_dev + t_add) * t_mul
  long long t_add, t_mul;
  int n, gamma;
  double sigma;
  float* mu_vm;
  double* y_lm;
  double* g_lm;
};

// Each warp runs the two ndtri regions over compacted lists of its 128
// samples (central ~73%, tail ~27%): ceil(n_central/32) + ceil(n_tail/32)
// (typically 3 + 2) warp-rounds instead of 4 + 4 with both branches taken per
// position -- the kernel is issue-bound on fp64 (ncu: issue slots 79%).
__global__ void __launch_bounds__(THREADS) channel_kernel(ChanArgs a) {
  __shared__ double qu[THREADS / 32][128];        // central from the front, tail from the back
  __shared__ unsigned char qslot[THREADS / 32][128];
  __shared__ double res[THREADS / 32][128];       // slot k*32 + lane
  pdl_trigger();
  pdl_wait();
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
  // 32-bit index math (the host keeps blocks x gamma < 2^31): a 64-bit
  // division / remainder per thread was ~8% of the kernel's instructions
  const unsigned tid = blockIdx.x * blockDim.x + threadIdx.x;
  if (a.t_dev) a.start += (uint64_t)((*a.t_dev + a.t_add) * a.t_mul);
  if (a.lane0_dev) a.lane0 = *a.lane0_dev;
  const uint64_t first = a.start >> 2;
  const unsigned off = (unsigned)(a.start & 3);
  const unsigned total = ((off + (unsigned)a.n + 3u) >> 2) * (unsigned)a.gamma;
  if ((tid & ~31u) >= total) return;    // whole warp out of range
  const bool valid = tid < total;
  unsigned g = 0, b = 0;
  if (valid) {
    b = tid / (unsigned)a.gamma;
    g = tid - b * (unsigned)a.gamma;
  }
  uint64_t w[4] = {0, 0, 0, 0};
  if (valid) philox4x64_10(first + (uint64_t)b + 1ull, a.lane0 + (uint64_t)g, 0ull, 0ull, a.k0, a.k1, w);
  const unsigned lt = (1u << lane) - 1u;
  int nc = 0, nt = 0;
  bool ok[4];
  int pos[4];
#pragma unroll
  for (int k = 0; k < 4; ++k) {
    pos[k] = (int)(b * 4u + (unsigned)k) - (int)off;      // (first + b) * 4 + k - start
    ok[k] = valid && pos[k] >= 0 && pos[k] < a.n;
    const double u = word_to_uniform(w[k]);
    const bool cen = ok[k] && ndtri_is_central(u);
    const bool tl = ok[k] && !cen;
    const unsigned mc = __ballot_sync(0xffffffffu, cen), mt = __ballot_sync(0xffffffffu, tl);
    if (cen) {
      const int o = nc + __popc(mc & lt);
      qu[wid][o] = u;
      qslot[wid][o] = (unsigned char)(k * 32 + lane);
    }
    if (tl) {
      const int o = 127 - (nt + __popc(mt & lt));
      qu[wid][o] = u;
      qslot[wid][o] = (unsigned char)(k * 32 + lane);
    }
    nc += __popc(mc);
    nt += __popc(mt);
  }
  __syncwarp();
  for (int i = lane; i < nc; i += 32) res[wid][qslot[wid][i]] = ndtri_central(qu[wid][i]);
  for (int i = lane; i < nt; i += 32) res[wid][qslot[wid][127 - i]] = ndtri_tail(qu[wid][127 - i]);
  __syncwarp();
  const double s2 = __dmul_rn(a.sigma, a.sigma);
#pragma unroll
  for (int k = 0; k < 4; ++k) {
    if (!ok[k]) continue;
    const double gv = res[wid][k * 32 + lane];
    const double y = __dadd_rn(1.0, __dmul_rn(a.sigma, gv));
    if (a.g_lm) a.g_lm[(size_t)g * a.n + pos[k]] = gv;
    if (a.y_lm) a.y_lm[(size_t)g * a.n + pos[k]] = y;
    if (a.mu_vm) {
      double mu = __ddiv_rn(__dmul_rn(2.0, y), s2);
      mu = mu < -50.0 ? -50.0 : (mu > 50.0 ? 50.0 : mu);
      a.mu_vm[(size_t)pos[k] * a.gamma + g] = __double2float_rn(mu);
    }
  }
}

}  // namespace

namespace qcb {
int launch_channel(uint64_t k0, uint64_t k1, uint64_t lane0, uint64_t start, int n, int gamma,
                   double sigma, float* mu_vm, double* y_lm, double* g_lm, cudaStream_t s) {
  ChanArgs a{k0, k1, lane0, start, nullptr, nullptr, 0, 0, n, gamma, sigma, mu_vm, y_lm, g_lm};
  long long nblk = (long long)(((start & 3) + (uint64_t)n + 3) >> 2);
  long long threads = nblk * gamma;
  if (threads == 0) return 0;
  if (threads >= (1ll << 31)) return fail_arg("channel: n x gamma too large for one launch");
  launch_pdl(channel_kernel, dim3(blocks_for(threads)), THREADS, s, a);
  return check_launch("channel");
}
// device-indexed variant for graph-captured slots: positions start at
// start + (*t_dev + t_add) * t_mul and/or the first lane is *lane0_dev.
int launch_channel_t(uint64_t k0, uint64_t k1, uint64_t lane0, const uint64_t* lane0_dev, uint64_t start,
                     const int64_t* t_dev, long long t_add, long long t_mul, int n, int gamma, double sigma,
                     float* mu_vm, cudaStream_t s) {
  if (!t_dev && !lane0_dev)
    return launch_channel(k0, k1, lane0, start + (uint64_t)(t_add * t_mul), n, gamma, sigma, mu_vm, nullptr,
                          nullptr, s);
  uint64_t st = start;
  if (!t_dev) st += (uint64_t)(t_add * t_mul);
  ChanArgs a{k0, k1, lane0, st, lane0_dev, t_dev, t_add, t_mul, n, gamma, sigma, mu_vm, nullptr, nullptr};
  // the start may be known only on the device: cover the worst-case block count
  long long threads = (long long)((n + 3) / 4 + 1) * gamma;
  if (threads == 0) return 0;
  if (threads >= (1ll << 31)) return fail_arg("channel: n x gamma too large for one launch");
  launch_pdl(channel_kernel, dim3(blocks_for(threads)), THREADS, s, a);
  return check_launch("channel");
}
}  // namespace qcb

extern "C" int qc_channel(uint64_t seed_lo, uint64_t seed_hi, uint64_t lane0, uint64_t start, int n,
                          int gamma, double sigma, float* mu_vm, double* y_lm, double* g_lm,
                          void* stream) {
  if (n < 0 || gamma < 1) return fail_arg("n must be >= 0 and gamma >= 1");
  if (mu_vm && gamma % 32) return fail_arg("variable-major mu output needs gamma % 32 == 0");
  return launch_channel(seed_lo, seed_hi, lane0, start, n, gamma, sigma, mu_vm, y_lm, g_lm,
                        as_stream(stream));
}

namespace {
__global__ void lane_advance_kernel(uint64_t* p, uint64_t k) { *p += k; }
}

extern "C" int qc_channel_dev(uint64_t seed_lo, uint64_t seed_hi, const uint64_t* lane0_dev, uint64_t start,
                              int n, int gamma, double sigma, float* mu_vm, void* stream) {
  if (!lane0_dev || !mu_vm) return fail_arg("null argument");
  if (n < 0 || gamma < 1 || gamma % 32) return fail_arg("n must be >= 0 and gamma a positive multiple of 32");
  return launch_channel_t(seed_lo, seed_hi, 0, lane0_dev, start, nullptr, 0, 0, n, gamma, sigma, mu_vm,
                          as_stream(stream));
}

extern "C" int qc_lane_advance(uint64_t* lane0_dev, uint64_t k, void* stream) {
  if (!lane0_dev) return fail_arg("null argument");
  lane_advance_kernel<<<1, 1, 0, as_stream(stream)>>>(lane0_dev, k);
  return check_launch("lane_advance");
}
