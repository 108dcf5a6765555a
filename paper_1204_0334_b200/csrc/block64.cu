// Float64 "conformance" build of the block decoder: the reference's own
// arithmetic, on the GPU, for callers that rely on its 1e-12 tolerances.
//
// Check rule exactly as /root/reference/pkg/src/qcldpc/bp.py:134-162:
//   t_k = tanh(0.5 beta_k); forward / backward exclusive products in the same
//   sequential order (bp.py:120-131); clip to +-(1 - 1e-12); alpha = 2 atanh;
//   clip +-50.  Variable rule as bp.py:165-188 (running total in increasing
//   edge order, beta = clip(total - alpha), posterior = clip(total)).
// Differences from numpy are only the libm ulps of tanh/atanh (CUDA's double
// tanh/atanh vs numpy's SIMD ones): messages agree to ~1e-15 relative.
// One thread per (node, lane); packages are gamma doubles, edge-major.
#include <cuda_runtime.h>

#include <algorithm>

#include "common.cuh"
#include "plan.h"

using namespace qcb;

namespace {

constexpr double L_MAX64 = 50.0;
constexpr double CLAMP64 = 1.0 - 1e-12;

__device__ __forceinline__ double clampd(double x, double lim) { return fmin(fmax(x, -lim), lim); }

__device__ __forceinline__ bool lane_on(const uint32_t* active, int g) {
  return !active || ((active[g >> 5] >> (g & 31)) & 1u);
}

template <int DC, bool REG>
__global__ void __launch_bounds__(THREADS) cnu64_kernel(double* msgs, const int32_t* check_ptr, const uint32_t* active,
                                                        const int32_t* done, int M, int gamma) {
  if (done && *done) return;
  long long tid = (long long)blockIdx.x * blockDim.x + threadIdx.x;
  if (tid >= (long long)M * gamma) return;
  int m = (int)(tid / gamma), g = (int)(tid - (long long)m * gamma);
  if (!lane_on(active, g)) return;
  int e0, deg;
  if constexpr (REG) { e0 = m * DC; deg = DC; }
  else { e0 = check_ptr[m]; deg = check_ptr[m + 1] - e0; }
  double t[DC];
#pragma unroll
  for (int k = 0; k < DC; ++k)
    t[k] = (k < deg) ? tanh(__dmul_rn(0.5, msgs[(size_t)(e0 + k) * gamma + g])) : 1.0;
  double fwd[DC];
  fwd[0] = 1.0;
#pragma unroll
  for (int k = 1; k < DC; ++k) fwd[k] = __dmul_rn(fwd[k - 1], t[k - 1]);
  double bwd = 1.0;   // bwd[k] for k = deg-1 .. 0
#pragma unroll
  for (int k = DC - 1; k >= 0; --k) {
    if (k < deg) {
      double pr = clampd(__dmul_rn(fwd[k], bwd), CLAMP64);
      double a = clampd(__dmul_rn(2.0, atanh(pr)), L_MAX64);
      bwd = __dmul_rn(bwd, t[k]);
      msgs[(size_t)(e0 + k) * gamma + g] = a;
    }
  }
}

template <int DV, bool QC>
__global__ void __launch_bounds__(THREADS) vnu64_kernel(double* msgs, const double* mu, double* post, uint32_t* hb,
                                                        const int32_t* var_pad, const uint32_t* active,
                                                        const int32_t* done, int N, int gamma, int dv,
                                                        int write_beta) {
  if (done && *done) return;
  long long tid = (long long)blockIdx.x * blockDim.x + threadIdx.x;
  bool valid = tid < (long long)N * gamma;
  int n = valid ? (int)(tid / gamma) : 0, g = valid ? (int)(tid - (long long)n * gamma) : 0;
  // write_beta bit 0: write beta packages (active lanes only); bit 1: posteriors
  // for every lane, frozen ones included (public single step, bp.py:183)
  bool on = valid && lane_on(active, g);
  bool calc = valid && (on || (write_beta & 2));
  unsigned bit = 0;
  if (calc) {
    int e[DV];
    double a[DV];
    double tot = mu[(size_t)n * gamma + g];
#pragma unroll
    for (int j = 0; j < DV; ++j) {
      e[j] = j < dv ? var_pad[(size_t)n * dv + j] : -1;
      a[j] = e[j] >= 0 ? msgs[(size_t)e[j] * gamma + g] : 0.0;
      tot = __dadd_rn(tot, a[j]);        // pads add 0.0 (bp.py:227-230)
    }
    if (on && (write_beta & 1)) {
#pragma unroll
      for (int j = 0; j < DV; ++j)
        if (e[j] >= 0) msgs[(size_t)e[j] * gamma + g] = clampd(__dsub_rn(tot, a[j]), L_MAX64);
    }
    double p = clampd(tot, L_MAX64);
    if (post) post[(size_t)n * gamma + g] = p;
    bit = p < 0.0 ? 1u : 0u;
  }
  if (hb) {
    unsigned w = __ballot_sync(0xffffffffu, bit);   // 32 consecutive lanes of one variable
    if (valid && (threadIdx.x & 31) == 0) hb[(size_t)n * (gamma >> 5) + (g >> 5)] = w;
  }
}

__global__ void init64_kernel(const double* mu, double* msgs, const int32_t* edge_var, int E, int gamma) {
  long long tid = (long long)blockIdx.x * blockDim.x + threadIdx.x;
  if (tid >= (long long)E * gamma) return;
  int e = (int)(tid / gamma), g = (int)(tid - (long long)e * gamma);
  msgs[tid] = mu[(size_t)edge_var[e] * gamma + g];
}

__global__ void lane_major64_kernel(const double* post, double* post_out, uint8_t* bits_out, int N, int gamma,
                                    int gamma_out) {
  __shared__ double tile[32][33];
  int n0 = blockIdx.x * 32, g0 = blockIdx.y * 32;
  for (int dy = threadIdx.y; dy < 32; dy += blockDim.y) {
    int n = n0 + dy, g = g0 + threadIdx.x;
    tile[dy][threadIdx.x] = (n < N) ? post[(size_t)n * gamma + g] : 0.0;
  }
  __syncthreads();
  for (int dy = threadIdx.y; dy < 32; dy += blockDim.y) {
    int g = g0 + dy, n = n0 + threadIdx.x;
    if (g < gamma_out && n < N) {
      double v = tile[threadIdx.x][dy];
      if (post_out) post_out[(size_t)g * N + n] = v;
      if (bits_out) bits_out[(size_t)g * N + n] = v < 0.0 ? 1 : 0;
    }
  }
}

__global__ void mu64_from_lane_major_kernel(const double* x, double* mu, int N, int gamma, int gamma_in,
                                            double sigma, int clip) {
  long long tid = (long long)blockIdx.x * blockDim.x + threadIdx.x;
  if (tid >= (long long)N * gamma) return;
  int n = (int)(tid / gamma), g = (int)(tid - (long long)n * gamma);
  double v = L_MAX64;
  if (g < gamma_in) {
    v = x[(size_t)g * N + n];
    if (sigma > 0.0) v = __ddiv_rn(__dmul_rn(2.0, v), __dmul_rn(sigma, sigma));
    if (clip) v = clampd(v, L_MAX64);
  }
  mu[tid] = v;
}

// early-stop helpers shared with the fp32 path are re-declared here (tiny)
__global__ void es64_update_kernel(uint32_t* active, uint32_t* bad, int32_t* iters_run, int32_t* done, int W,
                                   int it) {
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

__global__ void es64_start_kernel(uint32_t* active, uint32_t* bad, int32_t* iters_run, int32_t* done, int W,
                                  int iters) {
  for (int w = threadIdx.x; w < W; w += blockDim.x) {
    active[w] = 0xffffffffu;
    bad[w] = 0;
    for (int b = 0; b < 32; ++b) iters_run[w * 32 + b] = iters;
  }
  if (threadIdx.x == 0) *done = 0;
}

__global__ void syndrome64_kernel(const uint32_t* hb, uint32_t* bad, const int32_t* check_ptr,
                                  const int32_t* edge_var, int M, int W, const int32_t* done) {
  if (done && *done) return;
  long long tid = (long long)blockIdx.x * blockDim.x + threadIdx.x;
  if (tid >= (long long)M * W) return;
  int m = (int)(tid / W), w = (int)(tid - (long long)m * W);
  uint32_t par = 0;
  for (int k = check_ptr[m]; k < check_ptr[m + 1]; ++k) par ^= hb[(size_t)edge_var[k] * W + w];
  if (par) atomicOr(bad + w, par);
}

__global__ void ok64_kernel(const uint32_t* bad, const uint32_t* active, uint8_t* ok, int32_t* iters_run,
                            int gamma, int iters, int fill) {
  int g = blockIdx.x * blockDim.x + threadIdx.x;
  if (g >= gamma) return;
  uint32_t b = active ? active[g >> 5] : bad[g >> 5];
  ok[g] = ((b >> (g & 31)) & 1u) ? 0 : 1;
  if (fill) iters_run[g] = iters;
}

__global__ void hb64_kernel(const double* post, uint32_t* hb, int N, int gamma) {
  long long tid = (long long)blockIdx.x * blockDim.x + threadIdx.x;
  bool valid = tid < (long long)N * gamma;
  unsigned bit = valid && post[tid] < 0.0 ? 1u : 0u;
  unsigned w = __ballot_sync(0xffffffffu, bit);
  if (valid && (threadIdx.x & 31) == 0) hb[tid >> 5] = w;
}

int bucket(int d) {
  static const int B[] = {4, 8, 16, 24, 32};
  for (int b : B)
    if (d <= b) return b;
  return -1;
}

template <int DC>
void cnu64_dc(const qc_plan* p, double* msgs, const uint32_t* active, const int32_t* done, int gamma, cudaStream_t s) {
  unsigned nb = blocks_for((long long)p->M * gamma);
  if (p->check_regular == DC) cnu64_kernel<DC, true><<<nb, THREADS, 0, s>>>(msgs, p->d_check_ptr, active, done, p->M, gamma);
  else cnu64_kernel<DC, false><<<nb, THREADS, 0, s>>>(msgs, p->d_check_ptr, active, done, p->M, gamma);
}

int launch_cnu64(const qc_plan* p, double* msgs, const uint32_t* active, const int32_t* done, int gamma,
                 cudaStream_t s) {
  if (p->E == 0 || p->M == 0) return 0;
  switch (bucket(p->dc_max)) {
    case 4: cnu64_dc<4>(p, msgs, active, done, gamma, s); break;
    case 8: cnu64_dc<8>(p, msgs, active, done, gamma, s); break;
    case 16: cnu64_dc<16>(p, msgs, active, done, gamma, s); break;
    case 24: cnu64_dc<24>(p, msgs, active, done, gamma, s); break;
    case 32: cnu64_dc<32>(p, msgs, active, done, gamma, s); break;
    default: return fail_arg("check degree > 32 is not supported");
  }
  return check_launch("cnu64");
}

int launch_vnu64(const qc_plan* p, double* msgs, const double* mu, double* post, uint32_t* hb,
                 const uint32_t* active, const int32_t* done, int gamma, int write_beta, cudaStream_t s) {
  if (p->N == 0) return 0;
  unsigned nb = blocks_for((long long)p->N * gamma);
  const int dv = p->dv_max;
  if (dv <= 4) vnu64_kernel<4, false><<<nb, THREADS, 0, s>>>(msgs, mu, post, hb, p->d_var_pad, active, done, p->N, gamma, dv, write_beta);
  else if (dv <= 8) vnu64_kernel<8, false><<<nb, THREADS, 0, s>>>(msgs, mu, post, hb, p->d_var_pad, active, done, p->N, gamma, dv, write_beta);
  else if (dv <= 16) vnu64_kernel<16, false><<<nb, THREADS, 0, s>>>(msgs, mu, post, hb, p->d_var_pad, active, done, p->N, gamma, dv, write_beta);
  else return fail_arg("variable degree > 16 is not supported");
  return check_launch("vnu64");
}

int gamma_ok(int gamma) {
  if (gamma <= 0 || gamma % 32) return fail_arg("gamma must be a positive multiple of 32");
  return 0;
}

}  // namespace

extern "C" {

int qc64_init(const qc_plan* p, int gamma, const double* mu, double* msgs, void* stream) {
  if (int r = gamma_ok(gamma)) return r;
  if (!p || !mu || !msgs) return fail_arg("null argument");
  if (p->E == 0) return 0;
  init64_kernel<<<blocks_for((long long)p->E * gamma), THREADS, 0, as_stream(stream)>>>(mu, msgs, p->d_edge_var,
                                                                                       p->E, gamma);
  return check_launch("qc64_init");
}

int qc64_cnu(const qc_plan* p, int gamma, double* msgs, const uint32_t* active, void* stream) {
  if (int r = gamma_ok(gamma)) return r;
  if (!p || !msgs) return fail_arg("null argument");
  return launch_cnu64(p, msgs, active, nullptr, gamma, as_stream(stream));
}

int qc64_vnu(const qc_plan* p, int gamma, double* msgs, const double* mu, double* post, uint32_t* hb,
             const uint32_t* active, void* stream) {
  if (int r = gamma_ok(gamma)) return r;
  if (!p || !msgs || !mu) return fail_arg("null argument");
  return launch_vnu64(p, msgs, mu, post, hb, active, nullptr, gamma, 3, as_stream(stream));
}

int qc64_hard_bits(const qc_plan* p, int gamma, const double* post, uint32_t* hb, void* stream) {
  if (int r = gamma_ok(gamma)) return r;
  if (!p || !post || !hb) return fail_arg("null argument");
  hb64_kernel<<<blocks_for((long long)p->N * gamma), THREADS, 0, as_stream(stream)>>>(post, hb, p->N, gamma);
  return check_launch("qc64_hard_bits");
}

int qc64_decode(const qc_plan* p, int gamma, int iters, int early_stop, const double* mu, double* msgs,
                double* post, uint32_t* hb, uint32_t* work, uint8_t* ok, int32_t* iters_run, void* stream) {
  if (int r = gamma_ok(gamma)) return r;
  if (iters < 1) return fail_arg("need at least one iteration");
  if (!p || !mu || !msgs || !post || !hb || !work || !ok || !iters_run) return fail_arg("null argument");
  cudaStream_t s = as_stream(stream);
  const int W = gamma / 32;
  uint32_t* bad = work;
  uint32_t* active = work + W;
  int32_t* done = reinterpret_cast<int32_t*>(work + 2 * W);
  int rc;
  if (p->E) init64_kernel<<<blocks_for((long long)p->E * gamma), THREADS, 0, s>>>(mu, msgs, p->d_edge_var, p->E, gamma);
  if (!early_stop) {
    cudaMemsetAsync(bad, 0, sizeof(uint32_t) * W, s);
    for (int it = 1; it <= iters; ++it) {
      if ((rc = launch_cnu64(p, msgs, nullptr, nullptr, gamma, s))) return rc;
      if ((rc = launch_vnu64(p, msgs, mu, it == iters ? post : nullptr, it == iters ? hb : nullptr, nullptr, nullptr,
                             gamma, 1, s)))
        return rc;
    }
    if (p->M)
      syndrome64_kernel<<<blocks_for((long long)p->M * W), THREADS, 0, s>>>(hb, bad, p->d_check_ptr, p->d_edge_var,
                                                                          p->M, W, nullptr);
    ok64_kernel<<<blocks_for(gamma), THREADS, 0, s>>>(bad, nullptr, ok, iters_run, gamma, iters, 1);
  } else {
    es64_start_kernel<<<1, 256, 0, s>>>(active, bad, iters_run, done, W, iters);
    for (int it = 1; it <= iters; ++it) {
      if ((rc = launch_cnu64(p, msgs, active, done, gamma, s))) return rc;
      if ((rc = launch_vnu64(p, msgs, mu, post, hb, active, done, gamma, 1, s))) return rc;
      if (p->M)
        syndrome64_kernel<<<blocks_for((long long)p->M * W), THREADS, 0, s>>>(hb, bad, p->d_check_ptr,
                                                                            p->d_edge_var, p->M, W, done);
      es64_update_kernel<<<1, 256, 0, s>>>(active, bad, iters_run, done, W, it);
    }
    ok64_kernel<<<blocks_for(gamma), THREADS, 0, s>>>(bad, active, ok, iters_run, gamma, iters, 0);
    hb64_kernel<<<blocks_for((long long)p->N * gamma), THREADS, 0, s>>>(post, hb, p->N, gamma);
  }
  return check_launch("qc64_decode");
}

int qc64_lane_major(int n, int gamma, int gamma_out, const double* post, double* post_out, uint8_t* bits_out,
                    void* stream) {
  if (int r = gamma_ok(gamma)) return r;
  if (n < 0 || !post || gamma_out < 0 || gamma_out > gamma) return fail_arg("bad lane_major arguments");
  if (n == 0 || gamma_out == 0) return 0;
  dim3 grid((n + 31) / 32, (gamma_out + 31) / 32), block(32, 8);
  lane_major64_kernel<<<grid, block, 0, as_stream(stream)>>>(post, post_out, bits_out, n, gamma, gamma_out);
  return check_launch("qc64_lane_major");
}

int qc64_mu_from_lane_major(int n, int gamma, int gamma_in, const double* x, double sigma, int clip, double* mu,
                            void* stream) {
  if (int r = gamma_ok(gamma)) return r;
  if (n < 0 || gamma_in < 0 || gamma_in > gamma || (!x && gamma_in) || !mu) return fail_arg("bad mu arguments");
  if (n == 0) return 0;
  mu64_from_lane_major_kernel<<<blocks_for((long long)n * gamma), THREADS, 0, as_stream(stream)>>>(x, mu, n, gamma,
                                                                                                 gamma_in, sigma, clip);
  return check_launch("qc64_mu_from_lane_major");
}

}  // extern "C"
