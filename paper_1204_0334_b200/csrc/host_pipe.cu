// Host-buffer decode pipeline: the reference's decode_batch / decode_llr_batch
// (/root/reference/pkg/src/qcldpc/bp.py:213-274) with caller-owned HOST arrays,
// lane-major in and out exactly as DecodeResult (bp.py:87-100).
//
// A batch of gamma codewords is cut into chunks that rotate over `slots` CUDA
// streams, each with its own device buffers and instantiated CUDA graphs of
// the whole flooding loop (qc_decode) for chunk sizes C/8, C/4, C/2 and C lanes
// (C = `chunk`).  The chunk plan ramps up and down through the smaller sizes
// (C/4, C/2, C, ..., C, C/2, C/4 for C = 512): small first and last chunks
// shorten the pipeline fill (first copy-in) and drain (last copy-outs),
// full-size chunks in between keep the decode kernels at their large-gamma
// efficiency.  Decodes run in chunk order on one decode stream
// (two decodes running concurrently interfere, tools/chain_probe.py);
// copy-ins are serialised too, so the first chunk is not slowed by later ones
// sharing the link; copies in both directions overlap the decodes.  Per chunk:
//   H2D of the received values (fp64, lane-major)
//   -> LLR scale/clip/transpose kernel -> graph (init + iters x (check, variable)
//      + hard decision + syndrome) -> lane-major fp64 posteriors + u8 bits
//   -> D2H of posteriors, bits, syndrome flags, iteration counts.
// While one chunk decodes, the next is copied in and the previous one is read
// back, so PCIe (55 GB/s each way on the B200 box, profiles/r01/pcie.json)
// overlaps the kernels.  Host arrays that are page-locked (cudaHostAlloc /
// torch pin_memory / cudaHostRegister) are DMA'd in place; pageable arrays go
// through per-slot pinned staging: the staging threads convert them to fp32
// LLRs on the way (half the staged and PCIe bytes, bit-identical to the device
// conversion).
#include <cuda_runtime.h>

#include <algorithm>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <string>
#include <thread>
#include <vector>

#include "common.cuh"
#include "plan.h"

namespace {

using namespace qcb;

struct Slot {
  cudaStream_t st = nullptr;
  cudaEvent_t done = nullptr;
  static constexpr int NG = 4;
  cudaGraphExec_t graph[NG] = {};   // C/8, C/4, C/2, C lanes
  int size[NG] = {};
  cudaEvent_t decoded = nullptr;   // end of this slot's last decode (on the decode stream)
  cudaEvent_t ready = nullptr;     // this slot's LLRs converted (decode may start)
  cudaEvent_t copied_in = nullptr; // end of this slot's last copy-in (serialises copy-ins)
  double* x = nullptr;          // (chunk, N) fp64 lane-major input
  float* mu = nullptr;          // (N, chunk) fp32 LLRs
  float* msgs = nullptr;        // (E, chunk) packages
  float* post = nullptr;        // (N, chunk) fp32 posteriors
  uint32_t* hb = nullptr;       // (N, chunk/32) hard-bit planes
  uint32_t* work = nullptr;     // qc_decode scratch
  uint32_t* es_scratch = nullptr;  // early stop with lane compaction (qc_decode_es), or null
  uint8_t* ok = nullptr;        // (chunk)
  int32_t* its = nullptr;       // (chunk)
  double* post_lm = nullptr;    // (chunk, N) fp64 lane-major posteriors
  uint8_t* bits_lm = nullptr;   // (chunk, N) u8 lane-major hard bits
  // page-locked staging (allocated on first use with a pageable array)
  float* h_llr = nullptr;       // (chunk, N) fp32 lane-major LLRs (pageable input, converted on the host)
  double* h_post = nullptr;
  uint8_t* h_bits = nullptr;
  uint8_t* h_ok = nullptr;      // always used (small)
  int32_t* h_its = nullptr;
  // chunk in flight: lanes [a, b) of the current call, or a < 0
  long long a = -1, b = -1;
};

void par_copy(void* dst, const void* src, size_t bytes) {
  const size_t MIN_PER_THREAD = size_t(8) << 20;
  unsigned hw = std::max(1u, std::thread::hardware_concurrency());
  size_t T = std::min<size_t>({hw, 16, std::max<size_t>(1, bytes / MIN_PER_THREAD)});
  if (T <= 1) {
    std::memcpy(dst, src, bytes);
    return;
  }
  std::vector<std::thread> th;
  size_t per = (bytes + T - 1) / T;
  per = (per + 4095) & ~size_t(4095);
  for (size_t t = 0; t < T; ++t) {
    size_t lo = t * per;
    if (lo >= bytes) break;
    size_t n = std::min(per, bytes - lo);
    th.emplace_back([=] { std::memcpy(static_cast<char*>(dst) + lo, static_cast<const char*>(src) + lo, n); });
  }
  for (auto& t : th) t.join();
}

// Pageable input: the LLR conversion of the device kernel
// (llr_from_lane_major_kernel, block.cu: mu = clip(2 y / sigma^2, +-50) in
// fp64, rounded once to fp32) done by the staging threads instead of a plain
// copy -- the same IEEE operations, so the same bits -- which halves the bytes
// written to the staging buffer and sent over PCIe.
// no-trapping-math lets gcc vectorise the compare/selects (divpd, cmppd);
// results are unchanged (IEEE division, NaN passes both compares unclamped)
__attribute__((optimize("no-trapping-math"))) void llr_range(float* __restrict dst, const double* __restrict src,
                                                             size_t lo, size_t hi, double sigma) {
  const double s2 = sigma * sigma;
  if (sigma > 0.0) {
    for (size_t i = lo; i < hi; ++i) {
      double t = (2.0 * src[i]) / s2;
      t = t < -50.0 ? -50.0 : t;
      t = t > 50.0 ? 50.0 : t;
      dst[i] = static_cast<float>(t);
    }
  } else {
    for (size_t i = lo; i < hi; ++i) {
      double t = src[i];
      t = t < -50.0 ? -50.0 : t;
      t = t > 50.0 ? 50.0 : t;
      dst[i] = static_cast<float>(t);
    }
  }
}

void par_llr(float* dst, const double* src, size_t n, double sigma) {
  const size_t MIN_PER_THREAD = size_t(1) << 20;   // elements
  unsigned hw = std::max(1u, std::thread::hardware_concurrency());
  size_t T = std::min<size_t>({hw, 16, std::max<size_t>(1, n / MIN_PER_THREAD)});
  auto work = [=](size_t lo, size_t hi) { llr_range(dst, src, lo, hi, sigma); };
  if (T <= 1) {
    work(0, n);
    return;
  }
  std::vector<std::thread> th;
  size_t per = (n + T - 1) / T;
  per = (per + 1023) & ~size_t(1023);
  for (size_t t = 0; t < T; ++t) {
    const size_t lo = t * per;
    if (lo >= n) break;
    th.emplace_back(work, lo, std::min(n, lo + per));
  }
  for (auto& t : th) t.join();
}

// fp32 lane-major LLRs (chunk rows of N) -> variable-major mu (N, gamma);
// lanes >= gamma_in get the neutral +50 like llr_from_lane_major_kernel
__global__ void lm32_to_vm_kernel(const float* x, float* mu, int N, int gamma, int gamma_in) {
  __shared__ float tile[32][33];
  const int n0 = blockIdx.x * 32, g0 = blockIdx.y * 32;
  for (int dy = threadIdx.y; dy < 32; dy += blockDim.y) {
    const int g = g0 + dy, n = n0 + threadIdx.x;
    tile[dy][threadIdx.x] = (g < gamma_in && n < N) ? x[(size_t)g * N + n] : 50.0f;
  }
  __syncthreads();
  for (int dy = threadIdx.y; dy < 32; dy += blockDim.y) {
    const int n = n0 + dy, g = g0 + threadIdx.x;
    if (n < N) mu[(size_t)n * gamma + g] = tile[threadIdx.x][dy];
  }
}

bool pinned_one(const void* p) {
  cudaPointerAttributes at;
  if (cudaPointerGetAttributes(&at, p) != cudaSuccess) {
    cudaGetLastError();
    return false;
  }
  return at.type == cudaMemoryTypeHost;
}

// page-locked iff both ends are (a view into one pinned allocation)
bool pinned(const void* p, size_t bytes) {
  if (!p || bytes == 0) return false;
  return pinned_one(p) && pinned_one(static_cast<const char*>(p) + bytes - 1);
}

#define HP_CK(expr)                                                                   \
  do {                                                                                \
    cudaError_t e_ = (expr);                                                          \
    if (e_ != cudaSuccess) return fail_rt(std::string(#expr) + ": " + cudaGetErrorString(e_)); \
  } while (0)

struct DeviceGuard {
  int prev = -1;
  explicit DeviceGuard(int dev) {
    if (cudaGetDevice(&prev) != cudaSuccess) prev = -1;
    if (prev != dev) cudaSetDevice(dev);
  }
  ~DeviceGuard() {
    int cur;
    if (prev >= 0 && cudaGetDevice(&cur) == cudaSuccess && cur != prev) cudaSetDevice(prev);
  }
};

}  // namespace

struct qc_host_dec {
  const qc_plan* plan = nullptr;
  int chunk = 0, iters = 0, early_stop = 0, device = 0;
  std::vector<Slot> slots;
  cudaStream_t dstream = nullptr;   // every chunk's decode graph, in chunk order
};

static void free_slot(Slot& s) {
  for (auto& g : s.graph)
    if (g) cudaGraphExecDestroy(g);
  if (s.done) cudaEventDestroy(s.done);
  if (s.decoded) cudaEventDestroy(s.decoded);
  if (s.copied_in) cudaEventDestroy(s.copied_in);
  if (s.ready) cudaEventDestroy(s.ready);
  if (s.st) cudaStreamDestroy(s.st);
  void* dev[] = {s.x, s.mu, s.msgs, s.post, s.hb, s.work, s.es_scratch, s.ok, s.its, s.post_lm, s.bits_lm};
  for (void* d : dev)
    if (d) cudaFree(d);
  void* host[] = {s.h_llr, s.h_post, s.h_bits, s.h_ok, s.h_its};
  for (void* h : host)
    if (h) cudaFreeHost(h);
  s = Slot{};
}

static int init_slot(qc_host_dec* h, Slot& s) {
  const qc_plan* p = h->plan;
  const size_t C = h->chunk, N = p->N, E = std::max(p->E, 1);
  HP_CK(cudaStreamCreateWithFlags(&s.st, cudaStreamNonBlocking));
  HP_CK(cudaEventCreateWithFlags(&s.done, cudaEventDisableTiming));
  HP_CK(cudaMalloc(&s.x, C * N * sizeof(double)));
  HP_CK(cudaMalloc(&s.mu, N * C * sizeof(float)));
  HP_CK(cudaMalloc(&s.msgs, E * C * sizeof(float)));
  HP_CK(cudaMalloc(&s.post, N * C * sizeof(float)));
  HP_CK(cudaMalloc(&s.hb, N * (C / 32) * sizeof(uint32_t)));
  HP_CK(cudaMalloc(&s.work, qc_decode_work_words(p, h->chunk) * sizeof(uint32_t)));
  if (h->early_stop) {
    const size_t nes = qc_decode_es_scratch_words(p, h->chunk);
    if (nes) {
      HP_CK(cudaMalloc(&s.es_scratch, nes * sizeof(uint32_t)));
      HP_CK(cudaMemsetAsync(s.es_scratch, 0, nes * sizeof(uint32_t), s.st));
    }
  }
  HP_CK(cudaMalloc(&s.ok, C));
  HP_CK(cudaMalloc(&s.its, C * sizeof(int32_t)));
  HP_CK(cudaMalloc(&s.post_lm, C * N * sizeof(double)));
  HP_CK(cudaMalloc(&s.bits_lm, C * N));
  HP_CK(cudaMallocHost(&s.h_ok, C));
  HP_CK(cudaMallocHost(&s.h_its, C * sizeof(int32_t)));
  HP_CK(cudaEventCreateWithFlags(&s.decoded, cudaEventDisableTiming));
  HP_CK(cudaEventCreateWithFlags(&s.copied_in, cudaEventDisableTiming));
  HP_CK(cudaEventCreateWithFlags(&s.ready, cudaEventDisableTiming));
  HP_CK(cudaMemsetAsync(s.msgs, 0, E * C * sizeof(float), s.st));
  // the flooding loop for each chunk size, captured once and replayed per chunk
  // (a size-c decode uses the slot's buffers with row stride c)
  for (int i = 0; i < Slot::NG; ++i) {
    const int c = h->chunk >> (Slot::NG - 1 - i);
    if (c < 32 || c % 32) continue;
    s.size[i] = c;
    cudaGraph_t g = nullptr;
    HP_CK(cudaStreamBeginCapture(s.st, cudaStreamCaptureModeThreadLocal));
    // early stop: lane compaction where the plan / size allow it (else qc_decode_es
    // falls back to qc_decode's early-stop path)
    int rc = (h->early_stop && s.es_scratch)
                 ? qc_decode_es(p, c, h->iters, s.mu, s.msgs, s.post, s.hb, s.work, s.es_scratch, s.ok, s.its,
                                nullptr, s.st)
                 : qc_decode(p, c, h->iters, h->early_stop, s.mu, s.msgs, s.post, s.hb, s.work, s.ok, s.its,
                             nullptr, s.st);
    cudaError_t ce = cudaStreamEndCapture(s.st, &g);
    if (rc) {
      if (g) cudaGraphDestroy(g);
      return rc;
    }
    if (ce != cudaSuccess) return fail_rt(std::string("graph capture: ") + cudaGetErrorString(ce));
    ce = cudaGraphInstantiate(&s.graph[i], g, 0);
    cudaGraphDestroy(g);
    if (ce != cudaSuccess) return fail_rt(std::string("graph instantiate: ") + cudaGetErrorString(ce));
  }
  HP_CK(cudaStreamSynchronize(s.st));
  return 0;
}

extern "C" {

int qc_host_create(const qc_plan* plan, int chunk, int slots, int iters, int early_stop, qc_host_dec** out) {
  if (!plan || !out) return fail_arg("null argument");
  if (chunk <= 0 || chunk % 32) return fail_arg("chunk must be a positive multiple of 32");
  if (slots < 1 || slots > 8) return fail_arg("slots must be in [1, 8]");
  if (iters < 1) return fail_arg("need at least one iteration");
  *out = nullptr;
  auto* h = new qc_host_dec();
  h->plan = plan;
  h->chunk = chunk;
  h->iters = iters;
  h->early_stop = early_stop ? 1 : 0;
  if (cudaGetDevice(&h->device) != cudaSuccess) {
    delete h;
    return fail_rt("no CUDA device");
  }
  h->slots.resize(slots);
  cudaError_t ce = cudaStreamCreateWithFlags(&h->dstream, cudaStreamNonBlocking);
  int rc = ce == cudaSuccess ? 0 : fail_rt(std::string("decode stream: ") + cudaGetErrorString(ce));
  for (auto& s : h->slots)
    if (!rc) rc = init_slot(h, s);
  if (rc) {
    for (auto& t : h->slots) free_slot(t);
    if (h->dstream) cudaStreamDestroy(h->dstream);
    delete h;
    return rc;
  }
  *out = h;
  return 0;
}

void qc_host_destroy(qc_host_dec* h) {
  if (!h) return;
  DeviceGuard g(h->device);
  if (h->dstream) cudaStreamSynchronize(h->dstream);
  for (auto& s : h->slots) {
    if (s.st) cudaStreamSynchronize(s.st);
    free_slot(s);
  }
  if (h->dstream) cudaStreamDestroy(h->dstream);
  delete h;
}

int qc_host_is_pinned(const void* p, size_t bytes) { return pinned(p, bytes) ? 1 : 0; }

int qc_host_dims(const qc_host_dec* h, int64_t* dims) {
  if (!h || !dims) return fail_arg("null argument");
  dims[0] = h->chunk;
  dims[1] = (int64_t)h->slots.size();
  dims[2] = h->iters;
  dims[3] = h->early_stop;
  dims[4] = h->device;
  return 0;
}

}  // extern "C"

namespace {

struct Call {
  qc_host_dec* h;
  int N;
  double* post;
  uint8_t* bits;
  uint8_t* ok;
  int64_t* its;
  bool pin_post, pin_bits;
};

// wait for the slot's chunk and move its results into the caller's arrays
int finish(const Call& c, Slot& s) {
  if (s.a < 0) return 0;
  HP_CK(cudaEventSynchronize(s.done));
  const size_t n = (size_t)(s.b - s.a) * c.N;
  if (c.post && !c.pin_post) par_copy(c.post + (size_t)s.a * c.N, s.h_post, n * sizeof(double));
  if (c.bits && !c.pin_bits) par_copy(c.bits + (size_t)s.a * c.N, s.h_bits, n);
  for (long long g = s.a; g < s.b; ++g) {
    if (c.ok) c.ok[g] = s.h_ok[g - s.a] ? 1 : 0;
    if (c.its) c.its[g] = s.h_its[g - s.a];
  }
  s.a = s.b = -1;
  return 0;
}

int run(qc_host_dec* h, const double* x, int gamma, double sigma, uint8_t* bits, double* post, uint8_t* ok,
        int64_t* iters_run) {
  const qc_plan* p = h->plan;
  const int N = p->N;
  const size_t row = (size_t)N;
  Call c{h, N, post, bits, ok, iters_run, pinned(post, (size_t)gamma * row * sizeof(double)),
         pinned(bits, (size_t)gamma * row)};
  const bool pin_in = pinned(x, (size_t)gamma * row * sizeof(double));
  const int S = (int)h->slots.size();
  const int C = h->chunk;
  // chunk plan: ramp up through the captured sizes from min(128, C/4) lanes
  // (C/4, C/2 for C = 512), full chunks, then ramp down the same sizes.  Each
  // ramp step's decode outlasts the next chunk's copy-in (head) or the
  // previous chunk's copy-out (tail), so only the first copy-in and the last
  // copy-out stay exposed (QCB_HOST_PROFILE=1 shows the split).
  std::vector<int> plan, ramp_sizes;
  const Slot& s0 = h->slots[0];
  for (int i = 0; i < Slot::NG - 1; ++i)
    if (s0.size[i] && s0.size[i] >= std::min(128, C / 4)) ramp_sizes.push_back(s0.size[i]);
  long long ramp_lanes = 0;
  for (int r : ramp_sizes) ramp_lanes += r;
  const bool ramp = C % 128 == 0 && C / 4 >= 32;
  if (!ramp_sizes.empty() && gamma >= 2 * ramp_lanes + C) {
    long long body = gamma - 2 * ramp_lanes;
    plan = ramp_sizes;
    for (; body >= C; body -= C) plan.push_back(C);
    if (body > 0) plan.push_back((int)body);
    plan.insert(plan.end(), ramp_sizes.rbegin(), ramp_sizes.rend());
  } else {
    long long rem = gamma;
    if (gamma <= C) {
      plan.push_back(gamma);
      rem = 0;
    }
    for (int c : {C / 4, C / 2})
      if (c >= 32 && c % 32 == 0 && rem > c + C / 4) {
        plan.push_back(c);
        rem -= c;
      }
    while (rem > C + C / 4) {
      plan.push_back(C);
      rem -= C;
    }
    if (rem > C / 4 && ramp && !plan.empty()) {
      plan.push_back((int)(rem - C / 4));
      plan.push_back(C / 4);
    } else {
      while (rem > 0) {
        const int c = (int)std::min<long long>(rem, C);
        plan.push_back(c);
        rem -= c;
      }
    }
  }
  const long long nchunks = (long long)plan.size();
  // QCB_HOST_PROFILE=1: per-call breakdown on stderr (decode graph time vs the
  // whole call on the device clock)
  static const bool prof = [] {
    const char* e = std::getenv("QCB_HOST_PROFILE");
    return e && *e == '1';
  }();
  std::vector<cudaEvent_t> pev;
  auto tev = [&](cudaStream_t st) -> int {
    cudaEvent_t e;
    HP_CK(cudaEventCreate(&e));
    HP_CK(cudaEventRecord(e, st));
    pev.push_back(e);
    return 0;
  };
  cudaEvent_t prev_copied = nullptr;
  long long a = 0;
  for (long long k = 0; k < nchunks; ++k) {
    Slot& s = h->slots[k % S];
    if (int rc = finish(c, s)) return rc;
    const long long b = a + plan[k];
    const int gi = plan[k];
    int gsel = Slot::NG - 1;                        // smallest captured size holding the chunk
    while (gsel > 0 && s.size[gsel - 1] >= gi) --gsel;
    const int cs = s.size[gsel];
    const double* src = x + (size_t)a * row;
    if (!pin_in) {
      if (!s.h_llr) HP_CK(cudaMallocHost(&s.h_llr, (size_t)C * row * sizeof(float)));
      par_llr(s.h_llr, src, (size_t)gi * row, sigma);
    }
    // copy-ins in chunk order, one at a time: the first chunk gets the whole link
    if (prev_copied) HP_CK(cudaStreamWaitEvent(s.st, prev_copied, 0));
    if (prof && k == 0) tev(s.st);
    if (pin_in)
      HP_CK(cudaMemcpyAsync(s.x, src, (size_t)gi * row * sizeof(double), cudaMemcpyHostToDevice, s.st));
    else
      HP_CK(cudaMemcpyAsync(s.x, s.h_llr, (size_t)gi * row * sizeof(float), cudaMemcpyHostToDevice, s.st));
    HP_CK(cudaEventRecord(s.copied_in, s.st));
    prev_copied = s.copied_in;
    // the LLR conversion only needs this chunk's copy-in; the decode graphs
    // all run on one stream (no cross-stream hand-off between decodes)
    if (pin_in) {
      if (int rc = qc_llr_from_lane_major(N, cs, gi, s.x, sigma, s.mu, s.st)) return rc;
    } else {
      lm32_to_vm_kernel<<<dim3((N + 31) / 32, cs / 32), dim3(32, 8), 0, s.st>>>(
          reinterpret_cast<const float*>(s.x), s.mu, N, cs, gi);
      HP_CK(cudaGetLastError());
    }
    HP_CK(cudaEventRecord(s.ready, s.st));
    HP_CK(cudaStreamWaitEvent(h->dstream, s.ready, 0));
    if (prof) tev(h->dstream);
    HP_CK(cudaGraphLaunch(s.graph[gsel], h->dstream));
    if (prof) tev(h->dstream);
    HP_CK(cudaEventRecord(s.decoded, h->dstream));
    HP_CK(cudaStreamWaitEvent(s.st, s.decoded, 0));
    if (int rc = qc_lane_major(N, cs, gi, s.post, post ? s.post_lm : nullptr, bits ? s.bits_lm : nullptr, s.st))
      return rc;
    if (post) {
      double* dst = c.pin_post ? post + (size_t)a * row : nullptr;
      if (!dst) {
        if (!s.h_post) HP_CK(cudaMallocHost(&s.h_post, (size_t)C * row * sizeof(double)));
        dst = s.h_post;
      }
      HP_CK(cudaMemcpyAsync(dst, s.post_lm, (size_t)gi * row * sizeof(double), cudaMemcpyDeviceToHost, s.st));
    }
    if (bits) {
      uint8_t* dst = c.pin_bits ? bits + (size_t)a * row : nullptr;
      if (!dst) {
        if (!s.h_bits) HP_CK(cudaMallocHost(&s.h_bits, (size_t)C * row));
        dst = s.h_bits;
      }
      HP_CK(cudaMemcpyAsync(dst, s.bits_lm, (size_t)gi * row, cudaMemcpyDeviceToHost, s.st));
    }
    HP_CK(cudaMemcpyAsync(s.h_ok, s.ok, gi, cudaMemcpyDeviceToHost, s.st));
    HP_CK(cudaMemcpyAsync(s.h_its, s.its, gi * sizeof(int32_t), cudaMemcpyDeviceToHost, s.st));
    HP_CK(cudaEventRecord(s.done, s.st));
    s.a = a;
    s.b = b;
    a = b;
  }
  if (prof) tev(h->slots[(nchunks - 1) % S].st);
  for (long long k = std::max<long long>(0, nchunks - S); k < nchunks; ++k)
    if (int rc = finish(c, h->slots[k % S])) return rc;
  if (prof) {
    HP_CK(cudaDeviceSynchronize());
    float dec = 0.0f, gaps = 0.0f, ms;
    for (long long k = 0; k < nchunks; ++k) {
      cudaEventElapsedTime(&ms, pev[1 + 2 * k], pev[2 + 2 * k]);
      dec += ms;
      if (k) {
        cudaEventElapsedTime(&ms, pev[2 * k], pev[1 + 2 * k]);
        gaps += ms;
      }
    }
    float head, tail, total;
    cudaEventElapsedTime(&head, pev[0], pev[1]);
    cudaEventElapsedTime(&tail, pev[2 * nchunks], pev.back());
    cudaEventElapsedTime(&total, pev[0], pev.back());
    std::fprintf(stderr, "[qc_host] chunks=%lld decode_ms=%.3f gaps_ms=%.3f head_ms=%.3f tail_ms=%.3f total_ms=%.3f\n",
                 nchunks, dec, gaps, head, tail, total);
    for (auto e : pev) cudaEventDestroy(e);
  }
  return 0;
}

}  // namespace

extern "C" int qc_host_decode(qc_host_dec* h, const double* x, int gamma, double sigma, uint8_t* bits,
                              double* post, uint8_t* ok, int64_t* iters_run) {
  if (!h) return fail_arg("null decoder");
  if (gamma < 0) return fail_arg("gamma must be >= 0");
  if (gamma > 0 && !x) return fail_arg("null input");
  if (gamma == 0) return 0;
  DeviceGuard guard(h->device);
  int rc = run(h, x, gamma, sigma, bits, post, ok, iters_run);
  if (rc) {                       // leave no chunk in flight for the next call
    cudaStreamSynchronize(h->dstream);
    for (auto& s : h->slots) {
      cudaStreamSynchronize(s.st);
      s.a = s.b = -1;
    }
    cudaGetLastError();
  }
  return rc;
}
