// Persistent, software-pipelined check pass (phi form) for regular codes.
//
// Same arithmetic as cnu_kernel<DC, VEC, REG, CNU_PHI> (block_kernels.cuh), but
// memory latency is hidden by an asynchronous copy pipeline instead of by warp
// count: each CTA owns a strided sequence of tiles (one check x 256*VEC
// lanes); while a tile is computed from shared memory, the next tile's d_c
// packages stream into the other half of a double buffer with cp.async
// (LDGSTS).  Every thread consumes only the shared-memory slots it filled
// itself, so a cp.async.wait_group is the only synchronisation.
// Grid = 2 CTAs per SM (96 KB of shared memory each at d_c = 24, float2).
#include <cuda_runtime.h>

#include <algorithm>
#include <cstdlib>

#include "block_kernels.cuh"

namespace qcb {
namespace {

template <int BYTES>
__device__ __forceinline__ void cp_async(void* smem, const void* gmem) {
  unsigned s = static_cast<unsigned>(__cvta_generic_to_shared(smem));
  if constexpr (BYTES == 16)
    asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(s), "l"(gmem));
  else
    asm volatile("cp.async.ca.shared.global [%0], [%1], %2;" ::"r"(s), "l"(gmem), "n"(BYTES));
}
__device__ __forceinline__ void cp_async_commit() { asm volatile("cp.async.commit_group;"); }
template <int N>
__device__ __forceinline__ void cp_async_wait() { asm volatile("cp.async.wait_group %0;" ::"n"(N)); }

template <int DC, int VEC>
__global__ void __launch_bounds__(THREADS) cnu_phi_pipe_kernel(CnuArgs a, int ntiles, int tiles_per_check) {
  extern __shared__ float smem[];
  constexpr int SLOT = THREADS * VEC;            // floats per package slice of one tile
  float* const buf0 = smem;
  float* const buf1 = smem + DC * SLOT;
  const int tid = threadIdx.x;
  auto issue = [&](int tile, float* b) {
    const int m = tile / tiles_per_check, qb = tile - m * tiles_per_check;
    const float* src = a.msgs + (size_t)m * DC * a.gamma + (size_t)(qb * THREADS + tid) * VEC;
#pragma unroll
    for (int k = 0; k < DC; ++k) cp_async<VEC * 4>(b + k * SLOT + tid * VEC, src + (size_t)k * a.gamma);
  };
  int tile = blockIdx.x, cur = 0;
  if (tile < ntiles) issue(tile, buf0);
  cp_async_commit();
  for (; tile < ntiles; tile += gridDim.x) {
    const int nxt = tile + gridDim.x;
    if (nxt < ntiles) issue(nxt, cur ? buf0 : buf1);
    cp_async_commit();
    cp_async_wait<1>();                          // this tile's packages have landed
    float x[DC][VEC];
    const float* b = cur ? buf1 : buf0;
#pragma unroll
    for (int k = 0; k < DC; ++k) {
      if constexpr (VEC == 2) {
        float2 v = *reinterpret_cast<const float2*>(b + k * SLOT + tid * 2);
        x[k][0] = v.x; x[k][1] = v.y;
      } else if constexpr (VEC == 4) {
        float4 v = *reinterpret_cast<const float4*>(b + k * SLOT + tid * 4);
        x[k][0] = v.x; x[k][1] = v.y; x[k][2] = v.z; x[k][3] = v.w;
      } else {
        x[k][0] = b[k * SLOT + tid];
      }
    }
    cnu_core<DC, VEC, true>(x, DC, (1u << VEC) - 1u);
    const int m = tile / tiles_per_check, qb = tile - m * tiles_per_check;
    float* dst = a.msgs + (size_t)m * DC * a.gamma + (size_t)(qb * THREADS + tid) * VEC;
#pragma unroll
    for (int k = 0; k < DC; ++k) vstore<VEC>(dst + (size_t)k * a.gamma, x[k]);
    cur ^= 1;
  }
  cp_async_wait<0>();
}

}  // namespace

int cnu_pipe_mode() {
  static int v = [] {
    const char* e = std::getenv("QCB_CNU_PIPE");
    return e ? std::atoi(e) : 0;
  }();
  return v;
}

template <int VEC, int CTAS>
int launch_pipe_v(const qc_plan* p, const CnuArgs& a, cudaStream_t s) {
  constexpr int DC = 24;
  if (a.gamma % (THREADS * VEC)) return 0;
  static int nsm = 0;
  static bool attr = false;
  const size_t smem = 2ull * DC * THREADS * VEC * sizeof(float);
  if (!attr) {
    cudaFuncSetAttribute(cnu_phi_pipe_kernel<DC, VEC>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    int dev;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, dev);
    attr = true;
  }
  const int tpc = a.gamma / (THREADS * VEC);
  const int ntiles = p->M * tpc;
  const int grid = std::min(ntiles, nsm * CTAS);
  cnu_phi_pipe_kernel<DC, VEC><<<grid, THREADS, smem, s>>>(a, ntiles, tpc);
  return 1;
}

// returns 1 if launched, 0 if the shape is not supported (caller falls back)
// QCB_CNU_PIPE=1: float2 lanes, 96 KB smem, 2 CTAs/SM; =2: 1 lane, 48 KB, 4 CTAs/SM
int launch_cnu_phi_pipe(const qc_plan* p, const CnuArgs& a, cudaStream_t s) {
  if (p->check_regular != 24 || a.active) return 0;
  if (cnu_pipe_mode() == 2) return launch_pipe_v<1, 4>(p, a, s);
  return launch_pipe_v<2, 2>(p, a, s);
}

}  // namespace qcb
