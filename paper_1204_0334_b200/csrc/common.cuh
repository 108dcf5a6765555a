// Shared helpers of the qcldpc_b200 CUDA library (sm_100a).
#pragma once

#include <cuda_runtime.h>
#include <stdint.h>

#include <string>

#include "../../include/qcldpc_b200.h"

namespace qcb {

// thread-local last error (qc_last_error)
void set_error(const std::string& msg);
int fail_arg(const std::string& msg);      // returns a negative code (ValueError class)
int fail_rt(const std::string& msg);       // returns a positive code (RuntimeError class)
int check_launch(const char* what);        // cudaGetLastError -> code

constexpr float L_MAX = 50.0f;
// 2*atanh(fl(1 - 1e-12)) -- the reference's |alpha| cap (bp.py:50-51, test_bp.py:22)
constexpr float ALPHA_CAP = 28.324190418452803892f;
#ifndef QCB_THREADS
#define QCB_THREADS 128   // 128-thread CTAs: +12% check pass, +7-9% two-pass decode vs 256 (profiles/r01/kbench_threads128.jsonl)
#endif
constexpr int THREADS = QCB_THREADS;

inline cudaStream_t as_stream(void* s) { return reinterpret_cast<cudaStream_t>(s); }

// Programmatic dependent launch (sm_90+): a kernel launched with launch_pdl may
// be scheduled while its predecessor in the stream drains; it must call
// pdl_wait() before touching memory the predecessor writes (that wait covers
// the predecessor's completion and memory flush), and pdl_trigger() lets its
// own successor be scheduled early.
__device__ __forceinline__ void pdl_trigger() { asm volatile("griddepcontrol.launch_dependents;" ::: "memory"); }
__device__ __forceinline__ void pdl_wait() { asm volatile("griddepcontrol.wait;" ::: "memory"); }

bool pdl_enabled();   // QCB_PDL env (default on)

template <typename... KArgs, typename... Args>
inline void launch_pdl(void (*kern)(KArgs...), dim3 grid, unsigned block, cudaStream_t s, Args... args) {
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = grid;
  cfg.blockDim = dim3(block, 1, 1);
  cfg.dynamicSmemBytes = 0;
  cfg.stream = s;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  attr[0].val.programmaticStreamSerializationAllowed = pdl_enabled() ? 1 : 0;
  cfg.attrs = attr;
  cfg.numAttrs = 1;
  cudaLaunchKernelEx(&cfg, kern, args...);
}

inline unsigned blocks_for(long long threads, int per = THREADS) {
  return static_cast<unsigned>((threads + per - 1) / per);
}

// ---------------------------------------------------------------------------
// vector-of-lanes access: VEC consecutive lanes of one package per thread
// ---------------------------------------------------------------------------
template <int VEC> struct Vec;
template <> struct Vec<1> { using T = float; };
template <> struct Vec<2> { using T = float2; };
template <> struct Vec<4> { using T = float4; };

template <int VEC>
__device__ __forceinline__ void vload(const float* p, float (&v)[VEC]) {
  if constexpr (VEC == 4) {
    float4 t = *reinterpret_cast<const float4*>(p);
    v[0] = t.x; v[1] = t.y; v[2] = t.z; v[3] = t.w;
  } else if constexpr (VEC == 2) {
    float2 t = *reinterpret_cast<const float2*>(p);
    v[0] = t.x; v[1] = t.y;
  } else {
    v[0] = *p;
  }
}

template <int VEC>
__device__ __forceinline__ void vstore(float* p, const float (&v)[VEC]) {
  if constexpr (VEC == 4) {
    *reinterpret_cast<float4*>(p) = make_float4(v[0], v[1], v[2], v[3]);
  } else if constexpr (VEC == 2) {
    *reinterpret_cast<float2*>(p) = make_float2(v[0], v[1]);
  } else {
    *p = v[0];
  }
}

__device__ __forceinline__ float clampL(float x) { return fminf(fmaxf(x, -L_MAX), L_MAX); }

// lane mask bits (VEC lanes starting at lane g0, g0 % VEC == 0)
__device__ __forceinline__ unsigned lane_bits_of(const uint32_t* words, int g0, int vec) {
  if (!words) return (1u << vec) - 1u;
  return (words[g0 >> 5] >> (g0 & 31)) & ((1u << vec) - 1u);
}

// OR-reduce a VEC-lane bit group into its 32-lane word and store it once.
// Threads t..t+32/VEC-1 (aligned) share one word; q is the thread's lane-vector index.
template <int VEC>
__device__ __forceinline__ void store_bit_word(uint32_t* dst_word_base, int q, unsigned bits,
                                               bool valid) {
  constexpr int GROUP = 32 / VEC;
  unsigned w = valid ? (bits << ((q * VEC) & 31)) : 0u;
#pragma unroll
  for (int off = 1; off < GROUP; off <<= 1) w |= __shfl_xor_sync(0xffffffffu, w, off);
  if (valid && (q % GROUP) == 0) dst_word_base[(q * VEC) >> 5] = w;
}

}  // namespace qcb
