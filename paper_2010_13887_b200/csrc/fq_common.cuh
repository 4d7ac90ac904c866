// Shared helpers for the sm_100a kernels behind include/fq_abi.h.
#pragma once

#include <cuda_fp16.h>
#include <cuda_runtime.h>
#include <math.h>
#include <stdint.h>
#include <stdio.h>

#include "../../include/fq_abi.h"

namespace fq {

// Thread-local last error message for fq_last_error().
void set_error(const char* fmt, ...);

inline cudaStream_t as_stream(fq_stream_t s) { return reinterpret_cast<cudaStream_t>(s); }

// Map the last launch status to an fq_status.
int launch_status(const char* what);

#define FQ_CHECK_ARG(cond, code, ...)      \
  do {                                     \
    if (!(cond)) {                         \
      ::fq::set_error(__VA_ARGS__);        \
      return (code);                       \
    }                                      \
  } while (0)

__device__ __forceinline__ float warp_max(float v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v = fmaxf(v, __shfl_xor_sync(0xffffffffu, v, o));
  return v;
}
__device__ __forceinline__ float warp_min(float v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v = fminf(v, __shfl_xor_sync(0xffffffffu, v, o));
  return v;
}
__device__ __forceinline__ float warp_sum(float v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  return v;
}
__device__ __forceinline__ double warp_sum(double v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  return v;
}
__device__ __forceinline__ int warp_sum_i(int v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  return v;
}

// Block-wide sum of doubles; `red` needs blockDim/32 doubles of smem.
__device__ __forceinline__ double block_sum(double v, double* red) {
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5, nw = (blockDim.x + 31) >> 5;
  v = warp_sum(v);
  __syncthreads();
  if (lane == 0) red[w] = v;
  __syncthreads();
  double t = 0.0;
  for (int i = 0; i < nw; ++i) t += red[i];  // fixed order: deterministic
  return t;
}

// The 16-bit operand / storage type of the throughput mode (fp16: 11-bit
// significand, the paper's own half precision; fp32 accumulation everywhere).
using h16 = __half;
using h16x2 = __half2;

__device__ __forceinline__ float h2f(h16 x) { return __half2float(x); }
__device__ __forceinline__ h16 f2h(float x) { return __float2half_rn(x); }

// Exact-mode operand pair (OP_X3H GEMMs, 3xFP16): x = hi + lo * 2^-11 with
// hi = fp16(x) and lo = fp16((x - hi) * 2^11), both round-to-nearest. x - hi is
// exact in fp32 and the 2^11 scale keeps lo out of fp16's subnormal range, so
// the pair holds 22 significant bits (|x| < 65504).
constexpr float kXhScale = 2048.0f;
__device__ __forceinline__ void split_xh(float x, h16& hi, h16& lo) {
  hi = __float2half_rn(x);
  lo = __float2half_rn((x - __half2float(hi)) * kXhScale);
}
__device__ __forceinline__ void split_xh2(float x0, float x1, uint32_t& hi, uint32_t& lo) {
  const h16x2 h = __floats2half2_rn(x0, x1);
  const float2 hf = __half22float2(h);
  const h16x2 l = __floats2half2_rn((x0 - hf.x) * kXhScale, (x1 - hf.y) * kXhScale);
  hi = *reinterpret_cast<const uint32_t*>(&h);
  lo = *reinterpret_cast<const uint32_t*>(&l);
}

// fp32 ops with explicit rounding so nvcc never contracts them into FMA
// (two separately rounded fp32 operations).
__device__ __forceinline__ float fmul_rn(float a, float b) { return __fmul_rn(a, b); }
__device__ __forceinline__ float fadd_rn(float a, float b) { return __fadd_rn(a, b); }

// Activation on the fp32 pre-activation (kernels.py:45-50): ReLU by compare,
// GELU = 0.5 t (1 + erf(t/sqrt 2)) evaluated in f64 and rounded to fp32.
// The f64 GELU is out of line: inlined into every unrolled epilogue it grew
// the GEMM kernels' code past the instruction cache (ReLU stays inline).
static __device__ __noinline__ float gelu_f64(float t) {
  double td = (double)t;
  return (float)(0.5 * td * (1.0 + erf(td * 0.70710678118654752440)));
}
__device__ __forceinline__ float apply_act(float t, int act) {
  if (act == FQ_ACT_RELU) return t < 0.0f ? 0.0f : t;
  if (act == FQ_ACT_GELU) return gelu_f64(t);
  return t;
}

inline int ceil_div(int64_t a, int64_t b) { return (int)((a + b - 1) / b); }

// ---- programmatic dependent launch (PDL) ---------------------------------
// Every kernel is launched with programmatic stream serialization and starts
// with pdl_enter(): launch_dependents lets the NEXT kernel's CTAs launch and
// run their prologue while this grid drains, then griddepcontrol.wait blocks
// until the stream predecessor has completed and its writes are visible (so
// nothing below it may touch dependent global memory earlier). The tcgen05
// GEMMs go further: their TMA producer streams the first stages of the
// (constant) weight operand before the wait, so weight fetch latency overlaps
// the previous kernel. FQ_PDL=0 disables it.
__device__ __forceinline__ void pdl_enter() {
  asm volatile("griddepcontrol.launch_dependents;" ::: "memory");
  asm volatile("griddepcontrol.wait;" ::: "memory");
}
__device__ __forceinline__ void pdl_launch_dependents() {
  asm volatile("griddepcontrol.launch_dependents;" ::: "memory");
}
__device__ __forceinline__ void pdl_wait() { asm volatile("griddepcontrol.wait;" ::: "memory"); }

bool pdl_enabled();

template <typename... KArgs, typename... Args>
inline cudaError_t launch_kernel(void (*kernel)(KArgs...), dim3 grid, dim3 block, size_t smem,
                                 cudaStream_t s, unsigned cluster, Args... args) {
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = grid;
  cfg.blockDim = block;
  cfg.dynamicSmemBytes = smem;
  cfg.stream = s;
  cudaLaunchAttribute attr[2];
  unsigned n = 0;
  if (pdl_enabled()) {
    attr[n].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    attr[n].val.programmaticStreamSerializationAllowed = 1;
    ++n;
  }
  if (cluster > 1) {
    attr[n].id = cudaLaunchAttributeClusterDimension;
    attr[n].val.clusterDim.x = cluster;
    attr[n].val.clusterDim.y = 1;
    attr[n].val.clusterDim.z = 1;
    ++n;
  }
  cfg.attrs = attr;
  cfg.numAttrs = n;
  return cudaLaunchKernelEx(&cfg, kernel, static_cast<KArgs>(args)...);
}

}  // namespace fq
