// Per-SM ingest: 2D tensor TMA boxes (64 fp16 x 128 rows, 128-byte swizzle:
// the GEMM operand tiles) vs 1D cp.async.bulk of the same 16 KB, N copies in
// flight from one thread, L2-resident source; median over 148 CTAs.
#include <cstdio>
#include <cuda.h>
#include <cuda_runtime.h>
#include <stdint.h>
#include <algorithm>
#include <vector>
__device__ __forceinline__ uint32_t su32(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }
__global__ void probe(const __grid_constant__ CUtensorMap tm, const uint8_t* src, int n, int mode,
                      unsigned long long* out) {
  extern __shared__ __align__(1024) uint8_t smraw[];
  uint8_t* sm = smraw + ((1024 - (su32(smraw) & 1023)) & 1023);
  __shared__ __align__(8) uint64_t bars[16];
  if (threadIdx.x != 0) return;
  const int rows0 = blockIdx.x * 1024;  // each CTA its own 1024 rows x 1024 cols fp16 (2 MB)
  for (int i = 0; i < n; ++i) asm volatile("mbarrier.init.shared.b64 [%0], 1;" ::"r"(su32(&bars[i])));
  asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  for (int rep = 0; rep < 2; ++rep) {
    unsigned long long t0, t1;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t0));
    for (int i = 0; i < n; ++i) {
      asm volatile("mbarrier.arrive.expect_tx.shared.b64 _, [%0], %1;" ::"r"(su32(&bars[i])), "r"(16384) : "memory");
      if (mode == 0) {
        // box (64 cols, 128 rows) at col block i % 16, row block i / 16
        asm volatile(
            "cp.async.bulk.tensor.2d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3}], [%4];" ::"r"(
                su32(sm + i * 16384)), "l"(reinterpret_cast<uint64_t>(&tm)), "r"((i % 16) * 64),
            "r"(rows0 + (i / 16) * 128), "r"(su32(&bars[i])) : "memory");
      } else {
        asm volatile(
            "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
                su32(sm + i * 16384)), "l"(src + ((int64_t)rows0 * 1024) * 2 + (int64_t)i * 16384), "r"(16384),
            "r"(su32(&bars[i])) : "memory");
      }
    }
    for (int i = 0; i < n; ++i)
      asm volatile("{ .reg .pred p; W: mbarrier.try_wait.parity.shared.b64 p, [%0], %1; @!p bra W; }" ::"r"(
                       su32(&bars[i])), "r"(rep & 1) : "memory");
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t1));
    if (rep == 1) out[blockIdx.x] = t1 - t0;
  }
}
int main() {
  const int grid = 148;
  uint8_t* buf;
  unsigned long long* out;
  const size_t rows = (size_t)grid * 1024, cols = 1024;
  cudaMalloc(&buf, rows * cols * 2);
  cudaMemset(buf, 1, rows * cols * 2);
  cudaMalloc(&out, grid * 8);
  CUtensorMap tm;
  cuuint64_t dims[2] = {cols, rows}, strides[1] = {cols * 2};
  cuuint32_t box[2] = {64, 128}, es[2] = {1, 1};
  CUresult r = cuTensorMapEncodeTiled(&tm, CU_TENSOR_MAP_DATA_TYPE_FLOAT16, 2, buf, dims, strides, box, es,
                                      CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B,
                                      CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  if (r != CUDA_SUCCESS) { printf("encode failed %d\n", (int)r); return 1; }
  cudaFuncSetAttribute(probe, cudaFuncAttributeMaxDynamicSharedMemorySize, 210 * 1024);
  for (int mode = 0; mode < 2; ++mode)
    for (int n : {1, 2, 4, 8, 12})
      for (int g : {1, grid}) {
        probe<<<g, 32, n * 16384 + 1024>>>(tm, buf, n, mode, out);
        cudaDeviceSynchronize();
        std::vector<unsigned long long> h(g);
        cudaMemcpy(h.data(), out, g * 8, cudaMemcpyDeviceToHost);
        std::sort(h.begin(), h.end());
        printf("%s ctas %3d 16KB x %2d: %6llu ns  %6.1f GB/s per SM\n", mode ? "bulk1d" : "tma2d ", g, n,
               h[g / 2], 16384.0 * n / h[g / 2]);
      }
  printf("%s\n", cudaGetErrorString(cudaGetLastError()));
}
