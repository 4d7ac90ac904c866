// Do cp.async.bulk copies from one SM overlap? One thread issues N copies of P
// bytes (L2-resident source, one mbarrier each) back to back and waits for all;
// %globaltimer around it, median over CTAs. Also 2D-tensor-like sizes.
#include <cstdio>
#include <cuda_runtime.h>
#include <stdint.h>
#include <algorithm>
#include <vector>
__device__ __forceinline__ uint32_t su32(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }
__global__ void probe(const uint8_t* src, int n, int piece, unsigned long long* out) {
  extern __shared__ __align__(128) uint8_t sm[];
  __shared__ __align__(8) uint64_t bars[16];
  if (threadIdx.x != 0) return;
  const uint8_t* base = src + (int64_t)blockIdx.x * (4 << 20);
  for (int i = 0; i < n; ++i) asm volatile("mbarrier.init.shared.b64 [%0], 1;" ::"r"(su32(&bars[i])));
  asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  for (int rep = 0; rep < 2; ++rep) {  // rep 0 warms L2 / TLB
    unsigned long long t0, t1;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t0));
    for (int i = 0; i < n; ++i) {
      asm volatile("mbarrier.arrive.expect_tx.shared.b64 _, [%0], %1;" ::"r"(su32(&bars[i])), "r"(piece) : "memory");
      asm volatile(
          "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
              su32(sm + i * piece)), "l"(base + (int64_t)i * piece), "r"(piece), "r"(su32(&bars[i])) : "memory");
    }
    for (int i = 0; i < n; ++i)
      asm volatile("{ .reg .pred p; W: mbarrier.try_wait.parity.shared.b64 p, [%0], %1; @!p bra W; }" ::"r"(
                       su32(&bars[i])), "r"(rep & 1) : "memory");
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t1));
    if (rep == 1) out[blockIdx.x] = t1 - t0;
  }
}
int main() {
  uint8_t* buf;
  unsigned long long* out;
  const int grid = 148;
  cudaMalloc(&buf, (size_t)grid * (4 << 20));
  cudaMemset(buf, 1, (size_t)grid * (4 << 20));
  cudaMalloc(&out, grid * 8);
  cudaFuncSetAttribute(probe, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024);
  for (int piece : {4096, 16384, 32768, 65536})
    for (int n : {1, 2, 4, 8, 12}) {
      if ((size_t)piece * n > 200 * 1024) continue;
      for (int g : {1, grid}) {
        probe<<<g, 32, piece * n>>>(buf, n, piece, out);
        cudaDeviceSynchronize();
        std::vector<unsigned long long> h(g);
        cudaMemcpy(h.data(), out, g * 8, cudaMemcpyDeviceToHost);
        std::sort(h.begin(), h.end());
        const double ns = (double)h[g / 2];
        printf("ctas %3d piece %6d x %2d: %8.0f ns  %7.1f GB/s per SM\n", g, piece, n, ns,
               (double)piece * n / ns);
      }
    }
  printf("%s\n", cudaGetErrorString(cudaGetLastError()));
}
