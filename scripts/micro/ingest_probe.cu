// Per-SM ingest probe: how fast can ONE CTA per SM pull L2-resident data into
// shared memory through (0) the TMA unit (1D cp.async.bulk, 16 KB pieces,
// 4-deep mbarrier ring), (1) cp.async 16-byte copies (256 threads, LSU path),
// (2) both at once (half the bytes each)? At 32 .. 148 CTAs: if (2) beats (0)
// the decode GEMMs' per-SM operand ingest could be split across the paths.
#include <cstdio>
#include <cuda_runtime.h>
#include <stdint.h>

__device__ __forceinline__ uint32_t su32(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }
__device__ __forceinline__ void bar_init(uint64_t* b, int n) {
  asm volatile("mbarrier.init.shared.b64 [%0], %1;" ::"r"(su32(b)), "r"(n));
}
__device__ __forceinline__ void bar_expect(uint64_t* b, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared.b64 _, [%0], %1;" ::"r"(su32(b)), "r"(bytes) : "memory");
}
__device__ __forceinline__ void bar_wait(uint64_t* b, int ph) {
  asm volatile(
      "{ .reg .pred p; W: mbarrier.try_wait.parity.shared.b64 p, [%0], %1; @!p bra W; }" ::"r"(su32(b)),
      "r"(ph) : "memory");
}

constexpr int MAXNS = 16;
__constant__ int PIECE_c, NS_c;
// mode 0: bulk only; 1: cp.async only; 2: bulk for even pieces, cp.async for odd
__global__ void __launch_bounds__(256) ingest(const uint8_t* __restrict__ src, int64_t slice, int reps,
                                              int mode, float* sink) {
  extern __shared__ __align__(128) uint8_t ring[];  // NS pieces (bulk) + NS pieces (cp.async)
  __shared__ __align__(8) uint64_t full[MAXNS];
  const int PIECE = PIECE_c, NS = NS_c;
  const int tid = threadIdx.x;
  const uint8_t* base = src + (int64_t)blockIdx.x * slice;
  const int npiece = (int)(slice / PIECE) * reps;
  if (tid == 0) {
    for (int s = 0; s < NS; ++s) bar_init(&full[s], 1);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  __syncthreads();
  float acc = 0.f;
  // bulk ring: lane 0 of warp 0 keeps NS pieces in flight
  int bi = 0, bc = 0;  // bulk pieces issued / consumed (indices in the bulk sequence)
  int ci = 0;          // cp.async groups issued
  const int nb = mode == 0 ? npiece : mode == 2 ? (npiece + 1) / 2 : 0;
  const int nc = npiece - nb;
  auto piece_src = [&](int k) { return base + (int64_t)(k % (slice / PIECE)) * PIECE; };
  if (tid == 0)
    for (; bi < NS && bi < nb; ++bi) {
      bar_expect(&full[bi % NS], PIECE);
      asm volatile(
          "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
              su32(ring + (bi % NS) * PIECE)),
          "l"(piece_src(2 * bi)), "r"(PIECE), "r"(su32(&full[bi % NS]))
          : "memory");
    }
  uint8_t* cring = ring + NS * PIECE;
  auto cissue = [&](int k) {
    const uint8_t* p = piece_src(2 * k + 1);
    uint8_t* d = cring + (k % NS) * PIECE;
    for (int o = tid * 16; o < PIECE; o += 256 * 16)
      asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(su32(d + o)), "l"(p + o) : "memory");
    asm volatile("cp.async.commit_group;" ::: "memory");
  };
  for (; ci < 3; ++ci) {
    if (ci < nc) cissue(ci);
    else asm volatile("cp.async.commit_group;" ::: "memory");
  }
  int cc = 0;
  while (bc < nb || cc < nc) {
    if (bc < nb) {
      bar_wait(&full[bc % NS], (bc / NS) & 1);
      acc += (float)ring[(bc % NS) * PIECE + tid * 4];
      __syncthreads();
      if (tid == 0 && bi < nb) {
        bar_expect(&full[bi % NS], PIECE);
        asm volatile(
            "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
                su32(ring + (bi % NS) * PIECE)),
            "l"(piece_src(2 * bi)), "r"(PIECE), "r"(su32(&full[bi % NS]))
            : "memory");
        ++bi;
      }
      ++bc;
    }
    if (cc < nc) {
      asm volatile("cp.async.wait_group %0;" ::"n"(2) : "memory");
      __syncthreads();
      acc += (float)cring[(cc % NS) * PIECE + tid * 4];
      __syncthreads();
      if (ci < nc) cissue(ci);
      else asm volatile("cp.async.commit_group;" ::: "memory");
      ++ci;
      ++cc;
    }
  }
  if (acc == 1234.5f) sink[0] = acc;
}

int main() {
  const int64_t slice = 512 << 10;  // 512 KB per CTA, L2-resident (148 x 0.5 MB = 74 MB)
  uint8_t* buf;
  float* sink;
  cudaMalloc(&buf, 148 * slice);
  cudaMemset(buf, 1, 148 * slice);
  cudaMalloc(&sink, 4);
  cudaFuncSetAttribute(ingest, cudaFuncAttributeMaxDynamicSharedMemorySize, 220 * 1024);
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  const int reps = 4;
  const int cfgs[][2] = {{16384, 4}, {16384, 8}, {16384, 12}, {32768, 4}, {32768, 6}, {65536, 3}};
  for (int grid : {64, 148}) {
    for (auto& c : cfgs) {
      cudaMemcpyToSymbol(PIECE_c, &c[0], 4);
      cudaMemcpyToSymbol(NS_c, &c[1], 4);
      for (int mode = 0; mode < 3; mode += 2) {
        const int smem = (mode == 0 ? 1 : 2) * c[0] * c[1];
        if (smem > 220 * 1024) continue;
        for (int w = 0; w < 3; ++w) ingest<<<grid, 256, smem>>>(buf, slice, reps, mode, sink);
        cudaEventRecord(e0);
        const int it = 20;
        for (int w = 0; w < it; ++w) ingest<<<grid, 256, smem>>>(buf, slice, reps, mode, sink);
        cudaEventRecord(e1);
        cudaEventSynchronize(e1);
        float ms;
        cudaEventElapsedTime(&ms, e0, e1);
        const double us = ms * 1e3 / it, bytes = (double)slice * reps;
        printf("grid %3d piece %5d ns %2d mode %s: %8.2f us  per-SM %6.1f GB/s  chip %7.1f GB/s\n",
               grid, c[0], c[1], mode == 0 ? "bulk" : "both", us, bytes / us / 1e3,
               bytes * grid / us / 1e3);
      }
    }
  }
  cudaError_t err = cudaGetLastError();
  printf("%s\n", cudaGetErrorString(err));
  return 0;
}
