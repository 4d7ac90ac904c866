// bf16 GEMM on the 5th-generation tensor cores (tcgen05 + TMEM + TMA), sm_100a.
//
// C[M,N] = epilogue(A[M,K] . B[N,K]^T), A and B bf16 K-major (weights were
// re-laid out to [N,K] once at load), fp32 accumulation in TMEM. One CTA per
// 128 x BN output tile, warp-specialised:
//   warp 0      TMA producer: 2D tiled loads (128B swizzle) into a STAGES-deep
//               shared-memory ring, mbarrier complete_tx;
//   warp 1      TMEM allocator + single-thread tcgen05.mma issuer
//               (M=128, N=BN, K=16 per instruction), tcgen05.commit frees ring
//               slots and finally signals the accumulator;
//   warps 2..5  epilogue: tcgen05.ld (32 lanes x 16 columns per load), fused
//               (+C) (+bias) act (+residual), fp32 or bf16 stores.
// The fused epilogue is the reference's bias_residual_act pass (kernels.py:39-53)
// applied to the accumulator, so the [M,N] pre-activation never reaches HBM.
#include <cuda.h>
#include <cudaTypedefs.h>

#include "fq_common.cuh"

namespace fq {

namespace tc {

constexpr int BM = 128;
constexpr int BK = 64;  // 64 bf16 = 128 bytes = one swizzle row
constexpr int kThreads = 192;

__device__ __forceinline__ uint32_t smem_u32(const void* p) {
  return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}

__device__ __forceinline__ void mbar_init(uint64_t* bar, uint32_t count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count));
}

__device__ __forceinline__ void mbar_expect_tx(uint64_t* bar, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)),
               "r"(bytes)
               : "memory");
}

__device__ __forceinline__ bool mbar_try(uint64_t* bar, uint32_t parity) {
  uint32_t ok;
  asm volatile(
      "{\n\t.reg .pred p;\n\t"
      "mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\n\t"
      "selp.u32 %0, 1, 0, p;\n}"
      : "=r"(ok)
      : "r"(smem_u32(bar)), "r"(parity)
      : "memory");
  return ok != 0;
}

// Watchdog: a pipeline that never completes traps (error on the host)
// instead of hanging the GPU.
__device__ __forceinline__ void mbar_wait(uint64_t* bar, uint32_t parity) {
  if (mbar_try(bar, parity)) return;
  const long long t0 = clock64();
  while (!mbar_try(bar, parity)) {
    if (clock64() - t0 > (1LL << 33)) __trap();  // ~4 s at 2 GHz
  }
}

__device__ __forceinline__ void tma_load_2d(const CUtensorMap* map, uint64_t* bar, void* dst,
                                            int c0, int c1) {
  asm volatile(
      "cp.async.bulk.tensor.2d.shared::cluster.global.mbarrier::complete_tx::bytes"
      " [%0], [%1, {%2, %3}], [%4];" ::"r"(smem_u32(dst)),
      "l"(reinterpret_cast<uint64_t>(map)), "r"(c0), "r"(c1), "r"(smem_u32(bar))
      : "memory");
}

// K-major operand, 128-byte swizzle: rows of 128 B, 8-row atoms 1024 B apart.
__device__ __forceinline__ uint64_t sw128_desc(uint32_t saddr) {
  uint64_t d = 0;
  d |= (uint64_t)((saddr & 0x3FFFF) >> 4);  // start address
  d |= (uint64_t)1 << 16;                    // LBO (unused for swizzled K-major)
  d |= (uint64_t)(1024 >> 4) << 32;          // SBO: next 8-row atom
  d |= (uint64_t)1 << 46;                    // descriptor version (sm_100)
  d |= (uint64_t)2 << 61;                    // SWIZZLE_128B
  return d;
}

// kind::f16 instruction descriptor: bf16 x bf16 -> f32, both K-major.
__host__ __device__ constexpr uint32_t idesc_bf16(int m, int n) {
  return (1u << 4) | (1u << 7) | (1u << 10) | ((uint32_t)(n >> 3) << 17) |
         ((uint32_t)(m >> 4) << 24);
}

__device__ __forceinline__ void mma_bf16(uint32_t tmem_d, uint64_t adesc, uint64_t bdesc,
                                         uint32_t idesc, uint32_t accumulate) {
  asm volatile(
      "{\n\t.reg .pred p;\n\t"
      "setp.ne.b32 p, %4, 0;\n\t"
      "tcgen05.mma.cta_group::1.kind::f16 [%0], %1, %2, %3, p;\n}" ::"r"(tmem_d),
      "l"(adesc), "l"(bdesc), "r"(idesc), "r"(accumulate));
}

__device__ __forceinline__ void mma_commit(uint64_t* bar) {
  asm volatile(
      "tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(
          smem_u32(bar))
      : "memory");
}

__device__ __forceinline__ void tmem_ld32(uint32_t taddr, float* v) {
  uint32_t r[32];
  asm volatile(
      "tcgen05.ld.sync.aligned.32x32b.x32.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,"
      "%14,%15,%16,%17,%18,%19,%20,%21,%22,%23,%24,%25,%26,%27,%28,%29,%30,%31}, [%32];"
      : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]),
        "=r"(r[7]), "=r"(r[8]), "=r"(r[9]), "=r"(r[10]), "=r"(r[11]), "=r"(r[12]),
        "=r"(r[13]), "=r"(r[14]), "=r"(r[15]), "=r"(r[16]), "=r"(r[17]), "=r"(r[18]),
        "=r"(r[19]), "=r"(r[20]), "=r"(r[21]), "=r"(r[22]), "=r"(r[23]), "=r"(r[24]),
        "=r"(r[25]), "=r"(r[26]), "=r"(r[27]), "=r"(r[28]), "=r"(r[29]), "=r"(r[30]),
        "=r"(r[31])
      : "r"(taddr));
  asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
#pragma unroll
  for (int i = 0; i < 32; ++i) v[i] = __uint_as_float(r[i]);
}

__device__ __forceinline__ void mbar_arrive(uint64_t* bar) {
  asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem_u32(bar)) : "memory");
}

struct Epi {
  void* c;
  int64_t ldc;
  int c_bf16;
  int accumulate;
  const float* bias;
  const float* res;
  int64_t ldr;
  int act;
};

// Persistent: grid <= #SMs, CTA walks tiles t = blockIdx.x, +gridDim.x, ...
// (M-tile fastest so concurrent CTAs share the weight tile in L2). Two TMEM
// accumulator stages let the epilogue of tile i overlap the MMAs of tile i+1.
template <int BN, int STAGES>
__global__ void __launch_bounds__(kThreads, 1)
    tc_gemm_kernel(const __grid_constant__ CUtensorMap tma_a,
                   const __grid_constant__ CUtensorMap tma_b, const Epi ep, int M, int N, int K) {
  constexpr int A_BYTES = BM * BK * 2;
  constexpr int B_BYTES = BN * BK * 2;
  constexpr int STAGE_BYTES = A_BYTES + B_BYTES;
  constexpr uint32_t TMEM_COLS = 2 * BN < 32 ? 32 : 2 * BN;  // two accumulator stages
  extern __shared__ uint8_t smem_raw[];
  // 1024-B aligned (128B-swizzle atoms); pointer arithmetic keeps the shared
  // address space visible to the compiler (LDS/STS, not generic LD/ST)
  uint8_t* smem = smem_raw + ((1024u - (smem_u32(smem_raw) & 1023u)) & 1023u);
  float* stage_out = reinterpret_cast<float*>(smem + STAGES * STAGE_BYTES);  // 4 x [32][33]
  __shared__ __align__(8) uint64_t full_bar[STAGES];
  __shared__ __align__(8) uint64_t empty_bar[STAGES];
  __shared__ __align__(8) uint64_t tfull_bar[2];
  __shared__ __align__(8) uint64_t tempty_bar[2];
  __shared__ uint32_t tmem_base_sh;

  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int num_kb = (K + BK - 1) / BK;
  const int mt = (M + BM - 1) / BM;
  const int ntiles = mt * ((N + BN - 1) / BN);

  if (warp == 0 && lane == 0) {
    for (int s = 0; s < STAGES; ++s) {
      mbar_init(&full_bar[s], 1);
      mbar_init(&empty_bar[s], 1);
    }
    for (int s = 0; s < 2; ++s) {
      mbar_init(&tfull_bar[s], 1);
      mbar_init(&tempty_bar[s], 4);  // one arrive per epilogue warp
    }
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    asm volatile("prefetch.tensormap [%0];" ::"l"(reinterpret_cast<uint64_t>(&tma_a)));
    asm volatile("prefetch.tensormap [%0];" ::"l"(reinterpret_cast<uint64_t>(&tma_b)));
  }
  if (warp == 1) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(
                     smem_u32(&tmem_base_sh)),
                 "r"(TMEM_COLS));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
  const uint32_t tmem = tmem_base_sh;

  if (warp == 0) {
    if (lane == 0) {  // ---- TMA producer ----
      int it = 0;
      for (int t = blockIdx.x; t < ntiles; t += gridDim.x) {
        const int m0 = (t % mt) * BM, n0 = (t / mt) * BN;
        for (int kb = 0; kb < num_kb; ++kb, ++it) {
          const int s = it % STAGES;
          const uint32_t ph = (it / STAGES) & 1;
          mbar_wait(&empty_bar[s], ph ^ 1);
          uint8_t* sa = smem + s * STAGE_BYTES;
          mbar_expect_tx(&full_bar[s], STAGE_BYTES);
          tma_load_2d(&tma_a, &full_bar[s], sa, kb * BK, m0);
          tma_load_2d(&tma_b, &full_bar[s], sa + A_BYTES, kb * BK, n0);
        }
      }
    }
  } else if (warp == 1) {
    if (lane == 0) {  // ---- MMA issuer ----
      constexpr uint32_t idesc = idesc_bf16(BM, BN);
      int it = 0, local = 0;
      for (int t = blockIdx.x; t < ntiles; t += gridDim.x, ++local) {
        const int as = local & 1;
        mbar_wait(&tempty_bar[as], ((local >> 1) & 1) ^ 1);  // epilogue drained this stage
        asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
        const uint32_t acc = tmem + as * BN;
        for (int kb = 0; kb < num_kb; ++kb, ++it) {
          const int s = it % STAGES;
          const uint32_t ph = (it / STAGES) & 1;
          mbar_wait(&full_bar[s], ph);
          asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
          const uint32_t a_base = smem_u32(smem + s * STAGE_BYTES);
          const uint32_t b_base = a_base + A_BYTES;
#pragma unroll
          for (int k = 0; k < BK / 16; ++k) {
            mma_bf16(acc, sw128_desc(a_base + k * 32), sw128_desc(b_base + k * 32), idesc,
                     (kb | k) != 0);
          }
          mma_commit(&empty_bar[s]);  // ring slot reusable once these MMAs retire
        }
        mma_commit(&tfull_bar[as]);   // accumulator stage complete
      }
    }
  } else {  // ---- epilogue: warps 2..5 own TMEM lane quarters (warp % 4) ----
    const int q = warp & 3;
    float* st = stage_out + (warp - 2) * 32 * 33;
    float* c32 = reinterpret_cast<float*>(ep.c);
    __nv_bfloat16* c16 = reinterpret_cast<__nv_bfloat16*>(ep.c);
    int local = 0;
    for (int t = blockIdx.x; t < ntiles; t += gridDim.x, ++local) {
      const int as = local & 1;
      const int m0 = (t % mt) * BM, n0 = (t / mt) * BN;
      mbar_wait(&tfull_bar[as], (local >> 1) & 1);
      asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
      const int rbase = m0 + q * 32;
      const int nrows = min(32, M - rbase);
#pragma unroll 1
      for (int cc = 0; cc < BN; cc += 32) {
        float v[32];
        tmem_ld32(tmem + as * BN + ((uint32_t)(q * 32) << 16) + cc, v);
        if (cc + 32 >= BN) {  // last TMEM read of this stage: hand it back to the MMA warp
          asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
          __syncwarp();
          if (lane == 0) mbar_arrive(&tempty_bar[as]);
        }
        // transpose through smem: thread = row on the TMEM side, column on the store side
#pragma unroll
        for (int j = 0; j < 32; ++j) st[lane * 33 + j] = v[j];
        __syncwarp();
        const int col = n0 + cc + lane;
#pragma unroll 1
        for (int h0 = 0; h0 < 32; h0 += 16) {  // 16 rows at a time bounds register use
        float x[16];
#pragma unroll
        for (int i = 0; i < 16; ++i) x[i] = st[(h0 + i) * 33 + lane];
        const int nr = nrows - h0;
        if (col < N && nr > 0) {
          // every global read of the 32 rows is issued before any store
          // (no per-row dependent latency); each lane owns one column, so the
          // warp writes full 128-byte row segments
          const int64_t c0 = (int64_t)(rbase + h0) * ep.ldc + col;
          if (ep.accumulate) {
            float cv[16];
#pragma unroll
            for (int i = 0; i < 16; ++i)
              cv[i] = i < nr ? (ep.c_bf16 ? bf2f(c16[c0 + i * ep.ldc]) : c32[c0 + i * ep.ldc])
                                : 0.0f;
#pragma unroll
            for (int i = 0; i < 16; ++i) x[i] = fadd_rn(cv[i], x[i]);
          }
          if (ep.bias) {
            const float bias = __ldg(ep.bias + col);
#pragma unroll
            for (int i = 0; i < 16; ++i) x[i] = fadd_rn(x[i], bias);
          }
          if (ep.act) {
#pragma unroll
            for (int i = 0; i < 16; ++i) x[i] = apply_act(x[i], ep.act);
          }
          if (ep.res) {
            const float* rp = ep.res + (int64_t)(rbase + h0) * ep.ldr + col;
            float rv[16];
#pragma unroll
            for (int i = 0; i < 16; ++i) rv[i] = i < nr ? __ldg(rp + i * ep.ldr) : 0.0f;
#pragma unroll
            for (int i = 0; i < 16; ++i) x[i] = fadd_rn(x[i], rv[i]);
          }
          if (ep.c_bf16) {
#pragma unroll
            for (int i = 0; i < 16; ++i)
              if (i < nr) c16[c0 + i * ep.ldc] = f2bf(x[i]);
          } else {
#pragma unroll
            for (int i = 0; i < 16; ++i)
              if (i < nr) c32[c0 + i * ep.ldc] = x[i];
          }
        }
        }
        __syncwarp();  // staging free for the next chunk
      }
    }
  }
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  __syncthreads();
  if (warp == 1) {
    asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
    asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem),
                 "r"(TMEM_COLS));
  }
}

template <int BN, int STAGES>
constexpr int smem_bytes() {
  return STAGES * (BM * BK * 2 + BN * BK * 2) + 4 * 32 * 33 * 4 + 1024;
}

using EncodeFn = PFN_cuTensorMapEncodeTiled_v12000;

static EncodeFn get_encode() {
  static EncodeFn fn = nullptr;
  if (!fn) {
    void* p = nullptr;
    cudaDriverEntryPointQueryResult q;
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q) ==
            cudaSuccess &&
        q == cudaDriverEntryPointSuccess)
      fn = reinterpret_cast<EncodeFn>(p);
  }
  return fn;
}

// 2D bf16 map over a row-major [rows, cols] matrix with leading dim ld, box
// [box_rows, 64] with 128-byte swizzle; out-of-bounds elements read as zero.
static int make_map(CUtensorMap* map, const void* ptr, int64_t rows, int64_t cols, int64_t ld,
                    int box_rows) {
  EncodeFn enc = get_encode();
  if (!enc) {
    set_error("cuTensorMapEncodeTiled unavailable");
    return FQ_ERR_CUDA;
  }
  cuuint64_t dims[2] = {(cuuint64_t)cols, (cuuint64_t)rows};
  cuuint64_t strides[1] = {(cuuint64_t)(ld * 2)};
  cuuint32_t box[2] = {(cuuint32_t)BK, (cuuint32_t)box_rows};
  cuuint32_t estr[2] = {1, 1};
  CUresult r = enc(map, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2, const_cast<void*>(ptr), dims, strides,
                   box, estr, CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B,
                   CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  if (r != CUDA_SUCCESS) {
    set_error("cuTensorMapEncodeTiled failed (%d): rows=%lld cols=%lld ld=%lld", (int)r,
              (long long)rows, (long long)cols, (long long)ld);
    return FQ_ERR_CUDA;
  }
  return FQ_OK;
}

template <int BN, int STAGES>
static int launch(const void* a, int64_t lda, const void* b, int64_t ldb, const Epi& ep,
                  int64_t M, int64_t N, int64_t K, cudaStream_t s) {
  CUtensorMap ma, mb;
  int rc;
  if ((rc = make_map(&ma, a, M, K, lda, BM)) != FQ_OK) return rc;
  if ((rc = make_map(&mb, b, N, K, ldb, BN)) != FQ_OK) return rc;
  static int num_sms = 0;
  if (!num_sms) {
    int dev = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&num_sms, cudaDevAttrMultiProcessorCount, dev);
  }
  const int64_t ntiles = ((M + BM - 1) / BM) * ((N + BN - 1) / BN);
  const unsigned grid = (unsigned)(ntiles < num_sms ? ntiles : num_sms);
  tc_gemm_kernel<BN, STAGES><<<grid, kThreads, smem_bytes<BN, STAGES>(), s>>>(ma, mb, ep, (int)M,
                                                                             (int)N, (int)K);
  return launch_status("fq_gemm(tcgen05)");
}

template <int BN, int STAGES>
static int prep() {
  return cudaFuncSetAttribute(tc_gemm_kernel<BN, STAGES>,
                              cudaFuncAttributeMaxDynamicSharedMemorySize,
                              smem_bytes<BN, STAGES>()) == cudaSuccess
             ? FQ_OK
             : FQ_ERR_CUDA;
}

}  // namespace tc

int gemm_tc_prepare() {
  if (tc::prep<256, 4>() || tc::prep<128, 6>() || tc::prep<64, 8>() || tc::prep<32, 8>()) {
    set_error("fq_prepare: tcgen05 GEMM smem opt-in failed");
    return FQ_ERR_CUDA;
  }
  return FQ_OK;
}

int launch_tc_gemm(const void* a, int64_t lda, const void* b, int64_t ldb, void* c, int c_bf16,
                   int64_t ldc, int64_t M, int64_t N, int64_t K, int accumulate,
                   const float* bias, const float* res, int64_t ldr, int act, cudaStream_t s) {
  FQ_CHECK_ARG(lda % 8 == 0 && ldb % 8 == 0 && ((uintptr_t)a & 15) == 0 &&
                   ((uintptr_t)b & 15) == 0,
               FQ_ERR_DIMENSION, "tcgen05 GEMM: operands need 16-byte aligned rows (ld %% 8 == 0)");
  FQ_CHECK_ARG(M < (1LL << 31) && N < (1LL << 31) && K < (1LL << 31), FQ_ERR_DIMENSION,
               "tcgen05 GEMM: dimension too large");
  tc::Epi ep{c, ldc, c_bf16, accumulate, bias, res, ldr, act};
  // Widest N tile that still puts >= one CTA on every SM; the weight-streaming
  // decode GEMMs (M = rows <= 512) end up on narrow tiles.
  const int64_t mt = (M + tc::BM - 1) / tc::BM;
  auto tiles = [&](int bn) { return mt * ((N + bn - 1) / bn); };
  if (tiles(256) >= 148) return tc::launch<256, 4>(a, lda, b, ldb, ep, M, N, K, s);
  if (tiles(128) >= 148) return tc::launch<128, 6>(a, lda, b, ldb, ep, M, N, K, s);
  if (tiles(64) >= 148) return tc::launch<64, 8>(a, lda, b, ldb, ep, M, N, K, s);
  return tc::launch<32, 8>(a, lda, b, ldb, ep, M, N, K, s);
}

}  // namespace fq
