// Exact-mode fp32 GEMM (reference: tensor.py:179 gemm / :207 gemm_batched,
// numpy matmul -> OpenBLAS SGEMM).
//
// Why SIMT: SURVEY.md H1 measured that TF32 and fp16 operands flip beam
// selections while any fp32 (or f64) accumulation order keeps the tokens.
// This kernel therefore uses FFMA with a sequential K order per output element,
// independent of M and of the tiling, so results are bitwise invariant to
// batch sharding across GPUs (SURVEY §8(e) "Determinism across G").
// Fast (fp16) mode uses the tcgen05 kernel in fq_gemm_tc.cu instead.
//
// Epilogue (fused, fp32, separately rounded): t = acc (+C) (+bias); act; +res.
// This equals the reference's gemm followed by bias_residual_act_kernel
// bit for bit (kernels.py:45-53).
#include "fq_common.cuh"

namespace fq {

struct GemmArgs {
  const float* a;
  int64_t lda, sa0, sa1;
  const float* b;
  int64_t ldb, sb0, sb1;
  void* c;
  int64_t ldc, sc0, sc1;
  int64_t n1;  // inner batch extent (batch index z -> (z / n1, z % n1))
  int64_t M, N, K;
  int transpose_b, accumulate, act, c_f16;
  const float* bias;
  const float* res;
  int64_t ldr;
};

template <int BM, int BN, int BK, int TM, int TN>
__global__ void __launch_bounds__((BM / TM) * (BN / TN))
    sgemm_kernel(const GemmArgs p) {
  pdl_enter();
  constexpr int NT = (BM / TM) * (BN / TN);
  __shared__ float As[2][BK][BM + 4];
  __shared__ float Bs[2][BK][BN + 4];

  const int64_t z = blockIdx.z;
  const int64_t i0 = z / p.n1, i1 = z - i0 * p.n1;
  const float* A = p.a + i0 * p.sa0 + i1 * p.sa1;
  const float* B = p.b + i0 * p.sb0 + i1 * p.sb1;
  const int64_t m0 = (int64_t)blockIdx.y * BM, n0 = (int64_t)blockIdx.x * BN;
  const int tid = threadIdx.x;
  const int tx = tid % (BN / TN), ty = tid / (BN / TN);

  constexpr int A_PER = BM * BK / NT;  // elements of A tile per thread
  constexpr int B_PER = BN * BK / NT;
  float ra[A_PER], rb[B_PER];

  auto load_a = [&](int64_t k0) {
#pragma unroll
    for (int i = 0; i < A_PER; ++i) {
      int e = tid + i * NT;       // e in [0, BM*BK)
      int mm = e / BK, kk = e % BK;  // K fastest: coalesced along K
      int64_t gm = m0 + mm, gk = k0 + kk;
      ra[i] = (gm < p.M && gk < p.K) ? A[gm * p.lda + gk] : 0.0f;
    }
  };
  auto load_b = [&](int64_t k0) {
#pragma unroll
    for (int i = 0; i < B_PER; ++i) {
      int e = tid + i * NT;
      int nn, kk;
      if (p.transpose_b) { nn = e / BK; kk = e % BK; }  // B[N,K]: K fastest
      else { kk = e / BN; nn = e % BN; }                 // B[K,N]: N fastest
      int64_t gn = n0 + nn, gk = k0 + kk;
      float v = 0.0f;
      if (gn < p.N && gk < p.K) v = p.transpose_b ? B[gn * p.ldb + gk] : B[gk * p.ldb + gn];
      rb[i] = v;
    }
  };
  auto store_tiles = [&](int buf) {
#pragma unroll
    for (int i = 0; i < A_PER; ++i) {
      int e = tid + i * NT;
      As[buf][e % BK][e / BK] = ra[i];
    }
#pragma unroll
    for (int i = 0; i < B_PER; ++i) {
      int e = tid + i * NT;
      if (p.transpose_b) Bs[buf][e % BK][e / BK] = rb[i];
      else Bs[buf][e / BN][e % BN] = rb[i];
    }
  };

  float acc[TM][TN];
#pragma unroll
  for (int i = 0; i < TM; ++i)
#pragma unroll
    for (int j = 0; j < TN; ++j) acc[i][j] = 0.0f;

  const int64_t ktiles = (p.K + BK - 1) / BK;
  load_a(0);
  load_b(0);
  store_tiles(0);
  __syncthreads();
  for (int64_t kt = 0; kt < ktiles; ++kt) {
    const int buf = (int)(kt & 1);
    if (kt + 1 < ktiles) {
      load_a((kt + 1) * BK);
      load_b((kt + 1) * BK);
    }
#pragma unroll
    for (int kk = 0; kk < BK; ++kk) {
      float av[TM], bv[TN];
#pragma unroll
      for (int i = 0; i < TM; ++i) av[i] = As[buf][kk][ty * TM + i];
#pragma unroll
      for (int j = 0; j < TN; ++j) bv[j] = Bs[buf][kk][tx * TN + j];
#pragma unroll
      for (int i = 0; i < TM; ++i)
#pragma unroll
        for (int j = 0; j < TN; ++j) acc[i][j] = fmaf(av[i], bv[j], acc[i][j]);
    }
    if (kt + 1 < ktiles) {
      store_tiles(buf ^ 1);
    }
    __syncthreads();
  }

  // epilogue
  float* C32 = reinterpret_cast<float*>(p.c) + i0 * p.sc0 + i1 * p.sc1;
  h16* C16 = reinterpret_cast<fq::h16*>(p.c) + i0 * p.sc0 + i1 * p.sc1;
#pragma unroll
  for (int i = 0; i < TM; ++i) {
    int64_t gm = m0 + ty * TM + i;
    if (gm >= p.M) continue;
#pragma unroll
    for (int j = 0; j < TN; ++j) {
      int64_t gn = n0 + tx * TN + j;
      if (gn >= p.N) continue;
      float t = acc[i][j];
      if (p.accumulate) t = fadd_rn(p.c_f16 ? h2f(C16[gm * p.ldc + gn]) : C32[gm * p.ldc + gn], t);
      if (p.bias) t = fadd_rn(t, p.bias[gn]);
      t = apply_act(t, p.act);
      if (p.res) t = fadd_rn(t, p.res[gm * p.ldr + gn]);
      if (p.c_f16) C16[gm * p.ldc + gn] = f2h(t);
      else C32[gm * p.ldc + gn] = t;
    }
  }
}

int launch_sgemm(const GemmArgs& p, int64_t nbatch, cudaStream_t s) {
  // Pick the tile so the grid covers the 148 SMs; tiling never changes the
  // per-element K order, so both configs give identical bits.
  int64_t big_tiles = ((p.M + 127) / 128) * ((p.N + 127) / 128) * nbatch;
  if (big_tiles >= 2 * 148) {
    dim3 grid((unsigned)((p.N + 127) / 128), (unsigned)((p.M + 127) / 128), (unsigned)nbatch);
    launch_kernel(sgemm_kernel<128, 128, 8, 8, 8>, grid, 256, 0, s, 1u, p);
  } else if (p.M <= 16 || p.N <= 16) {
    dim3 grid((unsigned)((p.N + 31) / 32), (unsigned)((p.M + 31) / 32), (unsigned)nbatch);
    launch_kernel(sgemm_kernel<32, 32, 16, 2, 2>, grid, 256, 0, s, 1u, p);
  } else {
    dim3 grid((unsigned)((p.N + 63) / 64), (unsigned)((p.M + 63) / 64), (unsigned)nbatch);
    launch_kernel(sgemm_kernel<64, 64, 16, 4, 4>, grid, 256, 0, s, 1u, p);
  }
  return launch_status("fq_gemm(simt)");
}

// tcgen05 path (fq_gemm_tc.cu)
int launch_tc_gemm(const void* a, int64_t lda, const void* b, int64_t ldb, void* c, int c_f16,
                   int64_t ldc, int64_t M, int64_t N, int64_t K, int accumulate,
                   const float* bias, const float* res, int64_t ldr, int act, cudaStream_t s);

int launch_x3_gemm(const float* a, int64_t lda, const float* b, const float* b_lo, int64_t ldb,
                   float* c, int64_t ldc, int64_t M, int64_t N, int64_t K, int accumulate,
                   const float* bias, const float* res, int64_t ldr, int act, cudaStream_t s);

static bool ranges_overlap(const void* a, size_t na, const void* b, size_t nb) {
  const char* pa = (const char*)a;
  const char* pb = (const char*)b;
  return pa < pb + nb && pb < pa + na;
}

}  // namespace fq

using namespace fq;

extern "C" {

int fq_gemm(const void* a, int a_dtype, int64_t lda, const void* b, int b_dtype, int64_t ldb,
            int transpose_b, void* c, int c_dtype, int64_t ldc, int64_t M, int64_t N, int64_t K,
            int accumulate, const float* bias, const float* residual, int64_t ldr, int act,
            fq_stream_t stream) {
  FQ_CHECK_ARG(a && b && c && M >= 0 && N >= 0 && K >= 1, FQ_ERR_DIMENSION,
               "fq_gemm: bad shape M=%lld N=%lld K=%lld", (long long)M, (long long)N,
               (long long)K);
  FQ_CHECK_ARG(a_dtype == b_dtype, FQ_ERR_UNSUPPORTED, "fq_gemm: mixed operand dtypes");
  FQ_CHECK_ARG(act >= 0 && act <= 2, FQ_ERR_PARAMETER, "fq_gemm: unknown activation");
  if (M == 0 || N == 0) return FQ_OK;
  const size_t es = a_dtype == FQ_F32 ? 4 : 2;
  const size_t ces = c_dtype == FQ_F32 ? 4 : 2;
  const size_t ca = ((M - 1) * lda + K) * es;
  const size_t cb = (transpose_b ? (N - 1) * ldb + K : (K - 1) * ldb + N) * es;
  const size_t cc = ((M - 1) * ldc + N) * ces;
  FQ_CHECK_ARG(!ranges_overlap(c, cc, a, ca) && !ranges_overlap(c, cc, b, cb), FQ_ERR_ALIASING,
               "gemm output overlaps an input buffer");  // tensor.py:173-176
  if (a_dtype == FQ_F32 && transpose_b && c_dtype == FQ_F32 && lda % 4 == 0 && ldb % 4 == 0 &&
      ((uintptr_t)a & 15) == 0 && ((uintptr_t)b & 15) == 0 && getenv("FQ_SIMT_GEMM") == nullptr)
    return launch_x3_gemm((const float*)a, lda, (const float*)b, nullptr, ldb, (float*)c, ldc, M,
                          N, K, accumulate, bias, residual, ldr, act, as_stream(stream));
  if (a_dtype == FQ_F32) {
    GemmArgs p{};
    p.a = (const float*)a; p.lda = lda;
    p.b = (const float*)b; p.ldb = ldb;
    p.c = c; p.ldc = ldc; p.n1 = 1;
    p.M = M; p.N = N; p.K = K;
    p.transpose_b = transpose_b; p.accumulate = accumulate; p.act = act;
    p.c_f16 = c_dtype == FQ_F16;
    p.bias = bias; p.res = residual; p.ldr = ldr;
    return launch_sgemm(p, 1, as_stream(stream));
  }
  FQ_CHECK_ARG(a_dtype == FQ_F16 && transpose_b, FQ_ERR_UNSUPPORTED,
               "fp16 GEMM needs K-major B ([N,K], transpose_b=1)");
  return launch_tc_gemm(a, lda, b, ldb, c, c_dtype == FQ_F16, ldc, M, N, K, accumulate, bias,
                        residual, ldr, act, as_stream(stream));
}

int fq_gemm_batched(const float* a, int64_t lda, int64_t sa0, int64_t sa1, const float* b,
                    int64_t ldb, int64_t sb0, int64_t sb1, int transpose_b, float* c,
                    int64_t ldc, int64_t sc0, int64_t sc1, int64_t n0, int64_t n1, int64_t M,
                    int64_t N, int64_t K, fq_stream_t stream) {
  FQ_CHECK_ARG(a && b && c && n0 > 0 && n1 > 0 && M >= 0 && N >= 0 && K >= 1,
               FQ_ERR_DIMENSION, "fq_gemm_batched: bad shape");
  FQ_CHECK_ARG(n0 * n1 <= 65535, FQ_ERR_DIMENSION, "fq_gemm_batched: batch too large");
  if (M == 0 || N == 0) return FQ_OK;
  GemmArgs p{};
  p.a = a; p.lda = lda; p.sa0 = sa0; p.sa1 = sa1;
  p.b = b; p.ldb = ldb; p.sb0 = sb0; p.sb1 = sb1;
  p.c = c; p.ldc = ldc; p.sc0 = sc0; p.sc1 = sc1;
  p.n1 = n1; p.M = M; p.N = N; p.K = K;
  p.transpose_b = transpose_b;
  return launch_sgemm(p, n0 * n1, as_stream(stream));
}

}  // extern "C"
