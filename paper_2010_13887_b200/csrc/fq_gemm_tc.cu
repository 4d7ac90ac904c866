// fp16 GEMM on the 5th-generation tensor cores (tcgen05 + TMEM + TMA), sm_100a.
//
// C[M,N] = epilogue(A[M,K] . B[N,K]^T), A and B fp16 K-major (weights were
// re-laid out to [N,K] once at load), fp32 accumulation in TMEM.
//
// Persistent, warp-specialised, one 128 x BN output tile per CTA iteration:
//   warp 0      TMA producer: 2D tiled loads (128B swizzle) into a STAGES-deep
//               shared-memory ring, mbarrier complete_tx;
//   warp 1      TMEM allocator + single-thread tcgen05.mma issuer
//               (M=128, N=BN, K=16 per instruction); tcgen05.commit frees ring
//               slots and signals one of two TMEM accumulator stages;
//   warps 2..5  epilogue: tcgen05.ld 32x32b.x32, transpose through smem,
//               fused (+C) (+bias) act (+residual), coalesced fp32/fp16 stores,
//               overlapping the next tile's MMAs.
// Thread-block clusters of cm x cn CTAs share operands through TMA multicast:
// the cn CTAs of a cluster row (same M-tile) each load 1/cn of the A tile and
// multicast it to the row; the cm CTAs of a column (same N-tile) do the same
// for B. L2->SM traffic drops by cn (A) and cm (B) — the decode GEMMs
// (M = batch*beam = 512) were L2-bandwidth bound re-reading A once per N-tile.
// The fused epilogue is the reference's bias_residual_act pass (kernels.py:39-53)
// applied to the accumulator, so the [M,N] pre-activation never reaches HBM.
#include <cuda.h>
#include <cudaTypedefs.h>

#include <algorithm>
#include <cmath>
#include <cstdio>
#include <cstdlib>

#include "fq_common.cuh"

namespace fq {

namespace tc {

constexpr int BM = 128;
constexpr int BK = 64;  // 64 fp16 = 128 bytes = one swizzle row
constexpr int kThreads = 192;
// OP_X3 (exact fp32 mode, 3xTF32): 2 more warps split each staged fp32 tile
// (8 warps in all: 320 threads would cap registers at 168, below the
// epilogue's 128-float row accumulator + chunk registers)
// OP_X3H (exact fp32 mode, 3xFP16): operands arrive pre-split as fp16 pairs
// x = hi + lo * 2^-11 (hi = fp16(x), lo = fp16((x - hi) * 2^11): 22
// significant bits, the tf32 pair's precision at twice the kind::f16 MMA rate
// and half its bytes) written by the producing kernels; no converter warps.
constexpr int OP_F16 = 0, OP_X3 = 1, OP_X3H = 2;
constexpr int kThreadsX3 = 256;
constexpr int kConvThreads = kThreadsX3 - kThreads;
// OP_X3 / OP_X3H: K blocks (of 32 / 64 elements) per TMEM accumulation chunk,
// summed in registers: 128 K elements per chunk either way
constexpr int X3_CH = 4;
template <int OP>
__host__ __device__ constexpr int threads_of() { return OP == OP_X3 ? kThreadsX3 : kThreads; }
template <int OP>
__host__ __device__ constexpr int kblock() { return OP == OP_X3 ? 32 : BK; }  // K elements per 128-byte row
template <int OP>
__host__ __device__ constexpr int xchunk() { return OP == OP_X3 ? X3_CH : X3_CH / 2; }
template <int OP>
__host__ __device__ constexpr bool split3() { return OP == OP_X3 || OP == OP_X3H; }
// scale of the small-term accumulator (OP_X3H: lo carries 2^11)
template <int OP>
__host__ __device__ constexpr float small_scale() { return OP == OP_X3H ? 1.0f / 2048.0f : 1.0f; }

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

// TMA tensor store of one smem box (bulk-group completion).
__device__ __forceinline__ void tma_store_2d(const CUtensorMap* map, const void* src, int c0,
                                             int c1) {
  asm volatile(
      "cp.async.bulk.tensor.2d.global.shared::cta.bulk_group [%0, {%1, %2}], [%3];" ::"l"(
          reinterpret_cast<uint64_t>(map)),
      "r"(c0), "r"(c1), "r"(smem_u32(src))
      : "memory");
  asm volatile("cp.async.bulk.commit_group;" ::: "memory");
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

// kind::f16 instruction descriptor: f16 x f16 -> f32 (a/b format 0 = F16),
// both K-major.
__host__ __device__ constexpr uint32_t idesc_f16(int m, int n) {
  return (1u << 4) | ((uint32_t)(n >> 3) << 17) |
         ((uint32_t)(m >> 4) << 24);
}

__device__ __forceinline__ void mma_f16(uint32_t tmem_d, uint64_t adesc, uint64_t bdesc,
                                         uint32_t idesc, uint32_t accumulate) {
  asm volatile(
      "{\n\t.reg .pred p;\n\t"
      "setp.ne.b32 p, %4, 0;\n\t"
      "tcgen05.mma.cta_group::1.kind::f16 [%0], %1, %2, %3, p;\n}" ::"r"(tmem_d),
      "l"(adesc), "l"(bdesc), "r"(idesc), "r"(accumulate));
}

// kind::tf32 instruction descriptor: tf32 x tf32 -> f32, both K-major (K = 8 per MMA).
__host__ __device__ constexpr uint32_t idesc_tf32(int m, int n) {
  return (1u << 4) | (2u << 7) | (2u << 10) | ((uint32_t)(n >> 3) << 17) |
         ((uint32_t)(m >> 4) << 24);
}

__device__ __forceinline__ void mma_tf32(uint32_t tmem_d, uint64_t adesc, uint64_t bdesc,
                                         uint32_t idesc, uint32_t accumulate) {
  asm volatile(
      "{\n\t.reg .pred p;\n\t"
      "setp.ne.b32 p, %4, 0;\n\t"
      "tcgen05.mma.cta_group::1.kind::tf32 [%0], %1, %2, %3, p;\n}" ::"r"(tmem_d),
      "l"(adesc), "l"(bdesc), "r"(idesc), "r"(accumulate));
}

// 3xTF32 product of one 128-byte K block held in shared memory as hi/lo
// pairs (x = hi + lo, both exactly representable in tf32): per MMA-K step of
// 8, big += a_hi.b_hi and small += a_hi.b_lo + a_lo.b_hi (the a_lo.b_lo term,
// 2^-22 relative, is dropped). Two accumulators: the small terms never round
// against the large partial sum. Issued by one thread.
__device__ __forceinline__ void mma_x3_block(uint32_t big, uint32_t small, uint32_t a_hi,
                                             uint32_t a_lo, uint32_t b_hi, uint32_t b_lo,
                                             uint32_t idesc, bool first) {
#pragma unroll
  for (int k = 0; k < 4; ++k) {
    const uint32_t acc = (first && k == 0) ? 0u : 1u;
    mma_tf32(small, sw128_desc(a_hi + k * 32), sw128_desc(b_lo + k * 32), idesc, acc);
    mma_tf32(small, sw128_desc(a_lo + k * 32), sw128_desc(b_hi + k * 32), idesc, 1u);
    mma_tf32(big, sw128_desc(a_hi + k * 32), sw128_desc(b_hi + k * 32), idesc, acc);
  }
}

// Split n16 16-byte chunks of fp32 in shared memory in place into their
// tf32 "hi" part (round to nearest, ties away) and write the remainder, also
// rounded to tf32, at the same offset in `lo`: x = hi + lo + O(2^-22 |x|).
// Elementwise, so the 128B-swizzled layout the TMA wrote is preserved.
__device__ __forceinline__ uint32_t tf32_rna(float x) {
  uint32_t r;
  asm("cvt.rna.tf32.f32 %0, %1;" : "=r"(r) : "f"(x));
  return r;
}
__device__ __forceinline__ void split_tf32_smem(uint8_t* buf, uint8_t* lo, int n16, int t,
                                                int nt) {
  for (int i = t; i < n16; i += nt) {
    float4 x = *reinterpret_cast<const float4*>(buf + i * 16);
    uint4 h, l;
    h.x = tf32_rna(x.x); l.x = tf32_rna(x.x - __uint_as_float(h.x));
    h.y = tf32_rna(x.y); l.y = tf32_rna(x.y - __uint_as_float(h.y));
    h.z = tf32_rna(x.z); l.z = tf32_rna(x.z - __uint_as_float(h.z));
    h.w = tf32_rna(x.w); l.w = tf32_rna(x.w - __uint_as_float(h.w));
    *reinterpret_cast<uint4*>(buf + i * 16) = h;
    *reinterpret_cast<uint4*>(lo + i * 16) = l;
  }
}

// OP_X3H: the same three products on fp16 pairs, K = 16 per kind::f16 MMA:
// big += a_hi.b_hi, small += a_hi.b_lo + a_lo.b_hi (lo scaled by 2^11).
__device__ __forceinline__ void mma_xh_block(uint32_t big, uint32_t small, uint32_t a_hi,
                                             uint32_t a_lo, uint32_t b_hi, uint32_t b_lo,
                                             uint32_t idesc, bool first) {
#pragma unroll
  for (int k = 0; k < 4; ++k) {
    const uint32_t acc = (first && k == 0) ? 0u : 1u;
    mma_f16(small, sw128_desc(a_hi + k * 32), sw128_desc(b_lo + k * 32), idesc, acc);
    mma_f16(small, sw128_desc(a_lo + k * 32), sw128_desc(b_hi + k * 32), idesc, 1u);
    mma_f16(big, sw128_desc(a_hi + k * 32), sw128_desc(b_hi + k * 32), idesc, acc);
  }
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

// 32 columns without the wait (the caller batches several loads per wait::ld).
__device__ __forceinline__ void tmem_ld32_nowait(uint32_t taddr, uint32_t (&r)[32]) {
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
}

// 16 columns of this warp's 32 TMEM lanes (thread = lane = row).
__device__ __forceinline__ void tmem_ld16(uint32_t taddr, float* v) {
  uint32_t r[16];
  asm volatile(
      "tcgen05.ld.sync.aligned.32x32b.x16.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,"
      "%14,%15}, [%16];"
      : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]),
        "=r"(r[7]), "=r"(r[8]), "=r"(r[9]), "=r"(r[10]), "=r"(r[11]), "=r"(r[12]),
        "=r"(r[13]), "=r"(r[14]), "=r"(r[15])
      : "r"(taddr));
  asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
#pragma unroll
  for (int i = 0; i < 16; ++i) v[i] = __uint_as_float(r[i]);
}

// OP_X3 / OP_X3H: add one TMEM chunk slot (hi.hi at tb, small terms at tb +
// bn) to the thread's row accumulator: racc = racc + (big + small * SC), RN
// adds in a fixed order (SC a power of two: exact).
template <int BN, int OP>
__device__ __forceinline__ void x3_add_chunk(float (&racc)[BN], uint32_t tb, bool first) {
  if constexpr (BN % 32 == 0) {  // 32 columns of each accumulator per tcgen05.wait::ld
#pragma unroll
    for (int j = 0; j < BN / 32; ++j) {
      uint32_t rb[32], rs[32];
      tmem_ld32_nowait(tb + j * 32, rb);
      tmem_ld32_nowait(tb + BN + j * 32, rs);
      asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
#pragma unroll
      for (int i = 0; i < 32; ++i) {
        const float vs = __uint_as_float(rs[i]);
        const float t = fadd_rn(__uint_as_float(rb[i]),
                                OP == OP_X3H ? vs * small_scale<OP>() : vs);
        racc[j * 32 + i] = first ? t : fadd_rn(racc[j * 32 + i], t);
      }
    }
  } else {
#pragma unroll
    for (int j = 0; j < BN / 16; ++j) {
      float vb[16], vs[16];
      tmem_ld16(tb + j * 16, vb);
      tmem_ld16(tb + BN + j * 16, vs);
#pragma unroll
      for (int i = 0; i < 16; ++i) {
        const float t = fadd_rn(vb[i], OP == OP_X3H ? vs[i] * small_scale<OP>() : vs[i]);
        racc[j * 16 + i] = first ? t : fadd_rn(racc[j * 16 + i], t);
      }
    }
  }
}

__device__ __forceinline__ void mbar_arrive(uint64_t* bar) {
  asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem_u32(bar)) : "memory");
}

struct Epi {
  void* c;
  int64_t ldc;
  int c_f16;
  int accumulate;
  const float* bias;
  const float* res;
  int64_t ldr;
  int act;
  unsigned long long* dbg;  // per-CTA [start, end] %globaltimer (profiling only)
  int tstore;  // 1: C through TMA tensor stores (tma_c: 32-row x 128-byte boxes)
  int b_presplit;  // OP_X3: B arrives as tf32 hi (tma_b) + lo (tma_blo) pairs
  int chunk_kb;    // OP_X3H: K blocks per TMEM accumulation chunk (0: xchunk)
  void* c_lo;      // non-null (with c_f16): C is the exact mode's fp16 pair, hi at c, lo here
};

// HARS stage-1 statistics computed in the logits GEMM's epilogue (the [rows,
// V] logits are never written): per row and column tile the strided group
// maxima (published to the row's running maxima with global atomics), the
// tile-row maximum and sum of exp(x - max), and every element >= the row's
// current bound min_g(running group max) <= R as a survivor.
struct HarsEpi {
  const int32_t* dk;  // [M] group count per row (0: row not searched)
  int* gmax;          // [M][32] row group maxima, ordered ints (-inf between steps)
  float* tmax;        // [M][ldt] tile-row maxima
  double* tsum;       // [M][ldt] sum over the tile-row of exp(x - tmax)
  int* sv_cnt;        // [M][ldt] survivors of the tile-row (may exceed sv_cap: overflow)
  int2* sv;           // [M][ldt][sv_cap] survivors (column, value bits)
  int sv_cap;
  int ldt;
};

// LayerNorm of the split-K GEMM's output rows folded into its epilogue
// (bias + residual + LN, kernels.py:57-73): every CTA of the row block
// publishes per-row partial statistics of its 32 x BN slice (sum and the sum
// of squared deviations from the slice mean), the row block's CTAs meet at a
// global counter (all CTAs of the launch are co-resident: checked at launch),
// combine the N/BN partials (parallel-variance formula, f64) and normalise
// their own slice. ctr [mt][2] int32, zero between launches (self-resetting).
struct LnEpi {
  const float* gamma;
  const float* beta;
  double eps;
  float* out;
  int64_t ldo;
  h16* out16;
  int64_t ldo16;
  double2* stats;  // [M][nt]
  int* ctr;
  int nt;
};

__device__ __forceinline__ int hs_f2ord(float f) {
  const int i = __float_as_int(f);
  return i >= 0 ? i : i ^ 0x7fffffff;
}
__device__ __forceinline__ float hs_ord2f(int i) {
  return __int_as_float(i >= 0 ? i : i ^ 0x7fffffff);
}
__device__ __forceinline__ float hs_ex2(float x) {
  float y;
  asm("ex2.approx.ftz.f32 %0, %1;" : "=f"(y) : "f"(x));
  return y;
}

__device__ __forceinline__ uint32_t cluster_rank() {
  uint32_t r;
  asm volatile("mov.u32 %0, %%cluster_ctarank;" : "=r"(r));
  return r;
}

__device__ __forceinline__ void cluster_sync_all() {
  asm volatile("barrier.cluster.arrive.release.aligned;\n\tbarrier.cluster.wait.acquire.aligned;"
               ::: "memory");
}

__device__ __forceinline__ void tma_load_2d_mc(const CUtensorMap* map, uint64_t* bar, void* dst,
                                               int c0, int c1, uint16_t mask) {
  asm volatile(
      "cp.async.bulk.tensor.2d.shared::cluster.global.mbarrier::complete_tx::bytes"
      ".multicast::cluster [%0], [%1, {%2, %3}], [%4], %5;" ::"r"(smem_u32(dst)),
      "l"(reinterpret_cast<uint64_t>(map)), "r"(c0), "r"(c1), "r"(smem_u32(bar)), "h"(mask)
      : "memory");
}

__device__ __forceinline__ void mma_commit_mc(uint64_t* bar, uint16_t mask) {
  asm volatile(
      "tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.multicast::cluster.b64"
      " [%0], %1;" ::"r"(smem_u32(bar)),
      "h"(mask)
      : "memory");
}

// End of a TMA-store epilogue: the bulk stores complete (smem read, global
// writes performed) before the CTA moves on or exits. (Waiting only for the
// smem reads, .read, measured neutral at C2: the dependent grid waits for
// this grid's completion either way.)
__device__ __forceinline__ void tma_store_drain() {
  asm volatile("cp.async.bulk.wait_group %0;" ::"n"(0) : "memory");
}

// Per-CTA phase stamps for scripts/xh_cta_anatomy.py: compiled in only with
// -DFQ_GEMM_STAMPS (scripts/build_variant.sh), off the product path.
__device__ __forceinline__ void dbg_stamp(unsigned long long* dbg, int slot) {
#ifdef FQ_GEMM_STAMPS
  if (dbg) {
    unsigned long long t_;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t_));
    dbg[8 * blockIdx.x + slot] = t_;
  }
#else
  (void)dbg;
  (void)slot;
#endif
}

// Persistent over tile groups: a cluster (cm x cn CTAs, rank r -> (ry = r / cn,
// rx = r % cn)) walks groups g = cluster_id, +num_clusters, ...; group g covers
// M-tiles [gm*cm, +cm) x N-tiles [gn*cn, +cn) with the M-group fastest so
// concurrent clusters share weight tiles in L2. Two TMEM accumulator stages let
// the epilogue of one tile overlap the MMAs of the next.
//
// OP_X3 (exact fp32 mode): A and B are fp32, each K block of 32 elements is one
// 128-byte swizzle row, and a stage holds [A hi | A lo | B hi | B lo]. The TMA
// writes raw fp32 A into "A hi" (and raw B into "B hi" unless B arrives
// pre-split); converter warps 6..7 split it in place into tf32 hi + lo, then
// the MMA warp issues three kind::tf32 MMAs per K step (mma_x3_block).
template <int BN, int STAGES, bool HS = false, int OP = OP_F16>
__global__ void __launch_bounds__(threads_of<OP>(), 1)
    tc_gemm_kernel(const __grid_constant__ CUtensorMap tma_a,
                   const __grid_constant__ CUtensorMap tma_b, const Epi ep, int M, int N, int K,
                   int cm, int cn, const HarsEpi he, const __grid_constant__ CUtensorMap tma_c,
                   const __grid_constant__ CUtensorMap tma_blo,
                   const __grid_constant__ CUtensorMap tma_alo,
                   const __grid_constant__ CUtensorMap tma_clo) {
  static_assert(OP == OP_F16 || !HS, "the HARS epilogue is fp16-only");
  constexpr bool X3 = OP == OP_X3;
  constexpr bool XH = OP == OP_X3H;
  constexpr bool XS = split3<OP>();
  constexpr int KB = kblock<OP>();
  constexpr int A_BYTES = BM * 128;
  constexpr int B_BYTES = BN * 128;
  constexpr int STAGE_BYTES = XS ? 2 * (A_BYTES + B_BYTES) : A_BYTES + B_BYTES;
  constexpr int B_OFF = XS ? 2 * A_BYTES : A_BYTES;  // B (hi) inside a stage
  // two accumulator stages (OP_X3: two chunk slots x {hi.hi, small terms});
  // the allocation is a power of two >= 32 columns
  constexpr int TCOLS = XS ? 4 * BN : 2 * BN;
  static_assert(TCOLS <= 512, "TMEM holds 512 columns");
  constexpr uint32_t TMEM_COLS = TCOLS <= 32 ? 32 : TCOLS <= 64 ? 64 : TCOLS <= 128 ? 128
                                 : TCOLS <= 256 ? 256 : 512;
  extern __shared__ uint8_t smem_raw[];
  // 1024-B aligned (128B-swizzle atoms); identical offset in every CTA, so a
  // multicast lands at the same place cluster-wide. Pointer arithmetic keeps
  // the shared address space visible (LDS/STS, not generic LD/ST).
  uint8_t* smem = smem_raw + ((1024u - (smem_u32(smem_raw) & 1023u)) & 1023u);
  float* stage_out = reinterpret_cast<float*>(smem + STAGES * STAGE_BYTES);  // 4 x [32][33]
  __shared__ __align__(8) uint64_t full_bar[STAGES];
  __shared__ __align__(8) uint64_t empty_bar[STAGES];
  __shared__ __align__(8) uint64_t tfull_bar[2];
  __shared__ __align__(8) uint64_t tempty_bar[2];
  __shared__ __align__(8) uint64_t edone_bar;  // the 4 epilogue warps finished with TMEM
  __shared__ __align__(8) uint64_t conv_bar[X3 ? STAGES : 1];  // stage split (OP_X3)
  __shared__ uint32_t tmem_base_sh;

  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  pdl_launch_dependents();
  if (threadIdx.x == 0) dbg_stamp(ep.dbg, 0);
  const int csize = cm * cn;
  const int rank = csize > 1 ? (int)cluster_rank() : 0;
  const int ry = rank / cn, rx = rank % cn;
  const int num_kb = (K + KB - 1) / KB;
  // bytes one stage's TMA loads deliver
  const uint32_t tx_bytes = X3 ? A_BYTES + (ep.b_presplit ? 2 : 1) * B_BYTES : STAGE_BYTES;
  const int mt = (M + BM - 1) / BM, nt = (N + BN - 1) / BN;
  const int mg = mt / cm;                     // cm | mt and cn | nt (host guarantees)
  const int ngroups = mg * (nt / cn);
  const int cluster_id = blockIdx.x / csize, nclusters = gridDim.x / csize;
  uint16_t row_mask = 0, col_mask = 0;        // CTAs sharing my A tile / my B tile
  for (int x = 0; x < cn; ++x) row_mask |= (uint16_t)(1u << (ry * cn + x));
  for (int y = 0; y < cm; ++y) col_mask |= (uint16_t)(1u << (y * cn + rx));
  const uint16_t peer_mask = row_mask | col_mask;

  if (warp == 0 && lane == 0) {
    for (int s = 0; s < STAGES; ++s) {
      mbar_init(&full_bar[s], 1);
      mbar_init(&empty_bar[s], cm + cn - 1);  // every CTA that multicasts into my ring
    }
    for (int s = 0; s < 2; ++s) {
      mbar_init(&tfull_bar[s], 1);
      mbar_init(&tempty_bar[s], 4);  // one arrive per epilogue warp
    }
    mbar_init(&edone_bar, 4);
    if constexpr (X3)
      for (int s = 0; s < STAGES; ++s) mbar_init(&conv_bar[s], kConvThreads / 32);  // one per converter warp
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
  if (csize > 1) cluster_sync_all();  // peers' barriers initialised before any multicast
  else __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
  const uint32_t tmem = tmem_base_sh;
  if (threadIdx.x == 0) dbg_stamp(ep.dbg, 1);

  if (warp == 0) {
    if (lane == 0) {  // ---- TMA producer ----
      const int a_rows = BM / cn, b_rows = BN / cm;
      // Weights (B) do not depend on the previous kernel: stream the first
      // tile's first stages of B before the grid-dependency wait.
      int npre = 0;
      if (csize == 1 && cluster_id < ngroups) {
        const int n0 = (cluster_id / mg) * BN;
        npre = num_kb < STAGES ? num_kb : STAGES;
        for (int kb = 0; kb < npre; ++kb) {
          uint8_t* sa = smem + kb * STAGE_BYTES;
          mbar_expect_tx(&full_bar[kb], tx_bytes);
          tma_load_2d(&tma_b, &full_bar[kb], sa + B_OFF, kb * KB, n0);
          if ((X3 && ep.b_presplit) || XH)
            tma_load_2d(&tma_blo, &full_bar[kb], sa + B_OFF + B_BYTES, kb * KB, n0);
        }
      }
      pdl_wait();  // activations (A) are written by the previous kernel
      int it = 0;
      for (int g = cluster_id; g < ngroups; g += nclusters) {
        const int m0 = ((g % mg) * cm + ry) * BM, n0 = ((g / mg) * cn + rx) * BN;
        for (int kb = 0; kb < num_kb; ++kb, ++it) {
          const int s = it % STAGES;
          const uint32_t ph = (it / STAGES) & 1;
          uint8_t* sa = smem + s * STAGE_BYTES;
          if (it < npre) {  // B already in flight
            tma_load_2d(&tma_a, &full_bar[s], sa, kb * KB, m0);
            if (XH) tma_load_2d(&tma_alo, &full_bar[s], sa + A_BYTES, kb * KB, m0);
            continue;
          }
          mbar_wait(&empty_bar[s], ph ^ 1);  // free in every CTA I multicast into
          mbar_expect_tx(&full_bar[s], tx_bytes);
          if (cn > 1)
            tma_load_2d_mc(&tma_a, &full_bar[s], sa + rx * a_rows * 128, kb * KB,
                           m0 + rx * a_rows, row_mask);
          else
            tma_load_2d(&tma_a, &full_bar[s], sa, kb * KB, m0);
          if (XH) tma_load_2d(&tma_alo, &full_bar[s], sa + A_BYTES, kb * KB, m0);
          if (cm > 1)
            tma_load_2d_mc(&tma_b, &full_bar[s], sa + B_OFF + ry * b_rows * 128, kb * KB,
                           n0 + ry * b_rows, col_mask);
          else
            tma_load_2d(&tma_b, &full_bar[s], sa + B_OFF, kb * KB, n0);
          if ((X3 && ep.b_presplit) || XH)
            tma_load_2d(&tma_blo, &full_bar[s], sa + B_OFF + B_BYTES, kb * KB, n0);
        }
      }
      // drain: every peer's release of my last fills has landed before teardown
      for (int j = 0; j < STAGES; ++j, ++it) mbar_wait(&empty_bar[it % STAGES], ((it / STAGES) & 1) ^ 1);
    }
  } else if (warp == 1) {
    if (lane == 0) {  // ---- MMA issuer ----
      constexpr uint32_t idesc = X3 ? idesc_tf32(BM, BN) : idesc_f16(BM, BN);
      int it = 0, local = 0;
      if constexpr (XS) {  // chunks of xchunk K blocks into ping-pong TMEM slots
        const int CH = (XH && ep.chunk_kb > 0) ? ep.chunk_kb : xchunk<OP>();
        int gc = 0;
        for (int g = cluster_id; g < ngroups; g += nclusters) {
          for (int kb0 = 0; kb0 < num_kb; kb0 += CH, ++gc) {
            const int slot = gc & 1;
            mbar_wait(&tempty_bar[slot], ((gc >> 1) & 1) ^ 1);  // epilogue read the slot
            asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
            const uint32_t big = tmem + slot * 2 * BN;
            const int kb1 = min(num_kb, kb0 + CH);
            for (int kb = kb0; kb < kb1; ++kb, ++it) {
              const int s = it % STAGES;
              if constexpr (X3) mbar_wait(&conv_bar[s], (it / STAGES) & 1);
              else mbar_wait(&full_bar[s], (it / STAGES) & 1);
              if (it == 0) dbg_stamp(ep.dbg, 2);
              asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
              const uint32_t a_base = smem_u32(smem + s * STAGE_BYTES);
              const uint32_t b_base = a_base + B_OFF;
              if constexpr (X3)
                mma_x3_block(big, big + BN, a_base, a_base + A_BYTES, b_base, b_base + B_BYTES,
                             idesc, kb == kb0);
              else
                mma_xh_block(big, big + BN, a_base, a_base + A_BYTES, b_base, b_base + B_BYTES,
                             idesc, kb == kb0);
              mma_commit(&empty_bar[s]);
            }
            mma_commit(&tfull_bar[slot]);
          }
        }
      }
      for (int g = cluster_id; g < ngroups && !XS; g += nclusters, ++local) {
        const int as = local & 1;
        mbar_wait(&tempty_bar[as], ((local >> 1) & 1) ^ 1);  // epilogue drained this stage
        asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
        const uint32_t acc = tmem + as * BN;
        for (int kb = 0; kb < num_kb; ++kb, ++it) {
          const int s = it % STAGES;
          const uint32_t ph = (it / STAGES) & 1;
          mbar_wait(X3 ? &conv_bar[s] : &full_bar[s], ph);
          if (it == 0) dbg_stamp(ep.dbg, 2);
          asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
          const uint32_t a_base = smem_u32(smem + s * STAGE_BYTES);
          const uint32_t b_base = a_base + B_OFF;
#pragma unroll
          for (int k = 0; k < BK / 16; ++k) {
            mma_f16(acc, sw128_desc(a_base + k * 32), sw128_desc(b_base + k * 32), idesc,
                     (kb | k) != 0);
          }
          // ring slot reusable (in me and in every CTA that multicasts into me)
          if (csize > 1) mma_commit_mc(&empty_bar[s], peer_mask);
          else mma_commit(&empty_bar[s]);
        }
        mma_commit(&tfull_bar[as]);   // accumulator stage complete
        if (local == 0) dbg_stamp(ep.dbg, 3);  // first tile's MMAs issued
      }
      dbg_stamp(ep.dbg, 7);  // every tile's MMAs issued
    }
  } else if (X3 && warp >= 6) {  // ---- converter: fp32 stage -> tf32 hi + lo ----
    const int t = threadIdx.x - 192;
    int it = 0;
    for (int g = cluster_id; g < ngroups; g += nclusters) {
      for (int kb = 0; kb < num_kb; ++kb, ++it) {
        const int s = it % STAGES;
        mbar_wait(&full_bar[s], (it / STAGES) & 1);
        uint8_t* sa = smem + s * STAGE_BYTES;
        split_tf32_smem(sa, sa + A_BYTES, A_BYTES / 16, t, kConvThreads);
        if (!ep.b_presplit)
          split_tf32_smem(sa + B_OFF, sa + B_OFF + B_BYTES, B_BYTES / 16, t, kConvThreads);
        asm volatile("fence.proxy.async.shared::cta;" ::: "memory");  // visible to the MMA
        __syncwarp();
        if (lane == 0) mbar_arrive(&conv_bar[s]);
      }
    }
  } else if constexpr (HS) {  // ---- HARS statistics epilogue (thread = row) ----
    pdl_wait();  // the group counts / running maxima come from the previous kernel
    const int q = warp & 3;
    float* gms = stage_out + 4 * 32 * 33 + ((warp - 2) * 32 + lane) * 33;  // per-thread scratch
    constexpr float L2E = 1.4426950408889634f;
    int local = 0;
    for (int g = cluster_id; g < ngroups; g += nclusters, ++local) {
      const int as = local & 1;
      const int m0 = ((g % mg) * cm + ry) * BM, n0 = ((g / mg) * cn + rx) * BN;
      const int r = m0 + q * 32 + lane;
      const int k = r < M ? he.dk[r] : 0;
      // running lower bound of the row's R from the group maxima other tiles
      // have already published (each read <= that group's final maximum, so
      // the min over groups <= R): tightens the survivor bound of later tiles
      // at no wait — the loads are in flight under this tile's mainloop
      float rest = -INFINITY;
      if (k == 8) {
        const int4 a0 = __ldcg(reinterpret_cast<const int4*>(he.gmax + (int64_t)r * 32));
        const int4 a1 = __ldcg(reinterpret_cast<const int4*>(he.gmax + (int64_t)r * 32 + 4));
        rest = fminf(fminf(fminf(hs_ord2f(a0.x), hs_ord2f(a0.y)), fminf(hs_ord2f(a0.z), hs_ord2f(a0.w))),
                     fminf(fminf(hs_ord2f(a1.x), hs_ord2f(a1.y)), fminf(hs_ord2f(a1.z), hs_ord2f(a1.w))));
      } else if (k > 0) {
        float mn = INFINITY;
        for (int gq = 0; gq < k; ++gq) mn = fminf(mn, hs_ord2f(__ldcg(he.gmax + (int64_t)r * 32 + gq)));
        rest = mn;
      }
      mbar_wait(&tfull_bar[as], (local >> 1) & 1);
      asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
      for (int gq = 0; gq < k; ++gq) gms[gq] = -INFINITY;
      // pass 1: tile-row maximum and group maxima (group of column c: c % k).
      // k = 8 (the steady beam-4 step, K + live): 32 % 8 == 0, so column j of
      // every 32-column chunk is in group (n0 + j) % 8 -> 8 register maxima
      // indexed at compile time; other k: per-thread shared-memory maxima.
      float mt = -INFINITY;
      float g8[8] = {-INFINITY, -INFINITY, -INFINITY, -INFINITY,
                     -INFINITY, -INFINITY, -INFINITY, -INFINITY};
      int gi = k > 0 ? n0 % k : 0;
#pragma unroll 1
      for (int cc = 0; cc < BN; cc += 32) {
        float v[32];
        tmem_ld32(tmem + as * BN + ((uint32_t)(q * 32) << 16) + cc, v);
        if (k == 8) {
          if (n0 + cc + 32 <= N) {
#pragma unroll
            for (int j = 0; j < 32; ++j) g8[j & 7] = fmaxf(g8[j & 7], v[j]);
          } else {
#pragma unroll
            for (int j = 0; j < 32; ++j)
              if (n0 + cc + j < N) g8[j & 7] = fmaxf(g8[j & 7], v[j]);
          }
        } else if (k > 0) {
#pragma unroll
          for (int j = 0; j < 32; ++j) {
            if (n0 + cc + j < N) gms[gi] = fmaxf(gms[gi], v[j]);
            if (++gi == k) gi = 0;
          }
        }
      }
      if (k == 8) {  // register q holds group (n0 + q) % 8
#pragma unroll
        for (int qq = 0; qq < 8; ++qq) gms[(n0 + qq) & 7] = g8[qq];
      }
      for (int gq = 0; gq < k; ++gq) mt = fmaxf(mt, gms[gq]);
      // publish the tile's group maxima into the row maxima (fire-and-forget
      // reductions); the survivor bound is the tile-local min over groups of the
      // tile's maxima (<= the row's R), so no global round trip is waited on
      float bound = INFINITY;
      if (k > 0) {
#pragma unroll
        for (int gq = 0; gq < 32; ++gq)
          if (gq < k) {
            atomicMax(he.gmax + (int64_t)r * 32 + gq, hs_f2ord(gms[gq]));
            bound = fminf(bound, gms[gq]);
          }
        bound = fmaxf(bound, rest);
      }
      // pass 2: sum exp(x - mt) (fp32 per 32-column chunk, f64 across chunks)
      // and survivors x >= bound: a branch-free per-chunk bit mask, then the set
      // bits (a few per chunk) re-read from the warp's staging row and stored to
      // the tile-row's own slots (no atomics)
      const float mL = mt * L2E;
      const int tn = n0 / BN;
      int2* svr = he.sv + ((int64_t)r * he.ldt + tn) * he.sv_cap;
      float* strow = stage_out + ((warp - 2) * 32 + lane) * 33;
      double s = 0.0;
      int ns = 0;
#pragma unroll 1
      for (int cc = 0; cc < BN; cc += 32) {
        float v[32];
        tmem_ld32(tmem + as * BN + ((uint32_t)(q * 32) << 16) + cc, v);
        if (cc + 32 >= BN) {  // last TMEM read of this stage: hand it back to the MMA warp
          asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
          __syncwarp();
          if (lane == 0) mbar_arrive(&tempty_bar[as]);
        }
        if (k > 0) {
          const int nval = min(32, N - (n0 + cc));  // valid columns of this chunk
          float t = 0.0f;
          uint32_t mask = 0u;
          if (nval >= 32) {
#pragma unroll
            for (int j = 0; j < 32; ++j) {
              t += hs_ex2(fmaf(v[j], L2E, -mL));  // fp16 mode: one-FMA argument
              mask |= (v[j] >= bound ? 1u : 0u) << j;
            }
          } else {
#pragma unroll
            for (int j = 0; j < 32; ++j)
              if (j < nval) {
                t += hs_ex2(fmaf(v[j], L2E, -mL));
                mask |= (v[j] >= bound ? 1u : 0u) << j;
              }
          }
          s += (double)t;
          if (mask) {
#pragma unroll
            for (int j = 0; j < 32; ++j) strow[j] = v[j];
            while (mask) {
              const int j = __ffs(mask) - 1;
              mask &= mask - 1u;
              if (ns < he.sv_cap) svr[ns] = make_int2(n0 + cc + j, __float_as_int(strow[j]));
              ++ns;
            }
          }
        }
      }
      if (k > 0) {
        he.sv_cnt[(int64_t)r * he.ldt + tn] = ns;
        he.tmax[(int64_t)r * he.ldt + tn] = mt;
        he.tsum[(int64_t)r * he.ldt + tn] = s;
      }
    }
  } else {  // ---- epilogue: warps 2..5 own TMEM lane quarters (warp % 4) ----
    pdl_wait();  // C / residual / bias may be touched by the previous kernel
    const int q = warp & 3;
    float* st = stage_out + (warp - 2) * 32 * 33;
    float* c32 = reinterpret_cast<float*>(ep.c);
    h16* c16 = reinterpret_cast<fq::h16*>(ep.c);
    int local = 0, gc = 0;
    for (int g = cluster_id; g < ngroups; g += nclusters, ++local) {
      const int as = local & 1;
      const int m0 = ((g % mg) * cm + ry) * BM, n0 = ((g / mg) * cn + rx) * BN;
      // the tile's bias columns are requested before the accumulator wait, so
      // their latency hides under the mainloop (per-chunk loads after the wait
      // cost one L2/HBM round trip per 32 columns: 7.7 -> ~1 us epilogue)
      float bpre[BN / 32];
#pragma unroll
      for (int j = 0; j < BN / 32; ++j) {
        const int bc = n0 + j * 32 + lane;
        bpre[j] = (ep.bias && bc < N) ? __ldg(ep.bias + bc) : 0.0f;
      }
      const int rbase = m0 + q * 32;
      const int nrows = min(32, M - rbase);
      // one 32-column chunk of this thread's row (thread = row): fused
      // epilogue and store
      auto store_chunk = [&](float (&v)[32], const int cc) {
        if (ep.tstore) {
          // thread = row: epilogue math on the tcgen05.ld registers, the
          // 32 x 32 chunk written swizzled into this warp's 4 KB box area
          // (conflict-free 16-byte stores), then one TMA tensor store per chunk
          // (full-line writes; fp32: one 4 KB box, fp16: two 2 KB boxes)
          uint8_t* box = reinterpret_cast<uint8_t*>(stage_out) + (warp - 2) * 4096;
          const int col0 = n0 + cc;
          if (ep.bias) {
#pragma unroll
            for (int j = 0; j < 8; ++j) {
              const float4 b = (col0 + 4 * j + 3 < N)
                                   ? __ldg(reinterpret_cast<const float4*>(ep.bias + col0 + 4 * j))
                                   : make_float4(0.f, 0.f, 0.f, 0.f);
              v[4 * j] = fadd_rn(v[4 * j], b.x);
              v[4 * j + 1] = fadd_rn(v[4 * j + 1], b.y);
              v[4 * j + 2] = fadd_rn(v[4 * j + 2], b.z);
              v[4 * j + 3] = fadd_rn(v[4 * j + 3], b.w);
            }
          }
          if (ep.act) {
#pragma unroll
            for (int j = 0; j < 32; ++j) v[j] = apply_act(v[j], ep.act);
          }
          if (lane == 0) {  // my box area is free again (fp16: the one two chunks back)
            if (ep.c_f16 && !ep.c_lo) asm volatile("cp.async.bulk.wait_group.read %0;" ::"n"(1) : "memory");
            else asm volatile("cp.async.bulk.wait_group.read %0;" ::"n"(0) : "memory");
          }
          __syncwarp();
          if (ep.c_lo) {  // exact-mode pair: hi box + lo box (32 rows x 64 B each)
#pragma unroll
            for (int j = 0; j < 4; ++j) {
              uint4 ph, pl;
              split_xh2(v[8 * j], v[8 * j + 1], ph.x, pl.x);
              split_xh2(v[8 * j + 2], v[8 * j + 3], ph.y, pl.y);
              split_xh2(v[8 * j + 4], v[8 * j + 5], ph.z, pl.z);
              split_xh2(v[8 * j + 6], v[8 * j + 7], ph.w, pl.w);
              const int off = lane * 64 + ((j ^ ((lane >> 1) & 3)) << 4);
              *reinterpret_cast<uint4*>(box + off) = ph;
              *reinterpret_cast<uint4*>(box + 2048 + off) = pl;
            }
            asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
            __syncwarp();
            if (lane == 0) {
              tma_store_2d(&tma_c, box, col0, rbase);
              tma_store_2d(&tma_clo, box + 2048, col0, rbase);
            }
          } else if (ep.c_f16) {
            uint8_t* bx = box + ((cc >> 5) & 1) * 2048;  // 32 rows x 64 B, 64-byte swizzle
#pragma unroll
            for (int j = 0; j < 4; ++j) {
              uint4 pk;
              h16x2 hh;
              hh = __floats2half2_rn(v[8 * j], v[8 * j + 1]);
              pk.x = *reinterpret_cast<uint32_t*>(&hh);
              hh = __floats2half2_rn(v[8 * j + 2], v[8 * j + 3]);
              pk.y = *reinterpret_cast<uint32_t*>(&hh);
              hh = __floats2half2_rn(v[8 * j + 4], v[8 * j + 5]);
              pk.z = *reinterpret_cast<uint32_t*>(&hh);
              hh = __floats2half2_rn(v[8 * j + 6], v[8 * j + 7]);
              pk.w = *reinterpret_cast<uint32_t*>(&hh);
              *reinterpret_cast<uint4*>(bx + lane * 64 + ((j ^ ((lane >> 1) & 3)) << 4)) = pk;
            }
            asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
            __syncwarp();
            if (lane == 0) tma_store_2d(&tma_c, bx, col0, rbase);
          } else {  // 32 rows x 128 B, 128-byte swizzle
#pragma unroll
            for (int j = 0; j < 8; ++j)
              *reinterpret_cast<float4*>(box + lane * 128 + ((j ^ (lane & 7)) << 4)) =
                  make_float4(v[4 * j], v[4 * j + 1], v[4 * j + 2], v[4 * j + 3]);
            asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
            __syncwarp();
            if (lane == 0) tma_store_2d(&tma_c, box, col0, rbase);
          }
          return;
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
            // all global reads of the rows issue before any store (no per-row
            // dependent latency); lanes own columns: 128-byte row segments
            const int64_t c0 = (int64_t)(rbase + h0) * ep.ldc + col;
            if (ep.accumulate) {
              float cv[16];
#pragma unroll
              for (int i = 0; i < 16; ++i)
                cv[i] = i < nr ? (ep.c_f16 ? h2f(c16[c0 + i * ep.ldc]) : c32[c0 + i * ep.ldc])
                               : 0.0f;
#pragma unroll
              for (int i = 0; i < 16; ++i) x[i] = fadd_rn(cv[i], x[i]);
            }
            if (ep.bias) {
              float bias = bpre[0];
#pragma unroll
              for (int j = 1; j < BN / 32; ++j)
                if (cc == j * 32) bias = bpre[j];
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
            if (ep.c_lo) {
              h16* c16lo = reinterpret_cast<fq::h16*>(ep.c_lo);
#pragma unroll
              for (int i = 0; i < 16; ++i)
                if (i < nr) split_xh(x[i], c16[c0 + i * ep.ldc], c16lo[c0 + i * ep.ldc]);
            } else if (ep.c_f16) {
#pragma unroll
              for (int i = 0; i < 16; ++i)
                if (i < nr) c16[c0 + i * ep.ldc] = f2h(x[i]);
            } else {
#pragma unroll
              for (int i = 0; i < 16; ++i)
                if (i < nr) c32[c0 + i * ep.ldc] = x[i];
            }
          }
        }
        __syncwarp();  // staging free for the next chunk
      };
      if constexpr (XS) {
        // the tile's K chunks (X3_CH K blocks each, ping-pong TMEM slots): per
        // chunk the hi.hi and the small-term accumulators are read and added
        // to this thread's row in registers with IEEE round-to-nearest adds
        // (the tensor core's own long accumulation is not RN: this bounds it
        // to X3_CH * 32 K elements)
        float racc[BN];
        const int CH = (XH && ep.chunk_kb > 0) ? ep.chunk_kb : xchunk<OP>();
        for (int kb0 = 0; kb0 < num_kb; kb0 += CH, ++gc) {
          const int slot = gc & 1;
          mbar_wait(&tfull_bar[slot], (gc >> 1) & 1);
          asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
          x3_add_chunk<BN, OP>(racc, tmem + slot * 2 * BN + ((uint32_t)(q * 32) << 16), kb0 == 0);
          asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
          __syncwarp();
          if (lane == 0) mbar_arrive(&tempty_bar[slot]);
        }
        if (local == 0 && threadIdx.x == 64) dbg_stamp(ep.dbg, 4);
#pragma unroll
        for (int j = 0; j < BN / 32; ++j) {
          float v[32];
#pragma unroll
          for (int i = 0; i < 32; ++i) v[i] = racc[j * 32 + i];
          store_chunk(v, j * 32);
        }
      } else {
        mbar_wait(&tfull_bar[as], (local >> 1) & 1);
        if (local == 0 && threadIdx.x == 64) dbg_stamp(ep.dbg, 4);
        asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
#pragma unroll 1
        for (int cc = 0; cc < BN; cc += 32) {
          float v[32];
          tmem_ld32(tmem + as * BN + ((uint32_t)(q * 32) << 16) + cc, v);
          if (cc + 32 >= BN) {  // last TMEM read of this stage: hand it back to the MMA warp
            asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
            __syncwarp();
            if (lane == 0) mbar_arrive(&tempty_bar[as]);
          }
          store_chunk(v, cc);
        }
      }
    }
  }
  if constexpr (!HS) {  // TMA stores complete before exit
    if (ep.tstore && warp >= 2 && warp < 6 && lane == 0) tma_store_drain();
  }
  if (threadIdx.x == 64) dbg_stamp(ep.dbg, 5);  // epilogue done
  __syncwarp();
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  if (warp >= 2 && warp < 6 && lane == 0) mbar_arrive(&edone_bar);
  if (csize > 1) cluster_sync_all();  // no CTA leaves while peers may still signal it
  else __syncthreads();
  if (threadIdx.x == 0) dbg_stamp(ep.dbg, 6);
  if (warp == 1) {
    // dealloc strictly after every epilogue warp's last tcgen05.ld (measured:
    // the block barrier alone released warps 0-1 before the epilogue ended)
    mbar_wait(&edone_bar, 0);
    asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
    asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem),
                 "r"(TMEM_COLS));
  }
}

// ---------------------------------------------------------------------------
// Split-K over a thread-block cluster for small-M GEMMs (the decode step's
// M = batch*beam rows). Per-SM TMA ingest (~40 B/clk measured) bounds these
// GEMMs: a 128 x BN tile needs (128 + BN) * K * 2 bytes per SM. Splitting K
// across the S CTAs of a cluster cuts each SM's bytes by S; the fp32 partial
// tiles are then reduced through distributed shared memory — CTA r sums rows
// [r*128/S, (r+1)*128/S) over all S partials in fixed rank order (deterministic)
// and applies the fused epilogue with 128-bit coalesced stores.
// ---------------------------------------------------------------------------
__device__ __forceinline__ uint32_t cluster_nrank() {
  uint32_t r;
  asm volatile("mov.u32 %0, %%cluster_nctarank;" : "=r"(r));
  return r;
}

__device__ __forceinline__ float4 ld_dsmem_f4(uint32_t local_addr, uint32_t rank) {
  uint32_t ra;
  asm("mapa.shared::cluster.u32 %0, %1, %2;" : "=r"(ra) : "r"(local_addr), "r"(rank));
  float4 v;
  // not volatile, no memory clobber: ordering comes from the cluster barrier,
  // and independent remote loads must be free to overlap (~200-cycle latency)
  asm("ld.shared::cluster.v4.f32 {%0, %1, %2, %3}, [%4];"
      : "=f"(v.x), "=f"(v.y), "=f"(v.z), "=f"(v.w)
      : "r"(ra));
  return v;
}

// SLAB: no cluster and no in-kernel reduction — split s writes its fp32
// partial tile to slab s of ep.c ([S][M][ldc], plain coalesced stores) and the
// consumer (fq_splitk_bias_residual_layer_norm) sums the S slabs in split
// order, so the result is bit-identical to the DSMEM reduction's.
// OP_X3: the exact-mode 3xTF32 operands (see tc_gemm_kernel).
template <int BN, int STAGES, bool LNF = false, bool SLAB = false, int OP = OP_F16>
__global__ void __launch_bounds__(threads_of<OP>(), 1)
    tc_gemm_splitk_kernel(const __grid_constant__ CUtensorMap tma_a,
                          const __grid_constant__ CUtensorMap tma_b, const Epi ep, int M, int N,
                          int K, int kb_per_split, const LnEpi ln, int nsplit,
                          const __grid_constant__ CUtensorMap tma_c,
                          const __grid_constant__ CUtensorMap tma_blo,
                          const __grid_constant__ CUtensorMap tma_alo) {
  static_assert(OP == OP_F16 || !LNF, "the in-kernel LN is fp16-only");
  constexpr bool X3 = OP == OP_X3;
  constexpr bool XH = OP == OP_X3H;
  constexpr bool XS = split3<OP>();
  constexpr int KB = kblock<OP>();
  constexpr int A_BYTES = BM * 128;
  constexpr int B_BYTES = BN * 128;
  constexpr int STAGE_BYTES = XS ? 2 * (A_BYTES + B_BYTES) : A_BYTES + B_BYTES;
  constexpr int B_OFF = XS ? 2 * A_BYTES : A_BYTES;
  // OP_X3: two chunk slots x {hi.hi, small terms} (see tc_gemm_kernel)
  constexpr uint32_t TMEM_COLS = XS ? 4 * BN : (BN < 32 ? 32 : BN);
  static_assert(TMEM_COLS <= 512, "TMEM holds 512 columns");
  constexpr int PLD = BN + 4;  // padded partial row (floats): conflict-free v4 rows
  static_assert(BM * PLD * 4 <= STAGES * STAGE_BYTES, "partial tile must fit the ring");
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = smem_raw + ((1024u - (smem_u32(smem_raw) & 1023u)) & 1023u);
  float* part = reinterpret_cast<float*>(smem);  // reuses the ring once all MMAs retired
  __shared__ __align__(8) uint64_t full_bar[STAGES];
  __shared__ __align__(8) uint64_t empty_bar[STAGES];
  __shared__ __align__(8) uint64_t tfull_bar;
  __shared__ __align__(8) uint64_t conv_bar[X3 ? STAGES : 1];
  __shared__ __align__(8) uint64_t xfull_bar[2], xempty_bar[2];  // OP_X3 chunk slots
  __shared__ uint32_t tmem_base_sh;

  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  pdl_launch_dependents();
  if (threadIdx.x == 0) dbg_stamp(ep.dbg, 0);
  const int S = SLAB ? nsplit : (int)cluster_nrank();
  const int rank = SLAB ? (int)(blockIdx.x % nsplit) : (int)cluster_rank();
  const int mt = (M + BM - 1) / BM;
  const int tile = blockIdx.x / S;
  const int m0 = (tile % mt) * BM, n0 = (tile / mt) * BN;
  const int num_kb = (K + KB - 1) / KB;
  const uint32_t tx_bytes = X3 ? A_BYTES + (ep.b_presplit ? 2 : 1) * B_BYTES : STAGE_BYTES;
  const int kb0 = rank * kb_per_split;
  const int kb1 = min(num_kb, kb0 + kb_per_split);

  if (warp == 0 && lane == 0) {
    for (int s = 0; s < STAGES; ++s) {
      mbar_init(&full_bar[s], 1);
      mbar_init(&empty_bar[s], 1);
      if constexpr (X3) mbar_init(&conv_bar[s], kConvThreads / 32);
    }
    mbar_init(&tfull_bar, 1);
    for (int s = 0; s < 2; ++s) {
      mbar_init(&xfull_bar[s], 1);
      mbar_init(&xempty_bar[s], 4);
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
  if (threadIdx.x == 0) dbg_stamp(ep.dbg, 1);

  if (warp == 0) {
    if (lane == 0) {  // ---- TMA producer: this CTA's K slice ----
      // weight stages first (independent of the previous kernel), then wait
      const int npre = (kb1 - kb0) < STAGES ? (kb1 - kb0) : STAGES;
      for (int it = 0; it < npre; ++it) {
        uint8_t* sa = smem + it * STAGE_BYTES;
        mbar_expect_tx(&full_bar[it], tx_bytes);
        tma_load_2d(&tma_b, &full_bar[it], sa + B_OFF, (kb0 + it) * KB, n0);
        if ((X3 && ep.b_presplit) || XH)
          tma_load_2d(&tma_blo, &full_bar[it], sa + B_OFF + B_BYTES, (kb0 + it) * KB, n0);
      }
      pdl_wait();
      for (int kb = kb0, it = 0; kb < kb1; ++kb, ++it) {
        const int s = it % STAGES;
        uint8_t* sa = smem + s * STAGE_BYTES;
        if (it < npre) {
          tma_load_2d(&tma_a, &full_bar[s], sa, kb * KB, m0);
          if (XH) tma_load_2d(&tma_alo, &full_bar[s], sa + A_BYTES, kb * KB, m0);
          continue;
        }
        mbar_wait(&empty_bar[s], ((it / STAGES) & 1) ^ 1);
        mbar_expect_tx(&full_bar[s], tx_bytes);
        tma_load_2d(&tma_a, &full_bar[s], sa, kb * KB, m0);
        if (XH) tma_load_2d(&tma_alo, &full_bar[s], sa + A_BYTES, kb * KB, m0);
        tma_load_2d(&tma_b, &full_bar[s], sa + B_OFF, kb * KB, n0);
        if ((X3 && ep.b_presplit) || XH)
          tma_load_2d(&tma_blo, &full_bar[s], sa + B_OFF + B_BYTES, kb * KB, n0);
      }
    }
  } else if (warp == 1) {
    if (lane == 0) {  // ---- MMA issuer ----
      constexpr uint32_t idesc = X3 ? idesc_tf32(BM, BN) : idesc_f16(BM, BN);
      if constexpr (XS) {  // chunks of xchunk K blocks into ping-pong TMEM slots
        const int CH = (XH && ep.chunk_kb > 0) ? ep.chunk_kb : xchunk<OP>();
        int it = 0, gc = 0;
        for (int c0 = kb0; c0 < kb1; c0 += CH, ++gc) {
          const int slot = gc & 1;
          mbar_wait(&xempty_bar[slot], ((gc >> 1) & 1) ^ 1);
          asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
          const uint32_t big = tmem + slot * 2 * BN;
          for (int kb = c0; kb < min(kb1, c0 + CH); ++kb, ++it) {
            const int s = it % STAGES;
            if constexpr (X3) mbar_wait(&conv_bar[s], (it / STAGES) & 1);
            else mbar_wait(&full_bar[s], (it / STAGES) & 1);
            if (it == 0) dbg_stamp(ep.dbg, 2);
            asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
            const uint32_t a_base = smem_u32(smem + s * STAGE_BYTES);
            const uint32_t b_base = a_base + B_OFF;
            if constexpr (X3)
              mma_x3_block(big, big + BN, a_base, a_base + A_BYTES, b_base, b_base + B_BYTES,
                           idesc, kb == c0);
            else
              mma_xh_block(big, big + BN, a_base, a_base + A_BYTES, b_base, b_base + B_BYTES,
                           idesc, kb == c0);
            mma_commit(&empty_bar[s]);
          }
          mma_commit(&xfull_bar[slot]);
        }
        dbg_stamp(ep.dbg, 7);  // every MMA issued
      } else {
        for (int kb = kb0, it = 0; kb < kb1; ++kb, ++it) {
          const int s = it % STAGES;
          mbar_wait(&full_bar[s], (it / STAGES) & 1);
          asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
          const uint32_t a_base = smem_u32(smem + s * STAGE_BYTES);
          const uint32_t b_base = a_base + B_OFF;
#pragma unroll
          for (int k = 0; k < BK / 16; ++k)
            mma_f16(tmem, sw128_desc(a_base + k * 32), sw128_desc(b_base + k * 32), idesc,
                     (it | k) != 0);
          mma_commit(&empty_bar[s]);
        }
        mma_commit(&tfull_bar);
      }
    }
  } else if (X3 && warp >= 6) {  // ---- converter: fp32 stage -> tf32 hi + lo ----
    const int t = threadIdx.x - 192;
    for (int kb = kb0, it = 0; kb < kb1; ++kb, ++it) {
      const int s = it % STAGES;
      mbar_wait(&full_bar[s], (it / STAGES) & 1);
      uint8_t* sa = smem + s * STAGE_BYTES;
      split_tf32_smem(sa, sa + A_BYTES, A_BYTES / 16, t, kConvThreads);
      if (!ep.b_presplit)
        split_tf32_smem(sa + B_OFF, sa + B_OFF + B_BYTES, B_BYTES / 16, t, kConvThreads);
      asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
      __syncwarp();
      if (lane == 0) mbar_arrive(&conv_bar[s]);
    }
  } else {  // ---- epilogue warps: TMEM partial -> own smem [128][PLD] ----
    pdl_wait();
    const int q = warp & 3;
    // OP_X3: the K slice's chunks summed in registers (RN adds, fixed order)
    float racc[XS ? BN : 1];
    if constexpr (XS) {
#pragma unroll
      for (int i = 0; i < BN; ++i) racc[i] = 0.0f;
      int gc = 0;
      const int CH = (XH && ep.chunk_kb > 0) ? ep.chunk_kb : xchunk<OP>();
      for (int c0 = kb0; c0 < kb1; c0 += CH, ++gc) {
        const int slot = gc & 1;
        mbar_wait(&xfull_bar[slot], (gc >> 1) & 1);
        asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
        x3_add_chunk<XS ? BN : 1, OP>(racc, tmem + slot * 2 * BN + ((uint32_t)(q * 32) << 16),
                                  c0 == kb0);
        asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
        __syncwarp();
        if (lane == 0) mbar_arrive(&xempty_bar[slot]);
      }
    } else {
      mbar_wait(&tfull_bar, 0);
      asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
    }
    if (threadIdx.x == 64) dbg_stamp(ep.dbg, 4);  // the slice's chunks summed
    auto acc_chunk = [&](float (&v)[32], const int cc) {
      if constexpr (XS) {
#pragma unroll
        for (int i = 0; i < 32; ++i) v[i] = racc[(cc + i) % (XS ? BN : 1)];
      } else {
        tmem_ld32(tmem + ((uint32_t)(q * 32) << 16) + cc, v);
      }
    };
    float* prow = part + (q * 32 + lane) * PLD;
    if constexpr (SLAB) {
      if (ep.tstore) {
        // slab tile straight from TMEM through TMA tensor stores: per warp and
        // 32-column chunk one swizzled 32 x 128 B box in the (idle) ring, rows
        // rank * M + m0 + q * 32 of the [S * M, N] slab map
#pragma unroll
        for (int cc = 0; cc < BN; cc += 32) {
          float v[32];
          acc_chunk(v, cc);
          uint8_t* box = smem + q * (BN / 32) * 4096 + (cc / 32) * 4096;
#pragma unroll
          for (int j = 0; j < 8; ++j)
            *reinterpret_cast<float4*>(box + lane * 128 + ((j ^ (lane & 7)) << 4)) =
                make_float4(v[4 * j], v[4 * j + 1], v[4 * j + 2], v[4 * j + 3]);
          asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
          __syncwarp();
          if (lane == 0 && m0 + q * 32 < M)  // M % 32 == 0: whole boxes inside the slab
            tma_store_2d(&tma_c, box, n0 + cc, rank * M + m0 + q * 32);
        }
        if (lane == 0) tma_store_drain();
        __syncwarp();
      }
    }
#pragma unroll
    for (int cc = 0; cc < BN; cc += 32) {
      if (SLAB && ep.tstore) break;
      float v[32];
      acc_chunk(v, cc);
#pragma unroll
      for (int j = 0; j < 32; j += 4)
        *reinterpret_cast<float4*>(prow + cc + j) = make_float4(v[j], v[j + 1], v[j + 2], v[j + 3]);
    }
    if (SLAB && !ep.tstore) {  // my 32 rows, one row (BN * 4 contiguous bytes) per warp pass
      __syncwarp();
      float* slab = reinterpret_cast<float*>(ep.c) + (int64_t)rank * M * ep.ldc;
#pragma unroll 4
      for (int r = 0; r < 32; ++r) {
        const int lr = q * 32 + r, row = m0 + lr;
        if (row >= M) break;
#pragma unroll
        for (int c4 = lane; c4 < BN / 4; c4 += 32) {
          const int col = n0 + c4 * 4;
          if (col < N)
            *reinterpret_cast<float4*>(slab + (int64_t)row * ep.ldc + col) =
                *reinterpret_cast<const float4*>(part + lr * PLD + c4 * 4);
        }
      }
    }
  }
  if (threadIdx.x == 64) dbg_stamp(ep.dbg, 5);  // epilogue stores issued
  if constexpr (SLAB) {
    asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
    __syncthreads();
    if (threadIdx.x == 0) dbg_stamp(ep.dbg, 6);
    if (warp == 1) {
      asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
      asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem),
                   "r"(TMEM_COLS));
    }
    return;
  }
  __syncwarp();
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  cluster_sync_all();  // every partial tile of the cluster is in shared memory

  if (warp >= 2 && warp < 6) {  // ---- reduce my row slice over the S partials, fused epilogue ----
    const int t = threadIdx.x - 64;  // 0..127
    const int rows_per = (BM + S - 1) / S;          // S need not divide 128
    const int r_lo = rank * rows_per;
    const int rows = max(0, min(BM, r_lo + rows_per) - r_lo);
    constexpr int C4 = BN / 4;
    float* c32 = reinterpret_cast<float*>(ep.c);
    h16* c16 = reinterpret_cast<fq::h16*>(ep.c);
    const uint32_t part_s = smem_u32(part);
    // Two output float4 per thread per pass; every remote partial and the
    // residual / bias vectors of both are requested before the first use, so
    // a pass costs one DSMEM + one global round trip, not one per element.
    const bool vec_io = (ep.ldc % 4) == 0 && (!ep.res || (ep.ldr % 4) == 0) &&
                        !ep.accumulate && (N % 4) == 0;
    constexpr int U = 2;
    for (int idx0 = t; idx0 < rows * C4; idx0 += U * 128) {
      float4 pv[U][8];
      float4 rv[U], bv[U];
#pragma unroll
      for (int u = 0; u < U; ++u) {
        const int idx = idx0 + u * 128;
        rv[u] = make_float4(0.f, 0.f, 0.f, 0.f);
        bv[u] = rv[u];
        if (idx >= rows * C4) continue;
        const int lr = r_lo + idx / C4, c = (idx % C4) * 4;
        const uint32_t off = part_s + (uint32_t)(lr * PLD + c) * 4u;
#pragma unroll
        for (int p = 0; p < 8; ++p)
          if (p < S) pv[u][p] = ld_dsmem_f4(off, p);
        const int row = m0 + lr, col = n0 + c;
        if (vec_io && row < M && col < N) {
          if (ep.res) rv[u] = __ldg(reinterpret_cast<const float4*>(ep.res + (int64_t)row * ep.ldr + col));
          if (ep.bias) bv[u] = __ldg(reinterpret_cast<const float4*>(ep.bias + col));
        }
      }
#pragma unroll
      for (int u = 0; u < U; ++u) {
        const int idx = idx0 + u * 128;
        if (idx >= rows * C4) continue;
        const int lr = r_lo + idx / C4, c = (idx % C4) * 4;
        const int row = m0 + lr, col = n0 + c;
        float4 a = pv[u][0];
#pragma unroll
        for (int p = 1; p < 8; ++p)
          if (p < S) { a.x += pv[u][p].x; a.y += pv[u][p].y; a.z += pv[u][p].z; a.w += pv[u][p].w; }
        if (row >= M) continue;
        float x[4] = {a.x, a.y, a.z, a.w};
        const int64_t ci = (int64_t)row * ep.ldc + col;
        if (vec_io) {
          const float bb[4] = {bv[u].x, bv[u].y, bv[u].z, bv[u].w};
          const float rr[4] = {rv[u].x, rv[u].y, rv[u].z, rv[u].w};
#pragma unroll
          for (int j = 0; j < 4; ++j) {
            float y = x[j];
            if (ep.bias) y = fadd_rn(y, bb[j]);
            y = apply_act(y, ep.act);
            if (ep.res) y = fadd_rn(y, rr[j]);
            x[j] = y;
          }
        } else {
#pragma unroll
          for (int j = 0; j < 4; ++j) {
            if (col + j >= N) break;
            float y = x[j];
            if (ep.accumulate) y = fadd_rn(ep.c_f16 ? h2f(c16[ci + j]) : c32[ci + j], y);
            if (ep.bias) y = fadd_rn(y, __ldg(ep.bias + col + j));
            y = apply_act(y, ep.act);
            if (ep.res) y = fadd_rn(y, __ldg(ep.res + (int64_t)row * ep.ldr + col + j));
            x[j] = y;
          }
        }
        if constexpr (LNF) {  // keep the pre-LN row slice (my own rows of my partial)
          *reinterpret_cast<float4*>(part + lr * PLD + c) = make_float4(x[0], x[1], x[2], x[3]);
        } else if (ep.c_lo) {  // exact-mode pair output
          h16* c16lo = reinterpret_cast<fq::h16*>(ep.c_lo);
          for (int j = 0; j < 4 && col + j < N; ++j) split_xh(x[j], c16[ci + j], c16lo[ci + j]);
        } else if (col + 3 < N && ((ci & 3) == 0)) {
          if (ep.c_f16) {
            h16x2 lo = __floats2half2_rn(x[0], x[1]), hi = __floats2half2_rn(x[2], x[3]);
            uint2 pk;
            pk.x = *reinterpret_cast<uint32_t*>(&lo);
            pk.y = *reinterpret_cast<uint32_t*>(&hi);
            *reinterpret_cast<uint2*>(c16 + ci) = pk;
          } else {
            *reinterpret_cast<float4*>(c32 + ci) = make_float4(x[0], x[1], x[2], x[3]);
          }
        } else {
          for (int j = 0; j < 4 && col + j < N; ++j) {
            if (ep.c_f16) c16[ci + j] = f2h(x[j]);
            else c32[ci + j] = x[j];
          }
        }
      }
    }
  }
  if constexpr (LNF) {
    if (warp >= 2) {  // ---- LayerNorm of my 32 x BN slice (thread = row quarter) ----
      const int t = threadIdx.x - 64;
      const int rows_per = (BM + S - 1) / S;
      const int r_lo = rank * rows_per;
      const int rows = max(0, min(BM, r_lo + rows_per) - r_lo);
      asm volatile("bar.sync 1, 128;" ::: "memory");  // the slice is complete in smem
      constexpr int QW = BN / 4;                      // columns per thread
      const int lrl = t >> 2, qd = t & 3;
      const int lr = r_lo + lrl, row = m0 + lr;
      const bool rv = lrl < rows && row < M;
      const float* prow = part + lr * PLD + qd * QW;
      double sm = 0.0;
      if (rv)
        for (int j = 0; j < QW; ++j) sm += (double)prow[j];
      sm += __shfl_xor_sync(0xffffffffu, sm, 1);
      sm += __shfl_xor_sync(0xffffffffu, sm, 2);
      const double tmean = sm / BN;
      double m2 = 0.0;
      if (rv)
        for (int j = 0; j < QW; ++j) {
          const double dd = (double)prow[j] - tmean;
          m2 += dd * dd;
        }
      m2 += __shfl_xor_sync(0xffffffffu, m2, 1);
      m2 += __shfl_xor_sync(0xffffffffu, m2, 2);
      const int tn = n0 / BN, mtile = m0 / BM;
      if (rv && qd == 0) {
        __stcg(reinterpret_cast<double2*>(ln.stats + (int64_t)row * ln.nt + tn), make_double2(sm, m2));
        __threadfence();
      }
      asm volatile("bar.sync 1, 128;" ::: "memory");
      const int target = ln.nt * S;  // every CTA of the row block
      if (t == 0) {
        __threadfence();
        atomicAdd(ln.ctr + 2 * mtile, 1);
        int seen;
        do {
          asm volatile("ld.acquire.gpu.global.b32 %0, [%1];" : "=r"(seen) : "l"(ln.ctr + 2 * mtile) : "memory");
          if (seen < target) __nanosleep(64);
        } while (seen < target);
      }
      asm volatile("bar.sync 1, 128;" ::: "memory");
      if (rv) {
        double tot = 0.0;
        for (int tt = 0; tt < ln.nt; ++tt) tot += __ldcg(ln.stats + (int64_t)row * ln.nt + tt).x;
        const double mean = tot / N;
        double M2 = 0.0;
        for (int tt = 0; tt < ln.nt; ++tt) {
          const double2 st = __ldcg(ln.stats + (int64_t)row * ln.nt + tt);
          const double dm = st.x / BN - mean;
          M2 += st.y + (double)BN * dm * dm;
        }
        const double inv = 1.0 / sqrt(M2 / N + ln.eps);
        const int c0 = n0 + qd * QW;
        for (int j = 0; j < QW; j += 4) {
          const float4 g = __ldg(reinterpret_cast<const float4*>(ln.gamma + c0 + j));
          const float4 bb = __ldg(reinterpret_cast<const float4*>(ln.beta + c0 + j));
          float4 o;  // kernels.py:35: fp32((x - mean) * inv) * gamma + beta, two roundings
          o.x = fadd_rn(fmul_rn((float)(((double)prow[j] - mean) * inv), g.x), bb.x);
          o.y = fadd_rn(fmul_rn((float)(((double)prow[j + 1] - mean) * inv), g.y), bb.y);
          o.z = fadd_rn(fmul_rn((float)(((double)prow[j + 2] - mean) * inv), g.z), bb.z);
          o.w = fadd_rn(fmul_rn((float)(((double)prow[j + 3] - mean) * inv), g.w), bb.w);
          if (ln.out) *reinterpret_cast<float4*>(ln.out + (int64_t)row * ln.ldo + c0 + j) = o;
          if (ln.out16) {
            h16x2 lo = __floats2half2_rn(o.x, o.y), hi = __floats2half2_rn(o.z, o.w);
            uint2 pk;
            pk.x = *reinterpret_cast<uint32_t*>(&lo);
            pk.y = *reinterpret_cast<uint32_t*>(&hi);
            *reinterpret_cast<uint2*>(ln.out16 + (int64_t)row * ln.ldo16 + c0 + j) = pk;
          }
        }
      }
      asm volatile("bar.sync 1, 128;" ::: "memory");
      if (t == 0) {  // the last CTA to finish reading resets the row block's counters
        __threadfence();
        if (atomicAdd(ln.ctr + 2 * mtile + 1, 1) == target - 1) {
          ln.ctr[2 * mtile] = 0;
          ln.ctr[2 * mtile + 1] = 0;
        }
      }
    }
  }
  __syncwarp();
  cluster_sync_all();  // peers finished reading my partial
  if (threadIdx.x == 0) dbg_stamp(ep.dbg, 6);
  if (warp == 1) {
    asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
    asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem),
                 "r"(TMEM_COLS));
  }
}

// ---------------------------------------------------------------------------
// Exact-mode (3xFP16) GEMM on CTA pairs (tcgen05 cta_group::2). A 2-CTA
// cluster computes a 256 x BN tile: CTA r holds the A rows [128 r, +128) and
// the B rows [r BN/2, +BN/2) of every K block (hi + lo pairs), so each SM
// ingests 2 x (16 KB + BN/2 x 128 B) per 64-K block instead of 2 x (16 KB +
// BN x 128 B) — the decode GEMMs (M = 512) are bound by that per-SM TMA
// ingest. The leader CTA's single thread issues cta_group::2 MMAs (M = 256)
// that read both CTAs' shared memory and accumulate each CTA's 128 rows in its
// own TMEM; commits multicast to both CTAs' barriers; both CTAs' TMA loads
// complete on the leader's full barrier. The epilogue is per CTA (its 128
// rows), with the same TMEM chunking as the 1-CTA kernel: identical numerics.
// Epilogue: bias, activation, then an fp32 C or the exact mode's fp16 pair
// (c_lo) through TMA stores (no residual / accumulate on this path).
// ---------------------------------------------------------------------------
// Exact-mode HARS stage-1 statistics of one row's BN-column tile, from the
// thread's fp32 accumulator (thread = row r). gms: 32 floats of per-thread
// scratch (group counts other than 8).
template <int BN>
__device__ __forceinline__ void hars_tile_stats(const float (&v)[BN], const HarsEpi& he, int r,
                                                int M, int n0, float* gms) {
  const int k = r < M ? he.dk[r] : 0;
  if (k <= 0) return;
  // running lower bound of the row's R from the maxima other tiles published
  float rest = -INFINITY;
  if (k == 8) {
    const int4 a0 = __ldcg(reinterpret_cast<const int4*>(he.gmax + (int64_t)r * 32));
    const int4 a1 = __ldcg(reinterpret_cast<const int4*>(he.gmax + (int64_t)r * 32 + 4));
    rest = fminf(fminf(fminf(hs_ord2f(a0.x), hs_ord2f(a0.y)), fminf(hs_ord2f(a0.z), hs_ord2f(a0.w))),
                 fminf(fminf(hs_ord2f(a1.x), hs_ord2f(a1.y)), fminf(hs_ord2f(a1.z), hs_ord2f(a1.w))));
  } else {
    float mn = INFINITY;
    for (int g = 0; g < k; ++g) mn = fminf(mn, hs_ord2f(__ldcg(he.gmax + (int64_t)r * 32 + g)));
    rest = mn;
  }
  // pass 1: group maxima (column c in group c % k; n0 % 8 == 0 so for k = 8
  // column j of the tile is in group j & 7) and the tile maximum
  float g8[8] = {-INFINITY, -INFINITY, -INFINITY, -INFINITY,
                 -INFINITY, -INFINITY, -INFINITY, -INFINITY};
  float mt = -INFINITY, bound = INFINITY;
  if (k == 8) {
#pragma unroll
    for (int j = 0; j < BN; ++j) g8[j & 7] = fmaxf(g8[j & 7], v[j]);
#pragma unroll
    for (int g = 0; g < 8; ++g) {
      mt = fmaxf(mt, g8[g]);
      bound = fminf(bound, g8[g]);
      atomicMax(he.gmax + (int64_t)r * 32 + g, hs_f2ord(g8[g]));
    }
  } else {
    for (int g = 0; g < k; ++g) gms[g] = -INFINITY;
    int gi = n0 % k;
#pragma unroll
    for (int j = 0; j < BN; ++j) {
      gms[gi] = fmaxf(gms[gi], v[j]);
      if (++gi == k) gi = 0;
    }
    for (int g = 0; g < k; ++g) {
      mt = fmaxf(mt, gms[g]);
      bound = fminf(bound, gms[g]);
      atomicMax(he.gmax + (int64_t)r * 32 + g, hs_f2ord(gms[g]));
    }
  }
  bound = fmaxf(bound, rest);  // still <= the row's R: the candidate set is unchanged
  // pass 2: sum exp(x - mt) (each term 2^(x log2e - mt log2e) with log2e as hi +
  // lo fp32 parts, summed in f64) and the survivors x >= bound
  constexpr float L2E = 1.4426950408889634f;
  constexpr float L2E_LO = 1.925963033500011e-08f;
  const float mL = mt * L2E;
  double s = 0.0;
  const int tn = n0 / BN;
  int2* svr = he.sv + ((int64_t)r * he.ldt + tn) * he.sv_cap;
  int ns = 0;
#pragma unroll
  for (int j = 0; j < BN; ++j) {
    s += (double)hs_ex2(fmaf(v[j], L2E_LO, fmaf(v[j], L2E, -mL)));
    if (v[j] >= bound) {
      if (ns < he.sv_cap) svr[ns] = make_int2(n0 + j, __float_as_int(v[j]));
      ++ns;
    }
  }
  he.sv_cnt[(int64_t)r * he.ldt + tn] = ns;
  he.tmax[(int64_t)r * he.ldt + tn] = mt;
  he.tsum[(int64_t)r * he.ldt + tn] = s;
}

__device__ __forceinline__ void mma_f16_pair(uint32_t tmem_d, uint64_t adesc, uint64_t bdesc,
                                             uint32_t idesc, uint32_t accumulate) {
  asm volatile(
      "{\n\t"
      ".reg .pred p;\n\t"
      "setp.ne.b32 p, %4, 0;\n\t"
      "tcgen05.mma.cta_group::2.kind::f16 [%0], %1, %2, %3, p;\n}" ::"r"(tmem_d),
      "l"(adesc), "l"(bdesc), "r"(idesc), "r"(accumulate));
}

__device__ __forceinline__ void mma_xh_block_pair(uint32_t big, uint32_t small, uint32_t a_hi,
                                                  uint32_t a_lo, uint32_t b_hi, uint32_t b_lo,
                                                  uint32_t idesc, bool first) {
#pragma unroll
  for (int k = 0; k < 4; ++k) {
    const uint32_t acc = (first && k == 0) ? 0u : 1u;
    mma_f16_pair(small, sw128_desc(a_hi + k * 32), sw128_desc(b_lo + k * 32), idesc, acc);
    mma_f16_pair(small, sw128_desc(a_lo + k * 32), sw128_desc(b_hi + k * 32), idesc, 1u);
    mma_f16_pair(big, sw128_desc(a_hi + k * 32), sw128_desc(b_hi + k * 32), idesc, acc);
  }
}

__device__ __forceinline__ void commit_pair_mc(uint64_t* bar) {
  asm volatile(
      "tcgen05.commit.cta_group::2.mbarrier::arrive::one.shared::cluster.multicast::cluster.b64"
      " [%0], %1;" ::"r"(smem_u32(bar)),
      "h"((uint16_t)3)
      : "memory");
}

__device__ __forceinline__ uint32_t mapa_u32(uint32_t addr, uint32_t rank) {
  uint32_t r;
  asm volatile("mapa.shared::cluster.u32 %0, %1, %2;" : "=r"(r) : "r"(addr), "r"(rank));
  return r;
}

// TMA load into this CTA's shared memory whose completion is counted on the
// pair leader's mbarrier (bar: its shared::cluster address)
__device__ __forceinline__ void tma_load_2d_pair(const CUtensorMap* map, uint32_t bar, void* dst,
                                                 int c0, int c1) {
  asm volatile(
      "cp.async.bulk.tensor.2d.cta_group::2.shared::cluster.global.mbarrier::complete_tx::bytes"
      " [%0], [%1, {%2, %3}], [%4];" ::"r"(smem_u32(dst)),
      "l"(reinterpret_cast<uint64_t>(map)), "r"(c0), "r"(c1), "r"(bar)
      : "memory");
}

// Arrive on the pair leader's TMEM-slot barrier. Only the TMEM reads must be
// complete (tcgen05.wait::ld + tcgen05.fence::before_thread_sync order them);
// no smem / global data is handed over, so the default CTA-scope release
// suffices -- .release.cluster compiled to MEMBAR.ALL.GPU per chunk (ncu
// membar stalls, 14% of the pair GEMM's samples).
__device__ __forceinline__ void mbar_arrive_remote(uint32_t cluster_addr) {
  asm volatile("mbarrier.arrive.shared::cluster.b64 _, [%0];" ::"r"(cluster_addr) : "memory");
}

// HS: the exact mode's logits GEMM with the HARS stage-1 statistics epilogue
// (see HarsEpi): per row and 128-column tile the strided group maxima
// (published to the row's maxima with atomics), the tile maximum, the f64 sum
// of exp(x - tile max) and the survivors x >= a bound <= R, computed on the
// thread's fp32 row accumulator — the [rows, V] logits are never written.
template <int BN, int STAGES, bool HS = false>
__global__ void __launch_bounds__(kThreads, 1)
    xh_pair_gemm_kernel(const __grid_constant__ CUtensorMap tma_a,
                        const __grid_constant__ CUtensorMap tma_alo,
                        const __grid_constant__ CUtensorMap tma_b,
                        const __grid_constant__ CUtensorMap tma_blo,
                        const __grid_constant__ CUtensorMap tma_c,
                        const __grid_constant__ CUtensorMap tma_clo, const Epi ep, int M, int N,
                        int K, const HarsEpi he) {
  constexpr int KB = 64;
  constexpr int BH = BN / 2;  // B rows per CTA
  constexpr int A_BYTES = BM * 128;
  constexpr int B_BYTES = BH * 128;
  constexpr int STAGE_BYTES = 2 * (A_BYTES + B_BYTES);
  constexpr int B_OFF = 2 * A_BYTES;
  // 2 chunk slots x {hi.hi, small terms}; allocations are powers of two
  constexpr uint32_t TMEM_COLS = 4 * BN <= 128 ? 128 : (4 * BN <= 256 ? 256 : 512);
  static_assert(4 * BN <= 512, "TMEM holds 512 columns");
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = smem_raw + ((1024u - (smem_u32(smem_raw) & 1023u)) & 1023u);
  uint8_t* boxes = smem + STAGES * STAGE_BYTES;  // 4 epilogue warps x 4 KB
  __shared__ __align__(8) uint64_t full_bar[STAGES];
  __shared__ __align__(8) uint64_t empty_bar[STAGES];
  __shared__ __align__(8) uint64_t tfull_bar[2];
  __shared__ __align__(8) uint64_t tempty_bar[2];
  __shared__ __align__(8) uint64_t edone_bar;
  __shared__ uint32_t tmem_base_sh;

  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  pdl_launch_dependents();
  const uint32_t rank = cluster_rank();  // 0: the pair leader (issues the MMAs)
  const int num_kb = (K + KB - 1) / KB;
  const int mt = (M + 2 * BM - 1) / (2 * BM), nt = N / BN;
  const int ngroups = mt * nt;
  const int pid = blockIdx.x >> 1, npairs = gridDim.x >> 1;
  const int CH = ep.chunk_kb > 0 ? ep.chunk_kb : 4;

  if (warp == 0 && lane == 0) {
    for (int s = 0; s < STAGES; ++s) {
      mbar_init(&full_bar[s], 1);   // the leader's expect_tx arrive (+ both CTAs' bytes)
      mbar_init(&empty_bar[s], 1);  // the leader's multicast commit
    }
    for (int s = 0; s < 2; ++s) {
      mbar_init(&tfull_bar[s], 1);
      mbar_init(&tempty_bar[s], 8);  // both CTAs' 4 epilogue warps (leader's barrier)
    }
    mbar_init(&edone_bar, 4);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    asm volatile("prefetch.tensormap [%0];" ::"l"(reinterpret_cast<uint64_t>(&tma_a)));
    asm volatile("prefetch.tensormap [%0];" ::"l"(reinterpret_cast<uint64_t>(&tma_b)));
  }
  if (warp == 1) {  // both CTAs' warp 1 (same warp id): the pair's TMEM
    asm volatile("tcgen05.alloc.cta_group::2.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(
                     smem_u32(&tmem_base_sh)),
                 "r"(TMEM_COLS));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::2.sync.aligned;");
  }
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  cluster_sync_all();
  asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
  const uint32_t tmem = tmem_base_sh;
  const uint32_t full0 = mapa_u32(smem_u32(&full_bar[0]), 0);      // leader's, cluster space
  const uint32_t tempty0 = mapa_u32(smem_u32(&tempty_bar[0]), 0);

  if (warp == 0) {
    if (lane == 0) {  // ---- TMA producer (both CTAs) ----
      // the weights (B) do not depend on the previous kernel: the first
      // tile's first stages of B stream in before the grid-dependency wait
      int npre = 0;
      if (pid < ngroups) {
        const int n0 = (pid / mt) * BN + (int)rank * BH;
        npre = num_kb < STAGES ? num_kb : STAGES;
        for (int kb = 0; kb < npre; ++kb) {
          uint8_t* sa = smem + kb * STAGE_BYTES;
          if (rank == 0) mbar_expect_tx(&full_bar[kb], 2 * STAGE_BYTES);
          const uint32_t fb = full0 + 8u * (uint32_t)kb;
          tma_load_2d_pair(&tma_b, fb, sa + B_OFF, kb * KB, n0);
          tma_load_2d_pair(&tma_blo, fb, sa + B_OFF + B_BYTES, kb * KB, n0);
        }
      }
      pdl_wait();  // the activations are written by the previous kernel
      int it = 0;
      for (int g = pid; g < ngroups; g += npairs) {
        const int m0 = (g % mt) * 2 * BM + (int)rank * BM, n0 = (g / mt) * BN + (int)rank * BH;
        for (int kb = 0; kb < num_kb; ++kb, ++it) {
          const int s = it % STAGES;
          const uint32_t ph = (it / STAGES) & 1;
          uint8_t* sa = smem + s * STAGE_BYTES;
          if (it < npre) {  // B already in flight
            const uint32_t fb = full0 + 8u * (uint32_t)s;
            tma_load_2d_pair(&tma_a, fb, sa, kb * KB, m0);
            tma_load_2d_pair(&tma_alo, fb, sa + A_BYTES, kb * KB, m0);
            continue;
          }
          mbar_wait(&empty_bar[s], ph ^ 1);
          if (rank == 0) mbar_expect_tx(&full_bar[s], 2 * STAGE_BYTES);
          const uint32_t fb = full0 + 8u * (uint32_t)s;
          tma_load_2d_pair(&tma_a, fb, sa, kb * KB, m0);
          tma_load_2d_pair(&tma_alo, fb, sa + A_BYTES, kb * KB, m0);
          tma_load_2d_pair(&tma_b, fb, sa + B_OFF, kb * KB, n0);
          tma_load_2d_pair(&tma_blo, fb, sa + B_OFF + B_BYTES, kb * KB, n0);
        }
      }
      for (int j = 0; j < STAGES; ++j, ++it)
        mbar_wait(&empty_bar[it % STAGES], ((it / STAGES) & 1) ^ 1);
    }
  } else if (warp == 1) {
    if (lane == 0 && rank == 0) {  // ---- MMA issuer (the leader) ----
      constexpr uint32_t idesc = idesc_f16(2 * BM, BN);
      int it = 0, gc = 0;
      for (int g = pid; g < ngroups; g += npairs) {
        for (int kb0 = 0; kb0 < num_kb; kb0 += CH, ++gc) {
          const int slot = gc & 1;
          mbar_wait(&tempty_bar[slot], ((gc >> 1) & 1) ^ 1);
          asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
          const uint32_t big = tmem + slot * 2 * BN;
          const int kb1 = min(num_kb, kb0 + CH);
          for (int kb = kb0; kb < kb1; ++kb, ++it) {
            const int s = it % STAGES;
            mbar_wait(&full_bar[s], (it / STAGES) & 1);
            asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
            const uint32_t a_base = smem_u32(smem + s * STAGE_BYTES);
            const uint32_t b_base = a_base + B_OFF;
            mma_xh_block_pair(big, big + BN, a_base, a_base + A_BYTES, b_base, b_base + B_BYTES,
                              idesc, kb == kb0);
            commit_pair_mc(&empty_bar[s]);
          }
          commit_pair_mc(&tfull_bar[slot]);
        }
      }
    }
  } else {  // ---- epilogue: warps 2..5, this CTA's 128 rows ----
    const int q = warp & 3;
    uint8_t* box = boxes + (warp - 2) * 4096;
    // the tile's bias (a constant) staged in shared memory while the MMAs run:
    // the first tile's before the grid-dependency wait, so the epilogue's adds
    // do not wait on a global round trip
    __shared__ __align__(16) float s_bias[BN];
    const int et = threadIdx.x - 64;  // 0..127
    auto stage_bias = [&](int n0) {
      if (!ep.bias) return;
      asm volatile("bar.sync 1, 128;" ::: "memory");  // previous tile's reads done
      if (et < BN) s_bias[et] = __ldg(ep.bias + n0 + et);
      asm volatile("bar.sync 1, 128;" ::: "memory");
    };
    if (pid < ngroups) stage_bias((pid / mt) * BN);
    pdl_wait();
    int gc = 0;
    for (int g = pid; g < ngroups; g += npairs) {
      const int m0 = (g % mt) * 2 * BM + (int)rank * BM, n0 = (g / mt) * BN;
      const int rbase = m0 + q * 32;
      if (g != pid) stage_bias(n0);
      float racc[BN];
      for (int kb0 = 0; kb0 < num_kb; kb0 += CH, ++gc) {
        const int slot = gc & 1;
        mbar_wait(&tfull_bar[slot], (gc >> 1) & 1);
        asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
        x3_add_chunk<BN, OP_X3H>(racc, tmem + slot * 2 * BN + ((uint32_t)(q * 32) << 16),
                                 kb0 == 0);
        asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
        __syncwarp();
        if (lane == 0) mbar_arrive_remote(tempty0 + 8u * (uint32_t)slot);
      }
      if (rbase >= M) continue;  // this warp's rows are beyond the matrix
      if constexpr (HS) {
        hars_tile_stats<BN>(racc, he, rbase + lane, M, n0,
                            reinterpret_cast<float*>(boxes) + ((warp - 2) * 32 + lane) * 32);
        continue;
      }
#pragma unroll
      for (int j = 0; j < BN / 32; ++j) {
        float v[32];
#pragma unroll
        for (int i = 0; i < 32; ++i) v[i] = racc[j * 32 + i];
        const int col0 = n0 + j * 32;
        if (ep.bias) {
#pragma unroll
          for (int i = 0; i < 8; ++i) {
            const float4 b = *reinterpret_cast<const float4*>(s_bias + j * 32 + 4 * i);
            v[4 * i] = fadd_rn(v[4 * i], b.x);
            v[4 * i + 1] = fadd_rn(v[4 * i + 1], b.y);
            v[4 * i + 2] = fadd_rn(v[4 * i + 2], b.z);
            v[4 * i + 3] = fadd_rn(v[4 * i + 3], b.w);
          }
        }
        if (ep.act) {
#pragma unroll
          for (int i = 0; i < 32; ++i) v[i] = apply_act(v[i], ep.act);
        }
        if (lane == 0) asm volatile("cp.async.bulk.wait_group.read %0;" ::"n"(0) : "memory");
        __syncwarp();
        if (ep.c_lo) {  // the exact mode's fp16 pair: hi box + lo box (32 rows x 64 B each)
#pragma unroll
          for (int i = 0; i < 4; ++i) {
            uint4 ph, pl;
            split_xh2(v[8 * i], v[8 * i + 1], ph.x, pl.x);
            split_xh2(v[8 * i + 2], v[8 * i + 3], ph.y, pl.y);
            split_xh2(v[8 * i + 4], v[8 * i + 5], ph.z, pl.z);
            split_xh2(v[8 * i + 6], v[8 * i + 7], ph.w, pl.w);
            const int off = lane * 64 + ((i ^ ((lane >> 1) & 3)) << 4);
            *reinterpret_cast<uint4*>(box + off) = ph;
            *reinterpret_cast<uint4*>(box + 2048 + off) = pl;
          }
          asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
          __syncwarp();
          if (lane == 0) {
            tma_store_2d(&tma_c, box, col0, rbase);
            tma_store_2d(&tma_clo, box + 2048, col0, rbase);
          }
        } else {  // fp32: 32 rows x 128 B, 128-byte swizzle
#pragma unroll
          for (int i = 0; i < 8; ++i)
            *reinterpret_cast<float4*>(box + lane * 128 + ((i ^ (lane & 7)) << 4)) =
                make_float4(v[4 * i], v[4 * i + 1], v[4 * i + 2], v[4 * i + 3]);
          asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
          __syncwarp();
          if (lane == 0) tma_store_2d(&tma_c, box, col0, rbase);
        }
      }
    }
    if (lane == 0) tma_store_drain();
  }
  __syncwarp();
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  if (warp >= 2 && lane == 0) mbar_arrive(&edone_bar);
  cluster_sync_all();  // no CTA leaves while its peer may still signal or read it
  if (warp == 1) {
    mbar_wait(&edone_bar, 0);
    asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
    asm volatile("tcgen05.dealloc.cta_group::2.sync.aligned.b32 %0, %1;" ::"r"(tmem),
                 "r"(TMEM_COLS));
  }
}

template <int BN, int STAGES>
constexpr int smem_bytes_pair() {
  return STAGES * 2 * (BM * 128 + (BN / 2) * 128) + 4 * 4096 + 1024;
}

template <int BN, int OP>
constexpr int stage_bytes() {
  return (split3<OP>() ? 2 : 1) * (BM * 128 + BN * 128);
}

template <int BN, int STAGES, int OP = OP_F16>
constexpr int smem_bytes_splitk() {
  return STAGES * stage_bytes<BN, OP>() + 1024;
}

template <int BN, int STAGES, bool HS = false, int OP = OP_F16>
constexpr int smem_bytes() {
  return STAGES * stage_bytes<BN, OP>() + (HS ? 8 : 4) * 32 * 33 * 4 + 1024;
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

// 2D map over a row-major [rows, cols] matrix with leading dim ld, box
// [box_rows, one 128-byte row] (64 fp16 / 32 fp32) with 128-byte swizzle;
// out-of-bounds elements read as zero.
static int make_map(CUtensorMap* map, const void* ptr, int64_t rows, int64_t cols, int64_t ld,
                    int box_rows, bool f32 = false) {
  EncodeFn enc = get_encode();
  if (!enc) {
    set_error("cuTensorMapEncodeTiled unavailable");
    return FQ_ERR_CUDA;
  }
  const int es = f32 ? 4 : 2;
  cuuint64_t dims[2] = {(cuuint64_t)cols, (cuuint64_t)rows};
  cuuint64_t strides[1] = {(cuuint64_t)(ld * es)};
  cuuint32_t box[2] = {(cuuint32_t)(128 / es), (cuuint32_t)box_rows};
  cuuint32_t estr[2] = {1, 1};
  CUresult r = enc(map, f32 ? CU_TENSOR_MAP_DATA_TYPE_FLOAT32 : CU_TENSOR_MAP_DATA_TYPE_FLOAT16,
                   2, const_cast<void*>(ptr), dims, strides,
                   box, estr, CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B,
                   CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  if (r != CUDA_SUCCESS) {
    set_error("cuTensorMapEncodeTiled failed (%d): rows=%lld cols=%lld ld=%lld", (int)r,
              (long long)rows, (long long)cols, (long long)ld);
    return FQ_ERR_CUDA;
  }
  return FQ_OK;
}

// Output map for the TMA-store epilogue: [rows, cols] row-major (ld elements),
// box 32 rows x 32 elements (fp32: 128 B rows, 128-byte swizzle; fp16: 64 B
// rows, 64-byte swizzle) — the layout the epilogue writes its boxes in.
static int make_map_c(CUtensorMap* map, void* ptr, int64_t rows, int64_t cols, int64_t ld,
                      bool fp16) {
  EncodeFn enc = get_encode();
  if (!enc) return FQ_ERR_CUDA;
  const int es = fp16 ? 2 : 4;
  cuuint64_t dims[2] = {(cuuint64_t)cols, (cuuint64_t)rows};
  cuuint64_t strides[1] = {(cuuint64_t)(ld * es)};
  cuuint32_t box[2] = {32u, 32u};
  cuuint32_t estr[2] = {1, 1};
  CUresult r = enc(map, fp16 ? CU_TENSOR_MAP_DATA_TYPE_FLOAT16 : CU_TENSOR_MAP_DATA_TYPE_FLOAT32,
                   2, ptr, dims, strides, box, estr, CU_TENSOR_MAP_INTERLEAVE_NONE,
                   fp16 ? CU_TENSOR_MAP_SWIZZLE_64B : CU_TENSOR_MAP_SWIZZLE_128B,
                   CU_TENSOR_MAP_L2_PROMOTION_NONE, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  return r == CUDA_SUCCESS ? FQ_OK : FQ_ERR_CUDA;
}

static bool tma_store_enabled() {
  static int on = -1;
  if (on < 0) {
    const char* e = getenv("FQ_TMA_STORE");
    on = (e && e[0] == '0') ? 0 : 1;
  }
  return on == 1;
}

}  // namespace tc

// 2D fp16 tensor map with 128-byte swizzle for other kernels (attention):
// [rows, cols] row-major with leading dimension ld elements, box
// [box_rows, box_cols] (box_cols * 2 == 128 bytes for the swizzle).
int make_tmap_f16_sw128(CUtensorMap* map, const void* ptr, int64_t rows, int64_t cols,
                         int64_t ld, int box_cols, int box_rows) {
  tc::EncodeFn enc = tc::get_encode();
  if (!enc) {
    set_error("cuTensorMapEncodeTiled unavailable");
    return FQ_ERR_CUDA;
  }
  cuuint64_t dims[2] = {(cuuint64_t)cols, (cuuint64_t)rows};
  cuuint64_t strides[1] = {(cuuint64_t)(ld * 2)};
  cuuint32_t box[2] = {(cuuint32_t)box_cols, (cuuint32_t)box_rows};
  cuuint32_t estr[2] = {1, 1};
  CUresult r = enc(map, CU_TENSOR_MAP_DATA_TYPE_FLOAT16, 2, const_cast<void*>(ptr), dims, strides,
                   box, estr, CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B,
                   CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  if (r != CUDA_SUCCESS) {
    set_error("cuTensorMapEncodeTiled failed (%d)", (int)r);
    return FQ_ERR_CUDA;
  }
  return FQ_OK;
}

namespace tc {

static int num_sms() {
  static int n = 0;
  if (!n) {
    int dev = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&n, cudaDevAttrMultiProcessorCount, dev);
  }
  return n;
}

template <int BN, int STAGES, bool HS = false, int OP = OP_F16>
static int launch(const void* a, int64_t lda, const void* b, int64_t ldb, const Epi& ep,
                  int64_t M, int64_t N, int64_t K, int cm, int cn, cudaStream_t s,
                  const HarsEpi& he = HarsEpi{}, const void* b_lo = nullptr,
                  const void* a_lo = nullptr) {
  constexpr bool X3 = OP == OP_X3, XH = OP == OP_X3H;
  CUtensorMap ma, mb, mc, mblo, malo;
  int rc;
  if ((rc = make_map(&ma, a, M, K, lda, BM / cn, X3)) != FQ_OK) return rc;
  if ((rc = make_map(&mb, b, N, K, ldb, BN / cm, X3)) != FQ_OK) return rc;
  Epi e2 = ep;
  e2.tstore = 0;
  e2.b_presplit = (X3 || XH) && b_lo != nullptr;
  mblo = mb;
  malo = ma;
  if (e2.b_presplit && (rc = make_map(&mblo, b_lo, N, K, ldb, BN / cm, X3)) != FQ_OK) return rc;
  if (XH && (rc = make_map(&malo, a_lo, M, K, lda, BM / cn, false)) != FQ_OK) return rc;
  mc = ma;
  CUtensorMap mclo = ma;
  if (!HS && ep.c && !ep.accumulate && !ep.res && N % 32 == 0 && tma_store_enabled() &&
      ((uintptr_t)ep.c & 15) == 0 && (ep.ldc * (ep.c_f16 ? 2 : 4)) % 16 == 0 &&
      (!ep.c_lo || ((uintptr_t)ep.c_lo & 15) == 0) &&
      make_map_c(&mc, ep.c, M, N, ep.ldc, ep.c_f16 != 0) == FQ_OK &&
      (!ep.c_lo || make_map_c(&mclo, ep.c_lo, M, N, ep.ldc, true) == FQ_OK))
    e2.tstore = 1;
  const int csize = cm * cn;
  const int64_t groups = ((M + BM - 1) / BM / cm) * ((N + BN - 1) / BN / cn);
  const int64_t max_clusters = num_sms() / csize;
  const int64_t clusters = groups < max_clusters ? groups : max_clusters;
  cudaError_t e = launch_kernel(tc_gemm_kernel<BN, STAGES, HS, OP>,
                                dim3((unsigned)(clusters * csize)), dim3(threads_of<OP>()),
                                smem_bytes<BN, STAGES, HS, OP>(), s, (unsigned)csize, ma, mb, e2,
                                (int)M, (int)N, (int)K, cm, cn, he, mc, mblo, malo, mclo);
  if (e != cudaSuccess) {
    set_error("fq_gemm(tcgen05): launch failed: %s", cudaGetErrorString(e));
    return FQ_ERR_CUDA;
  }
  return launch_status("fq_gemm(tcgen05)");
}

template <int BN, int STAGES, bool LNF = false, bool SLAB = false, int OP = OP_F16>
static int launch_splitk(const void* a, int64_t lda, const void* b, int64_t ldb, const Epi& ep,
                         int64_t M, int64_t N, int64_t K, int S, cudaStream_t s,
                         const LnEpi& ln = LnEpi{}, const void* b_lo = nullptr,
                         const void* a_lo = nullptr) {
  constexpr bool X3 = OP == OP_X3, XH = OP == OP_X3H;
  CUtensorMap ma, mb, mc, mblo, malo;
  int rc;
  if ((rc = make_map(&ma, a, M, K, lda, BM, X3)) != FQ_OK) return rc;
  if ((rc = make_map(&mb, b, N, K, ldb, BN, X3)) != FQ_OK) return rc;
  Epi e2 = ep;
  e2.tstore = 0;
  e2.b_presplit = (X3 || XH) && b_lo != nullptr;
  mblo = mb;
  malo = ma;
  if (e2.b_presplit && (rc = make_map(&mblo, b_lo, N, K, ldb, BN, X3)) != FQ_OK) return rc;
  if (XH && (rc = make_map(&malo, a_lo, M, K, lda, BM, false)) != FQ_OK) return rc;
  mc = ma;
  if (SLAB && M % 32 == 0 && N % 32 == 0 && tma_store_enabled() && ((uintptr_t)ep.c & 15) == 0 &&
      (ep.ldc * 4) % 16 == 0 && make_map_c(&mc, ep.c, S * M, N, ep.ldc, false) == FQ_OK)
    e2.tstore = 1;
  const int64_t tiles = ((M + BM - 1) / BM) * ((N + BN - 1) / BN);
  const int nkb = (int)((K + kblock<OP>() - 1) / kblock<OP>());
  const int kbs = (nkb + S - 1) / S;
  cudaError_t e = launch_kernel(tc_gemm_splitk_kernel<BN, STAGES, LNF, SLAB, OP>,
                                dim3((unsigned)(tiles * S)), dim3(threads_of<OP>()),
                                smem_bytes_splitk<BN, STAGES, OP>(), s, SLAB ? 1u : (unsigned)S, ma,
                                mb, e2, (int)M, (int)N, (int)K, kbs, ln, S, mc, mblo, malo);
  if (e != cudaSuccess) {
    set_error("fq_gemm(tcgen05 split-K): launch failed: %s", cudaGetErrorString(e));
    return FQ_ERR_CUDA;
  }
  return launch_status("fq_gemm(tcgen05 split-K)");
}

template <int BN, int STAGES, bool LNF = false, bool SLAB = false, int OP = OP_F16>
static int prep_splitk() {
  return cudaFuncSetAttribute(tc_gemm_splitk_kernel<BN, STAGES, LNF, SLAB, OP>,
                              cudaFuncAttributeMaxDynamicSharedMemorySize,
                              smem_bytes_splitk<BN, STAGES, OP>()) == cudaSuccess
             ? FQ_OK
             : FQ_ERR_CUDA;
}

// Exact-mode pair GEMM launch: a, a_lo [M, K] and b, b_lo [N, K] fp16 pairs;
// C fp32 [M, ldc] (c_lo == NULL) or the fp16 pair (c, c_lo). N % BN == 0.
template <int BN, int STAGES, bool HS = false>
static int launch_pair(const void* a, const void* a_lo, int64_t lda, const void* b,
                       const void* b_lo, int64_t ldb, const Epi& ep, int64_t M, int64_t N,
                       int64_t K, cudaStream_t s, const HarsEpi& he = HarsEpi{}) {
  CUtensorMap ma, malo, mb, mblo, mc, mclo;
  int rc;
  if ((rc = make_map(&ma, a, M, K, lda, BM, false)) != FQ_OK) return rc;
  if ((rc = make_map(&malo, a_lo, M, K, lda, BM, false)) != FQ_OK) return rc;
  if ((rc = make_map(&mb, b, N, K, ldb, BN / 2, false)) != FQ_OK) return rc;
  if ((rc = make_map(&mblo, b_lo, N, K, ldb, BN / 2, false)) != FQ_OK) return rc;
  mc = ma;
  if (!HS && make_map_c(&mc, ep.c, M, N, ep.ldc, ep.c_lo != nullptr) != FQ_OK) {
    set_error("fq_gemm_x3h (pair): output tensor map");
    return FQ_ERR_CUDA;
  }
  mclo = mc;
  if (!HS && ep.c_lo && make_map_c(&mclo, ep.c_lo, M, N, ep.ldc, true) != FQ_OK) {
    set_error("fq_gemm_x3h (pair): output tensor map");
    return FQ_ERR_CUDA;
  }
  const int64_t groups = ((M + 2 * BM - 1) / (2 * BM)) * (N / BN);
  const int64_t max_pairs = num_sms() / 2;
  const int64_t pairs = groups < max_pairs ? groups : max_pairs;
  cudaError_t e = launch_kernel(xh_pair_gemm_kernel<BN, STAGES, HS>, dim3((unsigned)(2 * pairs)),
                                dim3(kThreads), smem_bytes_pair<BN, STAGES>(), s, 2u, ma, malo,
                                mb, mblo, mc, mclo, ep, (int)M, (int)N, (int)K, he);
  if (e != cudaSuccess) {
    set_error("fq_gemm_x3h (pair): launch failed: %s", cudaGetErrorString(e));
    return FQ_ERR_CUDA;
  }
  return launch_status("fq_gemm_x3h (pair)");
}

template <int BN, int STAGES, bool HS = false>
static int prep_pair() {
  return cudaFuncSetAttribute(xh_pair_gemm_kernel<BN, STAGES, HS>,
                              cudaFuncAttributeMaxDynamicSharedMemorySize,
                              smem_bytes_pair<BN, STAGES>()) == cudaSuccess
             ? FQ_OK
             : FQ_ERR_CUDA;
}

template <int BN, int STAGES, bool HS = false, int OP = OP_F16>
static int prep() {
  return cudaFuncSetAttribute(tc_gemm_kernel<BN, STAGES, HS, OP>,
                              cudaFuncAttributeMaxDynamicSharedMemorySize,
                              smem_bytes<BN, STAGES, HS, OP>()) == cudaSuccess
             ? FQ_OK
             : FQ_ERR_CUDA;
}

}  // namespace tc

int gemm_tc_prepare() {
  if (tc::prep<256, 4>() || tc::prep<224, 4>() || tc::prep<192, 4>() || tc::prep<128, 6>() ||
      tc::prep<96, 7>() ||
      tc::prep<224, 4, true>() ||
      tc::prep<64, 8>() || tc::prep<32, 8>() ||
      tc::prep_splitk<256, 4>() || tc::prep_splitk<128, 6>() || tc::prep_splitk<64, 8>() ||
      tc::prep_splitk<128, 6, true>() || tc::prep_splitk<128, 6, false, true>() ||
      tc::prep<128, 3, false, tc::OP_X3>() || tc::prep<64, 4, false, tc::OP_X3>() ||
      tc::prep_splitk<128, 3, false, false, tc::OP_X3>() ||
      tc::prep_splitk<128, 3, false, true, tc::OP_X3>() ||
      tc::prep<128, 3, false, tc::OP_X3H>() || tc::prep<64, 4, false, tc::OP_X3H>() ||
      tc::prep_splitk<128, 3, false, false, tc::OP_X3H>() ||
      tc::prep_splitk<128, 3, false, true, tc::OP_X3H>() || tc::prep_pair<128, 4>() ||
      tc::prep_pair<96, 4>() ||
      tc::prep_pair<128, 4, true>()) {
    set_error("fq_prepare: tcgen05 GEMM smem opt-in failed");
    return FQ_ERR_CUDA;
  }
  return FQ_OK;
}

// Tile / split choice from the measured bottleneck: per-SM TMA ingest
// (~40 B/clk, ~80 GB/s per SM on this B200 pool, fq_gemm_tc phase traces): a
// CTA streams (128 + BN) * K_slice * 2 bytes per tile. Persistent tiles overlap
// the epilogue with the next tile; a split-K cluster additionally reduces
// 512 * BN bytes of fp32 partials through DSMEM per CTA. Multicast clusters
// (cm x cn) stay available through fq_gemm_force_plan but never won on the
// sweep (ingest, not L2, is the limit), so the model picks cm = cn = 1.
struct TcPlan {
  int bn, cm, cn, split;  // split > 1: split-K cluster kernel (cm = cn = 1)
};

static TcPlan g_forced{0, 0, 0, 1};
unsigned long long* g_gemm_dbg = nullptr;
extern "C" void fq_gemm_debug_timestamps(unsigned long long* p) { g_gemm_dbg = p; }

static TcPlan plan_tc(int64_t M, int64_t N, int64_t K) {
  const int64_t mt = (M + tc::BM - 1) / tc::BM;
  const int nkb = (int)((K + tc::BK - 1) / tc::BK);
  if (g_forced.bn) {
    const int64_t nt = (N + g_forced.bn - 1) / g_forced.bn;
    if (mt % g_forced.cm == 0 && nt % g_forced.cn == 0 &&
        (g_forced.split == 1 || (mt * nt * g_forced.split <= tc::num_sms() &&
                                 g_forced.split <= nkb && g_forced.cm * g_forced.cn == 1)))
      return g_forced;
  }
  // Measured table (scripts/gemm_graph_sweep.py, CUDA-graph back-to-back
  // launches on B200): small-M GEMMs are bound by the chip-wide L2->SM
  // operand traffic and per-launch overhead, large ones by per-SM ingest.
  const int64_t nt128 = (N + 127) / 128;
  if (mt <= 8) {
    if (N <= 1024 && nkb >= 16 && mt * nt128 * 4 <= tc::num_sms())
      return {128, 1, 1, 4};                       // K >= 1024: split-K over 4 CTAs
    if (N <= 1024) return {32, 1, 1, 1};
    // N = 3072 (QKV): 96-wide tiles put 128 CTAs (not 96) on the GPU, each
    // streaming 10% fewer operand bytes
    if (N % 96 == 0 && N % 128 == 0 && mt * (N / 96) <= tc::num_sms() &&
        mt * (N / 128) < tc::num_sms() * 3 / 4 && getenv("FQ_NO_BN96") == nullptr)
      return {96, 1, 1, 1};
    if (N < 8192) return {128, 1, 1, 1};
  }
  // Large GEMMs are tensor-bound: pick the tile width minimising the busiest
  // CTA's work, ceil(tiles / SMs) * BN (wave quantisation over 148 SMs).
  int best = 256;
  int64_t best_cost = -1;
  for (int bn : {256, 224, 192}) {
    const int64_t tiles = mt * ((N + bn - 1) / bn);
    const int64_t cost = (tiles + tc::num_sms() - 1) / tc::num_sms() * bn;
    if (best_cost < 0 || cost < best_cost) { best = bn; best_cost = cost; }
  }
  return {best, 1, 1, 1};
}

int launch_tc_gemm(const void* a, int64_t lda, const void* b, int64_t ldb, void* c, int c_f16,
                   int64_t ldc, int64_t M, int64_t N, int64_t K, int accumulate,
                   const float* bias, const float* res, int64_t ldr, int act, cudaStream_t s) {
  FQ_CHECK_ARG(lda % 8 == 0 && ldb % 8 == 0 && ((uintptr_t)a & 15) == 0 &&
                   ((uintptr_t)b & 15) == 0,
               FQ_ERR_DIMENSION, "tcgen05 GEMM: operands need 16-byte aligned rows (ld %% 8 == 0)");
  FQ_CHECK_ARG(M < (1LL << 31) && N < (1LL << 31) && K < (1LL << 31), FQ_ERR_DIMENSION,
               "tcgen05 GEMM: dimension too large");
  tc::Epi ep{c, ldc, c_f16, accumulate, bias, res, ldr, act, g_gemm_dbg};
  const TcPlan p = plan_tc(M, N, K);
  if (p.split > 1) {
    switch (p.bn) {
      case 256: return tc::launch_splitk<256, 4>(a, lda, b, ldb, ep, M, N, K, p.split, s);
      case 128: return tc::launch_splitk<128, 6>(a, lda, b, ldb, ep, M, N, K, p.split, s);
      default: return tc::launch_splitk<64, 8>(a, lda, b, ldb, ep, M, N, K, p.split, s);
    }
  }
  switch (p.bn) {
    case 256: return tc::launch<256, 4>(a, lda, b, ldb, ep, M, N, K, p.cm, p.cn, s);
    case 224: return tc::launch<224, 4>(a, lda, b, ldb, ep, M, N, K, p.cm, p.cn, s);
    case 192: return tc::launch<192, 4>(a, lda, b, ldb, ep, M, N, K, p.cm, p.cn, s);
    case 128: return tc::launch<128, 6>(a, lda, b, ldb, ep, M, N, K, p.cm, p.cn, s);
    case 96: return tc::launch<96, 7>(a, lda, b, ldb, ep, M, N, K, p.cm, p.cn, s);
    case 64: return tc::launch<64, 8>(a, lda, b, ldb, ep, M, N, K, p.cm, p.cn, s);
    default: return tc::launch<32, 8>(a, lda, b, ldb, ep, M, N, K, p.cm, p.cn, s);
  }
}

// ---------------------------------------------------------------------------
// Exact fp32 mode on the tensor cores (3xTF32, OP_X3). The plan is a function
// of (N, K) only — never of M — so every output element sees the same K
// reduction order whatever the batch (bitwise invariant to batch sharding):
// sequential K through one TMEM accumulator, or for N <= 1024 with K >= 1024
// four K slices summed in slice order (DSMEM cluster reduction, or slabs summed
// by the consumer).
struct X3Plan {
  int bn, split;
};

static X3Plan plan_x3(int64_t N, int64_t K) {
  const int64_t nkb = (K + 31) / 32;
  if (N <= 1024 && nkb >= 32) return {128, 4};
  if (N <= 512) return {64, 1};
  return {128, 1};
}

static int check_x3(const void* a, int64_t lda, const void* b, const void* b_lo, int64_t ldb,
                    int64_t M, int64_t N, int64_t K) {
  FQ_CHECK_ARG(lda % 4 == 0 && ldb % 4 == 0 && ((uintptr_t)a & 15) == 0 &&
                   ((uintptr_t)b & 15) == 0 && ((uintptr_t)b_lo & 15) == 0,
               FQ_ERR_DIMENSION, "3xTF32 GEMM: operands need 16-byte aligned rows (ld %% 4 == 0)");
  FQ_CHECK_ARG(M < (1LL << 31) && N < (1LL << 31) && K < (1LL << 31), FQ_ERR_DIMENSION,
               "3xTF32 GEMM: dimension too large");
  return FQ_OK;
}

int launch_x3_gemm(const float* a, int64_t lda, const float* b, const float* b_lo, int64_t ldb,
                   float* c, int64_t ldc, int64_t M, int64_t N, int64_t K, int accumulate,
                   const float* bias, const float* res, int64_t ldr, int act, cudaStream_t s) {
  int rc = check_x3(a, lda, b, b_lo, ldb, M, N, K);
  if (rc != FQ_OK) return rc;
  tc::Epi ep{c, ldc, 0, accumulate, bias, res, ldr, act, g_gemm_dbg};
  const X3Plan p = plan_x3(N, K);
  if (p.split > 1)
    return tc::launch_splitk<128, 3, false, false, tc::OP_X3>(a, lda, b, ldb, ep, M, N, K,
                                                              p.split, s, tc::LnEpi{}, b_lo);
  if (p.bn == 64)
    return tc::launch<64, 4, false, tc::OP_X3>(a, lda, b, ldb, ep, M, N, K, 1, 1, s,
                                               tc::HarsEpi{}, b_lo);
  return tc::launch<128, 3, false, tc::OP_X3>(a, lda, b, ldb, ep, M, N, K, 1, 1, s,
                                              tc::HarsEpi{}, b_lo);
}

// Exact-mode GEMM (see include/fq_abi.h): c = act(a . b^T (+c) (+bias)) (+res),
// a [M,K] fp32, b [N,K] fp32 K-major given either raw (b_lo = NULL: split in
// shared memory) or pre-split into tf32 hi (b) + lo (b_lo).
extern "C" int fq_gemm_f32x3(const float* a, int64_t lda, const float* b, const float* b_lo,
                             int64_t ldb, float* c, int64_t ldc, int64_t M, int64_t N, int64_t K,
                             int accumulate, const float* bias, const float* residual,
                             int64_t ldr, int act, fq_stream_t stream) {
  FQ_CHECK_ARG(a && b && c && M >= 0 && N >= 0 && K >= 1, FQ_ERR_DIMENSION,
               "fq_gemm_f32x3: bad shape M=%lld N=%lld K=%lld", (long long)M, (long long)N,
               (long long)K);
  FQ_CHECK_ARG(act >= 0 && act <= 2, FQ_ERR_PARAMETER, "fq_gemm_f32x3: unknown activation");
  if (M == 0 || N == 0) return FQ_OK;
  return launch_x3_gemm(a, lda, b, b_lo, ldb, c, ldc, M, N, K, accumulate, bias, residual, ldr,
                        act, as_stream(stream));
}

// Exact-mode GEMM + bias + residual + LayerNorm (the encoder's / decoder's
// closing pairs, model.py:339-358, :582-626): with the 4-slice plan the split
// K slices go to ws as slabs and fq_splitk_bias_residual_layer_norm sums them
// in slice order (the DSMEM reduction's additions, same bits); else the GEMM
// with its fused bias + residual, then fq_layer_norm.
extern "C" int fq_gemm_f32x3_ln(const float* a, int64_t lda, const float* b, const float* b_lo,
                                int64_t ldb, const float* bias, const float* res, int64_t ldr,
                                const float* gamma, const float* beta, double eps, float* out,
                                int64_t ldo, void* ws, int64_t ws_bytes, int64_t M, int64_t N,
                                int64_t K, fq_stream_t stream) {
  FQ_CHECK_ARG(a && b && bias && res && gamma && beta && out && M > 0 && N > 0 && K > 0,
               FQ_ERR_DIMENSION, "fq_gemm_f32x3_ln: bad args");
  int rc = check_x3(a, lda, b, b_lo, ldb, M, N, K);
  if (rc != FQ_OK) return rc;
  const X3Plan p = plan_x3(N, K);
  const int64_t slab_need = (int64_t)p.split * M * N * (int64_t)sizeof(float);
  if (p.split > 1 && ws && ws_bytes >= slab_need && ((uintptr_t)ws & 15) == 0 &&
      (N == 512 || N == 1024)) {
    tc::Epi ep{ws, N, 0, 0, nullptr, nullptr, 0, 0, g_gemm_dbg};
    rc = tc::launch_splitk<128, 3, false, true, tc::OP_X3>(a, lda, b, ldb, ep, M, N, K, p.split,
                                                           as_stream(stream), tc::LnEpi{}, b_lo);
    if (rc != FQ_OK) return rc;
    return fq_splitk_bias_residual_layer_norm(reinterpret_cast<const float*>(ws), p.split, N,
                                              bias, res, ldr, gamma, beta, eps, M, N, out, ldo,
                                              nullptr, 0, stream);
  }
  rc = launch_x3_gemm(a, lda, b, b_lo, ldb, out, ldo, M, N, K, 0, bias, res, ldr, 0,
                      as_stream(stream));
  if (rc != FQ_OK) return rc;
  return fq_layer_norm(out, ldo, gamma, beta, eps, M, N, out, ldo, nullptr, 0, stream);
}

// ---------------------------------------------------------------------------
// Exact fp32 mode, 3xFP16 (OP_X3H): operands as fp16 pairs (split_xh), same
// M-independent plan as 3xTF32 (K slices of 1024 for N <= 1024 and K >= 2048
// ... in units of 64-element K blocks), 128-element accumulation chunks.
static int check_xh(const void* a, const void* a_lo, int64_t lda, const void* b,
                    const void* b_lo, int64_t ldb, int64_t M, int64_t N, int64_t K) {
  FQ_CHECK_ARG(a && a_lo && b && b_lo, FQ_ERR_DIMENSION, "3xFP16 GEMM: null operand");
  FQ_CHECK_ARG(lda % 8 == 0 && ldb % 8 == 0 &&
                   (((uintptr_t)a | (uintptr_t)a_lo | (uintptr_t)b | (uintptr_t)b_lo) & 15) == 0,
               FQ_ERR_DIMENSION, "3xFP16 GEMM: operands need 16-byte aligned rows (ld %% 8 == 0)");
  FQ_CHECK_ARG(M < (1LL << 31) && N < (1LL << 31) && K < (1LL << 31), FQ_ERR_DIMENSION,
               "3xFP16 GEMM: dimension too large");
  return FQ_OK;
}

// The exact mode's numerics are fixed by (N, K) alone: K runs in chunks of
// 256 elements (4 K blocks) — or, for N <= 1024 and K >= 1024, in 4 slices of
// K/4 — each accumulated in TMEM and added to the fp32 result with RN adds in
// K order. The kernel is then a free, M-dependent choice with identical bits:
// the 4-slice shapes run split-K over 4 CTAs (DSMEM reduction, or slabs summed
// by the consumer) for M <= 1024 (the decode step) and the persistent kernel
// with slice-long chunks for larger M (the encoder).
struct XhPlan {
  int bn, split, chunk_kb;
};

static XhPlan plan_xh(int64_t M, int64_t N, int64_t K) {
  const int nkb = (int)((K + 63) / 64);
  static int dbg_chunk = -1;  // experiments only: FQ_XH_CHUNK=<K blocks> (changes numerics)
  if (dbg_chunk < 0) {
    const char* e = getenv("FQ_XH_CHUNK");
    dbg_chunk = e ? atoi(e) : 0;
  }
  if (dbg_chunk > 0) return XhPlan{128, 1, dbg_chunk};
  if (N <= 1024 && nkb >= 16) {
    const int slice = (nkb + 3) / 4;
    return M <= 1024 ? XhPlan{128, 4, slice} : XhPlan{128, 1, slice};
  }
  return XhPlan{N <= 512 ? 64 : 128, 1, 4};
}

// The CTA-pair kernel takes the unsplit shapes whose epilogue is bias / act
// into a TMA-stored C (the QKV, FFN1, logits, cross-K/V and encoder
// projections). It is chosen by (N, epilogue) only, never by M, so the bits
// stay M-independent. FQ_XH_PAIR=0 disables it (A/B).
static bool pair_ok(int64_t N, int accumulate, const float* res, const void* c, int64_t ldc,
                    bool half_out) {
  static int on = -1;
  if (on < 0) {
    const char* e = getenv("FQ_XH_PAIR");
    on = (e && e[0] == '0') ? 0 : 1;
  }
  return on && N % 128 == 0 && !accumulate && !res && ((uintptr_t)c & 15) == 0 &&
         (ldc * (half_out ? 2 : 4)) % 16 == 0;
}

// Pair tile width: 96 columns when 128 would leave over a quarter of the SMs
// idle and 96 fills one wave (the decode QKV projection: 96 -> 128 CTAs). The
// tile width never changes the bits (same K chunks per element).
static bool pair_bn96(int64_t M, int64_t N) {
  const int64_t mp = (M + 255) / 256, sms = tc::num_sms();
  return N % 96 == 0 && 2 * mp * (N / 128) < (3 * sms) / 4 && 2 * mp * (N / 96) <= sms;
}

int launch_xh_gemm(const void* a, const void* a_lo, int64_t lda, const void* b,
                   const void* b_lo, int64_t ldb, float* c, int64_t ldc, int64_t M, int64_t N,
                   int64_t K, int accumulate, const float* bias, const float* res, int64_t ldr,
                   int act, cudaStream_t s) {
  int rc = check_xh(a, a_lo, lda, b, b_lo, ldb, M, N, K);
  if (rc != FQ_OK) return rc;
  const XhPlan p = plan_xh(M, N, K);
  tc::Epi ep{c, ldc, 0, accumulate, bias, res, ldr, act, g_gemm_dbg};
  ep.chunk_kb = p.chunk_kb;
  if (p.split == 1 && pair_ok(N, accumulate, res, c, ldc, false))
    return pair_bn96(M, N) ? tc::launch_pair<96, 4>(a, a_lo, lda, b, b_lo, ldb, ep, M, N, K, s)
                           : tc::launch_pair<128, 4>(a, a_lo, lda, b, b_lo, ldb, ep, M, N, K, s);
  if (p.split > 1)
    return tc::launch_splitk<128, 3, false, false, tc::OP_X3H>(a, lda, b, ldb, ep, M, N, K,
                                                               p.split, s, tc::LnEpi{}, b_lo, a_lo);
  if (p.bn == 64)
    return tc::launch<64, 4, false, tc::OP_X3H>(a, lda, b, ldb, ep, M, N, K, 1, 1, s,
                                                tc::HarsEpi{}, b_lo, a_lo);
  return tc::launch<128, 3, false, tc::OP_X3H>(a, lda, b, ldb, ep, M, N, K, 1, 1, s,
                                               tc::HarsEpi{}, b_lo, a_lo);
}

extern "C" int fq_gemm_x3h(const void* a, const void* a_lo, int64_t lda, const void* b,
                           const void* b_lo, int64_t ldb, float* c, int64_t ldc, int64_t M,
                           int64_t N, int64_t K, int accumulate, const float* bias,
                           const float* residual, int64_t ldr, int act, fq_stream_t stream) {
  FQ_CHECK_ARG(c && M >= 0 && N >= 0 && K >= 1, FQ_ERR_DIMENSION,
               "fq_gemm_x3h: bad shape M=%lld N=%lld K=%lld", (long long)M, (long long)N,
               (long long)K);
  FQ_CHECK_ARG(act >= 0 && act <= 2, FQ_ERR_PARAMETER, "fq_gemm_x3h: unknown activation");
  if (M == 0 || N == 0) return FQ_OK;
  return launch_xh_gemm(a, a_lo, lda, b, b_lo, ldb, c, ldc, M, N, K, accumulate, bias, residual,
                        ldr, act, as_stream(stream));
}

// The exact-mode GEMM whose output is written only as the next GEMM's fp16
// pair (c = hi, c_lo = lo, both [M, ldc]): the FFN1 / cross-K/V producers.
extern "C" int fq_gemm_x3h_pair(const void* a, const void* a_lo, int64_t lda, const void* b,
                                const void* b_lo, int64_t ldb, void* c, void* c_lo, int64_t ldc,
                                int64_t M, int64_t N, int64_t K, const float* bias, int act,
                                fq_stream_t stream) {
  FQ_CHECK_ARG(c && c_lo && M >= 0 && N >= 0 && K >= 1, FQ_ERR_DIMENSION,
               "fq_gemm_x3h_pair: bad args");
  FQ_CHECK_ARG(act >= 0 && act <= 2, FQ_ERR_PARAMETER, "fq_gemm_x3h_pair: unknown activation");
  if (M == 0 || N == 0) return FQ_OK;
  int rc = check_xh(a, a_lo, lda, b, b_lo, ldb, M, N, K);
  if (rc != FQ_OK) return rc;
  const XhPlan p = plan_xh(M, N, K);
  tc::Epi ep{c, ldc, 1, 0, bias, nullptr, 0, act, g_gemm_dbg};
  ep.chunk_kb = p.chunk_kb;
  ep.c_lo = c_lo;
  cudaStream_t s = as_stream(stream);
  if (p.split == 1 && pair_ok(N, 0, nullptr, c, ldc, true) && ((uintptr_t)c_lo & 15) == 0)
    return pair_bn96(M, N) ? tc::launch_pair<96, 4>(a, a_lo, lda, b, b_lo, ldb, ep, M, N, K, s)
                           : tc::launch_pair<128, 4>(a, a_lo, lda, b, b_lo, ldb, ep, M, N, K, s);
  if (p.split > 1)
    return tc::launch_splitk<128, 3, false, false, tc::OP_X3H>(a, lda, b, ldb, ep, M, N, K,
                                                               p.split, s, tc::LnEpi{}, b_lo, a_lo);
  if (p.bn == 64)
    return tc::launch<64, 4, false, tc::OP_X3H>(a, lda, b, ldb, ep, M, N, K, 1, 1, s,
                                                tc::HarsEpi{}, b_lo, a_lo);
  return tc::launch<128, 3, false, tc::OP_X3H>(a, lda, b, ldb, ep, M, N, K, 1, 1, s,
                                               tc::HarsEpi{}, b_lo, a_lo);
}

// The exact-mode GEMM as its split-K partial slabs only ([S][M][N] fp32 in ws,
// slab s = K slice s; the consumer sums them in slice order, e.g. the exact
// cross-attention's query load): for the shapes whose numerics are K/4
// slices (N <= 1024, K >= 1024); *nslab receives S. FQ_ERR_UNSUPPORTED otherwise.
extern "C" int fq_gemm_x3h_slabs(const void* a, const void* a_lo, int64_t lda, const void* b,
                                 const void* b_lo, int64_t ldb, void* ws, int64_t ws_bytes,
                                 int64_t M, int64_t N, int64_t K, int32_t* nslab,
                                 fq_stream_t stream) {
  FQ_CHECK_ARG(ws && nslab && M > 0 && N > 0 && K > 0, FQ_ERR_DIMENSION,
               "fq_gemm_x3h_slabs: bad args");
  int rc = check_xh(a, a_lo, lda, b, b_lo, ldb, M, N, K);
  if (rc != FQ_OK) return rc;
  const XhPlan p = plan_xh(M, N, K);
  FQ_CHECK_ARG(p.split > 1 && ws_bytes >= (int64_t)p.split * M * N * (int64_t)sizeof(float) &&
                   ((uintptr_t)ws & 15) == 0 && M % 32 == 0 && N % 32 == 0,
               FQ_ERR_UNSUPPORTED, "fq_gemm_x3h_slabs: not a split-K slice shape");
  tc::Epi ep{ws, N, 0, 0, nullptr, nullptr, 0, 0, g_gemm_dbg};
  ep.chunk_kb = p.chunk_kb;
  *nslab = p.split;
  return tc::launch_splitk<128, 3, false, true, tc::OP_X3H>(a, lda, b, ldb, ep, M, N, K, p.split,
                                                            as_stream(stream), tc::LnEpi{}, b_lo,
                                                            a_lo);
}

extern "C" int fq_gemm_x3h_ln(const void* a, const void* a_lo, int64_t lda, const void* b,
                              const void* b_lo, int64_t ldb, const float* bias, const float* res,
                              int64_t ldr, const float* gamma, const float* beta, double eps,
                              float* out, int64_t ldo, void* out16, void* out16_lo,
                              int64_t ldo16, void* ws, int64_t ws_bytes, int64_t M, int64_t N,
                              int64_t K, fq_stream_t stream) {
  FQ_CHECK_ARG(bias && res && gamma && beta && out && M > 0 && N > 0 && K > 0,
               FQ_ERR_DIMENSION, "fq_gemm_x3h_ln: bad args");
  int rc = check_xh(a, a_lo, lda, b, b_lo, ldb, M, N, K);
  if (rc != FQ_OK) return rc;
  const XhPlan p = plan_xh(M, N, K);
  const int64_t slab_need = (int64_t)p.split * M * N * (int64_t)sizeof(float);
  if (p.split > 1 && ws && ws_bytes >= slab_need && ((uintptr_t)ws & 15) == 0 &&
      (N == 512 || N == 1024)) {
    tc::Epi ep{ws, N, 0, 0, nullptr, nullptr, 0, 0, g_gemm_dbg};
    ep.chunk_kb = p.chunk_kb;
    rc = tc::launch_splitk<128, 3, false, true, tc::OP_X3H>(a, lda, b, ldb, ep, M, N, K, p.split,
                                                            as_stream(stream), tc::LnEpi{}, b_lo,
                                                            a_lo);
    if (rc != FQ_OK) return rc;
    return fq_splitk_bias_residual_layer_norm_xh(reinterpret_cast<const float*>(ws), p.split, N,
                                                 bias, res, ldr, gamma, beta, eps, M, N, out,
                                                 ldo, out16, out16_lo, ldo16, stream);
  }
  rc = launch_xh_gemm(a, a_lo, lda, b, b_lo, ldb, out, ldo, M, N, K, 0, bias, res, ldr, 0,
                      as_stream(stream));
  if (rc != FQ_OK) return rc;
  return fq_layer_norm_xh(out, ldo, gamma, beta, eps, M, N, out, ldo, out16, out16_lo, ldo16,
                          stream);
}

// Logits GEMM with the HARS statistics epilogue (see HarsEpi): x16 [rows, d]
// fp16, emb16 [vocab, d] fp16 (K-major). Column tile width 224 (ncu: the
// C2 logits GEMM's best wave quantisation;
// tiles; ldt >= ceil(vocab / 224) = the number of column tiles).
extern "C" int fq_logits_hars(const void* x16, int64_t ldx, const void* emb16, int64_t lde,
                              int64_t rows, int64_t vocab, int64_t d, const int32_t* dk,
                              int32_t* gmax, float* tmax, double* tsum, int64_t ldt,
                              int32_t* sv_cnt, void* sv, int64_t sv_cap, fq_stream_t stream) {
  FQ_CHECK_ARG(x16 && emb16 && dk && gmax && tmax && tsum && sv_cnt && sv && rows > 0 &&
                   vocab > 0 && d > 0 && ldt >= (vocab + 223) / 224 && sv_cap >= 1 &&
                   ldx % 8 == 0 && lde % 8 == 0,
               FQ_ERR_DIMENSION, "fq_logits_hars: bad args");
  tc::Epi ep{nullptr, 0, 0, 0, nullptr, nullptr, 0, 0, g_gemm_dbg};
  tc::HarsEpi he{dk, gmax, tmax, tsum, sv_cnt, reinterpret_cast<int2*>(sv), (int)sv_cap,
                 (int)ldt};
  return tc::launch<224, 4, true>(x16, ldx, emb16, lde, ep, rows, vocab, d, 1, 1,
                                  as_stream(stream), he);
}

// Exact mode's output layer: the 3xFP16 logits GEMM (CTA pairs, 128-column
// tiles) whose epilogue emits the HARS stage-1 statistics of every (row, tile)
// (hars_tile_stats) for fq_hars_merge_step; x (hi, lo) [rows, d] and the
// output matrix (hi, lo) [vocab, d] are fp16 pairs; vocab % 128 == 0,
// ldt >= vocab / 128.
extern "C" int fq_logits_hars_x3h(const void* x, const void* x_lo, int64_t ldx, const void* emb,
                                  const void* emb_lo, int64_t lde, int64_t rows, int64_t vocab,
                                  int64_t d, const int32_t* dk, int32_t* gmax, float* tmax,
                                  double* tsum, int64_t ldt, int32_t* sv_cnt, void* sv,
                                  int64_t sv_cap, fq_stream_t stream) {
  FQ_CHECK_ARG(dk && gmax && tmax && tsum && sv_cnt && sv && rows > 0 && vocab > 0 && d > 0 &&
                   vocab % 128 == 0 && ldt >= vocab / 128 && sv_cap >= 1,
               FQ_ERR_DIMENSION, "fq_logits_hars_x3h: bad args");
  int rc = check_xh(x, x_lo, ldx, emb, emb_lo, lde, rows, vocab, d);
  if (rc != FQ_OK) return rc;
  const XhPlan p = plan_xh(rows, vocab, d);
  FQ_CHECK_ARG(p.split == 1, FQ_ERR_UNSUPPORTED, "fq_logits_hars_x3h: split-K plan");
  tc::Epi ep{nullptr, 0, 0, 0, nullptr, nullptr, 0, 0, g_gemm_dbg};
  ep.chunk_kb = p.chunk_kb;
  tc::HarsEpi he{dk, gmax, tmax, tsum, sv_cnt, reinterpret_cast<int2*>(sv), (int)sv_cap,
                 (int)ldt};
  return tc::launch_pair<128, 4, true>(x, x_lo, ldx, emb, emb_lo, lde, ep, rows, vocab, d,
                                       as_stream(stream), he);
}

// fp16 GEMM + bias + residual + LayerNorm (the decode step's self-out/LN1,
// cross-out/LN2, FFN2/LN3): the split-K x4 kernel with the LN epilogue when
// the plan is split-K over 128-column tiles and every cluster of the launch can
// be resident at once (the row-block statistics exchange waits for all CTAs of
// the row block), else the GEMM then fq_layer_norm. ws: stats [M][N/128]
// double2 then counters [ceil(M/128)][2] int32, zeroed once by the caller.
extern "C" int fq_gemm_ln(const void* a, int64_t lda, const void* w, int64_t ldw,
                          const float* bias, const float* res, int64_t ldr, const float* gamma,
                          const float* beta, double eps, float* out, int64_t ldo, void* out16,
                          int64_t ldo16, void* ws, int64_t ws_bytes, int64_t M, int64_t N,
                          int64_t K, fq_stream_t stream) {
  FQ_CHECK_ARG(a && w && gamma && beta && out && M > 0 && N > 0 && K > 0, FQ_ERR_DIMENSION,
               "fq_gemm_ln: bad args");
  const TcPlan p = plan_tc(M, N, K);
  const int64_t slab_need = (int64_t)p.split * M * N * (int64_t)sizeof(float);
  if (p.split > 1 && p.bn == 128 && p.cm == 1 && p.cn == 1 && bias && res && ws &&
      ws_bytes >= slab_need && ((uintptr_t)ws & 15) == 0 && N % 4 == 0 &&
      (p.split == 2 || p.split == 4) && (N == 512 || N == 1024 || N == 2048)) {
    tc::Epi ep{ws, N, 0, 0, nullptr, nullptr, 0, 0, g_gemm_dbg};
    int rc = tc::launch_splitk<128, 6, false, true>(a, lda, w, ldw, ep, M, N, K, p.split,
                                                    as_stream(stream));
    if (rc != FQ_OK) return rc;
    return fq_splitk_bias_residual_layer_norm(reinterpret_cast<const float*>(ws), p.split, N,
                                              bias, res, ldr, gamma, beta, eps, M, N, out, ldo,
                                              out16, ldo16, stream);
  }
  const int64_t mt = (M + 127) / 128, nt = N / 128;
  const int64_t need = M * nt * (int64_t)sizeof(double2) + mt * 2 * (int64_t)sizeof(int);
  bool fused = p.split == 4 && p.bn == 128 && p.cm == 1 && p.cn == 1 && N % 128 == 0 &&
               ws && ws_bytes >= need && ((uintptr_t)ws & 15) == 0 && ldo % 4 == 0 &&
               (!out16 || ldo16 % 4 == 0) && (!res || ldr % 4 == 0) &&
               ((uintptr_t)gamma & 15) == 0 && ((uintptr_t)beta & 15) == 0;
  if (fused) {  // every cluster resident at once?
    static int max_clusters = -1;
    if (max_clusters < 0) {
      cudaLaunchConfig_t cfg = {};
      cfg.gridDim = dim3(4);
      cfg.blockDim = dim3(tc::kThreads);
      cfg.dynamicSmemBytes = tc::smem_bytes_splitk<128, 6>();
      cudaLaunchAttribute at;
      at.id = cudaLaunchAttributeClusterDimension;
      at.val.clusterDim.x = 4;
      at.val.clusterDim.y = 1;
      at.val.clusterDim.z = 1;
      cfg.attrs = &at;
      cfg.numAttrs = 1;
      int n = 0;
      if (cudaOccupancyMaxActiveClusters(&n, tc::tc_gemm_splitk_kernel<128, 6, true>, &cfg) !=
          cudaSuccess)
        n = 0;
      cudaGetLastError();
      max_clusters = n;
    }
    fused = mt * nt <= max_clusters;
  }
  if (fused) {
    tc::Epi ep{nullptr, 0, 0, 0, bias, res, ldr, 0, g_gemm_dbg};
    tc::LnEpi ln{gamma, beta, eps, out, ldo, reinterpret_cast<fq::h16*>(out16), ldo16,
                 reinterpret_cast<double2*>(ws),
                 reinterpret_cast<int*>(reinterpret_cast<char*>(ws) + M * nt * sizeof(double2)),
                 (int)nt};
    return tc::launch_splitk<128, 6, true>(a, lda, w, ldw, ep, M, N, K, 4, as_stream(stream),
                                           ln);
  }
  int rc = launch_tc_gemm(a, lda, w, ldw, out, 0, ldo, M, N, K, 0, bias, res, ldr, 0,
                          as_stream(stream));
  if (rc != FQ_OK) return rc;
  return fq_layer_norm(out, ldo, gamma, beta, eps, M, N, out, ldo, out16, ldo16, stream);
}

// The split-K GEMM's K-slice partials as slabs (no reduction): ws [nslab][M][N]
// fp32, slab s = a[:, slice s] . w[:, slice s]^T. *nslab = 0 (nothing launched)
// when the plan for this shape is not split-K or ws is too small.
extern "C" int fq_gemm_splitk_slabs(const void* a, int64_t lda, const void* w, int64_t ldw,
                                    void* ws, int64_t ws_bytes, int64_t M, int64_t N, int64_t K,
                                    int* nslab, fq_stream_t stream) {
  FQ_CHECK_ARG(a && w && nslab && M > 0 && N > 0 && K > 0 && lda % 8 == 0 && ldw % 8 == 0,
               FQ_ERR_DIMENSION, "fq_gemm_splitk_slabs: bad args");
  *nslab = 0;
  const TcPlan p = plan_tc(M, N, K);
  if (!(p.split > 1 && p.bn == 128 && p.cm == 1 && p.cn == 1 && ws && N % 4 == 0 &&
        ((uintptr_t)ws & 15) == 0 && ws_bytes >= (int64_t)p.split * M * N * (int64_t)sizeof(float)))
    return FQ_OK;
  tc::Epi ep{ws, N, 0, 0, nullptr, nullptr, 0, 0, g_gemm_dbg};
  const int rc = tc::launch_splitk<128, 6, false, true>(a, lda, w, ldw, ep, M, N, K, p.split,
                                                        as_stream(stream));
  if (rc == FQ_OK) *nslab = p.split;
  return rc;
}

// Benchmarks only: force (bn, cm, cn) for shapes it divides; bn = 0 restores auto.
extern "C" int fq_gemm_force_plan(int bn, int cm, int cn, int split) {
  g_forced = {bn, cm, cn, split < 1 ? 1 : split};
  return FQ_OK;
}

// Exposed for tests/benchmarks: the plan the dispatcher would pick.
extern "C" int fq_gemm_plan(int64_t M, int64_t N, int64_t K, int* bn, int* cm, int* cn,
                            int* split) {
  const TcPlan p = plan_tc(M, N, K);
  *bn = p.bn;
  *cm = p.cm;
  *cn = p.cn;
  *split = p.split;
  return FQ_OK;
}

}  // namespace fq
