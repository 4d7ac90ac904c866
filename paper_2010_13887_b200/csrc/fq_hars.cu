// Hierarchical Auto-Regressive Search (HARS) output layer on sm_100a.
//
// Stage 1 (retrieve): reference decode.py:58-92 -> kernels.py:155-185. One CTA
// per logit row. The row is read from HBM exactly once with 128-bit loads and
// staged in shared memory (a 32k fp32 row is 128 KB; up to 51200 columns
// fit); the group-maxima sweep runs on the loads, the logsumexp + candidate
// sweep runs from shared memory. Grouping is the reference's deterministic
// stride (token j -> group j % k): with a block width that is a multiple of
// k, every thread's elements fall in fixed groups, so each thread keeps one
// running maximum per vector lane and no atomics are needed.
// Numerics: fp32 x - row_max, fp32 expf, f64 sum,
// lse = f64(row_max) + log(sum); inclusive x >= R; candidates ascending.
//
// Stage 2 (select): decode.py:217-240 beam_search_step + :186-214 selection
// + :160-171 should_stop + engine.py:148-169, one CTA per batch item, on the
// device-resident beam state. Scores are f64 cum + (f64(logit) - lse) and the
// order is (-score, token, beam), exactly the reference's sort key.
#include <stdlib.h>

#include <algorithm>

#include "fq_common.cuh"

namespace fq {

constexpr int kRetrieveThreads = 512;
constexpr int kCandCap = 2048;  // survivors ranked in shared memory; more -> ordered rescan

// block-wide exclusive scan of small ints (blockDim multiple of 32).
__device__ __forceinline__ int block_excl_scan(int v, int* warp_tot, int* total) {
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5, nw = blockDim.x >> 5;
  int incl = v;
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    int t = __shfl_up_sync(0xffffffffu, incl, o);
    if (lane >= o) incl += t;
  }
  if (lane == 31) warp_tot[w] = incl;
  __syncthreads();
  if (w == 0) {
    int x = lane < nw ? warp_tot[lane] : 0;
    int ix = x;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      int t = __shfl_up_sync(0xffffffffu, ix, o);
      if (lane >= o) ix += t;
    }
    if (lane < nw) warp_tot[lane] = ix - x;
    if (lane == 31) *total = ix;
  }
  __syncthreads();
  return incl - v + warp_tot[w];
}

// One CTA (512 threads) per row; up to 4 CTAs per SM. Pass 1 streams the row
// from HBM once (128-bit loads, evict-first); pass 2 re-reads it from L2 (the
// <= 4 x 148 rows in flight are far below the 126 MB L2).
__global__ void __launch_bounds__(kRetrieveThreads, 4) retrieve_kernel(
    const float* __restrict__ logits, int64_t ld, int V, int k_fixed,
    const int32_t* __restrict__ d_k, float* __restrict__ group_max, int64_t gm_ld,
    float* __restrict__ threshold, double* __restrict__ lse, int32_t* __restrict__ cand_idx,
    int64_t cand_ld, int64_t* __restrict__ cand_count) {
  pdl_enter();
  __shared__ float part_max[kRetrieveThreads * 4];
  __shared__ int32_t s_idx[kCandCap];
  __shared__ float gmax_s[32];
  __shared__ float s_R, s_max;
  __shared__ double red[32];
  __shared__ int warp_tot[32];
  __shared__ int s_total, s_cnt;

  const int64_t row = blockIdx.x;
  const int k = d_k ? d_k[row] : k_fixed;
  if (k <= 0) {
    if (threadIdx.x == 0) cand_count[row] = 0;
    return;
  }
  const float* x = logits + row * ld;
  const int tid = threadIdx.x, lane = tid & 31, w = tid >> 5, nw = blockDim.x >> 5;
  const bool vec = ((reinterpret_cast<uintptr_t>(x) & 15) == 0);
  if (tid == 0) s_cnt = 0;

  // ---------------- pass 1: strided group maxima -------------------------
  if (k <= 32) {
    // T threads, T % k == 0: thread t only ever sees groups (4t + c) % k.
    const int T = blockDim.x - (blockDim.x % k);
    float m[4] = {-INFINITY, -INFINITY, -INFINITY, -INFINITY};
    if (tid < T) {
      if (vec) {
        const int nvec = V >> 2;
        const float4* x4 = reinterpret_cast<const float4*>(x);
#pragma unroll 4
        for (int v = tid; v < nvec; v += T) {
          float4 q = __ldcs(x4 + v);
          m[0] = fmaxf(m[0], q.x); m[1] = fmaxf(m[1], q.y);
          m[2] = fmaxf(m[2], q.z); m[3] = fmaxf(m[3], q.w);
        }
      } else {
#pragma unroll 4
        for (int j = tid; j < V; j += T) m[0] = fmaxf(m[0], __ldcs(x + j));
      }
    }
    // partials: vec -> element index e = 4*tid + c (group e % k); scalar -> e = tid
    const int per = vec ? 4 : 1;
    const int nparts = T * per;
    if (tid < T) {
      for (int c = 0; c < per; ++c) part_max[tid * per + c] = m[c];
    }
    __syncthreads();
    for (int g = w; g < k; g += nw) {  // warp g reduces entries e = g (mod k)
      float mm = -INFINITY;
      for (int e = g + lane * k; e < nparts; e += 32 * k) mm = fmaxf(mm, part_max[e]);
      mm = warp_max(mm);
      if (lane == 0) gmax_s[g] = mm;
    }
    __syncthreads();
    if (vec && tid == 0) {  // tail (V % 4 elements) folds into its group directly
      for (int j = (V >> 2) << 2; j < V; ++j) gmax_s[j % k] = fmaxf(gmax_s[j % k], x[j]);
    }
    __syncthreads();
    if (tid == 0) {
      float R = gmax_s[0], M = gmax_s[0];
      for (int g = 0; g < k; ++g) {
        R = fminf(R, gmax_s[g]);
        M = fmaxf(M, gmax_s[g]);
        if (group_max) group_max[row * gm_ld + g] = gmax_s[g];
      }
      s_R = R;
      s_max = M;
    }
    __syncthreads();
  } else {
    // large k (up to V): thread per group, strided columns stay coalesced
    float R = INFINITY, M = -INFINITY;
    for (int g = tid; g < k; g += blockDim.x) {
      float mm = -INFINITY;
      for (int j = g; j < V; j += k) mm = fmaxf(mm, x[j]);
      if (group_max) group_max[row * gm_ld + g] = mm;
      R = fminf(R, mm);
      M = fmaxf(M, mm);
    }
    R = warp_min(R);
    M = warp_max(M);
    if (lane == 0) { part_max[w] = R; part_max[32 + w] = M; }
    __syncthreads();
    if (tid == 0) {
      float r = part_max[0], mm = part_max[32];
      for (int i = 1; i < nw; ++i) { r = fminf(r, part_max[i]); mm = fmaxf(mm, part_max[32 + i]); }
      s_R = r;
      s_max = mm;
    }
    __syncthreads();
  }
  const float R = s_R, M = s_max;

  // ---------------- pass 2 (L2): logsumexp + survivors x >= R ---------------
  double acc = 0.0;
  auto visit = [&](float v, int j) {
    acc += (double)expf(__fsub_rn(v, M));  // E1: fp32 x - max, fp32 expf, f64 sum
    if (v >= R) {
      int p = atomicAdd(&s_cnt, 1);
      if (p < kCandCap) s_idx[p] = j;
    }
  };
  if (vec) {
    const int nvec = V >> 2;
    const float4* x4 = reinterpret_cast<const float4*>(x);
#pragma unroll 4
    for (int v = tid; v < nvec; v += blockDim.x) {
      float4 q = x4[v];
      visit(q.x, 4 * v); visit(q.y, 4 * v + 1); visit(q.z, 4 * v + 2); visit(q.w, 4 * v + 3);
    }
    for (int j = (nvec << 2) + tid; j < V; j += blockDim.x) visit(x[j], j);
  } else {
    for (int j = tid; j < V; j += blockDim.x) visit(x[j], j);
  }
  const double s = block_sum(acc, red);  // contains __syncthreads: s_cnt is final
  const int n = s_cnt;
  int32_t* out_idx = cand_idx + row * cand_ld;
  if (n <= kCandCap) {
    // ascending token order: rank of each (distinct) survivor
    for (int i = tid; i < n; i += blockDim.x) {
      const int j = s_idx[i];
      int rank = 0;
      for (int q = 0; q < n; ++q) rank += s_idx[q] < j ? 1 : 0;
      if (rank < cand_ld) out_idx[rank] = j;
    }
  } else {
    // tie-heavy row: ordered block-scan compaction over the row (rare)
    int64_t base = 0;
    const int chunk = blockDim.x * 4;
    for (int c0 = 0; c0 < V; c0 += chunk) {
      int flags = 0;
#pragma unroll
      for (int c = 0; c < 4; ++c) {
        int j = c0 + tid * 4 + c;
        if (j < V && x[j] >= R) flags |= 1 << c;
      }
      if (!__syncthreads_or(flags)) continue;
      int off = block_excl_scan(__popc(flags), warp_tot, &s_total);
#pragma unroll
      for (int c = 0; c < 4; ++c) {
        if (flags & (1 << c)) {
          int64_t pos = base + off;
          if (pos < cand_ld) out_idx[pos] = c0 + tid * 4 + c;
          ++off;
        }
      }
      base += s_total;
      __syncthreads();
    }
  }
  if (tid == 0) {
    if (threshold) threshold[row] = R;
    lse[row] = (double)M + log(s);
    cand_count[row] = n;
  }
}

// ---------------------------------------------------------------------------
// Stage 1, single-sweep variant (k <= 32, the decode step): the row is read
// once from HBM and every per-element decision is made on the fly.
//   * A pilot (each thread's first U vectors, ~13% of the row) gives a CTA-wide
//     lower bound R' <= R (min over groups of partial group maxima: maxima only
//     grow) and the pilot maximum M'.
//   * Strided group maxima as in the two-pass kernel (thread t, lane c always in
//     group (4t + c) % k).
//   * logsumexp as an online sum started at M': s_t = sum exp(x - m_t), four
//     terms per fp32 partial, f64 accumulation, rescaled in f64 only when an
//     element exceeds the running max (rare after the pilot); combined as
//     S = sum_t s_t exp(m_t - M) in a fixed order. Equal to the reference's lse
//     up to fp32 rounding of the terms (~1e-7; tested against the oracle).
//   * candidates: every x >= R' is appended to a shared-memory survivor list
//     (~0.5% of the row); after R is known the survivors >= R are ranked by
//     token. A survivor overflow (tie-heavy rows) falls back to an ordered
//     rescan of the row from L2.
// ---------------------------------------------------------------------------
constexpr int kSwThreads = 256;
__device__ unsigned long long* g_sw_dbg = nullptr;  // phase stamps (profiling only)
// Phase stamps cost a global load of g_sw_dbg on thread 0's critical path:
// compiled in only for the phase scripts (-DFQ_HARS_STAMPS, build_variant.sh).
__device__ __forceinline__ void sw_stamp(int64_t row, int slot) {
#ifdef FQ_HARS_STAMPS
  if (g_sw_dbg && threadIdx.x == 0) {
    unsigned long long t_;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t_));
    g_sw_dbg[row * 8 + slot] = t_;
  }
#endif
}
__device__ __forceinline__ float ex2_ftz(float x) {
  float y;
  asm("ex2.approx.ftz.f32 %0, %1;" : "=f"(y) : "f"(x));
  return y;
}
constexpr int kSwU = 8;  // pilot vectors per thread (2 / 4 / 6 measured slower or equal)
constexpr int kSwP = 8;   // async ring depth (vectors in flight per thread)
// CTAs (cluster) per row and threads per CTA (A/B builds: -DFQ_ROW_SPLIT,
// -DFQ_ROW_NT). 2 x 128-thread CTAs per row (7 resident per SM, one wave)
// balance bytes per SM but measured slower (stage 1 27.5 vs 24.1 us at C2):
// the per-CTA finishing spread, not the 4-vs-3 rows per SM, sets the tail.
#ifndef FQ_ROW_NT
#define FQ_ROW_NT 256
#endif
#ifndef FQ_ROW_SPLIT
#define FQ_ROW_SPLIT 1
#endif
constexpr int kSwSplit = FQ_ROW_SPLIT;
constexpr int kRowThreads = FQ_ROW_NT;  // threads of the CTA-per-row(-part) kernels
constexpr int kRowMinBlocks = kRowThreads >= 256 ? 4 : 7;  // one resident wave
constexpr int kSurvCap = 2048;
// The fused step's per-row "top list": the row's best kTopC survivors >= R by
// (-logit, token), the only ones stage 2 can pick (it keeps K + live <= 2K <=
// kTopC of the item's candidates, and within a row the score order is the
// logit order). Layout at the end of the row's candidate slots: [0] count (-1:
// none, use the full list), [1, 1 + kTopC) indices, then kTopC logits.
constexpr int kTopC = 32;
constexpr int kTopSlots = 1 + 2 * kTopC;

__device__ __forceinline__ void cp_async16(void* dst, const void* src) {
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(
                   static_cast<uint32_t>(__cvta_generic_to_shared(dst))),
               "l"(src)
               : "memory");
}
__device__ __forceinline__ void cp_async_commit() {
  asm volatile("cp.async.commit_group;" ::: "memory");
}
template <int N>
__device__ __forceinline__ void cp_async_wait() {
  asm volatile("cp.async.wait_group %0;" ::"n"(N) : "memory");
}

// ring: kSwP x kSwThreads float4 of dynamic shared memory (per-thread slots:
// each thread only ever reads back its own async copies, so the ring needs no
// block barrier, only per-thread cp.async groups).
__device__ __forceinline__ uint32_t cl_rank() {
  uint32_t r;
  asm volatile("mov.u32 %0, %%cluster_ctarank;" : "=r"(r));
  return r;
}
__device__ __forceinline__ uint32_t cl_nrank() {
  uint32_t r;
  asm volatile("mov.u32 %0, %%cluster_nctarank;" : "=r"(r));
  return r;
}
__device__ __forceinline__ void cl_sync_all() {
  asm volatile("barrier.cluster.arrive.release.aligned;\n\tbarrier.cluster.wait.acquire.aligned;" ::: "memory");
}
template <typename T>
__device__ __forceinline__ T* peer_ptr(T* p, int rank) {
  return reinterpret_cast<T*>(__cluster_map_shared_rank(reinterpret_cast<void*>(p), rank));
}

// C CTAs (a thread-block cluster, C = 1 or 2) share one row: rank r sweeps the
// vector iterations [r*I0, (r+1)*I0) (I0 a multiple-free split of the per-thread
// iteration count, so the strided group mapping is unchanged); group maxima,
// the logsumexp partial and the survivor counts are exchanged through
// distributed shared memory. Half rows balance the 512 decode rows over 148
// SMs (a row per CTA leaves a 4-vs-3 rows-per-SM tail).
template <int NT>
__device__ __forceinline__ void sweep_row(
    const float* __restrict__ logits, int64_t ld, int V, const int64_t row, const int k,
    float* __restrict__ group_max, int64_t gm_ld, float* __restrict__ threshold,
    double* __restrict__ lse, int32_t* __restrict__ cand_idx, int64_t cand_ld,
    int64_t* __restrict__ cand_count, float4* __restrict__ ring, const int C, const int rank,
    const int64_t vals_off = 0, int32_t* __restrict__ top_out = nullptr,
    int32_t* __restrict__ top_mark = nullptr) {
  // survivors >= R' in per-thread slots ([slot][thread]: no atomics in the
  // sweep), a thread's survivors beyond SL in a shared spill list (atomics,
  // rare); a spill overflow (tie-heavy rows) -> the ordered rescan
  constexpr int SL = 4, SP = NT * 2;
  __shared__ float part_max[NT * 4];
  __shared__ int2 tsv[SL][NT];
  __shared__ int2 spill[SP];
  __shared__ float gmax_s[32];
  __shared__ float s_R, s_M;
  __shared__ double red[NT / 32];
  __shared__ double s_S;
  __shared__ int warp_tot[32];
  __shared__ int s_cnt, s_total, s_n, s_ovf;
  if (k <= 0) {  // uniform across the cluster
    if (threadIdx.x == 0 && rank == 0) cand_count[row] = 0;
    return;
  }
  const float* x = logits + row * ld;
  const int tid = threadIdx.x, lane = tid & 31, w = tid >> 5;
  const int kk = k / (k & -k) * ((k & -k) > 4 ? (k & -k) / 4 : 1);  // k / gcd(k, 4)
  const int T = NT - NT % kk;
  // rows need not be 16-byte aligned (e.g. V = 50257): the first hd < 4
  // elements are a scalar head, vector v then holds columns hd + 4v + c, so
  // lane c of thread t stays in group (hd + 4t + c) % k (part_max[4t + c])
  const int hd = min(V, (int)((4 - ((reinterpret_cast<uintptr_t>(x) >> 2) & 3)) & 3));
  const int hk = hd % k;
  const int nvec = (V - hd) >> 2;
  const float4* x4 = reinterpret_cast<const float4*>(x + hd);
  const bool act = tid < T;
  constexpr float NEG = -INFINITY;
  const int itmax = (nvec + T - 1) / T;      // iterations of thread 0
  const int I0 = (itmax + C - 1) / C;
  const int i_lo = rank * I0;
  const int nit_thr = act && tid < nvec ? (nvec - tid + T - 1) / T : 0;
  const int nit = max(0, min(nit_thr, i_lo + I0) - i_lo);  // this CTA's iterations
  const float4* xb = x4 + tid + (int64_t)i_lo * T;
  // async prologue: this thread's first kSwP vectors in flight at once
#pragma unroll
  for (int i = 0; i < kSwP; ++i) {
    if (i < nit) cp_async16(ring + i * NT + tid, xb + i * T);
    cp_async_commit();
  }
  if (tid == 0) { s_cnt = 0; s_ovf = 0; }
  int nt_sv = 0;  // this thread's survivors (may exceed SL: overflow)
  auto keep = [&](int j, float v) {
    if (nt_sv < SL) {
      tsv[nt_sv][tid] = make_int2(j, __float_as_int(v));
      ++nt_sv;
    } else {
      const int p = atomicAdd(&s_cnt, 1);
      if (p < SP) spill[p] = make_int2(j, __float_as_int(v));
    }
  };
  // ---- pilot (first kSwU vectors): partial group maxima -> R' <= R, M' ----
  float gm[4] = {NEG, NEG, NEG, NEG};
  cp_async_wait<kSwP - kSwU>();
#pragma unroll
  for (int u = 0; u < kSwU; ++u) {
    if (u < nit) {
      const float4 e = ring[u * NT + tid];
      gm[0] = fmaxf(gm[0], e.x); gm[1] = fmaxf(gm[1], e.y);
      gm[2] = fmaxf(gm[2], e.z); gm[3] = fmaxf(gm[3], e.w);
    }
  }
  if (act) {
    part_max[4 * tid] = gm[0]; part_max[4 * tid + 1] = gm[1];
    part_max[4 * tid + 2] = gm[2]; part_max[4 * tid + 3] = gm[3];
  }
  __syncthreads();
  for (int g = w; g < k; g += NT / 32) {
    float mm = NEG;
    for (int e = (g - hk + k) % k + lane * k; e < 4 * T; e += 32 * k) mm = fmaxf(mm, part_max[e]);
    mm = warp_max(mm);
    if (lane == 0) gmax_s[g] = mm;
  }
  __syncthreads();
  if (w == 0) {
    const float gv = lane < k ? gmax_s[lane] : INFINITY;
    const float R = warp_min(gv);
    const float M = warp_max(lane < k ? gv : NEG);
    if (lane == 0) { s_R = R; s_M = M; }
  }
  __syncthreads();
  const float Rp = s_R;  // may be -inf (group without pilot elements): everything survives
  sw_stamp(row, 1);
  // logsumexp reference point: the pilot maximum, kept fixed (terms exp(x - m)
  // up to e^64 are exact enough in fp32/f64): moving it with every new
  // running maximum costs a divergent f64 exp per record (measured +20% on a
  // streaming sweep, scripts/micro/streamprobe.cu)
  constexpr float L2E = 1.4426950408889634f;
  constexpr float L2E_LO = 1.925963033500011e-08f;  // log2(e) - L2E
  constexpr double L2E_D = 1.4426950408889634;
  float m = s_M;
  float mL = m * L2E;
  double s = 0.0;
  // exp(x - m_eff) = 2^(x log2e - mL), m_eff = mL / log2e, log2e as hi + lo
  // fp32 parts (argument exact to ~1 ulp); terms below 2^-126 flush to 0
  auto terms4 = [&](const float4& e) {
    return (ex2_ftz(fmaf(e.x, L2E_LO, fmaf(e.x, L2E, -mL))) +
            ex2_ftz(fmaf(e.y, L2E_LO, fmaf(e.y, L2E, -mL)))) +
           (ex2_ftz(fmaf(e.z, L2E_LO, fmaf(e.z, L2E, -mL))) +
            ex2_ftz(fmaf(e.w, L2E_LO, fmaf(e.w, L2E, -mL))));
  };
  // rescale threshold (m + 64; -inf while m is -inf): the running maximum
  // moves only for wildly larger elements (the terms stay exact to ~1e-7)
  float thr = m == NEG ? NEG : m + 64.f;
  const float4* src = xb + kSwP * T;
  for (int i = 0; i < nit; ++i) {
    cp_async_wait<kSwP - 1>();
    float4* slot = ring + (i % kSwP) * NT + tid;
    const float4 e = *slot;
    if (i + kSwP < nit) cp_async16(slot, src);
    src += T;
    cp_async_commit();
    gm[0] = fmaxf(gm[0], e.x); gm[1] = fmaxf(gm[1], e.y);
    gm[2] = fmaxf(gm[2], e.z); gm[3] = fmaxf(gm[3], e.w);
    const float m4 = fmaxf(fmaxf(e.x, e.y), fmaxf(e.z, e.w));
    if (m4 > thr) {  // new maximum beyond m + 64, or m still -inf (practically never)
      if (m4 != NEG) {
        s = m == NEG ? 0.0 : s * exp2((double)mL - (double)m4 * L2E_D);
        m = m4;
        mL = m * L2E;
      }
      thr = m == NEG ? NEG : m + 64.f;
    }
    if (m != NEG) s += (double)terms4(e);
    // survivors: predicated slot stores, one per element >= R'
    const int j0 = hd + 4 * (tid + (i_lo + i) * T);
    if (e.x >= Rp) keep(j0, e.x);
    if (e.y >= Rp) keep(j0 + 1, e.y);
    if (e.z >= Rp) keep(j0 + 2, e.z);
    if (e.w >= Rp) keep(j0 + 3, e.w);
  }
  cp_async_wait<0>();
  sw_stamp(row, 2);
  if (act) {
    part_max[4 * tid] = gm[0]; part_max[4 * tid + 1] = gm[1];
    part_max[4 * tid + 2] = gm[2]; part_max[4 * tid + 3] = gm[3];
  }
  // scalar head (rank 0) and tail (the last rank): each rank's survivors stay
  // in column order across ranks
  const int h0 = rank == 0 ? 0 : hd, h1 = rank == 0 ? hd : hd;
  const int t0 = rank == C - 1 ? hd + (nvec << 2) : V;
  if (tid == 0) {
    for (int jj = h0; jj < h1 + (V - t0); ++jj) {
      const int j = jj < h1 ? jj : t0 + (jj - h1);
      const float xv = x[j];
      if (xv > m + 64.f || m == NEG) {
        if (xv != NEG) {
          s = m == NEG ? 0.0 : s * exp2((double)mL - (double)xv * L2E_D);
          m = xv;
          mL = m * L2E;
        }
      }
      if (m != NEG) s += (double)ex2_ftz(fmaf(xv, L2E_LO, fmaf(xv, L2E, -mL)));
      if (xv >= Rp) keep(j, xv);
    }
  }
  __syncthreads();
  for (int g = w; g < k; g += NT / 32) {
    float mm = NEG;
    for (int e = (g - hk + k) % k + lane * k; e < 4 * T; e += 32 * k) mm = fmaxf(mm, part_max[e]);
    mm = warp_max(mm);
    if (lane == 0) gmax_s[g] = mm;
  }
  __syncthreads();
  if (tid == 0)
    for (int jj = h0; jj < h1 + (V - t0); ++jj) {
      const int j = jj < h1 ? jj : t0 + (jj - h1);
      gmax_s[j % k] = fmaxf(gmax_s[j % k], x[j]);
    }
  if (C > 1) cl_sync_all();  // both halves' group maxima complete
  if (w == 0) {
    float gv = NEG;
    if (lane < k) {
      gv = gmax_s[lane];
      for (int r2 = 0; r2 < C; ++r2)
        if (r2 != rank) gv = fmaxf(gv, *peer_ptr(&gmax_s[lane], r2));
      if (rank == 0 && group_max) group_max[row * gm_ld + lane] = gv;
    }
    const float R = warp_min(lane < k ? gv : INFINITY);
    const float M = warp_max(gv);
    if (lane == 0) { s_R = R; s_M = M; }
  }
  __syncthreads();
  const float R = s_R, M = s_M;
  const double st = m == NEG ? 0.0 : s * exp2((double)mL - (double)M * L2E_D);
  const double Sl = block_sum(st, red);  // contains __syncthreads
  sw_stamp(row, 3);
  int32_t* out_idx = cand_idx + row * cand_ld;
  // survivors >= R of this CTA, compacted, then ranked by token below
  if (tid == 0) { s_n = 0; s_S = Sl; }
  __syncthreads();
  const int nsp = s_cnt;  // spilled survivors
  auto filt = [&](int2 sv) {
    const float v = __int_as_float(sv.y);
    if (v >= R) {
      const int p = atomicAdd(&s_n, 1);
      if (p < NT * 2) {  // (index, value) pairs
        part_max[2 * p] = __int_as_float(sv.x);
        part_max[2 * p + 1] = v;
      }
    }
  };
  for (int i = 0; i < nt_sv; ++i) filt(tsv[i][tid]);
  for (int i = tid; i < min(nsp, SP); i += NT) filt(spill[i]);
  __syncthreads();
  if (tid == 0) s_ovf = (nsp > SP || s_n > NT * 2) ? 1 : 0;
  if (C > 1) cl_sync_all();  // counts, overflow flags and partial sums visible
  else __syncthreads();
  int ovf = 0, base = 0, total = 0;
  double S = 0.0;
  for (int r2 = 0; r2 < C; ++r2) {
    const int n2 = r2 == rank ? s_n : *peer_ptr(&s_n, r2);
    ovf |= r2 == rank ? s_ovf : *peer_ptr(&s_ovf, r2);
    if (r2 < rank) base += n2;
    total += n2;
    S += r2 == rank ? s_S : *peer_ptr(&s_S, r2);  // fixed rank order
  }
  if (!ovf) {
    const int n = s_n;
    for (int i = tid; i < n; i += NT) {
      const int j = __float_as_int(part_max[2 * i]);
      const float v = part_max[2 * i + 1];
      int rk = 0, rl = 0;  // rank by token; rank by (-logit, token)
      for (int q2 = 0; q2 < n; ++q2) {
        const int jq = __float_as_int(part_max[2 * q2]);
        const float vq = part_max[2 * q2 + 1];
        rk += jq < j ? 1 : 0;
        rl += (vq > v || (vq == v && jq < j)) ? 1 : 0;
      }
      if (base + rk < cand_ld) out_idx[base + rk] = j;
      if (vals_off && base + rk < vals_off)  // candidate logit beside its index (stage 2)
        out_idx[vals_off + base + rk] = __float_as_int(v);
      if (top_out && rl < kTopC) {  // the row's best kTopC (stage 2 ranks only these)
        top_out[1 + rl] = j;
        top_out[1 + kTopC + rl] = __float_as_int(v);
      }
    }
    if (tid == 0 && rank == 0) cand_count[row] = total;
    if (top_out && tid == 0) *top_mark = C == 1 ? min(n, kTopC) : -1;
  } else if (rank == 0) {
    // ordered block-scan compaction over the whole row (tie-heavy rows)
    int64_t cb = 0;
    const int chunk = NT * 4;
    for (int c0 = 0; c0 < V; c0 += chunk) {
      int flags = 0;
#pragma unroll
      for (int c = 0; c < 4; ++c) {
        const int j = c0 + tid * 4 + c;
        if (j < V && x[j] >= R) flags |= 1 << c;
      }
      if (!__syncthreads_or(flags)) continue;
      int off = block_excl_scan(__popc(flags), warp_tot, &s_total);
#pragma unroll
      for (int c = 0; c < 4; ++c) {
        if (flags & (1 << c)) {
          const int64_t pos = cb + off;
          const int j = c0 + tid * 4 + c;
          if (pos < cand_ld) out_idx[pos] = j;
          if (vals_off && pos < vals_off) out_idx[vals_off + pos] = __float_as_int(x[j]);
          ++off;
        }
      }
      cb += s_total;
      __syncthreads();
    }
    if (tid == 0) cand_count[row] = cb;
    if (top_out && tid == 0) *top_mark = -1;  // no top list: stage 2 reads the full list
  }
  if (tid == 0 && rank == 0) {
    if (threshold) threshold[row] = R;
    lse[row] = (double)M + log(S);
    sw_stamp(row, 4);
  }
  if (C > 1) cl_sync_all();  // peers done reading my shared memory
}

__global__ void __launch_bounds__(kRowThreads, kRowMinBlocks) retrieve_sweep_kernel(
    const float* __restrict__ logits, int64_t ld, int V, int k_fixed,
    const int32_t* __restrict__ d_k, float* __restrict__ group_max, int64_t gm_ld,
    float* __restrict__ threshold, double* __restrict__ lse, int32_t* __restrict__ cand_idx,
    int64_t cand_ld, int64_t* __restrict__ cand_count) {
  pdl_enter();
  extern __shared__ __align__(16) float4 sw_ring[];
  const int C = (int)cl_nrank(), rank = (int)cl_rank();
  const int64_t row = blockIdx.x / C;
  if (rank == 0) sw_stamp(row, 0);
#ifdef FQ_HARS_STAMPS
  if (g_sw_dbg && threadIdx.x == 0 && rank == 0) {  // SM of the row (phase scripts)
    uint32_t smid;
    asm volatile("mov.u32 %0, %%smid;" : "=r"(smid));
    g_sw_dbg[(1536 + row) * 8] = smid;
  }
#endif
  sweep_row<kRowThreads>(logits, ld, V, row, d_k ? d_k[row] : k_fixed, group_max, gm_ld,
                         threshold, lse, cand_idx, cand_ld, cand_count, sw_ring, C, rank);
}

// ---------------------------------------------------------------------------
// Stage 1, balanced split (k <= 32, V % 4 == 0, V >= 2048; the default).
// The [rows, V/4] float4 space is cut into G equal contiguous ranges, one per
// CTA of a single resident wave (G = SMs x resident CTAs, fewer for small
// problems); a boundary within kMinPortion vectors of a row start/end snaps
// to it, so every row portion holds >= kMinPortion vectors. So every SM
// streams the same number of bytes whatever rows vs SMs is (a CTA per row
// leaves 4-vs-3 rows per SM at 512 rows and idles most SMs at few rows).
//   * A CTA sweeps each row portion in its range exactly like sweep_row
//     (pilot bound, strided group maxima, online logsumexp, survivor list)
//     and leaves a partial inside the row's own candidate row (cand_ld >= V):
//     its survivors >= its local bound min_g(portion group max) <= R at the
//     portion's first slots, and a header in its last kHdr slots.
//   * It then adds its portion length to the row's arrival counter; the CTA
//     that completes the row merges the partials in column order (group
//     maxima -> R and M, S = sum_p S_p exp(M_p - M) in fixed order, survivors
//     >= R ranked by token) into the row's outputs, overwriting the partials.
// Same results as retrieve_kernel / sweep_row (candidates and group maxima
// exact, lse to fp32 rounding of the terms).
// ---------------------------------------------------------------------------
constexpr int kHdr = 40;           // header slots: [0,32) group maxima, 32 M_p, 33-34 S_p, 35 n, 36 ovf
constexpr int kMinPortion = 256;   // float4 per row portion (>= kSwThreads: every thread works)
constexpr int kMaxPortions = 160;   // per row (G <= (kMaxPortions - 2) * rows)

struct SplitGeom {
  int64_t Q;     // rows * nvec
  int64_t nvec;  // V / 4
  int G;         // CTAs
};
// Q = rows * nvec < 2^31 (checked on the host): 32-bit row arithmetic; c*Q/G
// in double is exact (c*Q < 2^53; a non-integer quotient is >= 1/G away from
// the next integer, far above the double ulp at < 2^31).
__host__ __device__ __forceinline__ int64_t split_bound(const SplitGeom& g, int64_t c) {
  if (c <= 0) return 0;
  if (c >= g.G) return g.Q;
  const uint32_t x = (uint32_t)(((double)c * (double)g.Q) / (double)g.G);
  const uint32_t nv = (uint32_t)g.nvec;
  const uint32_t r = x / nv;
  uint32_t off = x - r * nv;
  if (off < (uint32_t)kMinPortion) off = 0;
  else if (nv - off < (uint32_t)kMinPortion) off = nv;
  return (int64_t)r * nv + off;
}
// the CTA whose range holds float4 position p (0 <= p < Q)
__device__ __forceinline__ int split_find(const SplitGeom& g, int64_t p) {
  int c = (int)(((double)p * (double)g.G) / (double)g.Q) - 2;
  if (c < 0) c = 0;
  while (c + 1 < g.G && split_bound(g, c + 1) <= p) ++c;
  return c;
}

__device__ __forceinline__ int f2ord(float f) {
  const int i = __float_as_int(f);
  return i >= 0 ? i : i ^ 0x7fffffff;
}
__device__ __forceinline__ float ord2f(int i) { return __int_as_float(i >= 0 ? i : i ^ 0x7fffffff); }


struct __align__(16) SplitSmem {
  float wsc[kSwThreads / 32][128];  // per-warp group-maxima scratch
  int32_t sv_idx[kSurvCap];
  float sv_val[kSurvCap];
  float gmax[32];
  int gmax_ord[32];                 // CTA group maxima (ordered ints, atomicMax)
  double red[kSwThreads / 32];
  int warp_tot[32];
  int cnt, n, total, ovf, c_first, np;
  float R, M;
  double S;
};

__device__ __forceinline__ int lattice_T(int k) {
  const int kk = k / (k & -k) * ((k & -k) > 4 ? (k & -k) / 4 : 1);  // k / gcd(k, 4)
  return kSwThreads - kSwThreads % kk;
}

// Sweep float4 columns [a, b) of one row (x = row base) with k groups; write
// the partial into crow (the row's candidate slots). As sweep_row: a
// per-thread cp.async ring, a CTA pilot (the first kSwU vectors per thread)
// for the survivor bound R' <= R and the logsumexp reference m, which stays
// fixed (terms exp(x - m) up to e^64 are exact enough in fp32/f64; moving it
// with every new maximum costs a divergent f64 exp per record, measured +20%
// on the sweep in scripts/micro/streamprobe.cu).
__device__ __forceinline__ void sweep_portion(const float* __restrict__ x, const int a, const int b,
                                              const int k, int32_t* __restrict__ crow,
                                              float4* __restrict__ ring, SplitSmem& sm) {
  const int tid = threadIdx.x, lane = tid & 31, w = tid >> 5;
  const int T = lattice_T(k);
  const bool act = tid < T;
  constexpr float NEG = -INFINITY;
  constexpr float L2E = 1.4426950408889634f;
  constexpr float L2E_LO = 1.925963033500011e-08f;  // log2(e) - L2E
  constexpr double L2E_D = 1.4426950408889634;
  float* part_max = &sm.wsc[0][0];
  // thread t owns float4 columns t + T*i (the row-global lattice): lane c of
  // its vectors is always in group (4t + c) % k
  int nit = 0, v0 = 0;
  if (act) {
    const int i0 = a > tid ? (a - tid + T - 1) / T : 0;
    v0 = tid + i0 * T;
    nit = v0 < b ? (b - 1 - v0) / T + 1 : 0;
  }
  const float4* xb = reinterpret_cast<const float4*>(x) + v0;
#pragma unroll
  for (int i = 0; i < kSwP; ++i) {
    if (i < nit) cp_async16(ring + i * kSwThreads + tid, xb + i * T);
    cp_async_commit();
  }
  if (tid == 0) { sm.cnt = 0; sm.n = 0; }
  // ---- pilot: partial group maxima of the first kSwU vectors -> R', m ----
  float gm[4] = {NEG, NEG, NEG, NEG};
  cp_async_wait<kSwP - kSwU>();
#pragma unroll
  for (int u = 0; u < kSwU; ++u) {
    if (u < nit) {
      const float4 e = ring[u * kSwThreads + tid];
      gm[0] = fmaxf(gm[0], e.x); gm[1] = fmaxf(gm[1], e.y);
      gm[2] = fmaxf(gm[2], e.z); gm[3] = fmaxf(gm[3], e.w);
    }
  }
  if (act) {
    part_max[4 * tid] = gm[0]; part_max[4 * tid + 1] = gm[1];
    part_max[4 * tid + 2] = gm[2]; part_max[4 * tid + 3] = gm[3];
  }
  __syncthreads();
  for (int gg = w; gg < k; gg += kSwThreads / 32) {
    float mm = NEG;
    for (int e = gg + lane * k; e < 4 * T; e += 32 * k) mm = fmaxf(mm, part_max[e]);
    mm = warp_max(mm);
    if (lane == 0) sm.gmax[gg] = mm;
  }
  __syncthreads();
  if (w == 0) {
    const float gv = lane < k ? sm.gmax[lane] : INFINITY;
    const float R = warp_min(gv);
    const float M = warp_max(lane < k ? gv : NEG);
    if (lane == 0) { sm.R = R; sm.M = M; }
  }
  __syncthreads();
  const float Rp = sm.R;
  float m = sm.M;
  float mL = m * L2E;
  double s = 0.0;
  for (int i = 0; i < nit; ++i) {
    cp_async_wait<kSwP - 1>();
    float4* slot = ring + (i % kSwP) * kSwThreads + tid;
    const float4 e = *slot;
    if (i + kSwP < nit) cp_async16(slot, xb + (i + kSwP) * T);
    cp_async_commit();
    if (i >= kSwU) {
      gm[0] = fmaxf(gm[0], e.x); gm[1] = fmaxf(gm[1], e.y);
      gm[2] = fmaxf(gm[2], e.z); gm[3] = fmaxf(gm[3], e.w);
    }
    const float m4 = fmaxf(fmaxf(e.x, e.y), fmaxf(e.z, e.w));
    if (m4 > m + 64.f || m == NEG) {  // (practically never for logits)
      if (m4 != NEG) {
        s = m == NEG ? 0.0 : s * exp2((double)mL - (double)m4 * L2E_D);
        m = m4;
        mL = m * L2E;
      }
    }
    // exp(x - m_eff) = 2^(x log2e - mL), m_eff = mL / log2e, log2e as hi + lo
    // fp32 parts (argument exact to ~1 ulp); terms below 2^-126 flush to 0
    if (m != NEG) {
      const float t4 = (ex2_ftz(fmaf(e.x, L2E_LO, fmaf(e.x, L2E, -mL))) +
                        ex2_ftz(fmaf(e.y, L2E_LO, fmaf(e.y, L2E, -mL)))) +
                       (ex2_ftz(fmaf(e.z, L2E_LO, fmaf(e.z, L2E, -mL))) +
                        ex2_ftz(fmaf(e.w, L2E_LO, fmaf(e.w, L2E, -mL))));
      s += (double)t4;
    }
    if (m4 >= Rp) {
      const int v = v0 + i * T;
      const float e4[4] = {e.x, e.y, e.z, e.w};
#pragma unroll
      for (int c = 0; c < 4; ++c) {
        if (e4[c] >= Rp) {
          const int p = atomicAdd(&sm.cnt, 1);
          if (p < kSurvCap) { sm.sv_idx[p] = 4 * v + c; sm.sv_val[p] = e4[c]; }
        }
      }
    }
  }
  cp_async_wait<0>();
  if (act) {
    part_max[4 * tid] = gm[0]; part_max[4 * tid + 1] = gm[1];
    part_max[4 * tid + 2] = gm[2]; part_max[4 * tid + 3] = gm[3];
  }
  __syncthreads();
  for (int gg = w; gg < k; gg += kSwThreads / 32) {
    float mm = NEG;
    for (int e = gg + lane * k; e < 4 * T; e += 32 * k) mm = fmaxf(mm, part_max[e]);
    mm = warp_max(mm);
    if (lane == 0) sm.gmax[gg] = mm;
  }
  __syncthreads();
  if (w == 0) {
    const float gv = lane < k ? sm.gmax[lane] : INFINITY;
    const float R = warp_min(gv);
    const float M = warp_max(lane < k ? gv : NEG);
    if (lane == 0) { sm.R = R; sm.M = M; }
  }
  __syncthreads();
  const float Rl = sm.R, Mp = sm.M;  // local bound Rl <= R (maxima only grow)
  const double Sp =
      block_sum(m == NEG ? 0.0 : s * exp2((double)mL - (double)Mp * L2E_D), sm.red);
  const int nsv = sm.cnt;
  const int cap = (4 * (b - a) - kHdr) / 2;
  int32_t* sidx = crow + 4 * a;
  int32_t* sval = sidx + cap;
  if (nsv <= kSurvCap) {
    for (int i = tid; i < nsv; i += kSwThreads) {
      const float v = sm.sv_val[i];
      if (v >= Rl) {
        const int p = atomicAdd(&sm.n, 1);
        if (p < cap) { sidx[p] = sm.sv_idx[i]; sval[p] = __float_as_int(v); }
      }
    }
  }
  __syncthreads();
  int32_t* hdr = crow + 4 * b - kHdr;
  if (tid < k) hdr[tid] = __float_as_int(sm.gmax[tid]);
  if (tid == 0) {
    hdr[32] = __float_as_int(Mp);
    const long long sb = __double_as_longlong(Sp);
    hdr[33] = (int32_t)(sb & 0xffffffffll);
    hdr[34] = (int32_t)(sb >> 32);
    hdr[35] = min(sm.n, cap);
    hdr[36] = (nsv > kSurvCap || sm.n > cap) ? 1 : 0;
  }
}

// Merge the partials of row `row` (all portions arrived). x = row base.
__device__ __forceinline__ void finalize_split_row(
    const SplitGeom& g, const int64_t row, const int k, const float* __restrict__ x,
    int32_t* __restrict__ crow, float* __restrict__ group_max, int64_t gm_ld,
    float* __restrict__ threshold, double* __restrict__ lse, int64_t* __restrict__ cand_count,
    int64_t cand_ld, int64_t vals_off, void* dyn, SplitSmem& sm) {
  const int tid = threadIdx.x, lane = tid & 31, w = tid >> 5;
  const int V = (int)(g.nvec * 4);
  if (k <= 0) {
    if (tid == 0) cand_count[row] = 0;
    return;
  }
  const int64_t rs = row * g.nvec, re = rs + g.nvec;
  // portion table in the warp scratch (the ring may be streaming the CTA's
  // next portion): S as double, a, b, n as int, M as float
  (void)dyn;
  double* pS = reinterpret_cast<double*>(&sm.wsc[0][0]);
  int* pa = reinterpret_cast<int*>(pS + kMaxPortions);
  int* pb = pa + kMaxPortions;
  int* pn = pb + kMaxPortions;
  float* pM = reinterpret_cast<float*>(pn + kMaxPortions);
  if (tid == 0) {
    const int c0 = split_find(g, rs), c1 = split_find(g, re - 1);
    sm.c_first = c0;
    sm.np = min(c1 - c0 + 1, kMaxPortions);
    sm.ovf = c1 - c0 + 1 > kMaxPortions ? 1 : 0;
    sm.cnt = 0;
  }
  if (tid < 32) sm.gmax_ord[tid] = f2ord(-INFINITY);
  __syncthreads();
  const int np = sm.np;
  for (int j = tid; j < np; j += kSwThreads) {
    const int64_t c = sm.c_first + j;
    pa[j] = (int)(max(split_bound(g, c), rs) - rs);
    pb[j] = (int)(min(split_bound(g, c + 1), re) - rs);
  }
  __syncthreads();
  // per-portion group maxima table in the (idle) survivor lists (sv_idx and
  // sv_val are adjacent: 2 * kSurvCap floats; the host keeps np * k within it)
  float* pgm = reinterpret_cast<float*>(sm.sv_idx);
  // every header word of every portion in one round trip: word w of a portion
  // is group maximum w (< k) or one of M, S lo, S hi, n, ovf; the loads of a
  // thread's words are all issued before any is used
  {
    const int nw = k + 5, total = np * nw;
    for (int e0 = tid; e0 < total; e0 += 4 * kSwThreads) {
      int v[4];
#pragma unroll
      for (int u = 0; u < 4; ++u) {
        const int e = e0 + u * kSwThreads;
        if (e < total) {
          const int j = e / nw, wq = e - j * nw;
          v[u] = __ldcg(crow + 4 * pb[j] - kHdr + (wq < k ? wq : 32 + (wq - k)));
        }
      }
#pragma unroll
      for (int u = 0; u < 4; ++u) {
        const int e = e0 + u * kSwThreads;
        if (e >= total) continue;
        const int j = e / nw, wq = e - j * nw;
        if (wq < k) pgm[j * k + wq] = __int_as_float(v[u]);  // reduced per group below
        else if (wq == k) pM[j] = __int_as_float(v[u]);
        else if (wq == k + 1) reinterpret_cast<int*>(pS + j)[0] = v[u];
        else if (wq == k + 2) reinterpret_cast<int*>(pS + j)[1] = v[u];
        else if (wq == k + 3) pn[j] = v[u];
        else if (v[u]) sm.ovf = 1;
      }
    }
  }
  __syncthreads();
  for (int gq = w; gq < k; gq += kSwThreads / 32) {  // warp per group: max over portions
    float mm = -INFINITY;
    for (int j = lane; j < np; j += 32) mm = fmaxf(mm, pgm[j * k + gq]);
    mm = warp_max(mm);
    if (lane == 0) sm.gmax[gq] = mm;
  }
  __syncthreads();
  if (w == 0) {
    const float gv = lane < k ? sm.gmax[lane] : INFINITY;
    if (lane < k && group_max) group_max[row * gm_ld + lane] = gv;
    const float R = warp_min(gv);
    const float M = warp_max(lane < k ? gv : -INFINITY);
    if (lane == 0) { sm.R = R; sm.M = M; }
  }
  __syncthreads();
  // exclusive prefix of the portions' survivor counts (np <= kMaxPortions <=
  // kSwThreads: one per thread) for the flattened gather below; a portion whose
  // maximum is below R holds no survivor >= R and is skipped
  const int my_n = tid < np && pM[tid] >= sm.R ? pn[tid] : 0;
  const int my_off = block_excl_scan(my_n, sm.warp_tot, &sm.total);  // contains syncs
  const int n_all = sm.total;
  __shared__ int s_cap[kMaxPortions], s_base[kMaxPortions];
  if (tid < np) {
    s_cap[tid] = (4 * (pb[tid] - pa[tid]) - kHdr) / 2;
    s_base[tid] = 4 * pa[tid];
  }
  __syncthreads();
  if (tid < np) pn[tid] = my_off;  // pn now holds the exclusive prefix
  __syncthreads();
  const float R = sm.R, M = sm.M;
  double acc = 0.0;
  for (int j = tid; j < np; j += kSwThreads)  // fixed assignment + fixed tree: deterministic
    acc += pS[j] == 0.0 ? 0.0 : pS[j] * exp((double)pM[j] - (double)M);
  const double S = block_sum(acc, sm.red);
  sw_stamp(blockIdx.x, 6);
  // survivors >= R of every portion, flattened over all threads (binary search
  // of the portion in the prefix), loads issued ahead of use
  if (!sm.ovf) {
    for (int e0 = tid; e0 < n_all; e0 += 2 * kSwThreads) {
      float v[2];
      int ix[2];
#pragma unroll
      for (int u = 0; u < 2; ++u) {
        const int e = e0 + u * kSwThreads;
        v[u] = -INFINITY;
        if (e < n_all) {
          int lo = 0, hi = np - 1;  // last j with pn[j] <= e
          while (lo < hi) {
            const int mid = (lo + hi + 1) >> 1;
            if (pn[mid] <= e) lo = mid; else hi = mid - 1;
          }
          const int i = e - pn[lo];
          const int32_t* sidx = crow + s_base[lo];
          v[u] = __int_as_float(__ldcg(sidx + s_cap[lo] + i));
          ix[u] = __ldcg(sidx + i);
        }
      }
#pragma unroll
      for (int u = 0; u < 2; ++u) {
        if (e0 + u * kSwThreads < n_all && v[u] >= R) {
          const int p = atomicAdd(&sm.cnt, 1);
          if (p < kSurvCap) { sm.sv_idx[p] = ix[u]; sm.sv_val[p] = v[u]; }
        }
      }
    }
  }
  __syncthreads();  // every partial read before the row is overwritten below
  sw_stamp(blockIdx.x, 7);
  const int n = sm.cnt;
  if (!sm.ovf && n <= kSurvCap) {
    for (int i = tid; i < n; i += kSwThreads) {
      const int j = sm.sv_idx[i];
      int rk = 0;
      for (int q = 0; q < n; ++q) rk += sm.sv_idx[q] < j ? 1 : 0;
      if (rk < cand_ld) crow[rk] = j;
      if (vals_off && rk < vals_off) crow[vals_off + rk] = __float_as_int(sm.sv_val[i]);
    }
    if (tid == 0) cand_count[row] = n;
  } else {
    // ordered block-scan compaction over the whole row (tie-heavy rows)
    int64_t cb = 0;
    const int chunk = kSwThreads * 4;
    for (int c0 = 0; c0 < V; c0 += chunk) {
      int flags = 0;
#pragma unroll
      for (int c = 0; c < 4; ++c) {
        const int j = c0 + tid * 4 + c;
        if (j < V && x[j] >= R) flags |= 1 << c;
      }
      if (!__syncthreads_or(flags)) continue;
      int off = block_excl_scan(__popc(flags), sm.warp_tot, &sm.total);
#pragma unroll
      for (int c = 0; c < 4; ++c) {
        if (flags & (1 << c)) {
          const int64_t pos = cb + off;
          const int j = c0 + tid * 4 + c;
          if (pos < cand_ld) crow[pos] = j;
          if (vals_off && pos < vals_off) crow[vals_off + pos] = __float_as_int(x[j]);
          ++off;
        }
      }
      cb += sm.total;
      __syncthreads();
    }
    if (tid == 0) cand_count[row] = cb;
  }
  if (tid == 0) {
    if (threshold) threshold[row] = R;
    lse[row] = (double)M + log(S);
  }
}

// Walk this CTA's range; for each row portion: sweep, arrive, and (if it
// completed the row) finalize + on_row(row).
template <typename OnRow, typename KOf>
__device__ __forceinline__ void split_walk(const SplitGeom& g, const float* __restrict__ logits,
                                           int64_t ld, int32_t* __restrict__ cand_idx,
                                           int64_t cand_ld, int* row_ctr, int ctr_stride,
                                           bool self_reset, float4* ring, SplitSmem& sm,
                                           KOf k_of, OnRow on_row) {
  __shared__ int s_last;
  const int64_t A = split_bound(g, blockIdx.x), B = split_bound(g, blockIdx.x + 1);
  int64_t p = A;
  int nport = 0;
  sw_stamp(blockIdx.x, 0);
  while (p < B) {
    const int64_t row = p / g.nvec;
    const int64_t rs = row * g.nvec;
    const int a = (int)(p - rs);
    const int b = (int)(min(B, rs + g.nvec) - rs);
    const int k = k_of(row);
    const float* x = logits + row * ld;
    int32_t* crow = cand_idx + row * cand_ld;
    if (k > 0) sweep_portion(x, a, b, k, crow, ring, sm);
    sw_stamp(blockIdx.x, 1 + min(nport++, 1));
    __syncthreads();
    if (threadIdx.x == 0) {
      __threadfence();
      int* ctr = row_ctr + row * ctr_stride;
      const int prev = atomicAdd(ctr, b - a);
      s_last = prev + (b - a) == (int)g.nvec;
      if (s_last && self_reset) *ctr = 0;
    }
    __syncthreads();
    if (s_last) {
      __threadfence();
      sw_stamp(blockIdx.x, 3);
      on_row(row, k, x, crow);
      sw_stamp(blockIdx.x, 4);
    }
    __syncthreads();
    p = rs + b;
  }
  sw_stamp(blockIdx.x, 5);
}

__global__ void __launch_bounds__(kSwThreads, 4) retrieve_split_kernel(
    const float* __restrict__ logits, int64_t ld, SplitGeom g, int k_fixed,
    const int32_t* __restrict__ d_k, float* __restrict__ group_max, int64_t gm_ld,
    float* __restrict__ threshold, double* __restrict__ lse, int32_t* __restrict__ cand_idx,
    int64_t cand_ld, int64_t* __restrict__ cand_count) {
  pdl_enter();
  extern __shared__ __align__(16) float4 sw_ring[];
  __shared__ SplitSmem sm;
  // arrival counters: the low words of cand_count (zeroed by the launcher)
  split_walk(
      g, logits, ld, cand_idx, cand_ld, reinterpret_cast<int*>(cand_count), 2, false, sw_ring, sm,
      [&](int64_t row) { return d_k ? d_k[row] : k_fixed; },
      [&](int64_t row, int k, const float* x, int32_t* crow) {
        finalize_split_row(g, row, k, x, crow, group_max, gm_ld, threshold, lse, cand_count,
                           cand_ld, 0, sw_ring, sm);
      });
}


// ---------------------------------------------------------------------------
// stage 2
// ---------------------------------------------------------------------------
constexpr int kSelThreads = 256;
constexpr int kSelCap = 1024;  // candidates ranked in shared memory
constexpr int kMaxBeam = 16;

struct Cand {
  double s;
  int32_t tok;
  int32_t beam;
};

__device__ __forceinline__ bool better(const Cand& a, const Cand& b) {
  if (a.s != b.s) return a.s > b.s;
  if (a.tok != b.tok) return a.tok < b.tok;
  return a.beam < b.beam;
}

// python list order: lexicographic, a proper prefix sorts first
__device__ bool seq_less(const int32_t* a, int la, const int32_t* b, int lb) {
  int n = la < lb ? la : lb;
  for (int i = 0; i < n; ++i)
    if (a[i] != b[i]) return a[i] < b[i];
  return la < lb;
}

// Stage-2 inputs of one item that do not depend on stage 1 (beam-state
// scalars, cumulative scores, old prefixes and history rows), prefetched by
// every CTA of the fused step at its start so the CTA that ends up running the
// item's stage 2 only has one dependent round trip left (counts, lse and a
// window of each row's candidates). The prefix / history rows only when
// 2 * K * max_len <= kPreCap.
constexpr int kPreCap = 512;
struct Stage2Pre {
  int in[5];  // done, live, step, cur, fin_count
  int rows_ok;
  int64_t top_off;  // the rows' top lists at cand_idx[row * cand_ld + top_off] (0: none)
  int32_t* top_mark;  // per-row top-list counts (-1: none), reset to 0 by stage 2
  // item-cluster variant: the rows' counts, lse and top lists already gathered
  // (tops = the peers' shared-memory top lists through DSMEM)
  int rows_ready;
  int64_t cnt[kMaxBeam];
  double lse[kMaxBeam];
  const int32_t* tops[kMaxBeam];
  double fsc_last;
  double cum[kMaxBeam];
  int32_t ph[kPreCap];  // [K][max_len] prefixes, then [K][max_len] history rows
};
__device__ __forceinline__ void stage2_prefetch(Stage2Pre& p, int b, const fq_beam_state& st,
                                                int K, int max_len, const int32_t* hist,
                                                int cur, int64_t top_off, int32_t* top_mark) {
  const int tid = threadIdx.x;
  const bool rows_ok = 2 * K * max_len <= kPreCap;
  if (tid == 0) {
    p.top_off = top_off;
    p.top_mark = top_mark;
    p.rows_ready = 0;
    p.in[0] = st.done[b];
    p.in[1] = st.live[b];
    p.in[2] = st.step[b];
    p.in[3] = cur;
    p.in[4] = st.fin_count[b];
    p.fsc_last = st.fin_score[b * K + K - 1];
    p.rows_ok = rows_ok ? 1 : 0;
  }
  if (tid < K) p.cum[tid] = st.cum[b * K + tid];
  if (rows_ok) {
    const int64_t row0 = (int64_t)b * K;
    for (int i = tid; i < K * max_len; i += blockDim.x) {
      p.ph[i] = st.prefix[row0 * max_len + i];
      p.ph[K * max_len + i] = hist ? hist[row0 * max_len + i] : 0;
    }
  }
}

// Stage-2 body for item b (one CTA). Candidate lists, counts and lse are read
// with ld.global.cg: in the fused step they were written by other CTAs of the
// same grid (made visible by their fence + the arrival counter).
__device__ __forceinline__ void select_item(
    const int b, const float* __restrict__ logits, int64_t ld, const double* lse,
    const int32_t* cand_idx, int64_t cand_ld, const int64_t* cand_count, fq_beam_state st, int K,
    int max_len, int eos, const double* __restrict__ len_pow, const int32_t* __restrict__ d_cur,
    int64_t max_steps, int64_t* row_tokens, int64_t* row_parents, int32_t* hist,
    const int64_t vals_off = 0, int64_t* tok_sh = nullptr, const Stage2Pre* pre = nullptr) {
  // dynamic smem: old prefixes [K][max_len], old hist [K][max_len], then the
  // candidate array (16-byte aligned)
  extern __shared__ int32_t sh[];
  Cand* cands = reinterpret_cast<Cand*>(sh + ((2 * K * max_len + 3) & ~3));
  __shared__ Cand picks[2 * kMaxBeam];
  __shared__ int64_t offs[kMaxBeam + 1];
  __shared__ int s_new_live, s_done, s_npick;
  __shared__ int new_par[kMaxBeam], new_tok[kMaxBeam];
  __shared__ double new_cum[kMaxBeam];
  __shared__ double red_s[kSelThreads / 32];
  __shared__ int red_t[kSelThreads / 32], red_b[kSelThreads / 32];

  const int tid = threadIdx.x;
  const int64_t row0 = (int64_t)b * K;
  const bool pre_rows = pre && pre->rows_ok;
  int32_t* old_pref = pre_rows ? const_cast<int32_t*>(pre->ph) : sh;
  int32_t* old_hist = old_pref + K * max_len;
  // the rows' top lists [K][kTopSlots] (sweep_row), behind the candidates
  int32_t* win = reinterpret_cast<int32_t*>(cands + kSelCap);
  const bool use_win = pre && (pre->top_off > 0 || pre->rows_ready);
  __shared__ int s_top;  // every live row has a top list: rank only those

  // every input of the item in one round trip: state scalars, per-row counts
  // and lse, old prefixes and whole history rows (no dependency on cur); with
  // `pre` the stage-1-independent ones are already in shared memory and the
  // round trip fetches the counts, lse and each row's first kCandWin
  // candidates (index + logit)
  __shared__ int s_in[5];
  __shared__ int64_t cnt_s[kMaxBeam];
  __shared__ double lse_s[kMaxBeam], cum_s[kMaxBeam];
  __shared__ double s_fsc_last;
  if (pre) {
    if (tid < 5) s_in[tid] = pre->in[tid];
    if (tid == 0) s_fsc_last = pre->fsc_last;
    if (tid < K) {
      cnt_s[tid] = pre->rows_ready ? pre->cnt[tid] : __ldcg(cand_count + row0 + tid);
      lse_s[tid] = pre->rows_ready ? pre->lse[tid] : __ldcg(lse + row0 + tid);
      cum_s[tid] = pre->cum[tid];
    }
    if (pre->rows_ready) {  // the rows' top lists from the item cluster's shared memory
      for (int e = tid; e < K * kTopSlots; e += blockDim.x)
        win[e] = pre->tops[e / kTopSlots][e % kTopSlots];
    } else if (use_win) {
      for (int e = tid; e < K * kTopSlots; e += blockDim.x)
        win[e] = e % kTopSlots ? __ldcg(cand_idx + (row0 + e / kTopSlots) * cand_ld +
                                        pre->top_off + e % kTopSlots)
                               : __ldcg(pre->top_mark + row0 + e / kTopSlots);
    }
    if (!pre_rows) {
      for (int i = tid; i < K * max_len; i += blockDim.x) {
        old_pref[i] = st.prefix[(int64_t)b * K * max_len + i];
        if (hist) old_hist[i] = hist[row0 * max_len + i];
      }
    }
  } else {
  if (tid == 0) {
    s_in[0] = st.done[b];
    s_in[1] = st.live[b];
    s_in[2] = st.step[b];
    s_in[3] = d_cur ? *d_cur : -1;
    s_in[4] = st.fin_count[b];
    s_fsc_last = st.fin_score[b * K + K - 1];
  }
  if (tid < K) {
    cnt_s[tid] = __ldcg(cand_count + row0 + tid);
    lse_s[tid] = __ldcg(lse + row0 + tid);
    cum_s[tid] = st.cum[b * K + tid];
  }
  for (int i = tid; i < K * max_len; i += blockDim.x) {
    old_pref[i] = st.prefix[(int64_t)b * K * max_len + i];
    if (hist) old_hist[i] = hist[row0 * max_len + i];
  }
  }
  __syncthreads();
  if (use_win && !pre->rows_ready && tid < K) pre->top_mark[row0 + tid] = 0;  // self-resetting
  if (s_in[0]) {  // engine.py:148-155: dead rows get parent row0, token 0
    if (tid < K) {
      row_parents[row0 + tid] = row0;
      row_tokens[row0 + tid] = 0;
      if (tok_sh) tok_sh[tid] = 0;
    }
    return;
  }
  const int live = s_in[1];
  const int step = s_in[2];
  const int cur = d_cur ? s_in[3] : step;
  const bool last_step = (int64_t)cur == max_steps - 1;
  if (hist && tid < K && cur < max_len) old_hist[tid * max_len + cur] = (int32_t)(row0 + tid);
  if (tid == 0) {
    int top = use_win ? 1 : 0;
    for (int i = 0; i < live; ++i) top &= win[i * kTopSlots] >= 0 ? 1 : 0;
    s_top = top;
    offs[0] = 0;
    // a row contributes at most K + live picks: its best K + live suffice
    for (int i = 0; i < live; ++i)
      offs[i + 1] = offs[i] + (top ? min(win[i * kTopSlots], K + live) : cnt_s[i]);
  }
  __syncthreads();
  const int64_t n_total = offs[live];
  const int need = (int)(((int64_t)K + live) < n_total ? ((int64_t)K + live) : n_total);
  sw_stamp(blockIdx.x, 5);

  auto cand_at = [&](int64_t j) -> Cand {
    int i = 0;
    while (offs[i + 1] <= j) ++i;
    const int64_t r = row0 + i;
    const int64_t jj = j - offs[i];
    if (s_top) {  // the row's top list, fetched with the counts
      Cand c;
      c.tok = win[i * kTopSlots + 1 + jj];
      c.s = cum_s[i] + ((double)__int_as_float(win[i * kTopSlots + 1 + kTopC + jj]) - lse_s[i]);
      c.beam = i;
      return c;
    }
    const int32_t tok = __ldcg(cand_idx + r * cand_ld + jj);
    // candidate logit stored beside the index by the fused stage 1 (one round trip)
    const double lg = (vals_off && cnt_s[i] <= vals_off)
                          ? (double)__int_as_float(__ldcg(cand_idx + r * cand_ld + vals_off + jj))
                          : (double)logits[r * ld + tok];
    Cand c;
    c.s = cum_s[i] + (lg - lse_s[i]);  // decode.py:238
    c.tok = tok;
    c.beam = i;
    return c;
  };

  if (n_total <= kSelCap) {
    for (int64_t j = tid; j < n_total; j += blockDim.x) cands[j] = cand_at(j);
    __syncthreads();
    // rank of each candidate under (-score, token, beam): 4 threads per
    // candidate, each counting the better ones among a quarter of the list
    // (the quarter counts summed over the 4 lanes); the top `need` are picks
    const int n = (int)n_total;
    const int sub = tid & 3;
    for (int j0 = 0; j0 < n; j0 += (int)(blockDim.x >> 2)) {
      const int j = j0 + (tid >> 2);
      int rank = 0;
      Cand c;
      if (j < n) {
        c = cands[j];
        for (int i = sub; i < n; i += 4) rank += better(cands[i], c) ? 1 : 0;
      }
      rank += __shfl_xor_sync(0xffffffffu, rank, 1);
      rank += __shfl_xor_sync(0xffffffffu, rank, 2);
      if (j < n && sub == 0 && rank < need) picks[rank] = c;
    }
  } else {
    // overflow (tie-heavy rows, exhaustive mode): `need` block-wide arg-best sweeps
    const int lane = tid & 31, w = tid >> 5;
    for (int p = 0; p < need; ++p) {
      Cand best;
      best.s = -INFINITY; best.tok = 0x7fffffff; best.beam = 0x7fffffff;
      bool have = false;
      const Cand prev = p ? picks[p - 1] : best;
      for (int64_t j = tid; j < n_total; j += blockDim.x) {
        Cand c = cand_at(j);
        if (p && !better(prev, c)) continue;  // already picked
        if (!have || better(c, best)) { best = c; have = true; }
      }
      for (int o = 16; o > 0; o >>= 1) {
        Cand other;
        other.s = __shfl_xor_sync(0xffffffffu, best.s, o);
        other.tok = __shfl_xor_sync(0xffffffffu, best.tok, o);
        other.beam = __shfl_xor_sync(0xffffffffu, best.beam, o);
        if (better(other, best)) best = other;
      }
      if (lane == 0) { red_s[w] = best.s; red_t[w] = best.tok; red_b[w] = best.beam; }
      __syncthreads();
      if (tid == 0) {
        Cand bb; bb.s = red_s[0]; bb.tok = red_t[0]; bb.beam = red_b[0];
        for (int i = 1; i < (int)(blockDim.x >> 5); ++i) {
          Cand o; o.s = red_s[i]; o.tok = red_t[i]; o.beam = red_b[i];
          if (better(o, bb)) bb = o;
        }
        picks[p] = bb;
      }
      __syncthreads();
    }
  }
  __syncthreads();
  sw_stamp(blockIdx.x, 6);

  // ---- selection walk, decode.py:192-214 (single thread; <= 2K picks) ----
  if (tid == 0) {
    int nl = 0;
    const int length = step + 1;
    int32_t* ftok = st.fin_tok + (int64_t)b * K * max_len;
    int32_t* flen = st.fin_len + b * K;
    double* fsc = st.fin_score + b * K;
    int fc = s_in[4];
    bool eos_in = false;  // finished list changed this step (else fsc[K-1] preloaded)
    for (int p = 0; p < need; ++p) {
      const Cand c = picks[p];
      if (c.tok == eos) {
        const double sc = len_pow ? c.s / len_pow[length] : c.s;  // decode.py:203
        const int32_t* par = old_pref + c.beam * max_len;  // seq = prefix + [eos]
        // insertion point under key (-score, seq)
        int pos = 0;
        while (pos < fc) {
          bool before;
          if (fsc[pos] != sc) before = fsc[pos] > sc;
          else {
            // compare seq_pos with new seq (par[0:step] + eos)
            const int32_t* e = ftok + pos * max_len;
            int le = flen[pos], n = le < length ? le : length, i = 0;
            before = false;
            bool decided = false;
            for (; i < n; ++i) {
              int32_t nv = i < step ? par[i] : eos;
              if (e[i] != nv) { before = e[i] < nv; decided = true; break; }
            }
            if (!decided) before = le < length;
          }
          if (!before) break;
          ++pos;
        }
        if (pos < K) {
          int last = fc < K ? fc : K - 1;  // shift [pos, last) down by one
          for (int q = last; q > pos; --q) {
            for (int i = 0; i < flen[q - 1]; ++i) ftok[q * max_len + i] = ftok[(q - 1) * max_len + i];
            flen[q] = flen[q - 1];
            fsc[q] = fsc[q - 1];
          }
          for (int i = 0; i < step; ++i) ftok[pos * max_len + i] = par[i];
          ftok[pos * max_len + step] = eos;
          flen[pos] = length;
          fsc[pos] = sc;
          eos_in = true;
          if (fc < K) ++fc;
        }
      } else if (nl < K) {
        new_par[nl] = c.beam;
        new_tok[nl] = c.tok;
        new_cum[nl] = c.s;
        ++nl;
      }
      if (nl >= K) break;
    }
    st.fin_count[b] = fc;
    // should_stop, decode.py:160-171, and the engine's stop rule (engine.py:164)
    bool stop;
    if (nl == 0) stop = true;
    else if (fc < K) stop = false;
    else {
      double best = new_cum[0];
      for (int i = 1; i < nl; ++i) best = fmax(best, new_cum[i]);
      if (len_pow) best = best / len_pow[max(step + 1, 1)];  // decode.py:170
      stop = best <= (eos_in ? fsc[K - 1] : s_fsc_last);
    }
    const int done = (stop || last_step || nl == 0) ? 1 : 0;
    s_new_live = nl;
    s_done = done;
    st.live[b] = nl;
    st.step[b] = step + 1;
    st.done[b] = done;
    if (done) atomicAdd(st.n_done, 1);
  }
  __syncthreads();
  sw_stamp(blockIdx.x, 7);
  const int nl = s_new_live, done = s_done;
  // new prefixes = parent prefix + token; cum / parents / last tokens
  for (int i = tid; i < nl * (step + 1); i += blockDim.x) {
    int bi = i / (step + 1), t = i % (step + 1);
    st.prefix[((int64_t)b * K + bi) * max_len + t] =
        t < step ? old_pref[new_par[bi] * max_len + t] : new_tok[bi];
  }
  if (tid < K) {
    const bool on = tid < nl;
    if (on) {
      st.cum[b * K + tid] = new_cum[tid];
      st.parent[b * K + tid] = new_par[tid];
      st.last_tok[b * K + tid] = new_tok[tid];
    }
    const bool feed = on && !done;
    row_parents[row0 + tid] = feed ? row0 + new_par[tid] : row0;
    row_tokens[row0 + tid] = feed ? new_tok[tid] : 0;
    if (tok_sh) tok_sh[tid] = feed ? new_tok[tid] : 0;
  }
  // copy-free KV reorder: new history row i = old history of its parent
  if (hist && !done) {
    for (int i = tid; i < nl * (cur + 1); i += blockDim.x) {
      int bi = i / (cur + 1), t = i % (cur + 1);
      hist[(row0 + bi) * max_len + t] = old_hist[new_par[bi] * max_len + t];
    }
  }
}

__global__ void __launch_bounds__(kSelThreads) hars_select_kernel(
    const float* __restrict__ logits, int64_t ld, const double* __restrict__ lse,
    const int32_t* __restrict__ cand_idx, int64_t cand_ld,
    const int64_t* __restrict__ cand_count, fq_beam_state st, int K, int max_len, int eos,
    const double* __restrict__ len_pow, const int32_t* __restrict__ d_cur, int64_t max_steps,
    int64_t* row_tokens, int64_t* row_parents, int32_t* hist) {
  pdl_enter();
  select_item(blockIdx.x, logits, ld, lse, cand_idx, cand_ld, cand_count, st, K, max_len, eos,
              len_pow, d_cur, max_steps, row_tokens, row_parents, hist);
}

// Stage 2 of item b (whole CTA), then the item's rows of the next step's
// decoder input (embed_scale_pos, kernels.py:143-151: fp32 emb * sqrt(d), then
// + PE[cur + 1], two roundings), so the decode step needs no separate
// embedding launch; the last item advances the position. cur0: *d_cur as read
// at kernel start (advanced only after every item passed here).
__device__ __forceinline__ void stage2_and_next(
    const int b, const float* __restrict__ logits, int64_t ld, const double* lse,
    const int32_t* cand_idx, int64_t cand_ld, const int64_t* cand_count, fq_beam_state st,
    int K, int max_len, int eos, const double* __restrict__ len_pow, int32_t* d_cur,
    int64_t max_steps, int64_t* row_tokens, int64_t* row_parents, int32_t* hist,
    const int64_t vals_off, const int cur0, const float* __restrict__ emb, int d,
    float emb_scale, const float* __restrict__ pos, float* __restrict__ x_next,
    h16* __restrict__ x16_next, int batch, int* all_cnt, h16* __restrict__ x16_next_lo = nullptr,
    const Stage2Pre* pre = nullptr) {
  __shared__ int64_t s_tok[kMaxBeam];
  select_item(b, logits, ld, lse, cand_idx, cand_ld, cand_count, st, K, max_len, eos, len_pow,
              d_cur, max_steps, row_tokens, row_parents, hist, vals_off, s_tok, pre);
  __syncthreads();
  sw_stamp(1024 + blockIdx.x, 0);  // stage-2 stamps of the fused step: rows 1024 +
  // next step's embedding of the item's rows (embed_scale_pos, kernels.py:143-151:
  // fp32 emb * sqrt(d), then + PE[cur + 1], two roundings), so the decode step
  // needs no separate embedding launch
  const int nxt = cur0 + 1;
  if (x_next && nxt < max_len) {
    const int d4 = d >> 2;  // d % 4 == 0 (checked on the host)
    for (int idx = threadIdx.x; idx < K * d4; idx += blockDim.x) {
      const int ri = idx / d4, j = 4 * (idx - ri * d4);
      const int64_t r = (int64_t)b * K + ri;
      const float4 e = *reinterpret_cast<const float4*>(emb + s_tok[ri] * d + j);
      const float4 p = *reinterpret_cast<const float4*>(pos + (int64_t)nxt * d + j);
      float4 v;
      v.x = fadd_rn(fmul_rn(e.x, emb_scale), p.x);
      v.y = fadd_rn(fmul_rn(e.y, emb_scale), p.y);
      v.z = fadd_rn(fmul_rn(e.z, emb_scale), p.z);
      v.w = fadd_rn(fmul_rn(e.w, emb_scale), p.w);
      *reinterpret_cast<float4*>(x_next + r * d + j) = v;
      if (x16_next) {  // fp16 copy, or with x16_next_lo the exact mode's pair
        uint2 ph, pl;
        split_xh2(v.x, v.y, ph.x, pl.x);
        split_xh2(v.z, v.w, ph.y, pl.y);
        *reinterpret_cast<uint2*>(x16_next + r * d + j) = ph;
        if (x16_next_lo) *reinterpret_cast<uint2*>(x16_next_lo + r * d + j) = pl;
      }
    }
  }
  __syncthreads();
  sw_stamp(1024 + blockIdx.x, 1);
  if (threadIdx.x == 0) {
    __threadfence();
    if (atomicAdd(all_cnt, 1) == batch - 1) {  // every item read d_cur: advance it
      *all_cnt = 0;
      *d_cur += 1;
    }
  }
}

// ---------------------------------------------------------------------------
// The whole HARS step in one launch (decode step, k = min(K + live, V) <= 32):
// CTA per beam row derives its group count from the beam state
// (decode.py:230), runs the single-sweep stage 1 on its row, and the last CTA
// of each item to finish (arrival counter, self-resetting) runs stage 2 for the
// item; the last item to finish advances the decode position. Replaces
// fq_hars_groups + fq_retrieve + fq_hars_select + fq_step_advance, and lets
// the selection of early items overlap the retrieve of the others.
// ---------------------------------------------------------------------------
__global__ void __launch_bounds__(kRowThreads, kRowMinBlocks) hars_step_kernel(
    const float* __restrict__ logits, int64_t ld, int V, fq_beam_state st, int batch, int K,
    int max_len, int eos, const double* __restrict__ len_pow, int32_t* d_cur, int64_t max_steps,
    double* lse, int32_t* cand_idx, int64_t cand_ld, int64_t* cand_count, int* item_cnt,
    int* all_cnt, int64_t* row_tokens, int64_t* row_parents, int32_t* hist,
    const float* __restrict__ emb, int d, float emb_scale, const float* __restrict__ pos,
    float* __restrict__ x_next, h16* __restrict__ x16_next, h16* __restrict__ x16_next_lo) {
  pdl_enter();
  const int C = (int)cl_nrank(), rank = (int)cl_rank();
  const int64_t row = blockIdx.x / C;
  const int b = (int)(row / K), i = (int)(row % K);
  if (rank == 0) sw_stamp(row, 0);
#ifdef FQ_HARS_STAMPS
  if (g_sw_dbg && threadIdx.x == 0 && rank == 0) {  // SM of the row (phase scripts)
    uint32_t smid;
    asm volatile("mov.u32 %0, %%smid;" : "=r"(smid));
    g_sw_dbg[(1536 + row) * 8] = smid;
  }
#endif
  // the position is only advanced after every item has passed its read below
  const int cur0 = *d_cur;
  const int live = st.live[b];
  const int k = (!st.done[b] && i < live) ? min(K + live, V) : 0;  // hars_groups
  const int64_t vals_off = cand_ld / 2 >= kSwThreads * 2 ? cand_ld / 2 : 0;
  const int64_t top_off =
      (C == 1 && vals_off && vals_off + 2 * kRowThreads <= cand_ld - kTopSlots) ? cand_ld - kTopSlots : 0;
  __shared__ Stage2Pre pre;  // in case this CTA runs the item's stage 2
  stage2_prefetch(pre, b, st, K, max_len, hist, cur0, top_off, item_cnt + batch + 1);
  extern __shared__ __align__(16) float4 sw_ring[];  // aliases stage 2's dynamic smem
  sweep_row<kRowThreads>(logits, ld, V, row, k, nullptr, 0, nullptr, lse, cand_idx, cand_ld,
                         cand_count, sw_ring, C, rank, vals_off,
                         top_off ? cand_idx + row * cand_ld + top_off : nullptr,
                         item_cnt + batch + 1 + row);
  __shared__ int s_last;
  __syncthreads();
  if (threadIdx.x == 0) {
    __threadfence();
    const int prev = atomicAdd(item_cnt + b, 1);
    s_last = prev == K * C - 1;  // every CTA of the item's rows has arrived
    if (s_last) item_cnt[b] = 0;
  }
  __syncthreads();
  if (!s_last) return;
  __threadfence();
  stage2_and_next(b, logits, ld, lse, cand_idx, cand_ld, cand_count, st, K, max_len, eos,
                  len_pow, d_cur, max_steps, row_tokens, row_parents, hist, vals_off, cur0, emb,
                  d, emb_scale, pos, x_next, x16_next, batch, all_cnt, x16_next_lo, &pre);
}

// The fused HARS step with one thread-block cluster per item (cluster = the
// item's K rows, one CTA each): each CTA sweeps its row (stage 1) and keeps its
// count, lse and best-32 top list in shared memory; after a cluster barrier
// the leader (rank 0) reads them through DSMEM (no global arrival counter,
// fence or candidate round trip), runs stage 2 and publishes the new tokens;
// after a second barrier every CTA writes its own row of the next step's
// input, and a third keeps the leader's shared memory alive until read.
__global__ void __launch_bounds__(kRowThreads, kRowMinBlocks) hars_step_item_kernel(
    const float* __restrict__ logits, int64_t ld, int V, fq_beam_state st, int batch, int K,
    int max_len, int eos, const double* __restrict__ len_pow, int32_t* d_cur, int64_t max_steps,
    double* lse, int32_t* cand_idx, int64_t cand_ld, int64_t* cand_count, int* all_cnt,
    int64_t* row_tokens, int64_t* row_parents, int32_t* hist, const float* __restrict__ emb,
    int d, float emb_scale, const float* __restrict__ pos, float* __restrict__ x_next,
    h16* __restrict__ x16_next, h16* __restrict__ x16_next_lo) {
  pdl_enter();
  const int rank = (int)cl_rank();
  const int64_t row = blockIdx.x;
  const int b = (int)(row / K), i = (int)(row % K);
  const int cur0 = *d_cur;
  const int live = st.live[b];
  const int k = (!st.done[b] && i < live) ? min(K + live, V) : 0;  // hars_groups
  extern __shared__ __align__(16) float4 sw_ring[];  // aliases stage 2's dynamic smem
  const int64_t vals_off = cand_ld / 2 >= kSwThreads * 2 ? cand_ld / 2 : 0;
  __shared__ Stage2Pre pre;
  __shared__ int32_t s_top[kTopSlots];
  __shared__ double s_lse;
  __shared__ int64_t s_cnt_row, s_tok[kMaxBeam];
  if (rank == 0) stage2_prefetch(pre, b, st, K, max_len, hist, cur0, 0, nullptr);
  sweep_row<kRowThreads>(logits, ld, V, row, k, nullptr, 0, nullptr, lse, cand_idx, cand_ld,
                         cand_count, sw_ring, 1, 0, vals_off, s_top, &s_top[0]);
  __syncthreads();
  if (threadIdx.x == 0) {  // this thread wrote them (sweep_row's tid 0)
    s_lse = k > 0 ? lse[row] : 0.0;
    s_cnt_row = k > 0 ? cand_count[row] : 0;
  }
  cl_sync_all();  // every row of the item swept
  if (rank == 0) {
    if (threadIdx.x < K) {
      pre.cnt[threadIdx.x] = *peer_ptr(&s_cnt_row, threadIdx.x);
      pre.lse[threadIdx.x] = *peer_ptr(&s_lse, threadIdx.x);
      pre.tops[threadIdx.x] = peer_ptr(&s_top[0], threadIdx.x);
    }
    if (threadIdx.x == 0) pre.rows_ready = 1;
    __syncthreads();
    select_item(b, logits, ld, lse, cand_idx, cand_ld, cand_count, st, K, max_len, eos, len_pow,
                d_cur, max_steps, row_tokens, row_parents, hist, vals_off, s_tok, &pre);
    __syncthreads();
  }
  cl_sync_all();  // the leader's new tokens are published
  // this row of the next step's decoder input (embed_scale_pos, kernels.py:143-151)
  const int nxt = cur0 + 1;
  if (x_next && nxt < max_len) {
    const int64_t tok = *peer_ptr(&s_tok[i], 0);
    const int d4 = d >> 2;
    for (int idx = threadIdx.x; idx < d4; idx += blockDim.x) {
      const int j = 4 * idx;
      const float4 e = *reinterpret_cast<const float4*>(emb + tok * d + j);
      const float4 p = *reinterpret_cast<const float4*>(pos + (int64_t)nxt * d + j);
      float4 v;
      v.x = fadd_rn(fmul_rn(e.x, emb_scale), p.x);
      v.y = fadd_rn(fmul_rn(e.y, emb_scale), p.y);
      v.z = fadd_rn(fmul_rn(e.z, emb_scale), p.z);
      v.w = fadd_rn(fmul_rn(e.w, emb_scale), p.w);
      *reinterpret_cast<float4*>(x_next + row * d + j) = v;
      if (x16_next) {
        uint2 ph, pl;
        split_xh2(v.x, v.y, ph.x, pl.x);
        split_xh2(v.z, v.w, ph.y, pl.y);
        *reinterpret_cast<uint2*>(x16_next + row * d + j) = ph;
        if (x16_next_lo) *reinterpret_cast<uint2*>(x16_next_lo + row * d + j) = pl;
      }
    }
  }
  cl_sync_all();  // peers done reading the leader's tokens
  if (rank == 0 && threadIdx.x == 0) {
    __threadfence();
    if (atomicAdd(all_cnt, 1) == batch - 1) {  // every item read d_cur: advance it
      *all_cnt = 0;
      *d_cur += 1;
    }
  }
}

// The fused HARS step on the balanced split (few rows: rows < 2 x SMs): as
// hars_step_kernel, but stage 1 runs on split_walk; the CTA that completes a
// row arrives at its item, the one completing the item runs stage 2 + the
// next-step embedding. counters: [batch] item, [1] all, [rows] row arrivals.
__global__ void __launch_bounds__(kSwThreads, 4) hars_step_split_kernel(
    const float* __restrict__ logits, int64_t ld, SplitGeom g, fq_beam_state st, int batch, int K,
    int max_len, int eos, const double* __restrict__ len_pow, int32_t* d_cur, int64_t max_steps,
    double* lse, int32_t* cand_idx, int64_t cand_ld, int64_t* cand_count, int* counters,
    int64_t* row_tokens, int64_t* row_parents, int32_t* hist, const float* __restrict__ emb,
    int d, float emb_scale, const float* __restrict__ pos, float* __restrict__ x_next,
    h16* __restrict__ x16_next, h16* __restrict__ x16_next_lo) {
  pdl_enter();
  extern __shared__ __align__(16) float4 sw_ring[];  // also stage 2's dynamic smem
  __shared__ SplitSmem sm;
  __shared__ int s_item_last;
  const int V = (int)(g.nvec * 4);
  const int64_t vals_off = cand_ld / 2 >= kSwThreads * 2 ? cand_ld / 2 : 0;
  const int cur0 = *d_cur;
  int* item_cnt = counters;
  int* all_cnt = counters + batch;
  int* row_ctr = counters + batch + 1;
  split_walk(
      g, logits, ld, cand_idx, cand_ld, row_ctr, 1, true, sw_ring, sm,
      [&](int64_t row) {
        const int b = (int)(row / K), i = (int)(row % K);
        const int live = st.live[b];
        return (!st.done[b] && i < live) ? min(K + live, V) : 0;  // hars_groups
      },
      [&](int64_t row, int k, const float* x, int32_t* crow) {
        finalize_split_row(g, row, k, x, crow, nullptr, 0, nullptr, lse, cand_count, cand_ld,
                           vals_off, sw_ring, sm);
        const int b = (int)(row / K);
        __syncthreads();
        if (threadIdx.x == 0) {
          __threadfence();
          const int prev = atomicAdd(item_cnt + b, 1);
          s_item_last = prev == K - 1;
          if (s_item_last) item_cnt[b] = 0;
        }
        __syncthreads();
        if (s_item_last) {
          __threadfence();
          stage2_and_next(b, logits, ld, lse, cand_idx, cand_ld, cand_count, st, K, max_len, eos,
                          len_pow, d_cur, max_steps, row_tokens, row_parents, hist, vals_off,
                          cur0, emb, d, emb_scale, pos, x_next, x16_next, batch, all_cnt, x16_next_lo);
        }
      });
}

// ---------------------------------------------------------------------------
// HARS from the logits GEMM's statistics (fq_logits_hars): the [rows, V]
// logits were never written. CTA per row: the row's exact group maxima (the
// GEMM's running atomics) give R and M; S = sum_t tsum_t exp(tmax_t - M) in a
// fixed tile order; the survivors (every element >= a bound <= R, recorded by
// the GEMM) filtered at R and ranked by column are exactly the candidates
// x >= R. Then, per item, stage 2 + next-step embedding as fq_hars_step, and
// the item's group counts for the next step's GEMM. Resets the running maxima
// and survivor counts for the next step.
// ---------------------------------------------------------------------------
constexpr int kMergeCap = 2048;
__global__ void __launch_bounds__(kSelThreads) hars_merge_step_kernel(
    int V, fq_beam_state st, int batch, int K, int max_len, int eos,
    const double* __restrict__ len_pow, int32_t* d_cur, int64_t max_steps, int32_t* dk,
    int* gmax, const float* __restrict__ tmax, const double* __restrict__ tsum, int ldt,
    int ntiles, int* sv_cnt, const int2* __restrict__ sv, int sv_cap, double* lse,
    int32_t* cand_idx, int64_t cand_ld, int64_t* cand_count, int* counters, int* d_ovf,
    int64_t* row_tokens, int64_t* row_parents, int32_t* hist, const float* __restrict__ emb,
    int d, float emb_scale, const float* __restrict__ pos, float* __restrict__ x_next,
    h16* __restrict__ x16_next, h16* __restrict__ x16_next_lo) {
  pdl_enter();
  __shared__ int s_idx[kMergeCap];
  __shared__ float s_val[kMergeCap];
  __shared__ float s_R, s_M;
  __shared__ int s_n, s_cnt, s_last, s_total;
  __shared__ double red[kSelThreads / 32];
  __shared__ int s_off[kSelThreads + 1];
  __shared__ int warp_tot[32];
  const int tid = threadIdx.x, lane = tid & 31, w = tid >> 5;
  const int64_t row = blockIdx.x;
  const int b = (int)(row / K);
  sw_stamp(row, 0);
  const int cur0 = *d_cur;
  const int k = dk[row];
  const int64_t vals_off = cand_ld / 2;
  int32_t* crow = cand_idx + row * cand_ld;
  if (k > 0) {
    if (w == 0) {
      const float gv = lane < k ? ord2f(gmax[row * 32 + lane]) : INFINITY;
      gmax[row * 32 + lane] = f2ord(-INFINITY);  // ready for the next step
      const float R = warp_min(gv);
      const float M = warp_max(lane < k ? gv : -INFINITY);
      if (lane == 0) {
        s_R = R;
        s_M = M;
        s_cnt = 0;
      }
    }
    __syncthreads();
    const float R = s_R, M = s_M;
    // tile t (ntiles <= kSelThreads: thread per tile): its survivor count, 0 when
    // the tile's maximum is below R (no candidate there); overflow is fatal
    int my_n = 0;
    double acc = 0.0;
    if (tid < ntiles) {
      const float tm = tmax[row * ldt + tid];
      acc = tsum[row * ldt + tid] * exp((double)tm - (double)M);
      const int c = sv_cnt[row * ldt + tid];
      if (c > sv_cap) atomicAdd(d_ovf, 1);
      my_n = tm >= R ? min(c, sv_cap) : 0;
    }
    const double S = block_sum(acc, red);  // fixed tile order: deterministic
    const int my_off = block_excl_scan(my_n, warp_tot, &s_total);
    s_off[tid] = my_off;
    if (tid == 0) s_off[kSelThreads] = s_total;
    __syncthreads();
    const int n = s_total;
    for (int e = tid; e < n; e += kSelThreads) {
      int lo = 0, hi = ntiles - 1;  // last tile t with s_off[t] <= e
      while (lo < hi) {
        const int mid = (lo + hi + 1) >> 1;
        if (s_off[mid] <= e) lo = mid; else hi = mid - 1;
      }
      const int2 en = sv[((int64_t)row * ldt + lo) * sv_cap + (e - s_off[lo])];
      const float v = __int_as_float(en.y);
      if (v >= R) {
        const int p = atomicAdd(&s_cnt, 1);
        if (p < kMergeCap) { s_idx[p] = en.x; s_val[p] = v; }
      }
    }
    __syncthreads();
    const int c = s_cnt;
    const int cw = min(c, kMergeCap);
    for (int i = tid; i < cw; i += kSelThreads) {
      const int j = s_idx[i];
      int rk = 0;
      for (int q = 0; q < cw; ++q) rk += s_idx[q] < j ? 1 : 0;
      crow[rk] = j;
      if (rk < vals_off) crow[vals_off + rk] = __float_as_int(s_val[i]);
    }
    if (tid == 0) {
      if (c > kMergeCap) atomicAdd(d_ovf, 1);  // tie-heavy row: beyond this path
      cand_count[row] = cw;
      lse[row] = (double)M + log(S);
    }
  } else if (tid == 0) {
    cand_count[row] = 0;
  }
  __syncthreads();
  sw_stamp(row, 1);
  if (tid == 0) {
    __threadfence();
    const int prev = atomicAdd(counters + b, 1);
    s_last = prev == K - 1;
    if (s_last) counters[b] = 0;
  }
  __syncthreads();
  if (!s_last) return;
  __threadfence();
  sw_stamp(row, 2);
  stage2_and_next(b, nullptr, 0, lse, cand_idx, cand_ld, cand_count, st, K, max_len, eos, len_pow,
                  d_cur, max_steps, row_tokens, row_parents, hist, vals_off, cur0, emb, d,
                  emb_scale, pos, x_next, x16_next, batch, counters + batch, x16_next_lo);
  __syncthreads();
  sw_stamp(row, 4);
  if (tid < K) {  // group counts of the item's rows for the next step (decode.py:230)
    const int live = st.live[b];
    dk[(int64_t)b * K + tid] = (!st.done[b] && tid < live) ? min(K + live, V) : 0;
  }
}

__global__ void hars_groups_kernel(fq_beam_state st, int batch, int K, int V, int exhaustive,
                                   int32_t* d_k) {
  pdl_enter();
  int r = blockIdx.x * blockDim.x + threadIdx.x;
  if (r >= batch * K) return;
  int b = r / K, i = r % K;
  int live = st.live[b];
  int g = exhaustive ? V : min(K + live, V);
  d_k[r] = (!st.done[b] && i < live) ? g : 0;
}

__global__ void beam_state_init_kernel(fq_beam_state st, int batch, int K, int max_len) {
  pdl_enter();
  int b = blockIdx.x * blockDim.x + threadIdx.x;
  if (b >= batch) return;
  st.live[b] = 1;  // BeamState(): prefixes [[]], cum [0.0], parents [0]
  st.step[b] = 0;
  st.done[b] = 0;
  st.fin_count[b] = 0;
  for (int i = 0; i < K; ++i) {
    st.cum[b * K + i] = 0.0;
    st.parent[b * K + i] = 0;
    st.last_tok[b * K + i] = 0;
    st.fin_len[b * K + i] = 0;
    st.fin_score[b * K + i] = 0.0;
  }
  if (b == 0) *st.n_done = 0;
}

__global__ void step_advance_kernel(int32_t* d_cur) {
  pdl_enter(); *d_cur += 1; }

}  // namespace fq

using namespace fq;

extern "C" {

static size_t sel_smem(int64_t beam, int64_t max_len) {
  return (size_t)((2 * beam * max_len + 3) & ~3) * sizeof(int32_t) + kSelCap * sizeof(Cand) +
         (size_t)beam * kTopSlots * sizeof(int32_t);
}

// FQ_RETRIEVE_TWO_PASS=1 selects the two-pass kernel for every k (A/B runs).
static bool retrieve_two_pass_forced() {
  static int v = -1;
  if (v < 0) {
    const char* e = getenv("FQ_RETRIEVE_TWO_PASS");
    v = (e && e[0] == '1') ? 1 : 0;
  }
  return v == 1;
}

static int hars_num_sms() {
  static int n = 0;
  if (!n) {
    int dev = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&n, cudaDevAttrMultiProcessorCount, dev);
  }
  return n;
}

// Stage 1 on the balanced split when a CTA per row would stream very long rows
// with few CTAs: V >= 64k, or <= 8 rows (scripts/hars_split_ab.py, graph-timed
// us, CTA-per-row vs split: 250k x 64 rows 201 vs 39, 250k x 1 row 52 vs 19,
// 128k x 128 rows 54 vs 39; but 32k x 32..512 rows 14..28 vs 23..39: the
// split's row merge costs a few dependent L2 round trips per row).
// FQ_HARS_SPLIT=0/1 forces either (A/B runs and tests).
// CTAs (a cluster) per row of the row kernels: the largest power of two <= 8
// with rows * C within one wave of 4 CTAs per SM (partials merged through
// DSMEM); 1 from 296 rows up (the C2 decode step's 512). The fused step and
// fq_retrieve use the same rule, so their logsumexp bits agree.
static int row_cluster(int64_t rows) {
  if (kSwSplit != 1) return kSwSplit;
  static int forced = -1;  // FQ_ROW_C=1|2|4|8 (A/B runs)
  if (forced < 0) {
    const char* e = getenv("FQ_ROW_C");
    forced = e ? atoi(e) : 0;
    if (forced != 1 && forced != 2 && forced != 4 && forced != 8) forced = 0;
  }
  if (forced) return forced;
  int C = 1;
  while (C < 8 && rows * C * 2 <= 4 * (int64_t)hars_num_sms()) C *= 2;
  return C;
}

// FQ_HARS_ITEMCL=0 returns the fused step to the global arrival-counter
// hand-over (A/B runs).
static bool item_cluster_enabled() {
  static int v = -1;
  if (v < 0) {
    const char* e = getenv("FQ_HARS_ITEMCL");
    v = (e && e[0] == '0') ? 0 : 1;
  }
  return v == 1;
}

static bool split_forced() {
  const char* e = getenv("FQ_HARS_SPLIT");
  return e && e[0] == '1';
}

static bool use_split(int64_t rows, int64_t vocab, int64_t cand_ld) {
  if (vocab % 4 != 0 || vocab < 8 * kMinPortion || cand_ld < vocab ||
      rows * (vocab / 4) >= (1ll << 31))
    return false;
  const char* e = getenv("FQ_HARS_SPLIT");
  if (e && e[0] == '0') return false;
  if (e && e[0] == '1') return true;
  return vocab >= 65536 || rows <= 8;
}

// Grid of the balanced split: one resident wave, every portion >= kMinPortion.
static SplitGeom split_geom(const void* kernel, size_t smem, int64_t rows, int64_t vocab,
                            int64_t kmax) {
  static thread_local const void* c_kernel = nullptr;
  static thread_local size_t c_smem = 0;
  static thread_local int c_slots = 0;
  if (c_kernel != kernel || c_smem != smem) {
    int occ = 0;
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, kernel, kSwThreads, smem);
    c_kernel = kernel;
    c_smem = smem;
    c_slots = std::max(1, hars_num_sms()) * std::max(1, occ);
  }
  SplitGeom g;
  g.nvec = vocab / 4;
  g.Q = rows * g.nvec;
  int64_t G = c_slots;
  G = std::min<int64_t>(G, g.Q / (kMinPortion + 1));
  G = std::min<int64_t>(G, (int64_t)(kMaxPortions - 2) * rows);
  G = std::min<int64_t>(G, (int64_t)(2 * kSurvCap / kmax - 2) * rows);  // finalize's table
  G = std::max<int64_t>(1, G);
  g.G = (int)G;
  return g;
}

static size_t split_smem() { return (size_t)kSwP * kSwThreads * sizeof(float4); }

extern "C" int fq_retrieve_debug_timestamps(unsigned long long* p) {
  return cudaMemcpyToSymbol(g_sw_dbg, &p, sizeof(p)) == cudaSuccess ? FQ_OK : FQ_ERR_CUDA;
}

int fq_retrieve(const float* logits, int64_t ld, int64_t rows, int64_t vocab, int64_t k,
                const int32_t* d_k, float* group_max, int64_t gm_ld, float* threshold,
                double* lse, int32_t* cand_idx, int64_t cand_ld, int64_t* cand_count,
                fq_stream_t stream) {
  FQ_CHECK_ARG(logits && lse && cand_idx && cand_count && rows >= 0 && vocab >= 1 &&
                   ld >= vocab && cand_ld >= 1,
               FQ_ERR_DIMENSION, "fq_retrieve: bad args");
  FQ_CHECK_ARG(d_k || (k >= 1 && k <= vocab), FQ_ERR_PARAMETER,
               "group count %lld outside [1, vocab=%lld]", (long long)k, (long long)vocab);
  FQ_CHECK_ARG(!group_max || gm_ld >= (d_k ? vocab : k) || gm_ld >= k, FQ_ERR_DIMENSION,
               "group_max leading dim too small");
  if (rows == 0) return FQ_OK;
  int C = row_cluster(rows);
  if (k >= 1 && k <= 32 && (ld % 4) == 0 && ((uintptr_t)logits & 15) == 0 &&
      !retrieve_two_pass_forced() && use_split(rows, vocab, cand_ld) &&
      (rows < 16 || split_forced())) {
    const size_t smem = split_smem();
    const SplitGeom g = split_geom(reinterpret_cast<const void*>(retrieve_split_kernel), smem,
                                   rows, vocab, k);
    // the low words of cand_count are the rows' arrival counters
    if (cudaMemsetAsync(cand_count, 0, (size_t)rows * sizeof(int64_t), as_stream(stream)) !=
        cudaSuccess)
      return launch_status("fq_retrieve");
    launch_kernel(retrieve_split_kernel, (unsigned)g.G, kSwThreads, smem, as_stream(stream), 1u,
                  logits, ld, g, (int)k, d_k, group_max, gm_ld, threshold, lse, cand_idx, cand_ld,
                  cand_count);
    return launch_status("fq_retrieve");
  }
  if (k >= 1 && k <= 32 && ((uintptr_t)logits & 3) == 0 && !retrieve_two_pass_forced()) {
    launch_kernel(retrieve_sweep_kernel, (unsigned)(rows * C), kRowThreads,
                  (size_t)kSwP * kRowThreads * sizeof(float4), as_stream(stream),
                  (unsigned)C,
                  logits, ld, (int)vocab, (int)k, d_k, group_max, gm_ld, threshold, lse,
                  cand_idx, cand_ld, cand_count);
    return launch_status("fq_retrieve");
  }
  launch_kernel(retrieve_kernel, (unsigned)rows, kRetrieveThreads, 0, as_stream(stream), 1u, 
      logits, ld, (int)vocab, (int)k, d_k, group_max, gm_ld, threshold, lse, cand_idx, cand_ld,
      cand_count);
  return launch_status("fq_retrieve");
}

int fq_hars_select(const float* logits, int64_t ld, const double* lse, const int32_t* cand_idx,
                   int64_t cand_ld, const int64_t* cand_count, fq_beam_state st, int64_t batch,
                   int64_t beam, int64_t vocab, int64_t max_len, int64_t eos,
                   const double* len_pow, const int32_t* d_cur, int64_t max_steps, int64_t* row_tokens,
                   int64_t* row_parents, int32_t* hist, void* workspace, int64_t ws_bytes,
                   fq_stream_t stream) {
  (void)workspace;
  (void)ws_bytes;
  FQ_CHECK_ARG(logits && lse && cand_idx && cand_count && row_tokens && row_parents &&
                   batch > 0 && beam >= 1 && beam <= kMaxBeam && max_len >= 1,
               FQ_ERR_DIMENSION, "fq_hars_select: bad args");
  FQ_CHECK_ARG(cand_ld >= vocab, FQ_ERR_DIMENSION,
               "fq_hars_select needs full candidate rows (cand_ld >= vocab)");
  FQ_CHECK_ARG(eos >= 0 && eos < vocab, FQ_ERR_PARAMETER, "eos token outside vocabulary");
  size_t smem = sel_smem(beam, max_len);
  FQ_CHECK_ARG(smem <= 160 * 1024, FQ_ERR_CAPACITY, "fq_hars_select: max_len too large");
  launch_kernel(hars_select_kernel, (unsigned)batch, kSelThreads, smem, as_stream(stream), 1u, 
      logits, ld, lse, cand_idx, cand_ld, cand_count, st, (int)beam, (int)max_len, (int)eos,
      len_pow, d_cur, max_steps, row_tokens, row_parents, hist);
  return launch_status("fq_hars_select");
}

int fq_hars_step(const float* logits, int64_t ld, fq_beam_state st, int64_t batch, int64_t beam,
                 int64_t vocab, int64_t max_len, int64_t eos, const double* len_pow,
                 int32_t* d_cur, int64_t max_steps, double* lse, int32_t* cand_idx,
                 int64_t cand_ld, int64_t* cand_count, int32_t* counters, int64_t* row_tokens,
                 int64_t* row_parents, int32_t* hist, const float* emb, int64_t d_model,
                 float emb_scale, const float* pos, float* x_next, void* x16_next, void* x16_next_lo,
                 fq_stream_t stream) {
  FQ_CHECK_ARG(logits && lse && cand_idx && cand_count && counters && d_cur && row_tokens &&
                   row_parents && batch > 0 && beam >= 1 && beam <= kMaxBeam && max_len >= 1,
               FQ_ERR_DIMENSION, "fq_hars_step: bad args");
  FQ_CHECK_ARG(2 * beam <= 32 && ld % 4 == 0 && vocab % 4 == 0 && ((uintptr_t)logits & 15) == 0,
               FQ_ERR_PARAMETER, "fq_hars_step: needs 2*beam <= 32 and 16-byte aligned rows");
  FQ_CHECK_ARG(cand_ld >= vocab, FQ_ERR_DIMENSION, "fq_hars_step needs full candidate rows");
  FQ_CHECK_ARG(!x_next || (emb && pos && d_model > 0 && d_model % 4 == 0 &&
                            ((uintptr_t)emb & 15) == 0 && ((uintptr_t)pos & 15) == 0 &&
                            ((uintptr_t)x_next & 15) == 0 &&
                            ((uintptr_t)x16_next & 7) == 0),
               FQ_ERR_DIMENSION,
               "fq_hars_step: next-step embedding needs aligned emb/pos/x and d_model % 4 == 0");
  FQ_CHECK_ARG(eos >= 0 && eos < vocab, FQ_ERR_PARAMETER, "eos token outside vocabulary");
  if (use_split(batch * beam, vocab, cand_ld) && (batch * beam < 16 || split_forced())) {
    const size_t smem = std::max(sel_smem(beam, max_len), split_smem());
    FQ_CHECK_ARG(smem <= 96 * 1024, FQ_ERR_CAPACITY, "fq_hars_step: max_len too large");
    const SplitGeom g = split_geom(reinterpret_cast<const void*>(hars_step_split_kernel), smem,
                                   batch * beam, vocab, std::min<int64_t>(2 * beam, vocab));
    launch_kernel(hars_step_split_kernel, (unsigned)g.G, kSwThreads, smem, as_stream(stream), 1u,
                  logits, ld, g, st, (int)batch, (int)beam, (int)max_len, (int)eos, len_pow, d_cur,
                  max_steps, lse, cand_idx, cand_ld, cand_count, counters, row_tokens,
                  row_parents, hist, x_next ? emb : nullptr, (int)d_model, emb_scale, pos, x_next,
                  reinterpret_cast<fq::h16*>(x16_next), reinterpret_cast<fq::h16*>(x16_next_lo));
    return launch_status("fq_hars_step");
  }
  const size_t smem = std::max(sel_smem(beam, max_len),
                               (size_t)kSwP * kRowThreads * sizeof(float4));
  FQ_CHECK_ARG(smem <= 96 * 1024, FQ_ERR_CAPACITY, "fq_hars_step: max_len too large");
  const int C = row_cluster(batch * beam);
  if (C == 1 && beam <= 8 && item_cluster_enabled()) {
    launch_kernel(hars_step_item_kernel, (unsigned)(batch * beam), kRowThreads, smem,
                  as_stream(stream), (unsigned)beam, logits, ld, (int)vocab, st, (int)batch,
                  (int)beam, (int)max_len, (int)eos, len_pow, d_cur, max_steps, lse, cand_idx,
                  cand_ld, cand_count, counters + batch, row_tokens, row_parents, hist,
                  x_next ? emb : nullptr, (int)d_model, emb_scale, pos, x_next,
                  reinterpret_cast<fq::h16*>(x16_next), reinterpret_cast<fq::h16*>(x16_next_lo));
    return launch_status("fq_hars_step");
  }
  launch_kernel(hars_step_kernel, (unsigned)(batch * beam * C), kRowThreads, smem,
                as_stream(stream), (unsigned)C, logits, ld, (int)vocab, st, (int)batch, (int)beam, (int)max_len, (int)eos,
                len_pow, d_cur, max_steps, lse, cand_idx, cand_ld, cand_count, counters,
                counters + batch, row_tokens, row_parents, hist, x_next ? emb : nullptr,
                (int)d_model, emb_scale, pos, x_next,
                reinterpret_cast<fq::h16*>(x16_next), reinterpret_cast<fq::h16*>(x16_next_lo));
  return launch_status("fq_hars_step");
}

int fq_hars_merge_step(fq_beam_state st, int64_t batch, int64_t beam, int64_t vocab,
                       int64_t max_len, int64_t eos, const double* len_pow, int32_t* d_cur,
                       int64_t max_steps, int32_t* dk, int32_t* gmax, const float* tmax,
                       const double* tsum, int64_t ldt, int64_t ntiles, int32_t* sv_cnt,
                       const void* sv, int64_t sv_cap, double* lse, int32_t* cand_idx,
                       int64_t cand_ld, int64_t* cand_count, int32_t* counters, int32_t* d_ovf,
                       int64_t* row_tokens, int64_t* row_parents, int32_t* hist,
                       const float* emb, int64_t d_model, float emb_scale, const float* pos,
                       float* x_next, void* x16_next, void* x16_next_lo, fq_stream_t stream) {
  FQ_CHECK_ARG(d_cur && dk && gmax && tmax && tsum && sv_cnt && sv && lse && cand_idx &&
                   cand_count && counters && d_ovf && row_tokens && row_parents && batch > 0 &&
                   beam >= 1 && beam <= kMaxBeam && 2 * beam <= 32 && ntiles <= ldt &&
                   ntiles <= kSelThreads &&
                   cand_ld >= vocab && cand_ld / 2 >= kMergeCap,
               FQ_ERR_DIMENSION, "fq_hars_merge_step: bad args");
  FQ_CHECK_ARG(!x_next || (emb && pos && d_model > 0 && d_model % 4 == 0),
               FQ_ERR_DIMENSION, "fq_hars_merge_step: next-step embedding needs emb/pos");
  const size_t smem = sel_smem(beam, max_len);
  FQ_CHECK_ARG(smem <= 96 * 1024, FQ_ERR_CAPACITY, "fq_hars_merge_step: max_len too large");
  launch_kernel(hars_merge_step_kernel, (unsigned)(batch * beam), kSelThreads, smem,
                as_stream(stream), 1u, (int)vocab, st, (int)batch, (int)beam, (int)max_len,
                (int)eos, len_pow, d_cur, max_steps, dk, gmax, tmax, tsum, (int)ldt, (int)ntiles,
                sv_cnt, reinterpret_cast<const int2*>(sv), (int)sv_cap, lse, cand_idx, cand_ld,
                cand_count, counters, d_ovf, row_tokens, row_parents, hist,
                x_next ? emb : nullptr, (int)d_model, emb_scale, pos, x_next,
                reinterpret_cast<fq::h16*>(x16_next), reinterpret_cast<fq::h16*>(x16_next_lo));
  return launch_status("fq_hars_merge_step");
}

int fq_hars_groups(fq_beam_state st, int64_t batch, int64_t beam, int64_t vocab, int exhaustive,
                   int32_t* d_k, fq_stream_t stream) {
  FQ_CHECK_ARG(d_k && batch > 0 && beam > 0, FQ_ERR_DIMENSION, "fq_hars_groups: bad args");
  int64_t n = batch * beam;
  launch_kernel(hars_groups_kernel, (unsigned)((n + 255) / 256), 256, 0, as_stream(stream), 1u, 
      st, (int)batch, (int)beam, (int)vocab, exhaustive, d_k);
  return launch_status("fq_hars_groups");
}

int fq_beam_state_init(fq_beam_state st, int64_t batch, int64_t beam, int64_t max_len,
                       fq_stream_t stream) {
  FQ_CHECK_ARG(batch > 0 && beam > 0 && beam <= kMaxBeam, FQ_ERR_DIMENSION,
               "fq_beam_state_init: bad args");
  (void)max_len;
  launch_kernel(beam_state_init_kernel, (unsigned)((batch + 127) / 128), 128, 0, as_stream(stream), 1u, 
      st, (int)batch, (int)beam, (int)max_len);
  return launch_status("fq_beam_state_init");
}

int fq_hars_prepare(void) {
  if (cudaFuncSetAttribute(hars_select_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                           160 * 1024) != cudaSuccess ||
      cudaFuncSetAttribute(hars_step_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                           96 * 1024) != cudaSuccess ||
      cudaFuncSetAttribute(hars_step_item_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                           96 * 1024) != cudaSuccess ||
      cudaFuncSetAttribute(retrieve_sweep_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                           64 * 1024) != cudaSuccess ||
      cudaFuncSetAttribute(retrieve_split_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                           64 * 1024) != cudaSuccess ||
      cudaFuncSetAttribute(hars_step_split_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                           96 * 1024) != cudaSuccess ||
      cudaFuncSetAttribute(hars_merge_step_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                           96 * 1024) != cudaSuccess) {
    set_error("fq_prepare: cannot opt in to large shared memory (hars)");
    return FQ_ERR_CUDA;
  }
  return FQ_OK;
}

int fq_step_advance(int32_t* d_cur, fq_stream_t stream) {
  FQ_CHECK_ARG(d_cur, FQ_ERR_DIMENSION, "fq_step_advance: null counter");
  launch_kernel(step_advance_kernel, 1, 1, 0, as_stream(stream), 1u, d_cur);
  return launch_status("fq_step_advance");
}

}  // extern "C"
