// NEXT 3: the LM-head contraction z = W h on the tcgen05 tensor cores with the
// online log-softmax in its epilogue, so the [rows, V] logits never reach HBM.
//
// lmhead_fwd — persistent, warp-specialised, one CTA per SM (192 threads):
//   warp 0      TMA producer: 128 x 64 hidden tile (A) + 256 x 64 weight tile (B) per stage,
//               SWIZZLE_128B, into a LM_STAGES-deep shared-memory ring (mbarrier complete_tx);
//   warp 1      owns 512 TMEM columns (two 128 x 256 fp32 accumulators); lane 0 issues
//               tcgen05.mma.cta_group::1.kind::f16 (M=128, N=256, K=16; bf16 in, fp32 out)
//               and tcgen05.commit's the stage back to the producer / the tile to the epilogue;
//   warps 2-5   epilogue: each thread owns one row (TMEM lane), tcgen05.ld's its 256 logits in
//               32-column chunks, folds them into an online (max, sum 2^x) state in log2 units
//               and gathers z[y]; releases the accumulator for the next tile.
// Work item = (row block of 128, group of LM_G vocab tiles); items are rasterised in super-rows
// of LM_RB_SWZ row blocks (vocab groups outer, row blocks inner) so the CTAs running at one
// time share a few hidden blocks and weight groups in L2. Each item writes a per-(row, group)
// partial {max, sum}; lmhead_combine reduces the groups of a row in a fixed order (fp64) and
// writes the same per-row log-prob (fp64) as the logits path, so seq_head runs unchanged.
#include "tc_sm100.cuh"

namespace tba {
namespace {

constexpr int LM_BM = 128, LM_BN = 256, LM_BK = 64, LM_STAGES = 4, LM_G = 4, LM_RB_SWZ = 32;  // defaults (measured)
constexpr int LM_A_BYTES = LM_BM * LM_BK * 2;  // 16 KB
constexpr int LM_B_BYTES = LM_BN * LM_BK * 2;  // 32 KB
constexpr int LM_STAGE_BYTES = LM_A_BYTES + LM_B_BYTES;
constexpr int LM_THREADS = 192;
constexpr uint32_t LM_IDESC = tc_idesc_bf16(LM_BM, LM_BN);
static_assert(LM_BK == TC_BK, "one 128-byte swizzle row per K block");
constexpr size_t LM_SMEM = 1024 + (size_t)LM_STAGES * LM_STAGE_BYTES + 256;
// + the logits-store staging (one-call schedule): per epilogue warp two 32 x 32 fp32 boxes
constexpr int LM_ZSTG_BYTES = 2 * 32 * 32 * 4;
constexpr size_t LM_SMEM_Z = 1024 + (size_t)LM_STAGES * LM_STAGE_BYTES + 1024 + 4 * LM_ZSTG_BYTES;

// The same load multicast to the CTAs of `mask` (same shared offset in each; each destination's
// mbarrier at `bar`'s offset receives the complete_tx).
__device__ __forceinline__ void tma_load_2d_mc(uint32_t dst, const CUtensorMap* map, int x, int y, uint32_t bar,
                                               uint16_t mask, uint64_t pol) {
  asm volatile(
      "cp.async.bulk.tensor.2d.shared::cluster.global.mbarrier::complete_tx::bytes.multicast::cluster"
      ".L2::cache_hint [%0], [%1, {%2, %3}], [%4], %5, %6;" ::"r"(dst),
      "l"(reinterpret_cast<uint64_t>(map)), "r"(x), "r"(y), "r"(bar), "h"(mask), "l"(pol)
      : "memory");
}

// Commit arriving on the barrier at `bar`'s offset in every CTA of `mask`.
__device__ __forceinline__ void umma_commit_mc(uint64_t* bar, uint16_t mask) {
  asm volatile(
      "tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.multicast::cluster.b64 [%0], %1;" ::"r"(
          smem_u32(bar)),
      "h"(mask)
      : "memory");
}

struct LmGrid {
  int64_t rows, V;
  const int* act;    // [units] the row-block units holding a valid row, ascending (lm_compact_units)
  const int* n_act;  // [1] their number
  int n_tiles, n_groups, nkb;
  int G, swz;  // vocab tiles per item, row blocks per raster super-row
  int pol;     // L2 policy bits: 1 = weight loads evict_last, 2 = hidden loads evict_last, 4 = no hint (2-SM)
  float* zst;  // nullable: the fp32 logits are also stored here, row r at zst + r * zst_ld (the one-call
  int64_t zst_ld;  // forward + backward keeps them for its gradient pass instead of recomputing them)
};

// item -> (active unit index, vocab group): super-rows of g.swz active units, groups outer.
__device__ __forceinline__ void lm_item(const LmGrid& g, int nact, int64_t item, int& ui, int& grp) {
  const int64_t per_super = (int64_t)g.swz * g.n_groups;
  const int sup = (int)(item / per_super);
  const int64_t w = item - (int64_t)sup * per_super;
  const int u0 = sup * g.swz;
  const int nu = (nact - u0) < g.swz ? (nact - u0) : g.swz;
  grp = (int)(w / nu);
  ui = u0 + (int)(w % nu);
}

// Does row-block unit `u` (MC row blocks of 128 rows) hold any valid row? Work items of units with
// no valid row (the tail of short responses in ragged batches) are skipped by every role alike.
__device__ __forceinline__ bool lm_unit_active(const uint8_t* __restrict__ mask, int u, int MCu, int64_t rows) {
  const int64_t r0 = (int64_t)u * MCu * LM_BM;
  const int64_t n = (int64_t)MCu * LM_BM;
  const int64_t r1 = r0 + n < rows ? r0 + n : rows;
  if (r1 - r0 == n && (reinterpret_cast<uintptr_t>(mask + r0) & 15) == 0) {
    const uint4* p = reinterpret_cast<const uint4*>(mask + r0);
    uint32_t acc = 0;
    for (int i = 0; i < (int)(n / 16); ++i) {
      const uint4 v = __ldg(p + i);
      acc |= v.x | v.y | v.z | v.w;
    }
    return acc != 0;
  }
  for (int64_t r = r0; r < r1; ++r)
    if (mask[r]) return true;
  return false;
}

// One work item of the epilogue (one row per thread): fold the item's vocabulary tiles into an
// online (reference, sum) state, gather z[y], release each accumulator, write the item partial.
// tempty_addr: the accumulator-empty barriers (shared::cluster address when `cluster_arrive`,
// i.e. the leader CTA's barrier in the 2-SM kernel).
// Per element: one FFMA 2^(z sc - Rs) with Rs = fl(R sc) the exponent reference, one MUFU ex2,
// one FMNMX (chunk max) and the pairwise FADD tree; the vocabulary-tail mask runs only in the
// last tile and the z[y] gather only in the chunk that holds y. The partial is {R, S} with
// S = sum 2^(z sc - fl(R sc)); lmhead_combine re-forms fl(R sc) with the same fp32 multiply.
// NT = 2 (wide pair tiles): one accumulator of 2 x 256 columns holds vocabulary tiles t and t+1;
// it is waited for before the first and released after the second (or after the group's last).
// H = 2 (with NT = 2): two epilogue warps per TMEM lane quarter; warp-half h folds only the tiles
// t0 + h, t0 + h + 2, ... and writes its own partial (group slot grp * 2 + h), so the softmax of
// the two halves of a wide tile runs in parallel; lmhead_combine reduces 2 x n_groups partials.
template <int NT = 1, int H = 1>
__device__ __forceinline__ void lm_epilogue_item(const LmGrid& g, int rb, int grp, uint32_t& j, uint32_t tmem_lane,
                                                 int row_in, int lane, uint64_t* tfull, uint32_t tempty_addr,
                                                 bool cluster_arrive, const int64_t* __restrict__ tokens,
                                                 const RowScale& rs, float2* __restrict__ part,
                                                 float* __restrict__ zy_out, int h = 0,
                                                 const CUtensorMap* zmap = nullptr, uint32_t zstg = 0,
                                                 uint32_t* zcnt = nullptr) {
  const float sc = rs.sc;
  const int t0 = grp * g.G, t1 = min(g.n_tiles, t0 + g.G);
  const int64_t row = (int64_t)rb * LM_BM + row_in;
  const bool in_rows = row < g.rows;
  const int64_t y = in_rows ? tokens[row] : -1;
  float R = -INFINITY;  // reference in logit units (a running max, moved only by > slack)
  float Rs = -INFINITY; // fl(R sc): the exponent reference
  double S = 0.0;       // sum of 2^(z sc - Rs)
  float zy = 0.f;
  bool found = false;
  constexpr int NACC = 2 / NT;
  for (int t = t0; t < t1; ++t) {
    const int u = (t - t0) % NT;  // sub-tile of the accumulator (t0 is a multiple of NT)
    const uint32_t acc = j % NACC, aph = (j / NACC) & 1u;
    if (u == 0) {
      mbar_wait(&tfull[acc], aph);
      tc_fence_after();
    }
    const uint32_t col0 = (acc * NT + u) * LM_BN;
    const int64_t nb = (int64_t)t * LM_BN;
    const bool tail = nb + LM_BN > g.V;          // warp-uniform: only the last vocabulary tile
    const int64_t dyt = y - nb;
    const int cy = ((uint64_t)dyt < (uint64_t)LM_BN) ? (int)(dyt >> 5) : -1;  // chunk holding y, if any
#pragma unroll 1
    for (int c = 0; c < ((H == 1 || u == h) ? LM_BN / 32 : 0); ++c) {
      float v[32];
      tmem_ld32(tmem_lane + col0 + c * 32, v);
      if (zmap) {  // logits store through shared memory + one TMA bulk store per 32 x 32 box
        const uint32_t buf = zstg + (*zcnt & 1u) * (32 * 32 * 4);
        if (*zcnt >= 2 && lane == 0) asm volatile("cp.async.bulk.wait_group.read 1;" ::: "memory");
        __syncwarp();
#pragma unroll
        for (int q4 = 0; q4 < 8; ++q4)  // 16-byte chunk q4 of this row at (q4 ^ row % 8): conflict-free
          asm volatile("st.shared.v4.f32 [%0], {%1, %2, %3, %4};" ::"r"(buf + lane * 128 + ((q4 ^ (lane & 7)) << 4)),
                       "f"(v[4 * q4]), "f"(v[4 * q4 + 1]), "f"(v[4 * q4 + 2]), "f"(v[4 * q4 + 3])
                       : "memory");
        asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
        __syncwarp();
        if (lane == 0) {
          tma_store_2d(zmap, buf, (int)(nb + c * 32), (int)(rb * LM_BM + (row_in & ~31)));
          asm volatile("cp.async.bulk.commit_group;" ::: "memory");
        }
        ++*zcnt;
      } else if (g.zst && in_rows) {
        float* zp = g.zst + row * g.zst_ld + nb + c * 32;
        if (nb + c * 32 + 32 <= g.V) {
#pragma unroll
          for (int u = 0; u < 8; ++u)
            reinterpret_cast<float4*>(zp)[u] = make_float4(v[4 * u], v[4 * u + 1], v[4 * u + 2], v[4 * u + 3]);
        } else {
          for (int i = 0; i < 32; ++i)
            if (nb + c * 32 + i < g.V) zp[i] = v[i];
        }
      }
      if (tail) {
        const int64_t lim = g.V - (nb + c * 32);
#pragma unroll
        for (int i = 0; i < 32; ++i) v[i] = (i < lim) ? v[i] : -INFINITY;
      }
      if (c == cy) {
        const int k = (int)(dyt & 31);
#pragma unroll
        for (int i = 0; i < 32; ++i)
          if (i == k) zy = v[i];
        found = true;
      }
      float m[16];
#pragma unroll
      for (int i = 0; i < 16; ++i) m[i] = fmaxf(v[i], v[i + 16]);
#pragma unroll
      for (int w = 8; w >= 1; w >>= 1)
#pragma unroll
        for (int i = 0; i < w; ++i) m[i] = fmaxf(m[i], m[i + w]);
      const float cm = m[0];
      if (cm > R + rs.slack) {  // re-base (rare): exact fp64 rescale of the running sum
        const float Rs2 = cm * sc;
        S = (R == -INFINITY) ? 0.0 : S * exp2((double)Rs - (double)Rs2);
        R = cm;
        Rs = Rs2;
      }
#pragma unroll
      for (int i = 0; i < 32; ++i) v[i] = ex2(fmaf(v[i], sc, -Rs));
#pragma unroll
      for (int w = 16; w >= 1; w >>= 1)
#pragma unroll
        for (int i = 0; i < w; ++i) v[i] += v[i + w];
      S += (double)v[0];
    }
    if (u == NT - 1 || t + 1 == t1) {
      tc_fence_before();
      __syncwarp();
      if (lane == 0) {
        const uint32_t bar = tempty_addr + acc * 8u;
        if (cluster_arrive)
          asm volatile("mbarrier.arrive.release.cluster.shared::cluster.b64 _, [%0];" ::"r"(bar) : "memory");
        else
          asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(bar) : "memory");
      }
      ++j;
    }
  }
  if (in_rows) {
    part[((int64_t)grp * H + h) * g.rows + row] = make_float2(R, (float)S);
    if (found) zy_out[row] = zy;
  }
}

// MC = 1: one CTA per work item. MC = 2: a cluster of two CTAs takes row blocks 2u and 2u+1 of the
// same vocabulary tiles; each CTA loads half of every weight tile and multicasts it to both, so
// the weight is read from L2 once per pair (1/3 less L2 -> SM traffic). Each CTA's MMA frees a
// stage in both CTAs (multicast commit): a producer refills a stage only when both have used it.
template <int MC>
__global__ void __launch_bounds__(LM_THREADS, 1)
    lmhead_fwd(const __grid_constant__ CUtensorMap tmH, const __grid_constant__ CUtensorMap tmW, LmGrid g,
               const int64_t* __restrict__ tokens, const uint8_t* __restrict__ mask, RowScale rs,
               float2* __restrict__ part, float* __restrict__ zy_out, const __grid_constant__ CUtensorMap tmZ) {
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~(uintptr_t)1023);
  uint8_t* sA = smem;
  uint8_t* sB = smem + LM_STAGES * LM_A_BYTES;
  uint64_t* full = reinterpret_cast<uint64_t*>(smem + LM_STAGES * LM_STAGE_BYTES);
  uint64_t* empty = full + LM_STAGES;
  uint64_t* tfull = empty + LM_STAGES;
  uint64_t* tempty = tfull + 2;
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(tempty + 2);
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const uint32_t crank = MC > 1 ? cluster_ctarank() : 0u;
  const int64_t unit0 = blockIdx.x / MC, n_units = gridDim.x / MC;
  const int nact = *g.n_act;
  const int64_t n_items = (int64_t)nact * g.n_groups;

  if (threadIdx.x == 0) {
    for (int s = 0; s < LM_STAGES; ++s) {
      mbar_init(&full[s], 1);
      mbar_init(&empty[s], MC);
    }
    for (int a = 0; a < 2; ++a) {
      mbar_init(&tfull[a], 1);
      mbar_init(&tempty[a], 4);  // one arrive per epilogue warp
    }
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
  }
  if (warp == 1) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 512;" ::"r"(smem_u32(tmem_slot))
                 : "memory");
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;" ::: "memory");
  }
  tc_fence_before();
  __syncthreads();
  if (MC > 1) cluster_sync_all();  // the partner's barriers are initialised before any remote arrive
  tc_fence_after();
  const uint32_t tmem = *tmem_slot;

  if (warp == 0) {
    if (lane == 0) {  // ---- TMA producer
      asm volatile("prefetch.tensormap [%0];" ::"l"(reinterpret_cast<uint64_t>(&tmH)) : "memory");
      asm volatile("prefetch.tensormap [%0];" ::"l"(reinterpret_cast<uint64_t>(&tmW)) : "memory");
      const uint64_t pol_w = l2_policy(g.pol & 1), pol_h = l2_policy(g.pol & 2);
      int stage = 0;
      uint32_t phase = 0;
      for (int64_t it = unit0; it < n_items; it += n_units) {
        int rb, grp;
        lm_item(g, nact, it, rb, grp);
        rb = g.act[rb];
        rb = rb * MC + (int)crank;
        const int t0 = grp * g.G, t1 = min(g.n_tiles, t0 + g.G);
        for (int t = t0; t < t1; ++t) {
          for (int kb = 0; kb < g.nkb; ++kb) {
            mbar_wait(&empty[stage], phase ^ 1u);
            mbar_expect_tx(&full[stage], LM_STAGE_BYTES);
            tma_load_2d(smem_u32(sA + stage * LM_A_BYTES), &tmH, kb * LM_BK, rb * LM_BM, smem_u32(&full[stage]),
                        pol_h);
            if (MC == 1)
              tma_load_2d(smem_u32(sB + stage * LM_B_BYTES), &tmW, kb * LM_BK, t * LM_BN, smem_u32(&full[stage]),
                          pol_w);
            else
              tma_load_2d_mc(smem_u32(sB + stage * LM_B_BYTES + crank * (LM_B_BYTES / MC)), &tmW, kb * LM_BK,
                             t * LM_BN + (int)crank * (LM_BN / MC), smem_u32(&full[stage]), (uint16_t)((1u << MC) - 1),
                             pol_w);
            if (++stage == LM_STAGES) {
              stage = 0;
              phase ^= 1u;
            }
          }
        }
      }
    }
  } else if (warp == 1) {
    if (lane == 0) {  // ---- MMA issuer
      int stage = 0;
      uint32_t phase = 0;
      uint32_t j = 0;  // accumulator tile counter
      for (int64_t it = unit0; it < n_items; it += n_units) {
        int rb, grp;
        lm_item(g, nact, it, rb, grp);
        rb = g.act[rb];
        rb = rb * MC + (int)crank;
        const int t0 = grp * g.G, t1 = min(g.n_tiles, t0 + g.G);
        for (int t = t0; t < t1; ++t, ++j) {
          const uint32_t acc = j & 1u, aph = (j >> 1) & 1u;
          mbar_wait(&tempty[acc], aph ^ 1u);
          tc_fence_after();
          const uint32_t d_tmem = tmem + acc * LM_BN;
          for (int kb = 0; kb < g.nkb; ++kb) {
            mbar_wait(&full[stage], phase);
            tc_fence_after();
            const uint64_t a0 = umma_desc_sw128(smem_u32(sA + stage * LM_A_BYTES));
            const uint64_t b0 = umma_desc_sw128(smem_u32(sB + stage * LM_B_BYTES));
#pragma unroll
            for (int k = 0; k < LM_BK / 16; ++k)  // K = 16 per MMA: +32 bytes = +2 in the address field
              umma_bf16<LM_IDESC>(d_tmem, a0 + 2u * k, b0 + 2u * k, (kb | k) != 0);
            if (MC == 1) umma_commit(&empty[stage]);
            else umma_commit_mc(&empty[stage], (uint16_t)((1u << MC) - 1));
            if (++stage == LM_STAGES) {
              stage = 0;
              phase ^= 1u;
            }
          }
          umma_commit(&tfull[acc]);
        }
      }
    }
  } else {  // ---- epilogue: warps 2..5 own TMEM lane quarters (warp % 4)
    const int q = warp & 3;
    const int row_in = q * 32 + lane;
    const uint32_t lane_addr = (uint32_t)(q * 32) << 16;
    uint32_t j = 0;
    // one-call schedule: the logits go out through per-warp staging boxes and TMA stores
    const bool zt = g.zst != nullptr && MC == 1;
    const uint32_t zstg = smem_u32(smem + LM_STAGES * LM_STAGE_BYTES + 1024) + (uint32_t)q * LM_ZSTG_BYTES;
    uint32_t zcnt = 0;
    for (int64_t it = unit0; it < n_items; it += n_units) {
      int rb, grp;
      lm_item(g, nact, it, rb, grp);
      rb = g.act[rb];
      rb = rb * MC + (int)crank;
      lm_epilogue_item(g, rb, grp, j, tmem + lane_addr, row_in, lane, tfull, smem_u32(tempty), false, tokens, rs,
                       part, zy_out, 0, zt ? &tmZ : nullptr, zstg, &zcnt);
    }
    if (zt && lane == 0) asm volatile("cp.async.bulk.wait_group 0;" ::: "memory");
  }
  __syncthreads();
  if (MC > 1) cluster_sync_all();  // no CTA leaves while its partner may still write into it
  if (warp == 1) {
    tc_fence_after();
    asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 512;" ::"r"(tmem) : "memory");
  }
}

// Ordered list of the row-block units (MCu row blocks of 128 rows) that hold a valid row: one
// CTA, chunks of 1024 units, ballot + warp-total scan. Masked tails of short responses then cost
// no GEMM work and the persistent CTAs stay balanced over the units that remain.
__global__ void __launch_bounds__(1024) lm_compact_units(const uint8_t* __restrict__ mask, int64_t rows, int MCu,
                                                          int n_units, int* __restrict__ act, int* __restrict__ n_act) {
  __shared__ int warp_tot[32];
  __shared__ int base;
  const int tid = threadIdx.x, lane = tid & 31, wid = tid >> 5;
  if (tid == 0) base = 0;
  __syncthreads();
  for (int c0 = 0; c0 < n_units; c0 += 1024) {
    const int u = c0 + tid;
    const bool a = u < n_units && lm_unit_active(mask, u, MCu, rows);
    const unsigned bal = __ballot_sync(0xffffffffu, a);
    if (lane == 0) warp_tot[wid] = __popc(bal);
    __syncthreads();
    int off = 0;
    for (int w = 0; w < wid; ++w) off += warp_tot[w];
    if (a) act[base + off + __popc(bal & ((1u << lane) - 1u))] = u;
    __syncthreads();
    if (tid == 0) {
      int tot = 0;
      for (int w = 0; w < 32; ++w) tot += warp_tot[w];
      base += tot;
    }
    __syncthreads();
  }
  if (tid == 0) *n_act = base;
}

// Per valid row: fixed-order fp64 reduction of the group partials, then the same stats / log-prob
// outputs as the logits path (finalize_row's contract): stats = {M2, log2 S}, lp fp64.
__global__ void lmhead_combine(const float2* __restrict__ part, const float* __restrict__ zy_in, int64_t rows,
                               int n_groups, int64_t V, const int64_t* __restrict__ tokens,
                               const uint8_t* __restrict__ mask, RowScale rs, float2* __restrict__ stats,
                               double* __restrict__ lp, int32_t* dev_status) {
  for (int64_t r = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; r < rows; r += (int64_t)gridDim.x * blockDim.x) {
    if (!mask[r]) continue;
    float M = -INFINITY;  // logit units
    for (int k = 0; k < n_groups; ++k) M = fmaxf(M, part[(int64_t)k * rows + r].x);
    // sum over the vocabulary of 2^((z - M) sc): group k's sum is relative to fl(R_k sc) (the
    // kernel's fp32 product, re-formed identically here); M sc is exact in fp64
    const double Msc = (double)M * (double)rs.sc;
    double S = 0.0;
    for (int k = 0; k < n_groups; ++k) {
      const float2 p = part[(int64_t)k * rows + r];
      S += (double)p.y * exp2((double)(p.x * rs.sc) - Msc);
    }
    const double l2s = log2(S);
    const int64_t y = tokens[r];
    double out;
    if (y < 0 || y >= V) {
      out = __longlong_as_double(0x7ff8000000000000ll);
      if (dev_status) atomicOr(dev_status, TBA_DEV_TOKEN_RANGE);
    } else {
      // log softmax(inv_temp z)[y] = inv_temp (z_y - M) - ln 2 log2 sum 2^((z - M) sc)
      out = rs.inv_temp * ((double)zy_in[r] - (double)M) - kLN2 * l2s;
    }
    if (!(isfinite(M) && isfinite(l2s))) {
      out = __longlong_as_double(0x7ff8000000000000ll);
      if (dev_status) atomicOr(dev_status, TBA_DEV_NONFINITE_ROW);
    }
    // row statistics in the logits path's convention: M2 = M sc (log2 units), log2 S
    stats[r] = make_float2((float)((double)M * (double)rs.sc), (float)l2s);
    lp[r] = out;
  }
}

}  // namespace

size_t lmhead_partial_bytes(int64_t rows, int64_t V) {
  const int64_t groups = ((V + LM_BN - 1) / LM_BN + LM_G - 1) / LM_G;
  const int64_t blocks = (rows + LM_BM - 1) / LM_BM;
  return align_up((size_t)groups * (size_t)rows * sizeof(float2), 256) + align_up((size_t)rows * sizeof(float), 256) +
         align_up((size_t)(blocks + 1) * sizeof(int), 256);
}

int launch_lmhead_rows(const tba_lmhead* x, void* part_ws, const WsLayout& w, const RowScale& rs, int32_t* dev_status,
                       cudaStream_t s, float* zst, int64_t zst_ld) {
  const int64_t rows = x->n_seq * x->seq_len;
  if (rows == 0) return TBA_OK;
  constexpr int mc = 1;  // one CTA per work item (the cluster / cta_group::2 variants measured slower)
  const int n_rb = (int)((rows + LM_BM - 1) / LM_BM);
  const int n_units_total = (n_rb + mc - 1) / mc;  // row-block units (pairs when mc = 2)
  LmGrid g;
  g.rows = rows;
  g.V = x->vocab;
  g.n_tiles = (int)((x->vocab + LM_BN - 1) / LM_BN);
  g.G = LM_G;
  g.swz = LM_RB_SWZ;
  g.pol = 1;  // weight tiles evict_last (54.4-55.5 vs 62-63 ms with evict_normal)
  g.n_groups = (g.n_tiles + g.G - 1) / g.G;
  g.nkb = (int)((x->d + LM_BK - 1) / LM_BK);
  g.zst = zst;
  g.zst_ld = zst_ld;
  CUtensorMap mh, mw, mz;
  if (!make_map(&mh, x->hidden, rows, x->d, x->hidden_stride, LM_BM) ||
      !make_map(&mw, x->weight, x->vocab, x->d, x->weight_stride, LM_BN / mc))
    return TBA_ERR_CUDA;
  const bool ztma = zst != nullptr;  // the logits store goes out through TMA
  if (ztma ? !make_store_map_f32(&mz, zst, rows, x->vocab, zst_ld) : false) return TBA_ERR_CUDA;
  if (!ztma) mz = CUtensorMap{};
  char* pw = static_cast<char*>(part_ws);
  float2* part = reinterpret_cast<float2*>(pw);
  pw += align_up((size_t)g.n_groups * (size_t)rows * sizeof(float2), 256);
  float* zy = reinterpret_cast<float*>(pw);
  pw += align_up((size_t)rows * sizeof(float), 256);
  int* act = reinterpret_cast<int*>(pw);
  g.act = act;
  g.n_act = act + n_rb;
  lm_compact_units<<<1, 1024, 0, s>>>(x->mask, rows, mc, n_units_total, act, act + n_rb);
  if (cudaGetLastError() != cudaSuccess) return TBA_ERR_CUDA;
  static bool attr[64] = {};  // per device; benign race: idempotent
  int dev = 0;
  if (cudaGetDevice(&dev) != cudaSuccess || dev < 0 || dev >= 64) return TBA_ERR_CUDA;
  auto kern = lmhead_fwd<1>;
  const size_t smem = ztma ? LM_SMEM_Z : LM_SMEM;
  if (!attr[dev]) {
    if (cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)LM_SMEM_Z) != cudaSuccess)
      return TBA_ERR_CUDA;
    attr[dev] = true;
  }
  cudaLaunchConfig_t cfg = {};
  cfg.blockDim = dim3(LM_THREADS);
  cfg.dynamicSmemBytes = smem;
  cfg.stream = s;
  int64_t units = device_sms();
  const int64_t max_items = (int64_t)n_units_total * g.n_groups;  // the active count is known on the device only
  if (units > max_items) units = max_items;
  cfg.gridDim = dim3((unsigned)(units * mc));
  if (cudaLaunchKernelEx(&cfg, kern, mh, mw, g, x->tokens, x->mask, rs, part, zy, mz) != cudaSuccess)
    return TBA_ERR_CUDA;
  const int64_t blocks = (rows + 255) / 256 < 4096 ? (rows + 255) / 256 : 4096;
  lmhead_combine<<<(unsigned)blocks, 256, 0, s>>>(part, zy, rows, g.n_groups, x->vocab, x->tokens, x->mask, rs,
                                                  w.stats, w.lp, dev_status);
  return launch_status();
}

}  // namespace tba
