// NEXT 3, backward through the LM head: dL/dh and dL/dW for z = W h without
// materialising the [rows, V] logits or dlogits of the whole batch.
//
// App. A gives dL/dz_{r,v} = c_r (1[v = y_r] - softmax(inv_temp z_r)_v) with the
// per-row coefficient c_r = grad_scale * g * inv_temp * eps_s (TB, Eqs. 3-5) or
// grad_scale * g * coef_r (TBA', Eq. 16); the chain rule through z = W h gives
//   dL/dh_r = sum_v dz_{r,v} W_v        (dH = dZ W)
//   dL/dW_v = sum_r dz_{r,v} h_r        (dW = dZ^T H)
// The valid rows are processed in chunks of C rows (compacted: masked rows have dz = 0 and are
// never computed). Per chunk, all on the tcgen05 tensor cores with one persistent kernel shape:
//   1. lmb_gather_t   H rows of the chunk -> Hc [C, d] and Hc^T [d, C]            (bf16 copy)
//   2. tc_gemm<DZ>    z = Hc W^T recomputed tile by tile in TMEM; the epilogue forms dz from
//                     the forward's row statistics and writes it as bf16 to dZ [C, Vp] and
//                     dZ^T [V, C] (the logits themselves never reach HBM)
//   3. tc_gemm<STORE> dH rows = dZ (W^T)^T, scattered to the rows' places in dhidden
//   4. tc_gemm<STORE> dW (+)= dZ^T (Hc^T)^T, fp32, accumulated over the chunks
// W^T [d, Vp] is formed once per call. Every GEMM is D = A B^T with both operands K-major
// (TMA SWIZZLE_128B tiles, UMMA K = 16, fp32 accumulators in TMEM), so the transposed copies are
// what lets one mainloop serve all three products. dH and dW run by default on tc_gemm2<2>, the
// cta_group::2 form with 256 x 512 tiles per SM pair (half the single-SM kernel's L2 -> SM feed).
// The one-call schedule (launch_lmhead_fwd_bwd) takes chunks of whole groups: the forward stores
// the chunk's fp32 logits and lmb_dz_from_z replaces step 2's recompute GEMM.
#include <cmath>

#include "tc_sm100.cuh"

namespace tba {
namespace {

constexpr int GB_BM = 128, GB_BN = 256, GB_STAGES = 4, GB_THREADS = 192;
constexpr int GB_A_BYTES = GB_BM * TC_BK * 2;  // 16 KB
constexpr int GB_B_BYTES = GB_BN * TC_BK * 2;  // 32 KB
constexpr int GB_STAGE_BYTES = GB_A_BYTES + GB_B_BYTES;
constexpr uint32_t GB_IDESC = tc_idesc_bf16(GB_BM, GB_BN);
constexpr size_t GB_SMEM = 1024 + (size_t)GB_STAGES * GB_STAGE_BYTES + 256;
constexpr int64_t LMB_DEFAULT_CHUNK = 16384;

enum { EPI_DZ = 0, EPI_STORE = 1 };

// dz epilogue: the chunk's rows i -> batch rows idx[chunk0 + i]
struct DzArgs {
  const int* idx;
  const float2* stats;    // forward row statistics {M2 = M sc, log2 S}
  const int64_t* tokens;
  const double* resid;    // per sequence (TB) or nullptr
  const float* coef;      // per row (TBA') or nullptr
  int64_t T;
  double gs;              // grad_scale * inv_temp (TB) or grad_scale (TBA'), times *grad_out
  const double* grad_out;
  float sc;               // fl(log2(e) inv_temp)
  int64_t V, Vp, C;
  uint16_t* dz;           // [C, Vp]
  uint16_t* dzt;          // [V, C]
};

struct StoreArgs {
  void* D;
  int64_t ldd;
  const int* row_map;  // nullable: output row of tile row m = row_map[m]
  int out_bf16, add, vec;
};

struct GemmArgs {
  int64_t M, N, K;     // static extents; dyn = 1: M := the chunk's count, dyn = 2: K := the chunk's count
  const int* n_valid;  // device count of valid rows (dyn != 0)
  int64_t chunk0, cap;
  int dyn, swz, n_inner;
  int pol;             // bit 0: A loads evict_last, bit 1: B loads evict_last
  DzArgs dz;
  StoreArgs st;
  int ksplit;          // tc_gemm2 only: > 1 splits K into ksplit slices; slice sl of tile (m, n) stores
  float* part;         // its fp32 partial at part[(sl * cap + m) * part_ld + n] (lmb_splitk_reduce sums them)
  int64_t part_ld;
};

__device__ __forceinline__ int64_t chunk_count(const int* n_valid, int64_t chunk0, int64_t cap) {
  const int64_t n = (int64_t)*n_valid - chunk0;
  return n < 0 ? 0 : (n > cap ? cap : n);
}

struct Tiles {
  int64_t n_mt, n_nt, nkb;
  int swz, n_inner;
};

// tile t -> (mb, nb). n_inner: consecutive tiles share the m block (all N tiles of a row block
// are in flight together; the A slice is fetched once). Otherwise super-rows of swz m blocks,
// n outer, m inner (consecutive CTAs share the B tile).
__device__ __forceinline__ void tile_of(const Tiles& g, int64_t t, int64_t& mb, int64_t& nb) {
  if (g.n_inner) {
    mb = t / g.n_nt;
    nb = t - mb * g.n_nt;
    return;
  }
  const int64_t per = (int64_t)g.swz * g.n_nt;
  const int64_t sup = t / per, w = t - sup * per;
  const int64_t m0 = sup * g.swz;
  const int64_t nm = (g.n_mt - m0) < g.swz ? (g.n_mt - m0) : g.swz;
  nb = w / nm;
  mb = m0 + (w - nb * nm);
}

__device__ __forceinline__ void store_bf16x32(uint16_t* p, const float (&d)[32]) {
  uint4* q = reinterpret_cast<uint4*>(p);
#pragma unroll
  for (int u = 0; u < 4; ++u)
    q[u] = make_uint4(pack_bf16x2(d[8 * u + 0], d[8 * u + 1]), pack_bf16x2(d[8 * u + 2], d[8 * u + 3]),
                      pack_bf16x2(d[8 * u + 4], d[8 * u + 5]), pack_bf16x2(d[8 * u + 6], d[8 * u + 7]));
}

__device__ __forceinline__ float bf16_to_f(uint16_t b) { return __uint_as_float((uint32_t)b << 16); }

// D row segment [n0, n0 + 32) of one output row: store or add, fp32 or bf16.
__device__ __forceinline__ void store_row32(const StoreArgs& st, int64_t orow, int64_t n0, int64_t N, float (&v)[32]) {
  if (st.out_bf16) {
    uint16_t* p = static_cast<uint16_t*>(st.D) + orow * st.ldd + n0;
    if (st.vec && n0 + 32 <= N) {
      if (st.add) {
        const uint4* q = reinterpret_cast<const uint4*>(p);
#pragma unroll
        for (int u = 0; u < 4; ++u) {
          const uint4 w = q[u];
          const uint32_t ws[4] = {w.x, w.y, w.z, w.w};
#pragma unroll
          for (int e = 0; e < 4; ++e) {
            v[8 * u + 2 * e] += bf16_to_f((uint16_t)(ws[e] & 0xFFFFu));
            v[8 * u + 2 * e + 1] += bf16_to_f((uint16_t)(ws[e] >> 16));
          }
        }
      }
      store_bf16x32(p, v);
    } else {
#pragma unroll
      for (int e = 0; e < 32; ++e)
        if (n0 + e < N) p[e] = to_bf16(st.add ? v[e] + bf16_to_f(p[e]) : v[e]);
    }
  } else {
    float* p = static_cast<float*>(st.D) + orow * st.ldd + n0;
    if (st.vec && n0 + 32 <= N) {
      float4* q = reinterpret_cast<float4*>(p);
#pragma unroll
      for (int u = 0; u < 8; ++u) {
        float4 o = make_float4(v[4 * u], v[4 * u + 1], v[4 * u + 2], v[4 * u + 3]);
        if (st.add) {
          const float4 w = q[u];
          o.x += w.x;
          o.y += w.y;
          o.z += w.z;
          o.w += w.w;
        }
        q[u] = o;
      }
    } else {
#pragma unroll
      for (int e = 0; e < 32; ++e)
        if (n0 + e < N) p[e] = st.add ? v[e] + p[e] : v[e];
    }
  }
}

// Persistent D = A B^T over (M/128) x (N/256) tiles, K in blocks of 64, warp-specialised like
// lmhead_fwd: warp 0 lane 0 TMA producer (4-stage ring), warp 1 lane 0 MMA issuer (two TMEM
// accumulators of 256 columns), warps 2-5 epilogue (one TMEM lane = one tile row per thread).
template <int EPI>
__global__ void __launch_bounds__(GB_THREADS, 1)
    tc_gemm(const __grid_constant__ CUtensorMap tmA, const __grid_constant__ CUtensorMap tmB, GemmArgs a) {
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~(uintptr_t)1023);
  uint8_t* sA = smem;
  uint8_t* sB = smem + GB_STAGES * GB_A_BYTES;
  uint64_t* full = reinterpret_cast<uint64_t*>(smem + GB_STAGES * GB_STAGE_BYTES);
  uint64_t* empty = full + GB_STAGES;
  uint64_t* tfull = empty + GB_STAGES;
  uint64_t* tempty = tfull + 2;
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(tempty + 2);
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;

  int64_t M = a.M, K = a.K, n_c = 0;
  if (a.dyn) {
    n_c = chunk_count(a.n_valid, a.chunk0, a.cap);
    if (a.dyn == 1) M = n_c;
    else K = n_c;
  }
  Tiles g;
  g.n_mt = (M + GB_BM - 1) / GB_BM;
  g.n_nt = (a.N + GB_BN - 1) / GB_BN;
  g.nkb = (K + TC_BK - 1) / TC_BK;
  g.swz = a.swz;
  g.n_inner = a.n_inner;
  const int64_t n_tiles = g.n_mt * g.n_nt;
  const bool has_k = g.nkb > 0;

  if (threadIdx.x == 0) {
    for (int s = 0; s < GB_STAGES; ++s) {
      mbar_init(&full[s], 1);
      mbar_init(&empty[s], 1);
    }
    for (int q = 0; q < 2; ++q) {
      mbar_init(&tfull[q], 1);
      mbar_init(&tempty[q], 4);
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
  tc_fence_after();
  const uint32_t tmem = *tmem_slot;

  if (warp == 0) {
    if (lane == 0 && has_k) {  // ---- TMA producer
      asm volatile("prefetch.tensormap [%0];" ::"l"(reinterpret_cast<uint64_t>(&tmA)) : "memory");
      asm volatile("prefetch.tensormap [%0];" ::"l"(reinterpret_cast<uint64_t>(&tmB)) : "memory");
      const uint64_t pol_a = l2_policy(a.pol & 1), pol_b = l2_policy(a.pol & 2);
      int stage = 0;
      uint32_t phase = 0;
      for (int64_t t = blockIdx.x; t < n_tiles; t += gridDim.x) {
        int64_t mb, nb;
        tile_of(g, t, mb, nb);
        for (int64_t kb = 0; kb < g.nkb; ++kb) {
          mbar_wait(&empty[stage], phase ^ 1u);
          mbar_expect_tx(&full[stage], GB_STAGE_BYTES);
          tma_load_2d(smem_u32(sA + stage * GB_A_BYTES), &tmA, (int)(kb * TC_BK), (int)(mb * GB_BM),
                      smem_u32(&full[stage]), pol_a);
          tma_load_2d(smem_u32(sB + stage * GB_B_BYTES), &tmB, (int)(kb * TC_BK), (int)(nb * GB_BN),
                      smem_u32(&full[stage]), pol_b);
          if (++stage == GB_STAGES) {
            stage = 0;
            phase ^= 1u;
          }
        }
      }
    }
  } else if (warp == 1) {
    if (lane == 0 && has_k) {  // ---- MMA issuer
      int stage = 0;
      uint32_t phase = 0;
      uint32_t j = 0;
      for (int64_t t = blockIdx.x; t < n_tiles; t += gridDim.x, ++j) {
        const uint32_t acc = j & 1u, aph = (j >> 1) & 1u;
        mbar_wait(&tempty[acc], aph ^ 1u);
        tc_fence_after();
        const uint32_t d_tmem = tmem + acc * GB_BN;
        for (int64_t kb = 0; kb < g.nkb; ++kb) {
          mbar_wait(&full[stage], phase);
          tc_fence_after();
          const uint64_t a0 = umma_desc_sw128(smem_u32(sA + stage * GB_A_BYTES));
          const uint64_t b0 = umma_desc_sw128(smem_u32(sB + stage * GB_B_BYTES));
#pragma unroll
          for (int k = 0; k < TC_BK / 16; ++k)  // K = 16 per MMA: +32 bytes = +2 in the address field
            umma_bf16<GB_IDESC>(d_tmem, a0 + 2u * k, b0 + 2u * k, (kb | k) != 0);
          umma_commit(&empty[stage]);
          if (++stage == GB_STAGES) {
            stage = 0;
            phase ^= 1u;
          }
        }
        umma_commit(&tfull[acc]);
      }
    }
  } else {  // ---- epilogue: warps 2..5 own TMEM lane quarters (warp % 4)
    const int q = warp & 3;
    const int row_in = q * 32 + lane;
    const uint32_t lane_addr = tmem + ((uint32_t)(q * 32) << 16);
    uint32_t j = 0;
    for (int64_t t = blockIdx.x; t < n_tiles; t += gridDim.x, ++j) {
      int64_t mb, nb;
      tile_of(g, t, mb, nb);
      const uint32_t acc = j & 1u, aph = (j >> 1) & 1u;
      const int64_t m = mb * GB_BM + row_in;
      if (has_k) {
        mbar_wait(&tfull[acc], aph);
        tc_fence_after();
      }
      if (EPI == EPI_DZ) {
        const DzArgs& z = a.dz;
        const bool valid = m < n_c;
        float M2 = 0.f, L2S = 0.f, c = 0.f;
        int64_t y = -1;
        if (valid) {
          const int64_t r = z.idx[a.chunk0 + m];
          const float2 st = z.stats[r];
          M2 = st.x;
          L2S = st.y;
          const double gg = (z.grad_out ? *z.grad_out : 1.0) * z.gs;
          c = z.coef ? (float)(gg * (double)z.coef[r]) : (float)(gg * z.resid[r / z.T]);
          y = z.tokens[r];
        }
#pragma unroll 1
        for (int cc = 0; cc < GB_BN / 32; ++cc) {
          const int64_t v0 = nb * GB_BN + cc * 32;
          if (v0 >= z.V) break;  // warp-uniform
          float v[32];
          tmem_ld32(lane_addr + acc * GB_BN + cc * 32, v);
          const float nM2 = -M2;
#pragma unroll
          for (int e = 0; e < 32; ++e) {
            const float p = ex2(fmaf(v[e], z.sc, nM2) - L2S);
            v[e] = valid ? ((v0 + e == y) ? fmaf(-c, p, c) : -c * p) : 0.f;
          }
          uint16_t* zr = z.dz + m * z.Vp + v0;
          if (v0 + 32 <= z.V) {
            store_bf16x32(zr, v);
            if (z.dzt)
#pragma unroll
              for (int e = 0; e < 32; ++e) z.dzt[(v0 + e) * z.C + m] = to_bf16(v[e]);
          } else {
            for (int e = 0; e < 32; ++e)
              if (v0 + e < z.V) {
                const uint16_t b = to_bf16(v[e]);
                zr[e] = b;
                if (z.dzt) z.dzt[(v0 + e) * z.C + m] = b;
              }
          }
        }
      } else {
        const StoreArgs& st = a.st;
        const bool in = m < M;
        const int64_t orow = in ? (st.row_map ? (int64_t)st.row_map[m] : m) : 0;
#pragma unroll 1
        for (int cc = 0; cc < GB_BN / 32; ++cc) {
          const int64_t n0 = nb * GB_BN + cc * 32;
          if (n0 >= a.N) break;  // warp-uniform
          float v[32];
          if (has_k) {
            tmem_ld32(lane_addr + acc * GB_BN + cc * 32, v);
          } else {
#pragma unroll
            for (int e = 0; e < 32; ++e) v[e] = 0.f;
          }
          if (in && (has_k || !st.add)) store_row32(st, orow, n0, a.N, v);
        }
      }
      if (has_k) {
        tc_fence_before();
        __syncwarp();
        if (lane == 0) mbar_arrive(&tempty[acc]);
      }
    }
  }
  __syncthreads();
  if (warp == 1) {
    tc_fence_after();
    asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 512;" ::"r"(tmem) : "memory");
  }
}

// cta_group::2 form of tc_gemm<EPI_STORE>: an SM pair (cluster of 2) computes a 256 x 256 tile per
// MMA (M = 256 across the pair). Each CTA loads its 128 rows of A and its half (128 rows) of the
// B tile per stage, so per SM only 32 KB (2/3 of the single-SM kernel's 48 KB) move from L2 per
// 128 x 256 x 64 of MMA work. Both CTAs' TMA loads signal the leader's full barrier; the leader's
// lane issues the MMA, whose commits arrive on both CTAs' barriers; the epilogue warps of both CTAs
// release an accumulator on the leader's barrier (count 8). Same arithmetic per output element
// as tc_gemm (one K-ordered fp32 accumulation), so results are bitwise equal.
// NT = 2: each pair tile is 256 x 512 (two N = 256 MMAs per K step sharing the A stage; the two
// accumulators hold one tile, so the epilogue is not overlapped with the next tile's MMAs — fine
// when K is long): per SM 48 KB move from L2 per 128 x 512 x 64, half the single-SM kernel's rate.
template <int NT>
struct G2 {
  static constexpr int STAGES = NT == 1 ? 6 : 4;
  static constexpr int A_BYTES = 128 * TC_BK * 2;       // 16 KB: this CTA's 128 rows of A
  static constexpr int B_BYTES = NT * 128 * TC_BK * 2;  // this CTA's halves of the NT 256-row B tiles
  static constexpr int STAGE_BYTES = A_BYTES + B_BYTES;
  static constexpr size_t SMEM = 1024 + (size_t)STAGES * STAGE_BYTES + 256;
  static constexpr int NACC = 2 / NT;                   // accumulator buffers of NT x 256 columns
};
constexpr uint32_t G2_IDESC = tc_idesc_bf16(256, GB_BN);

// MN = true: both operands MN-major (A = dZ [K = rows, M = V], B = Hc [K = rows, N = d], read as
// stored, no transposed copies): each 128-wide operand slab is two TMA boxes of {64 MN, 64 K}
// placed 8 KB apart (the descriptor's LBO).
template <int NT, bool MN = false>
__global__ void __launch_bounds__(GB_THREADS, 1)
    tc_gemm2(const __grid_constant__ CUtensorMap tmA, const __grid_constant__ CUtensorMap tmB, GemmArgs a) {
  using C = G2<NT>;
  constexpr int G2_STAGES = C::STAGES, G2_A_BYTES = C::A_BYTES, G2_B_BYTES = C::B_BYTES,
                G2_STAGE_BYTES = C::STAGE_BYTES, NACC = C::NACC;
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~(uintptr_t)1023);
  uint8_t* sA = smem;
  uint8_t* sB = smem + G2_STAGES * G2_A_BYTES;
  uint64_t* full = reinterpret_cast<uint64_t*>(smem + G2_STAGES * G2_STAGE_BYTES);
  uint64_t* empty = full + G2_STAGES;
  uint64_t* tfull = empty + G2_STAGES;
  uint64_t* tempty = tfull + 2;
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(tempty + 2);
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const uint32_t crank = cluster_ctarank();
  const bool leader = crank == 0;
  const int64_t pair0 = blockIdx.x / 2, n_pairs = gridDim.x / 2;

  int64_t M = a.M, K = a.K;
  if (a.dyn) {
    const int64_t n_c = chunk_count(a.n_valid, a.chunk0, a.cap);
    if (a.dyn == 1) M = n_c;
    else K = n_c;
  }
  Tiles g;
  g.n_mt = (M + 255) / 256;
  g.n_nt = (a.N + NT * GB_BN - 1) / (NT * GB_BN);
  g.nkb = (K + TC_BK - 1) / TC_BK;
  g.swz = (a.swz + 1) / 2;
  g.n_inner = a.n_inner;
  const int64_t n_tiles = g.n_mt * g.n_nt;
  const bool has_k = g.nkb > 0;
  // split-K (K static, ksplit <= nkb): unit u = slice (u / n_tiles) of tile (u % n_tiles), k blocks
  // [sl nkb / S, (sl + 1) nkb / S): the slice boundaries depend on K and S only, never on the tiling.
  const int S = a.ksplit > 1 ? a.ksplit : 1;
  const int64_t n_units = n_tiles * S;

  if (threadIdx.x == 0) {
    for (int s = 0; s < G2_STAGES; ++s) {
      mbar_init(&full[s], 1);   // leader: its producer's arrive + both CTAs' bytes
      mbar_init(&empty[s], 1);  // the leader's multicast commit
    }
    for (int q = 0; q < 2; ++q) {
      mbar_init(&tfull[q], 1);
      mbar_init(&tempty[q], 8);  // leader: 4 epilogue warps x 2 CTAs
    }
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
  }
  if (warp == 1) {
    asm volatile("tcgen05.alloc.cta_group::2.sync.aligned.shared::cta.b32 [%0], 512;" ::"r"(smem_u32(tmem_slot))
                 : "memory");
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::2.sync.aligned;" ::: "memory");
  }
  tc_fence_before();
  __syncthreads();
  cluster_sync_all();
  tc_fence_after();
  const uint32_t tmem = *tmem_slot;

  if (warp == 0) {
    if (lane == 0 && has_k) {  // ---- TMA producer (both CTAs)
      asm volatile("prefetch.tensormap [%0];" ::"l"(reinterpret_cast<uint64_t>(&tmA)) : "memory");
      asm volatile("prefetch.tensormap [%0];" ::"l"(reinterpret_cast<uint64_t>(&tmB)) : "memory");
      const uint64_t pol_a = l2_policy(a.pol & 1), pol_b = l2_policy(a.pol & 2);
      int stage = 0;
      uint32_t phase = 0;
      for (int64_t u = pair0; u < n_units; u += n_pairs) {
        const int64_t t = u % n_tiles, sl = u / n_tiles;
        int64_t mb, nb;
        tile_of(g, t, mb, nb);
        for (int64_t kb = sl * g.nkb / S, kb1 = (sl + 1) * g.nkb / S; kb < kb1; ++kb) {
          mbar_wait(&empty[stage], phase ^ 1u);
          if (leader) mbar_expect_tx(&full[stage], 2 * G2_STAGE_BYTES);
          if (MN) {
#pragma unroll
            for (int hb = 0; hb < 2; ++hb)
              tma_load_2d_pair(smem_u32(sA + stage * G2_A_BYTES + hb * 8192), &tmA,
                               (int)(mb * 256 + crank * 128 + hb * 64), (int)(kb * TC_BK), smem_u32(&full[stage]),
                               pol_a, true);
#pragma unroll
            for (int u = 0; u < NT; ++u)
#pragma unroll
              for (int hb = 0; hb < 2; ++hb)
                tma_load_2d_pair(smem_u32(sB + stage * G2_B_BYTES + u * (128 * TC_BK * 2) + hb * 8192), &tmB,
                                 (int)((nb * NT + u) * GB_BN + crank * 128 + hb * 64), (int)(kb * TC_BK),
                                 smem_u32(&full[stage]), pol_b, true);
          } else {
            tma_load_2d_pair(smem_u32(sA + stage * G2_A_BYTES), &tmA, (int)(kb * TC_BK),
                             (int)(mb * 256 + crank * 128), smem_u32(&full[stage]), pol_a, true);
#pragma unroll
            for (int u = 0; u < NT; ++u)
              tma_load_2d_pair(smem_u32(sB + stage * G2_B_BYTES + u * (128 * TC_BK * 2)), &tmB, (int)(kb * TC_BK),
                               (int)((nb * NT + u) * GB_BN + crank * 128), smem_u32(&full[stage]), pol_b, true);
          }
          if (++stage == G2_STAGES) {
            stage = 0;
            phase ^= 1u;
          }
        }
      }
    }
  } else if (warp == 1) {
    if (lane == 0 && leader && has_k) {  // ---- MMA issuer (leader only)
      int stage = 0;
      uint32_t phase = 0;
      uint32_t j = 0;
      for (int64_t u = pair0; u < n_units; u += n_pairs, ++j) {
        const int64_t sl = u / n_tiles, kb0 = sl * g.nkb / S;
        const uint32_t acc = j % NACC, aph = (j / NACC) & 1u;
        mbar_wait(&tempty[acc], aph ^ 1u);
        tc_fence_after();
        const uint32_t d_tmem = tmem + acc * NT * GB_BN;
        for (int64_t kb = kb0, kb1 = (sl + 1) * g.nkb / S; kb < kb1; ++kb) {
          mbar_wait(&full[stage], phase);
          tc_fence_after();
          const uint32_t sa = smem_u32(sA + stage * G2_A_BYTES);
          const uint64_t a0 = MN ? umma_desc_mn_sw128(sa, 8192) : umma_desc_sw128(sa);
          constexpr uint32_t kstep = MN ? (16 * 128) >> 4 : 2;  // K = 16: 16 rows of 128 B, or +32 B in a row
          constexpr uint32_t IDESC = MN ? (G2_IDESC | kIdescMajorMN) : G2_IDESC;
#pragma unroll
          for (int k = 0; k < TC_BK / 16; ++k)
#pragma unroll
            for (int nu = 0; nu < NT; ++nu) {
              const uint32_t sb = smem_u32(sB + stage * G2_B_BYTES + nu * (128 * TC_BK * 2));
              const uint64_t b0 = MN ? umma_desc_mn_sw128(sb, 8192) : umma_desc_sw128(sb);
              umma_bf16_pair<IDESC>(d_tmem + nu * GB_BN, a0 + kstep * k, b0 + kstep * k, kb != kb0 || k != 0);
            }
          umma_commit_pair(&empty[stage]);
          if (++stage == G2_STAGES) {
            stage = 0;
            phase ^= 1u;
          }
        }
        umma_commit_pair(&tfull[acc]);
      }
    }
  } else {  // ---- epilogue (both CTAs): release on the leader's tempty
    const int q = warp & 3;
    const int row_in = q * 32 + lane;
    const uint32_t lane_addr = tmem + ((uint32_t)(q * 32) << 16);
    uint32_t tempty_leader;
    asm volatile("mapa.shared::cluster.u32 %0, %1, 0;" : "=r"(tempty_leader) : "r"(smem_u32(tempty)));
    const StoreArgs& st = a.st;
    uint32_t j = 0;
    for (int64_t u = pair0; u < n_units; u += n_pairs, ++j) {
      const int64_t t = u % n_tiles, sl = u / n_tiles;
      int64_t mb, nb;
      tile_of(g, t, mb, nb);
      const uint32_t acc = j % NACC, aph = (j / NACC) & 1u;
      const int64_t m = mb * 256 + (int64_t)crank * 128 + row_in;
      if (has_k) {
        mbar_wait(&tfull[acc], aph);
        tc_fence_after();
      }
      const bool in = m < M;
      const int64_t orow = in ? (st.row_map ? (int64_t)st.row_map[m] : m) : 0;
#pragma unroll 1
      for (int cc = 0; cc < NT * GB_BN / 32; ++cc) {
        const int64_t n0 = nb * NT * GB_BN + cc * 32;
        if (n0 >= a.N) break;  // warp-uniform
        float v[32];
        if (has_k) {
          tmem_ld32(lane_addr + acc * NT * GB_BN + cc * 32, v);
        } else {
#pragma unroll
          for (int e = 0; e < 32; ++e) v[e] = 0.f;
        }
        if (S > 1) {
          if (in) {  // fp32 partial of slice sl (part_ld is a multiple of 4 floats)
            float* p = a.part + (sl * a.cap + m) * a.part_ld + n0;
            if (n0 + 32 <= a.N) {
#pragma unroll
              for (int e = 0; e < 8; ++e)
                reinterpret_cast<float4*>(p)[e] = make_float4(v[4 * e], v[4 * e + 1], v[4 * e + 2], v[4 * e + 3]);
            } else {
#pragma unroll
              for (int e = 0; e < 32; ++e)
                if (n0 + e < a.N) p[e] = v[e];
            }
          }
        } else if (in && (has_k || !st.add)) {
          store_row32(st, orow, n0, a.N, v);
        }
      }
      if (has_k) {
        tc_fence_before();
        __syncwarp();
        if (lane == 0)
          asm volatile("mbarrier.arrive.release.cluster.shared::cluster.b64 _, [%0];" ::"r"(tempty_leader + acc * 8u)
                       : "memory");
      }
    }
  }
  __syncthreads();
  cluster_sync_all();
  if (warp == 1) {
    tc_fence_after();
    asm volatile("tcgen05.dealloc.cta_group::2.sync.aligned.b32 %0, 512;" ::"r"(tmem) : "memory");
  }
}

// Ascending list of the valid rows (mask != 0), stored as r0 + row: one CTA, chunks of 1024 rows,
// ballot + warp scan.
__global__ void __launch_bounds__(1024) lmb_compact_rows(const uint8_t* __restrict__ mask, int64_t rows, int64_t r0,
                                                         int* __restrict__ idx, int* __restrict__ n_out) {
  __shared__ int warp_tot[32];
  __shared__ int base;
  const int tid = threadIdx.x, lane = tid & 31, wid = tid >> 5;
  if (tid == 0) base = 0;
  __syncthreads();
  for (int64_t c0 = 0; c0 < rows; c0 += 1024) {
    const int64_t r = c0 + tid;
    const bool a = r < rows && mask[r] != 0;
    const unsigned bal = __ballot_sync(0xffffffffu, a);
    if (lane == 0) warp_tot[wid] = __popc(bal);
    __syncthreads();
    int off = 0;
    for (int w = 0; w < wid; ++w) off += warp_tot[w];
    if (a) idx[base + off + __popc(bal & ((1u << lane) - 1u))] = (int)(r0 + r);
    __syncthreads();
    if (tid == 0) {
      int tot = 0;
      for (int w = 0; w < 32; ++w) tot += warp_tot[w];
      base += tot;
    }
    __syncthreads();
  }
  if (tid == 0) *n_out = base;
}

// Row gather + transpose of a bf16 matrix in 64 x 64 tiles: for output rows i in [0, n_pad),
// src row = idx[chunk0 + i] (idx == nullptr: chunk0 + i), zero for i >= n (the chunk's count):
//   dst_rm[i, k] = src[row, k]   (nullable; row stride d)
//   dst_t [k, i] = src[row, k]   (row stride ld_t)
// n = clamp(*n_valid - chunk0, 0, cap) (n_valid == nullptr: n_static); n_pad = n rounded up to
// 128 when `pad` (so the GEMM tiles over the chunk read zeros), else n.
__global__ void __launch_bounds__(256) lmb_gather_t(const uint16_t* __restrict__ src, int64_t sstride, int64_t d,
                                                    const int* __restrict__ idx, const int* __restrict__ n_valid,
                                                    int64_t n_static, int64_t chunk0, int64_t cap, int pad,
                                                    uint16_t* __restrict__ dst_rm, uint16_t* __restrict__ dst_t,
                                                    int64_t ld_t) {
  __shared__ uint16_t tile[64][66];  // 33-word rows: the column reads below are conflict-free
  const int64_t n = n_valid ? chunk_count(n_valid, chunk0, cap) : n_static;
  const int64_t n_pad = pad ? (n + 127) / 128 * 128 : n;
  const int64_t i0 = (int64_t)blockIdx.y * 64, k0 = (int64_t)blockIdx.x * 64;
  if (i0 >= n_pad) return;
  const int tid = threadIdx.x;
#pragma unroll
  for (int p = 0; p < 2; ++p) {
    const int rl = tid / 8 + 32 * p, kl = (tid % 8) * 8;
    const int64_t i = i0 + rl, k = k0 + kl;
    uint4 val = make_uint4(0u, 0u, 0u, 0u);
    if (i < n && k < d) {
      const int64_t r = idx ? (int64_t)idx[chunk0 + i] : chunk0 + i;
      val = *reinterpret_cast<const uint4*>(src + r * sstride + k);
    }
    if (dst_rm && i < n_pad && k < d) *reinterpret_cast<uint4*>(dst_rm + i * d + k) = val;
    uint32_t* tp = reinterpret_cast<uint32_t*>(&tile[rl][kl]);
    tp[0] = val.x;
    tp[1] = val.y;
    tp[2] = val.z;
    tp[3] = val.w;
  }
  if (!dst_t) return;
  __syncthreads();
#pragma unroll
  for (int p = 0; p < 2; ++p) {
    const int kl = tid / 8 + 32 * p, il = (tid % 8) * 8;
    const int64_t k = k0 + kl, i = i0 + il;
    if (k < d && i < n_pad) {
      uint32_t w[4];
#pragma unroll
      for (int e = 0; e < 4; ++e)
        w[e] = (uint32_t)tile[il + 2 * e][kl] | ((uint32_t)tile[il + 2 * e + 1][kl] << 16);
      *reinterpret_cast<uint4*>(dst_t + k * ld_t + i) = make_uint4(w[0], w[1], w[2], w[3]);
    }
  }
}

// dz from stored fp32 logits (the one-call forward + backward): tiles of 64 compacted rows x 128
// vocabulary columns; row i of the chunk is batch row r = idx[i], its logits at zst + (r - zrow0) * zst_ld.
//   dz [i, v] = c_r (1[v = y_r] - 2^(z sc - M2 - log2 S))  (bf16)  and  dz^T [v, i] the same
// (rows i in [n, n rounded up to 128) are written as 0 so the GEMM tiles over them read zeros).
__global__ void __launch_bounds__(256) lmb_dz_from_z(DzArgs z, const int* __restrict__ n_valid, int64_t chunk0,
                                                     int64_t cap, const float* __restrict__ zst, int64_t zst_ld,
                                                     int64_t zrow0) {
  __shared__ uint16_t tile[64][130];  // 65-word rows: the column reads below hit distinct banks
  __shared__ float s_c[64], s_m2[64], s_l2s[64];
  __shared__ long long s_y[64], s_off[64];
  const int64_t n = chunk_count(n_valid, chunk0, cap);
  const int64_t n_pad = (n + 127) / 128 * 128;
  const int64_t i0 = (int64_t)blockIdx.y * 64, v0 = (int64_t)blockIdx.x * 128;
  if (i0 >= n_pad) return;
  const int tid = threadIdx.x;
  if (tid < 64) {
    const int64_t i = i0 + tid;
    float c = 0.f, M2 = 0.f, L2S = 0.f;
    long long y = -1, off = -1;
    if (i < n) {
      const int64_t r = z.idx[chunk0 + i];
      const float2 st = z.stats[r];
      M2 = st.x;
      L2S = st.y;
      const double gg = (z.grad_out ? *z.grad_out : 1.0) * z.gs;
      c = z.coef ? (float)(gg * (double)z.coef[r]) : (float)(gg * z.resid[r / z.T]);
      y = z.tokens[r];
      off = (r - zrow0) * zst_ld;
    }
    s_c[tid] = c;
    s_m2[tid] = M2;
    s_l2s[tid] = L2S;
    s_y[tid] = y;
    s_off[tid] = off;
  }
  __syncthreads();
  // 64 rows x 128 columns: each thread 4 consecutive columns of 8 rows (float4 loads, 32 threads per row)
#pragma unroll
  for (int p = 0; p < 8; ++p) {
    const int rl = tid / 32 + 8 * p, cl = (tid % 32) * 4;
    const int64_t i = i0 + rl, v = v0 + cl;
    float d[4] = {0.f, 0.f, 0.f, 0.f};
    if (i < n && v < z.V) {
      const float* zp = zst + s_off[rl] + v;
      float4 q;
      if (v + 4 <= z.V) q = __ldcs(reinterpret_cast<const float4*>(zp));
      else q = make_float4(zp[0], v + 1 < z.V ? zp[1] : 0.f, v + 2 < z.V ? zp[2] : 0.f, 0.f);
      const float zz[4] = {q.x, q.y, q.z, q.w};
      const float c = s_c[rl], nM2 = -s_m2[rl], L2S = s_l2s[rl];
#pragma unroll
      for (int e = 0; e < 4; ++e) {
        const float pr = ex2(fmaf(zz[e], z.sc, nM2) - L2S);
        d[e] = (v + e == s_y[rl]) ? fmaf(-c, pr, c) : -c * pr;
      }
    }
    const uint32_t lo = pack_bf16x2(d[0], d[1]), hi = pack_bf16x2(d[2], d[3]);
    if (v + 4 <= z.Vp && i < cap) *reinterpret_cast<uint2*>(z.dz + i * z.Vp + v) = make_uint2(lo, hi);
    uint32_t* tp = reinterpret_cast<uint32_t*>(&tile[rl][cl]);
    tp[0] = lo;
    tp[1] = hi;
  }
  if (!z.dzt) return;  // dW reads dz itself (MN-major operand)
  __syncthreads();
  // dz^T: 128 vocabulary rows of 64 chunk rows (128 B each): 8 threads x 16 B per row
#pragma unroll
  for (int p = 0; p < 4; ++p) {
    const int vl = tid / 8 + 32 * p, il = (tid % 8) * 8;
    const int64_t v = v0 + vl;
    if (v < z.V) {
      uint32_t w[4];
#pragma unroll
      for (int e = 0; e < 4; ++e)
        w[e] = (uint32_t)tile[il + 2 * e][vl] | ((uint32_t)tile[il + 2 * e + 1][vl] << 16);
      *reinterpret_cast<uint4*>(z.dzt + v * z.C + i0 + il) = make_uint4(w[0], w[1], w[2], w[3]);
    }
  }
}

// dH rows from the split-K partials of tc_gemm2: out[row_map[m]] (+)= sum over slices, in slice order
// (fixed order: deterministic). One thread per 4 consecutive columns; rows m < the chunk's count.
__global__ void __launch_bounds__(256) lmb_splitk_reduce(const float* __restrict__ part, int64_t part_ld, int S,
                                                         int64_t cap, const int* __restrict__ n_valid, int64_t chunk0,
                                                         int64_t N, StoreArgs st) {
  const int64_t M = chunk_count(n_valid, chunk0, cap);
  const int64_t n = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) * 4;
  if (n >= N) return;
  const bool full4 = n + 4 <= N;  // the tail reads only the columns the GEMM wrote
  for (int64_t m = blockIdx.y; m < M; m += gridDim.y) {
    float v[4] = {0.f, 0.f, 0.f, 0.f};
    for (int sl = 0; sl < S; ++sl) {
      const float* q = part + (sl * cap + m) * part_ld + n;
      if (full4) {
        const float4 w = __ldg(reinterpret_cast<const float4*>(q));
        v[0] += w.x;
        v[1] += w.y;
        v[2] += w.z;
        v[3] += w.w;
      } else {
        for (int e = 0; e < 4 && n + e < N; ++e) v[e] += __ldg(q + e);
      }
    }
    const int64_t orow = st.row_map ? (int64_t)st.row_map[m] : m;
#pragma unroll
    for (int e = 0; e < 4; ++e) {
      if (n + e >= N) break;
      if (st.out_bf16) {
        uint16_t* o = static_cast<uint16_t*>(st.D) + orow * st.ldd + n + e;
        *o = to_bf16(st.add ? v[e] + bf16_to_f(*o) : v[e]);
      } else {
        float* o = static_cast<float*>(st.D) + orow * st.ldd + n + e;
        *o = st.add ? v[e] + *o : v[e];
      }
    }
  }
}

constexpr int LMB_KSPLIT_MAX = 4;

// Kernel selection of the backward GEMMs, read ONCE per process (A/B and test switches; the
// defaults are the measured best): pair bit 0 dH / bit 1 dW on the cta_group::2
// kernel, wide = 256 x 512 pair tiles, dwmn = dW reads dZ and Hc as MN-major operands.
struct LmbKnobs {
  int swz, ninner, pol, pair, wide, dwmn, ksplit;
};
const LmbKnobs& lmb_knobs() {
  static const LmbKnobs k = [] {
    LmbKnobs v;
    v.swz = env_once("TBA_LMB_SWZ", 32);
    if (v.swz < 1) v.swz = 32;
    v.ninner = env_once("TBA_LMB_NINNER", 3);
    v.pol = env_once("TBA_LMB_POL", 0x8);  // dW: keep Hc^T in L2 (measured 198 vs 203 ms)
    v.pair = env_once("TBA_LMB_2SM", 3);   // measured: 196-203 ms vs 218-223 (one-call Qwen step)
    v.wide = env_once("TBA_LMB_NT2", 3);
    v.dwmn = env_once("TBA_LMB_DW_MN", 1) != 0 && (v.pair & 2) != 0;
    v.ksplit = env_once("TBA_LMB_KSPLIT", 0);
    return v;
  }();
  return k;
}
// The transposed copies dZ^T [V, C] and Hc^T [d, C] exist only for the K-major dW forms.
inline bool lmb_need_transposed() { return !lmb_knobs().dwmn; }

struct LmbWs {
  int* idx;  // [rows] + the count at idx[rows]
  uint16_t *wt, *hc, *hct, *dz, *dzt;
  float* part;  // dH split-K partials [LMB_KSPLIT_MAX][C][lmb_dp(d)]
};

inline int64_t lmb_vp(int64_t V) { return (V + 7) / 8 * 8; }
inline int64_t lmb_dp(int64_t d) { return (d + 3) / 4 * 4; }

LmbWs lmb_layout(void* base, int64_t rows, int64_t d, int64_t V, int64_t C) {
  char* p = static_cast<char*>(base);
  LmbWs w;
  size_t off = 0;
  auto take = [&](size_t bytes) {
    char* q = p + off;
    off = align_up(off + bytes, 256);
    return q;
  };
  w.idx = reinterpret_cast<int*>(take((size_t)(rows + 1) * sizeof(int)));
  w.wt = reinterpret_cast<uint16_t*>(take((size_t)d * (size_t)lmb_vp(V) * 2));
  w.hc = reinterpret_cast<uint16_t*>(take((size_t)C * (size_t)d * 2));
  const bool tr = lmb_need_transposed();
  w.hct = reinterpret_cast<uint16_t*>(take(tr ? (size_t)d * (size_t)C * 2 : 0));
  w.dz = reinterpret_cast<uint16_t*>(take((size_t)C * (size_t)lmb_vp(V) * 2));
  w.dzt = reinterpret_cast<uint16_t*>(take(tr ? (size_t)V * (size_t)C * 2 : 0));
  w.part = reinterpret_cast<float*>(take((size_t)LMB_KSPLIT_MAX * (size_t)C * (size_t)lmb_dp(d) * 4));
  return w;
}

template <int EPI>
int launch_gemm(const CUtensorMap& ma, const CUtensorMap& mb, const GemmArgs& a, int64_t max_tiles, cudaStream_t s) {
  static bool attr[2][64] = {};  // per variant and device; benign race: idempotent
  int dev = 0;
  if (cudaGetDevice(&dev) != cudaSuccess || dev < 0 || dev >= 64) return TBA_ERR_CUDA;
  if (!attr[EPI][dev]) {
    if (cudaFuncSetAttribute(tc_gemm<EPI>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)GB_SMEM) != cudaSuccess)
      return TBA_ERR_CUDA;
    attr[EPI][dev] = true;
  }
  int64_t grid = device_sms();
  if (grid > max_tiles) grid = max_tiles;
  if (grid < 1) grid = 1;
  tc_gemm<EPI><<<(unsigned)grid, GB_THREADS, GB_SMEM, s>>>(ma, mb, a);
  return launch_status();
}

template <int NT, bool MN = false>
int launch_gemm2(const CUtensorMap& ma, const CUtensorMap& mb, const GemmArgs& a, int64_t max_pair_tiles,
                 cudaStream_t s) {
  static bool attr[64] = {};
  int dev = 0;
  if (cudaGetDevice(&dev) != cudaSuccess || dev < 0 || dev >= 64) return TBA_ERR_CUDA;
  if (!attr[dev]) {
    if (cudaFuncSetAttribute(tc_gemm2<NT, MN>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)G2<NT>::SMEM) !=
        cudaSuccess)
      return TBA_ERR_CUDA;
    attr[dev] = true;
  }
  cudaLaunchConfig_t cfg = {};
  cudaLaunchAttribute at[1];
  at[0].id = cudaLaunchAttributeClusterDimension;
  at[0].val.clusterDim.x = 2;
  at[0].val.clusterDim.y = 1;
  at[0].val.clusterDim.z = 1;
  cfg.attrs = at;
  cfg.numAttrs = 1;
  cfg.blockDim = dim3(GB_THREADS);
  cfg.dynamicSmemBytes = G2<NT>::SMEM;
  cfg.stream = s;
  int64_t pairs = device_sms() / 2;
  cfg.gridDim = dim3((unsigned)(pairs * 2));
  int ncl = 0;
  if (cudaOccupancyMaxActiveClusters(&ncl, tc_gemm2<NT, MN>, &cfg) == cudaSuccess && ncl > 0 && ncl < pairs)
    pairs = ncl;
  if (pairs > max_pair_tiles) pairs = max_pair_tiles;
  if (pairs < 1) pairs = 1;
  cfg.gridDim = dim3((unsigned)(pairs * 2));
  if (cudaLaunchKernelEx(&cfg, tc_gemm2<NT, MN>, ma, mb, a) != cudaSuccess) return TBA_ERR_CUDA;
  return TBA_OK;
}

}  // namespace

int64_t lmhead_bwd_chunk(int64_t rows, int64_t chunk_rows) {
  int64_t c = chunk_rows > 0 ? chunk_rows : LMB_DEFAULT_CHUNK;
  if (c > rows) c = rows;
  if (c < 1) c = 1;
  return (c + 127) / 128 * 128;
}

size_t lmhead_bwd_ws_bytes(int64_t rows, int64_t d, int64_t V, int64_t chunk_rows) {
  const int64_t C = lmhead_bwd_chunk(rows, chunk_rows);
  const bool tr = lmb_need_transposed();
  return align_up((size_t)(rows + 1) * sizeof(int), 256) + align_up((size_t)d * (size_t)lmb_vp(V) * 2, 256) +
         align_up((size_t)C * (size_t)d * 2, 256) + (tr ? align_up((size_t)d * (size_t)C * 2, 256) : 0) +
         align_up((size_t)C * (size_t)lmb_vp(V) * 2, 256) + (tr ? align_up((size_t)V * (size_t)C * 2, 256) : 0) +
         align_up((size_t)LMB_KSPLIT_MAX * (size_t)C * (size_t)lmb_dp(d) * 4, 256);
}

namespace {

// Per-call state of the backward: workspace layout, tensor maps, knobs (TBA_LMB_SWZ dz raster,
// TBA_LMB_NINNER bit 0: dH / bit 1: dW tiles n-inner, TBA_LMB_POL bits 0-1 dH / 2-3 dW A / B loads
// evict_last: measurement knobs, read once).
struct LmbCtx {
  const tba_lmhead* x;
  int64_t C, Vp;
  LmbWs w;
  CUtensorMap m_hc, m_w, m_dz, m_wt, m_dzt, m_hct;
  int swz, ninner, pol, pair, wide;  // pair: bit 0 dH, bit 1 dW on the cta_group::2 kernel; wide: NT = 2
  bool dwmn;                         // dW reads dZ and Hc as MN-major operands (no transposed copies)
  int dh_split;                      // dH split-K slices on the pair kernel (lmb_dh_split)
  CUtensorMap m_dzmn, m_hcmn;
  CUtensorMap m_wt2, m_hct2;   // B operands with 128-row boxes for the pair kernel (A boxes are 128 rows already)
};

// dH = dZ W has few output tiles and a long K (= V): (C/256) x (d/512) pair tiles leave the last
// wave mostly idle (Qwen: 448 tiles on 74 pairs = 6.05 waves run as 7). Split K into S slices
// (TBA_LMB_KSPLIT: 0 auto, else forced 1..4). Auto: the smallest S whose waves over the nominal chunk
// (LMB_DEFAULT_CHUNK rows) come within 4 % of perfect balance. S depends on (d, V, SMs) only, so the
// one-call and two-call schedules split alike and their dH stay bitwise equal.
int lmb_dh_split(int64_t d, int64_t V, int nt) {
  const int knob = lmb_knobs().ksplit;
  const int64_t nkb = (V + TC_BK - 1) / TC_BK;
  int S = 1;
  if (knob > 0) {
    S = knob;
  } else {
    const double pairs = (double)(device_sms() / 2 > 0 ? device_sms() / 2 : 1);
    const double tiles = (double)((LMB_DEFAULT_CHUNK / 256) * ((d + nt * GB_BN - 1) / (nt * GB_BN)));
    const double ideal = tiles / pairs;
    double best = 1e30;
    for (int c = 1; c <= LMB_KSPLIT_MAX; ++c) {
      const double waves = std::ceil(tiles * c / pairs) / c;
      if (waves <= 1.04 * ideal) {
        S = c;
        break;
      }
      if (waves < best - 1e-9) {
        best = waves;
        S = c;
      }
    }
  }
  if (S > LMB_KSPLIT_MAX) S = LMB_KSPLIT_MAX;
  if (S > nkb) S = (int)nkb;
  return S < 1 ? 1 : S;
}

int lmb_prepare(LmbCtx& k, const tba_lmhead* x, int64_t idx_rows, int64_t C, void* bws, bool need_wt, cudaStream_t s) {
  const LmbKnobs& kn = lmb_knobs();
  const int pair = kn.pair, wide = kn.wide;
  const int64_t d = x->d, V = x->vocab;
  k.x = x;
  k.C = C;
  k.Vp = lmb_vp(V);
  k.w = lmb_layout(bws, idx_rows, d, V, C);
  k.swz = kn.swz;
  k.ninner = kn.ninner;
  k.pol = kn.pol;
  k.pair = pair;
  k.wide = wide;
  k.dwmn = kn.dwmn != 0;
  k.dh_split = (pair & 1) ? lmb_dh_split(d, V, (wide & 1) ? 2 : 1) : 1;
  if (need_wt) {
    const dim3 grid((unsigned)((d + 63) / 64), (unsigned)((V + 63) / 64));
    lmb_gather_t<<<grid, 256, 0, s>>>(static_cast<const uint16_t*>(x->weight), x->weight_stride, d, nullptr,
                                      nullptr, V, 0, V, 0, nullptr, k.w.wt, k.Vp);
    if (cudaGetLastError() != cudaSuccess) return TBA_ERR_CUDA;
  }
  if (!make_map(&k.m_hc, k.w.hc, C, d, d, GB_BM) || !make_map(&k.m_w, x->weight, V, d, x->weight_stride, GB_BN) ||
      !make_map(&k.m_dz, k.w.dz, C, V, k.Vp, GB_BM) || !make_map(&k.m_wt, k.w.wt, d, V, k.Vp, GB_BN) ||
      (!k.dwmn && (!make_map(&k.m_dzt, k.w.dzt, V, C, C, GB_BM) || !make_map(&k.m_hct, k.w.hct, d, C, C, GB_BN))))
    return TBA_ERR_CUDA;
  if (pair && !make_map(&k.m_wt2, k.w.wt, d, V, k.Vp, 128)) return TBA_ERR_CUDA;
  if (pair && !k.dwmn && !make_map(&k.m_hct2, k.w.hct, d, C, C, 128)) return TBA_ERR_CUDA;
  // MN-major boxes {64 along V (or d), 64 rows}
  if (k.dwmn && (!make_map(&k.m_dzmn, k.w.dz, C, V, k.Vp, 64) || !make_map(&k.m_hcmn, k.w.hc, C, d, d, 64)))
    return TBA_ERR_CUDA;
  return TBA_OK;
}

// One chunk: rows idx[chunk0 + i], i < clamp(*n_valid - chunk0, 0, C). dz from a GEMM recompute
// (zst == nullptr) or from the stored fp32 logits (zst, row r at zst + (r - zrow0) * zst_ld; chunk0 = 0).
int lmb_chunk(const LmbCtx& k, const int* n_valid, int64_t chunk0, DzArgs dz, const float* zst, int64_t zst_ld,
              int64_t zrow0, void* dh, int32_t dh_dt, int64_t dh_stride, bool dh_add, float* dw, int64_t dw_stride,
              bool dw_add, cudaStream_t s) {
  const tba_lmhead* x = k.x;
  const int64_t d = x->d, V = x->vocab, C = k.C;
  const int64_t nt_v = (V + GB_BN - 1) / GB_BN, nt_d = (d + GB_BN - 1) / GB_BN;
  const dim3 ggrid((unsigned)((d + 63) / 64), (unsigned)(C / 64));
  lmb_gather_t<<<ggrid, 256, 0, s>>>(static_cast<const uint16_t*>(x->hidden), x->hidden_stride, d, k.w.idx, n_valid, 0,
                                     chunk0, C, 1, k.w.hc, (dw && !k.dwmn) ? k.w.hct : nullptr, C);
  if (cudaGetLastError() != cudaSuccess) return TBA_ERR_CUDA;
  dz.V = V;
  dz.Vp = k.Vp;
  dz.C = C;
  dz.dz = k.w.dz;
  dz.dzt = (dw && !k.dwmn) ? k.w.dzt : nullptr;
  int rc;
  if (zst) {  // 2'. dz from the stored logits (rows idx[chunk0 ..] of the group chunk's own row list)
    dz.idx = k.w.idx;
    const dim3 grid((unsigned)((V + 127) / 128), (unsigned)(C / 64));
    lmb_dz_from_z<<<grid, 256, 0, s>>>(dz, n_valid, chunk0, C, zst, zst_ld, zrow0);
    rc = launch_status();
  } else {  // 2. dz tiles recomputed: M = the chunk's rows, N = V, K = d
    GemmArgs a{};
    a.n_valid = n_valid;
    a.chunk0 = chunk0;
    a.cap = C;
    a.M = C;
    a.N = V;
    a.K = d;
    a.dyn = 1;
    a.swz = k.swz;
    a.n_inner = 0;
    a.pol = 2;  // the weight tiles are shared by the row blocks in flight
    dz.idx = k.w.idx;
    a.dz = dz;
    rc = launch_gemm<EPI_DZ>(k.m_hc, k.m_w, a, (C / GB_BM) * nt_v, s);
  }
  if (rc) return rc;
  if (dh) {  // 3. dH rows = dZ W: M = the chunk's rows, N = d, K = V
    GemmArgs b{};
    b.n_valid = n_valid;
    b.chunk0 = chunk0;
    b.cap = C;
    b.M = C;
    b.N = d;
    b.K = V;
    b.dyn = 1;
    b.swz = k.swz;
    b.n_inner = k.ninner & 1;
    b.pol = k.pol & 3;
    const int64_t esz = dh_dt == TBA_BF16 ? 2 : 4;
    b.st = StoreArgs{dh, dh_stride, k.w.idx + chunk0, dh_dt == TBA_BF16, dh_add ? 1 : 0,
                     ((reinterpret_cast<uintptr_t>(dh) | (uintptr_t)(dh_stride * esz)) & 15) == 0};
    if (k.pair & 1) {
      b.ksplit = k.dh_split;
      b.part = k.w.part;
      b.part_ld = lmb_dp(d);
      const int64_t units = (C / 256 + 1) * nt_d * k.dh_split;
      rc = (k.wide & 1) ? launch_gemm2<2>(k.m_dz, k.m_wt2, b, units, s) : launch_gemm2<1>(k.m_dz, k.m_wt2, b, units, s);
      if (!rc && k.dh_split > 1) {
        const dim3 rg((unsigned)(((d + 3) / 4 + 255) / 256), (unsigned)(C < 65535 ? C : 65535));
        lmb_splitk_reduce<<<rg, 256, 0, s>>>(k.w.part, b.part_ld, k.dh_split, C, n_valid, chunk0, d, b.st);
        rc = launch_status();
      }
    } else {
      rc = launch_gemm<EPI_STORE>(k.m_dz, k.m_wt, b, (C / GB_BM) * nt_d, s);
    }
    if (rc) return rc;
  }
  if (dw) {  // 4. dW (+)= dZ^T H: M = V, N = d, K = the chunk's rows
    GemmArgs b{};
    b.n_valid = n_valid;
    b.chunk0 = chunk0;
    b.cap = C;
    b.M = V;
    b.N = d;
    b.K = C;
    b.dyn = 2;
    b.swz = k.swz;
    b.n_inner = (k.ninner >> 1) & 1;
    b.pol = (k.pol >> 2) & 3;
    b.st = StoreArgs{dw, dw_stride, nullptr, 0, dw_add ? 1 : 0,
                     ((reinterpret_cast<uintptr_t>(dw) | (uintptr_t)(dw_stride * 4)) & 15) == 0};
    const int64_t mt = ((V + 255) / 256) * nt_d;
    rc = k.dwmn ? ((k.wide & 2) ? launch_gemm2<2, true>(k.m_dzmn, k.m_hcmn, b, mt, s)
                                : launch_gemm2<1, true>(k.m_dzmn, k.m_hcmn, b, mt, s))
         : (k.pair & 2) ? ((k.wide & 2) ? launch_gemm2<2>(k.m_dzt, k.m_hct2, b, mt, s)
                                      : launch_gemm2<1>(k.m_dzt, k.m_hct2, b, mt, s))
                      : launch_gemm<EPI_STORE>(k.m_dzt, k.m_hct, b, ((V + GB_BM - 1) / GB_BM) * nt_d, s);
  }
  return rc;
}

int lmb_zero_outputs(const tba_lmhead* x, int64_t rows, void* dh, int32_t dh_dt, int64_t dh_stride, float* dw,
                     int64_t dw_stride, bool zero_dw, cudaStream_t s) {
  const size_t esz = dh_dt == TBA_BF16 ? 2 : 4;
  if (dh && rows > 0 &&
      cudaMemset2DAsync(dh, (size_t)dh_stride * esz, 0, (size_t)x->d * esz, (size_t)rows, s) != cudaSuccess)
    return TBA_ERR_CUDA;
  if (dw && zero_dw &&
      cudaMemset2DAsync(dw, (size_t)dw_stride * 4, 0, (size_t)x->d * 4, (size_t)x->vocab, s) != cudaSuccess)
    return TBA_ERR_CUDA;
  return TBA_OK;
}

DzArgs dz_args(const tba_lmhead* x, const float2* stats, const double* resid, const float* coef, double gs,
               const double* grad_out, float sc) {
  DzArgs z{};
  z.stats = stats;
  z.tokens = x->tokens;
  z.resid = resid;
  z.coef = coef;
  z.T = x->seq_len;
  z.gs = gs;
  z.grad_out = grad_out;
  z.sc = sc;
  return z;
}

}  // namespace

int launch_lmhead_bwd(const tba_lmhead* x, const float2* stats, const double* resid, const float* coef, double gs,
                      const double* grad_out, float sc, void* dh, int32_t dh_dt, int64_t dh_stride, float* dw,
                      int64_t dw_stride, bool accumulate, int64_t chunk_rows, void* bws, cudaStream_t s) {
  const int64_t rows = x->n_seq * x->seq_len;
  if (!accumulate) {
    const int rc = lmb_zero_outputs(x, rows, dh, dh_dt, dh_stride, dw, dw_stride, rows == 0, s);
    if (rc) return rc;
  }
  if (rows == 0 || (!dh && !dw)) return TBA_OK;
  LmbCtx k;
  int rc = lmb_prepare(k, x, rows, lmhead_bwd_chunk(rows, chunk_rows), bws, dh != nullptr, s);
  if (rc) return rc;
  int* n_valid = k.w.idx + rows;
  lmb_compact_rows<<<1, 1024, 0, s>>>(x->mask, rows, 0, k.w.idx, n_valid);
  if (cudaGetLastError() != cudaSuccess) return TBA_ERR_CUDA;
  const DzArgs dz = dz_args(x, stats, resid, coef, gs, grad_out, sc);
  const int64_t n_chunks = (rows + k.C - 1) / k.C;
  for (int64_t ch = 0; ch < n_chunks && !rc; ++ch)
    rc = lmb_chunk(k, n_valid, ch * k.C, dz, nullptr, 0, 0, dh, dh_dt, dh_stride, accumulate, dw, dw_stride,
                   accumulate || ch > 0, s);
  return rc;
}

// ---- one-call forward + backward: chunks of whole groups, logits stored once (fp32) per chunk
int64_t lmhead_fb_groups(int64_t groups, int64_t rows_per_group, int32_t groups_per_chunk) {
  int64_t g = groups_per_chunk > 0 ? groups_per_chunk : LMB_DEFAULT_CHUNK / (rows_per_group > 0 ? rows_per_group : 1);
  if (g < 1) g = 1;
  if (g > groups) g = groups;
  return g < 1 ? 1 : g;
}

size_t lmhead_fb_ws_bytes(int64_t n_seq, int64_t T, int64_t d, int64_t V, int32_t K, int32_t groups_per_chunk) {
  const int64_t gpc = lmhead_fb_groups(n_seq / K, (int64_t)K * T, groups_per_chunk);
  const int64_t R = gpc * K * T;  // rows per chunk (all stored as fp32 logits)
  const int64_t C = lmhead_bwd_chunk(R, R < LMB_DEFAULT_CHUNK ? R : LMB_DEFAULT_CHUNK);  // GEMM sub-chunk
  return lmhead_bwd_ws_bytes(R, d, V, C) + align_up((size_t)R * (size_t)lmb_vp(V) * 4, 256) +
         lmhead_partial_bytes(R, V);
}

int launch_lmhead_fwd_bwd(const tba_lmhead* x, const RowScale& rs, const WsLayout& w, const HeadArgs& ha0, int32_t K,
                          double grad_scale, double inv_n_global, void* dh, int32_t dh_dt, int64_t dh_stride, float* dw,
                          int64_t dw_stride, bool accumulate, int32_t groups_per_chunk, void* bws,
                          int32_t* dev_status, cudaStream_t s) {
  const int64_t T = x->seq_len, groups = x->n_seq / K, rows = x->n_seq * T;
  const int64_t gpc = lmhead_fb_groups(groups, (int64_t)K * T, groups_per_chunk);
  // R rows per group chunk (their fp32 logits stored); the compaction / GEMM chunk C is capped at
  // LMB_DEFAULT_CHUNK, so one group larger than that (Table 5: K = 16 x T = 2048) runs as several
  // sub-chunks of its stored logits instead of growing every backward buffer with the group.
  const int64_t R = gpc * K * T, C = lmhead_bwd_chunk(R, R < LMB_DEFAULT_CHUNK ? R : LMB_DEFAULT_CHUNK);
  int rc = TBA_OK;
  if (!accumulate) rc = lmb_zero_outputs(x, rows, dh, dh_dt, dh_stride, dw, dw_stride, false, s);
  if (rc) return rc;
  LmbCtx k;
  rc = lmb_prepare(k, x, R, C, bws, dh != nullptr, s);
  if (rc) return rc;
  char* tail = static_cast<char*>(bws) + lmhead_bwd_ws_bytes(R, x->d, x->vocab, C);
  float* zst = reinterpret_cast<float*>(tail);
  void* part_ws = tail + align_up((size_t)R * (size_t)k.Vp * 4, 256);
  int* n_valid = k.w.idx + R;
  const DzArgs dz0 = dz_args(x, w.stats, ha0.resid, nullptr, grad_scale * rs.inv_temp, nullptr, rs.sc);
  const int64_t n_chunks = (groups + gpc - 1) / gpc;
  for (int64_t c = 0; c < n_chunks && !rc; ++c) {
    const int64_t g0 = c * gpc, gc = (g0 + gpc <= groups) ? gpc : groups - g0;
    const int64_t s0 = g0 * K, r0 = s0 * T, rc_rows = gc * K * T;
    tba_lmhead xc = *x;
    xc.hidden = static_cast<const uint16_t*>(x->hidden) + r0 * x->hidden_stride;
    xc.tokens = x->tokens + r0;
    xc.mask = x->mask + r0;
    xc.n_seq = gc * K;
    const WsLayout wc{w.stats + r0, w.lp + r0, w.group_sq + g0, nullptr, nullptr, w.qy + r0};
    // forward of the chunk, logits kept (row r0 + i at zst + i * Vp)
    rc = launch_lmhead_rows(&xc, part_ws, wc, rs, dev_status, s, zst, k.Vp);
    if (rc) break;
    HeadArgs ha = ha0;
    ha.n_seq = xc.n_seq;
    ha.ref_logp += s0;
    ha.log_reward += s0;
    ha.seq_logp += s0;
    ha.n_tokens += s0;
    ha.log_z += g0;
    ha.resid += s0;
    ha.group_sq = wc.group_sq;
    if (ha.log_z_param) ha.log_z_param += g0;
    rc = launch_seq_head(true, wc, xc.mask, ha, s);  // wc.counter == NULL: no per-chunk reduction
    if (rc) break;
    // backward of the chunk from the stored logits
    lmb_compact_rows<<<1, 1024, 0, s>>>(xc.mask, rc_rows, r0, k.w.idx, n_valid);
    if ((rc = launch_status())) break;
    for (int64_t sub = 0; sub * C < rc_rows && !rc; ++sub)  // sub-chunks past *n_valid do no work
      rc = lmb_chunk(k, n_valid, sub * C, dz0, zst, k.Vp, r0, dh, dh_dt, dh_stride, accumulate, dw, dw_stride,
                     accumulate || c > 0 || sub > 0, s);
  }
  if (!rc) rc = launch_tb_finish(w.group_sq, groups, x->n_seq, inv_n_global, ha0.partial, s);
  return rc;
}

}  // namespace tba
