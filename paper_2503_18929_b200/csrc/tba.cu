// libtba.so — the VarGrad trajectory-balance loss head (TBA, arXiv 2503.18929) for B200.
//
// Kernels:
//   row_fwd   a1  stream each valid logits row from HBM once: online max + sum of
//                 2^(z*log2e - M2) in one MUFU ex2 per element, gather z[y]; writes per-row
//                 (M2, log2 S) and the token log-prob (fp64).
//   seq_head  a2+a3  per-sequence fixed-order fp64 sum of token log-probs (log pi(y|x)),
//                 token counts, then per group Eq. 4 log Z and the Eq. 5 residuals; the last
//                 CTA reduces the per-group sums of squares in fixed order (no float atomics).
//   row_bwd   a5  stream each valid row again: dz = c_s (1[v=y] - 2^(z*log2e - M2 - log2 S)),
//                 c_s = grad_scale * grad_out * eps_s; masked rows are zero-filled unread.
// All hot loops use 128-bit loads/stores (ld.global.nc.L1::no_allocate / st.global.cs),
// per-thread fp32 partial sums folded into fp64 every 32 elements, fp64 row finalisation.
#include <cstdint>
#include <cmath>
#include <cuda_runtime.h>

#include "../../include/tba.h"

namespace {

constexpr float kL2E = 1.4426950408889634f;  // fp32(log2 e); rows are softmax'd at this exact scale
constexpr double kLN2 = 0.69314718055994530942;

// ------------------------------------------------------------------------------ PTX helpers
__device__ __forceinline__ float ex2(float x) {
  float y;
  asm("ex2.approx.ftz.f32 %0, %1;" : "=f"(y) : "f"(x));
  return y;
}

__device__ __forceinline__ uint4 ldg_stream(const uint4* p) {
  uint4 r;
  asm volatile("ld.global.nc.L1::no_allocate.L2::256B.v4.u32 {%0, %1, %2, %3}, [%4];"
               : "=r"(r.x), "=r"(r.y), "=r"(r.z), "=r"(r.w)
               : "l"(p));
  return r;
}

__device__ __forceinline__ void stg_stream(uint4* p, uint4 v) {
  asm volatile("st.global.cs.v4.u32 [%0], {%1, %2, %3, %4};" ::"l"(p), "r"(v.x), "r"(v.y), "r"(v.z), "r"(v.w)
               : "memory");
}

// element traits: 16-byte vector of VEC elements
template <class T> struct Elem;
template <> struct Elem<uint16_t> {  // bf16 stored as raw bits
  static constexpr int VEC = 8;
  __device__ __forceinline__ static float get(const uint4& v, int e) {
    const uint32_t w = (&v.x)[e >> 1];
    return __uint_as_float((e & 1) ? (w & 0xFFFF0000u) : (w << 16));
  }
  __device__ __forceinline__ static float load1(const uint16_t* p) { return __uint_as_float(((uint32_t)__ldg(p)) << 16); }
  __device__ __forceinline__ static uint4 neg_inf() { return make_uint4(0xFF80FF80u, 0xFF80FF80u, 0xFF80FF80u, 0xFF80FF80u); }
};
template <> struct Elem<float> {
  static constexpr int VEC = 4;
  __device__ __forceinline__ static float get(const uint4& v, int e) { return __uint_as_float((&v.x)[e]); }
  __device__ __forceinline__ static float load1(const float* p) { return __ldg(p); }
  __device__ __forceinline__ static uint4 neg_inf() { return make_uint4(0xFF800000u, 0xFF800000u, 0xFF800000u, 0xFF800000u); }
};

__device__ __forceinline__ uint32_t pack_bf16x2(float lo, float hi) {
  uint32_t r;
  asm("cvt.rn.bf16x2.f32 %0, %1, %2;" : "=r"(r) : "f"(hi), "f"(lo));
  return r;
}

__device__ __forceinline__ uint16_t to_bf16(float x) {
  uint16_t r;
  asm("{ .reg .b32 t; cvt.rn.bf16x2.f32 t, %1, %1; mov.b32 {%0, _}, t; }" : "=h"(r) : "f"(x));
  return r;
}

// row split: [0, head) scalar, [head, head + nvec*VEC) 16-byte vectors, rest scalar tail
template <class T>
__device__ __forceinline__ int64_t head_elems(const T* row, int64_t V) {
  const uint64_t a = reinterpret_cast<uint64_t>(row);
  int64_t h = (int64_t)(((16u - (a & 15u)) & 15u) / sizeof(T));
  return h < V ? h : V;
}

// ------------------------------------------------------------------------------ fwd state
// Per-thread online state: m = running max, M2 = fl(m * kL2E), s = sum of 2^(fl(z*kL2E - M2))
struct OnlineState {
  float m, M2;
  double s;
  __device__ __forceinline__ void init() { m = -INFINITY; M2 = 0.f; s = 0.0; }
  __device__ __forceinline__ void raise_to(float cm) {  // called when cm > m
    const float M2n = cm * kL2E;
    s = (m == -INFINITY) ? 0.0 : s * exp2((double)M2 - (double)M2n);
    m = cm;
    M2 = M2n;
  }
  __device__ __forceinline__ void add1(float z) {
    if (z > m) raise_to(z);
    s += (double)ex2(fmaf(z, kL2E, -M2));
  }
};

template <class T, int U>
__device__ __forceinline__ void fwd_accumulate(const T* __restrict__ row, int64_t V, int tid, int nthr,
                                               OnlineState& st) {
  using E = Elem<T>;
  constexpr int VEC = E::VEC;
  const int64_t h = head_elems(row, V);
  const int64_t nvec = (V - h) / VEC;
  const int64_t tail0 = h + nvec * VEC;
  for (int64_t i = tid; i < h; i += nthr) st.add1(E::load1(row + i));
  for (int64_t i = tail0 + tid; i < V; i += nthr) st.add1(E::load1(row + i));
  const uint4* vp = reinterpret_cast<const uint4*>(row + h);
  for (int64_t k0 = tid; k0 < nvec; k0 += (int64_t)nthr * U) {
    uint4 v[U];
#pragma unroll
    for (int u = 0; u < U; ++u) {
      const int64_t k = k0 + (int64_t)u * nthr;
      v[u] = (k < nvec) ? ldg_stream(vp + k) : E::neg_inf();
    }
    float cm = -INFINITY;
#pragma unroll
    for (int u = 0; u < U; ++u)
#pragma unroll
      for (int e = 0; e < VEC; ++e) cm = fmaxf(cm, E::get(v[u], e));
    if (cm > st.m) st.raise_to(cm);
    const float nM2 = -st.M2;
    float acc[VEC];
#pragma unroll
    for (int e = 0; e < VEC; ++e) acc[e] = 0.f;
#pragma unroll
    for (int u = 0; u < U; ++u)
#pragma unroll
      for (int e = 0; e < VEC; ++e) acc[e] += ex2(fmaf(E::get(v[u], e), kL2E, nM2));
#pragma unroll
    for (int w = VEC / 2; w >= 1; w >>= 1)
#pragma unroll
      for (int e = 0; e < w; ++e) acc[e] += acc[e + w];
    st.s += (double)acc[0];
  }
}

// Combine states across the 32 lanes of a warp (result valid in every lane).
__device__ __forceinline__ void warp_combine(OnlineState& st) {
  float M = st.m;
#pragma unroll
  for (int o = 16; o >= 1; o >>= 1) M = fmaxf(M, __shfl_xor_sync(0xffffffffu, M, o));
  const float M2 = (M == -INFINITY) ? 0.f : M * kL2E;
  double s = (st.m == -INFINITY) ? 0.0 : st.s * exp2((double)st.M2 - (double)M2);
  // fixed butterfly: every lane ends with the same bits
#pragma unroll
  for (int o = 16; o >= 1; o >>= 1) s += __shfl_xor_sync(0xffffffffu, s, o);
  st.m = M;
  st.M2 = M2;
  st.s = s;
}

__device__ __forceinline__ void finalize_row(const OnlineState& st, float zy, bool tok_ok, int64_t row,
                                             float2* __restrict__ stats, double* __restrict__ lp,
                                             int32_t* dev_status) {
  const bool finite = (st.m > -INFINITY) && (st.m < INFINITY) && (st.s > 0.0) && (st.s < INFINITY);
  const double log2s = log2(st.s);
  stats[row] = make_float2(st.M2, (float)log2s);
  // lp = (z_y - M) - ln sum_v e^{kappa (z_v - M)},  kappa = kL2E / log2(e)
  double v = ((double)zy - (double)st.m) - kLN2 * (log2s + (double)st.M2 - (double)st.m * (double)kL2E);
  if (!tok_ok) v = nan("");
  lp[row] = v;
  if (dev_status) {
    int f = (tok_ok ? 0 : TBA_DEV_TOKEN_RANGE) | (finite ? 0 : TBA_DEV_NONFINITE_ROW);
    if (f) atomicOr(dev_status, f);
  }
}

// One CTA (NT threads) per row.
template <class T, int NT, int U>
__global__ void __launch_bounds__(NT) row_fwd_cta(const T* __restrict__ logits, int64_t rows, int64_t V,
                                                   int64_t stride, const int64_t* __restrict__ tokens,
                                                   const uint8_t* __restrict__ mask, float2* __restrict__ stats,
                                                   double* __restrict__ lp, int32_t* dev_status) {
  const int64_t row = blockIdx.x;
  if (row >= rows || mask[row] == 0) return;
  const T* rp = logits + row * stride;
  OnlineState st;
  st.init();
  fwd_accumulate<T, U>(rp, V, threadIdx.x, NT, st);
  warp_combine(st);
  __shared__ float sm_m[NT / 32], sm_M2[NT / 32];
  __shared__ double sm_s[NT / 32];
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  if (lane == 0) {
    sm_m[warp] = st.m;
    sm_M2[warp] = st.M2;
    sm_s[warp] = st.s;
  }
  __syncthreads();
  if (threadIdx.x == 0) {
    OnlineState tot;
    tot.init();
    for (int w = 0; w < NT / 32; ++w) tot.m = fmaxf(tot.m, sm_m[w]);
    tot.M2 = (tot.m == -INFINITY) ? 0.f : tot.m * kL2E;
    double s = 0.0;
    for (int w = 0; w < NT / 32; ++w)
      if (sm_m[w] > -INFINITY) s += sm_s[w] * exp2((double)sm_M2[w] - (double)tot.M2);
    tot.s = s;
    const int64_t y = tokens[row];
    const bool ok = (y >= 0 && y < V);
    const float zy = ok ? Elem<T>::load1(rp + y) : 0.f;
    finalize_row(tot, zy, ok, row, stats, lp, dev_status);
  }
}

// One warp per row, NT/32 rows per CTA (small vocabularies).
template <class T, int NT, int U>
__global__ void __launch_bounds__(NT) row_fwd_warp(const T* __restrict__ logits, int64_t rows, int64_t V,
                                                    int64_t stride, const int64_t* __restrict__ tokens,
                                                    const uint8_t* __restrict__ mask, float2* __restrict__ stats,
                                                    double* __restrict__ lp, int32_t* dev_status) {
  const int64_t row = (int64_t)blockIdx.x * (NT / 32) + (threadIdx.x >> 5);
  const int lane = threadIdx.x & 31;
  if (row >= rows || mask[row] == 0) return;  // warp-uniform
  const T* rp = logits + row * stride;
  OnlineState st;
  st.init();
  fwd_accumulate<T, U>(rp, V, lane, 32, st);
  warp_combine(st);
  if (lane == 0) {
    const int64_t y = tokens[row];
    const bool ok = (y >= 0 && y < V);
    const float zy = ok ? Elem<T>::load1(rp + y) : 0.f;
    finalize_row(st, zy, ok, row, stats, lp, dev_status);
  }
}

// ------------------------------------------------------------------------------ a2 + a3
// One CTA per group of K sequences (or per 8 sequences when !HEAD). Warps sum the token
// log-probs of one sequence each in a fixed order (lane-strided fp64 + xor butterfly).
template <bool HEAD>
__global__ void __launch_bounds__(256) seq_head(const double* __restrict__ lp, const uint8_t* __restrict__ mask,
                                                int64_t n_seq, int64_t T, int K, const double* __restrict__ ref_logp,
                                                const double* __restrict__ log_reward, double inv_beta,
                                                double inv_n_global, double* __restrict__ seq_logp,
                                                int32_t* __restrict__ n_tokens, double* __restrict__ log_z,
                                                double* __restrict__ resid, double* __restrict__ group_sq,
                                                double* __restrict__ partial, unsigned int* counter) {
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int per = HEAD ? K : 8;
  const int64_t s0 = (int64_t)blockIdx.x * per;
  for (int j = warp; j < per; j += 8) {
    const int64_t s = s0 + j;
    if (s >= n_seq) break;
    double acc = 0.0;
    int cnt = 0;
    for (int64_t t = lane; t < T; t += 32) {
      const int64_t r = s * T + t;
      if (mask[r]) {
        acc += lp[r];
        ++cnt;
      }
    }
#pragma unroll
    for (int o = 16; o >= 1; o >>= 1) {
      acc += __shfl_xor_sync(0xffffffffu, acc, o);
      cnt += __shfl_xor_sync(0xffffffffu, cnt, o);
    }
    if (lane == 0) {
      seq_logp[s] = acc;
      n_tokens[s] = cnt;
    }
  }
  if (!HEAD) return;
  __syncthreads();
  __shared__ bool am_last;
  if (threadIdx.x == 0) {
    // Eq. 4: log Z_i = 1/K sum_j delta_j, delta = rho - ell + r/beta; Eq. 5 residual eps = log Z - delta
    double sum = 0.0;
    for (int j = 0; j < K; ++j) {
      const int64_t s = s0 + j;
      sum += ref_logp[s] - seq_logp[s] + log_reward[s] * inv_beta;
    }
    const double lz = sum / (double)K;
    double sq = 0.0;
    for (int j = 0; j < K; ++j) {
      const int64_t s = s0 + j;
      const double delta = ref_logp[s] - seq_logp[s] + log_reward[s] * inv_beta;
      const double e = lz - delta;
      resid[s] = e;
      sq += e * e;
    }
    log_z[blockIdx.x] = lz;
    group_sq[blockIdx.x] = sq;
    __threadfence();
    am_last = (atomicAdd(counter, 1u) == gridDim.x - 1);
  }
  __syncthreads();
  if (am_last && threadIdx.x == 0) {
    __threadfence();
    const volatile double* gs = group_sq;
    double tot = 0.0;
    for (unsigned i = 0; i < gridDim.x; ++i) tot += gs[i];
    partial[0] = tot * inv_n_global;
    partial[1] = (double)n_seq;
    partial[2] = (double)gridDim.x;
    *counter = 0u;
  }
}

// ------------------------------------------------------------------------------ a5
template <class TO> struct Out;
template <> struct Out<uint16_t> {
  static constexpr int VEC = 8;  // outputs per 16-byte store
  __device__ __forceinline__ static void put1(uint16_t* p, float x) { *p = to_bf16(x); }
};
template <> struct Out<float> {
  static constexpr int VEC = 4;
  __device__ __forceinline__ static void put1(float* p, float x) { __stcs(p, x); }
};

// store VEC_IN computed values starting at o (16-byte aligned for the first element)
template <class TO, int N>
__device__ __forceinline__ void store_vals(TO* o, const float (&d)[N]) {
  if constexpr (sizeof(TO) == 2) {
    static_assert(N == 8 || N == 4, "");
    if constexpr (N == 8) {
      uint4 w = make_uint4(pack_bf16x2(d[0], d[1]), pack_bf16x2(d[2], d[3]), pack_bf16x2(d[4], d[5]),
                           pack_bf16x2(d[6], d[7]));
      stg_stream(reinterpret_cast<uint4*>(o), w);
    } else {
      uint2 w = make_uint2(pack_bf16x2(d[0], d[1]), pack_bf16x2(d[2], d[3]));
      asm volatile("st.global.cs.v2.u32 [%0], {%1, %2};" ::"l"(o), "r"(w.x), "r"(w.y) : "memory");
    }
  } else {
#pragma unroll
    for (int q = 0; q < N / 4; ++q)
      stg_stream(reinterpret_cast<uint4*>(o) + q,
                 make_uint4(__float_as_uint(d[4 * q]), __float_as_uint(d[4 * q + 1]), __float_as_uint(d[4 * q + 2]),
                            __float_as_uint(d[4 * q + 3])));
  }
}

template <class T, class TO, int U>
__device__ __forceinline__ void bwd_row(const T* __restrict__ rp, TO* __restrict__ op, int64_t V, int tid, int nthr,
                                        bool valid, float M2, float L2S, float c, int64_t y) {
  using E = Elem<T>;
  constexpr int VEC = E::VEC;
  const int64_t h = head_elems(rp, V);
  // vector path needs the output 16-byte aligned at the same element as the input
  const bool vec_ok = ((reinterpret_cast<uint64_t>(op + h) & 15u) == 0);
  const int64_t nvec = vec_ok ? (V - h) / VEC : 0;
  const int64_t vend = h + nvec * VEC;
  auto one = [&](int64_t i) {
    float d = 0.f;
    if (valid) {
      const float p = ex2(fmaf(E::load1(rp + i), kL2E, -M2) - L2S);
      d = (i == y) ? fmaf(-c, p, c) : -c * p;
    }
    Out<TO>::put1(op + i, d);
  };
  for (int64_t i = tid; i < (vec_ok ? h : V); i += nthr) one(i);
  if (!vec_ok) return;
  for (int64_t i = vend + tid; i < V; i += nthr) one(i);
  const uint4* vp = reinterpret_cast<const uint4*>(rp + h);
  TO* ob = op + h;
  if (!valid) {
    float z[VEC];
#pragma unroll
    for (int e = 0; e < VEC; ++e) z[e] = 0.f;
    for (int64_t k = tid; k < nvec; k += nthr) store_vals<TO, VEC>(ob + k * VEC, z);
    return;
  }
  const float nM2 = -M2;
  const int64_t ky = (y >= h && y < vend) ? (y - h) / VEC : -1;
  for (int64_t k0 = tid; k0 < nvec; k0 += (int64_t)nthr * U) {
    uint4 v[U];
#pragma unroll
    for (int u = 0; u < U; ++u) {
      const int64_t k = k0 + (int64_t)u * nthr;
      if (k < nvec) v[u] = ldg_stream(vp + k);
    }
#pragma unroll
    for (int u = 0; u < U; ++u) {
      const int64_t k = k0 + (int64_t)u * nthr;
      if (k < nvec) {
        float d[VEC];
#pragma unroll
        for (int e = 0; e < VEC; ++e) d[e] = -c * ex2(fmaf(E::get(v[u], e), kL2E, nM2) - L2S);
        if (k == ky) {
          const int e = (int)((y - h) - k * VEC);
#pragma unroll
          for (int q = 0; q < VEC; ++q)
            if (q == e) d[q] += c;
        }
        store_vals<TO, VEC>(ob + k * VEC, d);
      }
    }
  }
}

template <class T, class TO, int NT, int U, bool WARP>
__global__ void __launch_bounds__(NT) row_bwd(const T* __restrict__ logits, int64_t rows, int64_t T_len, int64_t V,
                                               int64_t stride, const int64_t* __restrict__ tokens,
                                               const uint8_t* __restrict__ mask, const float2* __restrict__ stats,
                                               const double* __restrict__ resid, double grad_scale,
                                               const double* __restrict__ grad_out, TO* __restrict__ dlogits,
                                               int64_t ostride) {
  const int64_t row = WARP ? (int64_t)blockIdx.x * (NT / 32) + (threadIdx.x >> 5) : (int64_t)blockIdx.x;
  if (row >= rows) return;
  const int tid = WARP ? (threadIdx.x & 31) : threadIdx.x;
  const int nthr = WARP ? 32 : NT;
  const bool valid = mask[row] != 0;
  float M2 = 0.f, L2S = 0.f, c = 0.f;
  int64_t y = -1;
  if (valid) {
    const float2 st = stats[row];
    M2 = st.x;
    L2S = st.y;
    const double g = grad_out ? *grad_out : 1.0;
    c = (float)(grad_scale * g * resid[row / T_len]);
    y = tokens[row];
  }
  bwd_row<T, TO, U>(logits + row * stride, dlogits + row * ostride, V, tid, nthr, valid, M2, L2S, c, y);
}

// ------------------------------------------------------------------------------ host side
constexpr int kNT = 256;
constexpr int kU = 4;
constexpr int64_t kWarpRowMaxBytes = 8192;  // rows up to 8 KB use one warp per row

struct WsLayout {
  float2* stats;
  double* lp;
  double* group_sq;
  unsigned int* counter;
};

inline size_t align_up(size_t x, size_t a) { return (x + a - 1) / a * a; }

WsLayout ws_layout(void* ws, int64_t n_seq, int64_t T) {
  const size_t rows = (size_t)n_seq * (size_t)T;
  char* p = static_cast<char*>(ws);
  WsLayout l;
  size_t off = 0;
  l.stats = reinterpret_cast<float2*>(p + off);
  off = align_up(off + rows * sizeof(float2), 256);
  l.lp = reinterpret_cast<double*>(p + off);
  off = align_up(off + rows * sizeof(double), 256);
  l.group_sq = reinterpret_cast<double*>(p + off);
  off = align_up(off + (size_t)n_seq * sizeof(double), 256);
  l.counter = reinterpret_cast<unsigned int*>(p + off);
  return l;
}

size_t ws_bytes(int64_t n_seq, int64_t T) {
  const size_t rows = (size_t)n_seq * (size_t)T;
  return align_up(rows * sizeof(float2), 256) + align_up(rows * sizeof(double), 256) +
         align_up((size_t)n_seq * sizeof(double), 256) + 256;
}

int validate_rows(const tba_rows* x) {
  if (!x) return TBA_ERR_INVALID_ARG;
  if (x->dtype != TBA_BF16 && x->dtype != TBA_FP32) return TBA_ERR_INVALID_ARG;
  if (x->n_seq < 0 || x->seq_len < 0 || x->vocab < 1 || x->row_stride < x->vocab) return TBA_ERR_INVALID_ARG;
  const int64_t esz = x->dtype == TBA_BF16 ? 2 : 4;
  const int64_t lim = INT64_MAX / 8;
  if (x->n_seq > 0 && x->seq_len > lim / x->n_seq) return TBA_ERR_INVALID_ARG;
  const int64_t rows = x->n_seq * x->seq_len;
  if (rows > 0 && x->row_stride > lim / esz / rows) return TBA_ERR_INVALID_ARG;
  if (rows > (int64_t)INT32_MAX * 1024) return TBA_ERR_INVALID_ARG;
  if (rows > 0) {
    if (!x->logits || !x->tokens || !x->mask) return TBA_ERR_INVALID_ARG;
    if (reinterpret_cast<uintptr_t>(x->logits) % esz) return TBA_ERR_INVALID_ARG;
    if (reinterpret_cast<uintptr_t>(x->tokens) % 8) return TBA_ERR_INVALID_ARG;
  }
  return TBA_OK;
}

int launch_fwd_rows(const tba_rows* x, const WsLayout& w, int32_t* dev_status, cudaStream_t s) {
  const int64_t rows = x->n_seq * x->seq_len;
  if (rows == 0) return TBA_OK;
  const int64_t V = x->vocab, stride = x->row_stride;
  const int64_t esz = x->dtype == TBA_BF16 ? 2 : 4;
  const bool warp = V * esz <= kWarpRowMaxBytes;
  const int64_t grid = warp ? (rows + kNT / 32 - 1) / (kNT / 32) : rows;
  if (x->dtype == TBA_BF16) {
    auto lg = static_cast<const uint16_t*>(x->logits);
    if (warp)
      row_fwd_warp<uint16_t, kNT, kU><<<(unsigned)grid, kNT, 0, s>>>(lg, rows, V, stride, x->tokens, x->mask, w.stats,
                                                                    w.lp, dev_status);
    else
      row_fwd_cta<uint16_t, kNT, kU><<<(unsigned)grid, kNT, 0, s>>>(lg, rows, V, stride, x->tokens, x->mask, w.stats,
                                                                   w.lp, dev_status);
  } else {
    auto lg = static_cast<const float*>(x->logits);
    if (warp)
      row_fwd_warp<float, kNT, kU><<<(unsigned)grid, kNT, 0, s>>>(lg, rows, V, stride, x->tokens, x->mask, w.stats,
                                                                 w.lp, dev_status);
    else
      row_fwd_cta<float, kNT, kU><<<(unsigned)grid, kNT, 0, s>>>(lg, rows, V, stride, x->tokens, x->mask, w.stats,
                                                                w.lp, dev_status);
  }
  return cudaGetLastError() == cudaSuccess ? TBA_OK : TBA_ERR_CUDA;
}

template <class T, class TO>
void launch_bwd_t(const tba_rows* x, const WsLayout& w, const double* resid, double gs, const double* go, TO* out,
                  int64_t ostride, cudaStream_t s) {
  const int64_t rows = x->n_seq * x->seq_len;
  const bool warp = x->vocab * (int64_t)sizeof(T) <= kWarpRowMaxBytes;
  auto lg = static_cast<const T*>(x->logits);
  if (warp) {
    const int64_t grid = (rows + kNT / 32 - 1) / (kNT / 32);
    row_bwd<T, TO, kNT, kU, true><<<(unsigned)grid, kNT, 0, s>>>(lg, rows, x->seq_len, x->vocab, x->row_stride,
                                                                 x->tokens, x->mask, w.stats, resid, gs, go, out,
                                                                 ostride);
  } else {
    row_bwd<T, TO, kNT, kU, false><<<(unsigned)rows, kNT, 0, s>>>(lg, rows, x->seq_len, x->vocab, x->row_stride,
                                                                  x->tokens, x->mask, w.stats, resid, gs, go, out,
                                                                  ostride);
  }
}

}  // namespace

// ================================================================================ C ABI
extern "C" {

int tba_abi_version(void) { return TBA_ABI_VERSION; }

const char* tba_status_string(int code) {
  switch (code) {
    case TBA_OK: return "TBA_OK";
    case TBA_ERR_INVALID_ARG: return "TBA_ERR_INVALID_ARG: invalid argument (null pointer, size, stride, alignment or N % K)";
    case TBA_ERR_INVALID_CONFIG: return "TBA_ERR_INVALID_CONFIG: invalid configuration (beta must be finite and > 0, K >= 2)";
    case TBA_ERR_CUDA: return "TBA_ERR_CUDA: CUDA launch failed";
    default: return "TBA: unknown status";
  }
}

size_t tba_workspace_bytes(int64_t n_seq, int64_t seq_len) {
  if (n_seq < 0 || seq_len < 0) return 0;
  return ws_bytes(n_seq, seq_len);
}

int tba_seq_logprob(const tba_rows* x, void* workspace, double* seq_logp, int32_t* n_tokens, int32_t* dev_status,
                    tba_stream_t stream) {
  int rc = validate_rows(x);
  if (rc) return rc;
  if (x->n_seq == 0) return TBA_OK;
  if (!workspace || !seq_logp || !n_tokens) return TBA_ERR_INVALID_ARG;
  if (reinterpret_cast<uintptr_t>(workspace) % 256) return TBA_ERR_INVALID_ARG;
  cudaStream_t s = reinterpret_cast<cudaStream_t>(stream);
  WsLayout w = ws_layout(workspace, x->n_seq, x->seq_len);
  rc = launch_fwd_rows(x, w, dev_status, s);
  if (rc) return rc;
  const int64_t grid = (x->n_seq + 7) / 8;
  seq_head<false><<<(unsigned)grid, 256, 0, s>>>(w.lp, x->mask, x->n_seq, x->seq_len, 8, nullptr, nullptr, 0.0, 0.0,
                                                 seq_logp, n_tokens, nullptr, nullptr, nullptr, nullptr, nullptr);
  return cudaGetLastError() == cudaSuccess ? TBA_OK : TBA_ERR_CUDA;
}

int tba_vargrad_tb_loss_fwd(const tba_rows* x, const double* ref_logp, const double* log_reward, double beta,
                            int32_t K, double n_seq_global, void* workspace, double* seq_logp, int32_t* n_tokens,
                            double* log_z, double* resid, double* partial, int32_t* dev_status,
                            tba_stream_t stream) {
  if (!(std::isfinite(beta) && beta > 0.0)) return TBA_ERR_INVALID_CONFIG;
  if (K < 2) return TBA_ERR_INVALID_CONFIG;
  int rc = validate_rows(x);
  if (rc) return rc;
  if (x->n_seq % K) return TBA_ERR_INVALID_ARG;
  if (!(std::isfinite(n_seq_global) && n_seq_global >= (double)x->n_seq && n_seq_global > 0.0))
    return TBA_ERR_INVALID_ARG;
  if (!partial) return TBA_ERR_INVALID_ARG;
  cudaStream_t s = reinterpret_cast<cudaStream_t>(stream);
  if (x->n_seq == 0) {  // a rank with zero groups contributes zero partials
    return cudaMemsetAsync(partial, 0, 3 * sizeof(double), s) == cudaSuccess ? TBA_OK : TBA_ERR_CUDA;
  }
  if (!workspace || !ref_logp || !log_reward || !seq_logp || !n_tokens || !log_z || !resid)
    return TBA_ERR_INVALID_ARG;
  if (reinterpret_cast<uintptr_t>(workspace) % 256) return TBA_ERR_INVALID_ARG;
  WsLayout w = ws_layout(workspace, x->n_seq, x->seq_len);
  if (cudaMemsetAsync(w.counter, 0, sizeof(unsigned int), s) != cudaSuccess) return TBA_ERR_CUDA;
  rc = launch_fwd_rows(x, w, dev_status, s);
  if (rc) return rc;
  const int64_t groups = x->n_seq / K;
  seq_head<true><<<(unsigned)groups, 256, 0, s>>>(w.lp, x->mask, x->n_seq, x->seq_len, K, ref_logp, log_reward,
                                                  1.0 / beta, 1.0 / n_seq_global, seq_logp, n_tokens, log_z, resid,
                                                  w.group_sq, partial, w.counter);
  return cudaGetLastError() == cudaSuccess ? TBA_OK : TBA_ERR_CUDA;
}

int tba_vargrad_tb_loss_bwd(const tba_rows* x, const void* workspace, const double* resid, double grad_scale,
                            const double* grad_out, void* dlogits, int32_t dlogits_dtype, int64_t dlogits_row_stride,
                            tba_stream_t stream) {
  int rc = validate_rows(x);
  if (rc) return rc;
  if (dlogits_dtype != TBA_BF16 && dlogits_dtype != TBA_FP32) return TBA_ERR_INVALID_ARG;
  if (dlogits_row_stride < x->vocab) return TBA_ERR_INVALID_ARG;
  if (!std::isfinite(grad_scale)) return TBA_ERR_INVALID_ARG;
  const int64_t rows = x->n_seq * x->seq_len;
  if (rows == 0) return TBA_OK;
  const int64_t oesz = dlogits_dtype == TBA_BF16 ? 2 : 4;
  if (dlogits_row_stride > INT64_MAX / 8 / oesz / rows) return TBA_ERR_INVALID_ARG;
  if (!workspace || !resid || !dlogits) return TBA_ERR_INVALID_ARG;
  if (reinterpret_cast<uintptr_t>(workspace) % 256 || reinterpret_cast<uintptr_t>(dlogits) % oesz)
    return TBA_ERR_INVALID_ARG;
  if (dlogits == x->logits && (dlogits_dtype != x->dtype || dlogits_row_stride != x->row_stride))
    return TBA_ERR_INVALID_ARG;  // aliasing is only supported element-for-element
  cudaStream_t s = reinterpret_cast<cudaStream_t>(stream);
  WsLayout w = ws_layout(const_cast<void*>(workspace), x->n_seq, x->seq_len);
  if (x->dtype == TBA_BF16) {
    if (dlogits_dtype == TBA_BF16)
      launch_bwd_t<uint16_t, uint16_t>(x, w, resid, grad_scale, grad_out, static_cast<uint16_t*>(dlogits),
                                       dlogits_row_stride, s);
    else
      launch_bwd_t<uint16_t, float>(x, w, resid, grad_scale, grad_out, static_cast<float*>(dlogits),
                                    dlogits_row_stride, s);
  } else {
    if (dlogits_dtype == TBA_BF16)
      launch_bwd_t<float, uint16_t>(x, w, resid, grad_scale, grad_out, static_cast<uint16_t*>(dlogits),
                                    dlogits_row_stride, s);
    else
      launch_bwd_t<float, float>(x, w, resid, grad_scale, grad_out, static_cast<float*>(dlogits), dlogits_row_stride,
                                 s);
  }
  return cudaGetLastError() == cudaSuccess ? TBA_OK : TBA_ERR_CUDA;
}

}  // extern "C"
