// CUDA twin of tba_synth (the seeded input generator). Bit-identical to the NumPy twin in
// tba_synth/__init__.py: same SplitMix64 counter hash, same Irwin-Hall logits, same peak,
// same integer round-to-nearest-even to bf16. Holds none of the method's arithmetic; it only
// fills device buffers with synthetic logits so that 20 GB inputs need not cross PCIe.
#include <cstdint>
#include <cstring>
#include <cuda_runtime.h>

namespace {

constexpr uint64_t GAMMA = 0x9E3779B97F4A7C15ull;

__host__ __device__ __forceinline__ uint64_t mix64(uint64_t z) {
  z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ull;
  z = (z ^ (z >> 27)) * 0x94D049BB133111EBull;
  return z ^ (z >> 31);
}

__host__ __device__ __forceinline__ uint64_t hash_at(uint64_t key, uint64_t i) { return mix64(key + (i + 1) * GAMMA); }

__host__ __device__ __forceinline__ float irwin_hall(uint64_t h) {
  int64_t acc = (int64_t)(h & 0xFFFF) + (int64_t)((h >> 16) & 0xFFFF) + (int64_t)((h >> 32) & 0xFFFF) +
                (int64_t)((h >> 48) & 0xFFFF) - 131070;
  return (float)((double)acc * (1.0 / 16384.0));
}

__host__ __device__ __forceinline__ uint32_t f32_bits(float x) {
#ifdef __CUDA_ARCH__
  return __float_as_uint(x);
#else
  uint32_t b;
  std::memcpy(&b, &x, 4);
  return b;
#endif
}

__host__ __device__ __forceinline__ uint64_t umulhi64(uint64_t a, uint64_t b) {
#ifdef __CUDA_ARCH__
  return __umul64hi(a, b);
#else
  return (uint64_t)(((unsigned __int128)a * b) >> 64);
#endif
}

__host__ __device__ __forceinline__ uint16_t bf16_rne(float x) {
  uint32_t b = f32_bits(x);
  return (uint16_t)((b + 0x7FFFu + ((b >> 16) & 1u)) >> 16);
}

template <bool BF16>
__global__ void synth_logits_kernel(void* out, uint64_t key_logits, uint64_t key_tok, uint64_t key_peak,
                                    int64_t row0, int64_t nrows, int64_t V, int64_t row_stride) {
  for (int64_t r = blockIdx.y; r < nrows; r += gridDim.y) {
    const uint64_t grow = (uint64_t)(row0 + r);
    const uint64_t y = umulhi64(hash_at(key_tok, grow), (uint64_t)V);
    const float peak = (float)(4 * (int)(hash_at(key_peak, grow) & 3ull));
    for (int64_t c = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; c < row_stride;
         c += (int64_t)gridDim.x * blockDim.x) {
      const int64_t o = r * row_stride + c;
      if (c >= V) {
        if (BF16) ((uint16_t*)out)[o] = 0x7FC0u;
        else ((uint32_t*)out)[o] = 0x7FC00000u;
        continue;
      }
      float z = irwin_hall(hash_at(key_logits, grow * (uint64_t)V + (uint64_t)c));
      if ((uint64_t)c == y) z = z + peak;
      if (BF16) ((uint16_t*)out)[o] = bf16_rne(z);
      else ((float*)out)[o] = z;
    }
  }
}

// LM-head inputs (hidden states / weight rows): element (r, i) from hash(key, r*d + i).
// kind 0: Irwin-Hall(4) * 2^scale_exp; kind 1: lattice {-2..2}/4. bf16 by integer RNE.
__global__ void synth_bf16_kernel(uint16_t* out, uint64_t key, int64_t row0, int64_t nrows, int64_t d,
                                  int64_t row_stride, int kind, double scale) {
  for (int64_t r = blockIdx.y; r < nrows; r += gridDim.y) {
    const uint64_t grow = (uint64_t)(row0 + r);
    for (int64_t c = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; c < d; c += (int64_t)gridDim.x * blockDim.x) {
      const uint64_t h = hash_at(key, grow * (uint64_t)d + (uint64_t)c);
      float x;
      if (kind == 1) {
        x = (float)((double)((int64_t)__umul64hi(h, 5ull) - 2) * 0.25);
      } else {
        const int64_t acc = (int64_t)(h & 0xFFFF) + (int64_t)((h >> 16) & 0xFFFF) + (int64_t)((h >> 32) & 0xFFFF) +
                            (int64_t)((h >> 48) & 0xFFFF) - 131070;
        x = (float)((double)acc * scale);
      }
      out[r * row_stride + c] = bf16_rne(x);
    }
  }
}

}  // namespace

extern "C" {

// Fill a bf16 [nrows, d] matrix (row stride row_stride elements) with global rows row0.. of
// tba_synth.hidden_rows / weight_rows (key = stream_key(seed, S_HIDDEN / S_WEIGHT)).
int tba_synth_bf16(void* out, uint64_t key, int64_t row0, int64_t nrows, int64_t d, int64_t row_stride, int kind,
                   int scale_exp, cudaStream_t stream) {
  if (!out || nrows < 0 || d <= 0 || row_stride < d || (kind != 0 && kind != 1)) return 1;
  if (nrows == 0) return 0;
  int64_t gx = (d + 255) / 256;
  if (gx > 64) gx = 64;
  const int64_t gy = nrows < 65535 ? nrows : 65535;
  double scale = 1.0;
  for (int i = 0; i < (scale_exp < 0 ? -scale_exp : scale_exp); ++i) scale = scale_exp < 0 ? scale * 0.5 : scale * 2.0;
  synth_bf16_kernel<<<dim3((unsigned)gx, (unsigned)gy), 256, 0, stream>>>(static_cast<uint16_t*>(out), key, row0,
                                                                          nrows, d, row_stride, kind, scale);
  return (int)cudaGetLastError();
}


// Fill rows [row0, row0+nrows) (global row ids) of a logits buffer laid out as
// [nrows, row_stride] elements; columns >= V get NaN. dtype 0 = bf16, 1 = fp32.
// Keys are tba_synth.stream_key(seed, S_LOGITS/S_TOKENS/S_PEAK). Returns 0 or a cudaError_t.
int tba_synth_logits(void* out, int dtype, uint64_t key_logits, uint64_t key_tok, uint64_t key_peak,
                     int64_t row0, int64_t nrows, int64_t V, int64_t row_stride, cudaStream_t stream) {
  if (!out || nrows < 0 || V <= 0 || row_stride < V || (dtype != 0 && dtype != 1)) return 1;
  if (nrows == 0) return 0;
  dim3 block(256);
  int64_t gx = (row_stride + 255) / 256;
  if (gx > 64) gx = 64;
  int64_t gy = nrows < 16384 ? nrows : 16384;
  dim3 grid((unsigned)gx, (unsigned)gy);
  if (dtype == 0)
    synth_logits_kernel<true><<<grid, block, 0, stream>>>(out, key_logits, key_tok, key_peak, row0, nrows, V, row_stride);
  else
    synth_logits_kernel<false><<<grid, block, 0, stream>>>(out, key_logits, key_tok, key_peak, row0, nrows, V, row_stride);
  return (int)cudaGetLastError();
}

// HOST twin (no GPU needed): the same element function on the CPU, for an arbitrary list of
// global rows, packed [nrows, V] (bf16 bits or fp32). Lets the test harness regenerate the
// oracle's input rows ~100x faster than the NumPy twin (which pins it bit for bit,
// tests/test_synth.py). Returns 0, or 1 on a bad argument.
int tba_synth_logits_host(void* out, int dtype, uint64_t key_logits, uint64_t key_tok, uint64_t key_peak,
                          const int64_t* rows, int64_t nrows, int64_t V) {
  if (!out || !rows || nrows < 0 || V <= 0 || (dtype != 0 && dtype != 1)) return 1;
  for (int64_t r = 0; r < nrows; ++r) {
    const uint64_t grow = (uint64_t)rows[r];
    const uint64_t y = umulhi64(hash_at(key_tok, grow), (uint64_t)V);
    const float peak = (float)(4 * (int)(hash_at(key_peak, grow) & 3ull));
    const uint64_t base = grow * (uint64_t)V;
    for (int64_t c = 0; c < V; ++c) {
      float z = irwin_hall(hash_at(key_logits, base + (uint64_t)c));
      if ((uint64_t)c == y) z = z + peak;
      if (dtype == 0) static_cast<uint16_t*>(out)[r * V + c] = bf16_rne(z);
      else static_cast<float*>(out)[r * V + c] = z;
    }
  }
  return 0;
}

}  // extern "C"
