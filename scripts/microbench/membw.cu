// Calibration microbenchmarks (not product code): achievable HBM read-only / write-only / copy
// bandwidth with 128-bit accesses, and MUFU.EX2 throughput, on this B200.
#include <cstdint>
#include <cuda_runtime.h>
__global__ void rd(const uint4* __restrict__ p, size_t n, unsigned* out) {
  unsigned acc = 0;
  for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < n; i += (size_t)gridDim.x * blockDim.x) {
    uint4 v;
    asm volatile("ld.global.nc.L1::no_allocate.v4.u32 {%0,%1,%2,%3}, [%4];" : "=r"(v.x), "=r"(v.y), "=r"(v.z), "=r"(v.w) : "l"(p + i));
    acc ^= v.x ^ v.y ^ v.z ^ v.w;
  }
  if (acc == 0x12345678u) out[0] = acc;
}
template <int U>
__global__ void rdu(const uint4* __restrict__ p, size_t n, unsigned* out) {
  unsigned acc = 0;
  size_t stride = (size_t)gridDim.x * blockDim.x;
  size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x;
  for (; i + (U - 1) * stride < n; i += U * stride) {
    uint4 v[U];
#pragma unroll
    for (int u = 0; u < U; ++u)
      asm volatile("ld.global.nc.L1::no_allocate.v4.u32 {%0,%1,%2,%3}, [%4];" : "=r"(v[u].x), "=r"(v[u].y), "=r"(v[u].z), "=r"(v[u].w) : "l"(p + i + u * stride));
#pragma unroll
    for (int u = 0; u < U; ++u) acc ^= v[u].x ^ v[u].y ^ v[u].z ^ v[u].w;
  }
  if (acc == 0x12345678u) out[0] = acc;
}
__global__ void wr(uint4* __restrict__ p, size_t n) {
  for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < n; i += (size_t)gridDim.x * blockDim.x)
    asm volatile("st.global.cs.v4.u32 [%0], {%1,%1,%1,%1};" ::"l"(p + i), "r"(0u) : "memory");
}
__global__ void cp(const uint4* __restrict__ a, uint4* __restrict__ b, size_t n) {
  for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < n; i += (size_t)gridDim.x * blockDim.x) {
    uint4 v;
    asm volatile("ld.global.nc.L1::no_allocate.v4.u32 {%0,%1,%2,%3}, [%4];" : "=r"(v.x), "=r"(v.y), "=r"(v.z), "=r"(v.w) : "l"(a + i));
    asm volatile("st.global.cs.v4.u32 [%0], {%1,%2,%3,%4};" ::"l"(b + i), "r"(v.x), "r"(v.y), "r"(v.z), "r"(v.w) : "memory");
  }
}
__global__ void mufu(float* out, int iters) {
  float x0 = threadIdx.x * 1e-3f, x1 = x0 + 0.1f, x2 = x0 + 0.2f, x3 = x0 + 0.3f;
  float a0 = 0, a1 = 0, a2 = 0, a3 = 0;
  for (int i = 0; i < iters; ++i) {
    float y0, y1, y2, y3;
    asm volatile("ex2.approx.ftz.f32 %0, %1;" : "=f"(y0) : "f"(x0));
    asm volatile("ex2.approx.ftz.f32 %0, %1;" : "=f"(y1) : "f"(x1));
    asm volatile("ex2.approx.ftz.f32 %0, %1;" : "=f"(y2) : "f"(x2));
    asm volatile("ex2.approx.ftz.f32 %0, %1;" : "=f"(y3) : "f"(x3));
    a0 += y0; a1 += y1; a2 += y2; a3 += y3;
  }
  if (a0 + a1 + a2 + a3 == 1.2345f) out[0] = a0;
}
static float timeit(void (*f)(void*), void* arg, int reps) {
  cudaEvent_t a, b; cudaEventCreate(&a); cudaEventCreate(&b);
  f(arg); cudaDeviceSynchronize();
  cudaEventRecord(a);
  for (int r = 0; r < reps; ++r) f(arg);
  cudaEventRecord(b); cudaEventSynchronize(b);
  float ms; cudaEventElapsedTime(&ms, a, b); return ms / reps;
}
struct Args { uint4* a; uint4* b; size_t n; unsigned* o; int grid, block; };
extern "C" int membw(size_t bytes, float* res /* [rd, rdu4, rdu8, wr, cp(GB/s as r+w), mufu ex2/clk/SM-ish Gop/s] */) {
  Args A; A.n = bytes / 16;
  if (cudaMalloc(&A.a, bytes) || cudaMalloc(&A.b, bytes) || cudaMalloc(&A.o, 4)) return 1;
  cudaMemset(A.a, 1, bytes); cudaMemset(A.b, 0, bytes);
  int sms; cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  A.grid = sms * 8; A.block = 256;
  res[0] = bytes / 1e6 / timeit([](void* p){ Args* x=(Args*)p; rd<<<x->grid, x->block>>>(x->a, x->n, x->o); }, &A, 10);
  res[1] = bytes / 1e6 / timeit([](void* p){ Args* x=(Args*)p; rdu<4><<<x->grid, x->block>>>(x->a, x->n, x->o); }, &A, 10);
  res[2] = bytes / 1e6 / timeit([](void* p){ Args* x=(Args*)p; rdu<8><<<x->grid, x->block>>>(x->a, x->n, x->o); }, &A, 10);
  res[3] = bytes / 1e6 / timeit([](void* p){ Args* x=(Args*)p; wr<<<x->grid, x->block>>>(x->b, x->n); }, &A, 10);
  res[4] = 2 * bytes / 1e6 / timeit([](void* p){ Args* x=(Args*)p; cp<<<x->grid, x->block>>>(x->a, x->b, x->n); }, &A, 10);
  float* fo; cudaMalloc(&fo, 4);
  struct M { float* o; int sms; } m{fo, sms};
  const int iters = 1 << 16;
  float ms = timeit([](void* p){ M* x=(M*)p; mufu<<<x->sms * 8, 256>>>(x->o, 1 << 16); }, &m, 5);
  res[5] = (double)sms * 8 * 256 * 4.0 * iters / (ms * 1e-3) / 1e9;  // Gex2/s
  cudaFree(A.a); cudaFree(A.b); cudaFree(A.o); cudaFree(fo);
  return (int)cudaGetLastError();
}
