// Microbenchmark (B200): throughput of the attention softmax inner loop per SM.
//  mode 0: ex2.approx only (MUFU rate)
//  mode 1..: the kernel's per-element sequence (FFMA2 scale, exp2, FADD row
//  sum, F2FP pack) with PE of every 8 exponentials on the FMA-pipe polynomial.
// Prints elements / clock / SM for warps-per-SM in {4, 8, 16}.
#include <cstdio>
#include <cuda_bf16.h>
#include <cstdint>

__device__ __forceinline__ float ex2a(float x) { float y; asm volatile("ex2.approx.ftz.f32 %0, %1;" : "=f"(y) : "f"(x)); return y; }
__device__ __forceinline__ float ex2p(float x) {
  constexpr float MAGIC = 12582912.f;
  x = fmaxf(x, -126.f);
  const float t = x + MAGIC;
  const float f = x - (t - MAGIC);
  const float p = fmaf(fmaf(fmaf(0.055171628f, f, 0.24261117f), f, 0.69326103f), f, 0.99992806f);
  return __int_as_float(__float_as_int(t) * (1 << 23) + __float_as_int(p));
}
__device__ __forceinline__ uint64_t pk2(float x, float y) { uint64_t r; asm("mov.b64 %0, {%1, %2};" : "=l"(r) : "f"(x), "f"(y)); return r; }
__device__ __forceinline__ float2 upk2(uint64_t r) { float2 v; asm("mov.b64 {%0, %1}, %2;" : "=f"(v.x), "=f"(v.y) : "l"(r)); return v; }
__device__ __forceinline__ uint64_t fma2(uint64_t a, uint64_t b, uint64_t c) { uint64_t r; asm("fma.rn.f32x2 %0, %1, %2, %3;" : "=l"(r) : "l"(a), "l"(b), "l"(c)); return r; }

__device__ __forceinline__ uint32_t ex2bf2(uint32_t x) { uint32_t y; asm volatile("ex2.approx.ftz.bf16x2 %0, %1;" : "=r"(y) : "r"(x)); return y; }

template <int MODE, int PE>
__global__ void k(float* out, long long* cyc, int iters, float sc, float nb) {
  float s[64];
#pragma unroll
  for (int i = 0; i < 64; ++i) s[i] = (threadIdx.x * 0.001f + i) * 0.01f;
  float acc = 0.f;
  uint32_t pkacc = 0;
  __syncthreads();
  long long t0 = clock64();
  for (int it = 0; it < iters; ++it) {
    if (MODE == 0) {
#pragma unroll
      for (int i = 0; i < 64; ++i) s[i] = ex2a(s[i]);
    } else if (MODE == 2) {
      // bf16x2 exponentials only
#pragma unroll
      for (int i = 0; i < 64; i += 2) {
        uint32_t u = __float_as_uint(s[i]);
        u = ex2bf2(u);
        s[i] = __uint_as_float(u);
      }
    } else if (MODE == 3) {
      // FFMA2 (fp32 scale - max) -> F2FP bf16x2 -> ex2.bf16x2 = packed P
      const uint64_t sc2 = pk2(sc, sc), nb2 = pk2(nb, nb);
#pragma unroll
      for (int i = 0; i < 64; i += 2) {
        const float2 x = upk2(fma2(pk2(s[i], s[i + 1]), sc2, nb2));
        __nv_bfloat162 xb = __floats2bfloat162_rn(x.x, x.y);
        const uint32_t p = ex2bf2(*reinterpret_cast<uint32_t*>(&xb));
        pkacc ^= p;
        s[i] = __uint_as_float(p & 0xffff0000u); s[i + 1] = __uint_as_float(p << 16);
      }
    } else {
      float ls8[8] = {0, 0, 0, 0, 0, 0, 0, 0};
      const uint64_t sc2 = pk2(sc, sc), nb2 = pk2(nb, nb);
#pragma unroll
      for (int i = 0; i < 64; i += 2) {
        const float2 x = upk2(fma2(pk2(s[i], s[i + 1]), sc2, nb2));
        const float e0 = ((i & 7) < PE) ? ex2p(x.x) : ex2a(x.x);
        const float e1 = (((i + 1) & 7) < PE) ? ex2p(x.y) : ex2a(x.y);
        ls8[i & 7] += e0;
        ls8[(i + 1) & 7] += e1;
        __nv_bfloat162 pp = __floats2bfloat162_rn(e0, e1);
        pkacc ^= *reinterpret_cast<uint32_t*>(&pp);
        s[i] = e0 * 0.5f; s[i + 1] = e1 * 0.5f;   // keep a dependency so nothing is hoisted
      }
      acc += ((ls8[0] + ls8[1]) + (ls8[2] + ls8[3])) + ((ls8[4] + ls8[5]) + (ls8[6] + ls8[7]));
    }
  }
  __syncthreads();
  long long t1 = clock64();
#pragma unroll
  for (int i = 0; i < 64; ++i) acc += s[i];
  out[blockIdx.x * blockDim.x + threadIdx.x] = acc + pkacc;
  if (threadIdx.x == 0) cyc[blockIdx.x] = t1 - t0;
}

template <int MODE, int PE>
void run(int warps) {
  const int blocks = 148, iters = 2000;
  float* out; long long* cyc;
  cudaMalloc(&out, blocks * warps * 32 * 4);
  cudaMalloc(&cyc, blocks * 8);
  k<MODE, PE><<<blocks, warps * 32>>>(out, cyc, 10, 1.0f, -0.5f);
  k<MODE, PE><<<blocks, warps * 32>>>(out, cyc, iters, 1.0f, -0.5f);
  long long h[148];
  cudaMemcpy(h, cyc, sizeof h, cudaMemcpyDeviceToHost);
  double mean = 0; for (int i = 0; i < blocks; ++i) mean += h[i]; mean /= blocks;
  double elems = (double)warps * 32 * 64 * iters * (MODE == 2 ? 0.5 : 1.0) * (MODE >= 2 ? 2.0 : 1.0);
  printf("mode %d PE %d warps/SM %2d: %.2f elements/clk/SM (%.0f cycles)\n", MODE, PE, warps, elems / mean, mean);
  cudaFree(out); cudaFree(cyc);
}

int main() {
  for (int w : {4, 8, 16}) run<0, 0>(w);
  for (int w : {4, 8, 16}) run<1, 0>(w);
  for (int w : {4, 8, 16}) run<1, 1>(w);
  for (int w : {4, 8, 16}) run<1, 2>(w);
  for (int w : {4, 8, 16}) run<1, 3>(w);
  for (int w : {4, 8, 16}) run<1, 4>(w);
  for (int w : {8}) run<1, 8>(w);
  for (int w : {4, 8, 16}) run<2, 0>(w);   // elements = 2 per bf16x2 op: printed rate is ops; x2 for elements
  for (int w : {4, 8, 16}) run<3, 0>(w);
  return 0;
}
