// Microbenchmark (B200): the attention softmax chunk body on TMEM, in
// isolation: per chunk each softmax thread loads its 128-column S row
// (tcgen05.ld 4 x 32x32b.x32), takes the row max (FMNMX3), computes
// P = 2^(s sc - m) as bf16x2 (FFMA2, cvt, ex2.bf16x2) and stores 64 packed
// columns (tcgen05.st 4 x x16).  256-thread CTAs, 2 per SM, warps 4-7 work.
// SPIN=1: warps 0/1 lane 0 spin on an mbarrier meanwhile (like the producer
// and MMA threads).  Prints cycles per chunk per CTA.
#include <cstdio>
#include <cstdint>
#include <cuda_bf16.h>

__device__ __forceinline__ uint32_t ex2_bf16x2(uint32_t x) { uint32_t y; asm volatile("ex2.approx.ftz.bf16x2 %0, %1;" : "=r"(y) : "r"(x)); return y; }
__device__ __forceinline__ uint32_t cvt_bf16x2(float lo, float hi) { uint32_t r; asm("cvt.rn.bf16x2.f32 %0, %1, %2;" : "=r"(r) : "f"(hi), "f"(lo)); return r; }
__device__ __forceinline__ uint64_t pk2(float x, float y) { uint64_t r; asm("mov.b64 %0, {%1, %2};" : "=l"(r) : "f"(x), "f"(y)); return r; }
__device__ __forceinline__ float2 upk2(uint64_t r) { float2 v; asm("mov.b64 {%0, %1}, %2;" : "=f"(v.x), "=f"(v.y) : "l"(r)); return v; }
__device__ __forceinline__ uint64_t fma2(uint64_t a, uint64_t b, uint64_t c) { uint64_t r; asm("fma.rn.f32x2 %0, %1, %2, %3;" : "=l"(r) : "l"(a), "l"(b), "l"(c)); return r; }
__device__ __forceinline__ float max3(float a, float b, float c) { float r; asm("max.f32 %0, %1, %2, %3;" : "=f"(r) : "f"(a), "f"(b), "f"(c)); return r; }
__device__ __forceinline__ void ld32(uint32_t t, uint32_t* r) {
  asm volatile("tcgen05.ld.sync.aligned.32x32b.x32.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,%16,%17,%18,%19,%20,%21,%22,%23,%24,%25,%26,%27,%28,%29,%30,%31}, [%32];"
    : "=r"(r[0]),"=r"(r[1]),"=r"(r[2]),"=r"(r[3]),"=r"(r[4]),"=r"(r[5]),"=r"(r[6]),"=r"(r[7]),"=r"(r[8]),"=r"(r[9]),"=r"(r[10]),"=r"(r[11]),"=r"(r[12]),"=r"(r[13]),"=r"(r[14]),"=r"(r[15]),"=r"(r[16]),"=r"(r[17]),"=r"(r[18]),"=r"(r[19]),"=r"(r[20]),"=r"(r[21]),"=r"(r[22]),"=r"(r[23]),"=r"(r[24]),"=r"(r[25]),"=r"(r[26]),"=r"(r[27]),"=r"(r[28]),"=r"(r[29]),"=r"(r[30]),"=r"(r[31]) : "r"(t));
}
__device__ __forceinline__ void st16(uint32_t t, const uint32_t* v) {
  asm volatile("tcgen05.st.sync.aligned.32x32b.x16.b32 [%0], {%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,%16};" :: "r"(t),
    "r"(v[0]),"r"(v[1]),"r"(v[2]),"r"(v[3]),"r"(v[4]),"r"(v[5]),"r"(v[6]),"r"(v[7]),"r"(v[8]),"r"(v[9]),"r"(v[10]),"r"(v[11]),"r"(v[12]),"r"(v[13]),"r"(v[14]),"r"(v[15]));
}

template <int SPIN, int MODE>
__global__ void __launch_bounds__(256, 2) k(int chunks, long long* cyc, float* out) {
  __shared__ uint32_t slot;
  __shared__ __align__(8) uint64_t bar;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  if (warp == 2) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"((uint32_t)__cvta_generic_to_shared(&slot)), "r"(256));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  if (threadIdx.x == 0) asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"((uint32_t)__cvta_generic_to_shared(&bar)), "r"(128));
  asm volatile("tcgen05.fence::before_thread_sync;");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;");
  const uint32_t tb = slot;
  if (warp >= 4) {
    asm volatile("setmaxnreg.inc.sync.aligned.u32 192;");
    const int ew = warp & 3;
    const uint32_t lo = (uint32_t)(ew * 32) << 16;
    // S = small values
    for (int c = 0; c < 128; c += 16) { uint32_t v[16]; for (int i = 0; i < 16; ++i) v[i] = __float_as_uint(0.01f * (lane + i + c)); st16(tb + lo + c, v); }
    asm volatile("tcgen05.wait::st.sync.aligned;");
    const float sc = 1.4427f / 8.f;
    float acc = 0.f;
    long long t0 = clock64();
    for (int j = 0; j < chunks; ++j) {
      uint32_t sr[128];
#pragma unroll
      for (int c = 0; c < 128; c += 32) ld32(tb + lo + c, sr + c);
      asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
      float m8[8];
#pragma unroll
      for (int i = 0; i < 8; ++i) m8[i] = -INFINITY;
#pragma unroll
      for (int i = 0; i < 128; i += 2) m8[(i >> 1) & 7] = max3(m8[(i >> 1) & 7], __uint_as_float(sr[i]), __uint_as_float(sr[i + 1]));
      const float m = fmaxf(fmaxf(fmaxf(m8[0], m8[1]), fmaxf(m8[2], m8[3])), fmaxf(fmaxf(m8[4], m8[5]), fmaxf(m8[6], m8[7]))) * sc;
      acc += m;
      const uint64_t sc2 = pk2(sc, sc), nb2 = pk2(-m, -m);
#pragma unroll
      for (int c = 0; c < 128; c += 32) {
        uint32_t pk[16];
#pragma unroll
        for (int i = 0; i < 32; i += 2) {
          const float2 x = upk2(fma2(pk2(__uint_as_float(sr[c + i]), __uint_as_float(sr[c + i + 1])), sc2, nb2));
          pk[i >> 1] = MODE == 0 ? ex2_bf16x2(cvt_bf16x2(x.x, x.y)) : cvt_bf16x2(x.x, x.y);
        }
        st16(tb + lo + 128 + c / 2, pk);   // P into other columns (keeps S intact)
      }
      asm volatile("tcgen05.wait::st.sync.aligned;" ::: "memory");
    }
    long long t1 = clock64();
    if (threadIdx.x == 128) cyc[blockIdx.x] = (t1 - t0);
    out[blockIdx.x * 256 + threadIdx.x] = acc;
    asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"((uint32_t)__cvta_generic_to_shared(&bar)) : "memory");
  } else {
    asm volatile("setmaxnreg.dec.sync.aligned.u32 64;");
    if (SPIN && lane == 0 && warp < 2) asm volatile("{\n.reg .pred p;\nW_%=:\nmbarrier.try_wait.parity.shared::cta.b64 p, [%0], 0;\n@!p bra W_%=;\n}\n" ::"r"((uint32_t)__cvta_generic_to_shared(&bar)) : "memory");
  }
  asm volatile("tcgen05.fence::before_thread_sync;");
  __syncthreads();
  if (warp == 2) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tb), "r"(256));
}

template <int SPIN, int MODE>
void run(int ctas_per_sm) {
  const int blocks = 148 * ctas_per_sm, chunks = 2000;
  long long* cyc; float* out;
  cudaMalloc(&cyc, blocks * 8); cudaMalloc(&out, blocks * 256 * 4);
  k<SPIN, MODE><<<blocks, 256>>>(10, cyc, out);
  k<SPIN, MODE><<<blocks, 256>>>(chunks, cyc, out);
  cudaError_t e = cudaDeviceSynchronize();
  long long h[296 * 2]; cudaMemcpy(h, cyc, blocks * 8, cudaMemcpyDeviceToHost);
  double mean = 0; for (int i = 0; i < blocks; ++i) mean += h[i]; mean /= blocks;
  printf("SPIN %d MODE %d (%s) CTAs/SM %d: %.0f cycles per 128x128 chunk per CTA; %.1f elem/clk/SM [%s]\n", SPIN, MODE,
         MODE == 0 ? "ex2.bf16x2" : "no exp", ctas_per_sm, mean / chunks, 128.0 * 128 * ctas_per_sm / (mean / chunks), cudaGetErrorString(e));
  cudaFree(cyc); cudaFree(out);
}
int main() {
  run<0, 0>(1); run<0, 0>(2); run<1, 0>(2); run<0, 1>(2);
  return 0;
}
