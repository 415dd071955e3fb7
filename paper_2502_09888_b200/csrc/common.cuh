// Internal definitions shared by the libclimber kernels and the C-ABI layer.
// Not part of the public ABI (see include/climber.h).
#pragma once
#include <cuda_bf16.h>
#include <cuda_runtime.h>
#include <stdint.h>

#include <cmath>

namespace climber {

typedef __nv_bfloat16 bf16;

// Model dimensions, passed by value to kernels.  The relative-bias pointers
// are ctx-lifetime device arrays (nullptr when rel_bias = 0, Eq. 3
// f_b = 0): tables b_pos [L][Nb][R][h][NB_POS], b_time [L][Nb][R][h][NB_TIME];
// hage [slot][Nb][nk] the age of every extracted history token at the request
// time, t_req - t_j in seconds (int32, saturating at 2^31 - 1 s ~ 68 years;
// t_i - t_j = age_j - age_i); cbias [slot][L][Nb][h][nk] the candidate-row
// bias over the history keys (the same for every candidate of a request).
struct Dims {
  int d, h, dh, L, Nb, nk, F, Dse, Hse, V, A, R, Mmax, causal, ppb;
  float eps;
  const float* bpos;
  const float* btime;
  int* hage;
  float* cbias;
};

// ---- relative attention bias buckets (Eq. 3 f_b^{p,t}; G6c) ----
constexpr int NB_POS = 128;   // 64 position-offset buckets per sign
constexpr int NB_TIME = 14;   // 7 time-delta buckets per sign
__host__ __device__ __forceinline__ int bucket_pos(int delta) {
  const int a = delta < 0 ? -delta : delta;
  int b;
  if (a < 16) {
    b = a;
  } else {
#ifdef __CUDA_ARCH__
    const int e = 31 - __clz(a);  // floor(log2 a)
#else
    int e = 31;
    while (!((a >> e) & 1)) --e;
#endif
    b = 16 + 4 * (e - 4) + ((a >> (e - 2)) & 3);
    b = b < 63 ? b : 63;
  }
  return b + (delta < 0 ? 64 : 0);
}
__host__ __device__ __forceinline__ int bucket_time(long long dt) {
  const long long a = dt < 0 ? -dt : dt;
  const int b = a == 0 ? 0 : a < 60 ? 1 : a < 3600 ? 2 : a < 86400 ? 3 : a < 604800 ? 4 : a < 2592000 ? 5 : 6;
  return b + (dt < 0 ? 7 : 0);
}
// the same buckets for a 32-bit delta (branch-free compares)
__host__ __device__ __forceinline__ int bucket_time32(int dt) {
  const int a = dt < 0 ? -dt : dt;
  const int b = (a > 0) + (a >= 60) + (a >= 3600) + (a >= 86400) + (a >= 604800) + (a >= 2592000);
  return b + (dt < 0 ? 7 : 0);
}
// the (layer, block, scenario, head) row of a bias table
__host__ __device__ __forceinline__ long long bias_row(const Dims& D, int l, int k, int r, int head) {
  return (((long long)l * D.Nb + k) * D.R + r) * D.h + head;
}

// Device error word bits (climber_stream_status maps them to statuses).
enum : int { ERR_RANGE = 1, ERR_UNSORTED = 2, ERR_CONFIG = 4, ERR_NUMERIC = 8 };

constexpr int PAGE = 64;  // tokens per K/V page

// ---- element conversion helpers -------------------------------------------
__device__ __forceinline__ float to_f(float x) { return x; }
__device__ __forceinline__ float to_f(bf16 x) { return __bfloat162float(x); }
template <typename T> __device__ __forceinline__ T from_f(float x);
template <> __device__ __forceinline__ float from_f<float>(float x) { return x; }
template <> __device__ __forceinline__ bf16 from_f<bf16>(float x) { return __float2bfloat16_rn(x); }

// Load / store 8 consecutive elements (16 B for bf16, 32 B for fp32).
__device__ __forceinline__ void load8(const bf16* p, float* v) {
  uint4 u = *reinterpret_cast<const uint4*>(p);
  const bf16* b = reinterpret_cast<const bf16*>(&u);
#pragma unroll
  for (int i = 0; i < 8; ++i) v[i] = __bfloat162float(b[i]);
}
__device__ __forceinline__ void load8(const float* p, float* v) {
  float4 a = *reinterpret_cast<const float4*>(p);
  float4 b = *reinterpret_cast<const float4*>(p + 4);
  v[0] = a.x; v[1] = a.y; v[2] = a.z; v[3] = a.w; v[4] = b.x; v[5] = b.y; v[6] = b.z; v[7] = b.w;
}
__device__ __forceinline__ void store8(bf16* p, const float* v) {
  uint4 u;
  bf16* b = reinterpret_cast<bf16*>(&u);
#pragma unroll
  for (int i = 0; i < 8; ++i) b[i] = __float2bfloat16_rn(v[i]);
  *reinterpret_cast<uint4*>(p) = u;
}
__device__ __forceinline__ void store8(float* p, const float* v) {
  *reinterpret_cast<float4*>(p) = make_float4(v[0], v[1], v[2], v[3]);
  *reinterpret_cast<float4*>(p + 4) = make_float4(v[4], v[5], v[6], v[7]);
}
// N consecutive bf16 (N = 4: 8-byte access, N % 8 == 0: 16-byte accesses)
template <int N>
__device__ __forceinline__ void load_n(const bf16* p, float* v) {
  if constexpr (N % 8 == 0) {
#pragma unroll
    for (int i = 0; i < N; i += 8) load8(p + i, v + i);
  } else {
    static_assert(N == 4, "load_n: N = 4 or a multiple of 8");
    const uint2 u = *reinterpret_cast<const uint2*>(p);
    const bf16* b = reinterpret_cast<const bf16*>(&u);
#pragma unroll
    for (int i = 0; i < 4; ++i) v[i] = __bfloat162float(b[i]);
  }
}
template <int N>
__device__ __forceinline__ void store_n(bf16* p, const float* v) {
  if constexpr (N % 8 == 0) {
#pragma unroll
    for (int i = 0; i < N; i += 8) store8(p + i, v + i);
  } else {
    static_assert(N == 4, "store_n: N = 4 or a multiple of 8");
    uint2 u;
    bf16* b = reinterpret_cast<bf16*>(&u);
#pragma unroll
    for (int i = 0; i < 4; ++i) b[i] = __float2bfloat16_rn(v[i]);
    *reinterpret_cast<uint2*>(p) = u;
  }
}

__device__ __forceinline__ float warp_sum(float v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  return v;
}

// Activations with one MUFU op each: sigma(x) = 1/2 tanh(x/2) + 1/2, so
// SiLU (G8) = x sigma(x) and the Eq. 4 gate use a single tanh.approx.f32
// (max rel. error ~2^-11, below the bf16 rounding of the GEMM outputs).
__device__ __forceinline__ float tanh_approx(float x) {
  float y;
  asm("tanh.approx.f32 %0, %1;" : "=f"(y) : "f"(x));
  return y;
}
// bf16 path: one MUFU op; fp32 verification build: accurate expf.
template <typename T> __device__ __forceinline__ float sigmoid_t(float x) {
  return fmaf(0.5f, tanh_approx(0.5f * x), 0.5f);
}
template <> __device__ __forceinline__ float sigmoid_t<float>(float x) { return 1.0f / (1.0f + expf(-x)); }
template <typename T> __device__ __forceinline__ float silu_t(float x) { return x * sigmoid_t<T>(x); }

// SUMI visibility rule in canonical coordinates (G1,
// G12, G14): slots 0..nk-1 are history (left-padded, valid iff >= nk - v),
// slots nk.. are candidates.  The attention kernels implement exactly these
// key ranges: history row t sees keys j <= t (causal) or j < v; candidate
// rows see keys 0..v-1 plus themselves.
__host__ __device__ __forceinline__ bool sumi_visible(int i, int j, int nk, int v, int causal) {
  const int first = nk - v;
  if (i < nk && i < first) return false;
  if (j < nk && j < first) return false;
  if (i < nk && j < nk) return causal ? (j <= i) : true;
  if (i < nk) return false;
  if (j < nk) return true;
  return i == j;
}

// ---- GEMM epilogues ---------------------------------------------------------
// D[m][n] = sum_k A[m][k] * B[n][k]  (both operands K-contiguous), fp32 accum.
enum EpiKind : int {
  EPI_STORE = 0,   // out_T[m*ldo + n] = act(acc + bias[n])
  EPI_RESID = 1,   // out_f32[m*ldo + n] += acc
  EPI_QKV_PAGES = 2, // columns (n + col_off) in [0,d): Q -> out_T[m*ldo + n]; [d,3d): K/V -> pages
  EPI_STORE_F32 = 3, // out_f32[m*ldo + n] = act(acc + bias[n])  (the sigmoid gate of Eq. 4)
  EPI_RESID_NORM = 4, // residual add that also prepares the next RMSNorm (tcgen05 GEMM only):
                      // C = C + acc (fp32, out), Cb = bf16(C) (out_b16), part[m*part_rs + n_tile] =
                      // sum over the tile's columns of C^2
};
enum ActKind : int { ACT_NONE = 0, ACT_SILU = 1, ACT_RELU = 2, ACT_SIGMOID = 3 };

template <typename T>
__device__ __forceinline__ float apply_act(int act, float a) {
  if (act == ACT_SILU) return silu_t<T>(a);
  if (act == ACT_RELU) return fmaxf(a, 0.0f);
  if (act == ACT_SIGMOID) return sigmoid_t<T>(a);
  return a;
}

struct Epilogue {
  int kind;
  int act;
  void* out;            // T* (STORE, QKV Q part) or float* (RESID, GATE)
  long long ldo;        // row stride of out, elements
  const float* bias;    // [N] or nullptr
  // EPI_QKV_PAGES: history row m = u * nk + t of wave user u
  void* pool;           // page pool base (T*)
  long long pool_rows;  // n_pages * 2 * PAGE
  const int* ptab;      // [slots][Nb][L][ppb]
  const int* wave_slot; // [U] slot of wave user u
  int col_off;          // 0 (full QKV) or d (last layer: K/V only)
  int blk, layer;       // (k, l)
  int d, h, dh, nk, Nb, L, ppb;
  // EPI_RESID_NORM outputs
  void* out_b16;        // bf16 copy of C, same [rows][ldo] layout
  float* part;          // per-row, per-column-tile sums of squares
  long long part_rs;    // row stride of part (floats)
  // RMSNorm folded into a consumer GEMM (gain pre-multiplied into the weights):
  // acc *= 1 / sqrt(sum_{j < rs_n} rs_part[m * rs_rs + j] * rs_inv_d + rs_eps)
  const float* rs_part;
  long long rs_rs;
  int rs_n;
  float rs_inv_d, rs_eps;
  // batched (grouped over the N_b blocks) GEMMs: element strides between the
  // batch entries of each output, and the block index taken from the batch
  long long out_bs, out_b16_bs, part_bs, rs_bs;
  int blk_from_batch;
};

// Page addressing: page = [2 (K,V)][PAGE tokens][d] elements (heads contiguous
// d_h column groups inside a token row).  Viewed as a 2-D [n_pages*2*PAGE][d]
// matrix, the K (or V) rows of 32 consecutive tokens of one page are one TMA
// box, which is how the QKV GEMM epilogue writes them.
__host__ __device__ __forceinline__ long long page_row(int page, int kv, int slot_t) {
  return ((long long)page * 2 + kv) * PAGE + slot_t;
}
__device__ __forceinline__ long long page_elem_offset(int page, int kv, int head, int slot_t, int dim,
                                                      int d, int dh) {
  return page_row(page, kv, slot_t) * d + (long long)head * dh + dim;
}

// Apply the epilogue to NC consecutive columns [n0, n0+NC) of row m.
template <typename T, int NC>
__device__ __forceinline__ void epilogue_chunk(const Epilogue& e, long long m, int n0, const float* v) {
  if (e.kind == EPI_STORE) {
    float x[NC];
#pragma unroll
    for (int i = 0; i < NC; ++i) x[i] = apply_act<T>(e.act, v[i] + (e.bias ? e.bias[n0 + i] : 0.0f));
    T* o = reinterpret_cast<T*>(e.out) + m * e.ldo + n0;
    if constexpr (NC % 8 == 0) {
#pragma unroll
      for (int i = 0; i < NC; i += 8) store8(o + i, x + i);
    } else {
#pragma unroll
      for (int i = 0; i < NC; ++i) o[i] = from_f<T>(x[i]);
    }
  } else if (e.kind == EPI_RESID) {
    float* o = reinterpret_cast<float*>(e.out) + m * e.ldo + n0;
#pragma unroll
    for (int i = 0; i < NC; ++i) o[i] += v[i];
  } else if (e.kind == EPI_STORE_F32) {
    float* o = reinterpret_cast<float*>(e.out) + m * e.ldo + n0;
#pragma unroll
    for (int i = 0; i < NC; ++i) o[i] = apply_act<T>(e.act, v[i] + (e.bias ? e.bias[n0 + i] : 0.0f));
  } else {  // EPI_QKV_PAGES
    int c = n0 + e.col_off;
    if (c < e.d) {
      T* o = reinterpret_cast<T*>(e.out) + m * e.ldo + c;
#pragma unroll
      for (int i = 0; i < NC; ++i) o[i] = from_f<T>(v[i]);
    } else {
      int u = (int)(m / e.nk), t = (int)(m % e.nk);
      int slot = e.wave_slot[u];
      int page = e.ptab[(((long long)slot * e.Nb + e.blk) * e.L + e.layer) * e.ppb + t / PAGE];
      int kv = (c >= 2 * e.d) ? 1 : 0;
      int cc = c - e.d * (1 + kv);
      int head = cc / e.dh, dim = cc % e.dh;   // NC divides dh: chunk stays in one head
      T* o = reinterpret_cast<T*>(e.pool) + page_elem_offset(page, kv, head, t % PAGE, dim, e.d, e.dh);
#pragma unroll
      for (int i = 0; i < NC; ++i) o[i] = from_f<T>(v[i]);
    }
  }
}

// Element-wise form of the same epilogues: one value of row m, column n.  The
// tensor-core GEMM transposes each 32x32 accumulator block through shared
// memory so that lane j handles column n0 + j of one row: every warp-level
// access is then a contiguous row segment (coalesced) instead of 32 rows.
template <typename T>
__device__ __forceinline__ void epilogue_elem(const Epilogue& e, long long m, int n, float v) {
  if (e.kind == EPI_STORE) {
    reinterpret_cast<T*>(e.out)[m * e.ldo + n] = from_f<T>(apply_act<T>(e.act, v + (e.bias ? e.bias[n] : 0.0f)));
  } else if (e.kind == EPI_RESID) {
    float* o = reinterpret_cast<float*>(e.out) + m * e.ldo + n;
    *o += v;
  } else if (e.kind == EPI_STORE_F32) {
    reinterpret_cast<float*>(e.out)[m * e.ldo + n] = apply_act<T>(e.act, v + (e.bias ? e.bias[n] : 0.0f));
  } else {  // EPI_QKV_PAGES
    int c = n + e.col_off;
    if (c < e.d) {
      reinterpret_cast<T*>(e.out)[m * e.ldo + c] = from_f<T>(v);
    } else {
      int u = (int)(m / e.nk), t = (int)(m % e.nk);
      int slot = e.wave_slot[u];
      int page = e.ptab[(((long long)slot * e.Nb + e.blk) * e.L + e.layer) * e.ppb + t / PAGE];
      int kv = (c >= 2 * e.d) ? 1 : 0;
      int cc = c - e.d * (1 + kv);
      reinterpret_cast<T*>(e.pool)[page_elem_offset(page, kv, cc / e.dh, t % PAGE, cc % e.dh, e.d, e.dh)] =
          from_f<T>(v);
    }
  }
}

}  // namespace climber
