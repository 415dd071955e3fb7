// tcgen05/TMEM attention for the bf16 path (Eq. 3 with f_b = 0;
// SUMI masks P:L255): softmax(q.k / (sqrt(d_h) tau)) v.
//
//   MODE_SUMI: a tile of 128 candidates of one (user, head) attends to the v
//              cached history keys of its (block, layer) plus itself.
//   MODE_HIST: 128 history rows of one (user, head) attend keys j <= t
//              (causal) or j < v (requires n_k % 128 == 0).
//
// CTA = 8 warps, one 128-row query tile (TMEM lane = query row); 2 CTAs/SM:
//   warp 0   TMA: Q (and SUMI k_self / v_self) tiles once; K and V of one
//            64-token page per chunk into a 5-stage ring (stages 3 and 4 reuse
//            the self tiles once the self term is read; TMA latency under load
//            is ~2000 cycles, so five pages stay in flight)
//   warp 1   MMA (one thread): S_j = Q K_j^T (M=128, N=64, K=d_h) into one of
//            three TMEM score buffers, issued two chunks ahead and interleaved
//            step by step with O += P_j V_j (M=128, N=d_h, K=64; P_j read from
//            TMEM where it overwrote S_j as packed bf16, V MN-major): chains of
//            N=64 MMAs are latency-bound, two independent chains overlap
//   warp 2   TMEM allocator (3 x 64 score columns + d_h output columns = 256)
//   warps 4-7 softmax, one thread per query row, two passes over its S row in
//            TMEM (max, then exp2 -> packed bf16 P; packed FFMA2/FADD2 and
//            3-input max); lazy online max (O in TMEM is rescaled only when the
//            row max grows by more than 2^8); epilogue O / l -> bf16 -> global.
// The SUMI self term initialises the row state: m = s_self, l = 1, O = v_self
// (tcgen05.st), so no candidate ever reads another candidate's K/V.
#include <cuda.h>
#include <cudaTypedefs.h>

#include <cstdio>
#include <cstdlib>
#include <mutex>

#include "kernels.cuh"
#include "tc_util.cuh"

namespace climber {
namespace at {
using namespace tcu;

constexpr int ROWS = 128;
constexpr int KEYS = PAGE;  // 64 keys per chunk = one K/V page
constexpr int STAGES = 5;  // K/V pages in flight (TMA latency under load is ~2000 cycles)
constexpr int FREE_STAGES = 3;  // stages 3, 4 alias the SUMI k_self / v_self tiles (free after init)
constexpr int NSB = 3;      // TMEM score/P buffers
constexpr int THREADS = 256;
constexpr float LOG2E = 1.4426950408889634f;
constexpr float RESCALE_LOG2 = 8.0f;

// 2^x on the MUFU (ex2.approx.ftz: -inf -> +0, no range fix-up instructions)
__device__ __forceinline__ float ex2_approx(float x) {
  float y;
  asm("ex2.approx.ftz.f32 %0, %1;" : "=f"(y) : "f"(x));
  return y;
}

// 2^x on the FMA pipe (FA4's MUFU offload): x = j + f, j = rne(x), f in
// [-1/2, 1/2]; 2^f by a degree-3 fit (max rel. error 7.5e-5, far below the
// bf16 rounding of P), 2^j added to the exponent field with one IMAD.
__device__ __forceinline__ float ex2_poly(float x) {
  constexpr float MAGIC = 12582912.f;  // 1.5 * 2^23: t's low mantissa bits hold rne(x)
  x = fmaxf(x, -126.f);
  const float t = x + MAGIC;
  const float f = x - (t - MAGIC);
  const float p = fmaf(fmaf(fmaf(0.055171628f, f, 0.24261117f), f, 0.69326103f), f, 0.99992806f);
  return __int_as_float(__float_as_int(t) * (1 << 23) + __float_as_int(p));
}

// Blackwell packed FP32x2 FMA / add and 3-input max (FFMA2, FADD2, FMNMX3):
// half the issue slots of the scalar forms in the softmax loop
__device__ __forceinline__ uint64_t pk2(float x, float y) {
  uint64_t r;
  asm("mov.b64 %0, {%1, %2};" : "=l"(r) : "f"(x), "f"(y));
  return r;
}
__device__ __forceinline__ float2 upk2(uint64_t r) {
  float2 v;
  asm("mov.b64 {%0, %1}, %2;" : "=f"(v.x), "=f"(v.y) : "l"(r));
  return v;
}
__device__ __forceinline__ uint64_t fma2(uint64_t a, uint64_t b, uint64_t c) {
  uint64_t r;
  asm("fma.rn.f32x2 %0, %1, %2, %3;" : "=l"(r) : "l"(a), "l"(b), "l"(c));
  return r;
}
__device__ __forceinline__ uint64_t add2(uint64_t a, uint64_t b) {
  uint64_t r;
  asm("add.rn.f32x2 %0, %1, %2;" : "=l"(r) : "l"(a), "l"(b));
  return r;
}
__device__ __forceinline__ float max3(float a, float b, float c) {
  float r;
  asm("max.f32 %0, %1, %2, %3;" : "=f"(r) : "f"(a), "f"(b), "f"(c));
  return r;
}

#ifdef CLIMBER_ATTN_SPIN
#define MBW mbar_wait_spin
#else
#define MBW mbar_wait
#endif

enum { MODE_SUMI = 0, MODE_HIST = 1 };

template <int DH>
struct Lay {
  static constexpr int RB = DH * 2;                      // bytes per Q/K/V row (128 or 64)
  static constexpr uint32_t SWZ = (DH == 64) ? 2u : 4u;  // descriptor swizzle: 128B / 64B
  static constexpr int Q_OFF = 0;
  static constexpr int Q_BYTES = ROWS * RB;
  static constexpr int KVB = KEYS * RB;                  // one K (or V) page slice of one head
  static constexpr int KS_OFF = Q_OFF + Q_BYTES;         // SUMI: the tile's k_self rows (same swizzle as Q)
  static constexpr int VS_OFF = KS_OFF + Q_BYTES;        // SUMI: the tile's v_self rows
  static constexpr int KV_OFF = VS_OFF + Q_BYTES;        // stage s < 3: K at KV_OFF + 2 s KVB, V at + KVB
  static_assert(2 * KVB == Q_BYTES, "one ring stage = one self tile");
  static constexpr int BAR_OFF = KV_OFF + 2 * FREE_STAGES * KVB;
  // stages 3 and 4 reuse the k_self / v_self tiles once the self term is read
  __device__ static constexpr int stage_off(int st) { return st < FREE_STAGES ? KV_OFF + 2 * st * KVB : KS_OFF + 2 * (st - FREE_STAGES) * KVB; }
  static constexpr int TOTAL = BAR_OFF + 512 + 1024;
  static constexpr int STG_OFF = KV_OFF;                 // epilogue staging reuses the K/V ring
};

struct Args {
  const bf16* Q;  // SUMI: QKV [P][3d] (q | k_self | v_self); HIST: Q [U*nk][d]
  const int64_t* cand_off;
  const int* wave_slot;
  const int* wave_r;
  const int* ptab;
  const int* vlen_all;
  const float* tau;
  bf16* O;        // [rows][d]
  int k, l;       // first block, layer
  int U;          // users in the wave
  long long rows_pb;  // grouped over nbk blocks: block kk's rows start at kk * rows_pb in Q/QKV and O
  Dims D;
  unsigned long long* trace;  // debug timeline (CLIMBER_ATTN_TRACE), nullptr normally
};
constexpr int TRACE_N = 48;  // CLIMBER_ATTN_TRACE_BUILD: 0-23 softmax timeline, 24-31 MMA p_full seen, 32-39 QK issue

// PE8: how many of every 8 scores take ex2_poly instead of the MUFU
template <int DH, int MODE, int PE8, int ES = 0, int BIAS = 0>
__global__ void __launch_bounds__(THREADS, 2)
    k_attn_tc(const __grid_constant__ CUtensorMap tmQ, const __grid_constant__ CUtensorMap tmKV, Args a) {
  using Ly = Lay<DH>;
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  uint64_t* bars = reinterpret_cast<uint64_t*>(smem + Ly::BAR_OFF);
  uint64_t* bar_q = bars + 0;
  uint64_t* kv_full = bars + 1;                // [STAGES]
  uint64_t* kv_empty = bars + 1 + STAGES;      // [STAGES]
  // s_full / p_full / o_done are per score buffer (chunk j uses buffer j % 3):
  // every waiter is then at most one phase behind its barrier, so a parity
  // wait can never be overtaken by two completions (ABA).
  uint64_t* s_full = bars + 1 + 2 * STAGES;    // [NSB]
  uint64_t* p_full = s_full + NSB;             // [NSB]
  uint64_t* o_done = p_full + NSB;             // [NSB]
  uint64_t* self_done = o_done + NSB;          // SUMI: k_self / v_self tiles read (stages 3, 4 free)
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(self_done + 1);

  const Dims& D = a.D;
  const int u = blockIdx.z % a.U, head = blockIdx.y, tile0 = blockIdx.x * ROWS;  // tiles of one (u, h) adjacent
  const int kk = blockIdx.z / a.U;  // block within a grouped launch
  const int kblk = a.k + kk;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int slot = a.wave_slot[u];
  const int r = a.wave_r[u];
  const int v = a.vlen_all[(long long)slot * D.Nb + kblk];
  const int* pages = a.ptab + (((long long)slot * D.Nb + kblk) * D.L + a.l) * D.ppb;
  const float sc = LOG2E / (sqrtf((float)DH) * a.tau[((a.l * D.Nb + kblk) * D.R + r) * D.h + head]);

  long long row_base;
  int n_rows, key_end;
  long long ldq;
  if (MODE == MODE_SUMI) {
    const long long p0 = a.cand_off[u], p1 = a.cand_off[u + 1];
    if (p0 + tile0 >= p1) return;  // CTA-uniform
    row_base = kk * a.rows_pb + p0 + tile0;
    n_rows = (int)((p1 - p0 - tile0) < ROWS ? (p1 - p0 - tile0) : ROWS);
    key_end = v;
    ldq = 3LL * D.d;
  } else {
    if (tile0 >= D.nk) return;
    row_base = kk * a.rows_pb + (long long)u * D.nk + tile0;
    n_rows = max(0, min(ROWS, v - tile0));
    key_end = D.causal ? min(v, tile0 + ROWS) : v;
    ldq = D.d;
  }
  const int n_chunks = (key_end + KEYS - 1) / KEYS;

  // page ids of this (user, block, layer), requested before the setup so the
  // global-load latency overlaps barrier init and TMEM allocation
  int pg0 = 0, pg1 = 0;
  if (warp == 0) {
    if (lane < n_chunks) pg0 = pages[lane];
    if (lane + 32 < n_chunks) pg1 = pages[lane + 32];
  }
  if (warp == 0 && lane == 0) {
    asm volatile("prefetch.tensormap [%0];" ::"l"(&tmQ) : "memory");
    asm volatile("prefetch.tensormap [%0];" ::"l"(&tmKV) : "memory");
    mbar_init(bar_q, 1);
    for (int s = 0; s < STAGES; ++s) {
      mbar_init(&kv_full[s], 1);
      mbar_init(&kv_empty[s], 1);
    }
    mbar_init(self_done, 128);
    for (int b = 0; b < NSB; ++b) {
      mbar_init(&s_full[b], 1);
      mbar_init(&p_full[b], 128);
      mbar_init(&o_done[b], 1);
    }
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    // the query-side tiles go out first: their TMA round trip (~3k cycles
    // under load) is the head of every CTA's critical path
    if (MODE == MODE_SUMI) {  // q, k_self, v_self of the tile's candidates
      mbar_expect_tx(bar_q, 3 * Ly::Q_BYTES);
      tma_load_2d(smem + Ly::Q_OFF, &tmQ, bar_q, head * DH, (int)row_base);
      tma_load_2d(smem + Ly::KS_OFF, &tmQ, bar_q, D.d + head * DH, (int)row_base);
      tma_load_2d(smem + Ly::VS_OFF, &tmQ, bar_q, 2 * D.d + head * DH, (int)row_base);
    } else if (n_chunks > 0) {
      mbar_expect_tx(bar_q, Ly::Q_BYTES);
      tma_load_2d(smem + Ly::Q_OFF, &tmQ, bar_q, head * DH, (int)row_base);
    }
  }
  if (warp == 2) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(smem_u32(tmem_slot)),
                 "r"(256));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
#ifdef CLIMBER_ATTN_TRACE_BUILD
  unsigned long long* tr = nullptr;
  const bool tracer = a.trace != nullptr && threadIdx.x == 128;
  if (a.trace != nullptr && (threadIdx.x >= 128 ? (threadIdx.x & 31) == 0 : threadIdx.x == 32))
    tr = a.trace + ((long long)(blockIdx.z * gridDim.y + blockIdx.y) * gridDim.x + blockIdx.x) * TRACE_N;
  if (tracer) tr[0] = clock64();
#else
  constexpr unsigned long long* tr = nullptr;
  constexpr bool tracer = false;
#endif
  fence_before();
  __syncthreads();
  fence_after();
  if (tracer) tr[1] = clock64();
  const uint32_t tmem_base = *tmem_slot;
  const uint32_t tO = tmem_base + NSB * KEYS;  // S/P buffers at tmem_base + b * KEYS

  if (warp == 0) {
    // page ids of this (user, block, layer): one warp-wide load into smem (up
    // to 64 pages), so the producer never waits on a global load per chunk
    int* spg = reinterpret_cast<int*>(smem + Ly::BAR_OFF + 256);
    if (lane < n_chunks) spg[lane] = pg0;
    if (lane + 32 < n_chunks) spg[lane + 32] = pg1;
    __syncwarp();
    if (lane == 0 && n_chunks > 0) {
      // ---------------- TMA producer (K/V pages; q tiles were issued at init) ----------------
      for (int j = 0; j < n_chunks; ++j) {
        const int st = j % STAGES;
        const int page = (j < 64) ? spg[j] : pages[j];
        MBW(&kv_empty[st], ((j / STAGES) & 1) ^ 1);
        if (MODE == MODE_SUMI && j == FREE_STAGES) MBW(self_done, 0);
        mbar_expect_tx(&kv_full[st], 2 * Ly::KVB);
        uint8_t* kd = smem + Ly::stage_off(st);
        tma_load_2d(kd, &tmKV, &kv_full[st], head * DH, (int)page_row(page, 0, 0));
        tma_load_2d(kd + Ly::KVB, &tmKV, &kv_full[st], head * DH, (int)page_row(page, 1, 0));
      }
    }
  } else if (warp == 1) {
    if (lane == 0 && n_chunks > 0) {
      // ---------------- MMA issuer ----------------
      constexpr uint32_t idesc_qk = idesc_bf16_major(ROWS, KEYS, 0, 0);
      constexpr uint32_t idesc_pv = idesc_bf16_major(ROWS, DH, 0, 1);
      const uint64_t qd = make_sdesc(smem_u32(smem + Ly::Q_OFF), 16, 8 * Ly::RB, Ly::SWZ);
      MBW(bar_q, 0);
      // S runs two chunks ahead of P: iteration j issues PV(j) and QK(j+2)
      // step by step interleaved (two independent accumulation chains keep the
      // tensor pipe busy; a lone chain of N=64 MMAs is latency-bound)
      auto kv_wait = [&](int j) {
        MBW(&kv_full[j % STAGES], (j / STAGES) & 1);
        fence_after();
      };
      auto kdesc = [&](int j) { return make_sdesc(smem_u32(smem + Ly::stage_off(j % STAGES)), 16, 8 * Ly::RB, Ly::SWZ); };
      for (int j = 0; j < 2 && j < n_chunks; ++j) {
        kv_wait(j);
        const uint64_t kd = kdesc(j);
        const uint32_t tSj = tmem_base + (j % NSB) * KEYS;
        if (tr && j < 8) tr[32 + j] = clock64();
#pragma unroll
        for (int s = 0; s < DH / 16; ++s) mma_bf16(tSj, qd + 2 * s, kd + 2 * s, idesc_qk, s > 0 ? 1u : 0u);
        mma_commit(&s_full[j % NSB]);
      }
      for (int j = 0; j < n_chunks; ++j) {
        const int st = j % STAGES;
        const int jq = j + 2;
        bool q = jq < n_chunks;
        uint64_t kd = 0;
        uint32_t tSq = 0;
        if (q) {
          if (j >= 1) MBW(&o_done[(j - 1) % NSB], ((j - 1) / NSB) & 1);  // buffer jq % 3: PV(j-1) read it
          kv_wait(jq);
          kd = kdesc(jq);
          tSq = tmem_base + (jq % NSB) * KEYS;
          if (ES) {  // S(j+2) now, before waiting for P(j)
#pragma unroll
            for (int s = 0; s < DH / 16; ++s) mma_bf16(tSq, qd + 2 * s, kd + 2 * s, idesc_qk, s > 0 ? 1u : 0u);
            mma_commit(&s_full[jq % NSB]);
            q = false;
          }
        }
        MBW(&p_full[j % NSB], (j / NSB) & 1);
        fence_after();
        if (tr && j < 8) tr[24 + j] = clock64();
        if (tr && q && jq < 8) tr[32 + jq] = clock64();
        const uint64_t vd = make_sdesc(smem_u32(smem + Ly::stage_off(st) + Ly::KVB), 16, 8 * Ly::RB, Ly::SWZ);
        const uint32_t tPj = tmem_base + (j % NSB) * KEYS;
#pragma unroll
        for (int s = 0; s < KEYS / 16; ++s) {
          const uint64_t vds = vd + (uint64_t)((16 * Ly::RB) >> 4) * s;  // 16 keys = 2 groups of 8 rows
          const uint32_t acc = (MODE == MODE_SUMI || j > 0 || s > 0) ? 1u : 0u;
          mma_bf16_ts(tO, tPj + 8 * s, vds, idesc_pv, acc);  // 16 keys of P = 8 packed columns
          if (q && s < DH / 16) mma_bf16(tSq, qd + 2 * s, kd + 2 * s, idesc_qk, s > 0 ? 1u : 0u);
        }
        mma_commit(&o_done[j % NSB]);
        mma_commit(&kv_empty[st]);
        if (q) mma_commit(&s_full[jq % NSB]);
      }
    }
  } else if (warp >= 4) {
    // ---------------- softmax + epilogue ----------------
    const int ew = warp - 4;
    const int row = ew * 32 + lane;  // query row = TMEM lane
    const uint32_t lane_off = (uint32_t)(ew * 32) << 16;
    const bool valid = row < n_rows;
    const int t_row = tile0 + row;
    // relative bias (Eq. 3 f_b, BIAS = 1): this (layer, block, scenario,
    // head)'s tables staged in smem; history token times / candidate-row bias
    float* sbp = reinterpret_cast<float*>(smem + Ly::BAR_OFF + 512);
    float* sbt = sbp + NB_POS;
    float* lut = sbt + 16;  // causal history: lut[bp * 7 + bt] = b_pos[bp] + b_time[bt], bp < 64, bt < 7
    const int* hag = nullptr;
    const float* cbr = nullptr;
    int t_age = 0;
    if constexpr (BIAS) {
      const long long br = bias_row(D, a.l, kblk, r, head);
      const int i = ew * 32 + lane;
      sbp[i] = D.bpos[br * NB_POS + i];
      if (i < NB_TIME) sbt[i] = D.btime[br * NB_TIME + i];
      if (MODE == MODE_HIST && D.causal)
        for (int e = i; e < 64 * 7; e += 128) lut[e] = D.bpos[br * NB_POS + e / 7] + D.btime[br * NB_TIME + e % 7];
      asm volatile("bar.sync 1, 128;" ::: "memory");
      hag = D.hage + ((long long)slot * D.Nb + kblk) * D.nk;
      cbr = D.cbias + ((((long long)slot * D.L + a.l) * D.Nb + kblk) * D.h + head) * D.nk;
      if (MODE == MODE_HIST && t_row < v) t_age = hag[t_row];
    }
    float m_used, l;
    if (MODE == MODE_SUMI) {
      // self term from the TMA-loaded q / k_self / v_self tiles (row = lane's
      // row, 16-byte chunks XOR-swizzled like the TMA box: 128B or 64B pattern)
      MBW(bar_q, 0);
      const uint8_t* qrow = smem + Ly::Q_OFF + row * Ly::RB;
      const uint8_t* krow = smem + Ly::KS_OFF + row * Ly::RB;
      const uint8_t* vrow = smem + Ly::VS_OFF + row * Ly::RB;
      auto swz = [&](int j) { return (DH == 64) ? (j ^ (row & 7)) : (j ^ ((row >> 1) & 3)); };
      float ss = 0.f;
#pragma unroll
      for (int j = 0; j < DH / 8; ++j) {
        float q[8], kk[8];
        load8(reinterpret_cast<const bf16*>(qrow + (swz(j) << 4)), q);
        load8(reinterpret_cast<const bf16*>(krow + (swz(j) << 4)), kk);
#pragma unroll
        for (int i = 0; i < 8; ++i) ss = fmaf(q[i], kk[i], ss);
      }
      if constexpr (BIAS) ss += sbp[bucket_pos(0)] + sbt[bucket_time(0)];  // self: offset 0, delta 0
      m_used = valid ? ss * sc : 0.f;
      l = 1.f;
#pragma unroll
      for (int c = 0; c < DH; c += 32) {  // O = v_self
        float vs[32];
#pragma unroll
        for (int cc = 0; cc < 32; cc += 8) {
          if (valid) {
            load8(reinterpret_cast<const bf16*>(vrow + (swz((c + cc) / 8) << 4)), vs + cc);
          } else {
#pragma unroll
            for (int i = 0; i < 8; ++i) vs[cc + i] = 0.f;
          }
        }
        tmem_st32(tO + lane_off + c, vs);
      }
      // the self tiles become K/V ring stages 3 and 4
      asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
      mbar_arrive(self_done);
    } else {
      m_used = -INFINITY;
      l = 0.f;
    }
    const bool causal_hist = (MODE == MODE_HIST) && D.causal;
    if (tracer) tr[2] = clock64();
    for (int j = 0; j < n_chunks; ++j) {
      const uint32_t tSj = tmem_base + (j % NSB) * KEYS + lane_off;
      MBW(&s_full[j % NSB], (j / NSB) & 1);
      fence_after();
      if (tracer && j < 9) tr[3 + 2 * j] = clock64();
      const int key0 = j * KEYS;
      int lim = key_end - key0;  // keys [0, lim) of the chunk are visible to this row
      if (causal_hist) lim = min(lim, t_row - key0 + 1);
      // pass 1: row max of the raw scores (8 independent partials)
      uint32_t sr[KEYS];
      tmem_ld32_nw(tSj, sr);
      tmem_ld32_nw(tSj + 32, sr + 32);
      tmem_ld_wait();
      if constexpr (BIAS) {  // R = QK^T + f_b (before the 1/(sqrt(d_h) tau) scaling, Eq. 3)
        if (MODE == MODE_SUMI) {
          const float4* c4 = reinterpret_cast<const float4*>(cbr + key0);
#pragma unroll
          for (int i = 0; i < KEYS; i += 4) {
            const float4 b = c4[i >> 2];
            sr[i] = __float_as_uint(__uint_as_float(sr[i]) + b.x);
            sr[i + 1] = __float_as_uint(__uint_as_float(sr[i + 1]) + b.y);
            sr[i + 2] = __float_as_uint(__uint_as_float(sr[i + 2]) + b.z);
            sr[i + 3] = __float_as_uint(__uint_as_float(sr[i + 3]) + b.w);
          }
        } else {
          // t_row - t_key = age_key - age_row; key ages 4 per 16-byte load
          const int4* a4 = reinterpret_cast<const int4*>(hag + key0);
          if (D.causal) {  // offsets >= 0 and time deltas >= 0 on every visible key: one 2-D lookup
#pragma unroll
            for (int i = 0; i < KEYS; i += 4) {
              const int4 ka = a4[i >> 2];
              const int kv4[4] = {ka.x, ka.y, ka.z, ka.w};
#pragma unroll
              for (int q = 0; q < 4; ++q) {
                const int bp = bucket_pos(t_row - (key0 + i + q)) & 63;   // masked keys (offset < 0) stay in range
                const int bt = bucket_time32(kv4[q] - t_age) % 7;
                sr[i + q] = __float_as_uint(__uint_as_float(sr[i + q]) + lut[bp * 7 + bt]);
              }
            }
          } else {
#pragma unroll
            for (int i = 0; i < KEYS; i += 4) {
              const int4 ka = a4[i >> 2];
              const int kv4[4] = {ka.x, ka.y, ka.z, ka.w};
#pragma unroll
              for (int q = 0; q < 4; ++q) {
                const float b = sbp[bucket_pos(t_row - (key0 + i + q))] + sbt[bucket_time32(kv4[q] - t_age)];
                sr[i + q] = __float_as_uint(__uint_as_float(sr[i + q]) + b);
              }
            }
          }
        }
      }
      float mx8[8];
#pragma unroll
      for (int i = 0; i < 8; ++i) mx8[i] = -INFINITY;
      const bool full = lim >= KEYS;  // no masking in full chunks (the common case)
      if (full) {
#pragma unroll
        for (int i = 0; i < KEYS; i += 2)
          mx8[(i >> 1) & 7] = max3(mx8[(i >> 1) & 7], __uint_as_float(sr[i]), __uint_as_float(sr[i + 1]));
      } else {
#pragma unroll
        for (int i = 0; i < KEYS; ++i)
          if (i < lim) mx8[i & 7] = fmaxf(mx8[i & 7], __uint_as_float(sr[i]));
      }
      const float mraw = fmaxf(fmaxf(fmaxf(mx8[0], mx8[1]), fmaxf(mx8[2], mx8[3])),
                               fmaxf(fmaxf(mx8[4], mx8[5]), fmaxf(mx8[6], mx8[7])));
      const float mx = mraw * sc;  // sc > 0
      // lazy rescale: per row, only when its max grew by > 2^8; the TMEM
      // ld/st are warp-collective (.sync.aligned), so the warp decides together
      const bool mine = mx > m_used + RESCALE_LOG2;
      const float alpha = mine ? exp2f(m_used - mx) : 1.f;  // m_used = -inf -> 0
      if (mine) {
        l *= alpha;
        m_used = mx;
      }
      if ((MODE == MODE_SUMI || j > 0) && __any_sync(0xffffffffu, mine)) {
        if (j > 0) MBW(&o_done[(j - 1) % NSB], ((j - 1) / NSB) & 1);  // PV(j-1) finished writing O
        fence_after();
#pragma unroll
        for (int c = 0; c < DH; c += 32) {
          float o[32];
          tmem_ld32(tO + lane_off + c, o);
#pragma unroll
          for (int i = 0; i < 32; ++i) o[i] *= alpha;
          tmem_st32(tO + lane_off + c, o);
        }
      }
      // pass 2: P = exp2(s sc - m) as packed bf16, written over S_j in TMEM
      const float nb = (m_used == -INFINITY) ? 0.f : -m_used;
      float ls8[8] = {0.f, 0.f, 0.f, 0.f, 0.f, 0.f, 0.f, 0.f};
      uint32_t pk[KEYS / 2];
      if (full) {
        const uint64_t sc2 = pk2(sc, sc), nb2 = pk2(nb, nb);
        uint64_t ls2[4] = {0ull, 0ull, 0ull, 0ull};  // packed (0.f, 0.f)
#pragma unroll
        for (int i = 0; i < KEYS; i += 2) {
          const float2 x = upk2(fma2(pk2(__uint_as_float(sr[i]), __uint_as_float(sr[i + 1])), sc2, nb2));
          const float e0 = ((i & 7) < PE8) ? ex2_poly(x.x) : ex2_approx(x.x);
          const float e1 = (((i + 1) & 7) < PE8) ? ex2_poly(x.y) : ex2_approx(x.y);
          ls2[(i >> 1) & 3] = add2(ls2[(i >> 1) & 3], pk2(e0, e1));
          __nv_bfloat162 pp = __floats2bfloat162_rn(e0, e1);
          pk[i >> 1] = *reinterpret_cast<uint32_t*>(&pp);
        }
#pragma unroll
        for (int q = 0; q < 4; ++q) {
          const float2 t = upk2(ls2[q]);
          ls8[2 * q] = t.x;
          ls8[2 * q + 1] = t.y;
        }
      } else {
#pragma unroll
        for (int i = 0; i < KEYS; i += 2) {
          const float e0 = (i < lim) ? ex2_approx(fmaf(__uint_as_float(sr[i]), sc, nb)) : 0.f;
          const float e1 = (i + 1 < lim) ? ex2_approx(fmaf(__uint_as_float(sr[i + 1]), sc, nb)) : 0.f;
          ls8[i & 7] += e0;
          ls8[(i + 1) & 7] += e1;
          __nv_bfloat162 pp = __floats2bfloat162_rn(e0, e1);
          pk[i >> 1] = *reinterpret_cast<uint32_t*>(&pp);
        }
      }
      tmem_st16u(tSj, pk);
      tmem_st16u(tSj + 16, pk + 16);
      tmem_st_wait();
      l += ((ls8[0] + ls8[1]) + (ls8[2] + ls8[3])) + ((ls8[4] + ls8[5]) + (ls8[6] + ls8[7]));
      fence_before();
      mbar_arrive(&p_full[j % NSB]);
      if (tracer && j < 9) tr[4 + 2 * j] = clock64();

    }
    // ---- epilogue: O / l -> bf16, staged in smem for coalesced stores
    if (n_chunks > 0) {
      MBW(&o_done[(n_chunks - 1) % NSB], ((n_chunks - 1) / NSB) & 1);
      fence_after();
    }
    if (tracer) tr[21] = clock64();
    const float inv = (valid && l > 0.f) ? 1.f / l : 0.f;
    constexpr int LDS = DH + 8;
    bf16* stg = reinterpret_cast<bf16*>(smem + Ly::STG_OFF);  // K/V ring fully consumed (last PV done)
#pragma unroll
    for (int c = 0; c < DH; c += 32) {
      float o[32];
      if (MODE == MODE_SUMI || n_chunks > 0) {
        tmem_ld32(tO + lane_off + c, o);
      } else {
#pragma unroll
        for (int i = 0; i < 32; ++i) o[i] = 0.f;
      }
#pragma unroll
      for (int cc = 0; cc < 32; cc += 8) {
        float y[8];
#pragma unroll
        for (int i = 0; i < 8; ++i) y[i] = o[cc + i] * inv;
        store8(stg + row * LDS + c + cc, y);
      }
    }
    __syncwarp();
    if (tracer) tr[23] = clock64();
    const int rows_out = (MODE == MODE_SUMI) ? n_rows : min(ROWS, D.nk - tile0);
    constexpr int LPR = DH / 8;      // lanes per row, 16 B (8 bf16) each
    constexpr int RPI = 32 / LPR;    // rows per warp instruction
#pragma unroll
    for (int i = 0; i < 32; i += RPI) {
      const int rr = ew * 32 + i + lane / LPR;
      const int cc = (lane % LPR) * 8;
      if (rr < rows_out) {
        const uint4 val = *reinterpret_cast<const uint4*>(stg + rr * LDS + cc);
        *reinterpret_cast<uint4*>(a.O + (row_base + rr) * D.d + head * DH + cc) = val;
      }
    }
    if (tracer) tr[22] = clock64();
  }
  fence_before();
  __syncthreads();
  if (warp == 2) {
    fence_after();
    asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem_base), "r"(256));
  }
}

// ===========================================================================
// Persistent two-tile attention (CLIMBER_ATTN_KERNEL=2).  One CTA per SM (all 512 TMEM
// columns) loops over work items; an item = two adjacent 128-row query tiles
// of one (user, block, head), so every K/V page loaded serves 256 query rows.
//   warp 0     K/V producer: streams 64-key pages of every item into a ring
//              that runs across items (the warp holds the item's page ids)
//   warp 1     MMA issuer of tile 0, warp 3 of tile 1 (one thread each): S =
//              Q K^T two chunks ahead, issued as soon as its TMEM buffer is
//              free, and O += P V (P from TMEM, V MN-major); the two tiles share
//              only the K/V ring (each stage is released by both threads)
//   warp 2     TMEM allocator, then item decoder + Q / k_self / v_self
//              producer: writes the item's descriptor to smem and loads its q
//              tiles into one of two buffers while the previous item still runs
//   warps 4-7  softmax + epilogue of tile 0, warps 8-11 of tile 1; each
//              warpgroup owns half of TMEM (3 x 64 score/P columns + d_h
//              output columns); the two ping-pong on the MUFU
// Row arithmetic is identical to k_attn_tc (same online-softmax steps).
// ===========================================================================
constexpr int PT_THREADS = 384;
constexpr int PT_WT = 2;  // query tiles per item

template <int DH>
struct PLay {
  static constexpr int RB = DH * 2;
  static constexpr uint32_t SWZ = (DH == 64) ? 2u : 4u;
  static constexpr int QB = ROWS * RB;   // one 128-row tile of q (or k_self, v_self)
  static constexpr int KVB = KEYS * RB;  // one 64-key page slice of K (or V) of one head
  static constexpr int Q_OFF = 0;        // [2 buffers][PT_WT tiles]
  static constexpr int KS_OFF = Q_OFF + 2 * PT_WT * QB;
  static constexpr int VS_OFF = KS_OFF + PT_WT * QB;
  static constexpr int KV_OFF = VS_OFF + PT_WT * QB;
  static constexpr int ST_RAW = (232448 - 1024 - 2048 - KV_OFF) / (2 * KVB);
  static constexpr int ST = ST_RAW > 8 ? 8 : ST_RAW;  // K/V ring stages
  static constexpr int BAR_OFF = KV_OFF + ST * 2 * KVB;
  static constexpr int DESC_OFF = BAR_OFF + 512;
  static constexpr int TOTAL = BAR_OFF + 1024 + 1024;
  static_assert(ST >= 4, "K/V ring too shallow");
  static_assert(TOTAL <= 232448, "smem");
};

struct PArgs {
  Args a;
  int n_pairs;  // items per (z, head)
  long long n_items;
};

// One work item as the decoder wrote it to shared memory.
struct PDesc {
  long long row_base[PT_WT];
  int n_rows[PT_WT], rows_out[PT_WT], nch[PT_WT], key_end[PT_WT], tile0[PT_WT];
  int nkv, head, end;
  float sc;
};

template <int DH, int MODE>
__device__ __forceinline__ bool pt_decode(const PArgs& pa, long long it, PDesc& I, const int** pages) {
  const Args& a = pa.a;
  const Dims& D = a.D;
  const int pair = (int)(it % pa.n_pairs);
  const long long rest = it / pa.n_pairs;
  I.head = (int)(rest % D.h);
  const int z = (int)(rest / D.h);
  const int u = z % a.U, kk = z / a.U, kblk = a.k + kk;
  const int slot = a.wave_slot[u];
  const int v = a.vlen_all[(long long)slot * D.Nb + kblk];
  *pages = a.ptab + (((long long)slot * D.Nb + kblk) * D.L + a.l) * D.ppb;
  I.nkv = 0;
  I.end = 0;
  bool live = false;
  long long p0 = 0, mu = 0;
  if (MODE == MODE_SUMI) {
    p0 = a.cand_off[u];
    mu = a.cand_off[u + 1] - p0;
  }
#pragma unroll
  for (int w = 0; w < PT_WT; ++w) {
    const int t0 = (pair * PT_WT + w) * ROWS;
    I.tile0[w] = t0;
    if (MODE == MODE_SUMI) {
      const long long left = mu - t0;
      I.n_rows[w] = left <= 0 ? 0 : (left < ROWS ? (int)left : ROWS);
      I.rows_out[w] = I.n_rows[w];
      I.key_end[w] = v;
      I.nch[w] = I.n_rows[w] > 0 ? (v + KEYS - 1) / KEYS : 0;
      I.row_base[w] = kk * a.rows_pb + p0 + t0;
    } else {
      I.rows_out[w] = t0 < D.nk ? min(ROWS, D.nk - t0) : 0;
      I.n_rows[w] = max(0, min(ROWS, v - t0));
      I.key_end[w] = D.causal ? min(v, t0 + ROWS) : v;
      I.nch[w] = I.n_rows[w] > 0 ? (I.key_end[w] + KEYS - 1) / KEYS : 0;
      I.row_base[w] = kk * a.rows_pb + (long long)u * D.nk + t0;
    }
    I.nkv = max(I.nkv, I.nch[w]);
    live = live || I.rows_out[w] > 0;
  }
  if (live) {
    const int r = a.wave_r[u];
    I.sc = LOG2E / (sqrtf((float)DH) * a.tau[((a.l * D.Nb + kblk) * D.R + r) * D.h + I.head]);
  }
  return live;
}

template <int DH, int MODE>
__global__ void __launch_bounds__(PT_THREADS, 1)
    k_attn_pt(const __grid_constant__ CUtensorMap tmQ, const __grid_constant__ CUtensorMap tmKV, PArgs pa) {
  using Ly = PLay<DH>;
  constexpr int ST = Ly::ST;
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  uint64_t* bars = reinterpret_cast<uint64_t*>(smem + Ly::BAR_OFF);
  uint64_t* q_full = bars + 0;        // [2] item descriptor + q tiles of buffer b
  uint64_t* q_empty = bars + 2;       // [2] MMA read q (last QK) and every softmax thread read the descriptor
  uint64_t* self_full = bars + 4;     // SUMI: k_self / v_self tiles landed
  uint64_t* self_empty = bars + 5;    // SUMI: both warpgroups read them
  uint64_t* kv_full = bars + 6;       // [ST]
  uint64_t* kv_empty = kv_full + ST;  // [ST]
  uint64_t* s_full = kv_empty + ST;   // [PT_WT][NSB]
  uint64_t* p_full = s_full + PT_WT * NSB;
  uint64_t* o_done = p_full + PT_WT * NSB;
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(o_done + PT_WT * NSB);
  PDesc* desc = reinterpret_cast<PDesc*>(smem + Ly::DESC_OFF);  // [2]

  const Args& a = pa.a;
  const Dims& D = a.D;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;

  if (warp == 0 && lane == 0) {
    asm volatile("prefetch.tensormap [%0];" ::"l"(&tmQ) : "memory");
    asm volatile("prefetch.tensormap [%0];" ::"l"(&tmKV) : "memory");
    for (int b = 0; b < 2; ++b) {
      mbar_init(&q_full[b], 1);
      mbar_init(&q_empty[b], 2 + 256);  // both MMA threads + every softmax thread
    }
    mbar_init(self_full, 1);
    mbar_init(self_empty, 256);
    for (int s = 0; s < ST; ++s) {
      mbar_init(&kv_full[s], 1);
      mbar_init(&kv_empty[s], 2);  // released by both tiles' MMA threads
    }
    for (int b = 0; b < PT_WT * NSB; ++b) {
      mbar_init(&s_full[b], 1);
      mbar_init(&p_full[b], 128);
      mbar_init(&o_done[b], 1);
    }
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  if (warp == 2) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(smem_u32(tmem_slot)),
                 "r"(512));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  fence_before();
  __syncthreads();
  fence_after();
  const uint32_t tmem_base = *tmem_slot;

  if (warp == 0) {
    // ---------------- K/V producer ----------------
    long long gk = 0;
    for (long long it = blockIdx.x; it < pa.n_items; it += gridDim.x) {
      PDesc I;
      const int* pages;
      if (!pt_decode<DH, MODE>(pa, it, I, &pages)) continue;
      const int pg0 = lane < I.nkv ? pages[lane] : 0;
      const int pg1 = lane + 32 < I.nkv ? pages[lane + 32] : 0;
      for (int j = 0; j < I.nkv; ++j, ++gk) {
        const int page = j < 64 ? __shfl_sync(0xffffffffu, j < 32 ? pg0 : pg1, j & 31) : pages[j];
        if (lane == 0) {
          const int st = (int)(gk % ST);
          MBW(&kv_empty[st], (uint32_t)((gk / ST) & 1) ^ 1);
          mbar_expect_tx(&kv_full[st], 2 * Ly::KVB);
          uint8_t* kd = smem + Ly::KV_OFF + st * 2 * Ly::KVB;
          tma_load_2d(kd, &tmKV, &kv_full[st], I.head * DH, (int)page_row(page, 0, 0));
          tma_load_2d(kd + Ly::KVB, &tmKV, &kv_full[st], I.head * DH, (int)page_row(page, 1, 0));
        }
      }
      __syncwarp();
    }
  } else if (warp == 2) {
    // ---------------- item decoder + q / self producer (after the TMEM alloc) ----------------
    if (lane == 0) {
      long long seq = 0;
      for (long long it = blockIdx.x;; it += gridDim.x) {
        PDesc I;
        const int* pages;
        const bool done = it >= pa.n_items;
        if (!done && !pt_decode<DH, MODE>(pa, it, I, &pages)) continue;
        const int b = (int)(seq & 1);
        MBW(&q_empty[b], (uint32_t)((seq >> 1) & 1) ^ 1);
        if (done) {
          desc[b].end = 1;
          mbar_arrive(&q_full[b]);
          break;
        }
        desc[b] = I;
        uint32_t bytes = 0;
#pragma unroll
        for (int w = 0; w < PT_WT; ++w)
          if (MODE == MODE_SUMI ? I.n_rows[w] > 0 : I.nch[w] > 0) bytes += Ly::QB;
        mbar_expect_tx(&q_full[b], bytes);
#pragma unroll
        for (int w = 0; w < PT_WT; ++w)
          if (MODE == MODE_SUMI ? I.n_rows[w] > 0 : I.nch[w] > 0)
            tma_load_2d(smem + Ly::Q_OFF + (b * PT_WT + w) * Ly::QB, &tmQ, &q_full[b], I.head * DH,
                        (int)I.row_base[w]);
        if (MODE == MODE_SUMI) {
          MBW(self_empty, (uint32_t)(seq & 1) ^ 1);
          uint32_t sb = 0;
#pragma unroll
          for (int w = 0; w < PT_WT; ++w)
            if (I.n_rows[w] > 0) sb += 2 * Ly::QB;
          mbar_expect_tx(self_full, sb);
#pragma unroll
          for (int w = 0; w < PT_WT; ++w) {
            if (I.n_rows[w] <= 0) continue;
            tma_load_2d(smem + Ly::KS_OFF + w * Ly::QB, &tmQ, self_full, D.d + I.head * DH, (int)I.row_base[w]);
            tma_load_2d(smem + Ly::VS_OFF + w * Ly::QB, &tmQ, self_full, 2 * D.d + I.head * DH, (int)I.row_base[w]);
          }
        }
        ++seq;
      }
    }
  } else if (warp == 1 || warp == 3) {
    if (lane == 0) {
      // ---------------- MMA issuer of one tile (warp 1: tile 0, warp 3: tile 1) ----------------
      // The two tiles share only the K/V ring (kv_empty needs both threads) and
      // the q buffers; each runs its own S -> P -> PV chain.
      const int w = warp == 1 ? 0 : 1;
      constexpr uint32_t idesc_qk = idesc_bf16_major(ROWS, KEYS, 0, 0);
      constexpr uint32_t idesc_pv = idesc_bf16_major(ROWS, DH, 0, 1);
      long long gk = 0, cs = 0;
      for (long long seq = 0;; ++seq) {
        const int b = (int)(seq & 1);
        MBW(&q_full[b], (uint32_t)((seq >> 1) & 1));
        fence_after();
        const PDesc& I = desc[b];
        if (I.end) break;
        const int nch = I.nch[w];
        const int nkv = I.nkv;
        auto kv_wait = [&](int j) {
          MBW(&kv_full[(gk + j) % ST], (uint32_t)(((gk + j) / ST) & 1));
          fence_after();
        };
        auto kdesc = [&](int j) {
          return make_sdesc(smem_u32(smem + Ly::KV_OFF + (int)((gk + j) % ST) * 2 * Ly::KVB), 16, 8 * Ly::RB, Ly::SWZ);
        };
        const uint64_t qd = make_sdesc(smem_u32(smem + Ly::Q_OFF + (b * PT_WT + w) * Ly::QB), 16, 8 * Ly::RB, Ly::SWZ);
        auto sbuf = [&](long long c) { return tmem_base + w * 256 + (uint32_t)(c % NSB) * KEYS; };
        const uint32_t tO = tmem_base + w * 256 + NSB * KEYS;
        for (int j = 0; j < 2 && j < nch; ++j) {
          kv_wait(j);
          const uint64_t kd = kdesc(j);
          const long long c = cs + j;  // score buffer c % 3 was last read by PV(c - 3)
          if (c >= 3) MBW(&o_done[w * NSB + (int)((c - 3) % NSB)], (uint32_t)(((c - 3) / NSB) & 1));
#pragma unroll
          for (int s = 0; s < DH / 16; ++s) mma_bf16(sbuf(c), qd + 2 * s, kd + 2 * s, idesc_qk, s > 0 ? 1u : 0u);
          mma_commit(&s_full[w * NSB + (int)(c % NSB)]);
        }
        if (nch <= 2) mma_commit(&q_empty[b]);
        for (int j = 0; j < nkv; ++j) {
          if (j >= nch) {  // chunk unused by this tile: release the stage once it has landed
            kv_wait(j);
            mbar_arrive(&kv_empty[(gk + j) % ST]);
            continue;
          }
          const int jq = j + 2;
          const long long c = cs + j;
          if (jq < nch) {  // S(j+2) as soon as its buffer is free (PV(j-1) done)
            kv_wait(jq);
            const uint64_t kq = kdesc(jq);
            if (c >= 1) MBW(&o_done[w * NSB + (int)((c - 1) % NSB)], (uint32_t)(((c - 1) / NSB) & 1));
            fence_after();
#pragma unroll
            for (int s = 0; s < DH / 16; ++s) mma_bf16(sbuf(c + 2), qd + 2 * s, kq + 2 * s, idesc_qk, s > 0 ? 1u : 0u);
            mma_commit(&s_full[w * NSB + (int)((c + 2) % NSB)]);
            if (jq == nch - 1) mma_commit(&q_empty[b]);  // this tile's last QK has been issued
          }
          if (j < 2) kv_wait(j);  // (chunks >= 2 were waited for when their S was issued)
          const uint64_t vd = kdesc(j) + (uint64_t)(Ly::KVB >> 4);
          MBW(&p_full[w * NSB + (int)(c % NSB)], (uint32_t)((c / NSB) & 1));
          fence_after();
#pragma unroll
          for (int s = 0; s < KEYS / 16; ++s) {
            const uint64_t vds = vd + (uint64_t)((16 * Ly::RB) >> 4) * s;
            const uint32_t acc = (MODE == MODE_SUMI || j > 0 || s > 0) ? 1u : 0u;
            mma_bf16_ts(tO, sbuf(c) + 8 * s, vds, idesc_pv, acc);
          }
          mma_commit(&o_done[w * NSB + (int)(c % NSB)]);
          mma_commit(&kv_empty[(gk + j) % ST]);
        }
        gk += nkv;
        cs += nch;
      }
    }
  } else if (warp >= 4) {
    // ---------------- softmax + epilogue, warpgroup wg owns tile wg ----------------
    const int wg = (warp - 4) >> 2;
    const int ew = (warp - 4) & 3;
    const int row = ew * 32 + lane;
    const uint32_t lane_off = (uint32_t)(ew * 32) << 16;
    const uint32_t tO = tmem_base + wg * 256 + NSB * KEYS + lane_off;
    long long cs = 0;
    for (long long seq = 0;; ++seq) {
      const int b = (int)(seq & 1);
      MBW(&q_full[b], (uint32_t)((seq >> 1) & 1));
      const PDesc& I = desc[b];
      if (I.end) break;
      const int nch = I.nch[wg];
      const int n_rows = I.n_rows[wg];
      const int key_end = I.key_end[wg];
      const int rows_out = I.rows_out[wg];
      const long long row_base = I.row_base[wg];
      const int tile0 = I.tile0[wg];
      const int head = I.head;
      const float sc = I.sc;
      const bool valid = row < n_rows;
      float m_used, l;
      if (MODE == MODE_SUMI) {
        MBW(self_full, (uint32_t)(seq & 1));
        if (n_rows > 0) {
          const uint8_t* qrow = smem + Ly::Q_OFF + (b * PT_WT + wg) * Ly::QB + row * Ly::RB;
          const uint8_t* krow = smem + Ly::KS_OFF + wg * Ly::QB + row * Ly::RB;
          const uint8_t* vrow = smem + Ly::VS_OFF + wg * Ly::QB + row * Ly::RB;
          auto swz = [&](int j) { return (DH == 64) ? (j ^ (row & 7)) : (j ^ ((row >> 1) & 3)); };
          float ss = 0.f;
#pragma unroll
          for (int j = 0; j < DH / 8; ++j) {
            float q[8], kk[8];
            load8(reinterpret_cast<const bf16*>(qrow + (swz(j) << 4)), q);
            load8(reinterpret_cast<const bf16*>(krow + (swz(j) << 4)), kk);
#pragma unroll
            for (int i = 0; i < 8; ++i) ss = fmaf(q[i], kk[i], ss);
          }
          m_used = valid ? ss * sc : 0.f;
          l = 1.f;
#pragma unroll
          for (int c = 0; c < DH; c += 32) {  // O = v_self
            float vs[32];
#pragma unroll
            for (int cc = 0; cc < 32; cc += 8) {
              if (valid) {
                load8(reinterpret_cast<const bf16*>(vrow + (swz((c + cc) / 8) << 4)), vs + cc);
              } else {
#pragma unroll
                for (int i = 0; i < 8; ++i) vs[cc + i] = 0.f;
              }
            }
            tmem_st32(tO + c, vs);
          }
        } else {
          m_used = 0.f;
          l = 1.f;
        }
        fence_before();
        mbar_arrive(self_empty);
      } else {
        m_used = -INFINITY;
        l = 0.f;
      }
      mbar_arrive(&q_empty[b]);  // descriptor (and q rows) read
      const bool causal_hist = (MODE == MODE_HIST) && D.causal;
      const int t_row = tile0 + row;
      for (int j = 0; j < nch; ++j) {
        const long long c = cs + j;
        const int bb = (int)(c % NSB);
        const uint32_t tSj = tmem_base + wg * 256 + bb * KEYS + lane_off;
        MBW(&s_full[wg * NSB + bb], (uint32_t)((c / NSB) & 1));
        fence_after();
        const int key0 = j * KEYS;
        int lim = key_end - key0;
        if (causal_hist) lim = min(lim, t_row - key0 + 1);
        uint32_t sr[KEYS];
        tmem_ld32_nw(tSj, sr);
        tmem_ld32_nw(tSj + 32, sr + 32);
        tmem_ld_wait();
        float mx8[8];
#pragma unroll
        for (int i = 0; i < 8; ++i) mx8[i] = -INFINITY;
        const bool full = lim >= KEYS;
        if (full) {
#pragma unroll
          for (int i = 0; i < KEYS; i += 2)
            mx8[(i >> 1) & 7] = max3(mx8[(i >> 1) & 7], __uint_as_float(sr[i]), __uint_as_float(sr[i + 1]));
        } else {
#pragma unroll
          for (int i = 0; i < KEYS; ++i)
            if (i < lim) mx8[i & 7] = fmaxf(mx8[i & 7], __uint_as_float(sr[i]));
        }
        const float mraw = fmaxf(fmaxf(fmaxf(mx8[0], mx8[1]), fmaxf(mx8[2], mx8[3])),
                                 fmaxf(fmaxf(mx8[4], mx8[5]), fmaxf(mx8[6], mx8[7])));
        const float mx = mraw * sc;
        const bool mine = mx > m_used + RESCALE_LOG2;
        const float alpha = mine ? exp2f(m_used - mx) : 1.f;
        if (mine) {
          l *= alpha;
          m_used = mx;
        }
        if ((MODE == MODE_SUMI || j > 0) && __any_sync(0xffffffffu, mine)) {
          if (j > 0) MBW(&o_done[wg * NSB + (int)((c - 1) % NSB)], (uint32_t)(((c - 1) / NSB) & 1));
          fence_after();
#pragma unroll
          for (int cc = 0; cc < DH; cc += 32) {
            float o[32];
            tmem_ld32(tO + cc, o);
#pragma unroll
            for (int i = 0; i < 32; ++i) o[i] *= alpha;
            tmem_st32(tO + cc, o);
          }
        }
        const float nb = (m_used == -INFINITY) ? 0.f : -m_used;
        float ls8[8] = {0.f, 0.f, 0.f, 0.f, 0.f, 0.f, 0.f, 0.f};
        uint32_t pk[KEYS / 2];
        if (full) {
          const uint64_t sc2 = pk2(sc, sc), nb2 = pk2(nb, nb);
          uint64_t ls2[4] = {0ull, 0ull, 0ull, 0ull};
#pragma unroll
          for (int i = 0; i < KEYS; i += 2) {
            const float2 x = upk2(fma2(pk2(__uint_as_float(sr[i]), __uint_as_float(sr[i + 1])), sc2, nb2));
            const float e0 = ex2_approx(x.x);
            const float e1 = ex2_approx(x.y);
            ls2[(i >> 1) & 3] = add2(ls2[(i >> 1) & 3], pk2(e0, e1));
            __nv_bfloat162 pp = __floats2bfloat162_rn(e0, e1);
            pk[i >> 1] = *reinterpret_cast<uint32_t*>(&pp);
          }
#pragma unroll
          for (int q = 0; q < 4; ++q) {
            const float2 t = upk2(ls2[q]);
            ls8[2 * q] = t.x;
            ls8[2 * q + 1] = t.y;
          }
        } else {
#pragma unroll
          for (int i = 0; i < KEYS; i += 2) {
            const float e0 = (i < lim) ? ex2_approx(fmaf(__uint_as_float(sr[i]), sc, nb)) : 0.f;
            const float e1 = (i + 1 < lim) ? ex2_approx(fmaf(__uint_as_float(sr[i + 1]), sc, nb)) : 0.f;
            ls8[i & 7] += e0;
            ls8[(i + 1) & 7] += e1;
            __nv_bfloat162 pp = __floats2bfloat162_rn(e0, e1);
            pk[i >> 1] = *reinterpret_cast<uint32_t*>(&pp);
          }
        }
        tmem_st16u(tSj, pk);
        tmem_st16u(tSj + 16, pk + 16);
        tmem_st_wait();
        l += ((ls8[0] + ls8[1]) + (ls8[2] + ls8[3])) + ((ls8[4] + ls8[5]) + (ls8[6] + ls8[7]));
        fence_before();
        mbar_arrive(&p_full[wg * NSB + bb]);
      }
      // ---- epilogue: O / l -> bf16, one 2*DH-byte row per thread straight to global
      if (nch > 0) {
        const long long c = cs + nch - 1;
        MBW(&o_done[wg * NSB + (int)(c % NSB)], (uint32_t)((c / NSB) & 1));
        fence_after();
      }
      const bool have_o = (MODE == MODE_SUMI) ? n_rows > 0 : nch > 0;
      const float inv = (valid && l > 0.f) ? 1.f / l : 0.f;
      bf16* orow = a.O + (row_base + row) * D.d + head * DH;
      const bool wr_row = row < rows_out;
#pragma unroll
      for (int cc = 0; cc < DH; cc += 32) {
        float o[32];
        if (have_o) {
          tmem_ld32(tO + cc, o);
        } else {
#pragma unroll
          for (int i = 0; i < 32; ++i) o[i] = 0.f;
        }
        if (wr_row) {
#pragma unroll
          for (int q = 0; q < 32; q += 8) {
            float y[8];
#pragma unroll
            for (int i = 0; i < 8; ++i) y[i] = o[q + i] * inv;
            store8(orow + cc + q, y);
          }
        }
      }
      fence_before();  // TMEM reads of O complete before the next item's PV / init
      cs += nch;
    }
  }
  fence_before();
  __syncthreads();
  if (warp == 2) {
    fence_after();
    asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem_base), "r"(512));
  }
}

static PFN_cuTensorMapEncodeTiled_v12000 encoder() {
  static PFN_cuTensorMapEncodeTiled_v12000 fn = nullptr;
  static std::once_flag once;
  std::call_once(once, [] {
    void* p = nullptr;
    cudaDriverEntryPointQueryResult q;
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q) == cudaSuccess &&
        q == cudaDriverEntryPointSuccess)
      fn = reinterpret_cast<PFN_cuTensorMapEncodeTiled_v12000>(p);
  });
  return fn;
}

// 2-D bf16 map: [rows][cols] with row stride ld, box {box_cols, box_rows}, swizzle = box row bytes
static bool map2d(CUtensorMap* m, const void* base, long long rows, int cols, long long ld, int box_cols,
                  int box_rows) {
  auto enc = encoder();
  if (!enc) return false;
  cuuint64_t dims[2] = {(cuuint64_t)cols, (cuuint64_t)rows};
  cuuint64_t strides[1] = {(cuuint64_t)ld * 2};
  cuuint32_t box[2] = {(cuuint32_t)box_cols, (cuuint32_t)box_rows};
  cuuint32_t estr[2] = {1, 1};
  CUtensorMapSwizzle sw = box_cols * 2 == 128 ? CU_TENSOR_MAP_SWIZZLE_128B : CU_TENSOR_MAP_SWIZZLE_64B;
  return enc(m, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2, const_cast<void*>(base), dims, strides, box, estr,
             CU_TENSOR_MAP_INTERLEAVE_NONE, sw, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
             CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) == CUDA_SUCCESS;
}

template <int DH, int MODE, int PE8>
static void launch_pe(const CUtensorMap& mq, const CUtensorMap& mkv, const Args& a, dim3 grid, cudaStream_t s) {
  // CLIMBER_ATTN_1CTA=1 (measurement knob): request enough smem for 1 CTA/SM
  static const int smem = getenv("CLIMBER_ATTN_1CTA") ? 150 * 1024 : Lay<DH>::TOTAL;
  constexpr int smem_b = Lay<DH>::TOTAL + 3072;  // + the staged relative-bias tables and 2-D lookup
  static const bool es = [] { const char* e = getenv("CLIMBER_ATTN_EARLY_S"); return !(e && atoi(e) == 0); }();
  ensure_smem_attr((const void*)k_attn_tc<DH, MODE, PE8, 0>, smem);
  ensure_smem_attr((const void*)k_attn_tc<DH, MODE, PE8, 1>, smem);
  ensure_smem_attr((const void*)k_attn_tc<DH, MODE, PE8, 1, 1>, smem_b);
  if (a.D.bpos) k_attn_tc<DH, MODE, PE8, 1, 1><<<grid, THREADS, smem_b, s>>>(mq, mkv, a);
  else if (es) k_attn_tc<DH, MODE, PE8, 1><<<grid, THREADS, smem, s>>>(mq, mkv, a);
  else k_attn_tc<DH, MODE, PE8, 0><<<grid, THREADS, smem, s>>>(mq, mkv, a);
}

template <int DH, int MODE>
static void launch(const CUtensorMap& mq, const CUtensorMap& mkv, const Args& a, dim3 grid, cudaStream_t s) {
  // n of every 8 exponentials on the FMA pipe (degree-3 polynomial) instead of
  // the MUFU: 1 measured +0.8% (SUMI) over 0, 2 slower (CLIMBER_ATTN_PE8 = n)
  static const int pe8 = [] { const char* e = getenv("CLIMBER_ATTN_PE8"); return e ? atoi(e) : 1; }();
  switch (pe8) {
    case 1: launch_pe<DH, MODE, 1>(mq, mkv, a, grid, s); break;
    case 2: launch_pe<DH, MODE, 2>(mq, mkv, a, grid, s); break;
    default: launch_pe<DH, MODE, 0>(mq, mkv, a, grid, s); break;
  }
}

template <int DH, int MODE>
static void launch_pt(const CUtensorMap& mq, const CUtensorMap& mkv, const PArgs& pa, cudaStream_t s) {
  constexpr int smem = PLay<DH>::TOTAL;
  static bool attr = false;
  static int n_sm = 148;
  if (!attr) {
    cudaFuncSetAttribute(k_attn_pt<DH, MODE>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
    int dev = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&n_sm, cudaDevAttrMultiProcessorCount, dev);
    attr = true;
  }
  if (pa.n_items <= 0) return;
  const int grid = (int)(pa.n_items < n_sm ? pa.n_items : n_sm);
  k_attn_pt<DH, MODE><<<grid, PT_THREADS, smem, s>>>(mq, mkv, pa);
}

// CLIMBER_ATTN_KERNEL=2 selects the persistent two-tile kernel (measured 2%
// slower than two one-tile CTAs per SM at `large`; kept as a knob)
static bool use_pt() {
  static bool v = [] {
    const char* e = getenv("CLIMBER_ATTN_KERNEL");
    return e && atoi(e) == 2;
  }();
  return v;
}

}  // namespace at

// CLIMBER_ATTN_FA=0 keeps the one-tile kernel below for A/B measurements
static bool use_fa() {
  static const bool v = [] { const char* e = getenv("CLIMBER_ATTN_FA"); return !(e && atoi(e) == 0); }();
  return v;
}

bool attn_tc_supported(int dh, int nk, bool hist) {
  if (dh != 32 && dh != 64) return false;
  if (hist && nk % at::ROWS) return false;
  return at::encoder() != nullptr;
}

void launch_attn_sumi_tc(const bf16* QKV, long long P, const int64_t* cand_off, const int* wave_slot,
                         const int* wave_r, int U, int Mmax, const bf16* pool, long long pool_rows, const int* ptab,
                         const int* vlen_all, const float* tau, bf16* O, int k, int l, const Dims& D, cudaStream_t s,
                         int nbk) {
  if (!D.bpos && use_fa() && attn_fa_supported(D.dh, D.nk)) {
    launch_attn_sumi_fa(QKV, P, cand_off, wave_slot, wave_r, U, Mmax, pool, pool_rows, ptab, vlen_all, tau, O, k, l,
                        D, s, nbk);
    return;
  }
  CUtensorMap mq, mkv;
  if (!at::map2d(&mq, QKV, P * nbk, 3 * D.d, 3LL * D.d, D.dh, at::ROWS) ||
      !at::map2d(&mkv, pool, pool_rows, D.d, D.d, D.dh, at::KEYS)) {
    note_launch_error("SUMI attention: cuTensorMapEncodeTiled rejected a map (kernel not launched)");
    return;
  }
  at::Args a{QKV, cand_off, wave_slot, wave_r, ptab, vlen_all, tau, O, k, l, U, P, D, nullptr};
  dim3 grid((Mmax + at::ROWS - 1) / at::ROWS, D.h, U * nbk);
  if (at::use_pt() && !D.bpos) {
    at::PArgs pa{a, (int)((grid.x + at::PT_WT - 1) / at::PT_WT), 0};
    pa.n_items = (long long)pa.n_pairs * D.h * U * nbk;
    if (D.dh == 64) at::launch_pt<64, at::MODE_SUMI>(mq, mkv, pa, s);
    else at::launch_pt<32, at::MODE_SUMI>(mq, mkv, pa, s);
    return;
  }
  // debug timeline: CLIMBER_ATTN_TRACE=n records the n-th SUMI launch (clock64 per CTA)
  static int trace_at = [] { const char* t = getenv("CLIMBER_ATTN_TRACE"); return t ? atoi(t) : -1; }();
  static int n_launch = 0;
  unsigned long long* tbuf = nullptr;
  const long long n_cta = (long long)grid.x * grid.y * grid.z;
  if (trace_at >= 0 && n_launch++ == trace_at) {
    cudaMallocManaged(&tbuf, n_cta * at::TRACE_N * 8);
    cudaMemset(tbuf, 0, n_cta * at::TRACE_N * 8);
    a.trace = tbuf;
  }
  if (D.dh == 64) at::launch<64, at::MODE_SUMI>(mq, mkv, a, grid, s);
  else at::launch<32, at::MODE_SUMI>(mq, mkv, a, grid, s);
  if (tbuf) {
    cudaStreamSynchronize(s);
    double acc[at::TRACE_N] = {0};
    long long cnt = 0;
    for (long long c = 0; c < n_cta; ++c) {
      unsigned long long* t = tbuf + c * at::TRACE_N;
      if (!t[0] || !t[22]) continue;
      ++cnt;
      for (int i = 1; i < at::TRACE_N; ++i)
        if (t[i]) acc[i] += (double)(long long)(t[i] - t[0]);
    }
    fprintf(stderr, "[attn trace] %lld CTAs; mean cycles since start: prologue %.0f init %.0f", cnt, acc[1] / cnt,
            acc[2] / cnt);
    for (int j = 0; j < 9; ++j)
      if (acc[3 + 2 * j] > 0) fprintf(stderr, " | c%d S %.0f P %.0f", j, acc[3 + 2 * j] / cnt, acc[4 + 2 * j] / cnt);
    fprintf(stderr, " | o_done %.0f staged %.0f end %.0f\n", acc[21] / cnt, acc[23] / cnt, acc[22] / cnt);
    fprintf(stderr, "[attn trace] MMA p_full(j) seen: %.0f %.0f %.0f %.0f %.0f %.0f %.0f %.0f\n",
            acc[24] / cnt, acc[25] / cnt, acc[26] / cnt, acc[27] / cnt, acc[28] / cnt, acc[29] / cnt, acc[30] / cnt,
            acc[31] / cnt);
    fprintf(stderr, "[attn trace] QK issue:");
    for (int j = 0; j < 8; ++j) fprintf(stderr, " %.0f", acc[32 + j] / cnt);
    fprintf(stderr, "\n");
    cudaFree(tbuf);
  }
}

void launch_attn_hist_tc(const bf16* Q, const int* wave_slot, const int* wave_r, int U, const bf16* pool,
                         long long pool_rows, const int* ptab, const int* vlen_all, const float* tau, bf16* O, int k,
                         int l, const Dims& D, cudaStream_t s, int nbk) {
  if (!D.bpos && use_fa() && attn_fa_supported(D.dh, D.nk)) {
    launch_attn_hist_fa(Q, wave_slot, wave_r, U, pool, pool_rows, ptab, vlen_all, tau, O, k, l, D, s, nbk);
    return;
  }
  CUtensorMap mq, mkv;
  if (!at::map2d(&mq, Q, (long long)U * D.nk * nbk, D.d, D.d, D.dh, at::ROWS) ||
      !at::map2d(&mkv, pool, pool_rows, D.d, D.d, D.dh, at::KEYS)) {
    note_launch_error("history attention: cuTensorMapEncodeTiled rejected a map (kernel not launched)");
    return;
  }
  at::Args a{Q, nullptr, wave_slot, wave_r, ptab, vlen_all, tau, O, k, l, U, (long long)U * D.nk, D, nullptr};
  dim3 grid(D.nk / at::ROWS, D.h, U * nbk);
  if (at::use_pt() && !D.bpos) {
    at::PArgs pa{a, (int)((grid.x + at::PT_WT - 1) / at::PT_WT), 0};
    pa.n_items = (long long)pa.n_pairs * D.h * U * nbk;
    if (D.dh == 64) at::launch_pt<64, at::MODE_HIST>(mq, mkv, pa, s);
    else at::launch_pt<32, at::MODE_HIST>(mq, mkv, pa, s);
    return;
  }
  if (D.dh == 64) at::launch<64, at::MODE_HIST>(mq, mkv, a, grid, s);
  else at::launch<32, at::MODE_HIST>(mq, mkv, a, grid, s);
}

}  // namespace climber
