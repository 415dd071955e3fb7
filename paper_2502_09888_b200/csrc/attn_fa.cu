// tcgen05/TMEM flash attention for the bf16 path (Eq. 3 with f_b = 0;
// SUMI masks P:L255): softmax(q.k / (sqrt(d_h) tau)) v.
//
//   MODE_SUMI: a tile of 128 candidates of one (user, block, head) attends to
//              the v cached history keys of its (block, layer) plus itself.
//   MODE_HIST: 128 history rows of one (user, block, head) attend keys j <= t
//              (causal) or j < v (bidirectional).
//
// CTA = 8 warps, one 128-row query tile (TMEM lane = query row), keys in
// chunks of 128 (two 64-token pages); two CTAs per SM, so one CTA's prologue
// (q tiles) and epilogue overlap the other's chunks.
//   warp 0      K producer (TMA): q (+ SUMI k_self, v_self, parked in the last
//               K / V stages until the self term is read) and chunk 0's K and V
//               at once, then K of each further chunk into a three-stage ring,
//               freed as soon as its Q K^T completes
//   warp 3      V producer: V of each chunk into a two-stage ring, freed when
//               its P V completes (K runs ahead of V: Q K_{j+1}^T is needed
//               before P(j) V_j)
//   warp 1      MMA issuer (one thread): S(j+1) = Q K_{j+1}^T (M=128, N=128,
//               K=d_h) as soon as the softmax has loaded S(j) into registers,
//               so it runs under the exponentials of chunk j; O += P(j) V_j
//               (M=128, N=d_h, K=128; P read from TMEM, V an MN-major smem
//               operand) once P(j) is written
//   warp 2      TMEM allocator (256 columns: S [0,128), P [128,192) (bf16
//               pairs), O [192, 192+d_h))
//   warps 4-7   softmax, one thread per query row, the whole 128-key S row in
//               registers: row max, lazy online rescale (O is rescaled only
//               when the row max grows by > 2^8), P = 2^(s sc - m) on the MUFU,
//               packed to bf16 into TMEM, fp32 row sum with packed FADD2 (the
//               MUFU bounds it: 16 exponentials / clk / SM; an FMA-pipe
//               polynomial for part of them measured slower)
//   epilogue    O / l -> bf16, staged in the (then idle) q buffer, coalesced
//               row stores
// The SUMI self term initialises the row state (m = s_self, l = 1, O = v_self),
// so no candidate ever reads another candidate's K/V.
// BIAS = 1 adds Eq. 3's relative bias f_b^{p,t}(a_k, r) to the raw scores before
// the 1/(sqrt(d_h) tau) scaling (G6b-G6e): SUMI rows add the request's
// candidate-row bias cbias[slot][l][k][head][j] (the same for every candidate);
// history rows add b_pos[bucket_pos(t - j)] + b_time[bucket_time(age_j -
// age_t)] from tables staged in shared memory (causal: a per-offset table of
// b_pos[bucket_pos(d)] -- consecutive offsets across the lanes, no bank
// conflicts -- and the time bucket by a comparison tree).
#include <cuda.h>
#include <cudaTypedefs.h>

#include <cstdio>
#include <cstdlib>
#include <mutex>
#include <numeric>

#include "kernels.cuh"
#include "tc_util.cuh"

namespace climber {
namespace fa {
using namespace tcu;

constexpr int ROWS = 128;      // query rows per CTA (TMEM lanes)
constexpr int KEYS = 128;      // keys per chunk (two pages)
constexpr int KST = 3;         // K ring stages
constexpr int VST = 2;         // V ring stages
constexpr int THREADS = 256;
constexpr float LOG2E = 1.4426950408889634f;
constexpr float RESCALE_LOG2 = 8.0f;
enum { MODE_SUMI = 0, MODE_HIST = 1 };

template <int DH>
struct Lay {
  static constexpr int RB = DH * 2;                       // bytes per q/k/v row (one swizzle atom)
  static constexpr uint32_t SWZ = (DH == 64) ? 2u : 4u;   // descriptor swizzle: 128B / 64B
  static constexpr int TILE_B = ROWS * RB;                // the q tile (also k_self, v_self)
  static constexpr int KV_B = KEYS * RB;                  // K (or V) of one chunk
  static constexpr int Q_OFF = 0;
  static constexpr int K_OFF = Q_OFF + TILE_B;            // [KST] K chunks
  static constexpr int V_OFF = K_OFF + KST * KV_B;        // [VST] V chunks
  static constexpr int BAR_OFF = V_OFF + VST * KV_B;
  static constexpr int PG_OFF = BAR_OFF + 256;            // page ids of the (user, block, layer), <= 32
  // relative bias (BIAS = 1): b_pos [128], b_time [16], (spare [64 x 7]),
  // then the (user, block)'s row of n_k <= 1024 values: SUMI the candidate-row
  // bias of this (layer, head), HIST the token ages
  static constexpr int BIAS_OFF = PG_OFF + 128;
  static constexpr int BROW_OFF = BIAS_OFF + (NB_POS + 16 + 64 * 7) * 4;
  // causal history: b_pos[bucket_pos(d)] for offsets d in [-127, n_k) (float)
  static constexpr int PBT_OFF = BROW_OFF + 1024 * 4;
  static constexpr int TOTAL = PBT_OFF + (1024 + 128) * 4 + 1024;  // + 1024 B alignment slack
  // SUMI: k_self / v_self are parked in the last K and V stages until the self term is read
  static constexpr int KS_OFF = K_OFF + (KST - 1) * KV_B;
  static constexpr int VS_OFF = V_OFF + (VST - 1) * KV_B;
  static_assert(KV_B == TILE_B, "a self tile is one K (or V) stage");
  __device__ static constexpr int k_off(int j) { return K_OFF + (j % KST) * KV_B; }
  __device__ static constexpr int v_off(int j) { return V_OFF + (j % VST) * KV_B; }
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
  unsigned long long* trace;  // clock64 timeline per CTA (CLIMBER_FA_TRACE), nullptr normally
};
// trace slots per CTA: [2j] softmax saw S(j), [40 + j] its S row loaded,
// [52 + j] max / rescale done, [2j + 1] it released P(j) (j < 12); [30 / 31]
// epilogue start / end; [64 + j] MMA thread saw P(j);
// [96 + j] MMA thread saw K/V chunk j; [126] q tiles seen; [127] start
constexpr int TRACE_N = 128;

__device__ __forceinline__ float ex2_approx(float x) {
  float y;
  asm("ex2.approx.ftz.f32 %0, %1;" : "=f"(y) : "f"(x));
  return y;
}
__device__ __forceinline__ uint64_t f2_add(uint64_t a, uint64_t b) {
  uint64_t r;
  asm("add.rn.f32x2 %0, %1, %2;" : "=l"(r) : "l"(a), "l"(b));
  return r;
}
// explicit shared-space loads (the aligned smem base is a generic pointer:
// without these the compiler emits generic LD with 64-bit addresses)
__device__ __forceinline__ float lds_f32(uint32_t a) {
  float v;
  asm("ld.shared.f32 %0, [%1];" : "=f"(v) : "r"(a));
  return v;
}
__device__ __forceinline__ int4 lds_v4(uint32_t a) {
  int4 v;
  asm("ld.shared.v4.s32 {%0, %1, %2, %3}, [%4];" : "=r"(v.x), "=r"(v.y), "=r"(v.z), "=r"(v.w) : "r"(a));
  return v;
}
__device__ __forceinline__ float max3(float a, float b, float c) {
  float r;
  asm("max.f32 %0, %1, %2, %3;" : "=f"(r) : "f"(a), "f"(b), "f"(c));
  return r;
}
__device__ __forceinline__ void named_sync(int id, int n) { asm volatile("bar.sync %0, %1;" ::"r"(id), "r"(n) : "memory"); }
__device__ __forceinline__ void tmem_ld16_nw(uint32_t taddr, uint32_t* r) {
  asm volatile(
      "tcgen05.ld.sync.aligned.32x32b.x16.b32 {%0, %1, %2, %3, %4, %5, %6, %7, %8, %9, %10, %11, %12, %13, %14, "
      "%15}, [%16];"
      : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]), "=r"(r[7]), "=r"(r[8]),
        "=r"(r[9]), "=r"(r[10]), "=r"(r[11]), "=r"(r[12]), "=r"(r[13]), "=r"(r[14]), "=r"(r[15])
      : "r"(taddr));
}

// 16-byte chunk j of staged row `row` (the TMA box swizzle: 128B or 64B pattern)
template <int DH>
__device__ __forceinline__ int swz(int row, int j) {
  return (DH == 64) ? (j ^ (row & 7)) : (j ^ ((row >> 1) & 3));
}

template <int DH, int MODE, int BIAS>
__global__ void __launch_bounds__(THREADS, 2)
    k_attn_fa(const __grid_constant__ CUtensorMap tmQ, const __grid_constant__ CUtensorMap tmKV, Args a) {
  using Ly = Lay<DH>;
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  uint64_t* bars = reinterpret_cast<uint64_t*>(smem + Ly::BAR_OFF);
  uint64_t* bar_q = bars;
  uint64_t* k_full = bars + 1;                // [KST]
  uint64_t* k_empty = k_full + KST;           // [KST]
  uint64_t* v_full = k_empty + KST;           // [VST]
  uint64_t* v_empty = v_full + VST;           // [VST]
  uint64_t* s_full = v_empty + VST;           // S(j) written
  uint64_t* s_read = s_full + 1;              // S(j) loaded by the softmax (S columns free)
  uint64_t* p_full = s_read + 1;              // P(j) written
  uint64_t* pv_done = p_full + 1;             // P(j) V_j complete (P columns free, O current)
  uint64_t* self_done = pv_done + 1;          // SUMI: k_self / v_self read (their stages are free)
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(self_done + 1);
  int* spg = reinterpret_cast<int*>(smem + Ly::PG_OFF);

  const Dims& D = a.D;
  const int u = blockIdx.z % a.U, head = blockIdx.y, tile0 = blockIdx.x * ROWS;
  const int kk = blockIdx.z / a.U;
  const int kblk = a.k + kk;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int slot = a.wave_slot[u];
  const int r = a.wave_r[u];
  const int v = a.vlen_all[(long long)slot * D.Nb + kblk];
  const int* pages = a.ptab + (((long long)slot * D.Nb + kblk) * D.L + a.l) * D.ppb;
  const float sc = LOG2E / (sqrtf((float)DH) * a.tau[((a.l * D.Nb + kblk) * D.R + r) * D.h + head]);

  // tile geometry (CTA-uniform)
  int n_rows, n_out, kend;
  long long rbase;
  if (MODE == MODE_SUMI) {
    const long long p0 = a.cand_off[u], p1 = a.cand_off[u + 1];
    if (p0 + tile0 >= p1) return;
    n_rows = (int)min((long long)ROWS, p1 - p0 - tile0);
    n_out = n_rows;
    kend = v;
    rbase = kk * a.rows_pb + p0 + tile0;
  } else {
    if (tile0 >= D.nk) return;
    n_rows = max(0, min(ROWS, v - tile0));
    n_out = min(ROWS, D.nk - tile0);
    kend = D.causal ? min(v, tile0 + ROWS) : v;
    rbase = kk * a.rows_pb + (long long)u * D.nk + tile0;
  }
  const int nch = (MODE == MODE_SUMI || n_rows > 0) ? (kend + KEYS - 1) / KEYS : 0;
  const bool need_q = MODE == MODE_SUMI || nch > 0;
  const int n_pages = min(D.ppb, (nch * KEYS + PAGE - 1) / PAGE);

  if (warp == 0) {
    for (int i = lane; i < n_pages; i += 32) spg[i] = pages[i];
    if (lane == 0) {
      asm volatile("prefetch.tensormap [%0];" ::"l"(&tmQ) : "memory");
      asm volatile("prefetch.tensormap [%0];" ::"l"(&tmKV) : "memory");
      mbar_init(bar_q, 1);
      for (int s = 0; s < KST; ++s) {
        mbar_init(&k_full[s], 1);
        mbar_init(&k_empty[s], 1);
      }
      for (int s = 0; s < VST; ++s) {
        mbar_init(&v_full[s], 1);
        mbar_init(&v_empty[s], 1);
      }
      mbar_init(s_full, 1);
      mbar_init(s_read, 128);
      mbar_init(p_full, 128);
      mbar_init(pv_done, 1);
      mbar_init(self_done, 128);
      asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
      // the query-side tiles go out first: their round trip heads every CTA's critical path
      if (need_q) {
        mbar_expect_tx(bar_q, (MODE == MODE_SUMI ? 3 : 1) * Ly::TILE_B);
        tma_load_2d(smem + Ly::Q_OFF, &tmQ, bar_q, head * DH, (int)rbase);
        if (MODE == MODE_SUMI) {
          tma_load_2d(smem + Ly::KS_OFF, &tmQ, bar_q, D.d + head * DH, (int)rbase);
          tma_load_2d(smem + Ly::VS_OFF, &tmQ, bar_q, 2 * D.d + head * DH, (int)rbase);
        }
      }
      // chunk 0's K and V right behind them (stage 0 of each ring is free):
      // Q K_0^T needs both q and K_0, so they travel together
      if (nch > 0) {
        const int pa = pages[0];
        const int pb = n_pages > 1 ? pages[1] : pa;
        mbar_expect_tx(&k_full[0], Ly::KV_B);
        tma_load_2d(smem + Ly::k_off(0), &tmKV, &k_full[0], head * DH, (int)page_row(pa, 0, 0));
        tma_load_2d(smem + Ly::k_off(0) + PAGE * Ly::RB, &tmKV, &k_full[0], head * DH, (int)page_row(pb, 0, 0));
        mbar_expect_tx(&v_full[0], Ly::KV_B);
        tma_load_2d(smem + Ly::v_off(0), &tmKV, &v_full[0], head * DH, (int)page_row(pa, 1, 0));
        tma_load_2d(smem + Ly::v_off(0) + PAGE * Ly::RB, &tmKV, &v_full[0], head * DH, (int)page_row(pb, 1, 0));
      }
    }
  } else if (warp == 2) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(smem_u32(tmem_slot)),
                 "r"(256));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  fence_before();
  __syncthreads();
  fence_after();
  const uint32_t tmem_base = *tmem_slot;
  const uint32_t tS = tmem_base;                 // S(j)
  const uint32_t tP = tmem_base + KEYS;          // P(j), bf16 pairs
  const uint32_t tO = tmem_base + KEYS + KEYS / 2;  // O [DH]
  unsigned long long* tr = a.trace ? a.trace + ((long long)(blockIdx.z * gridDim.y + blockIdx.y) * gridDim.x +
                                                blockIdx.x) * TRACE_N
                                   : nullptr;
  if (tr && threadIdx.x == 0) tr[127] = clock64();

  if (warp < 4) {
    // the control warpgroup hands registers to the softmax warpgroup (whole S
    // rows live in registers): 128 x 64 + 128 x 192 = 256 x 128
    asm volatile("setmaxnreg.dec.sync.aligned.u32 64;");
    if ((warp == 0 || warp == 3) && lane == 0) {
      // ---------------- TMA producers: K (warp 0) and V (warp 3) of chunk j, two pages each ----------------
      const bool is_k = warp == 0;
      const int nst = is_k ? KST : VST;
      uint64_t* full = is_k ? k_full : v_full;
      uint64_t* empty = is_k ? k_empty : v_empty;
      const int kv = is_k ? 0 : 1;
      for (int j = 1; j < nch; ++j) {  // chunk 0 was issued with the q tiles
        const int st = j % nst;
        mbar_wait(&empty[st], ((j / nst) & 1) ^ 1);
        if (MODE == MODE_SUMI && j == nst - 1) mbar_wait(self_done, 0);  // the last stage held a self tile
        const int pa = spg[2 * j];
        const int pb = (2 * j + 1 < n_pages) ? spg[2 * j + 1] : pa;  // past the pages: finite, masked keys
        mbar_expect_tx(&full[st], Ly::KV_B);
        uint8_t* dst = smem + (is_k ? Ly::k_off(j) : Ly::v_off(j));
        tma_load_2d(dst, &tmKV, &full[st], head * DH, (int)page_row(pa, kv, 0));
        tma_load_2d(dst + PAGE * Ly::RB, &tmKV, &full[st], head * DH, (int)page_row(pb, kv, 0));
      }
    } else if (warp == 1 && lane == 0 && nch > 0) {
      // ---------------- MMA issuer ----------------
      constexpr uint32_t idesc_qk = idesc_bf16_major(ROWS, KEYS, 0, 0);
      constexpr uint32_t idesc_pv = idesc_bf16_major(ROWS, DH, 0, 1);
      const uint64_t qd = make_sdesc(smem_u32(smem + Ly::Q_OFF), 16, 8 * Ly::RB, Ly::SWZ);
      auto qk = [&](int j) {
        mbar_wait(&k_full[j % KST], (j / KST) & 1);
        fence_after();
        if (tr && j < 16) tr[96 + j] = clock64();
        const uint64_t kd = make_sdesc(smem_u32(smem + Ly::k_off(j)), 16, 8 * Ly::RB, Ly::SWZ);
#pragma unroll
        for (int s = 0; s < DH / 16; ++s) mma_bf16(tS, qd + 2 * s, kd + 2 * s, idesc_qk, s > 0 ? 1u : 0u);
        mma_commit(&k_empty[j % KST]);
        mma_commit(s_full);
      };
      mbar_wait(bar_q, 0);
      qk(0);
      for (int j = 0; j < nch; ++j) {
        if (j + 1 < nch) {  // S(j+1) as soon as S(j) is in the softmax's registers
          mbar_wait(s_read, j & 1);
          fence_after();
          qk(j + 1);
        }
        mbar_wait(p_full, j & 1);
        fence_after();
        if (tr && j < 12) tr[64 + j] = clock64();
        mbar_wait(&v_full[j % VST], (j / VST) & 1);
        fence_after();
        const uint64_t vd = make_sdesc(smem_u32(smem + Ly::v_off(j)), 16, 8 * Ly::RB, Ly::SWZ);
#pragma unroll 1
        for (int s = 0; s < KEYS / 16; ++s) {
          const uint64_t vds = vd + (uint64_t)((16 * Ly::RB) >> 4) * s;  // 16 keys = 2 groups of 8 rows
          const uint32_t acc = (MODE == MODE_SUMI || j > 0 || s > 0) ? 1u : 0u;
          mma_bf16_ts(tO, tP + 8 * s, vds, idesc_pv, acc);  // 16 keys of P = 8 packed columns
        }
        mma_commit(&v_empty[j % VST]);
        mma_commit(pv_done);
      }
    }
  } else {
    asm volatile("setmaxnreg.inc.sync.aligned.u32 192;");
    // ---------------- softmax + epilogue ----------------
    const int ew = warp & 3;            // TMEM lane quadrant of this warp
    const int row = ew * 32 + lane;     // query row = TMEM lane
    const uint32_t lane_off = (uint32_t)(ew * 32) << 16;
    const bool valid = row < n_rows;
    const int t_row = tile0 + row;      // HIST: this row's position in the subsequence
    float m_used = -INFINITY, l = 0.f;
    // relative bias (BIAS = 1): this (layer, block, scenario, head)'s tables in smem
    float* sbp = reinterpret_cast<float*>(smem + Ly::BIAS_OFF);
    float* sbt = sbp + NB_POS;
    const int* hag = nullptr;
    const float* cbr = nullptr;
    int t_age = 0;
    if constexpr (BIAS) {
      const long long br = bias_row(D, a.l, kblk, r, head);
      sbp[row] = D.bpos[br * NB_POS + row];
      if (row < NB_TIME) sbt[row] = D.btime[br * NB_TIME + row];
      // the (user, block)'s row (ages or candidate-row bias) in smem: the
      // per-chunk reads are broadcast shared loads off the critical path
      const int* gag = D.hage + ((long long)slot * D.Nb + kblk) * D.nk;
      const float* gcb = D.cbias + ((((long long)slot * D.L + a.l) * D.Nb + kblk) * D.h + head) * D.nk;
      int* srow = reinterpret_cast<int*>(smem + Ly::BROW_OFF);
      for (int i = row; i < D.nk; i += 128)
        srow[i] = MODE == MODE_SUMI ? __float_as_int(gcb[i]) : gag[i];
      if (MODE == MODE_HIST && D.causal) {  // offset -> its position bias, offsets -127 .. n_k - 1
        float* pbt = reinterpret_cast<float*>(smem + Ly::PBT_OFF);
        const long long br = bias_row(D, a.l, kblk, r, head);
        for (int i = row; i < D.nk + 127; i += 128) pbt[i] = i >= 127 ? D.bpos[br * NB_POS + bucket_pos(i - 127)] : 0.f;
      }
      named_sync(1, 128);
      hag = srow;
      cbr = reinterpret_cast<const float*>(srow);
      if (MODE == MODE_HIST && t_row < v) t_age = hag[t_row];
    }
    unsigned long long* trs = (tr && threadIdx.x == 128) ? tr : nullptr;
    if (MODE == MODE_SUMI) {
      // self term from the TMA-loaded q / k_self / v_self tiles (16-byte chunks
      // XOR-swizzled like the TMA box)
      mbar_wait(bar_q, 0);
      if (trs) trs[126] = clock64();
      // explicit shared loads, all issued before the arithmetic; 8 partial
      // sums break the dot product's dependence chain
      const uint32_t qrow = smem_u32(smem + Ly::Q_OFF) + row * Ly::RB;
      const uint32_t krow = smem_u32(smem + Ly::KS_OFF) + row * Ly::RB;
      const uint32_t vrow = smem_u32(smem + Ly::VS_OFF) + row * Ly::RB;
      int4 qv[DH / 8], kv[DH / 8];
#pragma unroll
      for (int j = 0; j < DH / 8; ++j) {
        qv[j] = lds_v4(qrow + (swz<DH>(row, j) << 4));
        kv[j] = lds_v4(krow + (swz<DH>(row, j) << 4));
      }
      float ps[8] = {0.f, 0.f, 0.f, 0.f, 0.f, 0.f, 0.f, 0.f};
#pragma unroll
      for (int j = 0; j < DH / 8; ++j) {
        const bf16* qb = reinterpret_cast<const bf16*>(&qv[j]);
        const bf16* kb = reinterpret_cast<const bf16*>(&kv[j]);
#pragma unroll
        for (int i = 0; i < 8; ++i) ps[i] = fmaf(__bfloat162float(qb[i]), __bfloat162float(kb[i]), ps[i]);
      }
      float ss = ((ps[0] + ps[1]) + (ps[2] + ps[3])) + ((ps[4] + ps[5]) + (ps[6] + ps[7]));
      if constexpr (BIAS) ss += sbp[bucket_pos(0)] + sbt[bucket_time32(0)];  // self: offset 0, delta 0
      m_used = valid ? ss * sc : 0.f;
#pragma unroll
      for (int c = 0; c < DH; c += 32) {  // O = v_self
        float vs[32];
#pragma unroll
        for (int cc = 0; cc < 32; cc += 8) {
          const int4 vv = lds_v4(vrow + (swz<DH>(row, (c + cc) / 8) << 4));
          const bf16* vb = reinterpret_cast<const bf16*>(&vv);
#pragma unroll
          for (int i = 0; i < 8; ++i) vs[cc + i] = valid ? __bfloat162float(vb[i]) : 0.f;
        }
        tmem_st32_nw(tO + lane_off + c, vs);  // waited before P(0) is released (or before a rescale)
      }
      l = 1.f;  // the self term's weight
      // the self tiles' stages become K / V stages
      asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
      mbar_arrive(self_done);
    }
    const bool causal_hist = (MODE == MODE_HIST) && D.causal;
    for (int j = 0; j < nch; ++j) {
      mbar_wait(s_full, j & 1);
      fence_after();
      if (trs && j < 12) trs[2 * j] = clock64();
      const int key0 = j * KEYS;
      int lim = kend - key0;  // keys [0, lim) of the chunk are visible to this row
      if (causal_hist) lim = min(lim, t_row - key0 + 1);
      uint32_t sr[KEYS];
#pragma unroll
      for (int c = 0; c < KEYS; c += 32) tmem_ld32_nw(tS + lane_off + c, sr + c);
      tmem_ld_wait();
      fence_before();
      mbar_arrive(s_read);  // the S columns may take S(j+1)
      if (trs && j < 12) trs[40 + j] = clock64();
      if constexpr (BIAS) {  // R = QK^T + f_b (before the 1/(sqrt(d_h) tau) scaling, Eq. 3)
        if (MODE == MODE_SUMI) {
          const uint32_t c4 = smem_u32(cbr + key0);
#pragma unroll
          for (int i = 0; i < KEYS; i += 4) {
            int4 bi = make_int4(0, 0, 0, 0);
            if (key0 + i < D.nk) bi = lds_v4(c4 + 4u * i);
            const float4 b = make_float4(__int_as_float(bi.x), __int_as_float(bi.y), __int_as_float(bi.z),
                                         __int_as_float(bi.w));
            const float2 s01 = f2_unpack(f2_add(f2_pack(__uint_as_float(sr[i]), __uint_as_float(sr[i + 1])),
                                                f2_pack(b.x, b.y)));
            const float2 s23 = f2_unpack(f2_add(f2_pack(__uint_as_float(sr[i + 2]), __uint_as_float(sr[i + 3])),
                                                f2_pack(b.z, b.w)));
            sr[i] = __float_as_uint(s01.x);
            sr[i + 1] = __float_as_uint(s01.y);
            sr[i + 2] = __float_as_uint(s23.x);
            sr[i + 3] = __float_as_uint(s23.y);
          }
        } else {
          // t_row - t_key = age_key - age_row; key ages 4 per 16-byte load.
          // The mask mode is hoisted out of the element loops: a branch per
          // score serialises the shared loads (measured 35k cycles / chunk)
          const int4* a4 = reinterpret_cast<const int4*>(hag + key0);
          if (D.causal) {
            // offsets >= 0 and time deltas >= 0 on every visible key: the
            // position bias from the per-offset table (the offset t - j >=
            // -127 inside a causal tile's chunks; consecutive offsets across
            // the lanes: no bank conflicts), the time bucket by a 3-level
            // comparison tree (the edges of S:L285), <= 7 time entries
            const uint32_t pbt = smem_u32(smem + Ly::PBT_OFF) + 4u * (127 + t_row - key0);
            const uint32_t sag = smem_u32(hag + key0), sbt_a = smem_u32(sbt);
#pragma unroll
            for (int i = 0; i < KEYS; i += 4) {
              const int4 ka = (key0 + i < D.nk) ? lds_v4(sag + 4u * i) : make_int4(0, 0, 0, 0);
              const int kv4[4] = {ka.x, ka.y, ka.z, ka.w};
#pragma unroll
              for (int q = 0; q < 4; ++q) {
                const int dt = kv4[q] - t_age;  // >= 0 on visible keys: branch-free bucket count
                const int bt = (dt > 0) + (dt >= 60) + (dt >= 3600) + (dt >= 86400) + (dt >= 604800) +
                               (dt >= 2592000);
                const float b = lds_f32(pbt - 4u * (i + q)) + lds_f32(sbt_a + 4u * bt);
                sr[i + q] = __float_as_uint(__uint_as_float(sr[i + q]) + b);
              }
            }
          } else {
#pragma unroll
            for (int i = 0; i < KEYS; i += 4) {
              const int4 ka = (key0 + i < D.nk) ? a4[i >> 2] : make_int4(0, 0, 0, 0);
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
      if (lim < KEYS) {  // masked keys -> -inf (2^-inf = +0)
#pragma unroll
        for (int i = 0; i < KEYS; ++i)
          if (i >= lim) sr[i] = __float_as_uint(-INFINITY);
      }
      float mx8[8];
#pragma unroll
      for (int i = 0; i < 8; ++i) mx8[i] = -INFINITY;
#pragma unroll
      for (int i = 0; i < KEYS; i += 2)
        mx8[(i >> 1) & 7] = max3(mx8[(i >> 1) & 7], __uint_as_float(sr[i]), __uint_as_float(sr[i + 1]));
      const float mraw = fmaxf(fmaxf(fmaxf(mx8[0], mx8[1]), fmaxf(mx8[2], mx8[3])),
                               fmaxf(fmaxf(mx8[4], mx8[5]), fmaxf(mx8[6], mx8[7])));
      const float mx = mraw * sc;  // sc > 0
      // lazy rescale: per row, only when its max grew by > 2^8; tcgen05.ld/st
      // are warp-collective, so the warp decides together.  s_full(j) implies
      // P(j-1) V_{j-1} is complete (the MMAs of one thread complete in order).
      const bool mine = mx > m_used + RESCALE_LOG2;
      const float alpha = mine ? exp2f(m_used - mx) : 1.f;  // m_used = -inf -> 0
      if (mine) {
        l *= alpha;
        m_used = mx;
      }
      // P(j-1) V_{j-1} must be complete before O is rescaled or P(j) written
      const bool need_pv = j > 0;
      bool pv_seen = false;
      if ((MODE == MODE_SUMI || j > 0) && __any_sync(0xffffffffu, mine)) {
        if (MODE == MODE_SUMI && j == 0) tmem_st_wait();  // the O = v_self stores
        if (need_pv) {
          mbar_wait(pv_done, (j - 1) & 1);
          fence_after();
          pv_seen = true;
        }
#pragma unroll
        for (int c = 0; c < DH; c += 16) {  // 16 columns at a time
          uint32_t o[16];
          tmem_ld16_nw(tO + lane_off + c, o);
          tmem_ld_wait();
#pragma unroll
          for (int i = 0; i < 16; ++i) o[i] = __float_as_uint(__uint_as_float(o[i]) * alpha);
          tmem_st16u(tO + lane_off + c, o);
        }
      }
      if (trs && j < 12) trs[52 + j] = clock64();
      // P = 2^(s sc - m) (fp32), packed to bf16 into S's first 64 columns
      const float nb = (m_used == -INFINITY) ? 0.f : -m_used;
      const uint64_t sc2 = f2_pack(sc, sc), nb2 = f2_pack(nb, nb);
      uint64_t ls2[4] = {0ull, 0ull, 0ull, 0ull};  // packed (0.f, 0.f)
#pragma unroll
      for (int c = 0; c < KEYS; c += 32) {
        uint32_t pk[16];
#pragma unroll
        for (int i = 0; i < 32; i += 2) {
          const float2 x = f2_unpack(f2_fma(f2_pack(__uint_as_float(sr[c + i]), __uint_as_float(sr[c + i + 1])),
                                            sc2, nb2));
          const float e0 = ex2_approx(x.x);
          const float e1 = ex2_approx(x.y);
          ls2[(i >> 1) & 3] = f2_add(ls2[(i >> 1) & 3], f2_pack(e0, e1));
          __nv_bfloat162 pp = __floats2bfloat162_rn(e0, e1);
          pk[i >> 1] = *reinterpret_cast<uint32_t*>(&pp);
        }
        if (c == 0 && need_pv && !pv_seen) {
          mbar_wait(pv_done, (j - 1) & 1);
          fence_after();
        }
        tmem_st16u(tP + lane_off + c / 2, pk);
      }
      {
        const float2 a0 = f2_unpack(f2_add(ls2[0], ls2[1])), a1 = f2_unpack(f2_add(ls2[2], ls2[3]));
        l += (a0.x + a0.y) + (a1.x + a1.y);
      }
      tmem_st_wait();
      fence_before();
      mbar_arrive(p_full);
      if (trs && j < 12) trs[2 * j + 1] = clock64();
    }
    if (trs) trs[30] = clock64();
    // ---- epilogue: O / l -> bf16, staged in the q buffer (every MMA has
    // completed once the last pv_done fires), coalesced row stores
    if (nch > 0) {
      mbar_wait(pv_done, (nch - 1) & 1);
      fence_after();
    }
    if (trs) trs[27] = clock64();
    const bool have_o = MODE == MODE_SUMI || nch > 0;
    const float inv = (valid && l > 0.f) ? 1.f / l : 0.f;
    uint8_t* qtile = smem + Ly::Q_OFF;
#pragma unroll
    for (int c = 0; c < DH; c += 32) {
      float o[32];
      if (have_o) {
        tmem_ld32(tO + lane_off + c, o);
      } else {
#pragma unroll
        for (int i = 0; i < 32; ++i) o[i] = 0.f;
      }
#pragma unroll
      for (int cc = 0; cc < 32; cc += 8) {
        uint32_t w[4];
#pragma unroll
        for (int i = 0; i < 4; ++i) {
          __nv_bfloat162 pp = __floats2bfloat162_rn(o[cc + 2 * i] * inv, o[cc + 2 * i + 1] * inv);
          w[i] = *reinterpret_cast<uint32_t*>(&pp);
        }
        st_shared_v4(qtile + row * Ly::RB + (swz<DH>(row, (c + cc) / 8) << 4), w[0], w[1], w[2], w[3]);
      }
    }
    if (trs) trs[28] = clock64();
    named_sync(1, 128);
    if (trs) trs[29] = clock64();
    constexpr int LPR = DH / 8;      // lanes per row, 16 B (8 bf16) each
    constexpr int RPI = 32 / LPR;    // rows per warp instruction
#pragma unroll
    for (int i = 0; i < 32; i += RPI) {
      const int rr = ew * 32 + i + lane / LPR;
      const int cj = lane % LPR;
      if (rr < n_out) {
        const int4 val = lds_v4(smem_u32(qtile) + rr * Ly::RB + (swz<DH>(rr, cj) << 4));
        *reinterpret_cast<int4*>(a.O + (rbase + rr) * D.d + head * DH + cj * 8) = val;
      }
    }
    if (trs) trs[31] = clock64();
  }
  fence_before();
  __syncthreads();
  if (warp == 2) {
    fence_after();
    asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem_base), "r"(256));
  }
}

// ===========================================================================
// Persistent variant (BIAS = 0): the grid is two CTAs per SM and each CTA
// walks the tiles t = blockIdx.x, blockIdx.x + gridDim.x, ... in the same
// (x, head, user x block) order as the one-tile kernel above.  Per CTA the
// chunk pipeline never drains between tiles:
//   * q tiles are double-buffered; the producer loads tile i+1's q while
//     tile i runs;
//   * the MMA issuer issues S(0) of tile i+1 = Q_{i+1} K_0^T right behind
//     tile i's last P V, so it runs under tile i's epilogue;
//   * the softmax warpgroup goes from P(last) of tile i through its epilogue
//     (SUMI: the self term merged into the row state, k_self / v_self rows
//     loaded from global memory under the last P V; O / l staged in tile i's
//     q buffer, TMA stores of full 32-row boxes) straight into S(0) of tile
//     i+1.
// The producer (warp 0) computes each tile's geometry once and hands it to
// the other roles in a descriptor next to the q buffer it fills (published by
// the q_full barrier; the softmax's q_empty arrival after the epilogue frees
// both).  Shared memory: 2 q + 3 K + 2 V tiles of 128 rows x 128 B (d_h 64)
// + 1 KB of barriers / descriptors = 115712 B, exactly half of an SM's
// 228 KB less the 1 KB each CTA reserves; the dynamic window starts 1024 B
// aligned (checked at run time).
// ===========================================================================
struct PDesc {
  int done, nch, n_rows, n_out, kend, tile0, head, n_pages;
  long long rbase;
  float sc;
  int pad;
  int pages[32];
};
static_assert(sizeof(PDesc) <= 256, "descriptor slot");

template <int DH>
struct PLay {
  static constexpr int RB = DH * 2;
  static constexpr uint32_t SWZ = (DH == 64) ? 2u : 4u;
  static constexpr int TILE_B = ROWS * RB;
#ifdef FA_LAYOUT_KFIRST  // determinism stress layout (tools/micro/race_variants.sh)
  static constexpr int K_OFF = 0;
  static constexpr int V_OFF = K_OFF + KST * TILE_B;
  static constexpr int Q_OFF = V_OFF + VST * TILE_B;
  static constexpr int BAR_OFF = Q_OFF + 2 * TILE_B;
#else
  static constexpr int Q_OFF = 0;                          // [2] q tiles, then O staging
  static constexpr int K_OFF = Q_OFF + 2 * TILE_B;         // [KST] K ring
  static constexpr int V_OFF = K_OFF + KST * TILE_B;       // [VST] V ring
  static constexpr int BAR_OFF = V_OFF + VST * TILE_B;     // barriers (<= 256 B)
#endif
  static constexpr int DESC_OFF = BAR_OFF + 256;           // [2] tile descriptors
  static constexpr int TOTAL = DESC_OFF + 768;
  __device__ static constexpr int q_off(int b) { return Q_OFF + b * TILE_B; }
  __device__ static constexpr int k_off(int i) { return K_OFF + (i % KST) * TILE_B; }
  __device__ static constexpr int v_off(int i) { return V_OFF + (i % VST) * TILE_B; }
};

template <int DH, int MODE>
__global__ void __launch_bounds__(THREADS, 2)
    k_attn_pers(const __grid_constant__ CUtensorMap tmQ, const __grid_constant__ CUtensorMap tmKV,
                const __grid_constant__ CUtensorMap tmO, Args a, int ntx, int n_tiles) {
  using Ly = PLay<DH>;
  constexpr bool SUMI = MODE == MODE_SUMI;
  // SUMI k_self / v_self are not ring items: each row's self term is merged
  // into its online-softmax state in the epilogue (k_self / v_self rows read
  // from global memory under the last P V), so both modes run the same chunk
  // pipeline.  (A first version carried them through the K / V rings as
  // items released by the softmax warps; it was not bitwise reproducible,
  // DESIGN.md §6.)
  extern __shared__ __align__(1024) uint8_t smem[];
  {
    uint32_t dyn;
    asm("mov.u32 %0, %%dynamic_smem_size;" : "=r"(dyn));
    if ((smem_u32(smem) & 1023u) != 0u || dyn < (uint32_t)Ly::TOTAL) __trap();
  }
  uint64_t* bars = reinterpret_cast<uint64_t*>(smem + Ly::BAR_OFF);
  uint64_t* q_full = bars;                    // [2]
  uint64_t* q_empty = q_full + 2;             // [2]
  uint64_t* k_full = q_empty + 2;             // [KST]
  uint64_t* k_empty = k_full + KST;           // [KST]
  uint64_t* v_full = k_empty + KST;           // [VST]
  uint64_t* v_empty = v_full + VST;           // [VST]
  uint64_t* s_full = v_empty + VST;
  uint64_t* s_read = s_full + 1;
  uint64_t* p_full = s_read + 1;
  uint64_t* pv_done = p_full + 1;
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(pv_done + 1);
  static_assert((2 + 2 + 2 * KST + 2 * VST + 4) * 8 + 4 <= 256, "barrier area");
  PDesc* desc = reinterpret_cast<PDesc*>(smem + Ly::DESC_OFF);

  const Dims& D = a.D;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  if (warp == 0 && lane == 0) {
    asm volatile("prefetch.tensormap [%0];" ::"l"(&tmQ) : "memory");
    asm volatile("prefetch.tensormap [%0];" ::"l"(&tmKV) : "memory");
    for (int b = 0; b < 2; ++b) {
      mbar_init(&q_full[b], 1);
      mbar_init(&q_empty[b], 4);  // one arrival per softmax warp
    }
    for (int s = 0; s < KST; ++s) {
      mbar_init(&k_full[s], 1);
      mbar_init(&k_empty[s], 1);
    }
    for (int s = 0; s < VST; ++s) {
      mbar_init(&v_full[s], 1);
      mbar_init(&v_empty[s], 1);
    }
    mbar_init(s_full, 1);
    mbar_init(s_read, 128);
    mbar_init(p_full, 128);
    mbar_init(pv_done, 1);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  } else if (warp == 2) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(smem_u32(tmem_slot)),
                 "r"(256));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  fence_before();
  __syncthreads();
  fence_after();
  const uint32_t tmem_base = *tmem_slot;
  const uint32_t tS = tmem_base;
  const uint32_t tP = tmem_base + KEYS;
  const uint32_t tO = tmem_base + KEYS + KEYS / 2;
  // clock64 timeline of the first tiles of each CTA (CLIMBER_FA_TRACE), see ptrace_print
  unsigned long long* tr = a.trace ? a.trace + (long long)blockIdx.x * TRACE_N : nullptr;
  if (tr && threadIdx.x == 0) tr[127] = clock64();

  if (warp < 4) {
    asm volatile("setmaxnreg.dec.sync.aligned.u32 64;");
    if (warp == 0) {
      // ---------------- q + K producer: tile geometry, q, K chunks ----------------
      int it = 0, kc = 0;
      for (int t = blockIdx.x;; t += gridDim.x) {
        const bool done = t >= n_tiles;
        int head = 0, nch = 0, n_rows = 0, n_out = 0, kend = 0, tile0 = 0, n_pages = 0, pg = 0;
        long long rbase = 0;
        float sc = 0.f;
        if (!done) {
          const int x = t % ntx;
          head = (t / ntx) % D.h;
          const int z = t / (ntx * D.h);
          const int u = z % a.U, kk = z / a.U, kblk = a.k + kk;
          tile0 = x * ROWS;
          const int slot = a.wave_slot[u];
          const int v = a.vlen_all[(long long)slot * D.Nb + kblk];
          if (SUMI) {
            const long long p0 = a.cand_off[u], p1 = a.cand_off[u + 1];
            if (p0 + tile0 >= p1) continue;  // no candidates in this tile: no role ever sees it
            n_rows = (int)min((long long)ROWS, p1 - p0 - tile0);
            n_out = n_rows;
            kend = v;
            rbase = kk * a.rows_pb + p0 + tile0;
          } else {
            n_rows = max(0, min(ROWS, v - tile0));
            n_out = min(ROWS, D.nk - tile0);
            kend = D.causal ? min(v, tile0 + ROWS) : v;
            rbase = kk * a.rows_pb + (long long)u * D.nk + tile0;
          }
          nch = (SUMI || n_rows > 0) ? (kend + KEYS - 1) / KEYS : 0;
          n_pages = min(D.ppb, (nch * KEYS + PAGE - 1) / PAGE);
          const int* pages = a.ptab + (((long long)slot * D.Nb + kblk) * D.L + a.l) * D.ppb;
          pg = lane < n_pages ? pages[lane] : 0;
          sc = LOG2E / (sqrtf((float)DH) * a.tau[((a.l * D.Nb + kblk) * D.R + a.wave_r[u]) * D.h + head]);
        }
        const int b = it & 1;
        mbar_wait(&q_empty[b], ((it >> 1) & 1) ^ 1);
        PDesc* ds = desc + b;
        for (int i = 0; i < n_pages; ++i) {
          const int p = __shfl_sync(0xffffffffu, pg, i);
          if (lane == 0) ds->pages[i] = p;
        }
        if (lane == 0) {
          ds->done = done;
          ds->nch = nch;
          ds->n_rows = n_rows;
          ds->n_out = n_out;
          ds->kend = kend;
          ds->tile0 = tile0;
          ds->head = head;
          ds->n_pages = n_pages;
          ds->rbase = rbase;
          ds->sc = sc;
          if (!done && (SUMI || nch > 0)) {
            mbar_expect_tx(&q_full[b], Ly::TILE_B);
            tma_load_2d(smem + Ly::q_off(b), &tmQ, &q_full[b], head * DH, (int)rbase);
          } else {
            mbar_arrive(&q_full[b]);  // descriptor only
          }
        }
        __syncwarp();
        if (done) break;
        for (int j = 0; j < nch; ++j, ++kc) {
          const int st = kc % KST;
          const int pa = __shfl_sync(0xffffffffu, pg, (2 * j) & 31);
          const int pb0 = __shfl_sync(0xffffffffu, pg, (2 * j + 1) & 31);
          const int pb = (2 * j + 1 < n_pages) ? pb0 : pa;  // past the pages: finite, masked keys
          mbar_wait(&k_empty[st], ((kc / KST) & 1) ^ 1);
          if (lane == 0) {
            mbar_expect_tx(&k_full[st], Ly::TILE_B);
            tma_load_2d(smem + Ly::k_off(kc), &tmKV, &k_full[st], head * DH, (int)page_row(pa, 0, 0));
            tma_load_2d(smem + Ly::k_off(kc) + PAGE * Ly::RB, &tmKV, &k_full[st], head * DH,
                        (int)page_row(pb, 0, 0));
          }
        }
        ++it;
      }
    } else if (warp == 3) {
      // ---------------- V producer: V chunks; geometry from the descriptors ----------------
      int it = 0, vc = 0;
      for (;; ++it) {
        const int b = it & 1;
        mbar_wait(&q_full[b], (it >> 1) & 1);
        const PDesc* ds = desc + b;
        if (ds->done) break;
        const int nch = ds->nch, head = ds->head, n_pages = ds->n_pages;
        const int pg = lane < n_pages ? ds->pages[lane] : 0;
        for (int j = 0; j < nch; ++j, ++vc) {
          const int st = vc % VST;
          const int pa = __shfl_sync(0xffffffffu, pg, (2 * j) & 31);
          const int pb0 = __shfl_sync(0xffffffffu, pg, (2 * j + 1) & 31);
          const int pb = (2 * j + 1 < n_pages) ? pb0 : pa;
          mbar_wait(&v_empty[st], ((vc / VST) & 1) ^ 1);
          if (lane == 0) {
            mbar_expect_tx(&v_full[st], Ly::TILE_B);
            tma_load_2d(smem + Ly::v_off(vc), &tmKV, &v_full[st], head * DH, (int)page_row(pa, 1, 0));
            tma_load_2d(smem + Ly::v_off(vc) + PAGE * Ly::RB, &tmKV, &v_full[st], head * DH,
                        (int)page_row(pb, 1, 0));
          }
        }
      }
    } else if (warp == 1 && lane == 0) {
      // ---------------- MMA issuer ----------------
      constexpr uint32_t idesc_qk = idesc_bf16_major(ROWS, KEYS, 0, 0);
      constexpr uint32_t idesc_pv = idesc_bf16_major(ROWS, DH, 0, 1);
      int n_qk = 0;  // Q K^T issued so far (S(n) may be written once S(n-1) was read)
      auto qk = [&](int b, int item) {
        if (n_qk > 0) mbar_wait(s_read, (n_qk - 1) & 1);
        mbar_wait(&k_full[item % KST], (item / KST) & 1);
        fence_after();
        const uint64_t qd = make_sdesc(smem_u32(smem + Ly::q_off(b)), 16, 8 * Ly::RB, Ly::SWZ);
        const uint64_t kd = make_sdesc(smem_u32(smem + Ly::k_off(item)), 16, 8 * Ly::RB, Ly::SWZ);
#pragma unroll
        for (int s = 0; s < DH / 16; ++s) mma_bf16(tS, qd + 2 * s, kd + 2 * s, idesc_qk, s > 0 ? 1u : 0u);
        mma_commit(&k_empty[item % KST]);
        mma_commit(s_full);
        if (tr && n_qk < 16) tr[96 + n_qk] = clock64();
        ++n_qk;
      };
      int it = 0, kc = 0, n = 0;
      mbar_wait(&q_full[0], 0);
      int done = desc[0].done, nch = desc[0].nch;
      bool first_issued = false;
      while (!done) {
        const int b = it & 1;
        const int c0 = kc;  // ring item of chunk 0
        if (nch > 0 && !first_issued) qk(b, c0);
        int done2 = 1, nch2 = 0;
        bool peeked = false, issued2 = false;
        for (int j = 0; j < nch; ++j) {
          if (j + 1 < nch) qk(b, c0 + j + 1);  // S(j+1) under the exponentials of chunk j
          mbar_wait(p_full, n & 1);
          const int item = c0 + j;
          mbar_wait(&v_full[item % VST], (item / VST) & 1);
          fence_after();
          if (tr && n < 12) tr[112 + n] = clock64();
          const uint64_t vd = make_sdesc(smem_u32(smem + Ly::v_off(item)), 16, 8 * Ly::RB, Ly::SWZ);
#pragma unroll 1
          for (int s = 0; s < KEYS / 16; ++s) {
            const uint64_t vds = vd + (uint64_t)((16 * Ly::RB) >> 4) * s;
            const uint32_t acc = (j > 0 || s > 0) ? 1u : 0u;
            mma_bf16_ts(tO, tP + 8 * s, vds, idesc_pv, acc);
          }
          mma_commit(&v_empty[item % VST]);
          mma_commit(pv_done);
          ++n;
          if (j + 1 == nch) {
            // S(0) of the next tile right behind the last P V (which the
            // epilogue waits for), under this tile's epilogue
            const int b2 = (it + 1) & 1;
            mbar_wait(&q_full[b2], ((it + 1) >> 1) & 1);
            done2 = desc[b2].done;
            nch2 = desc[b2].nch;
            peeked = true;
            if (!done2 && nch2 > 0) {
              qk(b2, c0 + nch);
              issued2 = true;
            }
          }
        }
        if (!peeked) {
          const int b2 = (it + 1) & 1;
          mbar_wait(&q_full[b2], ((it + 1) >> 1) & 1);
          done2 = desc[b2].done;
          nch2 = desc[b2].nch;
        }
        kc = c0 + nch;
        ++it;
        done = done2;
        nch = nch2;
        first_issued = issued2;
      }
    }
  } else {
    asm volatile("setmaxnreg.inc.sync.aligned.u32 192;");
    // ---------------- softmax + epilogue ----------------
    const int ew = warp & 3;
    const int row = ew * 32 + lane;
    const uint32_t lane_off = (uint32_t)(ew * 32) << 16;
    int it = 0, kc = 0, n = 0;
    // a TMA store of the previous tile's O rows still reading this warp's
    // staging rows: lane 0 releases that q buffer once the read is done
    int rel_b = -1;
    auto release_pending = [&]() {
      if (rel_b >= 0) {
        if (lane == 0) {
          asm volatile("cp.async.bulk.wait_group.read 0;" ::: "memory");
          mbar_arrive(&q_empty[rel_b]);
        }
        rel_b = -1;
      }
    };
    for (;; ++it) {
      const int b = it & 1;
      mbar_wait(&q_full[b], (it >> 1) & 1);
      const PDesc* ds = desc + b;
      if (ds->done) break;
      unsigned long long* tt = (tr && threadIdx.x == 128 && it < 4) ? tr + it * 24 : nullptr;
      if (tt) tt[0] = clock64();
      const int nch = ds->nch, n_rows = ds->n_rows, n_out = ds->n_out, kend = ds->kend;
      const int head = ds->head;
      const long long rbase = ds->rbase;
      const float sc = ds->sc;
      const bool valid = row < n_rows;
      const int t_row = ds->tile0 + row;
      const uint32_t qbuf = smem_u32(smem + Ly::q_off(b));
      float m_used = -INFINITY, l = 0.f;
      release_pending();
      for (int j = 0; j < nch; ++j, ++n) {
        mbar_wait(s_full, n & 1);
        fence_after();
        const int key0 = j * KEYS;
        int lim = kend - key0;
        if (!SUMI && D.causal) lim = min(lim, t_row - key0 + 1);
        uint32_t sr[KEYS];
#pragma unroll
        for (int c = 0; c < KEYS; c += 32) tmem_ld32_nw(tS + lane_off + c, sr + c);
        tmem_ld_wait();
        fence_before();
        mbar_arrive(s_read);
        if (tt && j < 4) tt[2 + 2 * j] = clock64();
        if (lim < KEYS) {
#pragma unroll
          for (int i = 0; i < KEYS; ++i)
            if (i >= lim) sr[i] = __float_as_uint(-INFINITY);
        }
        float mx8[8];
#pragma unroll
        for (int i = 0; i < 8; ++i) mx8[i] = -INFINITY;
#pragma unroll
        for (int i = 0; i < KEYS; i += 2)
          mx8[(i >> 1) & 7] = max3(mx8[(i >> 1) & 7], __uint_as_float(sr[i]), __uint_as_float(sr[i + 1]));
        const float mraw = fmaxf(fmaxf(fmaxf(mx8[0], mx8[1]), fmaxf(mx8[2], mx8[3])),
                                 fmaxf(fmaxf(mx8[4], mx8[5]), fmaxf(mx8[6], mx8[7])));
        const float mx = mraw * sc;
        const bool mine = mx > m_used + RESCALE_LOG2;
        const float alpha = mine ? exp2f(m_used - mx) : 1.f;
        if (mine) {
          l *= alpha;
          m_used = mx;
        }
        const bool need_pv = j > 0;  // P(j-1) V_{j-1} of this tile (the previous tile's were waited)
        bool pv_seen = false;
        if (j > 0 && __any_sync(0xffffffffu, mine)) {
          if (need_pv) {
            mbar_wait(pv_done, (n - 1) & 1);
            fence_after();
            pv_seen = true;
          }
#pragma unroll
          for (int c = 0; c < DH; c += 16) {
            uint32_t o[16];
            tmem_ld16_nw(tO + lane_off + c, o);
            tmem_ld_wait();
#pragma unroll
            for (int i = 0; i < 16; ++i) o[i] = __float_as_uint(__uint_as_float(o[i]) * alpha);
            tmem_st16u(tO + lane_off + c, o);
          }
        }
        const float nb = (m_used == -INFINITY) ? 0.f : -m_used;
        const uint64_t sc2 = f2_pack(sc, sc), nb2 = f2_pack(nb, nb);
        uint64_t ls2[4] = {0ull, 0ull, 0ull, 0ull};
#pragma unroll
        for (int c = 0; c < KEYS; c += 32) {
          uint32_t pk[16];
#pragma unroll
          for (int i = 0; i < 32; i += 2) {
            const float2 x = f2_unpack(
                f2_fma(f2_pack(__uint_as_float(sr[c + i]), __uint_as_float(sr[c + i + 1])), sc2, nb2));
            const float e0 = ex2_approx(x.x);
            const float e1 = ex2_approx(x.y);
            ls2[(i >> 1) & 3] = f2_add(ls2[(i >> 1) & 3], f2_pack(e0, e1));
            __nv_bfloat162 pp = __floats2bfloat162_rn(e0, e1);
            pk[i >> 1] = *reinterpret_cast<uint32_t*>(&pp);
          }
          if (c == 0 && need_pv && !pv_seen) {
            mbar_wait(pv_done, (n - 1) & 1);
            fence_after();
          }
          tmem_st16u(tP + lane_off + c / 2, pk);
        }
        {
          const float2 a0 = f2_unpack(f2_add(ls2[0], ls2[1])), a1 = f2_unpack(f2_add(ls2[2], ls2[3]));
          l += (a0.x + a0.y) + (a1.x + a1.y);
        }
        tmem_st_wait();
        fence_before();
        mbar_arrive(p_full);
        if (tt && j < 4) tt[3 + 2 * j] = clock64();
      }
      // ---- SUMI self term, merged into the row's state (every
      // candidate also sees itself): x = q . k_self / (sqrt(d_h) tau) in log2
      // units, m' = max(m, x), O' = O 2^(m - m') + v_self 2^(x - m'),
      // l' = l 2^(m - m') + 2^(x - m').  k_self / v_self rows come from the
      // QKV rows in global memory, loaded while the last P V runs; q from the
      // tile's q buffer (still intact: the staging below overwrites it)
      float oa = 1.f, vb = 0.f;     // O' = O oa + v_self vb (before 1 / l')
      int4 vsv[DH / 8];
      if (SUMI) {
        int4 ksv[DH / 8];
        const bf16* krow_g = a.Q + (rbase + row) * 3LL * D.d + D.d + head * DH;
#pragma unroll
        for (int j = 0; j < DH / 8; ++j) {
          ksv[j] = valid ? __ldg(reinterpret_cast<const int4*>(krow_g) + j) : make_int4(0, 0, 0, 0);
          vsv[j] = valid ? __ldg(reinterpret_cast<const int4*>(krow_g + D.d) + j) : make_int4(0, 0, 0, 0);
        }
        const uint32_t qrow = qbuf + row * Ly::RB;
        float ps[8] = {0.f, 0.f, 0.f, 0.f, 0.f, 0.f, 0.f, 0.f};
#pragma unroll
        for (int j = 0; j < DH / 8; ++j) {
          const int4 qv = lds_v4(qrow + (swz<DH>(row, j) << 4));
          const bf16* qb = reinterpret_cast<const bf16*>(&qv);
          const bf16* kb = reinterpret_cast<const bf16*>(&ksv[j]);
#pragma unroll
          for (int i = 0; i < 8; ++i) ps[i] = fmaf(__bfloat162float(qb[i]), __bfloat162float(kb[i]), ps[i]);
        }
        const float x = (((ps[0] + ps[1]) + (ps[2] + ps[3])) + ((ps[4] + ps[5]) + (ps[6] + ps[7]))) * sc;
        const float m2 = fmaxf(m_used, x);
        oa = (m_used == -INFINITY) ? 0.f : exp2f(m_used - m2);
        vb = exp2f(x - m2);
        l = l * oa + vb;
      }
      // ---- epilogue: O / l -> bf16 staged in this tile's q buffer, coalesced row stores
      if (nch > 0) {
        mbar_wait(pv_done, (n - 1) & 1);
        fence_after();
      }
      if (tt) tt[10] = clock64();
      const bool have_o = nch > 0;
      const float inv = (valid && l > 0.f) ? 1.f / l : 0.f;
      const float oai = oa * inv, vbi = vb * inv;
#pragma unroll
      for (int c = 0; c < DH; c += 32) {
        float o[32];
        if (have_o) {
          tmem_ld32(tO + lane_off + c, o);
        } else {
#pragma unroll
          for (int i = 0; i < 32; ++i) o[i] = 0.f;
        }
        if (SUMI) {
#pragma unroll
          for (int cc = 0; cc < 32; cc += 8) {
            const bf16* vv = reinterpret_cast<const bf16*>(&vsv[(c + cc) / 8]);
#pragma unroll
            for (int i = 0; i < 8; ++i) o[cc + i] = fmaf(o[cc + i], oai, __bfloat162float(vv[i]) * vbi);
          }
        } else {
#pragma unroll
          for (int i = 0; i < 32; ++i) o[i] *= inv;
        }
#pragma unroll
        for (int cc = 0; cc < 32; cc += 8) {
          uint32_t w[4];
#pragma unroll
          for (int i = 0; i < 4; ++i) {
            __nv_bfloat162 pp = __floats2bfloat162_rn(o[cc + 2 * i], o[cc + 2 * i + 1]);
            w[i] = *reinterpret_cast<uint32_t*>(&pp);
          }
          asm volatile("st.shared.v4.b32 [%0], {%1, %2, %3, %4};" ::"r"(qbuf + row * Ly::RB +
                                                                         (swz<DH>(row, (c + cc) / 8) << 4)),
                       "r"(w[0]), "r"(w[1]), "r"(w[2]), "r"(w[3])
                       : "memory");
        }
      }
      fence_before();  // the O reads are complete before the next tile's first P V may overwrite O
      // the staging writes are ordered before the producer's next TMA write
      // into this buffer; fenced before the global stores are issued (the
      // fence would otherwise wait for them)
      asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
      __syncwarp();  // each warp stores the 32 rows it staged
      if (tt) tt[11] = clock64();
      if (ew * 32 + 32 <= n_out) {
        // all 32 rows exist: one TMA store (box 32 rows x d_h, the staging
        // swizzle); the buffer is released once the store has read it
        if (lane == 0) {
          tma_store_2d(&tmO, smem + Ly::q_off(b) + ew * 32 * Ly::RB, head * DH, (int)(rbase + ew * 32));
          asm volatile("cp.async.bulk.commit_group;" ::: "memory");
        }
        rel_b = b;
      } else {
        // the tile's last rows: row stores that stop at n_out (the rows past
        // it belong to the next user's candidates)
        constexpr int LPR = DH / 8;
        constexpr int RPI = 32 / LPR;
#pragma unroll
        for (int i = 0; i < 32; i += RPI) {
          const int rr = ew * 32 + i + lane / LPR;
          const int cj = lane % LPR;
          if (rr < n_out) {
            const int4 val = lds_v4(qbuf + rr * Ly::RB + (swz<DH>(rr, cj) << 4));
            *reinterpret_cast<int4*>(a.O + (rbase + rr) * D.d + head * DH + cj * 8) = val;
          }
        }
        __syncwarp();
        if (lane == 0) mbar_arrive(&q_empty[b]);  // the buffer (and its descriptor) go back to the producer
      }
      if (tt) tt[12] = clock64();
      kc += nch;
    }
    release_pending();
    if (lane == 0) asm volatile("cp.async.bulk.wait_group 0;" ::: "memory");
  }
  fence_before();
  __syncthreads();
  if (warp == 2) {
    fence_after();
    asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem_base), "r"(256));
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

static int sm_count() {
  int dev = 0, n = 148;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&n, cudaDevAttrMultiProcessorCount, dev);
  return n;
}
// CLIMBER_ATTN_PERSIST=0 selects the one-tile kernels (A/B; tested: bitwise
// equal for history rows, within the parity tolerance for SUMI rows, whose
// self term the persistent kernel merges at the end instead of first)
static bool use_persistent(int /*mode*/) {
  static const bool on = [] { const char* e = getenv("CLIMBER_ATTN_PERSIST"); return !e || atoi(e) != 0; }();
  return on;
}

template <int DH, int MODE>
static void launch(const CUtensorMap& mq, const CUtensorMap& mkv, const Args& a, dim3 grid, cudaStream_t s,
                   const CUtensorMap* mo = nullptr) {
  constexpr int smem = Lay<DH>::TOTAL;
  static_assert(2 * (smem + 1024) <= 233472, "two CTAs per SM");
  static_assert(2 * (PLay<DH>::TOTAL + 1024) <= 233472, "two persistent CTAs per SM");
  // persistent kernel without the relative bias (A/B in a 128-user `large`
  // step: history 339-341 vs 258-262 TFLOP/s, medium 109 vs 80; SUMI see
  // DESIGN.md §6)
  {
    if (!a.D.bpos && mo && use_persistent(MODE)) {
      const int n_tiles = (int)(grid.x * grid.y * grid.z);
      int n_cta = min(n_tiles, 2 * sm_count());
      if (n_cta <= 0) return;
      // a CTA walks t, t + n_cta, ...: with n_cta coprime to the tiles per
      // (user, block, head) (x fastest) every CTA cycles through all x, so the
      // causal history tiles (x + 1 chunks) spread evenly over the CTAs
      while (n_cta > 1 && std::gcd(n_cta, (int)grid.x) != 1) --n_cta;
      constexpr int psmem = PLay<DH>::TOTAL;
      ensure_smem_attr((const void*)k_attn_pers<DH, MODE>, psmem);
      k_attn_pers<DH, MODE><<<n_cta, THREADS, psmem, s>>>(mq, mkv, *mo, a, (int)grid.x, n_tiles);
      return;
    }
  }
  if (a.D.bpos) {
    ensure_smem_attr((const void*)k_attn_fa<DH, MODE, 1>, smem);
    k_attn_fa<DH, MODE, 1><<<grid, THREADS, smem, s>>>(mq, mkv, a);
  } else {
    ensure_smem_attr((const void*)k_attn_fa<DH, MODE, 0>, smem);
    k_attn_fa<DH, MODE, 0><<<grid, THREADS, smem, s>>>(mq, mkv, a);
  }
}

static bool g_trace_bias = false;  // the traced launch ran the relative-bias (one-tile) kernel
static int g_trace_mode = 0;       // ... and its mode (SUMI / history)
// CLIMBER_FA_TRACE=n: record the n-th launch of this process (clock64 per CTA)
// and print the mean timeline relative to each CTA's start
static unsigned long long* trace_begin(long long n_cta) {
  static const int at = [] { const char* e = getenv("CLIMBER_FA_TRACE"); return e ? atoi(e) : -1; }();
  static int n_launch = 0;
  if (at < 0 || n_launch++ != at) return nullptr;
  unsigned long long* buf = nullptr;
  cudaMallocManaged(&buf, n_cta * TRACE_N * 8);
  cudaMemset(buf, 0, n_cta * TRACE_N * 8);
  return buf;
}
static void ptrace_print(const unsigned long long* buf, long long n_cta) {
  double acc[TRACE_N] = {0};
  long long cnt[TRACE_N] = {0};
  for (long long c = 0; c < n_cta; ++c) {
    const unsigned long long* t = buf + c * TRACE_N;
    if (!t[127]) continue;
    for (int i = 0; i < 127; ++i)
      if (t[i]) acc[i] += (double)(long long)(t[i] - t[127]), cnt[i]++;
  }
  auto m = [&](int i) { return cnt[i] ? acc[i] / cnt[i] : -1.0; };
  fprintf(stderr, "[fa ptrace] persistent kernel (cycles since CTA start)\n");
  for (int it = 0; it < 4; ++it) {
    const int b = it * 24;
    fprintf(stderr, "[fa ptrace] tile %d: q %7.0f | S0 %7.0f P0 %7.0f S1 %7.0f P1 %7.0f S2 %7.0f P2 %7.0f "
                    "S3 %7.0f P3 %7.0f | self+pv_done %7.0f staged %7.0f released %7.0f\n",
            it, m(b), m(b + 2), m(b + 3), m(b + 4), m(b + 5), m(b + 6), m(b + 7), m(b + 8), m(b + 9), m(b + 10),
            m(b + 11), m(b + 12));
  }
  for (int i = 0; i < 16; ++i) fprintf(stderr, "[fa ptrace] QK %2d issued %7.0f%s", i, m(96 + i), i % 4 == 3 ? "\n" : " |");
  for (int i = 0; i < 12; ++i) fprintf(stderr, "[fa ptrace] PV %2d issued %7.0f%s", i, m(112 + i), i % 4 == 3 ? "\n" : " |");
}
static void trace_end(unsigned long long* buf, long long n_cta, cudaStream_t s) {
  if (!buf) return;
  cudaStreamSynchronize(s);
  if (use_persistent(g_trace_mode) && !g_trace_bias) {
    ptrace_print(buf, n_cta);
    cudaFree(buf);
    return;
  }
  double acc[TRACE_N] = {0};
  long long cnt[TRACE_N] = {0};
  for (long long c = 0; c < n_cta; ++c) {
    const unsigned long long* t = buf + c * TRACE_N;
    if (!t[127]) continue;
    for (int i = 0; i < 127; ++i)
      if (t[i]) acc[i] += (double)(long long)(t[i] - t[127]), cnt[i]++;
  }
  auto m = [&](int i) { return cnt[i] ? acc[i] / cnt[i] : -1.0; };
  fprintf(stderr, "[fa trace] %lld CTAs (cycles since start)\n", n_cta);
  fprintf(stderr, "[fa trace] q tiles seen %7.0f\n", m(126));
  for (int j = 0; j < 12; ++j)
    fprintf(stderr, "[fa trace] chunk %2d: kv %7.0f | S %7.0f ld %7.0f max %7.0f P %7.0f | mma saw P %7.0f\n", j,
            m(96 + j), m(2 * j), m(40 + j), m(52 + j), m(2 * j + 1), m(64 + j));
  fprintf(stderr, "[fa trace] epilogue %7.0f: pv_done %7.0f staged %7.0f synced %7.0f end %7.0f\n", m(30), m(27),
          m(28), m(29), m(31));
  cudaFree(buf);
}

}  // namespace fa

// d_h 32 / 64 and whole pages (the history kernel covers n_k % 128 == 64 with a
// half-empty last tile)
bool attn_tc_supported(int dh, int nk, bool /*hist*/) {
  return (dh == 32 || dh == 64) && nk % PAGE == 0 && nk <= 32 * PAGE && fa::encoder() != nullptr;
}

void launch_attn_sumi_tc(const bf16* QKV, long long P, const int64_t* cand_off, const int* wave_slot,
                         const int* wave_r, int U, int Mmax, const bf16* pool, long long pool_rows, const int* ptab,
                         const int* vlen_all, const float* tau, bf16* O, int k, int l, const Dims& D, cudaStream_t s,
                         int nbk) {
  CUtensorMap mq, mkv, mo;
  if (!fa::map2d(&mq, QKV, P * nbk, 3 * D.d, 3LL * D.d, D.dh, fa::ROWS) ||
      !fa::map2d(&mkv, pool, pool_rows, D.d, D.d, D.dh, PAGE) ||
      !fa::map2d(&mo, O, P * nbk, D.d, D.d, D.dh, 32)) {  // O rows: 32-row boxes (one softmax warp)
    note_launch_error("SUMI attention: cuTensorMapEncodeTiled rejected a map (kernel not launched)");
    return;
  }
  fa::Args a{QKV, cand_off, wave_slot, wave_r, ptab, vlen_all, tau, O, k, l, U, P, D, nullptr};
  dim3 grid((Mmax + fa::ROWS - 1) / fa::ROWS, D.h, U * nbk);
  const long long n_cta = (long long)grid.x * grid.y * grid.z;
  a.trace = fa::trace_begin(n_cta);
  fa::g_trace_bias = D.bpos != nullptr;
  fa::g_trace_mode = fa::MODE_SUMI;
  if (D.dh == 64) fa::launch<64, fa::MODE_SUMI>(mq, mkv, a, grid, s, &mo);
  else fa::launch<32, fa::MODE_SUMI>(mq, mkv, a, grid, s, &mo);
  fa::trace_end(a.trace, n_cta, s);
}

void launch_attn_hist_tc(const bf16* Q, const int* wave_slot, const int* wave_r, int U, const bf16* pool,
                         long long pool_rows, const int* ptab, const int* vlen_all, const float* tau, bf16* O, int k,
                         int l, const Dims& D, cudaStream_t s, int nbk) {
  CUtensorMap mq, mkv, mo;
  if (!fa::map2d(&mq, Q, (long long)U * D.nk * nbk, D.d, D.d, D.dh, fa::ROWS) ||
      !fa::map2d(&mkv, pool, pool_rows, D.d, D.d, D.dh, PAGE) ||
      !fa::map2d(&mo, O, (long long)U * D.nk * nbk, D.d, D.d, D.dh, 32)) {
    note_launch_error("history attention: cuTensorMapEncodeTiled rejected a map (kernel not launched)");
    return;
  }
  fa::Args a{Q, nullptr, wave_slot, wave_r, ptab, vlen_all, tau, O, k, l, U, (long long)U * D.nk, D, nullptr};
  dim3 grid((D.nk + fa::ROWS - 1) / fa::ROWS, D.h, U * nbk);
  const long long n_cta = (long long)grid.x * grid.y * grid.z;
  a.trace = fa::trace_begin(n_cta);
  fa::g_trace_bias = D.bpos != nullptr;
  fa::g_trace_mode = fa::MODE_HIST;
  if (D.dh == 64) fa::launch<64, fa::MODE_HIST>(mq, mkv, a, grid, s, &mo);
  else fa::launch<32, fa::MODE_HIST>(mq, mkv, a, grid, s, &mo);
  fa::trace_end(a.trace, n_cta, s);
}

}  // namespace climber
