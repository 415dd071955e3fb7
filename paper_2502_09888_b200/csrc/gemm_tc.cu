// tcgen05 GEMM for sm_100a: D[m][n] = sum_k A[m][k] * B[n][k], bf16 operands
// (both K-contiguous), fp32 accumulation in TMEM, fused epilogues (QKV + K/V
// page write, fp32 residual add, SiLU/ReLU + bias, sigmoid gate) from
// common.cuh.  These are the f_QKV / W_O / f_FFN / squeeze-and-excitation
// contractions of PAPER.md Eq. 3-4.
//
// Structure (persistent over output tiles; default: CTA pairs, see CG below):
//   warp 0      TMA producer: A tile 128x64 and B tile BNx64 per k-block,
//               128B-swizzled, into a STAGES-deep smem ring (full/empty mbarriers)
//   warp 1      MMA issuer: one elected thread issues tcgen05.mma (M=128, N=BN,
//               K=16) into one of two TMEM accumulators, tcgen05.commit frees the
//               smem stage / publishes the accumulator
//   warp 2      TMEM allocator (2*BN columns)
//   warps 4..7  epilogue: tcgen05.ld 32 columns at a time, apply the epilogue,
//               release the accumulator so the MMA of the next tile overlaps
#include <cuda.h>
#include <cudaTypedefs.h>

#include <cstdio>
#include <cstdlib>
#include <mutex>

#include "kernels.cuh"
#include "tc_util.cuh"

namespace climber {
namespace tc {
using namespace tcu;

constexpr int BM = 128;
constexpr int BK = 64;  // 64 bf16 = 128 B rows = one SWIZZLE_128B atom width


template <int BN, int STAGES, int EPIW, int SBUF, int NORM = 0, int CG = 1>
struct Smem {
  static constexpr int A_BYTES = BM * BK * 2;
  static constexpr int B_BYTES = (BN / CG) * BK * 2;  // CG = 2: this CTA's half of the B tile
  static constexpr int STAGE_BYTES = A_BYTES + B_BYTES;
  static constexpr int STG_OFF = STAGES * STAGE_BYTES;  // epilogue staging: 4 warps x 2 x (32 rows x 128 B)
  // NORM (EPI_RESID_NORM): per warp NORM staging sets x (fp32 box 32x32 + bf16 box 32x32), 6 KB each
  static constexpr int STG_WARP = NORM ? NORM * 6144 : SBUF * 32 * 128;
  static constexpr int BAR_OFF = STG_OFF + EPIW * STG_WARP;
  static constexpr int TOTAL = BAR_OFF + 512 + 1024;  // barriers + tmem addr, + alignment slack
};

// EPIW epilogue warps (4 or 8), SBUF staging buffers per epilogue warp (1 or 2),
// NORM > 0: the EPI_RESID_NORM epilogue (residual add + bf16 copy + row sums of
// squares) with NORM staging sets per epilogue warp, so NORM - 1 chunks of the
// old residual are in flight ahead of the one being added
// CG = 2: CTA pair (2x1 cluster) computing a 256 x BN tile with cta_group::2
// MMAs issued by the leader; CTA r owns rows 128 r .. 128 r + 127 of the tile
// (its A half, its TMEM lanes, its epilogue) and loads B rows r BN/2 .. of it.
template <int BN, int STAGES, int EPIW, int SBUF, int NORM, int CG>
__global__ void __launch_bounds__(128 + 32 * EPIW, 1)
    k_gemm_tc(const __grid_constant__ CUtensorMap tmA, const __grid_constant__ CUtensorMap tmB,
              const __grid_constant__ CUtensorMap tmD, const __grid_constant__ CUtensorMap tmP,
              const __grid_constant__ CUtensorMap tmC16, long long M, int N, int K, int batch, Epilogue e) {
  using S = Smem<BN, STAGES, EPIW, SBUF, NORM, CG>;
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  uint64_t* full = reinterpret_cast<uint64_t*>(smem + S::BAR_OFF);
  uint64_t* empty = full + STAGES;
  uint64_t* tfull = empty + STAGES;
  uint64_t* tempty = tfull + 2;
  uint64_t* ldbar = tempty + 2;  // NORM: one TMA-load barrier per staging set per epilogue warp
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(ldbar + 4 * EPIW);

  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int crank = CG == 2 ? (int)cluster_rank() : 0;
  const long long tile_start = blockIdx.x / CG, tile_step = gridDim.x / CG;  // one tile per cluster
  const int n_tiles = N / BN;
  const long long m_tiles = (M + CG * BM - 1) / (CG * BM);
  const long long tiles_per_b = m_tiles * n_tiles;
  const long long num_tiles = tiles_per_b * batch;  // batch-major: t -> (b, m_blk, n_blk)
  const int kblocks = K / BK;

  if (warp == 0 && lane == 0) {
    asm volatile("prefetch.tensormap [%0];" ::"l"(&tmA) : "memory");
    asm volatile("prefetch.tensormap [%0];" ::"l"(&tmB) : "memory");
    asm volatile("prefetch.tensormap [%0];" ::"l"(&tmD) : "memory");
    asm volatile("prefetch.tensormap [%0];" ::"l"(&tmP) : "memory");
    asm volatile("prefetch.tensormap [%0];" ::"l"(&tmC16) : "memory");
    for (int s = 0; s < STAGES; ++s) {
      mbar_init(&full[s], 1);
      mbar_init(&empty[s], 1);
    }
    for (int a = 0; a < 2; ++a) {
      mbar_init(&tfull[a], 1);
      mbar_init(&tempty[a], CG * EPIW);  // one arrival per epilogue warp of the pair (leader's copy)
    }
    for (int a = 0; a < 4 * EPIW; ++a) mbar_init(&ldbar[a], 1);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  if (warp == 2) {
    if constexpr (CG == 2) {
      asm volatile("tcgen05.alloc.cta_group::2.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(smem_u32(tmem_slot)),
                   "r"(2 * BN));
      asm volatile("tcgen05.relinquish_alloc_permit.cta_group::2.sync.aligned;");
    } else {
      asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(smem_u32(tmem_slot)),
                   "r"(2 * BN));
      asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
    }
  }
  fence_before();
  if constexpr (CG == 2) cluster_sync();  // peer barriers initialised before any remote arrive / complete_tx
  else __syncthreads();
  fence_after();
  const uint32_t tmem_base = *tmem_slot;
  // the accumulator-empty barrier lives in the leader (cluster address)
  const uint32_t tempty_c0 = CG == 2 ? mapa(smem_u32(&tempty[0]), 0) : smem_u32(&tempty[0]);

  if (warp == 0) {
    if (lane == 0) {
      // ---------------- TMA producer ----------------
      int stage = 0;
      uint32_t phase = 0;
      for (long long t = tile_start; t < num_tiles; t += tile_step) {
        const int bt = (int)(t / tiles_per_b);
        const long long tr = t % tiles_per_b;
        const int m_blk = (int)(tr / n_tiles), n_blk = (int)(tr % n_tiles);
        const int arow = (m_blk * CG + crank) * BM, brow = n_blk * BN + crank * (BN / CG);
        for (int kb = 0; kb < kblocks; ++kb) {
          mbar_wait(&empty[stage], phase ^ 1);
          uint8_t* sa = smem + stage * S::STAGE_BYTES;
          uint8_t* sb = sa + S::A_BYTES;
          if constexpr (CG == 2) {  // both halves complete on the leader's full barrier
            const uint32_t fb = mapa(smem_u32(&full[stage]), 0);
            if (crank == 0) mbar_expect_tx(&full[stage], 2 * S::STAGE_BYTES);
            tma_load_3d_cg2(sa, &tmA, fb, kb * BK, arow, bt);
            tma_load_3d_cg2(sb, &tmB, fb, kb * BK, brow, bt);
          } else {
            mbar_expect_tx(&full[stage], S::STAGE_BYTES);
            tma_load_3d(sa, &tmA, &full[stage], kb * BK, arow, bt);
            tma_load_3d(sb, &tmB, &full[stage], kb * BK, brow, bt);
          }
          if (++stage == STAGES) { stage = 0; phase ^= 1; }
        }
      }
    }
  } else if (warp == 1) {
    if (lane == 0 && crank == 0) {
      // ---------------- MMA issuer (the pair's leader) ----------------
      constexpr uint32_t idesc = idesc_bf16(CG * BM, BN);
      int stage = 0;
      uint32_t phase = 0;
      int acc = 0;
      uint32_t acc_phase = 0;
      for (long long t = tile_start; t < num_tiles; t += tile_step) {
        mbar_wait(&tempty[acc], acc_phase ^ 1);
        fence_after();
        const uint32_t d_tmem = tmem_base + acc * BN;
        for (int kb = 0; kb < kblocks; ++kb) {
          mbar_wait(&full[stage], phase);
          fence_after();
          uint8_t* sa = smem + stage * S::STAGE_BYTES;
          uint8_t* sb = sa + S::A_BYTES;
          const uint64_t da = sdesc(sa), db = sdesc(sb);
#pragma unroll
          for (int k = 0; k < BK / 16; ++k) {  // +32 B along K inside the swizzle atom = +2 in the addr field
            if constexpr (CG == 2) mma_bf16_cg2(d_tmem, da + 2 * k, db + 2 * k, idesc, (kb | k) ? 1u : 0u);
            else mma_bf16(d_tmem, da + 2 * k, db + 2 * k, idesc, (kb | k) ? 1u : 0u);
          }
          if constexpr (CG == 2) mma_commit_cg2(&empty[stage]);
          else mma_commit(&empty[stage]);
          if (++stage == STAGES) { stage = 0; phase ^= 1; }
        }
        if constexpr (CG == 2) mma_commit_cg2(&tfull[acc]);
        else mma_commit(&tfull[acc]);
        if (++acc == 2) { acc = 0; acc_phase ^= 1; }
      }
    }
  } else if (warp >= 4) {
    // ---------------- epilogue ----------------
    // STORE / STORE_F32 / RESID: TMEM -> registers -> (bias, activation) ->
    // 128B-swizzled smem (32 rows x 128 B per warp, double buffered) -> one TMA
    // tile store (or TMA reduce-add into the fp32 residual) per 32-row chunk.
    // QKV_PAGES (d % 64 == 0): Q columns -> TMA store into Q, K/V columns ->
    // TMA store of 32 token rows straight into the user's K/V page (the 32-row
    // group lies in one user and one page since n_k % 32 == 0).
    // Otherwise: transpose through smem, lane = column, coalesced page stores.
    // 8 warps: warp w reads TMEM lane quadrant w % 4 (hardware rule), the two
    // warps of a quadrant split the tile's columns in halves
    const int ew = warp & 3;             // TMEM lanes 32*ew .. 32*ew+31
    constexpr int NCG = EPIW / 4;        // column groups
    const int cg = (warp - 4) >> 2;      // this warp's column group
    uint8_t* stg = smem + S::STG_OFF + (warp - 4) * S::STG_WARP;
    const bool tma_epi = e.kind != EPI_QKV_PAGES || (e.d % 64 == 0);
    const bool f32_out = e.kind == EPI_RESID || e.kind == EPI_STORE_F32;
    const int CW = f32_out ? 32 : 64;  // columns per 128-byte staged row
    int sbuf = 0;
    int acc = 0;
    uint32_t acc_phase = 0;
    if constexpr (NORM) {
      // EPI_RESID_NORM, per 32-column chunk: the old residual C (fp32 box 32x32,
      // 128B-swizzled) is TMA-loaded into one of two staging sets (two chunks in
      // flight), C += acc in registers (thread = row), the new C is written back
      // in place and as bf16 into a 32x32 box (64B-swizzled), two TMA stores; the
      // row's sum of squares over each 128 columns goes to part[m][n0 / 128].
      constexpr int NS = NORM;  // staging sets per warp (<= 4: the ldbar array)
      static_assert(NS <= 4, "at most four residual staging sets per warp");
      uint64_t* lb = ldbar + (warp - 4) * NS;
      uint32_t lph[NS];
#pragma unroll
      for (int i = 0; i < NS; ++i) lph[i] = 0u;
      constexpr int NCH = BN / 32;
      int bt = 0;
      auto issue = [&](long long r0, int n0, int set) {
        if (lane == 0) {
          asm volatile("cp.async.bulk.wait_group.read 0;" ::: "memory");  // staging no longer read by stores
          mbar_expect_tx(&lb[set], 4096);
          tma_load_3d(stg + set * 6144, &tmD, &lb[set], n0, (int)r0, bt);
        }
      };
      for (long long t = tile_start; t < num_tiles; t += tile_step) {
        bt = (int)(t / tiles_per_b);
        const long long trm = t % tiles_per_b;
        const int m_blk = (int)(trm / n_tiles), n_blk = (int)(trm % n_tiles);
        const long long row0 = (long long)(m_blk * CG + crank) * BM + ew * 32;
        const bool rows_ok = row0 < M;  // warp-uniform
        if (rows_ok) {  // the first NS chunks of old residual are requested before the accumulator wait
#pragma unroll
          for (int i = 0; i < NS; ++i)
            if (i < NCH) issue(row0, n_blk * BN + 32 * i, i);
        }
        mbar_wait(&tfull[acc], acc_phase);
        fence_after();
        const uint32_t taddr = tmem_base + ((uint32_t)(ew * 32) << 16) + acc * BN;
        float ss = 0.f;
#pragma unroll 1
        for (int q = 0; q < NCH; ++q) {
          const int set = q % NS;
          const int n0 = n_blk * BN + q * 32;
          // chunk q + NS - 1 into the set of chunk q - 1 (its stores were committed last)
          if (rows_ok && q >= 1 && q + NS - 1 < NCH) issue(row0, n0 + 32 * (NS - 1), (q - 1) % NS);
          float v[32];
          tmem_ld32(taddr + q * 32, v);
          if (rows_ok) {
            mbar_wait(&lb[set], lph[set]);
            lph[set] ^= 1;
            uint8_t* b = stg + set * 6144;
            uint8_t* rowp = b + lane * 128;
#pragma unroll
            for (int j = 0; j < 8; ++j) {
              float4* p4 = reinterpret_cast<float4*>(rowp + ((j ^ (lane & 7)) << 4));
              const float4 o = *p4;
              float* vv = v + 4 * j;
              vv[0] += o.x; vv[1] += o.y; vv[2] += o.z; vv[3] += o.w;
              ss = fmaf(vv[0], vv[0], fmaf(vv[1], vv[1], fmaf(vv[2], vv[2], fmaf(vv[3], vv[3], ss))));
              *p4 = make_float4(vv[0], vv[1], vv[2], vv[3]);
            }
            uint8_t* brow = b + 4096 + lane * 64;  // bf16 box: 64 B rows, 64B swizzle
#pragma unroll
            for (int j = 0; j < 4; ++j) {
              __nv_bfloat162 p0 = __floats2bfloat162_rn(v[8 * j], v[8 * j + 1]);
              __nv_bfloat162 p1 = __floats2bfloat162_rn(v[8 * j + 2], v[8 * j + 3]);
              __nv_bfloat162 p2 = __floats2bfloat162_rn(v[8 * j + 4], v[8 * j + 5]);
              __nv_bfloat162 p3 = __floats2bfloat162_rn(v[8 * j + 6], v[8 * j + 7]);
              st_shared_v4(brow + ((j ^ ((lane >> 1) & 3)) << 4), *reinterpret_cast<uint32_t*>(&p0),
                           *reinterpret_cast<uint32_t*>(&p1), *reinterpret_cast<uint32_t*>(&p2),
                           *reinterpret_cast<uint32_t*>(&p3));
            }
            asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
            __syncwarp();
            if (lane == 0) {
              tma_store_3d(&tmD, b, n0, (int)row0, bt);
              tma_store_3d(&tmC16, b + 4096, n0, (int)row0, bt);
              asm volatile("cp.async.bulk.commit_group;" ::: "memory");
            }
          }
          // one partial per 128 columns (the same slots whatever BN is)
          if ((q & 3) == 3) {
            if (rows_ok && row0 + lane < M)
              e.part[bt * e.part_bs + (row0 + lane) * e.part_rs + n_blk * (BN / 128) + (q >> 2)] = ss;
            ss = 0.f;
          }
        }
        fence_before();
        __syncwarp();
        if (lane == 0) mbar_arrive_cluster(tempty_c0 + acc * 8);
        if (++acc == 2) { acc = 0; acc_phase ^= 1; }
      }
    } else
    for (long long t = tile_start; t < num_tiles; t += tile_step) {
      const int bt = (int)(t / tiles_per_b);
      const long long trm = t % tiles_per_b;
      const int m_blk = (int)(trm / n_tiles), n_blk = (int)(trm % n_tiles);
      const long long row0 = (long long)(m_blk * CG + crank) * BM + ew * 32;
      // RMSNorm folded into this GEMM: the per-row 1/rms from the producer's
      // partials, loaded before the accumulator wait so the latency is hidden
      float rsc = 1.f;
      if (e.rs_part != nullptr && row0 + lane < M) {
        float sum = 0.f;
        for (int j = 0; j < e.rs_n; ++j) sum += e.rs_part[bt * e.rs_bs + (row0 + lane) * e.rs_rs + j];
        rsc = rsqrtf(sum * e.rs_inv_d + e.rs_eps);
      }
      mbar_wait(&tfull[acc], acc_phase);
      fence_after();
      const uint32_t taddr = tmem_base + ((uint32_t)(ew * 32) << 16) + acc * BN;
      if (tma_epi) {
#pragma unroll 1
        for (int c = cg * (BN / NCG); c < (cg + 1) * (BN / NCG); c += CW) {
          float v[64];
          tmem_ld32(taddr + c, v);  // lane = row row0 + lane
          if (!f32_out) tmem_ld32(taddr + c + 32, v + 32);
          const int n0 = n_blk * BN + c;
          // FFN-up (the epilogue paces these K = 512 launches): SiLU(x rs) =
          // h + h tanh(h) with h = x rs / 2 -- one multiply, one MUFU, one FMA
          const bool silu_fused = !f32_out && e.kind == EPI_STORE && e.act == ACT_SILU && e.bias == nullptr;
          if (silu_fused) {  // packed FP32x2 multiply / FMA: two elements per issue slot
            const uint64_t hs2 = f2_pack(0.5f * rsc, 0.5f * rsc);
#pragma unroll
            for (int i = 0; i < 64; i += 2) {
              const uint64_t h2 = f2_mul(f2_pack(v[i], v[i + 1]), hs2);
              const float2 h = f2_unpack(h2);
              const float2 y = f2_unpack(f2_fma(h2, f2_pack(tanh_approx(h.x), tanh_approx(h.y)), h2));
              v[i] = y.x;
              v[i + 1] = y.y;
            }
          } else if (e.rs_part != nullptr) {
            const uint64_t r2 = f2_pack(rsc, rsc);
#pragma unroll
            for (int i = 0; i < 64; i += 2) {
              const float2 y = f2_unpack(f2_mul(f2_pack(v[i], v[i + 1]), r2));
              v[i] = y.x;
              v[i + 1] = y.y;
            }
          }
          if (!silu_fused && e.kind != EPI_RESID && e.kind != EPI_QKV_PAGES) {
            // bias (vectorised) and activation, each hoisted out of the element loop
            if (e.bias != nullptr) {
              const float4* b4 = reinterpret_cast<const float4*>(e.bias + n0);
#pragma unroll
              for (int j = 0; j < 16; ++j) {
                if (4 * j < CW) {
                  const float4 b = b4[j];
                  v[4 * j] += b.x; v[4 * j + 1] += b.y; v[4 * j + 2] += b.z; v[4 * j + 3] += b.w;
                }
              }
            }
            const int act = e.act;
            if (act == ACT_SILU) {
#pragma unroll
              for (int i = 0; i < 64; ++i) v[i] = silu_t<bf16>(v[i]);
            } else if (act == ACT_SIGMOID) {
#pragma unroll
              for (int i = 0; i < 64; ++i) v[i] = sigmoid_t<bf16>(v[i]);
            } else if (act == ACT_RELU) {
#pragma unroll
              for (int i = 0; i < 64; ++i) v[i] = fmaxf(v[i], 0.f);
            }
          }
          uint8_t* buf = stg + sbuf * 4096;
          if (lane == 0) {
            if (SBUF == 2) asm volatile("cp.async.bulk.wait_group.read 1;" ::: "memory");
            else asm volatile("cp.async.bulk.wait_group.read 0;" ::: "memory");
          }
          __syncwarp();
          uint8_t* rowp = buf + lane * 128;
          if (f32_out) {
#pragma unroll
            for (int j = 0; j < 8; ++j)
              st_shared_v4(rowp + ((j ^ (lane & 7)) << 4), __float_as_uint(v[4 * j]), __float_as_uint(v[4 * j + 1]),
                           __float_as_uint(v[4 * j + 2]), __float_as_uint(v[4 * j + 3]));
          } else {
#pragma unroll
            for (int j = 0; j < 8; ++j) {
              __nv_bfloat162 p0 = __floats2bfloat162_rn(v[8 * j], v[8 * j + 1]);
              __nv_bfloat162 p1 = __floats2bfloat162_rn(v[8 * j + 2], v[8 * j + 3]);
              __nv_bfloat162 p2 = __floats2bfloat162_rn(v[8 * j + 4], v[8 * j + 5]);
              __nv_bfloat162 p3 = __floats2bfloat162_rn(v[8 * j + 6], v[8 * j + 7]);
              st_shared_v4(rowp + ((j ^ (lane & 7)) << 4), *reinterpret_cast<uint32_t*>(&p0),
                           *reinterpret_cast<uint32_t*>(&p1), *reinterpret_cast<uint32_t*>(&p2),
                           *reinterpret_cast<uint32_t*>(&p3));
            }
          }
          asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
          __syncwarp();
          if (lane == 0 && row0 < M) {
            if (e.kind == EPI_RESID) {
              tma_reduce_add_3d(&tmD, buf, n0, (int)row0, bt);
            } else if (e.kind == EPI_QKV_PAGES) {
              const int cg = n0 + e.col_off;
              if (cg < e.d) {
                tma_store_3d(&tmD, buf, cg, (int)row0, bt);
              } else {
                const int kv = cg >= 2 * e.d ? 1 : 0;
                const int cc = cg - e.d * (1 + kv);
                const int u = (int)(row0 / e.nk), tt = (int)(row0 % e.nk);
                const int slot = e.wave_slot[u];
                const int blk = e.blk_from_batch ? e.blk + bt : e.blk;
                const int page = e.ptab[(((long long)slot * e.Nb + blk) * e.L + e.layer) * e.ppb + tt / PAGE];
                tma_store_3d(&tmP, buf, cc, (int)page_row(page, kv, tt % PAGE), 0);
              }
            } else {
              tma_store_3d(&tmD, buf, n0, (int)row0, bt);
            }
            asm volatile("cp.async.bulk.commit_group;" ::: "memory");
          }
          sbuf = (SBUF == 2) ? (sbuf ^ 1) : 0;
        }
      } else {
        float (*tr)[33] = reinterpret_cast<float (*)[33]>(stg);
#pragma unroll 1
        for (int c = cg * (BN / NCG); c < (cg + 1) * (BN / NCG); c += 32) {
          float v[32];
          tmem_ld32(taddr + c, v);
#pragma unroll
          for (int i = 0; i < 32; ++i) tr[lane][i] = v[i];
          __syncwarp();
          const int n = n_blk * BN + c + lane;
#pragma unroll 4
          for (int i = 0; i < 32; ++i)  // row row0 + i, lane = column: coalesced
            if (row0 + i < M) epilogue_elem<bf16>(e, row0 + i, n, tr[i][lane]);
          __syncwarp();
        }
      }
      fence_before();
      __syncwarp();
      if (lane == 0) mbar_arrive_cluster(tempty_c0 + acc * 8);
      if (++acc == 2) { acc = 0; acc_phase ^= 1; }
    }
    if (lane == 0) asm volatile("cp.async.bulk.wait_group 0;" ::: "memory");
  }
  fence_before();
  if constexpr (CG == 2) cluster_sync();  // the leader's MMAs read the peer's smem until the last tile
  else __syncthreads();
  if (warp == 2) {
    fence_after();
    if constexpr (CG == 2)
      asm volatile("tcgen05.dealloc.cta_group::2.sync.aligned.b32 %0, %1;" ::"r"(tmem_base), "r"(2 * BN));
    else
      asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem_base), "r"(2 * BN));
  }
}

// ---------------------------------------------------------------------------
// host side
// ---------------------------------------------------------------------------
static PFN_cuTensorMapEncodeTiled_v12000 get_encode() {
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

// 3-D map [batch][rows][cols] (batch stride bs elements, may be < rows * ld for
// interleaved views such as the N_b block slots of one candidate row)
static bool make_map(CUtensorMap* map, const void* ptr, long long rows, int cols, long long ld, int box_rows,
                     int box_cols = BK, bool f32 = false, bool sw64 = false, int batch = 1, long long bs = 0) {
  auto enc = get_encode();
  if (!enc) return false;
  const int es = f32 ? 4 : 2;
  if (batch <= 1) bs = rows * ld;
  cuuint64_t dims[3] = {(cuuint64_t)cols, (cuuint64_t)rows, (cuuint64_t)(batch < 1 ? 1 : batch)};
  cuuint64_t strides[2] = {(cuuint64_t)ld * es, (cuuint64_t)bs * es};
  cuuint32_t box[3] = {(cuuint32_t)box_cols, (cuuint32_t)box_rows, 1};
  cuuint32_t estr[3] = {1, 1, 1};
  CUresult r = enc(map, f32 ? CU_TENSOR_MAP_DATA_TYPE_FLOAT32 : CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 3,
                   const_cast<void*>(ptr), dims, strides, box, estr,
                   CU_TENSOR_MAP_INTERLEAVE_NONE, sw64 ? CU_TENSOR_MAP_SWIZZLE_64B : CU_TENSOR_MAP_SWIZZLE_128B,
                   CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                   CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  if (r != CUDA_SUCCESS)
    fprintf(stderr, "[climber] cuTensorMapEncodeTiled failed (%d): rows %lld cols %d ld %lld batch %d bs %lld\n", (int)r,
            rows, cols, ld, batch, bs);
  return r == CUDA_SUCCESS;
}

static int num_sms() {
  static int n = 0;
  if (!n) {
    int dev = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&n, cudaDevAttrMultiProcessorCount, dev);
    if (n <= 0) n = 148;
  }
  return n;
}

template <int BN, int STAGES, int EPIW, int SBUF, int NORM = 0, int CG = 1>
static void launch(const bf16* A, long long lda, long long abs_, const bf16* B, long long ldb, long long bbs,
                   long long M, int N, int K, int batch, const Epilogue& e, cudaStream_t s) {
  CUtensorMap ma, mb, md, mp, mc;
  bool ok = make_map(&ma, A, M, K, lda, BM, BK, false, false, batch, abs_);
  ok = ok && make_map(&mb, B, N, K, ldb, BN / CG, BK, false, false, batch, bbs);
  mp = ma;  // unused unless QKV_PAGES
  mc = ma;  // unused unless RESID_NORM
  if (e.kind == EPI_RESID_NORM) ok = ok && make_map(&mc, e.out_b16, M, N, e.ldo, 32, 32, false, true, batch, e.out_b16_bs);
  if (e.kind == EPI_QKV_PAGES) {
    if (e.d % 64 == 0) {
      ok = ok && make_map(&md, e.out, M, e.d, e.ldo, 32, 64, false, false, batch, e.out_bs);  // Q buffer [b][M][d]
      ok = ok && make_map(&mp, e.pool, e.pool_rows, e.d, e.d, 32, 64, false);  // pages as [n_pages*2*64][d]
    } else {
      md = ma;
    }
  } else if (e.kind == EPI_STORE) {
    ok = ok && make_map(&md, e.out, M, N, e.ldo, 32, 64, false, false, batch, e.out_bs);
  } else {
    ok = ok && make_map(&md, e.out, M, N, e.ldo, 32, 32, true, false, batch, e.out_bs);
  }
  if (!ok) {
    note_launch_error("tcgen05 GEMM: cuTensorMapEncodeTiled rejected an operand map (kernel not launched)");
    return;
  }
  constexpr int smem = Smem<BN, STAGES, EPIW, SBUF, NORM, CG>::TOTAL;
  static_assert(smem <= 232448, "smem");
  auto kern = k_gemm_tc<BN, STAGES, EPIW, SBUF, NORM, CG>;
  ensure_smem_attr((const void*)kern, smem);
  const long long tiles = ((M + CG * BM - 1) / (CG * BM)) * (N / BN) * batch;  // per CTA (pair)
  const long long slots = num_sms() / CG;
  const int grid = (int)(tiles < slots ? tiles : slots) * CG;
  if constexpr (CG == 1) {
    kern<<<grid, 128 + 32 * EPIW, smem, s>>>(ma, mb, md, mp, mc, M, N, K, batch, e);
  } else {
    cudaLaunchConfig_t cfg{};
    cfg.gridDim = dim3(grid);
    cfg.blockDim = dim3(128 + 32 * EPIW);
    cfg.dynamicSmemBytes = smem;
    cfg.stream = s;
    cudaLaunchAttribute at[1];
    at[0].id = cudaLaunchAttributeClusterDimension;
    at[0].val.clusterDim.x = CG;
    at[0].val.clusterDim.y = 1;
    at[0].val.clusterDim.z = 1;
    cfg.attrs = at;
    cfg.numAttrs = 1;
    cudaLaunchKernelEx(&cfg, kern, ma, mb, md, mp, mc, M, N, K, batch, e);
  }
}

}  // namespace tc

bool gemm_tc_supported(long long M, int N, int K, long long lda, long long ldb) {
  if (M < 1 || M >= (1LL << 31) || K < tc::BK || K % tc::BK || N % 128) return false;
  if ((lda * 2) % 16 || (ldb * 2) % 16) return false;
  return tc::get_encode() != nullptr;
}

bool gemm_tc_available() { return tc::get_encode() != nullptr; }

void launch_gemm_tc_batched(const bf16* A, long long lda, long long a_bs, const bf16* B, long long ldb,
                            long long b_bs, long long M, int N, int K, int batch, const Epilogue& e, cudaStream_t s) {
  // small launches: 128 x 128 single-CTA tiles (4x the tiles) below
  // CLIMBER_GEMM_SMALL_WAVES (2) waves of pair CTAs and below
  // CLIMBER_GEMM_SMALL_GFLOP (1.5) GFLOP per launch.  Measured on one request
  // (latency graph with encode/score overlap): medium / small p50 0.54 / 0.44 ms
  // with small tiles vs 0.66 / 0.49 with pairs (launches <= 1.1 GF); at large
  // (launches >= 2.1 GF) pairs everywhere 1.51 ms vs 1.56-1.61 with small tiles
  const long long pair_ctas = ((M + 255) / 256) * (N / (N % 256 == 0 ? 256 : 128)) * batch * 2;
  // CLIMBER_GEMM_SMALL_WAVES (measurement knob): the threshold in waves of pair CTAs
  static const long long small_waves = [] {
    const char* e = getenv("CLIMBER_GEMM_SMALL_WAVES");
    return e ? atoll(e) : 2LL;
  }();
  static const double small_gflop = [] {
    const char* e = getenv("CLIMBER_GEMM_SMALL_GFLOP");
    return e ? atof(e) : 1.5;
  }();
  const double gflop = 2.0 * (double)M * N * K * batch * 1e-9;
  if (pair_ctas < small_waves * tc::num_sms() && gflop < small_gflop) {
    if (e.kind == EPI_RESID_NORM) {
      tc::launch<128, 4, 4, 2, 2>(A, lda, a_bs, B, ldb, b_bs, M, N, K, batch, e, s);
    } else {
      const bool heavy = (e.kind == EPI_STORE || e.kind == EPI_STORE_F32) && e.act != ACT_NONE;
      if (heavy) tc::launch<128, 5, 8, 2>(A, lda, a_bs, B, ldb, b_bs, M, N, K, batch, e, s);
      else tc::launch<128, 6, 4, 2>(A, lda, a_bs, B, ldb, b_bs, M, N, K, batch, e, s);
    }
    return;
  }
  {  // CTA pairs: 256 x BN tiles, each CTA streams half of B
    if (e.kind == EPI_RESID_NORM) {
      // K <= 512 (O-projection): HBM-bound on the residual stream -> four
      // staging sets per warp (three residual chunks in flight) over three
      // operand stages; longer K (FFN-down) keeps five operand stages
      if (N % 256 == 0 && K <= 512) tc::launch<256, 3, 4, 2, 4, 2>(A, lda, a_bs, B, ldb, b_bs, M, N, K, batch, e, s);
      else if (N % 256 == 0) tc::launch<256, 5, 4, 2, 2, 2>(A, lda, a_bs, B, ldb, b_bs, M, N, K, batch, e, s);
      else tc::launch<128, 6, 4, 2, 2, 2>(A, lda, a_bs, B, ldb, b_bs, M, N, K, batch, e, s);
      return;
    }
    // 8 epilogue warps for every store epilogue (QKV / K/V-page stores and the
    // activations): the K = 512 launches are paced by the epilogue, 993-1002
    // vs 895 TFLOP/s for the QKV class in the large step with 4 warps
    if (N % 256 == 0) tc::launch<256, 6, 8, 1, 0, 2>(A, lda, a_bs, B, ldb, b_bs, M, N, K, batch, e, s);
    else tc::launch<128, 8, 4, 2, 0, 2>(A, lda, a_bs, B, ldb, b_bs, M, N, K, batch, e, s);
  }
}

}  // namespace climber

namespace climber {
void launch_gemm_tc(const bf16* A, long long lda, const bf16* B, long long ldb, long long M, int N, int K,
                    const Epilogue& e, cudaStream_t s) {
  launch_gemm_tc_batched(A, lda, 0, B, ldb, 0, M, N, K, 1, e, s);
}
}  // namespace climber
