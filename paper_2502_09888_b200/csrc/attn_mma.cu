// Tensor-core attention for the bf16 path (Eq. 3 with f_b = 0;
// SUMI masks P:L255): softmax(q.k / (sqrt(d_h) tau)) v.
//
//   MODE_SUMI: each candidate row attends to the v cached history keys of its
//              (user, block, layer, head) plus its own (k_self, v_self).
//   MODE_HIST: history row t of a user attends keys j <= t (causal) or j < v.
//
// One CTA = 8 warps x 16 query rows = 128 rows of one (user, head).  K/V are
// streamed page by page (64 keys = one K/V page, PAGE) through a cp.async
// double buffer; S = Q K^T and O += P V use mma.sync m16n8k16 (bf16 in, fp32
// accumulate); the online softmax keeps fp32 row statistics in registers (a
// quad of lanes shares a row), P is re-packed from the S accumulators into
// A fragments without touching shared memory (FlashAttention-2 dataflow).
#include "kernels.cuh"

namespace climber {
namespace am {

constexpr int ROWS = 128;
constexpr int THREADS = 256;
constexpr int KEYS = PAGE;  // 64 keys per chunk = one page
constexpr float LOG2E = 1.4426950408889634f;

__device__ __forceinline__ uint32_t pack_bf16(float lo, float hi) {
  __nv_bfloat162 v = __floats2bfloat162_rn(lo, hi);
  return *reinterpret_cast<uint32_t*>(&v);
}

__device__ __forceinline__ void mma16816(float* c, const uint32_t* a, uint32_t b0, uint32_t b1) {
  asm volatile(
      "mma.sync.aligned.m16n8k16.row.col.f32.bf16.bf16.f32 {%0,%1,%2,%3}, {%4,%5,%6,%7}, {%8,%9}, "
      "{%0,%1,%2,%3};"
      : "+f"(c[0]), "+f"(c[1]), "+f"(c[2]), "+f"(c[3])
      : "r"(a[0]), "r"(a[1]), "r"(a[2]), "r"(a[3]), "r"(b0), "r"(b1));
}

__device__ __forceinline__ void cp_async16(void* smem, const void* gmem, bool valid) {
  uint32_t s = static_cast<uint32_t>(__cvta_generic_to_shared(smem));
  int n = valid ? 16 : 0;  // 0 -> zero fill
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16, %2;" ::"r"(s), "l"(gmem), "r"(n) : "memory");
}
__device__ __forceinline__ void cp_commit() { asm volatile("cp.async.commit_group;" ::: "memory"); }
template <int N>
__device__ __forceinline__ void cp_wait() { asm volatile("cp.async.wait_group %0;" ::"n"(N) : "memory"); }

__device__ __forceinline__ void ldsm_x4_trans(uint32_t* r, const void* smem) {
  uint32_t s = static_cast<uint32_t>(__cvta_generic_to_shared(smem));
  asm volatile("ldmatrix.sync.aligned.m8n8.x4.trans.shared.b16 {%0,%1,%2,%3}, [%4];"
               : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3])
               : "r"(s));
}

enum { MODE_SUMI = 0, MODE_HIST = 1 };

struct Args {
  const bf16* Q;          // SUMI: QKV [P][3d]; HIST: Q [U*nk][d]
  const int64_t* cand_off;
  const int* wave_slot;
  const int* wave_r;
  const bf16* pool;
  const int* ptab;
  const int* vlen_all;
  const float* tau;
  bf16* O;                // [rows][d]
  int k, l;
  Dims D;
};

template <int DH, int MODE>
__global__ void __launch_bounds__(THREADS) k_attn(Args a) {
  constexpr int LDS = DH + 8;  // padded smem row (bf16): conflict-free fragment loads
  __shared__ __align__(16) bf16 Ks[2][KEYS][LDS];
  __shared__ __align__(16) bf16 Vs[2][KEYS][LDS];
  const Dims& D = a.D;
  const int u = blockIdx.x, head = blockIdx.y;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int g = lane >> 2, t4 = lane & 3;
  const int slot = a.wave_slot[u];
  const int r = a.wave_r[u];
  const int v = a.vlen_all[(long long)slot * D.Nb + a.k];
  const int* pages = a.ptab + (((long long)slot * D.Nb + a.k) * D.L + a.l) * D.ppb;
  const float sc = LOG2E / (sqrtf((float)DH) * a.tau[((a.l * D.Nb + a.k) * D.R + r) * D.h + head]);

  // ---- rows of this CTA / warp ----
  long long row_base;   // global row index of tile row 0 (into Q / O)
  int n_rows;           // valid rows in this tile
  int key_end;          // keys [0, key_end) may be visible to some row of the tile
  const int tile0 = blockIdx.z * ROWS;
  long long ldq;
  if (MODE == MODE_SUMI) {
    const long long p0 = a.cand_off[u], p1 = a.cand_off[u + 1];
    if (p0 + tile0 >= p1) return;
    row_base = p0 + tile0;
    n_rows = (int)((p1 - row_base) < ROWS ? (p1 - row_base) : ROWS);
    key_end = v;
    ldq = 3LL * D.d;
  } else {
    if (tile0 >= D.nk) return;
    row_base = (long long)u * D.nk + tile0;
    n_rows = max(0, min(ROWS, v - tile0));  // rows >= v are pads (zero output)
    key_end = D.causal ? min(v, tile0 + ROWS) : v;
    ldq = D.d;
  }
  const int wr0 = warp * 16;  // warp's first tile row
  const int ra = wr0 + g, rb = wr0 + g + 8;
  const bool va = ra < n_rows, vb = rb < n_rows;

  // ---- Q fragments (A operand, row-major 16 x DH) ----
  uint32_t qf[DH / 16][4];
  {
    const bf16* qa = a.Q + (row_base + ra) * ldq + head * DH;
    const bf16* qb = a.Q + (row_base + rb) * ldq + head * DH;
#pragma unroll
    for (int kk = 0; kk < DH / 16; ++kk) {
      const int c = kk * 16 + 2 * t4;
      qf[kk][0] = va ? *reinterpret_cast<const uint32_t*>(qa + c) : 0u;
      qf[kk][1] = vb ? *reinterpret_cast<const uint32_t*>(qb + c) : 0u;
      qf[kk][2] = va ? *reinterpret_cast<const uint32_t*>(qa + c + 8) : 0u;
      qf[kk][3] = vb ? *reinterpret_cast<const uint32_t*>(qb + c + 8) : 0u;
    }
  }
  float o[DH / 8][4];
  float m_a, m_b, l_a, l_b;
  if (MODE == MODE_SUMI) {
    // self term first: s_self = q . k_self; o = v_self with weight exp2(0) = 1
    const bf16* ka = a.Q + (row_base + ra) * ldq + D.d + head * DH;
    const bf16* kb = a.Q + (row_base + rb) * ldq + D.d + head * DH;
    float sa = 0.f, sb = 0.f;
#pragma unroll
    for (int kk = 0; kk < DH / 16; ++kk) {
#pragma unroll
      for (int h2 = 0; h2 < 2; ++h2) {
        const int c = kk * 16 + 2 * t4 + 8 * h2;
        if (va) {
          float2 q2 = __bfloat1622float2(*reinterpret_cast<const __nv_bfloat162*>(&qf[kk][2 * h2]));
          float2 k2 = __bfloat1622float2(*reinterpret_cast<const __nv_bfloat162*>(ka + c));
          sa = fmaf(q2.x, k2.x, fmaf(q2.y, k2.y, sa));
        }
        if (vb) {
          float2 q2 = __bfloat1622float2(*reinterpret_cast<const __nv_bfloat162*>(&qf[kk][2 * h2 + 1]));
          float2 k2 = __bfloat1622float2(*reinterpret_cast<const __nv_bfloat162*>(kb + c));
          sb = fmaf(q2.x, k2.x, fmaf(q2.y, k2.y, sb));
        }
      }
    }
    sa += __shfl_xor_sync(0xffffffffu, sa, 1);
    sa += __shfl_xor_sync(0xffffffffu, sa, 2);
    sb += __shfl_xor_sync(0xffffffffu, sb, 1);
    sb += __shfl_xor_sync(0xffffffffu, sb, 2);
    m_a = sa * sc;
    m_b = sb * sc;
    // the quad shares a row: the self weight exp2(0) = 1 is counted on one lane
    l_a = l_b = (t4 == 0) ? 1.f : 0.f;
    const bf16* vsa = a.Q + (row_base + ra) * ldq + 2 * D.d + head * DH;
    const bf16* vsb = a.Q + (row_base + rb) * ldq + 2 * D.d + head * DH;
#pragma unroll
    for (int nt = 0; nt < DH / 8; ++nt) {
      const int c = nt * 8 + 2 * t4;
      float2 x = va ? __bfloat1622float2(*reinterpret_cast<const __nv_bfloat162*>(vsa + c)) : make_float2(0.f, 0.f);
      float2 y = vb ? __bfloat1622float2(*reinterpret_cast<const __nv_bfloat162*>(vsb + c)) : make_float2(0.f, 0.f);
      o[nt][0] = x.x; o[nt][1] = x.y; o[nt][2] = y.x; o[nt][3] = y.y;
    }
  } else {
    m_a = m_b = -INFINITY;
    l_a = l_b = 0.f;
#pragma unroll
    for (int nt = 0; nt < DH / 8; ++nt) o[nt][0] = o[nt][1] = o[nt][2] = o[nt][3] = 0.f;
  }

  // ---- K/V chunk loader (one page = 64 keys x DH, K then V) ----
  const int n_chunks = (key_end + KEYS - 1) / KEYS;
  auto load_chunk = [&](int j, int buf) {
    const int page = pages[j];
    const bf16* kg = a.pool + page_elem_offset(page, 0, head, 0, 0, D.d, DH);
    const bf16* vg = a.pool + page_elem_offset(page, 1, head, 0, 0, D.d, DH);
    const int nk = min(KEYS, key_end - j * KEYS);
    constexpr int VEC = DH / 8;  // 16-byte vectors per row
    for (int i = threadIdx.x; i < KEYS * VEC; i += THREADS) {
      const int row = i / VEC, cv = (i % VEC) * 8;
      const bool ok = row < nk;
      cp_async16(&Ks[buf][row][cv], kg + (long long)row * D.d + cv, ok);
      cp_async16(&Vs[buf][row][cv], vg + (long long)row * D.d + cv, ok);
    }
    cp_commit();
  };
  if (n_chunks > 0) load_chunk(0, 0);

  // causal: last query row (tile-relative) each warp row needs
  const int qa_t = tile0 + ra, qb_t = tile0 + rb;
  for (int j = 0; j < n_chunks; ++j) {
    const int buf = j & 1;
    if (j + 1 < n_chunks) {
      load_chunk(j + 1, buf ^ 1);
      cp_wait<1>();
    } else {
      cp_wait<0>();
    }
    __syncthreads();
    const int key0 = j * KEYS;
    const bool warp_needed = (MODE == MODE_SUMI) || !D.causal || (key0 <= tile0 + wr0 + 15);
    if (warp_needed && wr0 < n_rows) {
      // S = Q K^T : 16 x 64 per warp, 8 n-tiles of 8 keys
      float s[8][4];
#pragma unroll
      for (int nt = 0; nt < 8; ++nt) {
        s[nt][0] = s[nt][1] = s[nt][2] = s[nt][3] = 0.f;
#pragma unroll
        for (int kk = 0; kk < DH / 16; ++kk) {
          const bf16* kr = &Ks[buf][nt * 8 + g][kk * 16 + 2 * t4];
          uint32_t b0 = *reinterpret_cast<const uint32_t*>(kr);
          uint32_t b1 = *reinterpret_cast<const uint32_t*>(kr + 8);
          mma16816(s[nt], qf[kk], b0, b1);
        }
      }
      // mask + scale, row max
      float mxa = -INFINITY, mxb = -INFINITY;
#pragma unroll
      for (int nt = 0; nt < 8; ++nt) {
#pragma unroll
        for (int e = 0; e < 2; ++e) {
          const int key = key0 + nt * 8 + 2 * t4 + e;
          bool oka = key < key_end, okb = key < key_end;
          if (MODE == MODE_HIST && D.causal) {
            oka = oka && key <= qa_t;
            okb = okb && key <= qb_t;
          }
          s[nt][e] = oka ? s[nt][e] * sc : -INFINITY;
          s[nt][2 + e] = okb ? s[nt][2 + e] * sc : -INFINITY;
          mxa = fmaxf(mxa, s[nt][e]);
          mxb = fmaxf(mxb, s[nt][2 + e]);
        }
      }
      mxa = fmaxf(mxa, __shfl_xor_sync(0xffffffffu, mxa, 1));
      mxa = fmaxf(mxa, __shfl_xor_sync(0xffffffffu, mxa, 2));
      mxb = fmaxf(mxb, __shfl_xor_sync(0xffffffffu, mxb, 1));
      mxb = fmaxf(mxb, __shfl_xor_sync(0xffffffffu, mxb, 2));
      const float mna = fmaxf(m_a, mxa), mnb = fmaxf(m_b, mxb);
      const float ba = (mna == -INFINITY) ? 0.f : mna, bb = (mnb == -INFINITY) ? 0.f : mnb;
      const float alpha_a = exp2f(m_a - ba), alpha_b = exp2f(m_b - bb);
      m_a = mna;
      m_b = mnb;
      float suma = 0.f, sumb = 0.f;
#pragma unroll
      for (int nt = 0; nt < 8; ++nt) {
        s[nt][0] = exp2f(s[nt][0] - ba);
        s[nt][1] = exp2f(s[nt][1] - ba);
        s[nt][2] = exp2f(s[nt][2] - bb);
        s[nt][3] = exp2f(s[nt][3] - bb);
        suma += s[nt][0] + s[nt][1];
        sumb += s[nt][2] + s[nt][3];
      }
      l_a = l_a * alpha_a + suma;   // quad-partial sums; reduced at the end
      l_b = l_b * alpha_b + sumb;
#pragma unroll
      for (int nt = 0; nt < DH / 8; ++nt) {
        o[nt][0] *= alpha_a; o[nt][1] *= alpha_a;
        o[nt][2] *= alpha_b; o[nt][3] *= alpha_b;
      }
      // O += P V : k over 64 keys in 4 steps of 16, n over DH in tiles of 8
#pragma unroll
      for (int ks = 0; ks < 4; ++ks) {
        uint32_t pa[4];
        pa[0] = pack_bf16(s[2 * ks][0], s[2 * ks][1]);
        pa[1] = pack_bf16(s[2 * ks][2], s[2 * ks][3]);
        pa[2] = pack_bf16(s[2 * ks + 1][0], s[2 * ks + 1][1]);
        pa[3] = pack_bf16(s[2 * ks + 1][2], s[2 * ks + 1][3]);
#pragma unroll
        for (int np = 0; np < DH / 16; ++np) {
          uint32_t bv[4];
          const int krow = ks * 16 + (lane & 7) + ((lane >> 3) & 1) * 8;
          const int ncol = np * 16 + (lane >> 4) * 8;
          ldsm_x4_trans(bv, &Vs[buf][krow][ncol]);
          mma16816(o[2 * np], pa, bv[0], bv[1]);
          mma16816(o[2 * np + 1], pa, bv[2], bv[3]);
        }
      }
    }
    __syncthreads();
  }

  // ---- finalize: reduce the quad-partial row sums, normalise, store ----
  l_a += __shfl_xor_sync(0xffffffffu, l_a, 1);
  l_a += __shfl_xor_sync(0xffffffffu, l_a, 2);
  l_b += __shfl_xor_sync(0xffffffffu, l_b, 1);
  l_b += __shfl_xor_sync(0xffffffffu, l_b, 2);
  const float ia = (l_a > 0.f) ? 1.f / l_a : 0.f, ib = (l_b > 0.f) ? 1.f / l_b : 0.f;
  const int rows_to_write = (MODE == MODE_SUMI) ? n_rows : min(ROWS, D.nk - tile0);
  bf16* oa = a.O + (row_base + ra) * D.d + head * DH;
  bf16* ob = a.O + (row_base + rb) * D.d + head * DH;
#pragma unroll
  for (int nt = 0; nt < DH / 8; ++nt) {
    const int c = nt * 8 + 2 * t4;
    if (ra < rows_to_write)
      *reinterpret_cast<uint32_t*>(oa + c) = va ? pack_bf16(o[nt][0] * ia, o[nt][1] * ia) : 0u;
    if (rb < rows_to_write)
      *reinterpret_cast<uint32_t*>(ob + c) = vb ? pack_bf16(o[nt][2] * ib, o[nt][3] * ib) : 0u;
  }
}

}  // namespace am

bool attn_mma_supported(int dh) { return dh == 16 || dh == 32 || dh == 64; }

void launch_attn_sumi_mma(const bf16* QKV, const int64_t* cand_off, const int* wave_slot, const int* wave_r, int U,
                          int Mmax, const bf16* pool, const int* ptab, const int* vlen_all, const float* tau, bf16* O,
                          int k, int l, const Dims& D, cudaStream_t s) {
  am::Args a{QKV, cand_off, wave_slot, wave_r, pool, ptab, vlen_all, tau, O, k, l, D};
  dim3 grid(U, D.h, (Mmax + am::ROWS - 1) / am::ROWS);
  if (D.dh == 16) am::k_attn<16, am::MODE_SUMI><<<grid, am::THREADS, 0, s>>>(a);
  else if (D.dh == 32) am::k_attn<32, am::MODE_SUMI><<<grid, am::THREADS, 0, s>>>(a);
  else am::k_attn<64, am::MODE_SUMI><<<grid, am::THREADS, 0, s>>>(a);
}

void launch_attn_hist_mma(const bf16* Q, const int* wave_slot, const int* wave_r, int U, const bf16* pool,
                          const int* ptab, const int* vlen_all, const float* tau, bf16* O, int k, int l, const Dims& D,
                          cudaStream_t s) {
  am::Args a{Q, nullptr, wave_slot, wave_r, pool, ptab, vlen_all, tau, O, k, l, D};
  dim3 grid(U, D.h, (D.nk + am::ROWS - 1) / am::ROWS);
  if (D.dh == 16) am::k_attn<16, am::MODE_HIST><<<grid, am::THREADS, 0, s>>>(a);
  else if (D.dh == 32) am::k_attn<32, am::MODE_HIST><<<grid, am::THREADS, 0, s>>>(a);
  else am::k_attn<64, am::MODE_HIST><<<grid, am::THREADS, 0, s>>>(a);
}

}  // namespace climber
