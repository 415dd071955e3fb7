#include <algorithm>
#include <type_traits>
#include <mutex>
#include <map>
#include <set>
#include <string>
#include <cstdio>
// Non-GEMM kernels of the SUMI hot path (SURVEY §8(a) rows a1, a2, a4/a5
// attention, a6 head) and the SIMT GEMM used by the fp32 verification build.
//
// Every kernel is templated on the storage type T of activations / K/V pages
// (bf16 production path, fp32 verification build); statistics,
// softmax and residuals are fp32 in both.
#include "kernels.cuh"
#include "tc_util.cuh"

namespace climber {

static std::mutex g_launch_mu;
static std::string g_launch_err;
static std::map<std::pair<const void*, int>, int> g_attr_done;  // (kernel, device) -> bytes set

void note_launch_error(const char* what) {
  std::lock_guard<std::mutex> g(g_launch_mu);
  if (g_launch_err.empty()) g_launch_err = what;
}

bool take_launch_error(char* msg, int cap) {
  std::lock_guard<std::mutex> g(g_launch_mu);
  if (g_launch_err.empty()) return false;
  snprintf(msg, cap, "%s", g_launch_err.c_str());
  g_launch_err.clear();
  return true;
}

void ensure_smem_attr(const void* kern, int bytes) {
  int dev = 0;
  cudaGetDevice(&dev);
  std::lock_guard<std::mutex> g(g_launch_mu);
  int& have = g_attr_done[{kern, dev}];  // 0 when new; raised when a launch needs more
  if (bytes > have) {
    cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, bytes);
    have = bytes;
  }
}


// ===========================================================================
// a1: validation + multi-scale sequence extraction (Eq. 2)
// One CTA of 256 threads per user.  All threads validate the events
// (coalesced sweep); then the events are taken from the newest in
// super-chunks of 256 x EXT_EPT: thread t owns EXT_EPT consecutive events
// (thread 0 the newest) and counts its matches for every strategy; a
// block-wide exclusive scan (newest first) of the packed counts gives each
// match its rank from the newest, and matches of rank < n_k go to slot
// n_k - 1 - rank, so the most recent n_k matches land in canonical left-padded
// slots n_k-1, n_k-2, ... (G11, G12).  The sweep stops once every strategy
// has n_k matches: a user costs (events needed / 4096) steps of one coalesced
// load and one scan each.
// ===========================================================================
constexpr int EXT_EPT = 16;
constexpr int EXT_THREADS = 256;

__device__ __forceinline__ void ext_scan(uint64_t& a, uint64_t& b, uint64_t* sh, uint64_t& ta, uint64_t& tb) {
  // exclusive scan over the block of two packed vectors (4 x 16-bit counters each)
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  uint64_t ia = a, ib = b;
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    const uint64_t xa = __shfl_up_sync(0xffffffffu, ia, o), xb = __shfl_up_sync(0xffffffffu, ib, o);
    if (lane >= o) { ia += xa; ib += xb; }
  }
  if (lane == 31) { sh[2 * warp] = ia; sh[2 * warp + 1] = ib; }
  __syncthreads();
  uint64_t wa = 0, wb = 0;
  ta = 0; tb = 0;
#pragma unroll
  for (int w = 0; w < EXT_THREADS / 32; ++w) {
    if (w < warp) { wa += sh[2 * w]; wb += sh[2 * w + 1]; }
    ta += sh[2 * w]; tb += sh[2 * w + 1];
  }
  __syncthreads();
  a = wa + ia - a;
  b = wb + ib - b;
}
__device__ __forceinline__ int ext_get(uint64_t a, uint64_t b, int k) {
  return (int)(((k < 4 ? a : b) >> (16 * (k & 3))) & 0xFFFF);
}

__global__ void __launch_bounds__(EXT_THREADS) k_extract(const int32_t* __restrict__ item, const uint8_t* __restrict__ action,
                          const uint8_t* __restrict__ scenario, const int64_t* __restrict__ ts,
                          const int64_t* __restrict__ ev_off, const int* __restrict__ wave_slot,
                          const unsigned long long* __restrict__ amask,
                          const unsigned long long* __restrict__ smask, int* __restrict__ idx_all,
                          int* __restrict__ vlen_all, int* __restrict__ bad_all, int* __restrict__ err,
                          Dims D) {
  __shared__ uint64_t sh[2 * EXT_THREADS / 32];
  __shared__ unsigned long long sam[8], ssm[8];
  const int u = blockIdx.x;
  const long long s = ev_off[u], e = ev_off[u + 1];
  const int slot = wave_slot[u];
  int flags = 0;
  // validation sweep, 8 independent events per thread per step (the loads of a
  // step are all in flight together: the sweep is latency-, not issue-bound)
  constexpr int VU = 8;
  for (long long i0 = s + threadIdx.x; i0 < e; i0 += (long long)VU * EXT_THREADS) {
    int it[VU];
    unsigned ac[VU], sc[VU];
    long long t1[VU], t0[VU];
#pragma unroll
    for (int q = 0; q < VU; ++q) {
      const long long i = i0 + (long long)q * EXT_THREADS;
      const bool in = i < e;
      it[q] = in ? item[i] : 0;
      ac[q] = in ? action[i] : 0u;
      sc[q] = in ? scenario[i] : 0u;
      t1[q] = in ? ts[i] : 0;
      t0[q] = (in && i > s) ? ts[i - 1] : t1[q];
    }
#pragma unroll
    for (int q = 0; q < VU; ++q) {
      if (it[q] < 0 || it[q] >= D.V || ac[q] >= (unsigned)D.A || sc[q] >= (unsigned)D.R) flags |= ERR_RANGE;
      if (t1[q] < t0[q]) flags |= ERR_UNSORTED;
    }
  }
  if (threadIdx.x < D.Nb) {
    sam[threadIdx.x] = amask[threadIdx.x];
    ssm[threadIdx.x] = smask[threadIdx.x];
  }
  int any = __syncthreads_or(flags);
  if (flags) atomicOr(err, flags);
  if (threadIdx.x == 0) bad_all[slot] = any ? 1 : 0;

  int* idx_u = idx_all + (long long)slot * D.Nb * D.nk;
  int found[8] = {0, 0, 0, 0, 0, 0, 0, 0};  // matches so far per strategy (block-uniform)
  for (long long seg_end = e; seg_end > s; seg_end -= (long long)EXT_THREADS * EXT_EPT) {
    bool done = true;
#pragma unroll
    for (int k = 0; k < 8; ++k)
      if (k < D.Nb && found[k] < D.nk) done = false;
    if (done) break;
    const long long hi = seg_end - (long long)threadIdx.x * EXT_EPT;  // this thread: events [lo, hi)
    const long long lo = hi - EXT_EPT;
    uint8_t ac[EXT_EPT], sc[EXT_EPT];
#pragma unroll
    for (int q = 0; q < EXT_EPT; ++q) {  // q = 0 is the newest of the thread's events
      const long long i = hi - 1 - q;
      const bool in = i >= s && i >= lo;
      ac[q] = in ? action[i] : 0xFF;
      sc[q] = in ? scenario[i] : 0xFF;
    }
    uint64_t ca = 0, cb = 0;
#pragma unroll
    for (int k = 0; k < 8; ++k) {
      if (k >= D.Nb) break;
      const unsigned long long am = sam[k], sm = ssm[k];
      int c = 0;
#pragma unroll
      for (int q = 0; q < EXT_EPT; ++q)
        c += (ac[q] < 64 && sc[q] < 64 && ((am >> ac[q]) & 1ull) && ((sm >> sc[q]) & 1ull)) ? 1 : 0;
      if (k < 4) ca |= (uint64_t)c << (16 * k);
      else cb |= (uint64_t)c << (16 * (k - 4));
    }
    uint64_t pa = ca, pb = cb, ta, tb;
    ext_scan(pa, pb, sh, ta, tb);
#pragma unroll
    for (int k = 0; k < 8; ++k) {
      if (k >= D.Nb) break;
      int rank = found[k] + ext_get(pa, pb, k);
      if (rank < D.nk) {
        const unsigned long long am = sam[k], sm = ssm[k];
        int* idx = idx_u + (long long)k * D.nk;
#pragma unroll
        for (int q = 0; q < EXT_EPT; ++q) {
          const bool ok = ac[q] < 64 && sc[q] < 64 && ((am >> ac[q]) & 1ull) && ((sm >> sc[q]) & 1ull);
          if (ok) {
            if (rank < D.nk) idx[D.nk - 1 - rank] = (int)(hi - 1 - q - s);
            ++rank;
          }
        }
      }
      found[k] += ext_get(ta, tb, k);
    }
  }
  __syncthreads();
  for (int k = 0; k < D.Nb; ++k) {
    const int v = min(found[k], D.nk);
    int* idx = idx_u + (long long)k * D.nk;
    for (int p = threadIdx.x; p < D.nk - v; p += blockDim.x) idx[p] = -1;
    if (threadIdx.x == 0) vlen_all[(long long)slot * D.Nb + k] = v;
    if (D.hage && v > 0) {  // relative bias: age of history token p at the request time (G6e:
      __syncthreads();      // the request time is the last event's timestamp)
      int* hage = D.hage + ((long long)slot * D.Nb + k) * D.nk;
      const long long t_req = ts[e - 1];  // v > 0 implies e > s
      for (int p = threadIdx.x; p < v; p += blockDim.x) {
        const long long age = t_req - ts[s + idx[D.nk - v + p]];
        hage[p] = age < 0 ? 0 : (age > 2147483647LL ? 2147483647 : (int)age);
      }
    }
  }
}

// Relative bias of the candidate rows (Eq. 3 f_b, NEXT-1): a candidate sits at
// position v and time t_req, so its bias over history key j,
// b_pos[bucket_pos(v - j)] + b_time[bucket_time(t_req - t_j)], is the same for
// every candidate of the request: computed once per (user, layer, block, head)
// at encode.  grid (U, L * Nb * h), block 128 over the keys.
__global__ void k_cand_bias(const int* __restrict__ wave_slot, const int* __restrict__ wave_r,
                            const int* __restrict__ vlen_all, Dims D) {
  const int u = blockIdx.x;
  const int head = blockIdx.y % D.h, k = (blockIdx.y / D.h) % D.Nb, l = blockIdx.y / (D.h * D.Nb);
  const int slot = wave_slot[u], r = wave_r[u];
  const int v = vlen_all[(long long)slot * D.Nb + k];
  const long long row = bias_row(D, l, k, r, head);
  const float* bp = D.bpos + row * NB_POS;
  const float* bt = D.btime + row * NB_TIME;
  const int* age = D.hage + ((long long)slot * D.Nb + k) * D.nk;
  float* out = D.cbias + ((((long long)slot * D.L + l) * D.Nb + k) * D.h + head) * D.nk;
  for (int j = threadIdx.x; j < D.nk; j += blockDim.x)   // t_req - t_j = age_j
    out[j] = j < v ? bp[bucket_pos(v - j)] + bt[bucket_time32(age[j])] : 0.f;
}

// Block-parallel fusion input (NEXT-2): from the gathered fp32 block outputs
// C [rows][d], the bf16 copy and the per-128-column partial sums of squares
// that the RESID_NORM GEMM epilogue would have written, in the same order
// (32-column chunks, each 4 columns as fma(c3, fma(c2, fma(c1, fma(c0 ...)))))
// so the fused scores are bit-identical to the single-GPU path.
__global__ void k_row_prep(const float* __restrict__ C, bf16* __restrict__ Cb, float* __restrict__ part,
                           long long rows, int d, int pld) {
  const long long t = (long long)blockIdx.x * blockDim.x + threadIdx.x;  // (row, 128-column group)
  if (t >= rows * pld) return;
  const long long row = t / pld;
  const int g = (int)(t % pld);
  const int w = d < 128 ? d : 128;
  const float* x = C + row * d + g * w;
  bf16* xb = Cb + row * d + g * w;
  float ss = 0.f;
  for (int c = 0; c < w; c += 4) {
    const float4 v = *reinterpret_cast<const float4*>(x + c);
    ss = fmaf(v.x, v.x, fmaf(v.y, v.y, fmaf(v.z, v.z, fmaf(v.w, v.w, ss))));
    __nv_bfloat162 a = __floats2bfloat162_rn(v.x, v.y), b = __floats2bfloat162_rn(v.z, v.w);
    *reinterpret_cast<__nv_bfloat162*>(xb + c) = a;
    *reinterpret_cast<__nv_bfloat162*>(xb + c + 2) = b;
  }
  part[row * pld + g] = ss;
}

void launch_row_prep(const float* C, bf16* Cb, float* part, long long rows, int d, int pld, cudaStream_t s) {
  const long long n = rows * pld;
  k_row_prep<<<(unsigned)((n + 127) / 128), 128, 0, s>>>(C, Cb, part, rows, d, pld);
}

// Incremental cache update: flags[k] = 1 if an appended event e in [n0, n1)
// passes strategy a_k's filter (Eq. 2), i.e. S_k changed.
__global__ void k_append_flags(const uint8_t* __restrict__ action, const uint8_t* __restrict__ scenario, long long n0,
                               long long n1, const unsigned long long* __restrict__ amask,
                               const unsigned long long* __restrict__ smask, int* __restrict__ flags, Dims D) {
  for (long long i = n0 + (long long)blockIdx.x * blockDim.x + threadIdx.x; i < n1; i += (long long)gridDim.x * blockDim.x) {
    const unsigned a = action[i], sc = scenario[i];
    for (int k = 0; k < D.Nb; ++k)
      if (a < 64 && sc < 64 && ((amask[k] >> a) & 1ull) && ((smask[k] >> sc) & 1ull)) flags[k] = 1;
  }
}

void launch_append_flags(const uint8_t* action, const uint8_t* scenario, long long n0, long long n1,
                         const unsigned long long* amask, const unsigned long long* smask, int* flags, const Dims& D,
                         cudaStream_t s) {
  const long long n = n1 - n0;
  const int blocks = (int)((n + 255) / 256 < 148 ? (n + 255) / 256 : 148);
  k_append_flags<<<blocks > 0 ? blocks : 1, 256, 0, s>>>(action, scenario, n0, n1, amask, smask, flags, D);
}

// CLIMBER_SYNC_CHECK=1: flag non-finite scores (climber_status E_NUMERIC)
__global__ void k_check_finite(const float* __restrict__ x, long long n, int* __restrict__ err) {
  bool bad = false;
  for (long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (long long)gridDim.x * blockDim.x)
    bad |= !isfinite(x[i]);
  if (__syncthreads_or(bad) && threadIdx.x == 0) atomicOr(err, ERR_NUMERIC);
}

void launch_check_finite(const float* x, long long n, int* err, cudaStream_t s) {
  const long long b = (n + 255) / 256;
  k_check_finite<<<(unsigned)(b < 592 ? (b > 0 ? b : 1) : 592), 256, 0, s>>>(x, n, err);
}

void launch_cand_bias(const int* wave_slot, const int* wave_r, int U, const int* vlen_all, const Dims& D,
                      cudaStream_t s) {
  k_cand_bias<<<dim3(U, D.L * D.Nb * D.h), 128, 0, s>>>(wave_slot, wave_r, vlen_all, D);
}

// ===========================================================================
// a2: embedding gather-sum (G10).  Warp per row, 8 elems/lane.
// History row (u, t) of block k: E_item + E_act + E_scn of the t-th extracted
// event, zero for pad rows (t >= v).  Right-padded internal layout.
// ===========================================================================
template <typename T>
__global__ void k_embed_hist(const int32_t* __restrict__ item, const uint8_t* __restrict__ action,
                             const uint8_t* __restrict__ scenario, const int64_t* __restrict__ ev_off,
                             const int* __restrict__ wave_slot, const int* __restrict__ idx_all,
                             const int* __restrict__ vlen_all, const int* __restrict__ bad_all,
                             const T* __restrict__ e_item, const T* __restrict__ e_act,
                             const T* __restrict__ e_scn, float* __restrict__ X, T* __restrict__ Xb,
                             float* __restrict__ part, int pld, long long rows, int k, Dims D) {
  // Xb / part (fused-norm bf16 path): bf16 copy of the row and its sum of squares
  // (part[row][0]; the other pld-1 partial slots are 0) for the first GEMM's folded RMSNorm
  long long row = ((long long)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  int lane = threadIdx.x & 31;
  if (row >= rows) return;
  int u = (int)(row / D.nk), t = (int)(row % D.nk);
  int slot = wave_slot[u];
  int v = vlen_all[(long long)slot * D.Nb + k];
  float* out = X + row * D.d;
  if (t >= v) {
    float z[8] = {0, 0, 0, 0, 0, 0, 0, 0};
    for (int c = lane * 8; c < D.d; c += 256) {
      store8(out + c, z);
      if (Xb) store8(Xb + row * D.d + c, z);
    }
    if (part && lane < pld) part[row * pld + lane] = 0.f;
    return;
  }
  long long ev = ev_off[u] + idx_all[((long long)slot * D.Nb + k) * D.nk + (D.nk - v + t)];
  int it = item[ev], a = action[ev], sc = scenario[ev];
  bool bad = bad_all[slot] != 0;
  if (it < 0 || it >= D.V) it = 0;
  if (a >= D.A) a = 0;
  if (sc >= D.R) sc = 0;
  float ss = 0.f;
  for (int c = lane * 8; c < D.d; c += 256) {
    float x[8], y[8], z[8];
    load8(e_item + (long long)it * D.d + c, x);
    load8(e_act + (long long)a * D.d + c, y);
    load8(e_scn + (long long)sc * D.d + c, z);
#pragma unroll
    for (int i = 0; i < 8; ++i) {
      x[i] = bad ? __int_as_float(0x7fc00000) : x[i] + y[i] + z[i];
      ss = fmaf(x[i], x[i], ss);
    }
    store8(out + c, x);
    if (Xb) store8(Xb + row * D.d + c, x);
  }
  if (part) {
    ss = warp_sum(ss);
    if (lane < pld) part[row * pld + lane] = (lane == 0) ? ss : 0.f;
  }
}

// Binary search: wave user owning pair p, given cand_off[0..U] (wave-relative).
__device__ __forceinline__ int pair_user(const int64_t* cand_off, int U, long long p) {
  int lo = 0, hi = U - 1;
  while (lo < hi) {
    int mid = (lo + hi + 1) >> 1;
    if (cand_off[mid] <= p) lo = mid; else hi = mid - 1;
  }
  return lo;
}

// Candidate rows: c0 = E_item[item] + E_scn[r] (G10), replicated into the
// N_b block slots of the residual buffer C[p][k][d] (all blocks start from c0).
template <typename T>
__global__ void k_embed_cand(const int32_t* __restrict__ items, const int64_t* __restrict__ cand_off,
                             const int* __restrict__ wave_r, int U, long long P,
                             const T* __restrict__ e_item, const T* __restrict__ e_scn,
                             float* __restrict__ C, T* __restrict__ Cb, float* __restrict__ part, int pld,
                             int* __restrict__ err, Dims D) {
  long long p = ((long long)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  int lane = threadIdx.x & 31;
  if (p >= P) return;
  int u = pair_user(cand_off, U, p);
  int r = wave_r[u];
  int it = items[p];
  bool bad = it < 0 || it >= D.V;
  if (bad) {
    it = 0;
    if (lane == 0) atomicOr(err, ERR_RANGE);
  }
  float ss = 0.f;
  for (int c = lane * 8; c < D.d; c += 256) {
    float x[8], z[8];
    load8(e_item + (long long)it * D.d + c, x);
    load8(e_scn + (long long)r * D.d + c, z);
#pragma unroll
    for (int i = 0; i < 8; ++i) {
      x[i] = bad ? __int_as_float(0x7fc00000) : x[i] + z[i];
      ss = fmaf(x[i], x[i], ss);
    }
    for (int k = 0; k < D.Nb; ++k) {
      store8(C + (p * D.Nb + k) * D.d + c, x);
      if (Cb) store8(Cb + (p * D.Nb + k) * D.d + c, x);
    }
  }
  if (part) {
    ss = warp_sum(ss);
    for (int k = 0; k < D.Nb; ++k)
      if (lane < pld) part[(p * D.Nb + k) * pld + lane] = (lane == 0) ? ss : 0.f;
  }
}

// ===========================================================================
// RMSNorm (G7): out[row] = X[row] / sqrt(mean(X^2) + eps) * g.  Warp per row.
// ===========================================================================
template <typename T>
__global__ void k_rmsnorm(const float* __restrict__ X, long long ldx, const float* __restrict__ g,
                          T* __restrict__ out, long long ldo, long long rows, int d, float eps) {
  long long row = ((long long)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  int lane = threadIdx.x & 31;
  if (row >= rows) return;
  const float* x = X + row * ldx;
  float buf[4][8];
  float ss = 0.f;
#pragma unroll
  for (int j = 0; j < 4; ++j) {
    int c = (lane + 32 * j) * 8;
    if (c < d) {
      load8(x + c, buf[j]);
#pragma unroll
      for (int i = 0; i < 8; ++i) ss += buf[j][i] * buf[j][i];
    }
  }
  ss = warp_sum(ss);
  float rs = rsqrtf(ss / (float)d + eps);
#pragma unroll
  for (int j = 0; j < 4; ++j) {
    int c = (lane + 32 * j) * 8;
    if (c < d) {
      float gg[8], y[8];
      load8(g + c, gg);
#pragma unroll
      for (int i = 0; i < 8; ++i) y[i] = buf[j][i] * rs * gg[i];
      store8(out + row * ldo + c, y);
    }
  }
}

// fp32 -> T copy (vec(G) for the squeeze-and-excitation GEMM).
template <typename T>
__global__ void k_convert(const float* __restrict__ X, T* __restrict__ out, long long n8) {
  long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n8) return;
  float v[8];
  load8(X + i * 8, v);
  store8(out + i * 8, v);
}

// Eq. 4 gate product fused with the a6 head (G18):
//   score[p] = sum_c (G[p][c] * gate[p][c]) * w_head[c] + b_head,
// gate = sigmoid(f_gate(G)) from the SE GEMM epilogue.  Warp per row, fixed order.
__global__ void k_head(const float* __restrict__ Y, const float* __restrict__ gate, const float* __restrict__ w,
                       float b, float* __restrict__ scores, long long P, int D) {
  long long p = ((long long)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  int lane = threadIdx.x & 31;
  if (p >= P) return;
  float acc = 0.f;
  for (int c = lane * 8; c < D; c += 256) {
    float y[8], gg[8], ww[8];
    load8(Y + p * D + c, y);
    load8(gate + p * D + c, gg);
    load8(w + c, ww);
#pragma unroll
    for (int i = 0; i < 8; ++i) acc = fmaf(y[i] * gg[i], ww[i], acc);
  }
  acc = warp_sum(acc);
  if (lane == 0) scores[p] = acc + b;
}

// ===========================================================================
// Attention (Eq. 3 with f_b = 0, G2/G3): softmax(q.k / (sqrt(d_h) tau)).
// SIMT flash form: one thread owns one query row (q, o in registers), K/V
// chunks of KC keys are staged in shared memory (broadcast reads), online
// softmax in base 2 with fp32 statistics.
// ===========================================================================
constexpr int KC = 32;
constexpr float LOG2E = 1.4426950408889634f;

template <typename T, int DH>
__device__ __forceinline__ void load_kv_chunk(float (*Ks)[DH + 1], float (*Vs)[DH + 1], const T* pool,
                                              const int* pages, int t0, int nkeys, int head, int d) {
  // nkeys <= KC tokens starting at t0; a chunk never crosses a page (PAGE % KC == 0)
  const int page = pages[t0 / PAGE];
  const T* kb = pool + page_elem_offset(page, 0, head, t0 % PAGE, 0, d, DH);
  const T* vb = pool + page_elem_offset(page, 1, head, t0 % PAGE, 0, d, DH);
  for (int i = threadIdx.x; i < KC * DH; i += blockDim.x) {
    int j = i / DH, c = i % DH;
    float kv = 0.f, vv = 0.f;
    if (j < nkeys) {
      kv = to_f(kb[(long long)j * d + c]);
      vv = to_f(vb[(long long)j * d + c]);
    }
    Ks[j][c] = kv;
    Vs[j][c] = vv;
  }
}

// with a relative bias: bias(j) is the (already log2-scaled) bias of key j of the chunk
template <int DH, typename FB>
__device__ __forceinline__ void online_chunk_b(const float (*Ks)[DH + 1], const float (*Vs)[DH + 1],
                                               const float* q, float* o, float& m, float& l, int jmax, FB bias) {
  // keys j < jmax of the staged chunk are visible to this thread
  if (jmax <= 0) return;
  float s[KC];
  float cmax = -INFINITY;
#pragma unroll
  for (int j = 0; j < KC; ++j) {
    float acc = 0.f;
#pragma unroll
    for (int c = 0; c < DH; ++c) acc = fmaf(q[c], Ks[j][c], acc);
    s[j] = (j < jmax) ? acc + bias(j) : -INFINITY;
    cmax = fmaxf(cmax, s[j]);
  }
  float mn = fmaxf(m, cmax);
  float alpha = exp2f(m - mn);  // m = -inf -> 0
  l *= alpha;
#pragma unroll
  for (int c = 0; c < DH; ++c) o[c] *= alpha;
#pragma unroll
  for (int j = 0; j < KC; ++j) {
    float p = exp2f(s[j] - mn);
    l += p;
#pragma unroll
    for (int c = 0; c < DH; ++c) o[c] = fmaf(p, Vs[j][c], o[c]);
  }
  m = mn;
}

template <int DH>
__device__ __forceinline__ void online_chunk(const float (*Ks)[DH + 1], const float (*Vs)[DH + 1],
                                             const float* q, float* o, float& m, float& l, int jmax) {
  online_chunk_b<DH>(Ks, Vs, q, o, m, l, jmax, [](int) { return 0.f; });
}


// SUMI candidate attention: candidate (u, m) of block k,
// layer l attends to the v cached history keys of its user/block/layer and to
// itself (k_self, v_self) only.  grid (U, h, ceil(Mmax/128)), block 128.
template <typename T, int DH>
__global__ void __launch_bounds__(128) k_attn_sumi(const T* __restrict__ QKV, const int64_t* __restrict__ cand_off,
                                                   const int* __restrict__ wave_slot, const int* __restrict__ wave_r,
                                                   const T* __restrict__ pool, const int* __restrict__ ptab,
                                                   const int* __restrict__ vlen_all, const float* __restrict__ tau,
                                                   T* __restrict__ O, int k, int l, Dims D) {
  __shared__ float Ks[KC][DH + 1];
  __shared__ float Vs[KC][DH + 1];
  const int u = blockIdx.x, head = blockIdx.y;
  const long long p0 = cand_off[u], p1 = cand_off[u + 1];
  const long long p = p0 + (long long)blockIdx.z * blockDim.x + threadIdx.x;
  if (p0 + (long long)blockIdx.z * blockDim.x >= p1) return;  // whole CTA idle (uniform)
  const bool active = p < p1;
  const int slot = wave_slot[u];
  const int r = wave_r[u];
  const int v = vlen_all[(long long)slot * D.Nb + k];
  const int* pages = ptab + (((long long)slot * D.Nb + k) * D.L + l) * D.ppb;
  const float sc = LOG2E / (sqrtf((float)DH) * tau[((l * D.Nb + k) * D.R + r) * D.h + head]);

  float q[DH], o[DH];
  float m = -INFINITY, lsum = 0.f;
  if (active) {
    const T* row = QKV + p * (3LL * D.d);
    float ks[DH];
#pragma unroll
    for (int c = 0; c < DH; c += 8) {
      load8(row + head * DH + c, q + c);
      load8(row + D.d + head * DH + c, ks + c);
      load8(row + 2 * D.d + head * DH + c, o + c);
    }
    float ss = 0.f;
#pragma unroll
    for (int c = 0; c < DH; ++c) {
      q[c] *= sc;
      ss = fmaf(q[c], ks[c], ss);
    }
    if (D.bpos) {  // self: position offset 0, time delta 0
      const long long br = bias_row(D, l, k, r, head);
      ss += sc * (D.bpos[br * NB_POS + bucket_pos(0)] + D.btime[br * NB_TIME + bucket_time(0)]);
    }
    m = ss;      // self term first: weight exp2(0) = 1 on v_self
    lsum = 1.f;
  } else {
#pragma unroll
    for (int c = 0; c < DH; ++c) q[c] = o[c] = 0.f;
  }
  const float* cb = D.cbias ? D.cbias + ((((long long)slot * D.L + l) * D.Nb + k) * D.h + head) * D.nk : nullptr;
  for (int t0 = 0; t0 < v; t0 += KC) {
    int nkeys = min(KC, v - t0);
    __syncthreads();
    load_kv_chunk<T, DH>(Ks, Vs, pool, pages, t0, nkeys, head, D.d);
    __syncthreads();
    if (active) {
      if (cb) online_chunk_b<DH>(Ks, Vs, q, o, m, lsum, nkeys, [&](int j) { return sc * cb[t0 + j]; });
      else online_chunk<DH>(Ks, Vs, q, o, m, lsum, nkeys);
    }
  }
  if (active) {
    float inv = 1.f / lsum;
    T* out = O + p * D.d + head * DH;
#pragma unroll
    for (int c = 0; c < DH; c += 8) {
      float y[8];
#pragma unroll
      for (int i = 0; i < 8; ++i) y[i] = o[c + i] * inv;
      store8(out + c, y);
    }
  }
}

// History self-attention inside block k (Eq. 3 over S_k; causal G1 or
// bidirectional).  Query row t of user u attends keys j <= t (causal) or
// j < v.  Pad rows (t >= v) output zeros.  grid (U, h, nk/128), block 128.
template <typename T, int DH>
__global__ void __launch_bounds__(128) k_attn_hist(const T* __restrict__ Q, const int* __restrict__ wave_slot,
                                                   const int* __restrict__ wave_r, const T* __restrict__ pool,
                                                   const int* __restrict__ ptab, const int* __restrict__ vlen_all,
                                                   const float* __restrict__ tau, T* __restrict__ O, int k, int l,
                                                   Dims D) {
  __shared__ float Ks[KC][DH + 1];
  __shared__ float Vs[KC][DH + 1];
  const int u = blockIdx.x, head = blockIdx.y;
  const int t = blockIdx.z * blockDim.x + threadIdx.x;
  const int slot = wave_slot[u];
  const int r = wave_r[u];
  const int v = vlen_all[(long long)slot * D.Nb + k];
  const long long row = (long long)u * D.nk + t;
  const bool active = t < v;
  const int* pages = ptab + (((long long)slot * D.Nb + k) * D.L + l) * D.ppb;
  const float sc = LOG2E / (sqrtf((float)DH) * tau[((l * D.Nb + k) * D.R + r) * D.h + head]);
  float q[DH], o[DH];
  float m = -INFINITY, lsum = 0.f;
#pragma unroll
  for (int c = 0; c < DH; ++c) o[c] = 0.f;
  if (active) {
#pragma unroll
    for (int c = 0; c < DH; c += 8) load8(Q + row * D.d + head * DH + c, q + c);
#pragma unroll
    for (int c = 0; c < DH; ++c) q[c] *= sc;
  } else {
#pragma unroll
    for (int c = 0; c < DH; ++c) q[c] = 0.f;
  }
  const int tile_last = min(v, (int)(blockIdx.z + 1) * (int)blockDim.x) - 1;
  const int kend = D.causal ? tile_last + 1 : v;
  for (int t0 = 0; t0 < kend; t0 += KC) {
    int nkeys = min(KC, v - t0);
    __syncthreads();
    load_kv_chunk<T, DH>(Ks, Vs, pool, pages, t0, nkeys, head, D.d);
    __syncthreads();
    if (active) {
      int jmax = D.causal ? min(nkeys, t - t0 + 1) : nkeys;
      if (D.bpos) {  // relative bias of (row t, key t0 + j): offset and time delta
        const long long br = bias_row(D, l, k, r, head);
        const float* bp = D.bpos + br * NB_POS;
        const float* bt = D.btime + br * NB_TIME;
        const int* age = D.hage + ((long long)slot * D.Nb + k) * D.nk;
        const int at = age[t];   // t_t - t_j = age_j - age_t
        online_chunk_b<DH>(Ks, Vs, q, o, m, lsum, jmax, [&](int j) {
          return sc * (bp[bucket_pos(t - (t0 + j))] + bt[bucket_time32(age[t0 + j] - at)]);
        });
      } else {
        online_chunk<DH>(Ks, Vs, q, o, m, lsum, jmax);
      }
    }
  }
  T* out = O + row * D.d + head * DH;
  if (t < D.nk) {
    float inv = active ? 1.f / lsum : 0.f;
#pragma unroll
    for (int c = 0; c < DH; c += 8) {
      float y[8];
#pragma unroll
      for (int i = 0; i < 8; ++i) y[i] = o[c + i] * inv;
      store8(out + c, y);
    }
  }
}

// a5 fusion ATL attention (G16): the N_b tokens of one pair
// attend to each other (full visibility), temperature tau_f[r][head].
// One warp per (pair, head): 4 lanes per token (N_b <= 8), each lane owns
// d_h/4 dimensions of its token's q, k, v; K and V of the pair are staged in
// shared memory, scores are reduced over the 4 lanes with two shuffles.
// Memory: one read of the pair's Q, K, V head slices, one write of O.
template <typename T, int DH>
__global__ void __launch_bounds__(256) k_attn_fusion(const T* __restrict__ QKV, const int64_t* __restrict__ cand_off,
                                                     const int* __restrict__ wave_r, int U, long long P,
                                                     const float* __restrict__ tau_f, T* __restrict__ O, Dims D) {
  constexpr int PD = DH / 4;      // dims per lane (4, 8 or 16)
  constexpr int SEG = PD + 4;     // smem segment stride: the 4 parts land in distinct banks
  __shared__ __align__(16) float Ks[8][8][4 * SEG];
  __shared__ __align__(16) float Vs[8][8][4 * SEG];
  const int wib = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const long long gw = (long long)blockIdx.x * 8 + wib;  // (pair, head)
  if (gw >= P * D.h) return;
  const int head = (int)(gw % D.h);
  const long long p = gw / D.h;
  const int tok = lane >> 2, part = lane & 3;
  const bool act = tok < D.Nb;
  const int u = pair_user(cand_off, U, p);
  const int r = wave_r[u];
  const float sc = LOG2E / (sqrtf((float)DH) * tau_f[r * D.h + head]);
  const long long ld = 3LL * D.d;
  const T* row = QKV + (p * D.Nb + (act ? tok : 0)) * ld + head * DH + part * PD;
  float q[PD];
  float* ks = &Ks[wib][tok][part * SEG];
  float* vs = &Vs[wib][tok][part * SEG];
#pragma unroll
  for (int c = 0; c < PD; c += 4) {
    float x[8], y[8], z[8];
    if (PD >= 8 && c % 8 == 0) {
      if (act) {
        load8(row + c, x);
        load8(row + D.d + c, y);
        load8(row + 2 * D.d + c, z);
      } else {
#pragma unroll
        for (int i = 0; i < 8; ++i) x[i] = y[i] = z[i] = 0.f;
      }
#pragma unroll
      for (int i = 0; i < 8; ++i) q[c + i] = x[i] * sc;
      *reinterpret_cast<float4*>(ks + c) = make_float4(y[0], y[1], y[2], y[3]);
      *reinterpret_cast<float4*>(ks + c + 4) = make_float4(y[4], y[5], y[6], y[7]);
      *reinterpret_cast<float4*>(vs + c) = make_float4(z[0], z[1], z[2], z[3]);
      *reinterpret_cast<float4*>(vs + c + 4) = make_float4(z[4], z[5], z[6], z[7]);
    } else if (PD < 8) {
#pragma unroll
      for (int i = 0; i < 4; ++i) {
        q[c + i] = act ? to_f(row[c + i]) * sc : 0.f;
        ks[c + i] = act ? to_f(row[D.d + c + i]) : 0.f;
        vs[c + i] = act ? to_f(row[2 * D.d + c + i]) : 0.f;
      }
    }
  }
  __syncwarp();
  float s[8];
  float mx = -INFINITY;
#pragma unroll
  for (int j = 0; j < 8; ++j) {
    const float* kj = &Ks[wib][j][part * SEG];
    float acc = 0.f;
#pragma unroll
    for (int c = 0; c < PD; c += 4) {
      const float4 k4 = *reinterpret_cast<const float4*>(kj + c);
      acc = fmaf(q[c], k4.x, fmaf(q[c + 1], k4.y, fmaf(q[c + 2], k4.z, fmaf(q[c + 3], k4.w, acc))));
    }
    acc += __shfl_xor_sync(0xffffffffu, acc, 1);
    acc += __shfl_xor_sync(0xffffffffu, acc, 2);
    s[j] = (j < D.Nb) ? acc : -INFINITY;
    mx = fmaxf(mx, s[j]);
  }
  float l = 0.f;
#pragma unroll
  for (int j = 0; j < 8; ++j) {
    s[j] = (j < D.Nb) ? exp2f(s[j] - mx) : 0.f;
    l += s[j];
  }
  const float inv = 1.f / l;
  float o[PD];
#pragma unroll
  for (int c = 0; c < PD; ++c) o[c] = 0.f;
#pragma unroll
  for (int j = 0; j < 8; ++j) {
    const float* vj = &Vs[wib][j][part * SEG];
#pragma unroll
    for (int c = 0; c < PD; c += 4) {
      const float4 v4 = *reinterpret_cast<const float4*>(vj + c);
      o[c] = fmaf(s[j], v4.x, o[c]);
      o[c + 1] = fmaf(s[j], v4.y, o[c + 1]);
      o[c + 2] = fmaf(s[j], v4.z, o[c + 2]);
      o[c + 3] = fmaf(s[j], v4.w, o[c + 3]);
    }
  }
  if (act) {
    T* out = O + (p * D.Nb + tok) * D.d + head * DH + part * PD;
    if constexpr (PD % 8 == 0) {
#pragma unroll
      for (int c = 0; c < PD; c += 8) {
        float y[8];
#pragma unroll
        for (int i = 0; i < 8; ++i) y[i] = o[c + i] * inv;
        store8(out + c, y);
      }
    } else {
#pragma unroll
      for (int c = 0; c < PD; ++c) out[c] = from_f<T>(o[c] * inv);
    }
  }
}

// ===========================================================================
// Debug exports
// ===========================================================================
// Canonical SUMI mask of one handle: evaluated with
// sumi_visible(), the same key-range rule the attention kernels implement.
__global__ void k_debug_mask(const int* __restrict__ vlen_all, int slot, int M, uint8_t* __restrict__ mask,
                             Dims D) {
  const int T = D.nk + M;
  long long n = (long long)D.Nb * T * T;
  for (long long g = (long long)blockIdx.x * blockDim.x + threadIdx.x; g < n;
       g += (long long)gridDim.x * blockDim.x) {
    int k = (int)(g / ((long long)T * T));
    long long ij = g % ((long long)T * T);
    int i = (int)(ij / T), j = (int)(ij % T);
    int v = vlen_all[(long long)slot * D.Nb + k];
    mask[g] = sumi_visible(i, j, D.nk, v, D.causal) ? 1 : 0;
  }
}

template <typename T>
__global__ void k_debug_kv(const T* __restrict__ pool, const int* __restrict__ ptab,
                           const int* __restrict__ vlen_all, int slot, int k, int l, T* __restrict__ Kout,
                           T* __restrict__ Vout, Dims D) {
  int v = vlen_all[(long long)slot * D.Nb + k];
  const int* pages = ptab + (((long long)slot * D.Nb + k) * D.L + l) * D.ppb;
  long long n = (long long)v * D.d;
  for (long long g = (long long)blockIdx.x * blockDim.x + threadIdx.x; g < n;
       g += (long long)gridDim.x * blockDim.x) {
    int t = (int)(g / D.d), c = (int)(g % D.d);
    int head = c / D.dh, dim = c % D.dh;
    int page = pages[t / PAGE];
    Kout[g] = pool[page_elem_offset(page, 0, head, t % PAGE, dim, D.d, D.dh)];
    Vout[g] = pool[page_elem_offset(page, 1, head, t % PAGE, dim, D.d, D.dh)];
  }
}

// Mask probe (climber_debug_attn_probe): K = 0 and V[j] = one-hot on every
// page slot of one (user, block, layer), so that the production attention
// kernel, run on zero queries, gives every attended key weight 1/|set| and
// its output channel reveals which keys it read.  Head h maps key
// key_off + h (d_h - 1) + c to channel c < d_h - 1; channel d_h - 1 is left
// for the SUMI self term.  Every slot of the pages is written, pads included,
// so a kernel that reads past v_k shows it.
template <typename T>
__global__ void k_probe_pages(T* __restrict__ pool, const int* __restrict__ ptab, int slot, int k, int l,
                              int key_off, Dims D) {
  const int* pages = ptab + (((long long)slot * D.Nb + k) * D.L + l) * D.ppb;
  const long long n = (long long)D.ppb * PAGE * D.d;
  for (long long g = (long long)blockIdx.x * blockDim.x + threadIdx.x; g < n;
       g += (long long)gridDim.x * blockDim.x) {
    const int t = (int)(g / D.d), col = (int)(g % D.d);
    const int head = col / D.dh, c = col % D.dh;
    const int page = pages[t / PAGE];
    const bool hit = c < D.dh - 1 && t == key_off + head * (D.dh - 1) + c;
    pool[page_elem_offset(page, 0, head, t % PAGE, c, D.d, D.dh)] = T(0.f);
    pool[page_elem_offset(page, 1, head, t % PAGE, c, D.d, D.dh)] = T(hit ? 1.f : 0.f);
  }
}

// SUMI probe rows: q = k_self = 0, v_self = e_{d_h - 1} per head
template <typename T>
__global__ void k_probe_qkv(T* __restrict__ QKV, long long rows, Dims D) {
  const long long n = rows * 3 * D.d;
  for (long long g = (long long)blockIdx.x * blockDim.x + threadIdx.x; g < n;
       g += (long long)gridDim.x * blockDim.x) {
    const int col = (int)(g % (3 * D.d));
    QKV[g] = T((col >= 2 * D.d && (col - 2 * D.d) % D.dh == D.dh - 1) ? 1.f : 0.f);
  }
}

template <typename T>
void launch_probe_pages(T* pool, const int* ptab, int slot, int k, int l, int key_off, const Dims& D, cudaStream_t s) {
  k_probe_pages<T><<<296, 256, 0, s>>>(pool, ptab, slot, k, l, key_off, D);
}
template <typename T>
void launch_probe_qkv(T* QKV, long long rows, const Dims& D, cudaStream_t s) {
  k_probe_qkv<T><<<296, 256, 0, s>>>(QKV, rows, D);
}
template void launch_probe_pages<bf16>(bf16*, const int*, int, int, int, int, const Dims&, cudaStream_t);
template void launch_probe_pages<float>(float*, const int*, int, int, int, int, const Dims&, cudaStream_t);
template void launch_probe_qkv<bf16>(bf16*, long long, const Dims&, cudaStream_t);
template void launch_probe_qkv<float>(float*, long long, const Dims&, cudaStream_t);

// K/V slab export / import (multi-GPU candidate sharding): 16-byte copies of
// the handle's pages in page-table order, behind a 256-byte header.
constexpr int SLAB_MAGIC = 0x4B56534C;  // "KVSL"

__global__ void k_kv_export(const uint4* __restrict__ pool, const int* __restrict__ ptab, const int* __restrict__ vlen_all,
                            int slot, int per_slot, long long page_vec, int* __restrict__ hdr, uint4* __restrict__ body,
                            Dims D, int dtype, int r) {
  if (blockIdx.x == 0 && threadIdx.x == 0) {
    hdr[0] = SLAB_MAGIC; hdr[1] = 2; hdr[2] = D.Nb; hdr[3] = D.L; hdr[4] = D.ppb; hdr[5] = D.d; hdr[6] = dtype;
    hdr[7] = r;  // the handle's request scenario (for climber_kv_broadcast's receivers)
    for (int k = 0; k < D.Nb; ++k) hdr[8 + k] = vlen_all[(long long)slot * D.Nb + k];
    hdr[16] = D.hage != nullptr;  // version 2: relative-bias state (hage, cbias rows) follows the pages
  }
  const long long n = (long long)per_slot * page_vec;
  for (long long g = (long long)blockIdx.x * blockDim.x + threadIdx.x; g < n; g += (long long)gridDim.x * blockDim.x) {
    const long long i = g / page_vec, w = g % page_vec;
    body[g] = pool[(long long)ptab[(long long)slot * per_slot + i] * page_vec + w];
  }
}

__global__ void k_kv_import(uint4* __restrict__ pool, const int* __restrict__ ptab, int* __restrict__ vlen_all, int slot,
                            int per_slot, long long page_vec, const int* __restrict__ hdr, const uint4* __restrict__ body,
                            int* __restrict__ err, Dims D, int dtype) {
  const bool ok = hdr[0] == SLAB_MAGIC && hdr[1] == 2 && hdr[2] == D.Nb && hdr[3] == D.L && hdr[4] == D.ppb &&
                  hdr[5] == D.d && hdr[6] == dtype && hdr[16] == (D.hage != nullptr);
  if (!ok) {
    if (blockIdx.x == 0 && threadIdx.x == 0) {
      atomicOr(err, ERR_CONFIG);
      for (int k = 0; k < D.Nb; ++k) vlen_all[(long long)slot * D.Nb + k] = 0;
    }
    return;
  }
  if (blockIdx.x == 0 && threadIdx.x < D.Nb) vlen_all[(long long)slot * D.Nb + threadIdx.x] = hdr[8 + threadIdx.x];
  const long long n = (long long)per_slot * page_vec;
  for (long long g = (long long)blockIdx.x * blockDim.x + threadIdx.x; g < n; g += (long long)gridDim.x * blockDim.x) {
    const long long i = g / page_vec, w = g % page_vec;
    pool[(long long)ptab[(long long)slot * per_slot + i] * page_vec + w] = body[g];
  }
}

// Pipelined replication (climber_encode_user_bcast): the pages of one layer
// l of every block, [N_b][ppb] pages in that order, packed into / unpacked
// from one contiguous slab section with 16-byte copies.
__global__ void k_kv_layer_copy(uint4* __restrict__ pool, const int* __restrict__ ptab, int slot, int l,
                                long long page_vec, uint4* __restrict__ sec, int unpack, Dims D) {
  const long long n = (long long)D.Nb * D.ppb * page_vec;
  for (long long g = (long long)blockIdx.x * blockDim.x + threadIdx.x; g < n; g += (long long)gridDim.x * blockDim.x) {
    const long long i = g / page_vec, w = g % page_vec;
    const int k = (int)(i / D.ppb), pg = (int)(i % D.ppb);
    const long long at = (long long)ptab[(((long long)slot * D.Nb + k) * D.L + l) * D.ppb + pg] * page_vec + w;
    if (unpack) pool[at] = sec[g];
    else sec[g] = pool[at];
  }
}
void launch_kv_layer_copy(void* pool, const int* ptab, int slot, int l, long long page_bytes, void* sec, bool unpack,
                          const Dims& D, cudaStream_t s) {
  k_kv_layer_copy<<<296, 256, 0, s>>>((uint4*)pool, ptab, slot, l, page_bytes / 16, (uint4*)sec, unpack ? 1 : 0, D);
}

void launch_kv_export(const void* pool, const int* ptab, const int* vlen_all, int slot, int per_slot, long long page_bytes,
                      void* slab, const Dims& D, int dtype, int r, cudaStream_t s) {
  k_kv_export<<<592, 256, 0, s>>>((const uint4*)pool, ptab, vlen_all, slot, per_slot, page_bytes / 16, (int*)slab,
                                  (uint4*)((char*)slab + 256), D, dtype, r);
}

void launch_kv_import(void* pool, const int* ptab, int* vlen_all, int slot, int per_slot, long long page_bytes,
                      const void* slab, int* err, const Dims& D, int dtype, cudaStream_t s) {
  k_kv_import<<<592, 256, 0, s>>>((uint4*)pool, ptab, vlen_all, slot, per_slot, page_bytes / 16, (const int*)slab,
                                  (const uint4*)((const char*)slab + 256), err, D, dtype);
}

// Scatter the staged page-table rows of a call into the per-slot table.
__global__ void k_scatter_ptab(const int* __restrict__ staged, const int* __restrict__ slots, int B, int per,
                               int* __restrict__ ptab) {
  long long n = (long long)B * per;
  for (long long g = (long long)blockIdx.x * blockDim.x + threadIdx.x; g < n;
       g += (long long)gridDim.x * blockDim.x) {
    int b = (int)(g / per), i = (int)(g % per);
    ptab[(long long)slots[b] * per + i] = staged[g];
  }
}

// ===========================================================================
// SIMT GEMM (fp32 verification build; also a debug path for bf16):
// D[m][n] = sum_k A[m][k] B[n][k], 64x64 tile, BK = 16, 256 threads, 4x4 each.
// ===========================================================================
template <typename T>
__global__ void __launch_bounds__(256) k_gemm_simt(const T* __restrict__ A, long long lda, const T* __restrict__ B,
                                                   long long ldb, long long M, int N, int K, Epilogue e) {
  __shared__ float As[16][68];
  __shared__ float Bs[16][68];
  const int tx = threadIdx.x & 15, ty = threadIdx.x >> 4;
  const long long m0 = (long long)blockIdx.y * 64;
  const int n0 = blockIdx.x * 64;
  float acc[4][4] = {};
  for (int k0 = 0; k0 < K; k0 += 16) {
    for (int i = threadIdx.x; i < 64 * 16; i += 256) {
      int r = i / 16, c = i % 16;
      long long gm = m0 + r;
      int gn = n0 + r;
      As[c][r] = (gm < M) ? to_f(A[gm * lda + k0 + c]) : 0.f;
      Bs[c][r] = (gn < N) ? to_f(B[(long long)gn * ldb + k0 + c]) : 0.f;
    }
    __syncthreads();
#pragma unroll
    for (int kk = 0; kk < 16; ++kk) {
      float a[4], b[4];
#pragma unroll
      for (int i = 0; i < 4; ++i) {
        a[i] = As[kk][ty * 4 + i];
        b[i] = Bs[kk][tx * 4 + i];
      }
#pragma unroll
      for (int i = 0; i < 4; ++i)
#pragma unroll
        for (int j = 0; j < 4; ++j) acc[i][j] = fmaf(a[i], b[j], acc[i][j]);
    }
    __syncthreads();
  }
  const int n = n0 + tx * 4;
  if (n >= N) return;
#pragma unroll
  for (int i = 0; i < 4; ++i) {
    long long m = m0 + ty * 4 + i;
    if (m < M) epilogue_chunk<T, 4>(e, m, n, acc[i]);
  }
}

// ---------------------------------------------------------------------------
// launchers
// ---------------------------------------------------------------------------
static inline unsigned blocks_for(long long threads, int bs) { return (unsigned)((threads + bs - 1) / bs); }

void launch_extract(const EventsDev& ev, const int64_t* ev_off, const int* wave_slot, int U,
                    const unsigned long long* amask, const unsigned long long* smask, int* idx_all,
                    int* vlen_all, int* bad_all, int* err, const Dims& D, cudaStream_t s) {
  k_extract<<<U, EXT_THREADS, 0, s>>>(ev.item, ev.action, ev.scenario, ev.ts, ev_off, wave_slot, amask, smask, idx_all,
                              vlen_all, bad_all, err, D);
}

template <typename T>
void launch_embed_hist(const EventsDev& ev, const int64_t* ev_off, const int* wave_slot, int U, const int* idx_all,
                       const int* vlen_all, const int* bad_all, const T* e_item, const T* e_act, const T* e_scn,
                       float* X, T* Xb, float* part, int pld, int k, const Dims& D, cudaStream_t s) {
  long long rows = (long long)U * D.nk;
  k_embed_hist<T><<<blocks_for(rows * 32, 256), 256, 0, s>>>(ev.item, ev.action, ev.scenario, ev_off, wave_slot,
                                                           idx_all, vlen_all, bad_all, e_item, e_act, e_scn, X, Xb,
                                                           part, pld, rows, k, D);
}

template <typename T>
void launch_embed_cand(const int32_t* items, const int64_t* cand_off, const int* wave_r, int U, long long P,
                       const T* e_item, const T* e_scn, float* C, T* Cb, float* part, int pld, int* err,
                       const Dims& D, cudaStream_t s) {
  k_embed_cand<T><<<blocks_for(P * 32, 256), 256, 0, s>>>(items, cand_off, wave_r, U, P, e_item, e_scn, C, Cb, part,
                                                          pld, err, D);
}

template <typename T>
void launch_rmsnorm(const float* X, long long ldx, const float* g, T* out, long long ldo, long long rows, int d,
                    float eps, cudaStream_t s) {
  k_rmsnorm<T><<<blocks_for(rows * 32, 256), 256, 0, s>>>(X, ldx, g, out, ldo, rows, d, eps);
}

template <typename T>
void launch_convert(const float* X, T* out, long long n, cudaStream_t s) {
  k_convert<T><<<blocks_for(n / 8, 256), 256, 0, s>>>(X, out, n / 8);
}

void launch_head(const float* Y, const float* gate, const float* w, float b, float* scores, long long P, int Dse,
                 cudaStream_t s) {
  k_head<<<blocks_for(P * 32, 256), 256, 0, s>>>(Y, gate, w, b, scores, P, Dse);
}

template <typename T>
void launch_attn_sumi(const T* QKV, const int64_t* cand_off, const int* wave_slot, const int* wave_r, int U,
                      int Mmax, const T* pool, const int* ptab, const int* vlen_all, const float* tau, T* O, int k,
                      int l, const Dims& D, cudaStream_t s) {
  dim3 grid(U, D.h, (Mmax + 127) / 128);
#define CL_SUMI(DH) k_attn_sumi<T, DH><<<grid, 128, 0, s>>>(QKV, cand_off, wave_slot, wave_r, pool, ptab, vlen_all, tau, O, k, l, D)
  if (D.dh == 16) CL_SUMI(16);
  else if (D.dh == 32) CL_SUMI(32);
  else CL_SUMI(64);
#undef CL_SUMI
}

template <typename T>
void launch_attn_hist(const T* Q, const int* wave_slot, const int* wave_r, int U, const T* pool, const int* ptab,
                      const int* vlen_all, const float* tau, T* O, int k, int l, const Dims& D, cudaStream_t s) {
  dim3 grid(U, D.h, (D.nk + 127) / 128);
#define CL_HIST(DH) k_attn_hist<T, DH><<<grid, 128, 0, s>>>(Q, wave_slot, wave_r, pool, ptab, vlen_all, tau, O, k, l, D)
  if (D.dh == 16) CL_HIST(16);
  else if (D.dh == 32) CL_HIST(32);
  else CL_HIST(64);
#undef CL_HIST
}

// Fusion ATL attention, bf16 (G16): persistent CTAs, one candidate pair at a
// time, all heads.  The pair's N_b token rows of QKV (contiguous: rows
// p N_b .. p N_b + N_b - 1, 3 d bf16 each) arrive in shared memory by bulk
// async copies (one per row, into rows padded by 16 B so the 4-lane token
// groups hit distinct banks), double-buffered: the next pair streams in while
// this one is computed.  Every warp computes heads w, w + 8, ... (4 lanes per
// token, scores reduced over them with two shuffles); O is staged in shared
// memory and written back with coalesced 16-byte stores.  Traffic per pair:
// one read of 3 N_b d and one write of N_b d elements.
template <int DH>
__global__ void __launch_bounds__(256) k_attn_fusion_pair(const bf16* __restrict__ QKV,
                                                          const int64_t* __restrict__ cand_off,
                                                          const int* __restrict__ wave_r, int U, long long P,
                                                          const float* __restrict__ tau_f, bf16* __restrict__ O,
                                                          Dims D) {
  constexpr int PD = DH / 4;  // dims per lane
  extern __shared__ __align__(16) uint8_t fsm[];
  const int rs = 3 * D.d + 8;                       // token row stride (elements)
  const int ros = D.d + 8;
  bf16* sq0 = reinterpret_cast<bf16*>(fsm);          // [2][N_b][rs] double buffer
  bf16* so = sq0 + 2 * D.Nb * rs;                    // [N_b][ros] staged O
  uint64_t* bar = reinterpret_cast<uint64_t*>(so + D.Nb * ros);  // [2]
  const unsigned row_bytes = 3u * D.d * 2u;
  auto issue = [&](long long p, int b) {  // one thread: the pair's rows into buffer b
    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");  // after the generic reads of the buffer
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(tcu::smem_u32(&bar[b])),
                 "r"(row_bytes * D.Nb) : "memory");
    for (int t = 0; t < D.Nb; ++t)
      asm volatile(
          "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
              tcu::smem_u32(sq0 + (b * D.Nb + t) * rs)),
          "l"(QKV + (p * D.Nb + t) * 3LL * D.d), "r"(row_bytes), "r"(tcu::smem_u32(&bar[b]))
          : "memory");
  };
  if (threadIdx.x == 0) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(tcu::smem_u32(&bar[0])));
    asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(tcu::smem_u32(&bar[1])));
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  __syncthreads();
  if (threadIdx.x == 0 && (long long)blockIdx.x < P) issue(blockIdx.x, 0);
  const int wib = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int tok = lane >> 2, part = lane & 3;
  const bool act = tok < D.Nb;
  const int tk = act ? tok : 0;
  int it = 0;
  for (long long p = blockIdx.x; p < P; p += gridDim.x, ++it) {
    const int b = it & 1;
    // the other buffer was released by the __syncthreads that ended the previous pair
    if (threadIdx.x == 0 && p + gridDim.x < P) issue(p + gridDim.x, b ^ 1);
    {
      const uint32_t ba = tcu::smem_u32(&bar[b]), ph = (it >> 1) & 1;
      asm volatile(
          "{\n.reg .pred q;\nWF_%=:\nmbarrier.try_wait.parity.shared::cta.b64 q, [%0], %1;\n@!q bra WF_%=;\n}\n" ::"r"(ba),
          "r"(ph)
          : "memory");
    }
    const bf16* sq = sq0 + b * D.Nb * rs;
    const int u = pair_user(cand_off, U, p);
    const int r = wave_r[u];
    for (int head = wib; head < D.h; head += 8) {
      const float sc = LOG2E / (sqrtf((float)DH) * tau_f[r * D.h + head]);
      float q[PD];
      load_n<PD>(sq + tk * rs + head * DH + part * PD, q);
      float s[8];
      float mx = -INFINITY;
#pragma unroll
      for (int j = 0; j < 8; ++j) {
        float acc = 0.f;
        if (j < D.Nb) {
          float k[PD];
          load_n<PD>(sq + j * rs + D.d + head * DH + part * PD, k);
#pragma unroll
          for (int c = 0; c < PD; ++c) acc = fmaf(q[c], k[c], acc);
        }
        acc += __shfl_xor_sync(0xffffffffu, acc, 1);
        acc += __shfl_xor_sync(0xffffffffu, acc, 2);
        s[j] = (j < D.Nb) ? acc * sc : -INFINITY;
        mx = fmaxf(mx, s[j]);
      }
      float l = 0.f;
#pragma unroll
      for (int j = 0; j < 8; ++j) {
        s[j] = (j < D.Nb) ? exp2f(s[j] - mx) : 0.f;
        l += s[j];
      }
      const float inv = 1.f / l;
      float o[PD];
#pragma unroll
      for (int c = 0; c < PD; ++c) o[c] = 0.f;
#pragma unroll
      for (int j = 0; j < 8; ++j) {
        if (j < D.Nb) {
          float v[PD];
          load_n<PD>(sq + j * rs + 2 * D.d + head * DH + part * PD, v);
#pragma unroll
          for (int c = 0; c < PD; ++c) o[c] = fmaf(s[j], v[c], o[c]);
        }
      }
      if (act) {
#pragma unroll
        for (int c = 0; c < PD; ++c) o[c] *= inv;
        store_n<PD>(so + tok * ros + head * DH + part * PD, o);
      }
    }
    __syncthreads();
    {
      const int cpr = D.d / 8;
      uint4* g = reinterpret_cast<uint4*>(O + p * D.Nb * (long long)D.d);
      for (int i = threadIdx.x; i < D.Nb * cpr; i += blockDim.x) {
        const int t = i / cpr, c = i % cpr;
        g[i] = *reinterpret_cast<const uint4*>(so + t * ros + c * 8);
      }
    }
    __syncthreads();  // staging and this buffer free again
  }
}

template <typename T>
void launch_attn_fusion(const T* QKV, const int64_t* cand_off, const int* wave_r, int U, long long P,
                        const float* tau_f, T* O, const Dims& D, cudaStream_t s) {
  if constexpr (std::is_same<T, bf16>::value) {
    // bf16 path: one CTA per pair, coalesced row copies (k_attn_fusion_pair)
    if (D.dh >= 16 && P > 0) {
      const int smem = (2 * D.Nb * (3 * D.d + 8) + D.Nb * (D.d + 8)) * 2 + 16;
      static int n_sm = 0;
      if (!n_sm) {
        int dev = 0;
        cudaGetDevice(&dev);
        cudaDeviceGetAttribute(&n_sm, cudaDevAttrMultiProcessorCount, dev);
      }
      const int per_sm = std::max(1, std::min(8, (int)(227 * 1024 / (smem + 1024))));
      const unsigned grid = (unsigned)std::min<long long>(P, (long long)n_sm * per_sm);
#define CL_FP(DH)                                                                                          \
  do {                                                                                                     \
    ensure_smem_attr((const void*)k_attn_fusion_pair<DH>, smem);                                           \
    k_attn_fusion_pair<DH><<<grid, 256, smem, s>>>(QKV, cand_off, wave_r, U, P, tau_f, O, D);              \
  } while (0)
      if (D.dh == 16) CL_FP(16);
      else if (D.dh == 32) CL_FP(32);
      else CL_FP(64);
#undef CL_FP
      return;
    }
  }
  long long n = P * D.h;  // warps
  unsigned g = blocks_for(n, 8);
#define CL_FUS(DH) k_attn_fusion<T, DH><<<g, 256, 0, s>>>(QKV, cand_off, wave_r, U, P, tau_f, O, D)
  if (D.dh == 16) CL_FUS(16);
  else if (D.dh == 32) CL_FUS(32);
  else CL_FUS(64);
#undef CL_FUS
}

void launch_debug_mask(const int* vlen_all, int slot, int M, uint8_t* mask, const Dims& D, cudaStream_t s) {
  k_debug_mask<<<296, 256, 0, s>>>(vlen_all, slot, M, mask, D);
}

template <typename T>
void launch_debug_kv(const T* pool, const int* ptab, const int* vlen_all, int slot, int k, int l, T* K, T* V,
                     const Dims& D, cudaStream_t s) {
  k_debug_kv<T><<<296, 256, 0, s>>>(pool, ptab, vlen_all, slot, k, l, K, V, D);
}

void launch_scatter_ptab(const int* staged, const int* slots, int B, int per, int* ptab, cudaStream_t s) {
  k_scatter_ptab<<<296, 256, 0, s>>>(staged, slots, B, per, ptab);
}

template <typename T>
void launch_gemm_simt(const T* A, long long lda, const T* B, long long ldb, long long M, int N, int K,
                      const Epilogue& e, cudaStream_t s) {
  dim3 grid((N + 63) / 64, (unsigned)((M + 63) / 64));
  k_gemm_simt<T><<<grid, 256, 0, s>>>(A, lda, B, ldb, M, N, K, e);
}

#define INST(T)                                                                                                  \
  template void launch_embed_hist<T>(const EventsDev&, const int64_t*, const int*, int, const int*, const int*,  \
                                     const int*, const T*, const T*, const T*, float*, T*, float*, int, int,     \
                                     const Dims&, cudaStream_t);                                                 \
  template void launch_embed_cand<T>(const int32_t*, const int64_t*, const int*, int, long long, const T*,       \
                                     const T*, float*, T*, float*, int, int*, const Dims&, cudaStream_t);        \
  template void launch_rmsnorm<T>(const float*, long long, const float*, T*, long long, long long, int, float,   \
                                  cudaStream_t);                                                                 \
  template void launch_convert<T>(const float*, T*, long long, cudaStream_t);                                    \
  template void launch_attn_sumi<T>(const T*, const int64_t*, const int*, const int*, int, int, const T*,        \
                                    const int*, const int*, const float*, T*, int, int, const Dims&,             \
                                    cudaStream_t);                                                               \
  template void launch_attn_hist<T>(const T*, const int*, const int*, int, const T*, const int*, const int*,     \
                                    const float*, T*, int, int, const Dims&, cudaStream_t);                      \
  template void launch_attn_fusion<T>(const T*, const int64_t*, const int*, int, long long, const float*, T*,    \
                                      const Dims&, cudaStream_t);                                                \
  template void launch_debug_kv<T>(const T*, const int*, const int*, int, int, int, T*, T*, const Dims&,         \
                                   cudaStream_t);                                                                \
  template void launch_gemm_simt<T>(const T*, long long, const T*, long long, long long, int, int,               \
                                    const Epilogue&, cudaStream_t);
INST(float)
INST(bf16)
#undef INST

}  // namespace climber
