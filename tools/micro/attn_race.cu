// Determinism check of the tcgen05 attention kernels in isolation (debug
// tool): random bf16 q / k_self / v_self and K/V pages shaped like one
// `large` wave (64 users x 8 blocks x 8 heads, n_k = 512, M = 1000), the SUMI
// (and history) launch repeated on identical inputs, outputs compared bit for
// bit; differing rows are decoded to (block, user, tile, row, head).
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -lcuda \
//        -I paper_2502_09888_b200/csrc tools/micro/attn_race.cu \
//        paper_2502_09888_b200/csrc/attn_fa.cu -o attn_race
#include <cuda_runtime.h>

#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <vector>

#include "kernels.cuh"

namespace climber {
void note_launch_error(const char* what) { fprintf(stderr, "launch error: %s\n", what); }
void ensure_smem_attr(const void* kern, int bytes) {
  cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, bytes);
}
}  // namespace climber
using namespace climber;

static uint16_t rnd_bf16(uint64_t& s) {
  s = s * 6364136223846793005ULL + 1442695040888963407ULL;
  const float f = ((float)((s >> 33) & 0xFFFFFF) / 16777216.0f - 0.5f) * 2.0f;
  uint32_t u;
  memcpy(&u, &f, 4);
  return (uint16_t)(u >> 16);
}

int main(int argc, char** argv) {
  const int reps = argc > 1 ? atoi(argv[1]) : 4;
  const int mode = argc > 2 ? atoi(argv[2]) : 0;  // 0 SUMI, 1 history
  const char* ref_path = argc > 3 ? argv[3] : nullptr;  // "save:<file>" or "cmp:<file>"
  const int U = 64, nbk = 8, h = 8, dh = 64, d = 512, nk = 512, M = 1000;
  Dims D{};
  D.d = d; D.h = h; D.dh = dh; D.L = 1; D.Nb = nbk; D.nk = nk; D.F = 4 * d; D.R = 1; D.Mmax = M; D.causal = 1;
  D.ppb = nk / PAGE;
  const long long P = (long long)U * M;
  const long long n_pages = (long long)U * nbk * D.ppb;
  const long long pool_rows = n_pages * 2 * PAGE;
  const long long q_rows = mode == 0 ? P * nbk : (long long)U * nk * nbk;
  const int q_cols = mode == 0 ? 3 * d : d;
  std::vector<uint16_t> hq((size_t)q_rows * q_cols), hp((size_t)pool_rows * d);
  uint64_t s = 12345;
  for (auto& x : hq) x = rnd_bf16(s);
  for (auto& x : hp) x = rnd_bf16(s);
  std::vector<int> ptab(n_pages), slot(U), r(U, 0), vlen(U * nbk, nk);
  for (long long i = 0; i < n_pages; ++i) ptab[i] = (int)((i * 7919) % n_pages);  // scattered pages
  for (int u = 0; u < U; ++u) slot[u] = u;
  std::vector<int64_t> coff(U + 1);
  for (int u = 0; u <= U; ++u) coff[u] = (int64_t)u * M;
  std::vector<float> tau(nbk * h, 1.0f);
  bf16 *dq, *dp, *dO;
  int *dpt, *dsl, *dr, *dvl;
  int64_t* dco;
  float* dtau;
  const long long o_rows = q_rows;
  cudaMalloc(&dq, hq.size() * 2);
  cudaMalloc(&dp, hp.size() * 2);
  cudaMalloc(&dO, (size_t)o_rows * d * 2);
  cudaMalloc(&dpt, n_pages * 4);
  cudaMalloc(&dsl, U * 4);
  cudaMalloc(&dr, U * 4);
  cudaMalloc(&dvl, U * nbk * 4);
  cudaMalloc(&dco, (U + 1) * 8);
  cudaMalloc(&dtau, tau.size() * 4);
  cudaMemcpy(dq, hq.data(), hq.size() * 2, cudaMemcpyHostToDevice);
  cudaMemcpy(dp, hp.data(), hp.size() * 2, cudaMemcpyHostToDevice);
  cudaMemcpy(dpt, ptab.data(), n_pages * 4, cudaMemcpyHostToDevice);
  cudaMemcpy(dsl, slot.data(), U * 4, cudaMemcpyHostToDevice);
  cudaMemcpy(dr, r.data(), U * 4, cudaMemcpyHostToDevice);
  cudaMemcpy(dvl, vlen.data(), U * nbk * 4, cudaMemcpyHostToDevice);
  cudaMemcpy(dco, coff.data(), (U + 1) * 8, cudaMemcpyHostToDevice);
  cudaMemcpy(dtau, tau.data(), tau.size() * 4, cudaMemcpyHostToDevice);
  std::vector<uint16_t> ref((size_t)o_rows * d), got((size_t)o_rows * d);
  for (int rep = 0; rep < reps; ++rep) {
    cudaMemset(dO, 0xFF, (size_t)o_rows * d * 2);
    if (mode == 0)
      launch_attn_sumi_tc(dq, P, dco, dsl, dr, U, M, dp, pool_rows, dpt, dvl, dtau, dO, 0, 0, D, 0, nbk);
    else
      launch_attn_hist_tc(dq, dsl, dr, U, dp, pool_rows, dpt, dvl, dtau, dO, 0, 0, D, 0, nbk);
    cudaError_t e = cudaDeviceSynchronize();
    if (e != cudaSuccess) {
      printf("cuda error %s\n", cudaGetErrorString(e));
      return 1;
    }
    cudaMemcpy(rep == 0 ? ref.data() : got.data(), dO, ref.size() * 2, cudaMemcpyDeviceToHost);
    if (rep == 0 && ref_path && !strncmp(ref_path, "save:", 5)) {
      FILE* f = fopen(ref_path + 5, "wb");
      fwrite(ref.data(), 2, ref.size(), f);
      fclose(f);
    }
    if (rep == 0 && ref_path && !strncmp(ref_path, "cmp:", 4)) {  // rep 0 against a stored reference
      FILE* f = fopen(ref_path + 4, "rb");
      std::vector<uint16_t> stored(ref.size());
      const size_t nr = fread(stored.data(), 2, stored.size(), f);
      fclose(f);
      long long nd = 0;
      double mx = 0.0;
      auto f32 = [](uint16_t b) { uint32_t u = (uint32_t)b << 16; float f; memcpy(&f, &u, 4); return f; };
      for (size_t k = 0; k < ref.size() && k < nr; ++k)
        if (stored[k] != ref[k]) {
          ++nd;
          const double dd = fabs((double)f32(stored[k]) - (double)f32(ref[k]));
          mx = dd > mx ? dd : mx;
        }
      printf("rep 0 vs stored reference: %lld differing elements (max abs diff %.3g)\n", nd, mx);
    }
    if (rep == 0) continue;
    long long nd = 0, shown = 0;
    std::vector<long long> per_row_in_tile(128, 0), per_head(h, 0);
    for (long long i = 0; i < o_rows; ++i)
      for (int c = 0; c < d; ++c) {
        const size_t k = (size_t)i * d + c;
        if (ref[k] != got[k]) {
          ++nd;
          long long row_in_tile, tile, user, blk = i / (mode == 0 ? P : (long long)U * nk);
          const long long p = i % (mode == 0 ? P : (long long)U * nk);
          user = p / (mode == 0 ? M : nk);
          tile = (p % (mode == 0 ? M : nk)) / 128;
          row_in_tile = (p % (mode == 0 ? M : nk)) % 128;
          per_row_in_tile[row_in_tile]++;
          per_head[c / dh]++;
          if (shown < 12 && c % dh == 0) {
            printf("  diff: block %lld user %lld tile %lld row %lld head %d: %04x vs %04x\n", blk, user, tile,
                   row_in_tile, c / dh, ref[k], got[k]);
            ++shown;
          }
        }
      }
    printf("rep %d: %lld differing elements of %lld\n", rep, nd, o_rows * d);
    if (nd) {
      printf("  by row-in-tile quadrant: %lld %lld %lld %lld\n", [&] { long long t = 0; for (int q = 0; q < 32; ++q) t += per_row_in_tile[q]; return t; }(),
             [&] { long long t = 0; for (int q = 32; q < 64; ++q) t += per_row_in_tile[q]; return t; }(),
             [&] { long long t = 0; for (int q = 64; q < 96; ++q) t += per_row_in_tile[q]; return t; }(),
             [&] { long long t = 0; for (int q = 96; q < 128; ++q) t += per_row_in_tile[q]; return t; }());
    }
  }
  return 0;
}
