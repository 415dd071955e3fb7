// Launchers for the libclimber kernels (internal).
#pragma once
#include "common.cuh"

namespace climber {

// Host-side launch setup failures (a tensor map the driver rejects): the
// kernel is NOT launched, the failure is recorded, and the next status check
// of the C-ABI call (check_launch) returns CLIMBER_E_CUDA with the message.
void note_launch_error(const char* what);
bool take_launch_error(char* msg, int cap);
// cudaFuncSetAttribute(MaxDynamicSharedMemorySize) per (kernel, device), raised
// whenever a launch needs more than was set before (the attribute is per
// device, so a process driving several GPUs sets it on each).
void ensure_smem_attr(const void* kern, int bytes);

struct EventsDev {
  const int32_t* item;
  const uint8_t* action;
  const uint8_t* scenario;
  const int64_t* ts;
};

// relative bias (rel_bias = 1): candidate-row bias over the history keys, per (user, layer, block, head)
void launch_cand_bias(const int* wave_slot, const int* wave_r, int U, const int* vlen_all, const Dims& D,
                      cudaStream_t s);
// block-parallel fusion input: bf16 copy + norm partials of gathered fp32 rows
void launch_row_prep(const float* C, bf16* Cb, float* part, long long rows, int d, int pld, cudaStream_t s);
// incremental cache update: which strategies an appended event range matches
void launch_append_flags(const uint8_t* action, const uint8_t* scenario, long long n0, long long n1,
                         const unsigned long long* amask, const unsigned long long* smask, int* flags, const Dims& D,
                         cudaStream_t s);
// CLIMBER_SYNC_CHECK: flag non-finite values in the device error word
void launch_check_finite(const float* x, long long n, int* err, cudaStream_t s);
void launch_extract(const EventsDev& ev, const int64_t* ev_off, const int* wave_slot, int U,
                    const unsigned long long* amask, const unsigned long long* smask, int* idx_all,
                    int* vlen_all, int* bad_all, int* err, const Dims& D, cudaStream_t s);
template <typename T>
void launch_embed_hist(const EventsDev& ev, const int64_t* ev_off, const int* wave_slot, int U, const int* idx_all,
                       const int* vlen_all, const int* bad_all, const T* e_item, const T* e_act, const T* e_scn,
                       float* X, T* Xb, float* part, int pld, int k, const Dims& D, cudaStream_t s);
template <typename T>
void launch_embed_cand(const int32_t* items, const int64_t* cand_off, const int* wave_r, int U, long long P,
                       const T* e_item, const T* e_scn, float* C, T* Cb, float* part, int pld, int* err,
                       const Dims& D, cudaStream_t s);
template <typename T>
void launch_rmsnorm(const float* X, long long ldx, const float* g, T* out, long long ldo, long long rows, int d,
                    float eps, cudaStream_t s);
template <typename T>
void launch_convert(const float* X, T* out, long long n, cudaStream_t s);
void launch_head(const float* Y, const float* gate, const float* w, float b, float* scores, long long P, int Dse,
                 cudaStream_t s);
template <typename T>
void launch_attn_sumi(const T* QKV, const int64_t* cand_off, const int* wave_slot, const int* wave_r, int U,
                      int Mmax, const T* pool, const int* ptab, const int* vlen_all, const float* tau, T* O, int k,
                      int l, const Dims& D, cudaStream_t s);
template <typename T>
void launch_attn_hist(const T* Q, const int* wave_slot, const int* wave_r, int U, const T* pool, const int* ptab,
                      const int* vlen_all, const float* tau, T* O, int k, int l, const Dims& D, cudaStream_t s);
template <typename T>
void launch_attn_fusion(const T* QKV, const int64_t* cand_off, const int* wave_r, int U, long long P,
                        const float* tau_f, T* O, const Dims& D, cudaStream_t s);
void launch_debug_mask(const int* vlen_all, int slot, int M, uint8_t* mask, const Dims& D, cudaStream_t s);
template <typename T>
void launch_debug_kv(const T* pool, const int* ptab, const int* vlen_all, int slot, int k, int l, T* K, T* V,
                     const Dims& D, cudaStream_t s);
// mask probe (climber_debug_attn_probe)
template <typename T>
void launch_probe_pages(T* pool, const int* ptab, int slot, int k, int l, int key_off, const Dims& D, cudaStream_t s);
template <typename T>
void launch_probe_qkv(T* QKV, long long rows, const Dims& D, cudaStream_t s);
void launch_kv_layer_copy(void* pool, const int* ptab, int slot, int l, long long page_bytes, void* sec, bool unpack,
                          const Dims& D, cudaStream_t s);
void launch_kv_export(const void* pool, const int* ptab, const int* vlen_all, int slot, int per_slot, long long page_bytes,
                      void* slab, const Dims& D, int dtype, int r, cudaStream_t s);
void launch_kv_import(void* pool, const int* ptab, int* vlen_all, int slot, int per_slot, long long page_bytes,
                      const void* slab, int* err, const Dims& D, int dtype, cudaStream_t s);
void launch_scatter_ptab(const int* staged, const int* slots, int B, int per, int* ptab, cudaStream_t s);
template <typename T>
void launch_gemm_simt(const T* A, long long lda, const T* B, long long ldb, long long M, int N, int K,
                      const Epilogue& e, cudaStream_t s);

// Tensor-core (mma.sync) attention for the bf16 path, attn_mma.cu.
bool attn_mma_supported(int dh);
void launch_attn_sumi_mma(const bf16* QKV, const int64_t* cand_off, const int* wave_slot, const int* wave_r, int U,
                          int Mmax, const bf16* pool, const int* ptab, const int* vlen_all, const float* tau, bf16* O,
                          int k, int l, const Dims& D, cudaStream_t s);
void launch_attn_hist_mma(const bf16* Q, const int* wave_slot, const int* wave_r, int U, const bf16* pool,
                          const int* ptab, const int* vlen_all, const float* tau, bf16* O, int k, int l, const Dims& D,
                          cudaStream_t s);

// tcgen05/TMEM flash attention for the bf16 path, attn_fa.cu (d_h 32 / 64,
// n_k % 64 == 0; relative bias included).
bool attn_tc_supported(int dh, int nk, bool hist);
void launch_attn_sumi_tc(const bf16* QKV, long long P, const int64_t* cand_off, const int* wave_slot,
                         const int* wave_r, int U, int Mmax, const bf16* pool, long long pool_rows, const int* ptab,
                         const int* vlen_all, const float* tau, bf16* O, int k, int l, const Dims& D, cudaStream_t s,
                         int nbk = 1);
void launch_attn_hist_tc(const bf16* Q, const int* wave_slot, const int* wave_r, int U, const bf16* pool,
                         long long pool_rows, const int* ptab, const int* vlen_all, const float* tau, bf16* O, int k,
                         int l, const Dims& D, cudaStream_t s, int nbk = 1);

// tcgen05 GEMM (bf16 in, fp32 accumulate in TMEM), gemm_tc.cu.  Returns false
// if the shape is not supported by the tensor-core kernel.
bool gemm_tc_supported(long long M, int N, int K, long long lda, long long ldb);
bool gemm_tc_available();
void launch_gemm_tc(const bf16* A, long long lda, const bf16* B, long long ldb, long long M, int N, int K,
                    const Epilogue& e, cudaStream_t s);
// grouped over `batch` independent GEMMs (the N_b blocks): A_b = A + b * a_bs,
// B_b = B + b * b_bs, outputs offset by the Epilogue's *_bs strides
void launch_gemm_tc_batched(const bf16* A, long long lda, long long a_bs, const bf16* B, long long ldb,
                            long long b_bs, long long M, int N, int K, int batch, const Epilogue& e, cudaStream_t s);

}  // namespace climber
