// Internal launcher declarations shared by matq_abi.cu and the kernel units.
#pragma once
#include <cstdint>
#include <cuda_runtime.h>

#include "matq_common.cuh"

namespace mq {
#ifdef MQ_GEMV_TIMING
unsigned long long* gemm_dbg_buffer();  // K4 phase stamps [64 launches][160 CTAs][6]
#endif

cudaError_t launch_pack_planes(const uint8_t* codes, long long ldc, const Layout& L, int nbits,
                               uint32_t* blob, cudaStream_t s);
cudaError_t launch_pack_scales(const float* scales, const Layout& L, int ng, uint32_t* blob, float* ts,
                               cudaStream_t s);
cudaError_t launch_slice_codes(int r, bool child, const uint32_t* blob, const Layout& L, uint8_t* out,
                               long long ldo, cudaStream_t s);
cudaError_t launch_decode_dense(int r, bool child, const uint32_t* blob, const float* ts,
                                const Layout& L, float out_scale, int8_t* vals, float* W,
                                long long ldw, cudaStream_t s);
cudaError_t launch_materialize_child(int r, const uint32_t* blob, const Layout& Lp, uint32_t* child,
                                     cudaStream_t s);
cudaError_t launch_slice_elementwise(const uint8_t* q, long long n, int c, int r, int on_master,
                                     uint8_t* out, int* err, cudaStream_t s);
cudaError_t launch_dequant_f64(const uint8_t* codes, int N, int K, const float* scales, int ng,
                               int G, int c, int r, double* out, int* err, cudaStream_t s);
cudaError_t launch_dequant_value_f64(const uint8_t* q, const double* scale, long long n, int c,
                                     int r, double* out, int* err, cudaStream_t s);
cudaError_t launch_matmul_ref(const float* X, int B, int K, const float* W, int N, float* Y,
                              cudaStream_t s);
cudaError_t launch_pack_ref_layout(const uint8_t* codes, int N, int K, int bits,
                                   unsigned long long* base, uint32_t* b2, uint32_t* b3, int* err,
                                   cudaStream_t s);
cudaError_t launch_unpack_ref_layout(const unsigned long long* base, const uint32_t* b2,
                                     const uint32_t* b3, int N, int K, uint8_t* codes,
                                     cudaStream_t s);

// MatGPTQ quantiser (matq_quant.cu): the target set of a BitWidthSet
struct QuantTargets {
    int T, c;       // number of targets, master bit-width (the largest target)
    int r[8];       // targets, ascending
    double lam[8];  // importance weights
};
cudaError_t launch_select_codes(const double* W, long long ldw, int d_row, int d_col, const float* scales,
                                int ngs, int G, const QuantTargets& tg, uint8_t* codes, long long ldc,
                                cudaStream_t s);
cudaError_t launch_fit_grid(const double* W, long long ldw, int d_row, int d_col, int G, const QuantTargets& tg,
                            const double* alphas, int steps, float* scales, int ngs, cudaStream_t s);
cudaError_t launch_gptq_block(double* Wc, long long ldw, int d_row, int lo, int hi, const float* scales, int ngs,
                              int G, const double* chol, long long ldch, const QuantTargets& tg, uint8_t* codes,
                              long long ldc, double* comp, long long ldcomp, double* err, long long lde,
                              cudaStream_t s);
cudaError_t launch_rtn(const double* w, const double* s, long long n, int c, int mode, double* out_f,
                       long long* out_q, int* err, cudaStream_t st);

// full-model harness glue (matq_glue.cu), bf16
cudaError_t launch_add_rmsnorm(void* x, const void* delta, const float* w, void* y, int B, int h, float eps,
                               cudaStream_t s);
cudaError_t launch_rope_kv(const void* qkv, const void* cosv, const void* sinv, void* q, void* kc, void* vc, int B,
                           int nh, int nkv, int hd, int T, int pos, const float* qn, const float* kn, float eps,
                           cudaStream_t s);
cudaError_t launch_attn_decode(const void* qkv, const void* cosv, const void* sinv, const float* qn, const float* kn,
                               float eps, void* kc, void* vc, const int* kv_of_q, void* att, int B, int nh, int nkv,
                               int hd, int T, int pos, cudaStream_t s);
cudaError_t launch_silu_mul(const void* gu, void* y, int B, int inter, cudaStream_t s);

struct GemmConfig {
    int bn, n_tiles, S, cs, grid;
    int t1;  // tiles [0, t1) run whole (one unit each); tiles [t1, n_tiles) split S ways
};
// Split-K tickets at the head of the K4 workspace (same convention as K3's).
constexpr size_t kGemmTicketBytes = 64 * 1024;
// r < 0: the workspace query, which does not know r (the larger of both tilings)
GemmConfig choose_gemm_config(int N, int K, int B, int sms, int r);
#ifndef MQ_GEMM_BN512_R8
#define MQ_GEMM_BN512_R8 1
#endif
__host__ __device__ constexpr bool gemm_bn512_ok(int r) { return r >= 0 && (r <= 6 || MQ_GEMM_BN512_R8); }
size_t gemm_ws_bytes(const GemmConfig& c);
cudaError_t launch_gemm(const uint32_t* blob, const Layout& L, const void* X, int ldx, void* Y,
                        int ldy, int B, int r, bool child, float out_scale, bool y_f32,
                        const GemmConfig& c, void* ws, cudaStream_t stream, bool pdl,
                        const char** why);

}  // namespace mq
