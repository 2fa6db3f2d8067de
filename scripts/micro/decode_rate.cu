// Compute ceiling of the K3 register decode (no memory): weights/s for
// decode only, decode + mma.sync, per bit-width; varying warps per SM.
#include <cstdio>
#include "../../paper_2602_03537_b200/csrc/matq_common.cuh"
using namespace mq;

template <int R, bool RAW, bool MMA, bool F16 = false>
__global__ void k(uint32_t seed, int iters, float* out) {
    constexpr int NPL = PlaneCount<R, false>::value;
    uint32_t T[NPL];
    for (int j = 0; j < NPL; ++j) T[j] = seed * (j + 3) + threadIdx.x * 0x9E3779B9u;
    float acc[4] = {0, 0, 0, 0};
    uint32_t x = 0;
    const uint32_t b0 = 0x3f803f80u, b1 = 0x3f803f80u;
    for (int it = 0; it < iters; ++it) {
#pragma unroll
        for (int w = 0; w < 4; ++w) {
            uint32_t Tw[NPL];
#pragma unroll
            for (int j = 0; j < NPL; ++j) Tw[j] = T[j] ^ (w * 0x01010101u) ^ it;
            uint32_t S[R];
            slice_loaded<R, false>(Tw, S);
            uint32_t A[16];
            if constexpr (F16) decode_word_f16<R>(S, A);
            else decode_word<R, RAW>(S, A);
            if (MMA) {
#pragma unroll
                for (int s = 0; s < 4; ++s) {
                    if constexpr (F16) mma_acc_f16(acc, A[4 * s], A[4 * s + 1], A[4 * s + 2], A[4 * s + 3], b0, b1);
                    else mma_acc(acc, A[4 * s], A[4 * s + 1], A[4 * s + 2], A[4 * s + 3], b0, b1);
                }
            } else {
#pragma unroll
                for (int q = 0; q < 16; ++q) x ^= A[q];
            }
        }
    }
    if (x == 0x12345 || acc[0] == 1.2345f) out[0] = acc[0] + x;
}

template <int R, bool RAW, bool MMA, bool F16 = false>
void run(int sms, int warps) {
    float* d; cudaMalloc(&d, 4);
    const int iters = 2000;
    cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
    k<R, RAW, MMA, F16><<<sms, warps * 32>>>(1, 10, d);
    cudaEventRecord(e0);
    k<R, RAW, MMA, F16><<<sms, warps * 32>>>(1, iters, d);
    cudaEventRecord(e1); cudaEventSynchronize(e1);
    float ms; cudaEventElapsedTime(&ms, e0, e1);
    double w = (double)sms * warps * 32 * iters * 128;  // weights decoded
    double need = (R < 8 ? R + 1 : 8) / 8.0;            // bytes per weight (mode P)
    printf("R=%d raw=%d f16=%d mma=%d warps=%2d: %.2f Tw/s  (=> %.0f GB/s of mode-P planes)\n", R, RAW, F16, MMA, warps,
           w / (ms * 1e-3) / 1e12, w / (ms * 1e-3) * need / 1e9);
    cudaFree(d);
}
int main() {
    int sms; cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
    for (int warps : {16}) {
        run<2, true, false>(sms, warps); run<2, true, true>(sms, warps);
        run<4, true, false>(sms, warps); run<4, true, true>(sms, warps); run<4, false, true>(sms, warps);
        run<4, true, false, true>(sms, warps); run<4, true, true, true>(sms, warps);
        run<8, false, false>(sms, warps); run<8, false, true>(sms, warps);
        run<8, true, false, true>(sms, warps); run<8, true, true, true>(sms, warps);
    }
}
