// Microbenchmark: legacy mma.sync m16n8k16 bf16 throughput / latency on this GPU.
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>
template <int CH>
__global__ void k(float* out, int iters) {
    float acc[CH][4];
    for (int c = 0; c < CH; ++c) for (int i = 0; i < 4; ++i) acc[c][i] = 0.f;
    uint32_t a0 = threadIdx.x, a1 = a0 * 3, a2 = a0 * 5, a3 = a0 * 7, b0 = a0 ^ 0x3c003c00u, b1 = b0 + 1;
    for (int it = 0; it < iters; ++it) {
#pragma unroll
        for (int c = 0; c < CH; ++c)
            asm volatile("mma.sync.aligned.m16n8k16.row.col.f32.bf16.bf16.f32 {%0,%1,%2,%3}, {%4,%5,%6,%7}, {%8,%9}, {%0,%1,%2,%3};"
                         : "+f"(acc[c][0]), "+f"(acc[c][1]), "+f"(acc[c][2]), "+f"(acc[c][3])
                         : "r"(a0), "r"(a1), "r"(a2), "r"(a3), "r"(b0), "r"(b1));
    }
    float s = 0; for (int c = 0; c < CH; ++c) for (int i = 0; i < 4; ++i) s += acc[c][i];
    if (s == 123.f) out[0] = s;
}
template <int CH> void run(int warps_per_sm, int sms) {
    float* d; cudaMalloc(&d, 4);
    int iters = 4096;
    cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
    k<CH><<<sms, 32 * warps_per_sm>>>(d, 16);
    cudaEventRecord(e0);
    k<CH><<<sms, 32 * warps_per_sm>>>(d, iters);
    cudaEventRecord(e1); cudaEventSynchronize(e1);
    float ms; cudaEventElapsedTime(&ms, e0, e1);
    double mmas = (double)sms * warps_per_sm * iters * CH;
    printf("chains=%d warps/SM=%d: %.3f ms, %.1f TFLOP/s, %.2f ns/mma/warp-chain, %.1f cyc/HMMA/SM@1.9GHz\n", CH,
           warps_per_sm, ms, mmas * 4096 / (ms * 1e-3) / 1e12, ms * 1e6 / (iters), ms * 1e-3 * 1.9e9 / (mmas / sms));
    cudaFree(d);
}
int main() {
    int sms; cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
    for (int w : {4, 8, 16, 32}) { run<1>(w, sms); run<2>(w, sms); run<4>(w, sms); run<8>(w, sms); }
}
