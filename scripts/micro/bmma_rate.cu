// Microbenchmark: binary (b1, AND + popc) mma.sync throughput on sm_100a versus
// the bf16 m16n8k16 HMMA, plus int8 m16n8k32 IMMA: is a bit-plane x bit-serial
// GEMV (no weight decode) viable on this part?
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>
template <int OP, int CH>
__global__ void k(int* out, int iters) {
    int acc[CH][4];
    for (int c = 0; c < CH; ++c) for (int i = 0; i < 4; ++i) acc[c][i] = 0;
    uint32_t a0 = threadIdx.x * 0x9E3779B9u, a1 = a0 * 3, a2 = a0 * 5, a3 = a0 * 7, b0 = a0 ^ 0x3c003c00u, b1 = b0 + 1;
    for (int it = 0; it < iters; ++it) {
#pragma unroll
        for (int c = 0; c < CH; ++c) {
            if (OP == 0)
                asm volatile("mma.sync.aligned.m16n8k128.row.col.s32.b1.b1.s32.and.popc {%0,%1,%2,%3}, {%4,%5}, {%6}, {%0,%1,%2,%3};"
                             : "+r"(acc[c][0]), "+r"(acc[c][1]), "+r"(acc[c][2]), "+r"(acc[c][3])
                             : "r"(a0), "r"(a1), "r"(b0));
            if (OP == 1)
                asm volatile("mma.sync.aligned.m16n8k256.row.col.s32.b1.b1.s32.and.popc {%0,%1,%2,%3}, {%4,%5,%6,%7}, {%8,%9}, {%0,%1,%2,%3};"
                             : "+r"(acc[c][0]), "+r"(acc[c][1]), "+r"(acc[c][2]), "+r"(acc[c][3])
                             : "r"(a0), "r"(a1), "r"(a2), "r"(a3), "r"(b0), "r"(b1));
            if (OP == 2)
                asm volatile("mma.sync.aligned.m16n8k32.row.col.s32.s8.s8.s32 {%0,%1,%2,%3}, {%4,%5,%6,%7}, {%8,%9}, {%0,%1,%2,%3};"
                             : "+r"(acc[c][0]), "+r"(acc[c][1]), "+r"(acc[c][2]), "+r"(acc[c][3])
                             : "r"(a0), "r"(a1), "r"(a2), "r"(a3), "r"(b0), "r"(b1));
            if (OP == 3) {
                float* f = reinterpret_cast<float*>(acc[c]);
                asm volatile("mma.sync.aligned.m16n8k16.row.col.f32.bf16.bf16.f32 {%0,%1,%2,%3}, {%4,%5,%6,%7}, {%8,%9}, {%0,%1,%2,%3};"
                             : "+f"(f[0]), "+f"(f[1]), "+f"(f[2]), "+f"(f[3])
                             : "r"(a0), "r"(a1), "r"(a2), "r"(a3), "r"(b0), "r"(b1));
            }
        }
    }
    int s = 0; for (int c = 0; c < CH; ++c) for (int i = 0; i < 4; ++i) s += acc[c][i];
    if (s == 123) out[0] = s;
}
static const char* NAMES[] = {"b1 m16n8k128 and.popc", "b1 m16n8k256 and.popc", "s8 m16n8k32", "bf16 m16n8k16"};
template <int OP, int CH> void run(int warps_per_sm, int sms) {
    int* d; cudaMalloc(&d, 4);
    int iters = 2048;
    cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
    k<OP, CH><<<sms, 32 * warps_per_sm>>>(d, 16);
    cudaError_t e = cudaDeviceSynchronize();
    if (e != cudaSuccess) { printf("%s: %s\n", NAMES[OP], cudaGetErrorString(e)); return; }
    cudaEventRecord(e0);
    k<OP, CH><<<sms, 32 * warps_per_sm>>>(d, iters);
    cudaEventRecord(e1); cudaEventSynchronize(e1);
    float ms; cudaEventElapsedTime(&ms, e0, e1);
    double mmas = (double)sms * warps_per_sm * iters * CH;
    int clk; cudaDeviceGetAttribute(&clk, cudaDevAttrClockRate, 0);
    printf("%-24s chains=%d warps/SM=%2d: %.3f ms, %.3f mma/clk/SM, latency-ish %.1f clk/mma/chain\n", NAMES[OP], CH,
           warps_per_sm, ms, mmas / sms / (ms * 1e-3 * clk * 1e3), ms * 1e-3 * clk * 1e3 / (iters));
    cudaFree(d);
}
template <int OP> void sweep(int sms) {
    run<OP, 1>(4, sms); run<OP, 4>(4, sms); run<OP, 4>(8, sms); run<OP, 4>(16, sms); run<OP, 8>(16, sms);
}
int main() {
    int sms; cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
    sweep<0>(sms); sweep<1>(sms); sweep<2>(sms); sweep<3>(sms);
}
