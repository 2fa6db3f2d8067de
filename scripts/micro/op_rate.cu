// Per-SM throughput of integer/bf16 ops on sm_100a (8 independent chains/thread).
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>
#define CH 8
template <int OP>
__global__ void k(uint32_t seed, int iters, uint32_t* out) {
    uint32_t v[CH];
    for (int c = 0; c < CH; ++c) v[c] = seed * (c + 1) + threadIdx.x;
    const uint32_t m = 0x0F0F0F0Fu ^ seed, z = 0x43004300u + seed;
    for (int it = 0; it < iters; ++it) {
#pragma unroll
        for (int u = 0; u < 8; ++u)
#pragma unroll
        for (int c = 0; c < CH; ++c) {
            uint32_t a = v[c];
            if (OP == 0) asm volatile("lop3.b32 %0, %0, %1, %2, 0xEA;" : "+r"(a) : "r"(m), "r"(z));
            if (OP == 1) asm volatile("shf.r.wrap.b32 %0, %0, %0, 3;" : "+r"(a));
            if (OP == 2) asm volatile("mul.lo.u32 %0, %0, 16;" : "+r"(a));
            if (OP == 3) asm volatile("mul.hi.u32 %0, %0, 0x1000000;" : "+r"(a));
            if (OP == 4) asm volatile("fma.rn.bf16x2 %0, %0, %1, %2;" : "+r"(a) : "r"(m), "r"(z));
            if (OP == 5) { asm volatile("lop3.b32 %0, %0, %1, %2, 0xEA;" : "+r"(a) : "r"(m), "r"(z)); asm volatile("mul.lo.u32 %0, %0, 16;" : "+r"(a)); }
            if (OP == 6) { asm volatile("lop3.b32 %0, %0, %1, %2, 0xEA;" : "+r"(a) : "r"(m), "r"(z)); asm volatile("mul.hi.u32 %0, %0, 0x1000000;" : "+r"(a)); }
            if (OP == 7) { asm volatile("lop3.b32 %0, %0, %1, %2, 0xEA;" : "+r"(a) : "r"(m), "r"(z)); asm volatile("fma.rn.bf16x2 %0, %0, %1, %2;" : "+r"(a) : "r"(m), "r"(z)); }
            if (OP == 8) asm volatile("prmt.b32 %0, %0, %1, 0x5410;" : "+r"(a) : "r"(z));
            v[c] = a;
        }
    }
    uint32_t x = 0;
    for (int c = 0; c < CH; ++c) x ^= v[c];
    if (x == 0x1234567) out[0] = x;
}
template <int OP> void run(const char* name, int sms, int ops_per) {
    uint32_t* d; cudaMalloc(&d, 4);
    int iters = 4000, warps = 32;
    cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
    k<OP><<<sms, warps * 32>>>(1, 10, d);
    cudaEventRecord(e0); k<OP><<<sms, warps * 32>>>(1, iters, d); cudaEventRecord(e1); cudaEventSynchronize(e1);
    float ms; cudaEventElapsedTime(&ms, e0, e1);
    double instr = (double)sms * warps * iters * 8 * CH * ops_per;  // warp-instructions
    int clk; cudaDeviceGetAttribute(&clk, cudaDevAttrClockRate, 0);
    printf("%-22s %.2f warp-instr/cycle/SM (at %.0f MHz nominal)\n", name, instr / sms / (ms * 1e-3 * clk * 1e3), clk / 1e3);
}
int main() {
    int sms; cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
    run<0>("LOP3", sms, 1); run<1>("SHF", sms, 1); run<2>("IMAD.SHL(mul.lo)", sms, 1); run<3>("IMAD.HI(mul.hi)", sms, 1);
    run<4>("HFMA2.BF16", sms, 1); run<8>("PRMT", sms, 1); run<5>("LOP3+IMAD.SHL", sms, 2); run<6>("LOP3+IMAD.HI", sms, 2); run<7>("LOP3+HFMA2", sms, 2);
}
