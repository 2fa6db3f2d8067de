// Streaming-read bandwidth: LDG.128 vs per-warp cp.async.bulk rings of various sizes.
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>

__device__ __forceinline__ void mbar_init(uint32_t bar, uint32_t c) { asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(bar), "r"(c)); }
__device__ __forceinline__ void mbar_expect(uint32_t bar, uint32_t b) { asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(bar), "r"(b) : "memory"); }
__device__ __forceinline__ void mbar_wait(uint32_t bar, uint32_t ph) {
    asm volatile("{\n.reg .pred p;\nW%=:\nmbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n@!p bra W%=;\n}\n" ::"r"(bar), "r"(ph) : "memory");
}
__device__ __forceinline__ void bulk(uint32_t dst, const void* src, uint32_t n, uint32_t bar) {
    asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(dst), "l"(src), "r"(n), "r"(bar) : "memory");
}

__global__ void k_ldg(const uint4* __restrict__ p, size_t n16, uint32_t* out) {
    uint32_t acc = 0;
    for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < n16; i += (size_t)gridDim.x * blockDim.x) {
        uint4 v;
        asm volatile("ld.global.nc.L1::no_allocate.v4.u32 {%0,%1,%2,%3}, [%4];" : "=r"(v.x), "=r"(v.y), "=r"(v.z), "=r"(v.w) : "l"(p + i));
        acc ^= v.x ^ v.w;
    }
    if (acc == 0x12345678) out[0] = acc;
}

// each warp streams `chunk` bytes per request through a D-deep ring
__global__ void k_bulk(const uint8_t* __restrict__ p, size_t nbytes, int chunk, int D, uint32_t* out) {
    extern __shared__ __align__(128) uint8_t sm[];
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31, nw = blockDim.x >> 5;
    uint64_t* bars = reinterpret_cast<uint64_t*>(sm);
    uint8_t* ring = sm + 1024 + (size_t)warp * D * chunk;
    const uint32_t bar0 = (uint32_t)__cvta_generic_to_shared(bars + warp * 8);
    const uint32_t r0 = (uint32_t)__cvta_generic_to_shared(ring);
    if (lane == 0) { for (int i = 0; i < D; ++i) mbar_init(bar0 + 8 * i, 1); asm volatile("fence.mbarrier_init.release.cluster;"); }
    __syncwarp();
    const size_t nchunks = nbytes / chunk;
    const size_t gw = (size_t)blockIdx.x * nw + warp, W = (size_t)gridDim.x * nw;
    size_t mine = gw < nchunks ? (nchunks - 1 - gw) / W + 1 : 0;
    uint32_t acc = 0;
    if (lane == 0) for (int i = 0; i < D && i < (int)mine; ++i) { mbar_expect(bar0 + 8 * i, chunk); bulk(r0 + i * chunk, p + (gw + i * W) * chunk, chunk, bar0 + 8 * i); }
    for (size_t f = 0; f < mine; ++f) {
        const int st = f % D;
        mbar_wait(bar0 + 8 * st, (f / D) & 1);
        uint32_t v; asm volatile("ld.shared.u32 %0, [%1];" : "=r"(v) : "r"(r0 + st * chunk + lane * 4)); acc ^= v;
        __syncwarp();
        if (lane == 0 && f + D < mine) { asm volatile("fence.proxy.async.shared::cta;" ::: "memory"); mbar_expect(bar0 + 8 * st, chunk); bulk(r0 + st * chunk, p + (gw + (f + D) * W) * chunk, chunk, bar0 + 8 * st); }
    }
    if (acc == 0x12345678) out[0] = acc;
}

int main() {
    int sms; cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
    size_t nbytes = (size_t)2 << 30;
    uint8_t* p; cudaMalloc(&p, nbytes); cudaMemset(p, 1, nbytes);
    uint32_t* out; cudaMalloc(&out, 4);
    cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
    float ms;
    for (int blocks_per_sm : {2, 4, 8}) {
        k_ldg<<<sms * blocks_per_sm, 256>>>((const uint4*)p, nbytes / 16, out);
        cudaEventRecord(e0); k_ldg<<<sms * blocks_per_sm, 256>>>((const uint4*)p, nbytes / 16, out); cudaEventRecord(e1); cudaEventSynchronize(e1);
        cudaEventElapsedTime(&ms, e0, e1); printf("LDG.128 %d x 256 thr/SM: %.0f GB/s\n", blocks_per_sm, nbytes / (ms * 1e-3) / 1e9);
    }
    cudaFuncSetAttribute(k_bulk, cudaFuncAttributeMaxDynamicSharedMemorySize, 220 * 1024);
    for (int warps : {8, 16}) for (int chunk : {1024, 2688, 4096, 8192}) for (int D : {2, 4, 8}) {
        size_t smem = 1024 + (size_t)warps * D * chunk;
        if (smem > 220 * 1024) continue;
        k_bulk<<<sms, warps * 32, smem>>>(p, nbytes, chunk, D, out);
        cudaEventRecord(e0); k_bulk<<<sms, warps * 32, smem>>>(p, nbytes, chunk, D, out); cudaEventRecord(e1); cudaEventSynchronize(e1);
        cudaError_t e = cudaGetLastError();
        cudaEventElapsedTime(&ms, e0, e1);
        printf("bulk warps=%2d chunk=%5d D=%d: %.0f GB/s %s\n", warps, chunk, D, (nbytes / chunk * (size_t)chunk) / (ms * 1e-3) / 1e9, e ? cudaGetErrorString(e) : "");
    }
}
