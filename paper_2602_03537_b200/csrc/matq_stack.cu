// matq_stack.cu -- K3S instantiations and cooperative launcher.
#include <cstdio>
#include <cstdlib>
#include <atomic>
#include <mutex>

#include "matq_stack.cuh"

namespace mq {

namespace {
// the kernel's dynamic shared-memory limit only grows; serialised (plans and runs may
// come from several host threads)
template <int NT, int R, bool CHILD, bool XOPS>
cudaError_t set_smem(size_t smem) {
    static std::mutex mu;
    static int smem_set = 0;
    std::lock_guard<std::mutex> lk(mu);
    if ((int)smem > smem_set) {
        cudaError_t e = cudaFuncSetAttribute(k_stack<NT, R, CHILD, XOPS>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                             (int)smem);
        if (e != cudaSuccess) return e;
        smem_set = (int)smem;
    }
    return cudaSuccess;
}

// Every CTA must be resident: the layer barriers spin.  The launch is
// cooperative (the driver then guarantees co-residency or fails the launch),
// with the cluster dimension added for CTA pairs.  MQ_STACK_NOCOOP=1 drops the
// cooperative attribute from pair launches -- a profiling knob only: ncu's
// kernel replay rejects cooperative cluster launches.
bool stack_nocoop() {
    static const int v = [] {
        const char* e = getenv("MQ_STACK_NOCOOP");
        return e && e[0] == '1' ? 1 : 0;
    }();
    return v != 0;
}

// Programmatic dependent launch (the producer prefetches weights under the previous
// kernel's tail).  On by default; MQ_STACK_PDL=0 turns it off, and a driver that rejects
// it together with the cooperative / cluster attributes turns it off for the process.
std::atomic<int> g_stack_pdl{-1};
bool stack_pdl() {
    int v = g_stack_pdl.load();
    if (v < 0) {
        const char* e = getenv("MQ_STACK_PDL");
        v = (e && e[0] == '0') ? 0 : 1;
        g_stack_pdl.store(v);
    }
    return v != 0;
}

template <int NT, int R, bool CHILD, bool XOPS = false>
cudaError_t launch_one_stack(const StackParams& p, int grid, size_t smem, cudaStream_t stream) {
    auto kern = k_stack<NT, R, CHILD, XOPS>;
    cudaError_t e = set_smem<NT, R, CHILD, XOPS>(smem);
    if (e != cudaSuccess) return e;
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3(grid);
    cfg.blockDim = dim3(kStackThreads);
    cfg.dynamicSmemBytes = smem;
    cfg.stream = stream;
    cudaLaunchAttribute attr[3];
    int n = 0;
    if (!(p.cluster && stack_nocoop())) {
        attr[n].id = cudaLaunchAttributeCooperative;
        attr[n].val.cooperative = 1;
        ++n;
    }
    if (p.cluster) {
        attr[n].id = cudaLaunchAttributeClusterDimension;
        attr[n].val.clusterDim.x = 2;
        attr[n].val.clusterDim.y = 1;
        attr[n].val.clusterDim.z = 1;
        ++n;
    }
    const bool pdl = stack_pdl();
    if (pdl) {
        attr[n].id = cudaLaunchAttributeProgrammaticStreamSerialization;
        attr[n].val.programmaticStreamSerializationAllowed = 1;
        ++n;
    }
    cfg.attrs = attr;
    cfg.numAttrs = n;
    e = cudaLaunchKernelEx(&cfg, kern, p);
    if (pdl && (e == cudaErrorInvalidValue || e == cudaErrorNotSupported)) {
        (void)cudaGetLastError();
        g_stack_pdl.store(0);
        cfg.numAttrs = n - 1;
        e = cudaLaunchKernelEx(&cfg, kern, p);
    }
    if (getenv("MQ_STACK_LAUNCH_DEBUG"))
        fprintf(stderr, "k_stack launch cluster=%d coop=%d pdl=%d grid=%d smem=%zu -> %s\n", p.cluster,
                !(p.cluster && stack_nocoop()), (int)stack_pdl(), grid, smem, cudaGetErrorString(e));
    return e;
}

template <int NT, int R, bool CHILD, bool XOPS = false>
int pair_capacity(size_t smem) {
    if (set_smem<NT, R, CHILD, XOPS>(smem) != cudaSuccess) return 0;
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3(2);
    cfg.blockDim = dim3(kStackThreads);
    cfg.dynamicSmemBytes = smem;
    cudaLaunchAttribute attr[1];
    attr[0].id = cudaLaunchAttributeClusterDimension;
    attr[0].val.clusterDim.x = 2;
    attr[0].val.clusterDim.y = 1;
    attr[0].val.clusterDim.z = 1;
    cfg.attrs = attr;
    cfg.numAttrs = 1;
    int n = 0;
    if (cudaOccupancyMaxActiveClusters(&n, k_stack<NT, R, CHILD, XOPS>, &cfg) != cudaSuccess) {
        (void)cudaGetLastError();
        return 0;
    }
    return 2 * n;
}
}  // namespace

template <int R>
cudaError_t launch_stack_r(const StackParams& p, int nt, bool child, int grid, size_t smem,
                           cudaStream_t stream) {
    constexpr bool kChildOk = R < 8;
    if (p.xops) {  // fused prologues: parents at NT = 1 only (the planner checks)
        if (nt != 1 || (child && kChildOk)) return cudaErrorInvalidValue;
        return launch_one_stack<1, R, false, true>(p, grid, smem, stream);
    }
    if (child && kChildOk) {
        if (nt == 1) return launch_one_stack<1, R, kChildOk>(p, grid, smem, stream);
        return launch_one_stack<2, R, kChildOk>(p, grid, smem, stream);
    }
    if (nt == 1) return launch_one_stack<1, R, false>(p, grid, smem, stream);
    return launch_one_stack<2, R, false>(p, grid, smem, stream);
}

cudaError_t launch_stack_mixed(const StackParams& p, int nt, int grid, size_t smem, cudaStream_t stream) {
    if (p.xops) {
        if (nt != 1) return cudaErrorInvalidValue;
        return launch_one_stack<1, 0, false, true>(p, grid, smem, stream);
    }
    if (nt == 1) return launch_one_stack<1, 0, false>(p, grid, smem, stream);
    return launch_one_stack<2, 0, false>(p, grid, smem, stream);
}

// Plan-time probe: launch the planned kernel with the planned attributes and no
// layers (it returns at entry) and report whether the driver accepts it.
cudaError_t stack_probe(int nt, int r, bool child, int grid, size_t smem, bool cluster, bool xops) {
    StackParams p{};
    p.n_layers = 0;
    p.cluster = cluster ? 1 : 0;
    p.xops = xops ? 1 : 0;
    cudaError_t e = r == 0 ? launch_stack_mixed(p, nt, grid, smem, 0) : cudaSuccess;
    if (r != 0) {
        switch (r) {
            case 2: e = launch_stack_r<2>(p, nt, child, grid, smem, 0); break;
            case 3: e = launch_stack_r<3>(p, nt, child, grid, smem, 0); break;
            case 4: e = launch_stack_r<4>(p, nt, child, grid, smem, 0); break;
            case 6: e = launch_stack_r<6>(p, nt, child, grid, smem, 0); break;
            default: e = launch_stack_r<8>(p, nt, child, grid, smem, 0); break;
        }
    }
    if (e == cudaSuccess) e = cudaStreamSynchronize(0);
    if (e != cudaSuccess) (void)cudaGetLastError();
    return e;
}

int stack_pair_capacity(int nt, int r, bool child, size_t smem, bool xops) {
    const bool c = child && r < 8;
    if (xops) {
        if (nt != 1 || c) return 0;  // c: a child slice (r < 8)
        switch (r) {
            case 0: return pair_capacity<1, 0, false, true>(smem);
            case 2: return pair_capacity<1, 2, false, true>(smem);
            case 3: return pair_capacity<1, 3, false, true>(smem);
            case 4: return pair_capacity<1, 4, false, true>(smem);
            case 6: return pair_capacity<1, 6, false, true>(smem);
            default: return pair_capacity<1, 8, false, true>(smem);
        }
    }
#define MQ_CAP(R)                                                                   \
    if (r == R) {                                                                   \
        if (nt == 1) return c ? pair_capacity<1, R, (R < 8)>(smem) : pair_capacity<1, R, false>(smem); \
        return c ? pair_capacity<2, R, (R < 8)>(smem) : pair_capacity<2, R, false>(smem);             \
    }
    MQ_CAP(2) MQ_CAP(3) MQ_CAP(4) MQ_CAP(6) MQ_CAP(8)
#undef MQ_CAP
    return nt == 1 ? pair_capacity<1, 0, false>(smem) : pair_capacity<2, 0, false>(smem);
}

template cudaError_t launch_stack_r<2>(const StackParams&, int, bool, int, size_t, cudaStream_t);
template cudaError_t launch_stack_r<3>(const StackParams&, int, bool, int, size_t, cudaStream_t);
template cudaError_t launch_stack_r<4>(const StackParams&, int, bool, int, size_t, cudaStream_t);
template cudaError_t launch_stack_r<6>(const StackParams&, int, bool, int, size_t, cudaStream_t);
template cudaError_t launch_stack_r<8>(const StackParams&, int, bool, int, size_t, cudaStream_t);

}  // namespace mq
