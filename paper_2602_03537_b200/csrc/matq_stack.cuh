// matq_stack.cuh -- K3S: the whole decode step (every sliced linear of a model)
// as ONE persistent kernel.
//
// The per-layer K3 launch pays a fixed ~4-5 us per layer (grid launch and
// drain, the dependent-launch release, the weight ring refilling from empty,
// activation staging, zero-point constants) -- about a third of a Llama-3.1-8B
// decode step (scripts/phase_timing.py).  K3S keeps one CTA per SM resident
// for the whole step and walks a table of layers (StackLayer, in HBM):
//   * every warp owns a TMA bulk-copy ring of weight steps whose issue cursor
//     runs across layer boundaries: while a layer's last tiles finish, the
//     next layer's first steps are already streaming into shared memory;
//   * layer l+1 reads layer l's output, so before staging its activations a
//     CTA waits until every CTA has published layer l: __syncthreads, thread
//     0 fence + atomicAdd on the layer's counter (release), and the waiter's
//     thread 0 spins on ld.acquire.gpu (the cooperative-groups grid.sync
//     pattern, per layer).  Counters only grow: launch g waits for
//     (g + 1) * gridDim.x, g taken from a launch counter at entry, so a graph
//     replays without resets.  Co-residency of all CTAs is guaranteed by a
//     cooperative launch;
//   * the per-layer work split, slice, decode, zero-point folding, mma.sync
//     and split-K fixup are K3's (matq_gemv.cuh) -- the same device code paths.
// G = 128.  Uniform stacks run k_stack<NT, R>; heterogeneous stacks (per-layer
// r, parents) run k_stack<NT, 0>, which dispatches each layer on its r.  TP
// stacks use per-layer K3 launches in a CUDA graph.
#pragma once
#include <cuda_fp16.h>

#include "matq_common.cuh"

namespace mq {

// Staging / decode mode of a stack layer (the planner mirrors it for the shared-memory
// budget): fp16 decode for r in {4, 8}, else bf16 with the zero point folded into a
// per-(group, row) constant (r != 8), both at one n-tile (B <= 8).  MQ_STACK_WIDE_ZP=1
// extends them to B <= 16: correct (tests pass) but measured 3-9x slower -- the extra
// activation copies for 16 rows crowd shared memory, so K splits many ways.
#ifndef MQ_STACK_WIDE_ZP
#define MQ_STACK_WIDE_ZP 0
#endif
__host__ __device__ constexpr bool stack_f16(int r, int nt) { return (r == 4 || r == 8) && (nt == 1 || MQ_STACK_WIDE_ZP); }
__host__ __device__ constexpr bool stack_zp(int r, int nt) {
    return stack_f16(r, nt) || (r != 8 && (nt == 1 || MQ_STACK_WIDE_ZP));
}

struct __align__(8) StackLayer {
    const uint32_t* blob;
    long long step_words;
    const uint16_t* X;  // bf16 [B][ldx] (read when xll is null: activations from outside the step)
    uint16_t* Y;        // bf16 [B][ldy]
    long long xll;  // word offset in StackParams::ll of the producing layer's LL output at X's first
                    // column, or -1 (X from outside the step: plain loads)
    long long yll;  // word offset of this layer's LL output [B][ldyll], or -1 (no later layer reads it)
    int ldx, ldy, ldxll, ldyll;     // ldxll / ldyll in 8-byte words
    int N, Np, K, nsteps, n_rt;
    int S, cs, cpc;  // K chunks, steps per chunk, CTAs per chunk
    float out_scale;
    int r;            // slice width (the mixed kernel dispatches on it)
    int stage_bytes;  // one ring stage: 128 B of scales + the planes read at r
    int ext_pub;      // X comes from outside the step and a later layer overwrites it: count the
                      // CTAs that finished staging it (done[l])
    int war_wait;     // this layer overwrites layer war_wait's external X: wait until every CTA staged it, or -1
    int cl_base;      // pair layers (S == 2, CTA pairs): first slot of this layer's buffer -- pair
                      // layers alternate between two, so a partner one layer ahead never waits
    int flat;         // S == 1, stream-K split: CTA c takes pairs [c fq + min(c, fr), ...) of the layer's
    int fq, fr;       // n_rt * nsteps (tile, step) pairs (tile-major) -- every CTA within one step
                      // of the mean; a tile cut by a CTA boundary is summed through fl_off
    long long fl_off;  // word offset in StackParams::ll of [grid][32 lanes][NT * 4] LL words: slot c
                       // holds CTA c + 1's part of CTA c's last tile
    int xop;          // activation prologue fused into staging (MQ_XOP_*: 0 none, 1 add + RMSNorm, 2 SiLU gating)
    const uint16_t* res_in;  // xop 1: bf16 residual [B][ldres], or null: the smem residual of the previous xop-1 layer
    uint16_t* res_out;       // xop 1: CTA 0 writes the updated residual here (or null)
    const float* norm_w;     // xop 1: RMSNorm weight [K]
    int ldres;
    float eps;
    int yop;          // MQ_YOP_SILU_PAIRS: rows interleaved 8 gate / 8 up per tile; Y = silu(g) * u, N / 2 wide
    int tk_off;       // S > 1 through the workspace: this layer's own tickets (StackParams::tickets + tk_off)
    long long ws_off;  // and its own partials (StackParams::ws + ws_off): no layer reuses another's, since
                       // without grid barriers a fast CTA may already be a layer ahead
};

struct StackParams {
    const StackLayer* layers;  // device array
    int n_layers;
    int B;
    int xs_stride;     // smem activation row stride (elements), max over layers
    int xcopy_stride;  // elements between activation copies
    int cs_off;        // byte offset of the zero-point constants
    int xs_bytes;      // bytes of the staging area (activations + constants + partial slots)
    int slot_off;      // byte offset of the per-warp partial-tile slots [16][32 lanes][NT * 4]
    int table_off;     // byte offset of the shared-memory copy of the layer table
    int stages;        // per-warp ring depth
    int stage_stride;  // bytes per ring slot (the largest stage of the stack)
    int cluster;       // 1: CTA pairs (cluster of 2); S == 2 layers reduce through DSMEM
    int res_off;       // xop-1 stacks: byte offset of the kept residual [B][res_k] bf16 ...
    int rpart_off;     // ... and of its per-(row, 128-column group) sums of squares [B][res_k / 128]
    int nw_off;        // ... and of the layer's RMSNorm weight [res_k] fp32 (copied by the pre-pass), or 0
    int res_k;
    int xops;          // some layer has a fused prologue: the XOPS kernel instantiation (NT = 1, parents)
    int cl_off;        // byte offset of the pair-reduction area: [cl_tiles mbarriers][cl_tiles use counters][slots]
    int cl_tiles;      // most row tiles a CTA holds in an S == 2 layer
    float* ws;         // split-K partials (per layer: StackLayer::ws_off)
    int* tickets;      // split-K tickets, self-resetting (per layer: StackLayer::tk_off)
    unsigned long long* done;  // [n_layers] monotone external-staging counters (64-bit: never wrap)
    unsigned long long* launch_ctr;
    unsigned long long* ll;      // LL activation words of every producing layer (workspace)
    unsigned long long* dbg_ts;  // MQ_GEMV_TIMING builds: [n_layers][148][8] globaltimer stamps
};

#ifdef MQ_GEMV_TIMING
__device__ __forceinline__ unsigned long long stack_gtimer() {
    unsigned long long t;
    asm volatile("mov.u64 %0, %globaltimer;" : "=l"(t));
    return t;
}
#define MQ_STS(l, ev) do { if (threadIdx.x == 0 && p.dbg_ts && blockIdx.x < 148) \
    p.dbg_ts[((size_t)(l) * 148 + blockIdx.x) * 8 + (ev)] = stack_gtimer(); } while (0)
#define MQ_STS_WMAX(l, ev) do { if ((threadIdx.x & 31) == 0 && p.dbg_ts && blockIdx.x < 148) \
    atomicMax(&p.dbg_ts[((size_t)(l) * 148 + blockIdx.x) * 8 + (ev)], stack_gtimer()); } while (0)
#else
#define MQ_STS_WMAX(l, ev) do { } while (0)
#define MQ_STS(l, ev) do { } while (0)
#endif

#ifndef MQ_PROD_SLEEP_NS
#define MQ_PROD_SLEEP_NS 0
#endif
#ifndef MQ_STACK_SPIN_NS
#define MQ_STACK_SPIN_NS 0
#endif
#ifndef MQ_LL_SPIN_NS
#define MQ_LL_SPIN_NS 0
#endif

constexpr int kStackWarps = 15;                      // consumer (decode + MMA) warps
constexpr int kStackThreads = (kStackWarps + 1) * 32;  // + one producer warp issuing every ring's bulk copies
constexpr int kConsumerThreads = kStackWarps * 32;

// A warp's share of one layer.  CTA c works on K chunk kc = c % S and the
// contiguous row tiles [ta, ta + ntiles) of that chunk (near-equal split over
// the chunk's cpc CTAs); its ntiles x ns (tile, step) pairs, flattened
// tile-major, are split into 15 contiguous ranges [f0, f1), one per ring warp
// (sized per SMSP, below).  A tile cut by a warp boundary is summed in warp
// order through shared memory; a tile cut by a chunk boundary (S > 1) through
// the CTA pair's shared memory (S = 2) or the split-K workspace and a ticket --
// all deterministic.
// SMSP-balanced split: warp w runs on SMSP w % 4, and SMSP 3 also hosts the
// producer warp, so it has 3 consumer warps to the others' 4.  The ALU pipe is
// per SMSP: consumer warps on SMSPs 0-2 take 3 units of work, those on SMSP 3
// MQ_SMSP3_UNITS (U(w) = units before warp w, kSplitUnits in all).
#ifndef MQ_SMSP3_UNITS
#define MQ_SMSP3_UNITS 3
#endif
constexpr int kSplitUnits = 3 * kStackWarps + (MQ_SMSP3_UNITS - 3) * (kStackWarps / 4);
__device__ __forceinline__ int warp_units(int w) { return 3 * w + (MQ_SMSP3_UNITS - 3) * (w >> 2); }
struct WarpPlan {
    int ta, ntiles, ns, chunk0, kc, f0, f1;
    int fo, P;  // the CTA's pairs are [fo, fo + P) (flat index over tiles ta.. x ns steps); f0, f1 too
};
// a / b for 0 <= a < 2^22, 0 < b: float reciprocal + one-step correction
// (~10 instructions; the compiler's 32/64-bit division sequences cost 20-60,
// and these sit on every warp's per-layer path)
__device__ __forceinline__ int udiv_small(int a, int b) {
    int q = __float2int_rz(__int2float_rn(a) * __frcp_rn(__int2float_rn(b)));
    q -= (q * b > a);
    q += ((q + 1) * b <= a);
    return q;
}
__device__ __forceinline__ WarpPlan warp_plan(const StackLayer& L, int cta, int warp) {
    WarpPlan w{};
    if (L.flat) {  // stream-K over the whole layer (K in one chunk)
        w.ns = L.nsteps;
        w.fo = cta * L.fq + min(cta, L.fr);
        w.P = L.fq + (cta < L.fr ? 1 : 0);
    } else {
        if (cta >= L.cpc * L.S) return w;
        const int j = udiv_small(cta, L.S);
        w.kc = cta - j * L.S;
        w.ta = udiv_small(j * L.n_rt, L.cpc);
        w.ntiles = udiv_small((j + 1) * L.n_rt, L.cpc) - w.ta;
        w.chunk0 = w.kc * L.cs;
        w.ns = max(0, min(w.chunk0 + L.cs, L.nsteps) - w.chunk0);
        w.P = w.ntiles * w.ns;
    }
    w.f0 = w.fo + warp_units(warp) * w.P / kSplitUnits;
    w.f1 = w.fo + warp_units(warp + 1) * w.P / kSplitUnits;
    return w;
}
// local (CTA-relative) start of warp v's range
__device__ __forceinline__ int plan_f0(const WarpPlan& w, int warp) {
    return warp_units(warp) * w.P / kSplitUnits;
}
// The last warp whose range starts at or before local step x: the largest v with
// floor(U(v) P / kSplitUnits) <= x, i.e. U(v) <= umax = ceil(kSplitUnits (x + 1) / P) - 1
// (never an empty warp); the estimate 4 umax / (9 + U3) is off by at most one.
__device__ __forceinline__ int last_warp_at(const WarpPlan& w, int x) {
    const int P = w.P;
    const int umax = udiv_small(kSplitUnits * (x + 1) + P - 1, P) - 1;
    int v = min(kStackWarps - 1, 4 * umax / (9 + MQ_SMSP3_UNITS));
    while (v > 0 && warp_units(v) > umax) --v;
    while (v < kStackWarps - 1 && warp_units(v + 1) <= umax) ++v;
    return v;
}
// Warps after wa holding a part of the tile ending at step f_last: those whose
// range starts inside the tile and is not empty (a CTA with fewer (tile, step)
// pairs than warps leaves some warps without work; they never arrive).
__device__ __forceinline__ int tile_parts(const WarpPlan& w, int wa, int f_last) {
    const int vmax = last_warp_at(w, f_last);
    constexpr int kMinUnits = MQ_SMSP3_UNITS < 3 ? MQ_SMSP3_UNITS : 3;
    // every warp has >= floor(P kMinUnits / kSplitUnits) >= 1 steps
    if (w.P * kMinUnits >= kSplitUnits) return vmax - wa;
    int n = 0;
    for (int v = wa + 1; v <= vmax; ++v) n += plan_f0(w, v) < plan_f0(w, v + 1);
    return n;
}

// Publish: bar.sync orders the CTA's writes before thread 0's release at gpu
// scope (cumulative), which the waiters' ld.acquire.gpu synchronises with.
__device__ __forceinline__ void red_release_add(unsigned long long* p, unsigned long long v) {
    asm volatile("red.release.gpu.global.add.u64 [%0], %1;" ::"l"(p), "l"(v) : "memory");
}
// Explicit global stores: Y's pointer comes from the shared-memory layer table,
// so a plain store would be GENERIC -- and a generic store is ordered behind the
// warp's in-flight bulk copies into shared memory (~HBM latency).
__device__ __forceinline__ void st_global_u16(uint16_t* p, uint16_t v) {
    asm volatile("st.global.u16 [%0], %1;" ::"l"(p), "h"(v) : "memory");
}
__device__ __forceinline__ void st_global_f32(float* p, float v) {
    asm volatile("st.global.f32 [%0], %1;" ::"l"(p), "f"(v) : "memory");
}
__device__ __forceinline__ void named_bar_arrive(int id, int nthreads) {
    asm volatile("bar.arrive %0, %1;" ::"r"(id), "r"(nthreads) : "memory");
}
__device__ __forceinline__ void named_bar_sync(int id, int nthreads) {
    asm volatile("bar.sync %0, %1;" ::"r"(id), "r"(nthreads) : "memory");
}
__device__ __forceinline__ void st_release_cta(uint32_t saddr, unsigned v) {
    asm volatile("st.release.cta.shared.u32 [%0], %1;" ::"r"(saddr), "r"(v) : "memory");
}
__device__ __forceinline__ unsigned ld_acquire_cta(uint32_t saddr) {
    unsigned v;
    asm volatile("ld.acquire.cta.shared.u32 %0, [%1];" : "=r"(v) : "r"(saddr) : "memory");
    return v;
}
__device__ __forceinline__ unsigned long long ld_acquire_u64(const unsigned long long* p) {
    unsigned long long v;
    asm volatile("ld.acquire.gpu.global.u64 %0, [%1];" : "=l"(v) : "l"(p) : "memory");
    return v;
}
// pair-slot credits: chunk 0 releases a consumed slot to chunk 1 across the cluster
__device__ __forceinline__ void mbar_arrive_remote(uint32_t raddr) {
    asm volatile("mbarrier.arrive.relaxed.cluster.shared::cluster.b64 _, [%0];" ::"r"(raddr) : "memory");
}
__device__ __forceinline__ void mbar_wait_cluster(uint32_t bar, uint32_t parity) {
    asm volatile(
        "{\n"
        ".reg .pred p;\n"
        "WAITC_%=:\n"
        "mbarrier.try_wait.parity.acquire.cluster.shared::cta.b64 p, [%0], %1;\n"
        "@!p bra WAITC_%=;\n"
        "}\n" ::"r"(bar),
        "r"(parity)
        : "memory");
}
// the consumer warps only (the producer warp runs ahead across layers): named
// barrier 0 with the consumer thread count (1..15 are the tile hand-off barriers)
__device__ __forceinline__ void consumer_sync() {
    asm volatile("bar.sync 0, %0;" ::"n"(kConsumerThreads) : "memory");
}
// every lane of a consumer warp arrives (count 32): its reads of the slot are
// released to the producer's next bulk copy into it
__device__ __forceinline__ void mbar_arrive(uint32_t bar) {
    asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(bar) : "memory");
}
__device__ __forceinline__ bool mbar_test(uint32_t bar, uint32_t parity) {
    uint32_t r;
    asm volatile(
        "{\n.reg .pred p;\n"
        "mbarrier.test_wait.parity.shared::cta.b64 p, [%1], %2;\n"
        "selp.u32 %0, 1, 0, p;\n}\n"
        : "=r"(r) : "r"(bar), "r"(parity) : "memory");
    return r != 0;
}

constexpr int kSyncThread = 0;  // consumer warp 0, lane 0: layer barrier wait + publish

// Per-consumer weight ring: the producer warp's lane c walks consumer c's
// (layer, flattened step) sequence across layer boundaries and issues each
// step's bulk copy into the next free slot of c's ring; each layer's stage is
// its own size (scales + its plane count) in slots of the plan's largest stage.
// Slot s of ring c has a full barrier (count 1 + transaction bytes, completed by
// the TMA engine) and an empty barrier (count 32: every lane of consumer c
// arrives once it has read the slot).
struct RingCtx {
    uint32_t full0, empty0, ring0, stride;  // this ring's barriers and slots
    int D;
    uint64_t policy;
    int cta, warp, n_layers;  // warp = the consumer this ring feeds
    const StackLayer* tab;
};
struct StackCursor {
    int il, iff, istage, itile, isi, insteps;
    uint32_t cyc;  // completed passes over the ring's slots
    WarpPlan ip;
    const uint32_t* iblob;
    const uint32_t* isrc;  // the next step's block
    long long isw;
    uint32_t ibytes;
};
__device__ __forceinline__ void cursor_next_layer(StackCursor& c, const RingCtx& rc) {
    for (++c.il; c.il < rc.n_layers; ++c.il) {  // the next layer with work for this consumer
        const StackLayer& L = rc.tab[c.il];
        c.ip = warp_plan(L, rc.cta, rc.warp);
        if (c.ip.f1 > c.ip.f0) {
            c.iblob = L.blob;
            c.isw = L.step_words;
            c.insteps = L.nsteps;
            c.ibytes = (uint32_t)L.stage_bytes;
            c.iff = c.ip.f0;
            const int t0 = udiv_small(c.ip.f0, c.ip.ns);
            c.itile = c.ip.ta + t0;
            c.isi = c.ip.f0 - t0 * c.ip.ns;
            c.isrc = c.iblob + ((long long)c.itile * c.insteps + c.ip.chunk0 + c.isi) * c.isw;
            return;
        }
    }
}
// Issue the cursor's next step into slot c.istage (the caller checked that the
// slot is free).  FIXB: the stage size when every layer's is the same (uniform
// kernels), else 0.
template <uint32_t FIXB>
__device__ __forceinline__ void cursor_issue(StackCursor& c, const RingCtx& rc) {
    const uint32_t bytes = FIXB ? FIXB : c.ibytes, stride = FIXB ? FIXB : rc.stride;
    const uint32_t* src = c.isrc;
    if (++c.isi == c.ip.ns) {
        c.isi = 0;
        ++c.itile;
        c.isrc = c.iblob + ((long long)c.itile * c.insteps + c.ip.chunk0) * c.isw;
    } else {
        c.isrc += c.isw;
    }
    const uint32_t bar = rc.full0 + 8 * c.istage;
    mbar_expect_tx(bar, bytes);
    bulk_g2s(rc.ring0 + c.istage * stride, src, bytes, bar, rc.policy);
    if (++c.istage == rc.D) {
        c.istage = 0;
        ++c.cyc;
    }
    if (++c.iff == c.ip.f1) cursor_next_layer(c, rc);
}

// The producer warp: lane c < 15 feeds consumer c.  A slot is reused once its
// consumer's previous pass released it (empty barrier phase cyc - 1).  Lanes
// advance independently; a round in which no lane can issue backs off briefly
// so the polling does not take issue slots from the consumers on this SMSP.
template <uint32_t FIXB>
__device__ __noinline__ void stack_producer(RingCtx rc) {
    const int lane = threadIdx.x & 31;
    StackCursor cur{};
    cur.il = -1;
    if (lane < kStackWarps) cursor_next_layer(cur, rc);
    else cur.il = rc.n_layers;
    for (;;) {
        const bool live = cur.il < rc.n_layers;
        if (!__any_sync(0xffffffffu, live)) break;
        bool issued = false;
        if (live && (cur.cyc == 0 || mbar_test(rc.empty0 + 8 * cur.istage, (cur.cyc - 1) & 1u))) {
            cursor_issue<FIXB>(cur, rc);
            issued = true;
        }
#if MQ_PROD_SLEEP_NS
        if (!__any_sync(0xffffffffu, issued)) __nanosleep(MQ_PROD_SLEEP_NS);
#else
        (void)issued;
#endif
    }
}

struct StackShared {
    unsigned long long gen;
    uint32_t tag;  // this step's LL tag, in [1, 2^32 - 1]
};

// LL (low-latency) activation hand-off between layers.  A layer whose output a
// later layer reads also stores it as 8-byte words {bf16 y[2i], bf16 y[2i+1],
// tag} (tag = this step's id); the consumer polls its words until every tag
// matches.  The data IS the flag (the LL protocol of NCCL): 8-byte accesses are
// single-copy atomic, so no grid barrier, no release/acquire fence and no
// counter polling sit between two layers, and a CTA starts layer l+1 as soon as
// the words of ITS K chunk exist.
__device__ __forceinline__ void st_ll(unsigned long long* p, uint32_t data, uint32_t tag) {
    asm volatile("st.relaxed.gpu.global.u64 [%0], %1;" ::"l"(p), "l"(((unsigned long long)tag << 32) | data)
                 : "memory");
}
__device__ __forceinline__ void ld_ll2(const unsigned long long* p, unsigned long long& a, unsigned long long& b) {
    asm volatile("ld.relaxed.gpu.global.v2.u64 {%0, %1}, [%2];" : "=l"(a), "=l"(b) : "l"(p) : "memory");
}

// 16 bf16 activations of row b from column col (LL words polled until tagged,
// or plain loads): lo / hi halves guarded by the caller's bounds
__device__ __forceinline__ void load_x16(const StackParams& p, const StackLayer& L, int b, int col, bool hi_ok,
                                         uint32_t tag, uint32_t (&w)[8]) {
    if (L.xll >= 0) {
        const unsigned long long* src = p.ll + L.xll + (long long)b * L.ldxll + (col >> 1);
        unsigned long long v[8];
#pragma unroll
        for (int i = 0; i < 8; ++i) v[i] = (unsigned long long)tag << 32;
        for (;;) {
            ld_ll2(src, v[0], v[1]);
            ld_ll2(src + 2, v[2], v[3]);
            if (hi_ok) {
                ld_ll2(src + 4, v[4], v[5]);
                ld_ll2(src + 6, v[6], v[7]);
            }
            bool ok = true;
#pragma unroll
            for (int i = 0; i < 8; ++i) ok = ok && (uint32_t)(v[i] >> 32) == tag;
            if (ok) break;
        }
#pragma unroll
        for (int i = 0; i < 8; ++i) w[i] = (uint32_t)v[i];
    } else {
        const uint16_t* src = L.X + (long long)b * L.ldx + col;
        const uint4 a = __ldcg(reinterpret_cast<const uint4*>(src));
        w[0] = a.x; w[1] = a.y; w[2] = a.z; w[3] = a.w;
        w[4] = w[5] = w[6] = w[7] = 0u;
        if (hi_ok) {
            const uint4 c = __ldcg(reinterpret_cast<const uint4*>(src + 8));
            w[4] = c.x; w[5] = c.y; w[6] = c.z; w[7] = c.w;
        }
    }
}

// bf16x2 silu(g) * u, rounded like torch (silu to bf16, then the product to bf16)
__device__ __forceinline__ uint32_t silu_mul_bf16x2(uint32_t g, uint32_t u) {
    const float g0 = __uint_as_float(g << 16), g1 = __uint_as_float(g & 0xFFFF0000u);
    const float s0 = bf16_to_f32(f32_to_bf16_rn(__fdividef(g0, 1.0f + __expf(-g0))));
    const float s1 = bf16_to_f32(f32_to_bf16_rn(__fdividef(g1, 1.0f + __expf(-g1))));
    return (uint32_t)f32_to_bf16_rn(s0 * __uint_as_float(u << 16)) |
           ((uint32_t)f32_to_bf16_rn(s1 * __uint_as_float(u & 0xFFFF0000u)) << 16);
}

// Add + RMSNorm prologue, pass 1 (consumer threads; the layer is one K chunk):
// R <- bf16(R + X) into the kept residual (R from res_in, or the residual the
// previous add-norm layer kept), and per (row, 128-column group) sums of R^2 --
// summed in group order by the staging pass (deterministic).
__device__ __forceinline__ void stack_addnorm_prepass(const StackParams& p, const StackLayer& L, uint32_t tag,
                                                      uint8_t* smem_base, int l) {
    constexpr int kOctets = kConsumerThreads / 8;
    const int ol = threadIdx.x & 7;
    const int ngroups = L.K >> 7;
    uint16_t* res = reinterpret_cast<uint16_t*>(smem_base + p.res_off);
    float* part = reinterpret_cast<float*>(smem_base + p.rpart_off);
    const int oct0 = (threadIdx.x >> 5) * 4;
    for (int base = oct0; base < p.B * ngroups; base += kOctets) {  // warp-uniform trip count
        const int task = base + ((threadIdx.x >> 3) & 3);
        const bool active = task < p.B * ngroups;
        const int b = active ? udiv_small(task, ngroups) : 0, grp = task - b * ngroups;
        const int col = (grp << 7) + (ol << 4);
        float ss = 0.0f;
        if (active) {
            uint32_t d[8], r[8];
            // everything that does not wait on the producing layer is issued before the
            // LL polling (its loads are ordered after it): the residual, and the RMSNorm
            // weights the staging pass reads (into L1)
            float4 nw4[4];
            if (b == 0 && p.nw_off) {  // the staging pass reads the RMSNorm weight from shared memory
#pragma unroll
                for (int i = 0; i < 4; ++i) nw4[i] = __ldg(reinterpret_cast<const float4*>(L.norm_w + col) + i);
            }
            if (L.res_in) {
                const uint16_t* src = L.res_in + (long long)b * L.ldres + col;
                const uint4 a = __ldcg(reinterpret_cast<const uint4*>(src)), c = __ldcg(reinterpret_cast<const uint4*>(src + 8));
                r[0] = a.x; r[1] = a.y; r[2] = a.z; r[3] = a.w; r[4] = c.x; r[5] = c.y; r[6] = c.z; r[7] = c.w;
            } else {
                const uint4 a = *reinterpret_cast<const uint4*>(res + b * p.res_k + col);
                const uint4 c = *reinterpret_cast<const uint4*>(res + b * p.res_k + col + 8);
                r[0] = a.x; r[1] = a.y; r[2] = a.z; r[3] = a.w; r[4] = c.x; r[5] = c.y; r[6] = c.z; r[7] = c.w;
            }
            load_x16(p, L, b, col, true, tag, d);
            MQ_STS_WMAX(l + 128, 0);  // delta arrived (timing builds)
            if (b == 0 && p.nw_off) {
                float4* nw = reinterpret_cast<float4*>(smem_base + p.nw_off) + (col >> 2);
#pragma unroll
                for (int i = 0; i < 4; ++i) nw[i] = nw4[i];
            }
            uint32_t o[8];
#pragma unroll
            for (int i = 0; i < 8; ++i) {
                const uint16_t v0 = f32_to_bf16_rn(__uint_as_float(r[i] << 16) + __uint_as_float(d[i] << 16));
                const uint16_t v1 = f32_to_bf16_rn(__uint_as_float(r[i] & 0xFFFF0000u) + __uint_as_float(d[i] & 0xFFFF0000u));
                const float f0 = bf16_to_f32(v0), f1 = bf16_to_f32(v1);
                ss += f0 * f0 + f1 * f1;
                o[i] = (uint32_t)v0 | ((uint32_t)v1 << 16);
            }
            *reinterpret_cast<uint4*>(res + b * p.res_k + col) = make_uint4(o[0], o[1], o[2], o[3]);
            *reinterpret_cast<uint4*>(res + b * p.res_k + col + 8) = make_uint4(o[4], o[5], o[6], o[7]);
        }
        __syncwarp();
        ss += __shfl_xor_sync(0xffffffffu, ss, 4);
        ss += __shfl_xor_sync(0xffffffffu, ss, 2);
        ss += __shfl_xor_sync(0xffffffffu, ss, 1);
        if (active && ol == 0) part[b * (p.res_k >> 7) + grp] = ss;
    }
    MQ_STS_WMAX(l + 128, 1);
}

// Stage X[:, chunk] into shared memory (consumer threads).  An octet of lanes
// takes one (batch row, 128-column group); each lane 16 columns.  From LL words
// (polled) or plain bf16 (X from outside the step).  Per mode:
//   F16  (r in {4, 8}, B <= 8): fp16 copies x * lambda_g * 2^-o with a power of
//        two lambda_g = 2^(14 - e) per (row, group), max|x| in [2^e, 2^(e+1))
//        (exact unless subnormal), and per (group, row) {c / lambda_g, 1 / lambda_g}
//        for the output: tot += s * (acc / lambda_g - c / lambda_g);
//   ZP   (bf16, r != 8, one n-tile): copies x * 2^-o and the zero-point constant;
//   else a plain copy.
template <int R, int NT, bool F16, bool ZP, int NCOPY, bool XOPS>
__device__ __forceinline__ void stack_stage(const StackParams& p, const StackLayer& L, uint16_t* xs, float* zc,
                                            int col_base, int Kc, uint32_t tag, const uint8_t* smem_base, int l) {
    constexpr int kOctets = kConsumerThreads / 8;
    const int ol = threadIdx.x & 7;
    const int ngroups = Kc >> 7;
    const int ntask = p.B * ngroups;
    // warp-uniform trip count (full-mask shuffles: a partial mask after the
    // divergent polling loop costs the compiler's divergent-shuffle path);
    // octets past the last task run the shuffles on zeros and store nothing
    const int oct0 = (threadIdx.x >> 5) * 4;
    for (int base = oct0; base < ntask; base += kOctets) {
        const int task = base + ((threadIdx.x >> 3) & 3);
        const bool active = task < ntask;
        const int b = active ? udiv_small(task, ngroups) : 0, grp = task - b * ngroups;
        const int c0 = (grp << 7) + (ol << 4);  // column inside the chunk
        const int col = col_base + c0;
        uint32_t w[8];
#pragma unroll
        for (int i = 0; i < 8; ++i) w[i] = 0u;
        const bool lo_ok = active && col < L.K, hi_ok = active && col + 8 < L.K;  // K % 8 == 0
        if (XOPS && L.xop == 1) {
            // X' = bf16(R * rsqrt(mean(R^2) + eps) * w); R (already R + delta) kept in smem by the pre-pass
            if (lo_ok) {
                const uint16_t* rr = reinterpret_cast<const uint16_t*>(smem_base + p.res_off) + b * p.res_k + col;
                const float* part = reinterpret_cast<const float*>(smem_base + p.rpart_off) + b * (p.res_k >> 7);
                // fixed order (deterministic, the same in every thread); K % 512 == 0 takes
                // float4 loads (part is 16-byte aligned per row when res_k % 512 == 0)
                float ss = 0.0f;
                const int ng = L.K >> 7;
                if ((ng & 3) == 0 && ((p.res_k >> 7) & 3) == 0) {
                    float4 acc = make_float4(0.f, 0.f, 0.f, 0.f);
                    for (int gi = 0; gi < ng; gi += 4) {
                        const float4 v = *reinterpret_cast<const float4*>(part + gi);
                        acc.x += v.x; acc.y += v.y; acc.z += v.z; acc.w += v.w;
                    }
                    ss = (acc.x + acc.y) + (acc.z + acc.w);
                } else {
                    for (int gi = 0; gi < ng; ++gi) ss += part[gi];
                }
                const float inv = rsqrtf(ss / (float)L.K + L.eps);
                MQ_STS_WMAX(l + 128, 3);
                const uint4 r0 = *reinterpret_cast<const uint4*>(rr), r1 = *reinterpret_cast<const uint4*>(rr + 8);
                const uint32_t rw[8] = {r0.x, r0.y, r0.z, r0.w, r1.x, r1.y, r1.z, r1.w};
                const float4* nw4 = p.nw_off ? reinterpret_cast<const float4*>(smem_base + p.nw_off) + (col >> 2)
                                             : reinterpret_cast<const float4*>(L.norm_w + col);
                float nw[16];
#pragma unroll
                for (int i = 0; i < 4; ++i) {
                    const float4 v = nw4[i];
                    nw[4 * i] = v.x; nw[4 * i + 1] = v.y; nw[4 * i + 2] = v.z; nw[4 * i + 3] = v.w;
                }
#pragma unroll
                for (int i = 0; i < 8; ++i) {
                    const float a = __uint_as_float(rw[i] << 16) * inv * nw[2 * i];
                    const float c = __uint_as_float(rw[i] & 0xFFFF0000u) * inv * nw[2 * i + 1];
                    w[i] = (uint32_t)f32_to_bf16_rn(a) | ((uint32_t)f32_to_bf16_rn(c) << 16);
                }
                MQ_STS_WMAX(l + 128, 4);
            }
        } else if (XOPS && L.xop == 2 && L.xll >= 0) {
            // SiLU gating from LL words: g (columns col..) and u (K columns further) in one poll
            uint32_t u[8];
            if (lo_ok) {
                const unsigned long long* sg = p.ll + L.xll + (long long)b * L.ldxll + (col >> 1);
                const unsigned long long* su = sg + (L.K >> 1);
                unsigned long long v[16];
#pragma unroll
                for (int i = 0; i < 16; ++i) v[i] = (unsigned long long)tag << 32;
                for (;;) {
                    ld_ll2(sg, v[0], v[1]);
                    ld_ll2(sg + 2, v[2], v[3]);
                    ld_ll2(su, v[8], v[9]);
                    ld_ll2(su + 2, v[10], v[11]);
                    if (hi_ok) {
                        ld_ll2(sg + 4, v[4], v[5]);
                        ld_ll2(sg + 6, v[6], v[7]);
                        ld_ll2(su + 4, v[12], v[13]);
                        ld_ll2(su + 6, v[14], v[15]);
                    }
                    bool ok = true;
#pragma unroll
                    for (int i = 0; i < 16; ++i) ok = ok && (uint32_t)(v[i] >> 32) == tag;
                    if (ok) break;
                }
#pragma unroll
                for (int i = 0; i < 8; ++i) {
                    w[i] = (uint32_t)v[i];
                    u[i] = (uint32_t)v[8 + i];
                }
#pragma unroll
                MQ_STS_WMAX(l + 128, 4);  // g and u arrived
#pragma unroll
                for (int i = 0; i < 8; ++i) w[i] = silu_mul_bf16x2(w[i], u[i]);
                MQ_STS_WMAX(l + 128, 5);
            }
        } else if (L.xll >= 0) {
            const unsigned long long* src = p.ll + L.xll + (long long)b * L.ldxll + (col >> 1);
            unsigned long long v[8];
#pragma unroll
            for (int i = 0; i < 8; ++i) v[i] = (unsigned long long)tag << 32;
            for (;;) {
                if (lo_ok) {
                    ld_ll2(src, v[0], v[1]);
                    ld_ll2(src + 2, v[2], v[3]);
                }
                if (hi_ok) {
                    ld_ll2(src + 4, v[4], v[5]);
                    ld_ll2(src + 6, v[6], v[7]);
                }
                bool ok = true;
#pragma unroll
                for (int i = 0; i < 8; ++i) ok = ok && (uint32_t)(v[i] >> 32) == tag;
                if (ok) break;
#if MQ_LL_SPIN_NS
                __nanosleep(MQ_LL_SPIN_NS);  // fewer L2 polls while the producing CTAs finish
#endif
            }
#pragma unroll
            for (int i = 0; i < 8; ++i) w[i] = (uint32_t)v[i];
            MQ_STS_WMAX(l + 128, 4);  // X arrived
        } else {
            const uint16_t* src = L.X + (long long)b * L.ldx + col;
            if (lo_ok) {
                const uint4 a = __ldcg(reinterpret_cast<const uint4*>(src));
                w[0] = a.x; w[1] = a.y; w[2] = a.z; w[3] = a.w;
            }
            if (hi_ok) {
                const uint4 a = __ldcg(reinterpret_cast<const uint4*>(src + 8));
                w[4] = a.x; w[5] = a.y; w[6] = a.z; w[7] = a.w;
            }
        }
        if (XOPS && L.xop == 2 && L.xll < 0 && lo_ok) {  // SiLU gating, X from outside the step
            uint32_t u[8];
            load_x16(p, L, b, col + L.K, hi_ok, tag, u);
#pragma unroll
            for (int i = 0; i < 8; ++i) w[i] = silu_mul_bf16x2(w[i], u[i]);
        }
        __syncwarp();
        uint16_t* dst = xs + b * p.xs_stride + c0;
        float x[16];
#pragma unroll
        for (int i = 0; i < 8; ++i) {
            x[2 * i] = __uint_as_float(w[i] << 16);
            x[2 * i + 1] = __uint_as_float(w[i] & 0xFFFF0000u);
        }
        if constexpr (F16) {
            float m = 0.0f;
#pragma unroll
            for (int i = 0; i < 16; ++i) m = fmaxf(m, fabsf(x[i]));
            m = fmaxf(m, __shfl_xor_sync(0xffffffffu, m, 4));
            m = fmaxf(m, __shfl_xor_sync(0xffffffffu, m, 2));
            m = fmaxf(m, __shfl_xor_sync(0xffffffffu, m, 1));
            // lambda = 2^(14 - e): max|x| lambda < 2^15 < 65504 (fp16 max); e from the
            // exponent field (m = 0: e = 0; clamped so lambda and 1 / lambda stay normal)
            const int e = m > 0.0f ? max(-100, (int)((__float_as_uint(m) >> 23) & 0xFF) - 127) : 0;
            const float lam = __uint_as_float((uint32_t)(127 + 14 - e) << 23);
            const float il = __uint_as_float((uint32_t)(127 - 14 + e) << 23);
            const int o = zp_off16<R>(((c0 & 255) & 63) >> 4);  // one field offset per 16 columns
            float part = 0.0f;
#pragma unroll
            for (int cp = 0; cp < NCOPY; ++cp) {
                const int oc = cp ? 4 : 0;
                const float f = lam / (float)(1 << oc);
                float y[16];
#pragma unroll
                for (int i = 0; i < 16; ++i) y[i] = x[i] * f;  // exact in fp16 unless subnormal
                uint32_t hw[8];
#pragma unroll
                for (int i = 0; i < 8; ++i) {
                    const __half2 h2 = __floats2half2_rn(y[2 * i], y[2 * i + 1]);
                    hw[i] = *reinterpret_cast<const uint32_t*>(&h2);
                }
                if (active) {
                    uint4* d = reinterpret_cast<uint4*>(dst + cp * p.xcopy_stride);
                    d[0] = make_uint4(hw[0], hw[1], hw[2], hw[3]);
                    d[1] = make_uint4(hw[4], hw[5], hw[6], hw[7]);
                }
                // the constant uses the values the MMA sees: (1024 + z 2^o) x' (pairwise sum)
                if (oc == o) {
#pragma unroll
                    for (int st = 8; st >= 1; st >>= 1)
#pragma unroll
                        for (int i = 0; i < st; ++i) y[i] += y[i + st];
                    part = y[0];
                }
            }
            part *= 1024.0f + (float)((1 << (R - 1)) << o);
            part += __shfl_xor_sync(0xffffffffu, part, 4);
            part += __shfl_xor_sync(0xffffffffu, part, 2);
            part += __shfl_xor_sync(0xffffffffu, part, 1);
            if (active && ol == 0) {
                float* z = zc + ((c0 >> 7) * (NT * 8) + b) * 2;
                z[0] = part * il;
                z[1] = il;
            }
        } else {
            if (active) {
                uint4* d = reinterpret_cast<uint4*>(dst);
                d[0] = make_uint4(w[0], w[1], w[2], w[3]);
                d[1] = make_uint4(w[4], w[5], w[6], w[7]);
            }
            if constexpr (ZP) {
                // zero-point constant of the 128-column group: sum (128 2^-o + z) x; each
                // 8 columns share the field offset o
                float part = 0.0f;
#pragma unroll
                for (int h = 0; h < 2; ++h) {
                    const int cs_ = (c0 + 8 * h) & 255;
                    const int o = zp_off<R>((cs_ & 63) >> 4, (cs_ & 15) >> 3);
                    const float mo = 128.0f / (float)(1 << o) + (float)(1 << (R - 1));
                    const float sx = ((x[8 * h] + x[8 * h + 1]) + (x[8 * h + 2] + x[8 * h + 3])) +
                                     ((x[8 * h + 4] + x[8 * h + 5]) + (x[8 * h + 6] + x[8 * h + 7]));
                    part += sx * mo;
                }
                part += __shfl_xor_sync(0xffffffffu, part, 4);
                part += __shfl_xor_sync(0xffffffffu, part, 2);
                part += __shfl_xor_sync(0xffffffffu, part, 1);
                if (active && ol == 0) zc[(c0 >> 7) * (NT * 8) + b] = part;
            }
            if constexpr (NCOPY > 1) {
                if (active) {
#pragma unroll
                    for (int cp = 1; cp < NCOPY; ++cp) {
                        const float f = 1.0f / (float)(1 << zp_copy_off(R, cp));
                        uint32_t o2[8];
#pragma unroll
                        for (int i = 0; i < 8; ++i)
                            o2[i] = (uint32_t)f32_to_bf16_rn(x[2 * i] * f) |
                                    ((uint32_t)f32_to_bf16_rn(x[2 * i + 1] * f) << 16);
                        uint4* dc = reinterpret_cast<uint4*>(dst + cp * p.xcopy_stride);
                        dc[0] = make_uint4(o2[0], o2[1], o2[2], o2[3]);
                        dc[1] = make_uint4(o2[4], o2[5], o2[6], o2[7]);
                    }
                }
            }
        }
    }
}

// One layer of the step, slice width R.  Uniform stacks instantiate k_stack
// with R fixed; heterogeneous stacks (an EvoPress configuration: per-layer r)
// dispatch here on the layer table's r -- the ring and cursor are shared.
template <int R, int NT, bool CHILD, bool FIXED, bool XOPS>
__device__ __forceinline__ void stack_layer(const StackParams& p, const StackLayer* tab, int l,
                                            const RingCtx& rc, int& cstage, uint32_t& parity,
                                            StackShared& sh, uint8_t* smem, unsigned long long target) {
    constexpr int NPL = PlaneCount<R, CHILD>::value;
    constexpr uint32_t kSlab = 512, kScaleBytes = 128;
    constexpr uint32_t kStage = kScaleBytes + NPL * kSlab;
    const uint32_t stride = FIXED ? kStage : rc.stride;
    // fp16 decode (r in {4, 8}, B <= 8): fp16's 10-bit mantissa takes a nibble at
    // offsets 0 and 4 and a whole byte at 0, cutting the decode's ALU work by
    // 15-24% (scripts/micro/decode_rate.cu); activations are staged as fp16
    // scaled by a per-CTA power of two (exact; keeps them inside fp16's range)
    constexpr bool F16 = stack_f16(R, NT);
    constexpr bool ZP = stack_zp(R, NT);  // see k_gemv
    constexpr int NCOPY = F16 ? (R == 4 ? 2 : 1) : (ZP ? zp_ncopies(R) : 1);
    uint16_t* xs = reinterpret_cast<uint16_t*>(smem);
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int g = lane >> 2, t = lane & 3;
    const int D = rc.D;
    const uint32_t xs_saddr = smem_addr(xs);
    float* zc = reinterpret_cast<float*>(smem + p.cs_off);  // [2 cs groups][NT * 8] zero-point constants

    const StackLayer& L = tab[l];
    const WarpPlan wp = warp_plan(L, rc.cta, warp);
    const int Kc = L.cs * kStepCols;
    const int col_base = wp.chunk0 * kStepCols;  // every warp of the CTA shares its chunk

    // ---- stage X[:, chunk]: polls the producing layer's LL words ------------
    // (the previous layer's readers of the staging area are done: the
    // consumer_sync that ends every layer)
    MQ_STS(l, 0);
    if (XOPS && L.xop == 1) {  // add + RMSNorm: the residual update and the row sums first
        stack_addnorm_prepass(p, L, sh.tag, smem, l);
        consumer_sync();
        MQ_STS(l + 128, 2);
    }
    stack_stage<R, NT, F16, ZP, NCOPY, XOPS>(p, L, xs, zc, col_base, Kc, sh.tag, smem, l);
    MQ_STS_WMAX(l, 1);  // this warp's staging tasks done (max over warps)
    if (threadIdx.x == kSyncThread && L.war_wait >= 0 && L.war_wait < l) {
        // this layer overwrites a buffer an earlier layer read from outside the
        // step: every CTA must have staged it (almost always long done)
        while (ld_acquire_u64(p.done + L.war_wait) < target) {
        }
    }
    consumer_sync();
    if (L.ext_pub) {
        if (threadIdx.x == kSyncThread) red_release_add(p.done + l, 1ull);
        if (L.war_wait == l) {  // writes over its own external X: every CTA staged it first
            if (threadIdx.x == kSyncThread)
                while (ld_acquire_u64(p.done + l) < target) {
                }
            consumer_sync();
        }
    }
    if (XOPS && L.res_out && blockIdx.x == 0) {  // the updated residual for the next kernel (after the WAR wait)
        const uint16_t* res = reinterpret_cast<const uint16_t*>(smem + p.res_off);
        for (int i = threadIdx.x; i < p.B * (L.K >> 3); i += kConsumerThreads) {
            const int b = udiv_small(i, L.K >> 3), c = (i - b * (L.K >> 3)) * 8;
            *reinterpret_cast<uint4*>(L.res_out + (long long)b * L.ldres + c) =
                *reinterpret_cast<const uint4*>(res + b * p.res_k + c);
        }
    }
    MQ_STS(l, 2);

    uint32_t xrow_addr[NT][2];
#pragma unroll
    for (int nt = 0; nt < NT; ++nt) {
        int n = nt * 8 + (lane & 7);
        if (n >= p.B) n = 0;
#pragma unroll
        for (int s2 = 0; s2 < 2; ++s2) {
            const int mi = lane >> 3;
            int cp = 0;
            if constexpr (F16) {
                cp = zp_off16<R>(2 * s2 + (mi >> 1)) ? 1 : 0;
            } else if constexpr (ZP) {
                const int sx = 2 * s2 + (mi >> 1), hx = mi & 1;
                cp = zp_copy_of(R, zp_off<R>(sx, hx));
            }
            xrow_addr[nt][s2] = xs_saddr + (uint32_t)(cp * p.xcopy_stride + n * p.xs_stride + 8 * mi) * 2u;
        }
    }


    // ---- this warp's units of layer l --------------------------------------
    float tot[NT][4], acc[NT][4];
    auto process = [&](const uint4 (&buf)[NPL], const float (&sc)[4], uint32_t xcol) {
#pragma unroll
        for (int w = 0; w < 4; ++w) {
            uint32_t T[NPL];
#pragma unroll
            for (int jj = 0; jj < NPL; ++jj) T[jj] = word_of(buf[jj], w);
            uint32_t A[16];
            uint32_t Sl[R];
            slice_loaded<R, CHILD>(T, Sl);
            if constexpr (F16) decode_word_f16<R>(Sl, A);
            else decode_word<R, ZP>(Sl, A);
#pragma unroll
            for (int s2 = 0; s2 < 2; ++s2) {
                uint32_t bf[NT][4];
#pragma unroll
                for (int nt = 0; nt < NT; ++nt)
                    ldmatrix_x4(bf[nt], xrow_addr[nt][s2] + (xcol + 64 * w + 32 * s2) * 2u);
#pragma unroll
                for (int sh2 = 0; sh2 < 2; ++sh2) {
                    const int s = 2 * s2 + sh2;
#pragma unroll
                    for (int nt = 0; nt < NT; ++nt) {
                        if constexpr (F16) {
                            if ((w & 1) == 0 && s == 0)
                                mma_zero_f16(acc[nt], A[4 * s], A[4 * s + 1], A[4 * s + 2], A[4 * s + 3],
                                             bf[nt][2 * sh2], bf[nt][2 * sh2 + 1]);
                            else
                                mma_acc_f16(acc[nt], A[4 * s], A[4 * s + 1], A[4 * s + 2], A[4 * s + 3],
                                            bf[nt][2 * sh2], bf[nt][2 * sh2 + 1]);
                        } else {
                            if ((w & 1) == 0 && s == 0)
                                mma_zero(acc[nt], A[4 * s], A[4 * s + 1], A[4 * s + 2], A[4 * s + 3],
                                         bf[nt][2 * sh2], bf[nt][2 * sh2 + 1]);
                            else
                                mma_acc(acc[nt], A[4 * s], A[4 * s + 1], A[4 * s + 2], A[4 * s + 3],
                                        bf[nt][2 * sh2], bf[nt][2 * sh2 + 1]);
                        }
                    }
                }
            }
            if (w & 1) {
                const float s_lo = sc[(w >> 1) * 2], s_hi = sc[(w >> 1) * 2 + 1];
#pragma unroll
                for (int nt = 0; nt < NT; ++nt) {
                    if constexpr (F16) {
                        // {c / lambda_g, 1 / lambda_g} per batch row (stack_stage)
                        const float4 z = *reinterpret_cast<const float4*>(
                            zc + (((int)(xcol >> 7) + (w >> 1)) * (NT * 8) + nt * 8 + 2 * t) * 2);
                        tot[nt][0] = fmaf(s_lo, fmaf(z.y, acc[nt][0], -z.x), tot[nt][0]);
                        tot[nt][1] = fmaf(s_lo, fmaf(z.w, acc[nt][1], -z.z), tot[nt][1]);
                        tot[nt][2] = fmaf(s_hi, fmaf(z.y, acc[nt][2], -z.x), tot[nt][2]);
                        tot[nt][3] = fmaf(s_hi, fmaf(z.w, acc[nt][3], -z.z), tot[nt][3]);
                    } else if constexpr (ZP) {
                        const float* zp = zc + ((int)(xcol >> 7) + (w >> 1)) * (NT * 8) + nt * 8 + 2 * t;
                        const float c0 = zp[0], c1 = zp[1];
                        tot[nt][0] = fmaf(s_lo, acc[nt][0] - c0, tot[nt][0]);
                        tot[nt][1] = fmaf(s_lo, acc[nt][1] - c1, tot[nt][1]);
                        tot[nt][2] = fmaf(s_hi, acc[nt][2] - c0, tot[nt][2]);
                        tot[nt][3] = fmaf(s_hi, acc[nt][3] - c1, tot[nt][3]);
                    } else {
                        tot[nt][0] = fmaf(s_lo, acc[nt][0], tot[nt][0]);
                        tot[nt][1] = fmaf(s_lo, acc[nt][1], tot[nt][1]);
                        tot[nt][2] = fmaf(s_hi, acc[nt][2], tot[nt][2]);
                        tot[nt][3] = fmaf(s_hi, acc[nt][3], tot[nt][3]);
                    }
                }
            }
        }
    };
    // write a finished 16-row tile: Y (S == 1) or the chunk's split-K partial +
    // ticket, the last chunk to arrive summing the partials in chunk order
    const float out_scale_l = L.out_scale;
    const bool pair = p.cluster && L.S == 2;
    // the final values of a tile (row r0 + 8h, batch nt * 8 + 2t + c in v[nt][2h + c]):
    // plain bf16 Y and, when a later layer reads it, the LL words (row pairs)
    auto store_final = [&](int rt, const float (&v)[NT][4]) {
        if (XOPS && L.yop) {
            // gated output: lane (g, t) holds gate row g (h = 0) and its up row g + 8 (h = 1)
            // of tile rt for batch columns 2t, 2t + 1 -> act row 8 rt + g
            const int a = rt * 8 + g;
            uint16_t ab[NT][2];
#pragma unroll
            for (int nt = 0; nt < NT; ++nt)
#pragma unroll
                for (int c = 0; c < 2; ++c) {
                    const uint32_t gw = f32_to_bf16_rn(v[nt][c]), uw = f32_to_bf16_rn(v[nt][2 + c]);
                    const uint32_t o = silu_mul_bf16x2(gw, uw) & 0xFFFFu;
                    ab[nt][c] = (uint16_t)o;
                    const int b = nt * 8 + 2 * t + c;
                    if (b < p.B && 2 * a < L.N) st_global_u16(L.Y + (long long)b * L.ldy + a, ab[nt][c]);
                }
            if (L.yll >= 0) {
                // act rows (a, a + 1) pair up across lanes g, g + 1 (lane ^ 4): even g writes
#pragma unroll
                for (int nt = 0; nt < NT; ++nt)
#pragma unroll
                    for (int c = 0; c < 2; ++c) {
                        const uint32_t nb = __shfl_xor_sync(0xffffffffu, (uint32_t)ab[nt][c], 4);
                        const int b = nt * 8 + 2 * t + c;
                        if ((g & 1) == 0 && b < p.B && 2 * a < L.N)
                            st_ll(p.ll + L.yll + (long long)b * L.ldyll + (a >> 1), (uint32_t)ab[nt][c] | (nb << 16),
                                  sh.tag);
                    }
            }
            return;
        }
        const int r0 = rt * kTileRows + g;
        uint16_t yb[NT][4];
#pragma unroll
        for (int nt = 0; nt < NT; ++nt)
#pragma unroll
            for (int h = 0; h < 2; ++h)
#pragma unroll
                for (int c = 0; c < 2; ++c) {
                    const int row = r0 + 8 * h, b = nt * 8 + 2 * t + c;
                    yb[nt][2 * h + c] = f32_to_bf16_rn(v[nt][2 * h + c]);
                    if (b < p.B && row < L.N) st_global_u16(L.Y + (long long)b * L.ldy + row, yb[nt][2 * h + c]);
                }
        if (L.yll >= 0) {
            // even g: rows (g, g+1) from its h = 0 value and lane g+1's; odd g: rows (g+7, g+8)
            const bool odd = (g & 1) != 0;
            const int start = rt * kTileRows + (odd ? g + 7 : g);
#pragma unroll
            for (int nt = 0; nt < NT; ++nt)
#pragma unroll
                for (int c = 0; c < 2; ++c) {
                    const uint32_t send = odd ? yb[nt][c] : yb[nt][2 + c];
                    const uint32_t recv = __shfl_xor_sync(0xffffffffu, send, 4);
                    const uint32_t word = odd ? (recv | ((uint32_t)yb[nt][2 + c] << 16))
                                              : ((uint32_t)yb[nt][c] | (recv << 16));
                    const int b = nt * 8 + 2 * t + c;
                    if (b < p.B && start < L.N) st_ll(p.ll + L.yll + (long long)b * L.ldyll + (start >> 1), word, sh.tag);
                }
        }
    };
    auto emit = [&](int rt, const float (&v)[NT][4]) {
        if (pair) {
            const int li = L.cl_base + rt - wp.ta;  // this pair layer's slot buffer
            const uint32_t cl = smem_addr(smem + p.cl_off);
            const uint32_t bar = cl + 8 * li;
            const uint32_t slot = cl + 32u * p.cl_tiles + (uint32_t)((li * 32 + lane) * NT * 16);
            if (wp.kc == 1) {  // chunk 1: ship the scaled partial to chunk 0
                // credit: chunk 0 has consumed this slot's previous partial (no grid
                // barrier orders the two CTAs' layers any more)
                unsigned* fuses = reinterpret_cast<unsigned*>(smem + p.cl_off + 24 * p.cl_tiles);
                uint32_t fu = 0;
                if (lane == 0) {
                    fu = fuses[li];
                    fuses[li] = fu + 1u;
                }
                fu = __shfl_sync(0xffffffffu, fu, 0);
                if (fu > 0) mbar_wait_cluster(cl + 16 * p.cl_tiles + 8 * li, (fu - 1u) & 1u);
                const uint32_t rbar = mapa_rank(bar, 0), rslot = mapa_rank(slot, 0);
#pragma unroll
                for (int nt = 0; nt < NT; ++nt)
                    st_async_v4(rslot + 16 * nt, v[nt][0] * out_scale_l, v[nt][1] * out_scale_l,
                                v[nt][2] * out_scale_l, v[nt][3] * out_scale_l, rbar);
                return;
            }
            // chunk 0: arm the tile's barrier (its use count gives the phase), wait, add in chunk order
            unsigned* uses = reinterpret_cast<unsigned*>(smem + p.cl_off + 8 * p.cl_tiles);
            uint32_t par = 0;
            if (lane == 0) {
                par = uses[li] & 1u;
                uses[li] = uses[li] + 1u;
                mbar_expect_tx(bar, 32u * NT * 16u);
            }
            par = __shfl_sync(0xffffffffu, par, 0);
            mbar_wait(bar, par);
            float fin[NT][4];
#pragma unroll
            for (int nt = 0; nt < NT; ++nt) {
                const uint4 q = lds128(slot + 16 * nt);
                fin[nt][0] = v[nt][0] * out_scale_l + __uint_as_float(q.x);
                fin[nt][1] = v[nt][1] * out_scale_l + __uint_as_float(q.y);
                fin[nt][2] = v[nt][2] * out_scale_l + __uint_as_float(q.z);
                fin[nt][3] = v[nt][3] * out_scale_l + __uint_as_float(q.w);
            }
            store_final(rt, fin);
            // slot free: every lane's slot loads fed its Y stores, which are issued (in
            // order) before this point, so a relaxed arrive cannot overtake the reads --
            // a release would also wait for the global stores to complete (~1 us)
            __syncwarp();
            if (lane == 0) mbar_arrive_remote(mapa_rank(cl + 16 * p.cl_tiles + 8 * li, 1));
            return;
        }
        if (L.S == 1) {
            float fin[NT][4];
#pragma unroll
            for (int nt = 0; nt < NT; ++nt)
#pragma unroll
                for (int i = 0; i < 4; ++i) fin[nt][i] = v[nt][i] * out_scale_l;
            store_final(rt, fin);
            return;
        }
        const int r0 = rt * kTileRows + g;
#pragma unroll
        for (int nt = 0; nt < NT; ++nt)
#pragma unroll
            for (int h = 0; h < 2; ++h)
#pragma unroll
                for (int c = 0; c < 2; ++c) {
                    const int row = r0 + 8 * h, b = nt * 8 + 2 * t + c;
                    if (b < p.B && row < L.N)
                        st_global_f32(p.ws + L.ws_off + ((long long)wp.kc * p.B + b) * L.Np + row, v[nt][2 * h + c] * out_scale_l);
                }
        __syncwarp();
        int last = 0;
        // lane 1: lane 0's in-flight bulk copies would delay an acq_rel RMW
        if (lane == 1) last = (atom_add_acq_rel(p.tickets + L.tk_off + rt, 1) == L.S - 1);
        last = __shfl_sync(0xffffffffu, last, 1);
        if (!last) return;
        float fin[NT][4];
#pragma unroll
        for (int nt = 0; nt < NT; ++nt)
#pragma unroll
            for (int h = 0; h < 2; ++h)
#pragma unroll
                for (int c = 0; c < 2; ++c) {
                    const int row = r0 + 8 * h, b = nt * 8 + 2 * t + c;
                    float sum = 0.0f;
                    if (b < p.B && row < L.N) {
                        const float* wq = p.ws + L.ws_off + (long long)b * L.Np + row;
                        const long long cstride = (long long)p.B * L.Np;
                        int q = 0;
                        for (; q + 4 <= L.S; q += 4) {
                            const float a0 = __ldcg(wq + q * cstride), a1 = __ldcg(wq + (q + 1) * cstride);
                            const float a2 = __ldcg(wq + (q + 2) * cstride), a3 = __ldcg(wq + (q + 3) * cstride);
                            sum += a0; sum += a1; sum += a2; sum += a3;
                        }
                        for (; q < L.S; ++q) sum += __ldcg(wq + q * cstride);
                    }
                    fin[nt][2 * h + c] = sum;
                }
        store_final(rt, fin);
        __syncwarp();
        if (lane == 0) p.tickets[L.tk_off + rt] = 0;
    };
    // A tile cut by warp boundaries (warps wa < ... < wb) is emitted by wa, the
    // warp holding its first step: that is wa's LAST segment, so wa finishes it
    // last.  wa+1..wb park their parts in their slot (only their FIRST segment
    // can be such a part) and raise their flag; wa adds them in warp order.
    float* slots = reinterpret_cast<float*>(smem + p.slot_off);
    auto slot_ptr = [&](int w) { return slots + (w * 32 + lane) * (NT * 4); };
    const int first_lt = wp.ns > 0 ? udiv_small(wp.f0, wp.ns) : 0;
    int lt = first_lt, si = wp.ns > 0 ? wp.f0 - first_lt * wp.ns : 0;
    const int f_end = wp.fo + wp.P;  // this CTA's range: [fo, f_end)
    // stream-K boundary parts (flat layers): LL words {float, tag} per lane
    auto remote_slot = [&](int cta) {
        return p.ll + L.fl_off + ((long long)cta * 32 + lane) * (NT * 4);
    };
    // segment by segment: the steps of one row tile inside [f0, f1)
#pragma unroll 1
    for (int f = wp.f0; f < wp.f1;) {
        const int seg = min(wp.ns - si, wp.f1 - f);
        const int tstart = lt * wp.ns, tlast = tstart + wp.ns - 1;
        const int lfirst = max(tstart, wp.fo);  // the tile's first step inside this CTA
        const bool head = f == lfirst;           // this segment holds it
#pragma unroll
        for (int nt = 0; nt < NT; ++nt)
#pragma unroll
            for (int i = 0; i < 4; ++i) tot[nt][i] = 0.0f;
        uint32_t xcol = (uint32_t)(si * kStepCols);  // column of the step inside the staged chunk
#pragma unroll 1
        for (int k = 0; k < seg; ++k) {
            mbar_wait(rc.full0 + 8 * cstage, parity);
            const uint32_t src = rc.ring0 + cstage * stride;
            float sc[4];
            sc[0] = lds32f(src + g * 4);
            sc[1] = lds32f(src + (g + 8) * 4);
            sc[2] = lds32f(src + (16 + g) * 4);
            sc[3] = lds32f(src + (24 + g) * 4);
            uint4 buf[NPL];
#pragma unroll
            for (int jj = 0; jj < NPL; ++jj) buf[jj] = lds128(src + kScaleBytes + jj * kSlab + lane * 16);
            mbar_arrive(rc.empty0 + 8 * cstage);  // the slot is read: the producer may refill it
            if (++cstage == D) {
                cstage = 0;
                parity ^= 1u;
            }
            process(buf, sc, xcol);
            xcol += kStepCols;
        }
        f += seg;
        si += seg;
        if (f == wp.f1) MQ_STS_WMAX(l, 5);  // this warp's last step decoded
        const bool tile_end = si == wp.ns;
        const bool lend = tile_end || f == f_end;  // this segment reaches the tile's last step in this CTA
        const int llast = min(tlast, f_end - 1) - wp.fo;  // CTA-local index of that step
        if (head && lend && tstart >= wp.fo && tlast < f_end) {
            emit(wp.ta + lt, tot);  // the whole tile in this warp
        } else if (!head) {
            float* sp = slot_ptr(warp);
#pragma unroll
            for (int nt = 0; nt < NT; ++nt)
#pragma unroll
                for (int i = 0; i < 4; ++i) sp[nt * 4 + i] = tot[nt][i];
            // hand the part to the tile's head wa (holder of its first step here)
            // through named barrier wa + 1: bar.arrive orders the slot stores and
            // does not wait
            const int wa = last_warp_at(wp, lfirst - wp.fo);
            named_bar_arrive(wa + 1, 32 * (1 + tile_parts(wp, wa, llast)));
        } else {
            // head: own part, the later warps' parts in warp order, then the next
            // CTA's part (a tile running past this CTA's range), in that order.  (Issuing
            // the first poll of that part before the local-parts barrier measured no
            // faster and cost the r = 4 kernel 2% through register allocation.)
            if (!lend) {
                named_bar_sync(warp + 1, 32 * (1 + tile_parts(wp, warp, llast)));
                if (f == wp.f1) MQ_STS_WMAX(l, 3);  // the parts of this warp's last tile arrived
                const int vmax = last_warp_at(wp, llast);
                for (int w2 = warp + 1; w2 <= vmax; ++w2) {
                    if (plan_f0(wp, w2) == plan_f0(wp, w2 + 1)) continue;  // no steps: no part
                    const float* sp = slot_ptr(w2);
#pragma unroll
                    for (int nt = 0; nt < NT; ++nt)
#pragma unroll
                        for (int i = 0; i < 4; ++i) tot[nt][i] += sp[nt * 4 + i];
                }
            }
            if (tlast >= f_end) {  // the next CTA's part of this tile
                const unsigned long long* src = remote_slot(rc.cta);
                unsigned long long v[NT * 4];
                for (;;) {
                    bool ok = true;
#pragma unroll
                    for (int i = 0; i < NT * 4; i += 2) {
                        ld_ll2(src + i, v[i], v[i + 1]);
                        ok = ok && (uint32_t)(v[i] >> 32) == sh.tag && (uint32_t)(v[i + 1] >> 32) == sh.tag;
                    }
                    if (ok) break;
                }
                __syncwarp();
#pragma unroll
                for (int nt = 0; nt < NT; ++nt)
#pragma unroll
                    for (int i = 0; i < 4; ++i) tot[nt][i] += __uint_as_float((uint32_t)v[nt * 4 + i]);
                MQ_STS_WMAX(l, 7);  // the next CTA's part arrived
            }
            if (tstart < wp.fo) {  // the tile started in the previous CTA: ship this part there
                unsigned long long* dst = remote_slot(rc.cta - 1);
#pragma unroll
                for (int nt = 0; nt < NT; ++nt)
#pragma unroll
                    for (int i = 0; i < 4; ++i) st_ll(dst + nt * 4 + i, __float_as_uint(tot[nt][i]), sh.tag);
            } else {
                emit(wp.ta + lt, tot);
            }
        }
        if (tile_end) {
            si = 0;
            ++lt;
        }
    }
    MQ_STS_WMAX(l, 4);  // this warp's tiles emitted (max over warps)

    // ---- end of layer l: the staging area and the partial slots are free again
    consumer_sync();
    MQ_STS(l, 6);
}

// RFIX = the uniform slice width, or 0: per-layer r from the table (parents only)
// XOPS: the layers may carry fused activation prologues (mq_stack_layer.xop); the
// headline stacks run the XOPS = false instantiation, free of their code
template <int NT, int RFIX, bool CHILD, bool XOPS = false>
__global__ void __launch_bounds__(kStackThreads, 1) k_stack(const StackParams p) {
    extern __shared__ __align__(16) uint8_t smem[];
    __shared__ StackShared sh;
    if (p.n_layers == 0) return;  // plan-time launch probe

    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    // warps 0..14 decode + MMA (consumers); warp 15 issues every ring's bulk
    // copies (producer), so no consumer ever has a bulk copy in flight
    const int D = p.stages;
    uint64_t* full = reinterpret_cast<uint64_t*>(smem + p.xs_bytes);   // [15][8]
    uint64_t* empty = full + kStackWarps * 8;                           // [15][8]
    uint8_t* ring = smem + p.xs_bytes + kStackWarps * 8 * 16;
    if (threadIdx.x == kSyncThread) {
        sh.gen = atomicAdd(p.launch_ctr, 1ull) / gridDim.x;
        sh.tag = (uint32_t)(sh.gen % 0xFFFFFFFFull) + 1u;  // never 0 (zeroed buffers); consecutive steps differ
    }
    // the layer table lives in shared memory: a descriptor field re-read from
    // global memory mid-layer (register rematerialisation) waits behind the
    // weight stream for ~1-2 us
    StackLayer* tab = reinterpret_cast<StackLayer*>(smem + p.table_off);
    {
        const int words = p.n_layers * (int)(sizeof(StackLayer) / 4);
        const uint32_t* src = reinterpret_cast<const uint32_t*>(p.layers);
        uint32_t* dst = reinterpret_cast<uint32_t*>(tab);
        for (int i = threadIdx.x; i < words; i += blockDim.x) dst[i] = __ldg(src + i);
    }
    const bool producer = warp == kStackWarps;
    const int ring_of = producer ? (lane < kStackWarps ? lane : 0) : warp;  // the ring this thread serves
    RingCtx rc;
    rc.full0 = smem_addr(full + ring_of * 8);
    rc.empty0 = smem_addr(empty + ring_of * 8);
    rc.ring0 = smem_addr(ring + (size_t)ring_of * D * p.stage_stride);
    rc.stride = (uint32_t)p.stage_stride;
    rc.D = D;
    rc.policy = 0;
    rc.cta = blockIdx.x;
    rc.warp = ring_of;
    rc.n_layers = p.n_layers;
    rc.tab = tab;
    if (producer && lane < kStackWarps) {
        rc.policy = policy_evict_first();
        for (int i = 0; i < D; ++i) {
            mbar_init(rc.full0 + 8 * i, 1);
            mbar_init(rc.empty0 + 8 * i, 32);
        }
        fence_mbar_init();
    }
    if (p.cluster && threadIdx.x == kSyncThread) {
        // [full mbarriers][uses] (chunk 0 side), [free mbarriers][free uses] (chunk 1 side)
        const uint32_t cl = smem_addr(smem + p.cl_off);
        unsigned* uses = reinterpret_cast<unsigned*>(smem + p.cl_off + 8 * p.cl_tiles);
        unsigned* fuses = reinterpret_cast<unsigned*>(smem + p.cl_off + 24 * p.cl_tiles);
        for (int i = 0; i < p.cl_tiles; ++i) {
            mbar_init(cl + 8 * i, 1);
            mbar_init(cl + 16 * p.cl_tiles + 8 * i, 1);
            uses[i] = 0u;
            fuses[i] = 0u;
        }
        fence_mbar_init();
    }
    __syncthreads();
    if (p.cluster) cluster_sync_all();  // the peer's first st.async lands on initialised barriers

    if (producer) {
        // the same slot stride the consumer uses: the stage size in uniform kernels
        constexpr uint32_t kFix = RFIX ? 128u + 512u * PlaneCount<RFIX ? RFIX : 2, CHILD>::value : 0u;
        stack_producer<kFix>(rc);
        if (p.cluster) cluster_sync_all();  // see the end of the consumer path
        return;
    }
    // programmatic dependent launch: the producer warp streams the (static) weights while
    // the previous kernel drains; consumers touch activations / outputs only after it is done
#ifndef MQ_STACK_GDC
#define MQ_STACK_GDC 1
#endif
    if (MQ_STACK_GDC) asm volatile("griddepcontrol.wait;" ::: "memory");
    const unsigned long long target = (sh.gen + 1ull) * gridDim.x;
    int cstage = 0;
    uint32_t parity = 0;
#pragma unroll 1
    for (int l = 0; l < p.n_layers; ++l) {
        if constexpr (RFIX != 0) {
            stack_layer<RFIX, NT, CHILD, true, XOPS>(p, tab, l, rc, cstage, parity, sh, smem, target);
        } else {
            switch (tab[l].r) {
                case 2: stack_layer<2, NT, false, false, XOPS>(p, tab, l, rc, cstage, parity, sh, smem, target); break;
                case 3: stack_layer<3, NT, false, false, XOPS>(p, tab, l, rc, cstage, parity, sh, smem, target); break;
                case 4: stack_layer<4, NT, false, false, XOPS>(p, tab, l, rc, cstage, parity, sh, smem, target); break;
                case 6: stack_layer<6, NT, false, false, XOPS>(p, tab, l, rc, cstage, parity, sh, smem, target); break;
                default: stack_layer<8, NT, false, false, XOPS>(p, tab, l, rc, cstage, parity, sh, smem, target); break;
            }
        }
    }
    // a CTA pair touches each other's shared memory (partials, slot credits) until
    // the last pair layer: neither exits before both are done
    if (p.cluster) cluster_sync_all();
}

template <int R>
cudaError_t launch_stack_r(const StackParams& p, int nt, bool child, int grid, size_t smem,
                           cudaStream_t stream);
cudaError_t launch_stack_mixed(const StackParams& p, int nt, int grid, size_t smem, cudaStream_t stream);
// CTAs of k_stack<nt, r, child> (r = 0: the mixed kernel) that can be co-resident as
// clusters of 2 with `smem` bytes each, or 0 when unknown
int stack_pair_capacity(int nt, int r, bool child, size_t smem, bool xops);
// launch the planned configuration with no layers: does the driver accept it?
cudaError_t stack_probe(int nt, int r, bool child, int grid, size_t smem, bool cluster, bool xops);

}  // namespace mq
