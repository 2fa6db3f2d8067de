// Host emulation of the K1 pack + K3 register decode (test infrastructure).
//
// Compiles the same __host__ __device__ functions the GEMV kernel runs
// (matq_common.cuh) for the CPU and checks, for every r on the ladder and
// both parent (mode P) and child (mode C) planes, that the bf16 A registers
// produced by slice_loaded + decode_word hold exactly s_r(q) - 2^(r-1) for
// the weight the mma.m16n8k16 A-fragment layout assigns to that register
// slot (PTX ISA: a0/a1 row g cols 2t,2t+1; a2/a3 row g+8; a4..a7 cols +8).
// s_r is the reference rounding slice (slicing.py:31-48).
#include <cstdio>
#include <cstdlib>
#include <vector>

#include "../../paper_2602_03537_b200/csrc/matq_common.cuh"

using namespace mq;

static uint32_t rng_state = 12345u;
static uint32_t xrand() {
    rng_state ^= rng_state << 13;
    rng_state ^= rng_state >> 17;
    rng_state ^= rng_state << 5;
    return rng_state;
}

static int slice_ref(int q, int r) {  // slicing.py:31-48 with c = 8
    const int k = 8 - r;
    if (k == 0) return q;
    int v = (q + (1 << (k - 1))) >> k;
    return v > (1 << r) - 1 ? (1 << r) - 1 : v;
}

// host restatement of k_pack_planes (matq_aux.cu), step-interleaved blob
static void pack_planes(const std::vector<uint8_t>& codes, int N, int K, int nbits,
                        std::vector<uint32_t>& blob, Layout& L) {
    L = Layout::make(N, K, 128, nbits);
    blob.assign((size_t)L.total_words(), 0u);
    const long long total = (long long)L.n_rt * L.nsteps * 128;
    for (long long idx = 0; idx < total; ++idx) {
        const int w = (int)(idx & 3), lane = (int)((idx >> 2) & 31);
        const long long blk = idx >> 7;
        const int st = (int)(blk % L.nsteps), rt = (int)(blk / L.nsteps);
        for (int bit = 0; bit < 32; ++bit) {
            int ro, co;
            word_bit_pos(lane, w, bit, ro, co);
            const int row = rt * 16 + ro, col = st * 256 + co;
            const uint32_t q = (row < N && col < K) ? codes[(size_t)row * K + col] : 0u;
            for (int j = 0; j < nbits; ++j)
                blob[(size_t)L.plane_word(rt, st, j, lane, w)] |= ((q >> (nbits - 1 - j)) & 1u) << bit;
        }
    }
}

template <int R, bool CHILD>
static long long check(const std::vector<uint8_t>& parent, int N, int K) {
    constexpr int NPL = PlaneCount<R, CHILD>::value;
    std::vector<uint8_t> src = parent;
    int nbits = 8;
    if (CHILD) {
        for (auto& q : src) q = (uint8_t)slice_ref(q, R);
        nbits = R;
    }
    std::vector<uint32_t> planes;
    Layout L;
    pack_planes(src, N, K, nbits, planes, L);
    const long long total = (long long)L.n_rt * L.nsteps * 128;
    long long bad = 0;
    for (long long idx = 0; idx < total; ++idx) {
        const int w = (int)(idx & 3), lane = (int)((idx >> 2) & 31);
        const long long blk = idx >> 7;
        const int st = (int)(blk % L.nsteps), rt = (int)(blk / L.nsteps);
        uint32_t T[NPL];
        for (int j = 0; j < NPL; ++j) T[j] = planes[(size_t)L.plane_word(rt, st, j, lane, w)];
        uint32_t S[R];
        slice_loaded<R, CHILD>(T, S);
        uint32_t A[16], Araw[16];
        decode_word<R>(S, A);
        decode_word<R, true>(S, Araw);
        const int g = lane >> 2, t = lane & 3;
        for (int s = 0; s < 4; ++s)
            for (int q = 0; q < 4; ++q)
                for (int h = 0; h < 2; ++h) {
                    // mma.m16n8k16 A fragment (row-major), register q of step s
                    const int row = rt * 16 + g + 8 * (q & 1);
                    const int col = st * 256 + 64 * w + 16 * s + 8 * (q >> 1) + 2 * t + h;
                    const float v = host_bf16(A[4 * s + q] >> (16 * h));
                    int want = 0;
                    if (row < N && col < K)
                        want = slice_ref(parent[(size_t)row * K + col], R) - (1 << (R - 1));
                    else
                        want = (CHILD ? 0 : slice_ref(0, R)) - (1 << (R - 1));  // pad code 0
                    if (R != 8) {  // raw (zero-point folded) encoding: 128 + s * 2^o
                        const float raw = host_bf16(Araw[4 * s + q] >> (16 * h));
                        const int o = zp_off<R>(s, q >> 1);
                        const float dec = (raw - 128.0f) / (float)(1 << o) - (float)(1 << (R - 1));
                        if (dec != (float)want) {
                            if (bad < 5) std::printf("RAW R=%d row=%d col=%d got %g want %d\n", R, row, col, dec, want);
                            ++bad;
                        }
                    }
                    if (v != (float)want) {
                        if (bad < 5)
                            std::printf("R=%d child=%d row=%d col=%d got %g want %d\n", R, (int)CHILD,
                                        row, col, v, want);
                        ++bad;
                    }
                }
    }
    return bad;
}

int main(int argc, char** argv) {
    const int N = argc > 1 ? std::atoi(argv[1]) : 40;
    const int K = argc > 2 ? std::atoi(argv[2]) : 600;
    std::vector<uint8_t> parent((size_t)N * K);
    for (auto& q : parent) q = (uint8_t)(xrand() & 255u);
    for (int c = 0; c < K && c < 256 * 4; ++c) parent[c] = (uint8_t)(c & 255);  // every code
    long long bad = 0;
    bad += check<2, false>(parent, N, K);
    bad += check<3, false>(parent, N, K);
    bad += check<4, false>(parent, N, K);
    bad += check<6, false>(parent, N, K);
    bad += check<8, false>(parent, N, K);
    bad += check<2, true>(parent, N, K);
    bad += check<3, true>(parent, N, K);
    bad += check<4, true>(parent, N, K);
    bad += check<6, true>(parent, N, K);
    std::printf("%s mismatches=%lld N=%d K=%d\n", bad ? "FAIL" : "OK", bad, N, K);
    return bad ? 1 : 0;
}
