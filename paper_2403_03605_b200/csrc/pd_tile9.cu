// One-shot fused 2D fine step with TMA staging (tile v9), 28-offset stencil,
// fast mode: 31 x 31 owned elements, 32 x 32 force region (own + one recomputed
// ring), bond state at the lower end, integer candidate compare.  Inputs:
//
//   * one thread issues three cp.async.bulk.tensor loads completing on two
//     mbarriers -- at launch the node apron of the predictor displacement (needed
//     first, alone in the TMA unit), and after the ubar pass the owned nodes' rv
//     and {1/M, flags} (needed last: their latency hides behind the force pass).  Out-of-domain parts of
//     a box are zero-filled by the TMA unit, exactly the zeros the tile kernel
//     writes with bounds-checked loads (the tile kernel's ncu source page put
//     ~25 % of the stall samples on its staging phase and ~27 % on the
//     node-update loads).  The bond-state apron goes through 4-byte cp.async
//     with zero fill: a TMA box row must start 16-byte aligned in global
//     memory, which the mask apron (start column i0 - 4) is not, and the
//     aligned superset box would not leave room for three CTAs per SM;
//   * G aliases the ubar apron after the force pass, and the node flags ride
//     in the three low mantissa bits of 1/M (pmts_pd.cu encodes them for every
//     2D lattice kernel), so the CTA fits in 76.3 KB and three CTAs (24 warps)
//     stay resident per SM.
//
// TMA rules this layout honours (measured: violations fault with "illegal
// instruction" / "misaligned address"): 128-byte aligned shared destinations,
// 16-byte aligned global row starts (so the {1/M, flags} box starts at the
// even column i0 & ~1 of rows padded to an even length).  Reference semantics
// as in pd_stencil.cu.
#include <cstdlib>
#include <cstring>
#include <initializer_list>
#include <stdexcept>
#include <string>
#include <type_traits>

#include "pd_stencil.cuh"

namespace pmts {

namespace {

constexpr int TX = 31, TY = 31, R = kFusedR;
constexpr int GX = TX + 1, GY = TY + 1;          // force region (elements), 32 x 32
constexpr int AX = GX + 2 * R, AY = GY + 2 * R;  // ubar apron (elements), 38 x 38
constexpr int BX = AX + 1, BY = AY + 1;          // node apron, 39 x 39
constexpr int MY = GY + R;                       // bond-state apron rows the force pass reads
constexpr int IX = 32;                           // {1/M, flags} box row (from an even column)
#ifndef PMTS_T9_NW
#define PMTS_T9_NW 8
#endif
constexpr int NW = PMTS_T9_NW, NT = 32 * NW;  // 8 warps x 4 rows (3 CTAs/SM) or 16 x 2 (2 CTAs/SM)
constexpr int kMinBlocks = NW <= 8 ? 3 : 2;
constexpr int EPT = GY / NW;
constexpr int SHALF = kFusedS / 2;
static_assert(GX == 32 && EPT * NW == GY && EPT % 4 == 0, "lane = column, warp = EPT rows in blocks of 4");
static_assert(AX == kFusedAX, "Stencil2D apron offsets assume this width");

constexpr int rup(int x, int a) { return (x + a - 1) / a * a; }
constexpr int kNtBytes = BX * BY * 16;
constexpr int kRvBytes = TX * TY * 16;
constexpr int kImBytes = IX * TY * 8;
// TMA destinations (128-byte aligned) first, ordered to minimise padding
constexpr int kOffIm = 0;
constexpr int kOffNt = rup(kOffIm + kImBytes, 128);
constexpr int kOffRv = rup(kOffNt + kNtBytes, 128);
constexpr int kOffMa = rup(kOffRv + kRvBytes, 16);  // AX x MY bond-state words
constexpr int kOffUb = rup(kOffMa + AX * MY * 4, 16);
constexpr int kOffBar = rup(kOffUb + AX * AY * 16, 8);
constexpr int kOffPart = kOffUb + GX * GY * 16;  // in the ubar apron's tail, after G
constexpr int kOffRed = kOffBar + 16;            // screen: per-warp node-step maxima
constexpr int kSmem = kOffRed + 4 * NW * 4 + 8 + 128;  // + realignment slack of the dynamic base
static_assert(GX * GY * 16 + 8 * NW <= AX * AY * 16, "G and the partial counts fit in ub");
static_assert(TY < GY, "a band's last force row is never an owned node row");
static_assert(kSmem + 1024 <= 233472 / 3, "three CTAs per SM");

__device__ __forceinline__ long long dbits(double x) { return __double_as_longlong(x); }
__device__ __forceinline__ unsigned smem_u32(const void* p) {
    return (unsigned)__cvta_generic_to_shared(p);
}
__device__ __forceinline__ void mbar_init(uint64_t* b, unsigned count) {
    asm volatile("mbarrier.init.shared.b64 [%0], %1;\n" ::"r"(smem_u32(b)), "r"(count));
}
__device__ __forceinline__ void mbar_expect_tx(uint64_t* b, unsigned bytes) {
    asm volatile("mbarrier.arrive.expect_tx.shared.b64 _, [%0], %1;\n" ::"r"(smem_u32(b)),
                 "r"(bytes));
}
__device__ __forceinline__ void mbar_wait(uint64_t* b, unsigned phase) {
    asm volatile(
        "{\n"
        ".reg .pred P1;\n"
        "WAIT_%=:\n"
        "mbarrier.try_wait.parity.shared.b64 P1, [%0], %1;\n"
        "@!P1 bra WAIT_%=;\n"
        "}\n" ::"r"(smem_u32(b)),
        "r"(phase));
}
__device__ __forceinline__ void tma_load_2d(void* dst, const CUtensorMap* map, int x, int y,
                                            uint64_t* b) {
    asm volatile(
        "cp.async.bulk.tensor.2d.shared::cluster.global.mbarrier::complete_tx::bytes"
        " [%0], [%1, {%2, %3}], [%4];\n" ::"r"(smem_u32(dst)),
        "l"(map), "r"(x), "r"(y), "r"(smem_u32(b))
        : "memory");
}
__device__ __forceinline__ void tma_prefetch_2d(const CUtensorMap* map, int x, int y) {
    asm volatile("cp.async.bulk.prefetch.tensor.2d.L2.global.tile [%0, {%1, %2}];\n" ::"l"(map),
                 "r"(x), "r"(y)
                 : "memory");
}
__device__ __forceinline__ void cp_async4(void* dst, const void* src, bool valid) {
    asm volatile("cp.async.ca.shared.global [%0], [%1], 4, %2;\n" ::"r"(smem_u32(dst)), "l"(src),
                 "r"(valid ? 4 : 0)
                 : "memory");
}

// pair order = the column groups of the register-blocked full-tile path
// (|A| = 0, 1, 2, 3); the masked path accumulates in the same order
constexpr int kPairA[14] = {0, 0, 0, 1, 1, -1, 1, -1, 2, 2, -2, 2, -2, 3};
constexpr int kPairB[14] = {1, 2, 3, 0, 1, 1, 2, 2, 0, 1, 1, 2, 2, 0};

// One opposite-offset pair (o, -o) of every element of the thread: the two
// directed entries share xi xi^T, so their forces combine into one term of
// s = eta_o + eta_-o (G_e = -w c h^2 sum (o.s) o); the bond to e + o (state kept
// here, at its lower end) also gets the candidate break test.  Tiles with a
// broken or absent bond in reach take the MASKED instance, which is bitwise the
// same arithmetic for intact pairs -- so results do not depend on how the
// domain is cut into tiles or slabs.  The products
// with the integer offset components are compile-time (adds / small-constant
// multiplies); the apron offset itself comes from the parameter block, which
// keeps ptxas from hoisting all 112 loads of a thread to the top (immediate
// offsets did, and spilled).
// the arithmetic of one pair of one element (shared by every path, so they
// round identically)
template <bool DO_BREAK, bool MASKED, int K>
__device__ __forceinline__ void pair_math(double2 up, double2 um, double2 ue, bool actp, bool actm,
                                          double& G0, double& G1, bool& anyc,
                                          const PairStencil2D& ps) {
    static_assert(!DO_BREAK, "break tests run in cand_terms");
    constexpr int A = kPairA[K], B = kPairB[K];
    // s = eta_o + eta_-o with a broken bond's eta an exact zero.  (Measured: forming s as
    // (u_o + u_-o) - 2 u_e -- 4 instead of 6 fp64 operations per pair -- is not faster
    // here, 37.8 vs 37.3 us per cfg3 step; the fp32 variant below does use it.)
    const double ep0 = up.x - ue.x, ep1 = up.y - ue.y;
    double em0 = um.x - ue.x, em1 = um.y - ue.y;
    if (MASKED) {
        em0 = actm ? em0 : 0.0;
        em1 = actm ? em1 : 0.0;
    }
    const double fp0 = MASKED && !actp ? 0.0 : ep0, fp1 = MASKED && !actp ? 0.0 : ep1;
    if (B == 0) {
        G0 = fma(ps.fa[K], fp0 + em0, G0);
    } else if (A == 0) {
        G1 = fma(ps.fb[K], fp1 + em1, G1);
    } else {
        const double s0 = fp0 + em0, s1 = fp1 + em1;
        const double t = fma((double)A, s0, B * s1);
        G0 = fma(ps.fa[K], t, G0);
        G1 = fma(ps.fb[K], t, G1);
    }
}

// fp32-position variant (PMTS_FAST_F32POS): the ubar apron holds tile-relative
// fp32 displacements (ubar - ubar_ref, rounded once); the pair sum s = (u_o + u_-o) -
// 2 u_e (the masked form drops a broken bond's u and lowers the factor: -1 gives the
// single eta rounded once, 0 an exact zero) and t = o . s are fp32, each pair's t is
// widened to fp64 and accumulated into G in fp64 (the break tests run in cand_terms)
template <bool DO_BREAK, bool MASKED, int K>
__device__ __forceinline__ void pair_math(float2 up, float2 um, float2 ue, bool actp, bool actm,
                                          double& G0, double& G1, bool& anyc,
                                          const PairStencil2D& ps) {
    static_assert(!DO_BREAK, "break tests run in cand_terms");
    constexpr int A = kPairA[K], B = kPairB[K];
    float c = -2.0f;
    if (MASKED) {
        up.x = actp ? up.x : 0.0f;
        up.y = actp ? up.y : 0.0f;
        um.x = actm ? um.x : 0.0f;
        um.y = actm ? um.y : 0.0f;
        c = actp ? (actm ? -2.0f : -1.0f) : (actm ? -1.0f : 0.0f);
    }
    if (B == 0) {
        G0 = fma(ps.fa[K], (double)fmaf(c, ue.x, up.x + um.x), G0);
    } else if (A == 0) {
        G1 = fma(ps.fb[K], (double)fmaf(c, ue.y, up.y + um.y), G1);
    } else {
        const float s0 = fmaf(c, ue.x, up.x + um.x), s1 = fmaf(c, ue.y, up.y + um.y);
        const double t = fmaf((float)A, s0, (float)B * s1);
        G0 = fma(ps.fa[K], t, G0);
        G1 = fma(ps.fb[K], t, G1);
    }
}

template <bool DO_BREAK, bool MASKED, int K, typename V>
__device__ __forceinline__ void pair_term(const V* ubq, const uint32_t* maq,
                                          const V (&ue)[EPT], const uint32_t (&m0)[EPT],
                                          double (&G0)[EPT], double (&G1)[EPT],
                                          bool (&anyc)[EPT], const PairStencil2D& ps) {
    const int off = ps.off[K];
    const V* pp = ubq + off;
    const V* pm = ubq - off;
#pragma unroll
    for (int r = 0; r < EPT; ++r) {
        bool actp = true, actm = true;
        if (MASKED) {
            // bond e -> e+o lives at e, bond e-o -> e at e-o, both under the bit of +o;
            // a broken (or absent) bond contributes an exact zero, so a pair with both
            // bonds intact rounds exactly as on the unmasked path
            const int bit = ps.pbit[K];
            actp = (m0[r] >> bit) & 1u;
            actm = (maq[r * AX - off] >> bit) & 1u;
        }
        pair_math<DO_BREAK, MASKED, K>(pp[r * AX], pm[r * AX], ue[r], actp, actm, G0[r], G1[r],
                                       anyc[r], ps);
    }
}

// full tiles, register-blocked by column group: the 4 rows of column x need,
// for the pairs of one |A| group, the cells of columns x +- A at rows -3..6
// (A = 0), -2..5 (|A| = 1, 2, loaded per half of the rows to stay within 80
// registers) or 0..3 (|A| = 3): 62 shared loads per thread instead of 112 --
// the shared-memory pipe was the limiter (ncu: 67 % of peak)
// MASKED: the same cell loads with the bond states applied per pair (the bond e -> e + o
// under e's own word m0, the bond e - o -> e under the word of e - o, read from maq) --
// the pairs of an element accumulate in the same order as in pair_terms, so this is
// bitwise that instance at less than half its shared-memory traffic
template <bool DO_BREAK, bool MASKED, typename V>
__device__ __forceinline__ void pairs_blocked(const V* ubq, const V* ue, double* G0, double* G1,
                                              bool* anyc, const PairStencil2D& ps,
                                              const uint32_t* maq = nullptr,
                                              const uint32_t* m0 = nullptr) {
    // one block of 4 consecutive rows of the thread (ubq, ue, G, anyc, maq, m0 at its first row)
    constexpr int EPT = 4;
#define PMTS_PM(K, UP, UM, ROW)                                                              \
    {                                                                                        \
        bool ap_ = true, am_ = true;                                                         \
        if (MASKED) {                                                                        \
            const int bit_ = ps.pbit[K];                                                     \
            ap_ = (m0[ROW] >> bit_) & 1u;                                                    \
            am_ = (maq[(ROW)*AX - ps.off[K]] >> bit_) & 1u;                                  \
        }                                                                                    \
        pair_math<DO_BREAK, MASKED, K>(UP, UM, ue[ROW], ap_, am_, G0[ROW], G1[ROW], anyc[ROW], ps); \
    }
    {  // A = 0: (0,1) (0,2) (0,3)
        V c[10];
#pragma unroll
        for (int i = 0; i < 10; ++i) c[i] = (i >= 3 && i < 7) ? ue[i - 3] : ubq[(i - 3) * AX];
#pragma unroll
        for (int r = 0; r < EPT; ++r) {
            PMTS_PM(0, c[r + 4], c[r + 2], r)
            PMTS_PM(1, c[r + 5], c[r + 1], r)
            PMTS_PM(2, c[r + 6], c[r], r)
        }
    }
#pragma unroll
    for (int g = 1; g <= 2; ++g) {    // |A| = 1: pairs 3..7, |A| = 2: pairs 8..12
#pragma unroll
        for (int half = 0; half < 2; ++half) {  // rows 2 half .. 2 half + 1: cells rows -2..3 (+2 half)
            V p[6], m[6];
#pragma unroll
            for (int i = 0; i < 6; ++i) {
                p[i] = ubq[(i - 2 + 2 * half) * AX + g];
                m[i] = ubq[(i - 2 + 2 * half) * AX - g];
            }
#pragma unroll
            for (int rr = 0; rr < 2; ++rr) {
                const int r = 2 * half + rr, q = rr + 2;
                if (g == 1) {
                    PMTS_PM(3, p[q], m[q], r)
                    PMTS_PM(4, p[q + 1], m[q - 1], r)
                    PMTS_PM(5, m[q + 1], p[q - 1], r)
                    PMTS_PM(6, p[q + 2], m[q - 2], r)
                    PMTS_PM(7, m[q + 2], p[q - 2], r)
                } else {
                    PMTS_PM(8, p[q], m[q], r)
                    PMTS_PM(9, p[q + 1], m[q - 1], r)
                    PMTS_PM(10, m[q + 1], p[q - 1], r)
                    PMTS_PM(11, p[q + 2], m[q - 2], r)
                    PMTS_PM(12, m[q + 2], p[q - 2], r)
                }
            }
        }
    }
#pragma unroll
    for (int r = 0; r < EPT; ++r)  // |A| = 3: (3,0)
        PMTS_PM(13, ubq[r * AX + 3], ubq[r * AX - 3], r)
}
#undef PMTS_PM

template <bool DO_BREAK, bool MASKED, int K, typename V>
__device__ __forceinline__ void pair_terms(const V* ubq, const uint32_t* maq,
                                           const V (&ue)[EPT], const uint32_t (&m0)[EPT],
                                           double (&G0)[EPT], double (&G1)[EPT],
                                           bool (&anyc)[EPT], const PairStencil2D& ps) {
    if constexpr (K < 14) {
        pair_term<DO_BREAK, MASKED, K>(ubq, maq, ue, m0, G0, G1, anyc, ps);
        pair_terms<DO_BREAK, MASKED, K + 1>(ubq, maq, ue, m0, G0, G1, anyc, ps);
    }
}

// candidate break test of the bond e -> e + o (state kept at e) for the pairs of
// one element; only run on tiles the screen could not prove cold
template <bool MASKED, int K>
__device__ __forceinline__ void cand_terms(const double2* uq, double2 ue, uint32_t m0, bool& anyc,
                                           const PairStencil2D& ps) {
    if constexpr (K < 14) {
        constexpr int A = kPairA[K], B = kPairB[K];
        const double2 up = uq[ps.off[K]];
        const double ep0 = up.x - ue.x, ep1 = up.y - ue.y;
        double tp;
        if (B == 0) tp = A * ep0;
        else if (A == 0) tp = B * ep1;
        else tp = fma((double)A, ep0, B * ep1);
        const bool act = !MASKED || ((m0 >> ps.pbit[K]) & 1u);
        anyc |= act && dbits(fma(ps.h2, tp, fma(ep0, ep0, ep1 * ep1))) >= ps.cl[K];
        cand_terms<MASKED, K + 1>(uq, ue, m0, anyc, ps);
    }
}
// fp32 candidate test against thresholds lowered by 1e-4 (clf): a superset of
// the bonds whose fp64 test on the same fp32 ubar values can fire
template <bool MASKED, int K>
__device__ __forceinline__ void cand_terms(const float2* uq, float2 ue, uint32_t m0, bool& anyc,
                                           const PairStencil2D& ps) {
    if constexpr (K < 14) {
        constexpr int A = kPairA[K], B = kPairB[K];
        const float2 up = uq[ps.off[K]];
        const float ep0 = up.x - ue.x, ep1 = up.y - ue.y;
        float tp;
        if (B == 0) tp = A * ep0;
        else if (A == 0) tp = B * ep1;
        else tp = fmaf((float)A, ep0, B * ep1);
        const bool act = !MASKED || ((m0 >> ps.pbit[K]) & 1u);
        anyc |= act && fmaf(ps.h2f, tp, fmaf(ep0, ep0, ep1 * ep1)) >= ps.clf[K];
        cand_terms<MASKED, K + 1>(uq, ue, m0, anyc, ps);
    }
}

__device__ __forceinline__ double2 to_d2(double2 v) { return v; }
__device__ __forceinline__ double2 to_d2(float2 v) { return make_double2(v.x, v.y); }

template <bool F32> struct UbarT { using V = double2; };
template <> struct UbarT<true> { using V = float2; };

__device__ __forceinline__ int ps_a(int k) {
    return k == 13 ? 3 : (k >= 8 ? 2 : (k >= 3 ? 1 : 0));  // |A| of pair k
}
__device__ __forceinline__ int ps_b(int k) {
    constexpr unsigned kB = 0u | (1u << 0) | (2u << 2) | (3u << 4) | (0u << 6) | (1u << 8) |
                            (1u << 10) | (2u << 12) | (2u << 14) | (0u << 16) | (1u << 18) |
                            (1u << 20) | (2u << 22) | (2u << 24) | (0u << 26);
    return (kB >> (2 * k)) & 3u;  // |B| of pair k
}

// |d| <= hi_bound(max of hi_abs(d)): the high word of |d| orders like |d|
__device__ __forceinline__ unsigned hi_abs(double d) {
    return (unsigned)__double2hiint(d) & 0x7fffffffu;
}
__device__ __forceinline__ double hi_bound(unsigned m) {
    return __hiloint2double((int)m, (int)0xffffffffu);
}

}  // namespace

int tile9_pair_offset(int k, int* a, int* b) {
    static const int A[14] = {0, 0, 0, 1, 1, -1, 1, -1, 2, 2, -2, 2, -2, 3};
    static const int B[14] = {1, 2, 3, 0, 1, 1, 2, 2, 0, 1, 1, 2, 2, 0};
    *a = A[k];
    *b = B[k];
    return 14;
}

// PAIRS: the pair-symmetric force with the cold-tile break screen; otherwise
// per-offset sums with representative per-bond constants (lattice_h = 0)
template <bool DO_BREAK, bool PAIRS, bool REPORT, bool F32>
__global__ void __launch_bounds__(NT, kMinBlocks)
k_tile9(DevPD d, LatticeDev L, const __grid_constant__ Stencil2D st,
        const __grid_constant__ PairStencil2D ps,
        const __grid_constant__ Tile9Maps maps, FusedBufs bf, int step, double scale,
        int write_state) {
    constexpr bool SCREEN = PAIRS && DO_BREAK;
    static_assert(PAIRS || !F32, "the fp32-position variant runs the pair-symmetric force");
    using V = typename UbarT<F32>::V;
    extern __shared__ __align__(16) unsigned char smraw[];
    // the dynamic base is only guaranteed 16-byte aligned: realign for TMA
    unsigned char* sm = smraw + ((128u - (smem_u32(smraw) & 127u)) & 127u);
    const double2* nt = reinterpret_cast<const double2*>(sm + kOffNt);
    uint32_t* ma = reinterpret_cast<uint32_t*>(sm + kOffMa);
    const double2* rvs = reinterpret_cast<const double2*>(sm + kOffRv);
    const double* ims = reinterpret_cast<const double*>(sm + kOffIm);
    V* ub = reinterpret_cast<V*>(sm + kOffUb);
    double2* gt = reinterpret_cast<double2*>(sm + kOffUb);  // G aliases the ubar apron after the force pass
    uint64_t* bar = reinterpret_cast<uint64_t*>(sm + kOffBar);
    unsigned* red = reinterpret_cast<unsigned*>(sm + kOffRed);
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    const int nx = L.nx, ny = L.ny, NX = nx + 1, NY = ny + 1;
    // a launch may cover a range of tile rows (halo-overlap split, pmts_pd.cu)
    const int by = maps.row_base + blockIdx.y;
    const int i0 = blockIdx.x * TX, j0 = by * TY;
    const int ax0 = i0 - 1 - R, ay0 = j0 - 1 - R;
    const int ie = i0 & ~1;  // {1/M, flags} box start: 16-byte aligned global row start

    // (1) staging: TMA for the node apron and the node-update inputs; 4-byte
    //     cp.async (zero-filled outside the domain) for the bond-state apron (a
    //     TMA box must start 16-byte aligned, so the mask box would be 3 columns
    //     wider than the CTA's shared memory has room for; measured: no faster)
    // programmatic dependent launch: the next step's grid may launch now (its CTAs
    // take SM slots as this grid's last wave drains); everything this step reads was
    // written by the previous step, so wait for it before the first global access
    asm volatile("griddepcontrol.launch_dependents;\n" ::);
    if (threadIdx.x == 0) {
        mbar_init(&bar[0], 1);
        mbar_init(&bar[1], 1);
        asm volatile("fence.mbarrier_init.release.cluster;\n" ::);
    }
    asm volatile("griddepcontrol.wait;\n" ::: "memory");
    if (threadIdx.x == 0) {
        mbar_expect_tx(&bar[0], kNtBytes);
        tma_load_2d(sm + kOffNt, &maps.rd, 2 * ax0, ay0, &bar[0]);
    }
    if constexpr (REPORT) {
        // pmts_pd_step_tracked: the step's u is the predictor it consumes (beta = 0);
        // block (0, 0) copies the tracked dofs of it into mapped pinned host memory
        if ((blockIdx.x | by) == 0)
            for (int j = threadIdx.x; j < bf.n_trk; j += NT) bf.trk_host[j] = bf.rd_in[bf.trk_dofs[j]];
    }
    // clean tiles: the apron lies in the domain and the six tiles it overlaps (this one,
    // left, right and the three below: a bond's state lives at its lower element) have
    // every positive-stencil bit set in both bond-state buffers -- nothing to stage, test
    // or write back.  A flag read while its tile clears it in this same step is harmless:
    // the step's input words are still the full ones, and the full and the masked force
    // round identically for intact bonds.
    const bool interior = ax0 >= 0 && ay0 >= 0 && ax0 + AX <= nx && ay0 + MY <= ny;
    bool skip = false;
    if (bf.tclean && interior) {
        const uint32_t* tf = bf.tclean + (size_t)by * gridDim.x + blockIdx.x;
        const uint32_t* tb = tf - gridDim.x;
        skip = (tf[-1] & tf[0] & tf[1] & tb[-1] & tb[0] & tb[1]) != 0u;
    }
    // (re-read from shared memory after the force pass: no register held across it)
    if (threadIdx.x == 0) red[4 * NW] = skip ? 1u : 0u;
    if (skip) {
    } else if (interior) {
        // interior tile (most of them): no per-word bounds checks
        const uint32_t* src = bf.mask_in + (size_t)ay0 * nx + ax0;
        for (int y = warp; y < MY; y += NW) {
            cp_async4(ma + y * AX + lane, src + (size_t)y * nx + lane, true);
            if (lane < AX - 32) cp_async4(ma + y * AX + 32 + lane, src + (size_t)y * nx + 32 + lane, true);
        }
    } else {
        for (int y = warp; y < MY; y += NW) {
            const int gj = ay0 + y;
#pragma unroll
            for (int h = 0; h < 2; ++h) {
                const int x = lane + 32 * h, gi = ax0 + x;
                if (x < AX) {
                    const bool in = gi >= 0 && gj >= 0 && gi < nx && gj < ny;
                    cp_async4(ma + y * AX + x, bf.mask_in + (in ? (size_t)gj * nx + gi : 0), in);
                }
            }
        }
    }
    asm volatile("cp.async.commit_group;\n" ::);
    asm volatile("cp.async.wait_group 0;\n" ::: "memory");
    __syncthreads();
    mbar_wait(&bar[0], 0);
    // fp32 variant: the apron stores ubar - uref, uref = a node of the tile (in the
    // domain), so the fp32 rounding is relative to the tile's local variation
    double2 uref = make_double2(0.0, 0.0);
    if constexpr (F32) uref = nt[(min(j0 + TY / 2, ny) - ay0) * BX + min(i0 + TX / 2, nx) - ax0];

    // (2) ubar of the apron (column walk with carried node-pair sums); the
    //     positive-stencil completeness of every mask the force pass reads.
    //     Work item = (column x, block of UR ub rows): 228 items, one per thread.
    constexpr uint32_t kPos = ((1u << kFusedS) - 1u) & ~((1u << SHALF) - 1u);
    constexpr int UR = NW >= 8 ? 7 : 13, NYB = (AY + UR - 1) / UR;
    static_assert(AX * NYB <= NT, "one ubar work item per thread");
    bool tile_full = true;
    // screen: maxima of |node step| over the in-domain nodes of the apron, per
    // component and direction (x-step of u_x, y-step of u_x, x-step of u_y,
    // y-step of u_y), as high words (out-of-domain nodes are TMA zero fill)
    unsigned mxx = 0, mxy = 0, myx = 0, myy = 0;
    // (ALLIN: every node of the apron lies in the domain -- no per-node bounds tests)
    auto ubar_pass = [&](auto allin) {
        constexpr bool ALLIN = decltype(allin)::value;
        const int x = threadIdx.x % AX, y0 = (threadIdx.x / AX) * UR;
        const bool ca = ALLIN || (unsigned)(ax0 + x) <= (unsigned)nx;      // node column x in the domain
        const bool cb = ALLIN || (unsigned)(ax0 + x + 1) <= (unsigned)nx;  // node column x + 1
        double2 hs[UR + 1];
        double2 ap = make_double2(0.0, 0.0);
        bool rp = false;
#pragma unroll
        for (int i = 0; i <= UR; ++i) {
            const int y = min(y0 + i, BY - 1);
            const double2 a = nt[y * BX + x], b = nt[y * BX + x + 1];
            hs[i] = make_double2(a.x + b.x, a.y + b.y);
            if (SCREEN) {
                const bool rw = ALLIN || (unsigned)(ay0 + y) <= (unsigned)ny;
                if (rw && ca && cb) {
                    mxx = max(mxx, hi_abs(b.x - a.x));
                    myx = max(myx, hi_abs(b.y - a.y));
                }
                if (i > 0 && rw && (ALLIN || rp)) {
                    if (ca) {
                        mxy = max(mxy, hi_abs(a.x - ap.x));
                        myy = max(myy, hi_abs(a.y - ap.y));
                    }
                }
                ap = a;
                rp = rw;
            }
        }
#pragma unroll
        for (int i = 0; i < UR; ++i) {
            const int y = y0 + i;
            if (y < AY) {
                if constexpr (F32)
                    ub[y * AX + x] = make_float2((float)(d.Nsh * (hs[i].x + hs[i + 1].x) - uref.x),
                                                 (float)(d.Nsh * (hs[i].y + hs[i + 1].y) - uref.y));
                else
                    ub[y * AX + x] = make_double2(d.Nsh * (hs[i].x + hs[i + 1].x),
                                                  d.Nsh * (hs[i].y + hs[i + 1].y));
            }
        }
        // (staging tiles only; a uniform branch instead of a predicate per row)
        if (!skip) {
#pragma unroll
            for (int i = 0; i < UR; ++i) {
                const int y = y0 + i;
                if (y < MY) tile_full = tile_full && (ma[y * AX + x] & kPos) == kPos;
            }
        }
    };
    // the y-steps of the apron's last node column (b of x = AX - 1) are taken by the threads
    // the ubar pass leaves idle: inside the pass they were a divergent branch every warp paid
    auto last_column = [&](auto allin) {
        constexpr bool ALLIN = decltype(allin)::value;
        constexpr int NI = NT - AX * NYB;
        static_assert(NI >= 1, "idle threads for the last node column");
        const bool cb = ALLIN || (unsigned)(ax0 + BX - 1) <= (unsigned)nx;
        for (int p = threadIdx.x - AX * NYB; p < BY - 1; p += NI) {
            const bool rw = ALLIN || ((unsigned)(ay0 + p) <= (unsigned)ny &&
                                      (unsigned)(ay0 + p + 1) <= (unsigned)ny);
            if (cb && rw) {
                const double2 b0 = nt[p * BX + BX - 1], b1 = nt[(p + 1) * BX + BX - 1];
                mxy = max(mxy, hi_abs(b1.x - b0.x));
                myy = max(myy, hi_abs(b1.y - b0.y));
            }
        }
    };
    const bool allin = SCREEN && ax0 >= 0 && ay0 >= 0 && ax0 + BX - 1 <= nx && ay0 + BY - 1 <= ny;
    if (threadIdx.x < AX * NYB) {
        if (allin) ubar_pass(std::true_type{});
        else ubar_pass(std::false_type{});
    } else if (SCREEN) {
        if (allin) last_column(std::true_type{});
        else last_column(std::false_type{});
    }
    if (SCREEN) {
        mxx = __reduce_max_sync(0xffffffffu, mxx);
        mxy = __reduce_max_sync(0xffffffffu, mxy);
        myx = __reduce_max_sync(0xffffffffu, myx);
        myy = __reduce_max_sync(0xffffffffu, myy);
        if (lane == 0) {
            red[4 * warp + 0] = mxx;
            red[4 * warp + 1] = mxy;
            red[4 * warp + 2] = myx;
            red[4 * warp + 3] = myy;
        }
    }
    tile_full = __syncthreads_and(tile_full);
    // the node-update inputs are needed last: their loads are issued only now, so the node
    // apron above has the TMA unit to itself (35.16 -> 35.00 us per cfg3 step)
    if (threadIdx.x == 0) {
        mbar_expect_tx(&bar[1], kRvBytes + kImBytes);
        tma_load_2d(sm + kOffRv, &maps.rv, 2 * i0, j0, &bar[1]);
        tma_load_2d(sm + kOffIm, &maps.im, ie, j0, &bar[1]);
        // ... and the L2 prefetch for the tile that takes this CTA's slot a wave later
        // (35.05 -> 34.83 us)
        const int ahead = maps.prefetch_ahead;
        if (ahead > 0) {
            const int t = by * gridDim.x + blockIdx.x + ahead;
            if (t < gridDim.x * maps.grid_rows) {
                const int pi0 = (t % gridDim.x) * TX, pj0 = (t / gridDim.x) * TY;
                const int pax0 = pi0 - 1 - R, pay0 = pj0 - 1 - R;
                tma_prefetch_2d(&maps.rd, 2 * pax0, pay0);
                tma_prefetch_2d(&maps.rv, 2 * pi0, pj0);
                tma_prefetch_2d(&maps.im, pi0 & ~1, pj0);
            }
        }
    }
    // hot: some bond of the tile could reach its candidate threshold.  With the
    // node-step maxima D, |eta_x| <= E0 = |A| Dxx + |B| Dxy, |eta_y| <= E1 =
    // |A| Dyx + |B| Dyy, so 2 xi.eta + |eta|^2 <= 2h (|A| E0 + |B| E1) + E0^2 + E1^2.
    bool hot = DO_BREAK;
    if (SCREEN && ps.screen) {
        unsigned v = red[lane & (4 * NW - 1)];
#pragma unroll
        for (int o = 4; o < 4 * NW; o <<= 1) v = max(v, __shfl_xor_sync(0xffffffffu, v, o));
        const double Dxx = hi_bound(__shfl_sync(0xffffffffu, v, 0));
        const double Dxy = hi_bound(__shfl_sync(0xffffffffu, v, 1));
        const double Dyx = hi_bound(__shfl_sync(0xffffffffu, v, 2));
        const double Dyy = hi_bound(__shfl_sync(0xffffffffu, v, 3));
        const int k = lane < 14 ? lane : 0;
        const double A = fabs((double)ps_a(k)), B = fabs((double)ps_b(k));
        const double E0 = A * Dxx + B * Dxy, E1 = A * Dyx + B * Dyy;
        // (fp32 variant: against the lowered fp32 candidate thresholds, with room
        // for the fp32 rounding of the candidate's own lhs)
        const double bound =
            fma(ps.h2, A * E0 + B * E1, E0 * E0 + E1 * E1) * (F32 ? 1.0 + 1e-5 : 1.0 + 1e-6);
        const double cthr = F32 ? (double)ps.clf[k] : __longlong_as_double(ps.cl[k]);
        hot = __any_sync(0xffffffffu, lane < 14 && !(bound < cthr));
        if (ps.hot_count && threadIdx.x == 0) {
            atomicAdd(ps.hot_count, hot ? 1ull : 0ull);
            atomicAdd(ps.hot_count + 1, 1ull);
        }
    }

    // (3) forces of the 32 x 32 region: column = lane, rows EPT*warp + r
    const int gx = lane, gy0 = warp * EPT;
    const int ei = i0 - 1 + gx;
    const int q0 = (gy0 + R) * AX + gx + R;
    // only ue, G and the candidate flags stay live through the force pass (the
    // element ids and bond-state words are re-derived afterwards: registers)
    V ue[EPT];
    double G0[EPT], G1[EPT];
#pragma unroll
    for (int r = 0; r < EPT; ++r) {
        ue[r] = ub[q0 + r * AX];
        G0[r] = 0.0;
        G1[r] = 0.0;
    }
    bool anyc[EPT];
#pragma unroll
    for (int r = 0; r < EPT; ++r) anyc[r] = false;
    uint32_t cand = 0;  // bit r: row r has a break candidate
    if constexpr (PAIRS) {
        // candidate break tests first, on the tiles the screen could not prove cold
        // (rolled over the rows: the registers are free before the force pass)
        if (DO_BREAK && hot) {
#pragma unroll 1
            for (int r = 0; r < EPT; ++r) {
                const int q = q0 + r * AX;
                bool ac = false;
                if (tile_full) cand_terms<false, 0>(ub + q, ub[q], 0u, ac, ps);
                else cand_terms<true, 0>(ub + q, ub[q], ma[q], ac, ps);
                cand |= (ac ? 1u : 0u) << r;
            }
        }
        bool none[EPT];
        // a warp of a tile with broken or absent bonds still takes the unmasked instance
        // when every bond state its own rows read is full: the words of apron rows gy0 ..
        // gy0 + EPT + 2 (its elements and the partners up to three rows below), all columns
        // (fp64 cells only: the masked instance moves 2.4x the shared-memory bytes there --
        // cfg3 36.9 -> 35.1 us; with 8-byte cells the test costs more than it saves)
        bool wfull = tile_full;
        if (!F32 && !tile_full) {
            bool f = true;
            for (int idx = lane; idx < (EPT + R) * AX; idx += 32)
                f = f && (ma[gy0 * AX + idx] & kPos) == kPos;
            wfull = __all_sync(0xffffffffu, f);
        }
        if (wfull) {
#pragma unroll
            for (int sb = 0; sb < EPT; sb += 4)
                pairs_blocked<false, false>(ub + q0 + sb * AX, ue + sb, G0 + sb, G1 + sb, none + sb, ps);
        } else {
            uint32_t m0[EPT];
#pragma unroll
            for (int r = 0; r < EPT; ++r) m0[r] = ma[q0 + r * AX];
            // (the blocked loads with bond states fit the register budget with 8-byte cells
            // only: fp64 spilled ~100 B and ran 37.3 instead of 35.1 us; fp32 positions
            // 32.0 -> 31.7 us)
            if constexpr (F32) {
#pragma unroll
                for (int sb = 0; sb < EPT; sb += 4)
                    pairs_blocked<false, true>(ub + q0 + sb * AX, ue + sb, G0 + sb, G1 + sb,
                                               none + sb, ps, ma + q0 + sb * AX, m0 + sb);
            } else {
                pair_terms<false, true, 0>(ub + q0, ma + q0, ue, m0, G0, G1, none, ps);
            }
        }
    } else if (tile_full) {
#pragma unroll
        for (int k = 0; k < kFusedS; ++k) {
            const double xi0 = st.xi0[k], xi1 = st.xi1[k];
            const double fx0 = st.fx0[k], fx1 = st.fx1[k];
            const long long clo = dbits(st.clo[k]);
            const double2* up_base = ub + q0 + st.aoff[k];
#pragma unroll
            for (int r = 0; r < EPT; ++r) {
                const double2 up = up_base[r * AX];
                const double e0 = up.x - ue[r].x, e1 = up.y - ue[r].y;
                const double dot = fma(xi1, e1, xi0 * e0);
                G0[r] = fma(-dot, fx0, G0[r]);
                G1[r] = fma(-dot, fx1, G1[r]);
                if (DO_BREAK && k >= SHALF)
                    anyc[r] |= dbits(fma(2.0, dot, fma(e1, e1, e0 * e0))) >= clo;
            }
        }
    } else {
        uint32_t m0[EPT];
#pragma unroll
        for (int r = 0; r < EPT; ++r) m0[r] = ma[q0 + r * AX];
#pragma unroll
        for (int k = 0; k < kFusedS; ++k) {
            const double xi0 = st.xi0[k], xi1 = st.xi1[k];
            const double fx0 = st.fx0[k], fx1 = st.fx1[k];
            const long long clo = dbits(st.clo[k]);
            const int aoff = st.aoff[k];
            const double2* up_base = ub + q0 + aoff;
#pragma unroll
            for (int r = 0; r < EPT; ++r) {
                const bool act = k >= SHALF ? ((m0[r] >> k) & 1u)
                                            : ((ma[q0 + r * AX + aoff] >> (kFusedS - 1 - k)) & 1u);
                const double2 up = up_base[r * AX];
                const double e0 = up.x - ue[r].x, e1 = up.y - ue[r].y;
                const double dot = fma(xi1, e1, xi0 * e0);
                const double dm = act ? dot : 0.0;
                G0[r] = fma(-dm, fx0, G0[r]);
                G1[r] = fma(-dm, fx1, G1[r]);
                if (DO_BREAK && k >= SHALF)
                    anyc[r] |= act && dbits(fma(2.0, dot, fma(e1, e1, e0 * e0))) >= clo;
            }
        }
    }
    const bool skip2 = red[4 * NW] != 0u;
    unsigned long long nb = 0;
    if constexpr (!PAIRS) {
#pragma unroll
        for (int r = 0; r < EPT; ++r) cand |= (anyc[r] ? 1u : 0u) << r;
    }
    const bool anyw = cand != 0u;
    // (a clean tile without a candidate in the warp has no bond state to test or write)
    if (!skip2 || __any_sync(0xffffffffu, anyw)) {
    int e[EPT];
    uint32_t m0[EPT], m[EPT];
#pragma unroll
    for (int r = 0; r < EPT; ++r) {
        const int ej = j0 - 1 + gy0 + r;
        const bool in = ei >= 0 && ej >= 0 && ei < nx && ej < ny;
        e[r] = in ? ej * nx + ei : -1;
        m0[r] = skip2 ? 0u : ma[q0 + r * AX];
        m[r] = m0[r];
    }
    bool changed = false;
    if (DO_BREAK) {  // rare: exact per-bond thresholds for the flagged elements
#pragma unroll
        for (int r = 0; r < EPT; ++r) {
            const bool ac = (cand >> r) & 1u;
            if (skip2 && ac) m0[r] = m[r] = bf.mask_in[e[r]];  // (a clean tile staged nothing)
            uint32_t c = ac ? (m0[r] & kPos) : 0u;
            while (c) {
                const int k = __ffs(c) - 1;
                c &= c - 1;
                const double2 up = to_d2(ub[q0 + r * AX + st.aoff[k]]), uer = to_d2(ub[q0 + r * AX]);
                const double e0 = up.x - uer.x, e1 = up.y - uer.y;
                const double dot = fma(st.xi1[k], e1, st.xi0[k] * e0);
                const double lhs = fma(2.0, dot, fma(e1, e1, e0 * e0));
                double thr = st.cthr[k];
                if (d.spread != 0.0) {
                    const int p = e[r] + st.did[k];
                    const double sb =
                        bond_s_crit(d.s_crit, d.spread, d.seed, e[r] + d.goff, p + d.goff);
                    thr = fma(sb, sb, 2.0 * sb) * st.x2[k];
                }
                if (lhs >= thr) {
                    m[r] &= ~(1u << k);
                    if (gx >= 1 && gy0 + r >= 1 && e[r] >= d.own_lo && e[r] < d.own_hi) ++nb;
                }
            }
        }
    }
#pragma unroll
    for (int r = 0; r < EPT; ++r)
        if (e[r] >= 0 && gx >= 1 && gy0 + r >= 1) {
            if (!skip2 || m[r] != m0[r]) bf.mask_out[e[r]] = m[r];
            changed |= m[r] != m0[r];
        }
    if (DO_BREAK && bf.tclean && changed) bf.tclean[(size_t)by * gridDim.x + blockIdx.x] = 0u;
    }
    // the node update needs, per node, (G(x,y) + G(x+1,y)) + (G(x,y+1) + G(x+1,y+1)):
    // the horizontal pair sums come from the neighbour lane, the vertical partner
    // row from this thread's next row -- except for a band's last row, whose
    // partner is the next warp's first row (the only G that goes through smem)
    double2 hsum[EPT];
#pragma unroll
    for (int r = 0; r < EPT; ++r)
        hsum[r] = make_double2(G0[r] + __shfl_down_sync(0xffffffffu, G0[r], 1),
                               G1[r] + __shfl_down_sync(0xffffffffu, G1[r], 1));
    __syncthreads();  // every read of ub is done: the band rows may overwrite it
    if (warp > 0) gt[(warp - 1) * GX + lane] = hsum[0];
    mbar_wait(&bar[1], 0);
    __syncthreads();

    // (4) Verlet update of the owned nodes: column i0 + lane, rows j0 + 4*warp + r.
    //     The grid has floor(n/31) + 1 blocks per axis, so the last block owns at
    //     most 31 node columns / rows including the domain's far node line.
    const int ox = (blockIdx.x == gridDim.x - 1) ? NX - i0 : TX;
    const int oy = (by == maps.grid_rows - 1) ? NY - j0 : TY;
    double2* rdo = reinterpret_cast<double2*>(bf.rd_out);
    double2* rv2 = reinterpret_cast<double2*>(d.rv);
    const double2* P2 = reinterpret_cast<const double2*>(d.P);
    // one node: a = (P - K u) / M, the corrector, the next predictor (the same expressions
    // on both paths below, so they round identically)
    auto node = [&](int r, double im, int fl, bool ws) {
        const int lx = lane, ly = gy0 + r;
        const size_t n = (size_t)(j0 + ly) * NX + i0 + lx;
        const double2 hn = r + 1 < EPT ? hsum[r + 1] : gt[warp * GX + lx];  // row ly + 1
        const double k0 = d.Nsh * (hsum[r].x + hn.x);
        const double k1 = d.Nsh * (hsum[r].y + hn.y);
        double2 p = make_double2(0.0, 0.0);
        if (fl & 4) {
            const double sc = bf.scale_dev ? bf.scale_dev[step] : scale;
            p = P2[n];
            p.x *= sc;
            p.y *= sc;
        }
        const double a0 = (fl & 1) ? 0.0 : (p.x - k0) * im;
        const double a1 = (fl & 2) ? 0.0 : (p.y - k1) * im;
        const double2 rv = rvs[ly * TX + lx];
        const double2 rd = nt[(ly + 1 + R) * BX + lx + 1 + R];
        double v0 = rv.x + d.c_corr_v * a0, v1 = rv.y + d.c_corr_v * a1;
        const double u0 = rd.x + d.c_corr_d * a0, u1 = rd.y + d.c_corr_d * a1;
        if (fl & 3) {
            if (fl & 1) v0 = d.bcvel[2 * n];
            if (fl & 2) v1 = d.bcvel[2 * n + 1];
        }
        if (ws) {
            reinterpret_cast<double2*>(d.a)[n] = make_double2(a0, a1);
            reinterpret_cast<double2*>(d.v)[n] = make_double2(v0, v1);
            reinterpret_cast<double2*>(d.u)[n] = make_double2(u0, u1);
        }
        rv2[n] = make_double2(v0 + d.c_pred_v * a0, v1 + d.c_pred_v * a1);
        rdo[n] = make_double2(u0 + d.dt * v0 + d.c_pred_d * a0, u1 + d.dt * v1 + d.c_pred_d * a1);
    };
    // {1/M, flags} of the thread's nodes (lane 31 and row 31 are the apron: not owned)
    double imv[EPT];
    int flor = 0;
#pragma unroll
    for (int r = 0; r < EPT; ++r) {
        imv[r] = (lane < TX && gy0 + r < TY) ? ims[(gy0 + r) * IX + lane + (i0 - ie)] : 0.0;
        flor |= (int)dbits(imv[r]);
    }
    if (ox == TX && oy == TY && !write_state && !__any_sync(0xffffffffu, (flor & 7) != 0)) {
        // interior step of unconstrained, unloaded nodes (nearly every warp): straight-line
        if (lane < TX) {
#pragma unroll
            for (int r = 0; r < EPT; ++r)
                if (gy0 + r < TY) node(r, imv[r], 0, false);
        }
    } else {
#pragma unroll
        for (int r = 0; r < EPT; ++r) {
            if (lane >= ox || gy0 + r >= oy) continue;
            node(r, imv[r], (int)(dbits(imv[r]) & 7), write_state != 0);
        }
    }

    if (DO_BREAK) {  // per warp (no CTA barrier at the tail; breaks are rare)
        if (__any_sync(0xffffffffu, nb != 0)) {
            for (int o = 16; o > 0; o >>= 1) nb += __shfl_down_sync(0xffffffffu, nb, o);
            if (lane == 0) atomicAdd(d.broken_count + step, nb);
        }
    }
}

// clean-tile flags from the current bond states (and mask -> mask_alt, so that both
// ping-pong buffers hold every word before tiles stop re-writing theirs)
__global__ void __launch_bounds__(256) k_tile9_flags(int nx, int ny, const uint32_t* mask,
                                                     uint32_t* mask_alt, uint32_t* tclean) {
    constexpr uint32_t kPos = ((1u << kFusedS) - 1u) & ~((1u << SHALF) - 1u);
    const int i0 = blockIdx.x * TX, j0 = blockIdx.y * TY;
    bool full = true;
    for (int t = threadIdx.x; t < TX * TY; t += 256) {
        const int i = i0 + t % TX, j = j0 + t / TX;
        if (i < nx && j < ny) {
            const uint32_t m = mask[(size_t)j * nx + i];
            mask_alt[(size_t)j * nx + i] = m;
            full = full && (m & kPos) == kPos;
        }
    }
    full = __syncthreads_and(full);
    if (threadIdx.x == 0) tclean[(size_t)blockIdx.y * gridDim.x + blockIdx.x] = full ? 1u : 0u;
}

int tile9_rows(const LatticeDev& L) { return L.ny / TY + 1; }
int tile9_cols(const LatticeDev& L) { return L.nx / TX + 1; }
void launch_tile9_flags(const LatticeDev& L, const uint32_t* mask, uint32_t* mask_alt,
                        uint32_t* tclean, cudaStream_t s) {
    k_tile9_flags<<<dim3(tile9_cols(L), tile9_rows(L)), 256, 0, s>>>(L.nx, L.ny, mask, mask_alt,
                                                                     tclean);
    cudaError_t e = cudaGetLastError();
    if (e != cudaSuccess) throw std::runtime_error(std::string("CUDA: ") + cudaGetErrorString(e));
}
int tile9_tile_rows() { return TY; }

void tile9_boxes(int* rd_x, int* rd_y, int* rv_x, int* rv_y, int* im_x, int* im_y) {
    *rd_x = 2 * BX;
    *rd_y = BY;
    *rv_x = 2 * TX;
    *rv_y = TY;
    *im_x = IX;
    *im_y = TY;
}

namespace {
template <bool B, bool P, bool Q, bool F = false>
void t9_set_smem() {
    cudaError_t e = cudaFuncSetAttribute(k_tile9<B, P, Q, F>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                         kSmem);
    if (e != cudaSuccess) throw std::runtime_error(std::string("CUDA: ") + cudaGetErrorString(e));
}
}  // namespace

int tile9_configure() {
    t9_set_smem<true, false, false>();
    t9_set_smem<false, false, false>();
    t9_set_smem<true, true, false>();
    t9_set_smem<false, true, false>();
    t9_set_smem<true, false, true>();
    t9_set_smem<false, false, true>();
    t9_set_smem<true, true, true>();
    t9_set_smem<false, true, true>();
    t9_set_smem<true, true, false, true>();
    t9_set_smem<false, true, false, true>();
    t9_set_smem<true, true, true, true>();
    t9_set_smem<false, true, true, true>();
    int occ = 0;
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, k_tile9<true, true, false, false>, NT, kSmem);
    return occ;
}


void launch_tile9_step(const DevPD& d, const LatticeDev& L, const Stencil2D& st,
                       const PairStencil2D* ps, const Tile9Maps& maps, const FusedBufs& b,
                       int step, int do_break, double scale, int write_state, bool f32,
                       cudaStream_t s, int row_first, int row_end) {
    if (f32 && !ps) throw std::runtime_error("tile9: the fp32-position variant needs the pair stencil");
    const int rows = tile9_rows(L);
    if (row_end < 0) row_end = rows;
    if (row_first >= row_end) return;
    dim3 grid(L.nx / TX + 1, row_end - row_first, 1);
    Tile9Maps mp = maps;
    mp.row_base = row_first;
    mp.grid_rows = rows;
    const PairStencil2D none{};
    const PairStencil2D& p = ps ? *ps : none;
    cudaLaunchConfig_t cfg{};
    cfg.gridDim = grid;
    cfg.blockDim = dim3(NT, 1, 1);
    cfg.dynamicSmemBytes = kSmem;
    cfg.stream = s;
    cudaLaunchAttribute attr[1];
    attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    attr[0].val.programmaticStreamSerializationAllowed = 1;
    cfg.attrs = attr;
    cfg.numAttrs = 1;
#define PMTS_T9_LAUNCH(B, P, Q, F) \
    cudaLaunchKernelEx(&cfg, k_tile9<B, P, Q, F>, d, L, st, p, mp, b, step, scale, write_state)
#define PMTS_T9_PICK(Q)                                              \
    if (f32) {                                                       \
        if (do_break) PMTS_T9_LAUNCH(true, true, Q, true);           \
        else PMTS_T9_LAUNCH(false, true, Q, true);                   \
    } else if (ps) {                                                 \
        if (do_break) PMTS_T9_LAUNCH(true, true, Q, false);          \
        else PMTS_T9_LAUNCH(false, true, Q, false);                  \
    } else {                                                         \
        if (do_break) PMTS_T9_LAUNCH(true, false, Q, false);         \
        else PMTS_T9_LAUNCH(false, false, Q, false);                 \
    }
    if (b.n_trk > 0) {
        PMTS_T9_PICK(true)
    } else {
        PMTS_T9_PICK(false)
    }
#undef PMTS_T9_PICK
#undef PMTS_T9_LAUNCH
    cudaError_t e = cudaGetLastError();
    if (e != cudaSuccess) throw std::runtime_error(std::string("CUDA: ") + cudaGetErrorString(e));
}

}  // namespace pmts
