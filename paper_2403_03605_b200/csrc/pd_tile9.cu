// One-shot fused 2D fine step with TMA staging (tile v9), 28-offset stencil,
// fast mode.  Arithmetic is the tile kernel's (pd_stencil_fused.cu: 31 x 31
// owned elements, 32 x 32 force region, bond state at the lower end, integer
// candidate compare) -- the two kernels are bitwise equal -- what changes is
// how the CTA gets its inputs:
//
//   * at launch one thread issues three cp.async.bulk.tensor loads completing
//     on two mbarriers -- the node apron of the predictor displacement (needed
//     first), and the owned nodes' rv and {1/M, flags} (needed last, so their
//     latency hides behind the ubar and force passes).  Out-of-domain parts of
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
#include <stdexcept>
#include <string>

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
constexpr int kMinBlocks = NW == 8 ? 3 : 2;
constexpr int EPT = GY / NW;
constexpr int SHALF = kFusedS / 2;
constexpr int URB = (AY + NW - 1) / NW;
static_assert(GX == 32 && EPT * NW == GY, "lane = column, warp = EPT rows");
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
constexpr int kSmem = kOffBar + 16 + 128;        // + realignment slack of the dynamic base
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
    constexpr int A = kPairA[K], B = kPairB[K];
    const double ep0 = up.x - ue.x, ep1 = up.y - ue.y;
    double em0 = um.x - ue.x, em1 = um.y - ue.y;
    if (MASKED) {
        em0 = actm ? em0 : 0.0;
        em1 = actm ? em1 : 0.0;
    }
    const double fp0 = MASKED && !actp ? 0.0 : ep0, fp1 = MASKED && !actp ? 0.0 : ep1;
    double tp;
    if (B == 0) {
        const double s0 = fp0 + em0;
        G0 = fma(ps.fa[K], s0, G0);
        tp = A * ep0;
    } else if (A == 0) {
        const double s1 = fp1 + em1;
        G1 = fma(ps.fb[K], s1, G1);
        tp = B * ep1;
    } else {
        const double s0 = fp0 + em0, s1 = fp1 + em1;
        const double t = fma((double)A, s0, B * s1);
        G0 = fma(ps.fa[K], t, G0);
        G1 = fma(ps.fb[K], t, G1);
        tp = fma((double)A, ep0, B * ep1);
    }
    if (DO_BREAK)
        anyc |= (!MASKED || actp) && dbits(fma(ps.h2, tp, fma(ep0, ep0, ep1 * ep1))) >= ps.cl[K];
}

template <bool DO_BREAK, bool MASKED, int K>
__device__ __forceinline__ void pair_term(const double2* ubq, const uint32_t* maq,
                                          const double2 (&ue)[EPT], const uint32_t (&m0)[EPT],
                                          double (&G0)[EPT], double (&G1)[EPT],
                                          bool (&anyc)[EPT], const PairStencil2D& ps) {
    const int off = ps.off[K];
    const double2* pp = ubq + off;
    const double2* pm = ubq - off;
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
template <bool DO_BREAK>
__device__ __forceinline__ void pairs_blocked(const double2* ubq, const double2 (&ue)[EPT],
                                              double (&G0)[EPT], double (&G1)[EPT],
                                              bool (&anyc)[EPT], const PairStencil2D& ps) {
    static_assert(EPT == 4, "blocked path assumes 4 rows per thread");
    {  // A = 0: (0,1) (0,2) (0,3)
        double2 c[10];
#pragma unroll
        for (int i = 0; i < 10; ++i) c[i] = (i >= 3 && i < 7) ? ue[i - 3] : ubq[(i - 3) * AX];
#pragma unroll
        for (int r = 0; r < EPT; ++r) {
            pair_math<DO_BREAK, false, 0>(c[r + 4], c[r + 2], ue[r], true, true, G0[r], G1[r], anyc[r], ps);
            pair_math<DO_BREAK, false, 1>(c[r + 5], c[r + 1], ue[r], true, true, G0[r], G1[r], anyc[r], ps);
            pair_math<DO_BREAK, false, 2>(c[r + 6], c[r], ue[r], true, true, G0[r], G1[r], anyc[r], ps);
        }
    }
#pragma unroll
    for (int g = 1; g <= 2; ++g) {    // |A| = 1: pairs 3..7, |A| = 2: pairs 8..12
#pragma unroll
        for (int half = 0; half < 2; ++half) {  // rows 2 half .. 2 half + 1: cells rows -2..3 (+2 half)
            double2 p[6], m[6];
#pragma unroll
            for (int i = 0; i < 6; ++i) {
                p[i] = ubq[(i - 2 + 2 * half) * AX + g];
                m[i] = ubq[(i - 2 + 2 * half) * AX - g];
            }
#pragma unroll
            for (int rr = 0; rr < 2; ++rr) {
                const int r = 2 * half + rr, q = rr + 2;
                if (g == 1) {
                    pair_math<DO_BREAK, false, 3>(p[q], m[q], ue[r], true, true, G0[r], G1[r], anyc[r], ps);
                    pair_math<DO_BREAK, false, 4>(p[q + 1], m[q - 1], ue[r], true, true, G0[r], G1[r], anyc[r], ps);
                    pair_math<DO_BREAK, false, 5>(m[q + 1], p[q - 1], ue[r], true, true, G0[r], G1[r], anyc[r], ps);
                    pair_math<DO_BREAK, false, 6>(p[q + 2], m[q - 2], ue[r], true, true, G0[r], G1[r], anyc[r], ps);
                    pair_math<DO_BREAK, false, 7>(m[q + 2], p[q - 2], ue[r], true, true, G0[r], G1[r], anyc[r], ps);
                } else {
                    pair_math<DO_BREAK, false, 8>(p[q], m[q], ue[r], true, true, G0[r], G1[r], anyc[r], ps);
                    pair_math<DO_BREAK, false, 9>(p[q + 1], m[q - 1], ue[r], true, true, G0[r], G1[r], anyc[r], ps);
                    pair_math<DO_BREAK, false, 10>(m[q + 1], p[q - 1], ue[r], true, true, G0[r], G1[r], anyc[r], ps);
                    pair_math<DO_BREAK, false, 11>(p[q + 2], m[q - 2], ue[r], true, true, G0[r], G1[r], anyc[r], ps);
                    pair_math<DO_BREAK, false, 12>(m[q + 2], p[q - 2], ue[r], true, true, G0[r], G1[r], anyc[r], ps);
                }
            }
        }
    }
#pragma unroll
    for (int r = 0; r < EPT; ++r)  // |A| = 3: (3,0)
        pair_math<DO_BREAK, false, 13>(ubq[r * AX + 3], ubq[r * AX - 3], ue[r], true, true, G0[r],
                                       G1[r], anyc[r], ps);
}

template <bool DO_BREAK, bool MASKED, int K>
__device__ __forceinline__ void pair_terms(const double2* ubq, const uint32_t* maq,
                                           const double2 (&ue)[EPT], const uint32_t (&m0)[EPT],
                                           double (&G0)[EPT], double (&G1)[EPT],
                                           bool (&anyc)[EPT], const PairStencil2D& ps) {
    if constexpr (K < 14) {
        pair_term<DO_BREAK, MASKED, K>(ubq, maq, ue, m0, G0, G1, anyc, ps);
        pair_terms<DO_BREAK, MASKED, K + 1>(ubq, maq, ue, m0, G0, G1, anyc, ps);
    }
}

}  // namespace

int tile9_pair_offset(int k, int* a, int* b) {
    static const int A[14] = {0, 0, 0, 1, 1, -1, 1, -1, 2, 2, -2, 2, -2, 3};
    static const int B[14] = {1, 2, 3, 0, 1, 1, 2, 2, 0, 1, 1, 2, 2, 0};
    *a = A[k];
    *b = B[k];
    return 14;
}

template <bool DO_BREAK, bool PAIRS, bool REPORT>
__global__ void __launch_bounds__(NT, kMinBlocks)
k_tile9(DevPD d, LatticeDev L, const __grid_constant__ Stencil2D st,
        const __grid_constant__ PairStencil2D ps, const __grid_constant__ Tile9Maps maps,
        FusedBufs bf, int step, double scale, int write_state) {
    extern __shared__ __align__(16) unsigned char smraw[];
    // the dynamic base is only guaranteed 16-byte aligned: realign for TMA
    unsigned char* sm = smraw + ((128u - (smem_u32(smraw) & 127u)) & 127u);
    const double2* nt = reinterpret_cast<const double2*>(sm + kOffNt);
    uint32_t* ma = reinterpret_cast<uint32_t*>(sm + kOffMa);
    const double2* rvs = reinterpret_cast<const double2*>(sm + kOffRv);
    const double* ims = reinterpret_cast<const double*>(sm + kOffIm);
    double2* ub = reinterpret_cast<double2*>(sm + kOffUb);
    double2* gt = ub;  // G aliases the ubar apron once the force pass is done
    uint64_t* bar = reinterpret_cast<uint64_t*>(sm + kOffBar);
    unsigned long long* part = reinterpret_cast<unsigned long long*>(sm + kOffPart);
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    const int nx = L.nx, ny = L.ny, NX = nx + 1, NY = ny + 1;
    const int i0 = blockIdx.x * TX, j0 = blockIdx.y * TY;
    const int ax0 = i0 - 1 - R, ay0 = j0 - 1 - R;
    const int ie = i0 & ~1;  // {1/M, flags} box start: 16-byte aligned global row start

    // (1) staging: TMA for the node apron and the node-update inputs; 4-byte
    //     cp.async (zero-filled outside the domain) for the bond-state apron
    if (threadIdx.x == 0) {
        mbar_init(&bar[0], 1);
        mbar_init(&bar[1], 1);
        asm volatile("fence.mbarrier_init.release.cluster;\n" ::);
        mbar_expect_tx(&bar[0], kNtBytes);
        tma_load_2d(sm + kOffNt, &maps.rd, 2 * ax0, ay0, &bar[0]);
        mbar_expect_tx(&bar[1], kRvBytes + kImBytes);
        tma_load_2d(sm + kOffRv, &maps.rv, 2 * i0, j0, &bar[1]);
        tma_load_2d(sm + kOffIm, &maps.im, ie, j0, &bar[1]);
    }
    if constexpr (REPORT) {
        // pmts_pd_step_tracked: the step's u is the predictor it consumes (beta = 0);
        // block (0, 0) copies the tracked dofs of it into mapped pinned host memory
        if ((blockIdx.x | blockIdx.y) == 0)
            for (int j = threadIdx.x; j < bf.n_trk; j += NT) bf.trk_host[j] = bf.rd_in[bf.trk_dofs[j]];
    }
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
    asm volatile("cp.async.commit_group;\n" ::);
    asm volatile("cp.async.wait_group 0;\n" ::: "memory");
    __syncthreads();
    mbar_wait(&bar[0], 0);

    // (2) ubar of the apron (column walk with carried node-pair sums); the
    //     positive-stencil completeness of every mask the force pass reads
    constexpr uint32_t kPos = ((1u << kFusedS) - 1u) & ~((1u << SHALF) - 1u);
    bool tile_full = true;
#pragma unroll
    for (int h = 0; h < 2; ++h) {
        const int x = lane + 32 * h;
        const int y0 = URB * warp;
        if (x < AX && y0 < AY) {
            double2 hs[URB + 1];
#pragma unroll
            for (int i = 0; i <= URB; ++i) {
                const int y = min(y0 + i, BY - 1);
                const double2 a = nt[y * BX + x], b = nt[y * BX + x + 1];
                hs[i] = make_double2(a.x + b.x, a.y + b.y);
            }
#pragma unroll
            for (int i = 0; i < URB; ++i) {
                const int y = y0 + i;
                if (y < AY) {
                    ub[y * AX + x] = make_double2(d.Nsh * (hs[i].x + hs[i + 1].x),
                                                  d.Nsh * (hs[i].y + hs[i + 1].y));
                    if (y < MY) tile_full = tile_full && (ma[y * AX + x] & kPos) == kPos;
                }
            }
        }
    }
    tile_full = __syncthreads_and(tile_full);

    // (3) forces of the 32 x 32 region: column = lane, rows EPT*warp + r
    const int gx = lane, gy0 = warp * EPT;
    const int ei = i0 - 1 + gx;
    const int q0 = (gy0 + R) * AX + gx + R;
    // only ue, G and the candidate flags stay live through the force pass (the
    // element ids and bond-state words are re-derived afterwards: registers)
    double2 ue[EPT];
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
    if (PAIRS && tile_full) {
        pairs_blocked<DO_BREAK>(ub + q0, ue, G0, G1, anyc, ps);
    } else if (PAIRS) {
        uint32_t m0[EPT];
#pragma unroll
        for (int r = 0; r < EPT; ++r) m0[r] = ma[q0 + r * AX];
        pair_terms<DO_BREAK, true, 0>(ub + q0, ma + q0, ue, m0, G0, G1, anyc, ps);
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
    int e[EPT];
    uint32_t m0[EPT], m[EPT];
#pragma unroll
    for (int r = 0; r < EPT; ++r) {
        const int ej = j0 - 1 + gy0 + r;
        const bool in = ei >= 0 && ej >= 0 && ei < nx && ej < ny;
        e[r] = in ? ej * nx + ei : -1;
        m0[r] = ma[q0 + r * AX];
        m[r] = m0[r];
    }
    unsigned long long nb = 0;
    if (DO_BREAK) {  // rare: exact per-bond thresholds for the flagged elements
#pragma unroll
        for (int r = 0; r < EPT; ++r) {
            uint32_t c = anyc[r] ? (m0[r] & kPos) : 0u;
            while (c) {
                const int k = __ffs(c) - 1;
                c &= c - 1;
                const double2 up = ub[q0 + r * AX + st.aoff[k]];
                const double e0 = up.x - ue[r].x, e1 = up.y - ue[r].y;
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
        if (e[r] >= 0 && gx >= 1 && gy0 + r >= 1) bf.mask_out[e[r]] = m[r];
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
    const int oy = (blockIdx.y == gridDim.y - 1) ? NY - j0 : TY;
    double2* rdo = reinterpret_cast<double2*>(bf.rd_out);
    double2* rv2 = reinterpret_cast<double2*>(d.rv);
    const double2* P2 = reinterpret_cast<const double2*>(d.P);
#pragma unroll
    for (int r = 0; r < EPT; ++r) {
        const int lx = lane, ly = gy0 + r;
        if (lx >= ox || ly >= oy) continue;
        const size_t n = (size_t)(j0 + ly) * NX + i0 + lx;
        const double2 hn = r + 1 < EPT ? hsum[r + 1] : gt[warp * GX + lx];  // row ly + 1
        const double k0 = d.Nsh * (hsum[r].x + hn.x);
        const double k1 = d.Nsh * (hsum[r].y + hn.y);
        const double im = ims[ly * IX + lx + (i0 - ie)];
        const int fl = (int)(dbits(im) & 7);  // 1: x constrained, 2: y constrained, 4: loaded
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
        if (write_state) {
            reinterpret_cast<double2*>(d.a)[n] = make_double2(a0, a1);
            reinterpret_cast<double2*>(d.v)[n] = make_double2(v0, v1);
            reinterpret_cast<double2*>(d.u)[n] = make_double2(u0, u1);
        }
        rv2[n] = make_double2(v0 + d.c_pred_v * a0, v1 + d.c_pred_v * a1);
        rdo[n] = make_double2(u0 + d.dt * v0 + d.c_pred_d * a0, u1 + d.dt * v1 + d.c_pred_d * a1);
    }

    if (DO_BREAK) {
        for (int o = 16; o > 0; o >>= 1) nb += __shfl_down_sync(0xffffffffu, nb, o);
        if (lane == 0) part[warp] = nb;
        __syncthreads();
        if (threadIdx.x == 0) {
            unsigned long long t = 0;
            for (int w = 0; w < NW; ++w) t += part[w];
            if (t) atomicAdd(d.broken_count + step, t);
        }
    }
}

void tile9_boxes(int* rd_x, int* rd_y, int* rv_x, int* rv_y, int* im_x, int* im_y) {
    *rd_x = 2 * BX;
    *rd_y = BY;
    *rv_x = 2 * TX;
    *rv_y = TY;
    *im_x = IX;
    *im_y = TY;
}

namespace {
template <bool B, bool P, bool Q>
void t9_set_smem() {
    cudaError_t e = cudaFuncSetAttribute(k_tile9<B, P, Q>, cudaFuncAttributeMaxDynamicSharedMemorySize,
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
    int occ = 0;
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, k_tile9<true, true, false>, NT, kSmem);
    return occ;
}

void launch_tile9_step(const DevPD& d, const LatticeDev& L, const Stencil2D& st,
                       const PairStencil2D* ps, const Tile9Maps& maps, const FusedBufs& b,
                       int step, int do_break, double scale, int write_state, cudaStream_t s) {
    dim3 grid(L.nx / TX + 1, L.ny / TY + 1, 1);
    const PairStencil2D none{};
    const PairStencil2D& p = ps ? *ps : none;
#define PMTS_T9_LAUNCH(B, P, Q) \
    k_tile9<B, P, Q><<<grid, NT, kSmem, s>>>(d, L, st, p, maps, b, step, scale, write_state)
#define PMTS_T9_PICK(Q)                                              \
    if (ps) {                                                        \
        if (do_break) PMTS_T9_LAUNCH(true, true, Q);                 \
        else PMTS_T9_LAUNCH(false, true, Q);                         \
    } else {                                                         \
        if (do_break) PMTS_T9_LAUNCH(true, false, Q);                \
        else PMTS_T9_LAUNCH(false, false, Q);                        \
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
