// Fused one-kernel fine step for 2D lattices with the 28-offset stencil
// (delta in [3, sqrt(10)) dx -- BASELINE's 3.015 dx), fast mode.
//
// One CTA owns a 31 x 31 block of elements and the nodes at their lower-left
// corners.  It stages the predictor displacement of a node apron and the
// bond-state words of the element apron in shared memory, forms the centroid
// displacements (ubar) of the element apron, evaluates the bond forces of the
// 32 x 32 elements whose G the owned nodes need (its own block plus one ring of
// neighbours, recomputed -- ~7% extra arithmetic instead of a grid-wide
// dependency), and finishes with the Verlet update of the owned nodes.
// Nothing per element goes to HBM except one mask word.
//
// Bond state lives with the bond's lower element only ("positive" offsets,
// mask bits 14..27): the break test -- the |eta|^2 half of the fp64 work of a
// directed entry -- runs once per bond, from its lower end, and the upper end
// reads the state from the staged mask apron.  Bits 0..13 of a mask word are
// not maintained by this kernel (pmts_pd reads them through the lower element).
// The candidate test compares fp64 bit patterns as integers (exact for the
// positive thresholds), off the fp64 pipe.
//
// Thread layout everywhere: lane = column, warp = a band of rows -- no integer
// division in any index, every warp access to shared memory is 32 consecutive
// cells, and the ubar pass reuses the horizontal node-pair sums of a column
// walking up its rows.  8 warps; in the force pass warp w owns rows 4w..4w+3,
// so every per-offset constant (kernel parameter space) is fetched once per
// thread and used for 4 elements.  Displacement and mask are ping-ponged
// across steps so neighbouring CTAs never observe a half-updated step.
// Reference semantics as in pd_stencil.cu.
#include <stdexcept>
#include <string>

#include "pd_stencil.cuh"

namespace pmts {

namespace {

constexpr int TX = 31, TY = 31, R = kFusedR;
constexpr int GX = TX + 1, GY = TY + 1;          // force region (elements), 32 x 32
constexpr int AX = GX + 2 * R, AY = GY + 2 * R;  // ubar apron (elements), 38 x 38
constexpr int BX = AX + 1, BY = AY + 1;          // node apron, 39 x 39
constexpr int NW = 8, NT = 32 * NW;
constexpr int EPT = GY / NW;                     // 4 rows per warp
constexpr int SHALF = kFusedS / 2;               // offsets 0..13 negative, 14..27 positive
static_assert(GX == 32 && EPT * NW == GY, "lane = column, warp = EPT rows");
static_assert(AX == kFusedAX, "Stencil2D apron offsets assume this width");
constexpr int NRB = (BY + NW - 1) / NW;          // node-apron rows per warp (5)
constexpr int URB = (AY + NW - 1) / NW;          // ubar rows per warp (5)

constexpr size_t kSmem = sizeof(double2) * (BX * BY + AX * AY + GX * GY) +
                         sizeof(uint32_t) * AX * AY;

__device__ __forceinline__ long long dbits(double x) { return __double_as_longlong(x); }

}  // namespace

template <bool DO_BREAK>
__global__ void __launch_bounds__(NT, 3)
k_fused2d(DevPD d, LatticeDev L, const __grid_constant__ Stencil2D st, FusedBufs bf, int step,
          double scale, int write_state) {
    extern __shared__ __align__(16) double2 sm2[];
    double2* nt = sm2;                 // BX * BY node apron
    double2* ub = nt + BX * BY;        // AX * AY element apron
    double2* gt = ub + AX * AY;        // GX * GY element forces
    uint32_t* ma = reinterpret_cast<uint32_t*>(gt + GX * GY);  // AX * AY mask apron
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    const int nx = L.nx, ny = L.ny, NX = nx + 1, NY = ny + 1;
    const int i0 = blockIdx.x * TX, j0 = blockIdx.y * TY;
    const int ax0 = i0 - 1 - R, ay0 = j0 - 1 - R;  // apron origin (element = node index)
    const double2* rd2 = reinterpret_cast<const double2*>(bf.rd_in);

    // (1) stage the apron: warp w takes rows w, w+8, ...; lanes take columns
    //     lane and lane+32; every load of a thread is issued before any store
    {
        double2 nv[NRB][2];
        uint32_t mv[URB][2];
#pragma unroll
        for (int i = 0; i < NRB; ++i) {
            const int by = warp + NW * i, gj = ay0 + by;
#pragma unroll
            for (int h = 0; h < 2; ++h) {
                const int bx = lane + 32 * h, gi = ax0 + bx;
                nv[i][h] = make_double2(0.0, 0.0);
                if (by < BY && bx < BX && gi >= 0 && gj >= 0 && gi < NX && gj < NY)
                    nv[i][h] = rd2[(size_t)gj * NX + gi];
            }
        }
#pragma unroll
        for (int i = 0; i < URB; ++i) {
            const int y = warp + NW * i, gj = ay0 + y;
#pragma unroll
            for (int h = 0; h < 2; ++h) {
                const int x = lane + 32 * h, gi = ax0 + x;
                mv[i][h] = 0u;
                if (y < AY && x < AX && gi >= 0 && gj >= 0 && gi < nx && gj < ny)
                    mv[i][h] = bf.mask_in[(size_t)gj * nx + gi];
            }
        }
#pragma unroll
        for (int i = 0; i < NRB; ++i)
#pragma unroll
            for (int h = 0; h < 2; ++h) {
                const int by = warp + NW * i, bx = lane + 32 * h;
                if (by < BY && bx < BX) nt[by * BX + bx] = nv[i][h];
            }
#pragma unroll
        for (int i = 0; i < URB; ++i)
#pragma unroll
            for (int h = 0; h < 2; ++h) {
                const int y = warp + NW * i, x = lane + 32 * h;
                if (y < AY && x < AX) ma[y * AX + x] = mv[i][h];
            }
    }
    __syncthreads();

    // (2) ubar of the apron: a thread walks up a column band (rows URB*warp ..),
    //     carrying the horizontal node-pair sum of the row above to the next row
    constexpr uint32_t kPos = ((1u << kFusedS) - 1u) & ~((1u << SHALF) - 1u);
    bool tile_full = true;  // every apron element carries its full intact positive stencil
#pragma unroll
    for (int h = 0; h < 2; ++h) {
        const int x = lane + 32 * h;
        const int y0 = URB * warp;
        if (x < AX && y0 < AY) {
            // all node pairs of the band first (independent shared loads in flight),
            // then the sums; rows past the apron read the (zero-padded) top node row
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
                    tile_full = tile_full && (ma[y * AX + x] & kPos) == kPos;
                }
            }
        }
    }
    tile_full = __syncthreads_and(tile_full);

    // (3) forces of the 32 x 32 region: column = lane, rows EPT*warp + r
    const int gx = lane, gy0 = warp * EPT;
    const int ei = i0 - 1 + gx;
    const int q0 = (gy0 + R) * AX + gx + R;
    int e[EPT];
    uint32_t m0[EPT], m[EPT];
    double2 ue[EPT];
    double G0[EPT], G1[EPT];
#pragma unroll
    for (int r = 0; r < EPT; ++r) {
        const int ej = j0 - 1 + gy0 + r;
        const bool in = ei >= 0 && ej >= 0 && ei < nx && ej < ny;
        e[r] = in ? ej * nx + ei : -1;
        m0[r] = ma[q0 + r * AX];
        m[r] = m0[r];
        ue[r] = ub[q0 + r * AX];
        G0[r] = 0.0;
        G1[r] = 0.0;
    }
    bool anyc[EPT];
#pragma unroll
    for (int r = 0; r < EPT; ++r) anyc[r] = false;
    if (tile_full) {
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
    // rare: exact per-bond thresholds for the flagged elements
    unsigned long long nb = 0;
    if (DO_BREAK) {
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
    for (int r = 0; r < EPT; ++r) {
        if (e[r] >= 0 && gx >= 1 && gy0 + r >= 1) bf.mask_out[e[r]] = m[r];
        gt[(gy0 + r) * GX + gx] = make_double2(G0[r], G1[r]);
    }

    // (4) Verlet update of the owned nodes: column i0 + lane, rows j0 + 4*warp + r
    //     (the last block row/column also owns the domain's far node line, whose
    //     nodes sit at lane 31 / row 31 of the 32 x 32 node region)
    const int ox = (blockIdx.x == gridDim.x - 1) ? NX - i0 : TX;
    const int oy = (blockIdx.y == gridDim.y - 1) ? NY - j0 : TY;
    double2* rdo = reinterpret_cast<double2*>(bf.rd_out);
    double2* rv2 = reinterpret_cast<double2*>(d.rv);
    const double2* P2 = reinterpret_cast<const double2*>(d.P);
    double2 rvv[EPT];
    double imv[EPT];
    uint8_t flv[EPT];
#pragma unroll
    for (int r = 0; r < EPT; ++r) {
        const int ly = gy0 + r;
        rvv[r] = make_double2(0.0, 0.0);
        imv[r] = 0.0;
        flv[r] = 0;
        if (lane < ox && ly < oy) {
            const size_t n = (size_t)(j0 + ly) * NX + i0 + lane;
            rvv[r] = rv2[n];
            imv[r] = L.inv_mass[n];
            flv[r] = L.nflag[n];
        }
    }
    __syncthreads();
#pragma unroll
    for (int r = 0; r < EPT; ++r) {
        const int lx = lane, ly = gy0 + r;
        if (lx >= ox || ly >= oy) continue;
        const size_t n = (size_t)(j0 + ly) * NX + i0 + lx;
        // incident elements (ni-1|ni, nj-1|nj) sit at force-region (lx|lx+1, ly|ly+1)
        const double2 a = gt[ly * GX + lx];
        const double2 c = gt[(ly + 1 < GY ? ly + 1 : ly) * GX + lx];
        const double2 b = lx + 1 < GX ? gt[ly * GX + lx + 1] : make_double2(0.0, 0.0);
        const double2 f = (lx + 1 < GX && ly + 1 < GY) ? gt[(ly + 1) * GX + lx + 1]
                                                       : make_double2(0.0, 0.0);
        const double2 cc = ly + 1 < GY ? c : make_double2(0.0, 0.0);
        const double k0 = d.Nsh * ((a.x + b.x) + (cc.x + f.x));
        const double k1 = d.Nsh * ((a.y + b.y) + (cc.y + f.y));
        const uint8_t fl = flv[r];
        const double im = imv[r];
        double2 p = make_double2(0.0, 0.0);
        if (fl & 8) {
            p = P2[n];
            p.x *= scale;
            p.y *= scale;
        }
        const double a0 = (fl & 1) ? 0.0 : (p.x - k0) * im;
        const double a1 = (fl & 2) ? 0.0 : (p.y - k1) * im;
        const double2 rv = rvv[r];
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
        __shared__ unsigned long long part[NW];
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

void fused2d_configure() {
    for (auto fn : {k_fused2d<true>, k_fused2d<false>}) {
        cudaError_t e =
            cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)kSmem);
        if (e != cudaSuccess)
            throw std::runtime_error(std::string("CUDA: ") + cudaGetErrorString(e));
    }
}

void launch_fused2d_step(const DevPD& d, const LatticeDev& L, const Stencil2D& st,
                         const FusedBufs& b, int step, int do_break, double scale,
                         int write_state, cudaStream_t s) {
    dim3 grid((L.nx + TX - 1) / TX, (L.ny + TY - 1) / TY, 1);
    if (do_break) k_fused2d<true><<<grid, NT, kSmem, s>>>(d, L, st, b, step, scale, write_state);
    else k_fused2d<false><<<grid, NT, kSmem, s>>>(d, L, st, b, step, scale, write_state);
    cudaError_t e = cudaGetLastError();
    if (e != cudaSuccess) throw std::runtime_error(std::string("CUDA: ") + cudaGetErrorString(e));
}

}  // namespace pmts
