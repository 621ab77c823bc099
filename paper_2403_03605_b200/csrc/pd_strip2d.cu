// Row-streaming, bond-symmetric fused fine step for 2D lattices with the
// 28-offset stencil (delta in [3, sqrt(10)) dx; BASELINE's 3.015 dx), fast mode.
//
// Why: the per-directed-bond arithmetic (eta, xi.eta, force, |eta|^2, test) is
// fp64 work on the B200's fp64 pipe; the one-shot tile kernel evaluates every
// bond twice (once from each end).  Here each bond is evaluated ONCE, by its
// "source" element (the left end, or the lower end of a vertical bond), and the
// reaction reaches the other end through a warp shuffle (horizontal) or a
// register (vertical) -- no shared-memory atomics, no grid-wide dependency.
//
// Work unit = one warp = a strip of 32 element columns (lane = column; the 4
// leftmost lanes are margin: their G only feeds the useful columns) x one
// segment of H node rows.  The warp streams the segment bottom-up two source
// rows at a time: per iteration it extends a ring of centroid displacements
// (ubar) by two rows (from node rows fetched one iteration ahead), evaluates
// the 14 "positive" bonds of both source rows with each per-offset constant
// loaded once, accumulates own forces and reactions in a 7-row register
// window of G, and performs the Verlet update of the two node rows whose G is
// now final.  Margin rows (below / above the segment) take a filtered path
// that skips bonds with both ends outside the useful rows.
//
// Every useful element accumulates its 28 contributions in the same fixed
// order whatever strip or segment (or rank) it falls in, so results are
// bitwise independent of the decomposition.  The break test is evaluated once
// per bond (so both directed bits always agree); the rare breaking path
// (warp vote) applies the exact per-bond threshold and clears the source's
// bit directly and the target's through the same shuffle.
#include <stdexcept>
#include <string>

#include "pd_stencil.cuh"

namespace pmts {

namespace {

constexpr int NP = 14;                 // positive offsets
constexpr int SH = 36;                 // ring row stride (element columns cb .. cb+35)
constexpr int RING = 8;                // ubar ring rows
constexpr int NRING = 4;               // node ring rows
constexpr int WARPS = 4;
constexpr int kOwnLane0 = 4;           // lanes >= 4: own node / element column
constexpr int kColsPerStrip = 32 - kOwnLane0;  // 28

// Positive offsets (di >= 0; di == 0 -> dj > 0) of the 28-offset stencil, in
// this order:  (0,1) (0,2) (0,3) (1,-2) (1,-1) (1,0) (1,1) (1,2) (2,-2) (2,-1)
// (2,0) (2,1) (2,2) (3,0).  Plain conditional functions so that, inside the
// fully unrolled bond loop, every use folds to an immediate.
__host__ __device__ constexpr int pdi(int k) { return k < 3 ? 0 : k < 8 ? 1 : k < 13 ? 2 : 3; }
__host__ __device__ constexpr int pdj(int k) {
    return k < 3 ? k + 1 : k < 8 ? k - 5 : k < 13 ? k - 10 : 0;
}
// index of the offset / of its reverse in the 28-offset list sorted by (dj, di)
// -- the host's stencil order (ascending linear element-id delta)
__host__ __device__ constexpr int pkp(int k) {
    return k == 0 ? 19 : k == 1 ? 24 : k == 2 ? 27 : k == 3 ? 4 : k == 4 ? 9 : k == 5 ? 14
         : k == 6 ? 20 : k == 7 ? 25 : k == 8 ? 5 : k == 9 ? 10 : k == 10 ? 15 : k == 11 ? 21
         : k == 12 ? 26 : 16;
}
__host__ __device__ constexpr int pkn(int k) { return 27 - pkp(k); }  // list is point-symmetric

constexpr int stencil_index(int di, int dj) {
    int idx = 0;
    for (int j = -3; j <= 3; ++j)
        for (int i = -3; i <= 3; ++i) {
            if (i * i + j * j > 9 || (i == 0 && j == 0)) continue;
            if (j == dj && i == di) return idx;
            ++idx;
        }
    return -1;
}
static_assert(stencil_index(0, 1) == 19 && stencil_index(3, 0) == 16 &&
                  stencil_index(-2, 1) == 17 && stencil_index(0, -3) == 0 && pkn(0) == 8,
              "stencil order");

constexpr size_t kWarpSmem = sizeof(double2) * (RING * SH + NRING * SH);
constexpr size_t kSmem = kWarpSmem * WARPS;

struct RowCtx {  // per source row
    double2 ue;
    uint32_t m;
    long long eid;  // global-ish element id of (c, row) (local numbering)
    bool own;       // counted for broken bonds
};

}  // namespace

int strip2d_pos_offset(int k, int* di, int* dj) {
    *di = pdi(k);
    *dj = pdj(k);
    if (stencil_index(pdi(k), pdj(k)) != pkp(k) || stencil_index(-pdi(k), -pdj(k)) != pkn(k))
        throw std::logic_error("strip2d offset tables inconsistent");
    return pkp(k);
}

// Evaluate the 14 positive bonds of source row w (window index WS = 2 or 3).
// FILTER: margin rows -- skip bonds with neither end in the useful rows.
// ACTSEL: some lane lacks a full intact stencil -- select by the mask bit.
template <bool DO_BREAK, bool ACTSEL, bool FILTER, int WS>
__device__ __forceinline__ void bonds_row(const DevPD& d, const StripStencil& st,
                                          const double2* __restrict__ rowp[7], RowCtx& rc,
                                          double (&G0)[7], double (&G1)[7], uint32_t (&mw)[7],
                                          int lane, int ys, int y_lo, int y_hi,
                                          unsigned long long& nb) {
    const bool src_useful = ys >= y_lo - 1 && ys < y_hi;
#pragma unroll
    for (int k = 0; k < NP; ++k) {
        const int di = pdi(k), dj = pdj(k);
        if (FILTER) {
            const int tr = ys + dj;
            if (!src_useful && !(tr >= y_lo - 1 && tr < y_hi)) continue;  // warp-uniform
        }
        const double2 up = rowp[WS + dj][lane + di];
        const double e0 = up.x - rc.ue.x, e1 = up.y - rc.ue.y;
        const double dot = fma(st.xi1[k], e1, st.xi0[k] * e0);
        bool act = true;
        double dm = dot;
        if (ACTSEL) {
            act = (rc.m >> pkp(k)) & 1u;
            dm = act ? dot : 0.0;
        }
        G0[WS] = fma(-dm, st.fx0[k], G0[WS]);
        G1[WS] = fma(-dm, st.fx1[k], G1[WS]);
        // reaction at (lane + di, row + dj); lanes < di receive their own value --
        // they are margin lanes (< 4) whose G is never used
        const double rm = di > 0 ? __shfl_up_sync(0xffffffffu, dm, di) : dm;
        G0[WS + dj] = fma(rm, st.fx0[k], G0[WS + dj]);
        G1[WS + dj] = fma(rm, st.fx1[k], G1[WS + dj]);
        if (DO_BREAK) {
            const double lhs = fma(2.0, dot, fma(e1, e1, e0 * e0));
            const bool cand = act && lhs >= st.clo[k];
            if (__any_sync(0xffffffffu, cand)) {  // rare
                bool brk = false;
                if (cand) {
                    double thr = st.cthr[k];
                    if (d.spread != 0.0) {
                        const long long se = rc.eid, te = rc.eid + st.did[k];
                        const long long lo = se < te ? se : te, hi = se < te ? te : se;
                        const double sb =
                            bond_s_crit(d.s_crit, d.spread, d.seed, lo + d.goff, hi + d.goff);
                        thr = fma(sb, sb, 2.0 * sb) * st.x2[k];
                    }
                    brk = lhs >= thr;
                }
                if (brk) {
                    mw[WS] &= ~(1u << pkp(k));
                    if (rc.own) ++nb;
                }
                const bool tb = di > 0 ? __shfl_up_sync(0xffffffffu, brk, di) : brk;
                if (tb) mw[WS + dj] &= ~(1u << pkn(k));  // lanes < di: margin, never written
            }
        }
    }
}

template <bool DO_BREAK, int WS>
__device__ __forceinline__ void source_row(const DevPD& d, const StripStencil& st,
                                           const double2* __restrict__ rowp[7], double (&G0)[7],
                                           double (&G1)[7], uint32_t (&mw)[7], int lane, int c,
                                           bool own_col, bool col_ok, int nx, int ny, int ys,
                                           int y_lo, int y_hi, unsigned long long& nb) {
    if (ys < 0 || ys >= ny) return;  // no elements on this row (warp-uniform)
    RowCtx rc;
    rc.ue = rowp[WS][lane];
    rc.m = mw[WS];
    rc.eid = (long long)ys * nx + c;
    rc.own = own_col && col_ok && ys >= y_lo && ys < y_hi && rc.eid >= d.own_lo &&
             rc.eid < d.own_hi;
    constexpr uint32_t kFull = (1u << kFusedS) - 1u;
    const bool margin = !(ys >= y_lo - 1 && ys < y_hi);  // source G not needed: filter
    const bool fast = __all_sync(0xffffffffu, rc.m == kFull);
    if (margin) {
        bonds_row<DO_BREAK, true, true, WS>(d, st, rowp, rc, G0, G1, mw, lane, ys, y_lo, y_hi, nb);
    } else if (fast) {
        bonds_row<DO_BREAK, false, false, WS>(d, st, rowp, rc, G0, G1, mw, lane, ys, y_lo, y_hi,
                                              nb);
    } else {
        bonds_row<DO_BREAK, true, false, WS>(d, st, rowp, rc, G0, G1, mw, lane, ys, y_lo, y_hi,
                                             nb);
    }
}

template <bool DO_BREAK>
__global__ void __launch_bounds__(32 * WARPS)
k_strip2d(DevPD d, LatticeDev L, const __grid_constant__ StripStencil st, FusedBufs bf,
          int step, double scale, int write_state, int H) {
    extern __shared__ __align__(16) double2 sm2[];
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    const int nx = L.nx, ny = L.ny, NX = nx + 1, NY = ny + 1;
    const int n_strips = (NX + kColsPerStrip - 1) / kColsPerStrip;
    const int n_segs = (NY + H - 1) / H;
    const int unit = blockIdx.x * WARPS + warp;
    unsigned long long nb = 0;
    if (unit < n_strips * n_segs) {
        const int s = unit % n_strips, g = unit / n_strips;
        double2* ubr = sm2 + warp * (RING * SH + NRING * SH);
        double2* ndr = ubr + RING * SH;
        const int cb = kColsPerStrip * s - kOwnLane0;  // element / node column of lane 0
        const int c = cb + lane;                         // this lane's column
        const int y_lo = H * g, y_hi = min(H * (g + 1), NY);  // owned node rows
        const bool col_ok = c >= 0 && c < nx;
        const bool own_col = lane >= kOwnLane0;
        const double2* rd2 = reinterpret_cast<const double2*>(bf.rd_in);
        auto node_at = [&](int col, int row) {
            return (col >= 0 && col < NX && row >= 0 && row < NY) ? rd2[(size_t)row * NX + col]
                                                                   : make_double2(0.0, 0.0);
        };
        auto make_ubar = [&](int r) {  // ubar row r from node rows r, r+1 in the node ring
            const double2* na = ndr + (r & (NRING - 1)) * SH;
            const double2* nb2 = ndr + ((r + 1) & (NRING - 1)) * SH;
            double2* u = ubr + (r & (RING - 1)) * SH;
            for (int j = lane; j < SH - 1; j += 32) {
                const int ce = cb + j;
                double2 v = make_double2(0.0, 0.0);
                if (ce >= 0 && ce < nx && r >= 0 && r < ny) {
                    const double2 a = na[j], b = na[j + 1], cc = nb2[j + 1], e = nb2[j];
                    v = make_double2(d.Nsh * (((a.x + b.x) + cc.x) + e.x),
                                     d.Nsh * (((a.y + b.y) + cc.y) + e.y));
                }
                u[j] = v;
            }
        };
        auto load_node_row = [&](int r, double2& v0, double2& v1) {
            v0 = node_at(cb + lane, r);
            v1 = lane < SH - 32 ? node_at(cb + 32 + lane, r) : make_double2(0.0, 0.0);
        };
        auto store_node_row = [&](int r, const double2& v0, const double2& v1) {
            double2* n = ndr + (r & (NRING - 1)) * SH;
            n[lane] = v0;
            if (lane < SH - 32) n[32 + lane] = v1;
        };
        auto load_mask = [&](int r) -> uint32_t {
            return (col_ok && r >= 0 && r < ny) ? bf.mask_in[(size_t)r * nx + c] : 0u;
        };
        const double2* P2 = reinterpret_cast<const double2*>(d.P);
        auto node_update = [&](int t, double gp0, double gp1, double gf0, double gf1,
                               const double2& rv, double im, uint8_t fl, bool upd) {
            const double gl0 = __shfl_up_sync(0xffffffffu, gf0, 1);
            const double gl1 = __shfl_up_sync(0xffffffffu, gf1, 1);
            const double gpl0 = __shfl_up_sync(0xffffffffu, gp0, 1);
            const double gpl1 = __shfl_up_sync(0xffffffffu, gp1, 1);
            if (!upd) return;
            const size_t n_id = (size_t)t * NX + c;
            const double k0 = d.Nsh * ((gpl0 + gp0) + (gl0 + gf0));
            const double k1 = d.Nsh * ((gpl1 + gp1) + (gl1 + gf1));
            double2 p = make_double2(0.0, 0.0);
            if (fl & 8) {
                p = P2[n_id];
                p.x *= scale;
                p.y *= scale;
            }
            const double a0 = (fl & 1) ? 0.0 : (p.x - k0) * im;
            const double a1 = (fl & 2) ? 0.0 : (p.y - k1) * im;
            const double2 rdt = rd2[n_id];  // L2-resident: staged for the ubar rows earlier
            double v0 = rv.x + d.c_corr_v * a0, v1 = rv.y + d.c_corr_v * a1;
            const double u0 = rdt.x + d.c_corr_d * a0, u1 = rdt.y + d.c_corr_d * a1;
            if (fl & 1) v0 = d.bcvel[2 * n_id];
            if (fl & 2) v1 = d.bcvel[2 * n_id + 1];
            if (write_state) {
                reinterpret_cast<double2*>(d.a)[n_id] = make_double2(a0, a1);
                reinterpret_cast<double2*>(d.v)[n_id] = make_double2(v0, v1);
                reinterpret_cast<double2*>(d.u)[n_id] = make_double2(u0, u1);
            }
            reinterpret_cast<double2*>(d.rv)[n_id] =
                make_double2(v0 + d.c_pred_v * a0, v1 + d.c_pred_v * a1);
            reinterpret_cast<double2*>(bf.rd_out)[n_id] =
                make_double2(u0 + d.dt * v0 + d.c_pred_d * a0, u1 + d.dt * v1 + d.c_pred_d * a1);
        };

        // Source rows run over [ys0, ys_end] in pairs; window rows ys-2 .. ys+4.
        const int ys0 = y_lo - 4;
        int ys_end = y_hi + 1;
        if ((ys_end - ys0 + 1) & 1) ++ys_end;  // even number of source rows
        // prologue: node rows ys0-2 .. ys0+3 (ring holds 4: keep ys0+2 .. ys0+3 at the end),
        // ubar rows ys0-2 .. ys0+2, masks of rows ys0-2 .. ys0+2
        double2 p0, p1, q0, q1;
        for (int r = ys0 - 2; r <= ys0 + 3; ++r) {
            load_node_row(r, p0, p1);
            store_node_row(r, p0, p1);
            __syncwarp();
            if (r >= ys0 - 1) make_ubar(r - 1);
            __syncwarp();
        }
        load_node_row(ys0 + 4, p0, p1);  // prefetch for the first iteration
        load_node_row(ys0 + 5, q0, q1);
        double G0[7], G1[7];
        uint32_t mw[7];
#pragma unroll
        for (int w = 0; w < 7; ++w) {
            G0[w] = 0.0;
            G1[w] = 0.0;
            mw[w] = w < 5 ? load_mask(ys0 - 2 + w) : 0u;
        }
        double gp0 = 0.0, gp1 = 0.0;  // final G of the row below the next finished one

#pragma unroll 1
        for (int ys = ys0; ys < ys_end; ys += 2) {
            // (1) extend the rings: node rows ys+4, ys+5 (prefetched), ubar rows ys+3, ys+4,
            //     mask rows ys+3, ys+4; prefetch node rows ys+6, ys+7
            store_node_row(ys + 4, p0, p1);
            store_node_row(ys + 5, q0, q1);
            load_node_row(ys + 6, p0, p1);
            load_node_row(ys + 7, q0, q1);
            mw[5] = load_mask(ys + 3);
            mw[6] = load_mask(ys + 4);
            // node-update inputs of the node rows t = ys-2, ys-1 (in flight during the bonds)
            const int t0 = ys - 2;
            const bool upd0 = own_col && c < NX && t0 >= y_lo && t0 < y_hi;
            const bool upd1 = own_col && c < NX && t0 + 1 >= y_lo && t0 + 1 < y_hi;
            double2 rv0 = make_double2(0.0, 0.0), rv1 = rv0;
            double im0 = 0.0, im1 = 0.0;
            uint8_t fl0 = 0, fl1 = 0;
            if (upd0) {
                const size_t n = (size_t)t0 * NX + c;
                rv0 = reinterpret_cast<const double2*>(d.rv)[n];
                im0 = L.inv_mass[n];
                fl0 = L.nflag[n];
            }
            if (upd1) {
                const size_t n = (size_t)(t0 + 1) * NX + c;
                rv1 = reinterpret_cast<const double2*>(d.rv)[n];
                im1 = L.inv_mass[n];
                fl1 = L.nflag[n];
            }
            __syncwarp();
            make_ubar(ys + 3);
            make_ubar(ys + 4);
            __syncwarp();
            const double2* rowp[7];
#pragma unroll
            for (int w = 0; w < 7; ++w) rowp[w] = ubr + ((ys - 2 + w) & (RING - 1)) * SH;

            // (2) bonds of source rows ys (window 2) and ys+1 (window 3)
            source_row<DO_BREAK, 2>(d, st, rowp, G0, G1, mw, lane, c, own_col, col_ok, nx, ny,
                                    ys, y_lo, y_hi, nb);
            source_row<DO_BREAK, 3>(d, st, rowp, G0, G1, mw, lane, c, own_col, col_ok, nx, ny,
                                    ys + 1, y_lo, y_hi, nb);

            // (3) rows t0 = ys-2 and t0+1 are final: node updates, mask write-out
            node_update(t0, gp0, gp1, G0[0], G1[0], rv0, im0, fl0, upd0);
            node_update(t0 + 1, G0[0], G1[0], G0[1], G1[1], rv1, im1, fl1, upd1);
            if (own_col && col_ok && t0 >= y_lo && t0 < y_hi && t0 < ny)
                bf.mask_out[(size_t)t0 * nx + c] = mw[0];
            if (own_col && col_ok && t0 + 1 >= y_lo && t0 + 1 < y_hi && t0 + 1 < ny)
                bf.mask_out[(size_t)(t0 + 1) * nx + c] = mw[1];
            gp0 = G0[1];
            gp1 = G1[1];
            // (4) rotate the windows by two rows
#pragma unroll
            for (int w = 0; w < 5; ++w) {
                G0[w] = G0[w + 2];
                G1[w] = G1[w + 2];
                mw[w] = mw[w + 2];
            }
            G0[5] = G0[6] = 0.0;
            G1[5] = G1[6] = 0.0;
        }
    }
    if (DO_BREAK) {
        __shared__ unsigned long long part[WARPS];
        for (int o = 16; o > 0; o >>= 1) nb += __shfl_down_sync(0xffffffffu, nb, o);
        if (lane == 0) part[warp] = nb;
        __syncthreads();
        if (threadIdx.x == 0) {
            unsigned long long t = 0;
            for (int w = 0; w < WARPS; ++w) t += part[w];
            if (t) atomicAdd(d.broken_count + step, t);
        }
    }
}

void strip2d_configure() {
    for (auto fn : {k_strip2d<true>, k_strip2d<false>}) {
        cudaError_t e =
            cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)kSmem);
        if (e != cudaSuccess)
            throw std::runtime_error(std::string("CUDA: ") + cudaGetErrorString(e));
    }
}

void launch_strip2d_step(const DevPD& d, const LatticeDev& L, const StripStencil& st,
                         const FusedBufs& b, int step, int do_break, double scale,
                         int write_state, int H, cudaStream_t s) {
    const int n_strips = (L.nx + 1 + kColsPerStrip - 1) / kColsPerStrip;
    const int n_segs = (L.ny + 1 + H - 1) / H;
    const int units = n_strips * n_segs;
    const int grid = (units + WARPS - 1) / WARPS;
    if (do_break)
        k_strip2d<true><<<grid, 32 * WARPS, kSmem, s>>>(d, L, st, b, step, scale, write_state, H);
    else
        k_strip2d<false><<<grid, 32 * WARPS, kSmem, s>>>(d, L, st, b, step, scale, write_state, H);
    cudaError_t e = cudaGetLastError();
    if (e != cudaSuccess) throw std::runtime_error(std::string("CUDA: ") + cudaGetErrorString(e));
}

}  // namespace pmts
