// Fused one-kernel fine step for 2D lattices with the 28-offset stencil
// (delta in [3, sqrt(10)) dx -- BASELINE's 3.015 dx), fast mode.
//
// One CTA owns a 31 x 15 block of elements and the nodes at their lower-left
// corners.  It stages the predictor displacement of a node apron in shared
// memory, forms the centroid displacements of the element apron, evaluates the
// bond forces of the 32 x 16 elements whose G the owned nodes need (its own
// block plus one ring of neighbours, recomputed -- ~10% extra arithmetic
// instead of a grid-wide dependency), and finishes with the Verlet update of
// the owned nodes.  Nothing per-element goes to HBM except one mask word.
//
// Work split: 4 warps; lane = column of the 32-wide force region, warp w owns
// rows 4w..4w+3, so every per-offset constant (kernel parameter space) is
// fetched once per thread and used for 4 elements, and each shared-memory
// load of a warp touches 32 consecutive apron cells.  Displacement and mask
// are ping-ponged across steps so neighbouring CTAs never observe a
// half-updated step.  Reference semantics as in pd_stencil.cu.
#include <stdexcept>
#include <string>

#include "pd_stencil.cuh"

namespace pmts {

namespace {

constexpr int TX = kFusedTX, TY = kFusedTY, R = kFusedR;
constexpr int GX = TX + 1, GY = TY + 1;          // force region (elements)
constexpr int AX = GX + 2 * R, AY = GY + 2 * R;  // ubar apron (elements)
constexpr int BX = AX + 1, BY = AY + 1;          // node apron
constexpr int NT = 128;
constexpr int EPT = GY / (NT / 32);              // elements per thread (rows per warp)
static_assert(GX == 32 && EPT * (NT / 32) == GY, "lane = column, warp = EPT rows");
static_assert(AX == kFusedAX, "apron width");

constexpr size_t kSmem = sizeof(double2) * (BX * BY + AX * AY + GX * GY);

}  // namespace

template <bool DO_BREAK>
__global__ void __launch_bounds__(NT, 6)
k_fused2d(DevPD d, LatticeDev L, const __grid_constant__ Stencil2D st, FusedBufs bf, int step,
          double scale, int write_state) {
    extern __shared__ __align__(16) double2 sm2[];
    double2* nt = sm2;                 // BX * BY node apron
    double2* ub = nt + BX * BY;        // AX * AY element apron
    double2* gt = ub + AX * AY;        // GX * GY element forces
    const int tid = threadIdx.x;
    const int nx = L.nx, ny = L.ny, NX = nx + 1, NY = ny + 1;
    const int i0 = blockIdx.x * TX, j0 = blockIdx.y * TY;
    const double2* rd2 = reinterpret_cast<const double2*>(bf.rd_in);
    for (int q = tid; q < BX * BY; q += NT) {
        const int bx = q % BX, by = q / BX;
        const int gi = i0 - 1 - R + bx, gj = j0 - 1 - R + by;
        double2 v = make_double2(0.0, 0.0);
        if (gi >= 0 && gj >= 0 && gi < NX && gj < NY) v = rd2[(size_t)gj * NX + gi];
        nt[q] = v;
    }
    __syncthreads();
    for (int q = tid; q < AX * AY; q += NT) {
        const int ax = q % AX, ay = q / AX;
        const double2 a = nt[ay * BX + ax], b = nt[ay * BX + ax + 1];
        const double2 c = nt[(ay + 1) * BX + ax + 1], e = nt[(ay + 1) * BX + ax];
        ub[q] = make_double2(d.Nsh * (((a.x + b.x) + c.x) + e.x),
                             d.Nsh * (((a.y + b.y) + c.y) + e.y));
    }

    // per-thread elements: column gx = lane, rows gy = EPT*warp + r
    const int gx = tid & 31, gy0 = (tid >> 5) * EPT;
    const int ei = i0 - 1 + gx;
    int e[EPT];
    uint32_t m0[EPT], m[EPT];
    double2 ue[EPT];
    double G0[EPT], G1[EPT];
    const int q0 = (gy0 + R) * AX + gx + R;
#pragma unroll
    for (int r = 0; r < EPT; ++r) {
        const int ej = j0 - 1 + gy0 + r;
        const bool in = ei >= 0 && ej >= 0 && ei < nx && ej < ny;
        e[r] = in ? ej * nx + ei : -1;
        m0[r] = in ? bf.mask_in[e[r]] : 0u;
        m[r] = m0[r];
        G0[r] = 0.0;
        G1[r] = 0.0;
    }
    __syncthreads();
#pragma unroll
    for (int r = 0; r < EPT; ++r) ue[r] = ub[q0 + r * AX];

    // pass 1, branch-free: forces of all active bonds, and one flag per element
    // if any active bond reaches the smallest threshold of its offset.  Warps
    // whose elements all carry the full intact stencil (the interior, nearly
    // always) skip the per-bond activity selects.
    bool anyc[EPT];
#pragma unroll
    for (int r = 0; r < EPT; ++r) anyc[r] = false;
    constexpr uint32_t kFull = (1u << kFusedS) - 1u;
    bool full = true;
#pragma unroll
    for (int r = 0; r < EPT; ++r) full = full && m0[r] == kFull;
    if (__all_sync(0xffffffffu, full)) {
#pragma unroll
        for (int k = 0; k < kFusedS; ++k) {
            const double xi0 = st.xi0[k], xi1 = st.xi1[k];
            const double fx0 = st.fx0[k], fx1 = st.fx1[k], clo = st.clo[k];
            const double2* up_base = ub + q0 + st.aoff[k];
#pragma unroll
            for (int r = 0; r < EPT; ++r) {
                const double2 up = up_base[r * AX];
                const double e0 = up.x - ue[r].x, e1 = up.y - ue[r].y;
                const double dot = fma(xi1, e1, xi0 * e0);
                G0[r] = fma(-dot, fx0, G0[r]);
                G1[r] = fma(-dot, fx1, G1[r]);
                if (DO_BREAK) anyc[r] |= fma(2.0, dot, fma(e1, e1, e0 * e0)) >= clo;
            }
        }
    } else {
#pragma unroll
        for (int k = 0; k < kFusedS; ++k) {
            const double xi0 = st.xi0[k], xi1 = st.xi1[k];
            const double fx0 = st.fx0[k], fx1 = st.fx1[k], clo = st.clo[k];
            const double2* up_base = ub + q0 + st.aoff[k];
#pragma unroll
            for (int r = 0; r < EPT; ++r) {
                const bool act = (m0[r] >> k) & 1u;
                const double2 up = up_base[r * AX];
                const double e0 = up.x - ue[r].x, e1 = up.y - ue[r].y;
                const double dot = fma(xi1, e1, xi0 * e0);
                const double dm = act ? dot : 0.0;
                G0[r] = fma(-dm, fx0, G0[r]);
                G1[r] = fma(-dm, fx1, G1[r]);
                if (DO_BREAK) anyc[r] |= act && fma(2.0, dot, fma(e1, e1, e0 * e0)) >= clo;
            }
        }
    }
    // pass 2 (rare): exact per-bond thresholds for the flagged elements
    unsigned long long nb = 0;
    if (DO_BREAK) {
#pragma unroll
        for (int r = 0; r < EPT; ++r) {
            uint32_t c = anyc[r] ? m0[r] : 0u;
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
                    const int lo = e[r] < p ? e[r] : p, hi = e[r] < p ? p : e[r];
                    const double sb =
                        bond_s_crit(d.s_crit, d.spread, d.seed, lo + d.goff, hi + d.goff);
                    thr = fma(sb, sb, 2.0 * sb) * st.x2[k];
                }
                if (lhs >= thr) {
                    m[r] &= ~(1u << k);
                    if (gx >= 1 && gy0 + r >= 1 && st.did[k] > 0 && e[r] >= d.own_lo &&
                        e[r] < d.own_hi)
                        ++nb;
                }
            }
        }
    }
#pragma unroll
    for (int r = 0; r < EPT; ++r) {
        if (e[r] >= 0 && gx >= 1 && gy0 + r >= 1) bf.mask_out[e[r]] = m[r];
        gt[(gy0 + r) * GX + gx] = make_double2(G0[r], G1[r]);
    }
    __syncthreads();

    // Verlet update of the owned nodes (the last block row/column also owns the
    // domain's far node line)
    const int ox = (blockIdx.x == gridDim.x - 1) ? NX - i0 : TX;
    const int oy = (blockIdx.y == gridDim.y - 1) ? NY - j0 : TY;
    double2* rdo = reinterpret_cast<double2*>(bf.rd_out);
    double2* rv2 = reinterpret_cast<double2*>(d.rv);
    const double2* P2 = reinterpret_cast<const double2*>(d.P);
    for (int q = tid; q < ox * oy; q += NT) {
        const int lx = q % ox, ly = q / ox;
        const int ni = i0 + lx, nj = j0 + ly;
        const size_t n = (size_t)nj * NX + ni;
        // incident elements (ni-1|ni, nj-1|nj) sit at force-region (lx|lx+1, ly|ly+1)
        const double2 a = gt[ly * GX + lx], b = gt[ly * GX + lx + 1];
        const double2 c = gt[(ly + 1) * GX + lx], f = gt[(ly + 1) * GX + lx + 1];
        const double k0 = d.Nsh * ((a.x + b.x) + (c.x + f.x));
        const double k1 = d.Nsh * ((a.y + b.y) + (c.y + f.y));
        const uint8_t fl = L.nflag[n];
        const double im = L.inv_mass[n];
        double2 p = make_double2(0.0, 0.0);
        if (fl & 8) {
            p = P2[n];
            p.x *= scale;
            p.y *= scale;
        }
        const double a0 = (fl & 1) ? 0.0 : (p.x - k0) * im;
        const double a1 = (fl & 2) ? 0.0 : (p.y - k1) * im;
        const double2 rv = rv2[n];
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
        __shared__ unsigned long long part[NT / 32];
        for (int o = 16; o > 0; o >>= 1) nb += __shfl_down_sync(0xffffffffu, nb, o);
        if ((tid & 31) == 0) part[tid >> 5] = nb;
        __syncthreads();
        if (tid == 0) {
            unsigned long long t = 0;
            for (int w = 0; w < NT / 32; ++w) t += part[w];
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
