// Fused one-kernel fine step for 2D lattices with the 28-offset stencil
// (delta in [3, sqrt(10)) dx -- BASELINE's 3.015 dx), fast mode.
//
// One CTA owns a 31 x 15 block of elements and the nodes at their lower-left
// corners.  It stages the predictor displacement of a node apron in shared
// memory, forms the centroid displacements of the element apron, evaluates the
// bond forces of the 32 x 16 elements whose G the owned nodes need (its own
// block plus one ring of neighbours, recomputed -- ~10% extra arithmetic
// instead of a grid-wide dependency), and finishes with the Verlet update of
// the owned nodes.  Nothing per-element ever goes to HBM except one mask word;
// the per-offset constants live in the kernel's parameter space (constant
// bank operands of the fp64 instructions).  Displacement and mask are
// ping-ponged across steps so neighbouring CTAs never observe a half-updated
// step.  Reference semantics as in pd_stencil.cu.
#include <stdexcept>
#include <string>

#include "pd_stencil.cuh"

namespace pmts {

namespace {

constexpr int TX = kFusedTX, TY = kFusedTY, R = kFusedR;
constexpr int GX = TX + 1, GY = TY + 1;       // force region (elements)
constexpr int AX = GX + 2 * R, AY = GY + 2 * R;  // ubar apron (elements)
constexpr int BX = AX + 1, BY = AY + 1;          // node apron
constexpr int NT = 256;
static_assert(GX * GY == 2 * NT, "force region = 2 elements per thread");
static_assert(AX == kFusedAX, "apron width");

constexpr size_t kSmem = sizeof(double2) * (BX * BY + AX * AY + GX * GY);

}  // namespace

__global__ void __launch_bounds__(NT, 4)
k_fused2d(DevPD d, LatticeDev L, const __grid_constant__ Stencil2D st, FusedBufs bf, int step,
          int do_break, double scale, int write_state) {
    extern __shared__ __align__(16) double2 sm2[];
    double2* nt = sm2;                 // BX * BY node apron
    double2* ub = nt + BX * BY;        // AX * AY element apron
    double2* gt = ub + AX * AY;        // GX * GY element forces
    const int tid = threadIdx.x;
    const int nx = L.nx, ny = L.ny, NX = nx + 1, NY = ny + 1;
    const int i0 = blockIdx.x * TX, j0 = blockIdx.y * TY;
    // node apron: nodes [i0-1-R, i0-1-R+BX) x [j0-1-R, ...)
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
    __syncthreads();

    unsigned long long nb = 0;
#pragma unroll 1
    for (int r = 0; r < 2; ++r) {
        const int g = tid + r * NT;
        const int gx = g % GX, gy = g / GX;
        const int ei = i0 - 1 + gx, ej = j0 - 1 + gy;
        double G0 = 0.0, G1 = 0.0;
        if (ei >= 0 && ej >= 0 && ei < nx && ej < ny) {
            const int e = ej * nx + ei;
            const bool own = gx >= 1 && gy >= 1;
            const int q0 = (gy + R) * AX + gx + R;
            const double2 ue = ub[q0];
            const uint32_t m0 = bf.mask_in[e];
            uint32_t m = m0;
#pragma unroll
            for (int k = 0; k < kFusedS; ++k) {
                if (m0 & (1u << k)) {
                    const double2 up = ub[q0 + st.aoff[k]];
                    const double e0 = up.x - ue.x, e1 = up.y - ue.y;
                    const double dot = fma(st.xi1[k], e1, st.xi0[k] * e0);
                    const double fd = st.f[k] * dot;
                    G0 = fma(-fd, st.xi0[k], G0);
                    G1 = fma(-fd, st.xi1[k], G1);
                    if (do_break) {
                        const double lhs = fma(2.0, dot, fma(e1, e1, e0 * e0));
                        if (lhs >= st.clo[k]) {
                            double thr = st.cthr[k];
                            if (d.spread != 0.0) {
                                const int p = e + st.did[k];
                                const double sb = bond_s_crit(d.s_crit, d.spread, d.seed,
                                                              e < p ? e : p, e < p ? p : e);
                                thr = fma(sb, sb, 2.0 * sb) * st.x2[k];
                            }
                            if (lhs >= thr) {
                                m &= ~(1u << k);
                                if (own && st.did[k] > 0) ++nb;
                            }
                        }
                    }
                }
            }
            if (own) bf.mask_out[e] = m;
        }
        gt[g] = make_double2(G0, G1);
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
        const double2 c = gt[(ly + 1) * GX + lx], e = gt[(ly + 1) * GX + lx + 1];
        const double k0 = d.Nsh * ((a.x + b.x) + (c.x + e.x));
        const double k1 = d.Nsh * ((a.y + b.y) + (c.y + e.y));
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

    if (do_break) {
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
    cudaError_t e = cudaFuncSetAttribute(k_fused2d, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                         (int)kSmem);
    if (e != cudaSuccess) throw std::runtime_error(std::string("CUDA: ") + cudaGetErrorString(e));
}

void launch_fused2d_step(const DevPD& d, const LatticeDev& L, const Stencil2D& st,
                         const FusedBufs& b, int step, int do_break, double scale,
                         int write_state, cudaStream_t s) {
    dim3 grid((L.nx + TX - 1) / TX, (L.ny + TY - 1) / TY, 1);
    k_fused2d<<<grid, NT, kSmem, s>>>(d, L, st, b, step, do_break, scale, write_state);
    cudaError_t e = cudaGetLastError();
    if (e != cudaSuccess) throw std::runtime_error(std::string("CUDA: ") + cudaGetErrorString(e));
}

}  // namespace pmts
