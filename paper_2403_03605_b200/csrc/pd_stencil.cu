// Fast-mode lattice-stencil path (sm_100a, FMA allowed).
//
// When the mesh is the generated lattice (mesh.hpp:170-219 numbering) every
// element's family is a subset of one global offset stencil: partner =
// e + (di, dj, dk).  The family then needs no per-bond storage at all -- one
// bit per stencil offset per element ("active" = in the family and intact),
// and per-offset constants (xi, w c(|xi|), |xi|^2) shared by all elements.
// Compared with ELL families this drops the 12 B per directed entry (partner
// id + coefficient) that dominated HBM traffic; what remains per element is
// the centroid displacement, the bit mask and the element force.
//
// Per fine step (3 launches):
//   k_lat_ubar   ubar_e = N sum_a rd(node_a)                 (perifem.hpp:149-157)
//   k_lat_bond   CTA tile of elements + stencil apron of ubar staged in shared
//                memory; per active offset: eta = ubar_p - ubar_e,
//                G_e -= w c (xi.eta) xi, squared break test (one-way bits)
//   k_lat_node   K u at the nodes from the <= 2^d incident G_e, explicit
//                Newmark update (newmark.hpp:125-157) + next predictor
//                (newmark.hpp:61-69); u, v, a written on the batch's last step
#include <stdexcept>
#include <string>

#include "pd_stencil.cuh"

namespace pmts {

#define PMTS_CUDA_S(x)                                                                   \
    do {                                                                                 \
        cudaError_t err_ = (x);                                                          \
        if (err_ != cudaSuccess)                                                         \
            throw std::runtime_error(std::string("CUDA: ") + cudaGetErrorString(err_)); \
    } while (0)

template <int DIM>
__global__ void __launch_bounds__(256) k_lat_ubar(DevPD d, LatticeDev L) {
    const int e = blockIdx.x * blockDim.x + threadIdx.x;
    if (e >= d.E) return;
    const int i = e % L.nx, r = e / L.nx;
    const int j = r % L.ny, k = r / L.ny;
    const int NX = L.nx + 1, NY = L.ny + 1;
    double s[DIM];
    for (int c = 0; c < DIM; ++c) s[c] = 0.0;
    const int n00 = (k * NY + j) * NX + i;
    const int nodes2[4] = {n00, n00 + 1, n00 + NX + 1, n00 + NX};
#pragma unroll
    for (int a = 0; a < 4; ++a)
#pragma unroll
        for (int c = 0; c < DIM; ++c) s[c] += d.rd[(size_t)nodes2[a] * DIM + c];
    if constexpr (DIM == 3) {
        const int up = NX * NY;
#pragma unroll
        for (int a = 0; a < 4; ++a)
#pragma unroll
            for (int c = 0; c < DIM; ++c) s[c] += d.rd[(size_t)(nodes2[a] + up) * DIM + c];
    }
#pragma unroll
    for (int c = 0; c < DIM; ++c) d.ubar[(size_t)e * DIM + c] = d.Nsh * s[c];
}

template <int DIM, int TX, int TY, int TZ>
__global__ void __launch_bounds__(TX* TY* TZ)
k_lat_bond(DevPD d, LatticeDev L, int step, int do_break) {
    extern __shared__ double smem[];
    constexpr int NT = TX * TY * TZ;
    const int R = L.R;
    const int AX = TX + 2 * R, AY = TY + 2 * R, AZ = DIM == 3 ? TZ + 2 * R : 1;
    const int napron = AX * AY * AZ;
    // shared layout: ubar apron tile (SoA per component), then the stencil table
    double* ub = smem;                                  // DIM * napron
    double* tab = smem + (size_t)DIM * napron;          // S * 6: xi[3], f, x2, thr
    int* toff = reinterpret_cast<int*>(tab + 6 * L.S);  // S * 2: tile offset, id delta
    const int tid = threadIdx.x;
    for (int q = tid; q < L.S; q += NT) {
        for (int c = 0; c < 6; ++c) tab[6 * q + c] = L.table[6 * q + c];
        toff[2 * q] = (L.dk[q] * AY + L.dj[q]) * AX + L.di[q];
        toff[2 * q + 1] = L.delta_id[q];
    }
    const int i0 = blockIdx.x * TX, j0 = blockIdx.y * TY, k0 = blockIdx.z * TZ;
    for (int q = tid; q < napron; q += NT) {
        const int ax = q % AX, r = q / AX;
        const int ay = r % AY, az = r / AY;
        const int gi = i0 + ax - R, gj = j0 + ay - R, gk = DIM == 3 ? k0 + az - R : 0;
        const bool in = gi >= 0 && gj >= 0 && gk >= 0 && gi < L.nx && gj < L.ny && gk < L.nz;
        const size_t ge = ((size_t)gk * L.ny + gj) * L.nx + gi;
#pragma unroll
        for (int c = 0; c < DIM; ++c) ub[c * napron + q] = in ? d.ubar[ge * DIM + c] : 0.0;
    }
    __syncthreads();
    const int tx = tid % TX, ty = (tid / TX) % TY, tz = tid / (TX * TY);
    const int gi = i0 + tx, gj = j0 + ty, gk = k0 + tz;
    unsigned long long nb = 0;
    if (gi < L.nx && gj < L.ny && gk < L.nz) {
        const int e = (gk * L.ny + gj) * L.nx + gi;
        const int q0 = ((DIM == 3 ? tz + R : 0) * AY + ty + R) * AX + tx + R;
        double ue[DIM], G[DIM];
#pragma unroll
        for (int c = 0; c < DIM; ++c) {
            ue[c] = ub[c * napron + q0];
            G[c] = 0.0;
        }
        for (int w = 0; w < L.W; ++w) {
            uint32_t m = d.mask[(size_t)w * d.E + e];
            const uint32_t m0 = m;
            uint32_t live = m;
            while (live) {
                const int b = __ffs(live) - 1;
                live &= live - 1;
                const int s = 32 * w + b;
                const double* t = tab + 6 * s;
                const int q = q0 + toff[2 * s];
                double dot = 0.0, l2 = 0.0;
                double xi[DIM];
#pragma unroll
                for (int c = 0; c < DIM; ++c) {
                    xi[c] = t[c];
                    const double eta = ub[c * napron + q] - ue[c];
                    dot = fma(xi[c], eta, dot);
                    const double y = xi[c] + eta;
                    l2 = fma(y, y, l2);
                }
                const double fd = t[3] * dot;
#pragma unroll
                for (int c = 0; c < DIM; ++c) G[c] = fma(-fd, xi[c], G[c]);
                if (do_break) {
                    double thr = t[5];
                    if (d.spread != 0.0) {
                        const int p = e + toff[2 * s + 1];
                        const double s1 = 1.0 + bond_s_crit(d.s_crit, d.spread, d.seed,
                                                            e < p ? e : p, e < p ? p : e);
                        thr = s1 * s1 * t[4];
                    }
                    if (l2 >= thr) {
                        m &= ~(1u << b);
                        if (toff[2 * s + 1] > 0) ++nb;
                    }
                }
            }
            if (m != m0) d.mask[(size_t)w * d.E + e] = m;
        }
#pragma unroll
        for (int c = 0; c < DIM; ++c) d.G[(size_t)e * DIM + c] = G[c];
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

template <int DIM>
__global__ void __launch_bounds__(256)
k_lat_node(DevPD d, LatticeDev L, double scale, int write_state) {
    const int n = blockIdx.x * blockDim.x + threadIdx.x;
    if (n >= d.N) return;
    const int NX = L.nx + 1, NY = L.ny + 1;
    const int i = n % NX, r = n / NX;
    const int j = r % NY, k = r / NY;
    double Ku[DIM];
#pragma unroll
    for (int c = 0; c < DIM; ++c) Ku[c] = 0.0;
    // incident elements (i-1|i, j-1|j, k-1|k), ascending id
#pragma unroll
    for (int dz = (DIM == 3 ? -1 : 0); dz <= 0; ++dz)
#pragma unroll
        for (int dy = -1; dy <= 0; ++dy)
#pragma unroll
            for (int dx = -1; dx <= 0; ++dx) {
                const int ei = i + dx, ej = j + dy, ek = k + dz;
                if (ei < 0 || ej < 0 || ek < 0 || ei >= L.nx || ej >= L.ny || ek >= L.nz) continue;
                const size_t e = ((size_t)ek * L.ny + ej) * L.nx + ei;
#pragma unroll
                for (int c = 0; c < DIM; ++c) Ku[c] += d.G[e * DIM + c];
            }
#pragma unroll
    for (int c = 0; c < DIM; ++c) {
        const size_t q = (size_t)n * DIM + c;
        const bool bc = d.bcflag[q] != 0;
        const double acc = bc ? 0.0 : (d.P[q] * scale - d.Nsh * Ku[c]) / d.M[q];
        double vel = d.rv[q] + d.c_corr_v * acc;
        const double dis = d.rd[q] + d.c_corr_d * acc;
        if (bc) vel = d.bcvel[q];
        if (write_state) {
            d.a[q] = acc;
            d.v[q] = vel;
            d.u[q] = dis;
        }
        d.rv[q] = vel + d.c_pred_v * acc;
        d.rd[q] = dis + d.dt * vel + d.c_pred_d * acc;
    }
}

size_t lattice_smem_bytes(int dim, int R, int S) {
    const int TX = dim == 2 ? 32 : 16, TY = dim == 2 ? 8 : 4, TZ = dim == 2 ? 1 : 4;
    const size_t napron =
        (size_t)(TX + 2 * R) * (TY + 2 * R) * (dim == 3 ? TZ + 2 * R : 1);
    return sizeof(double) * (dim * napron + 6 * (size_t)S) + sizeof(int) * 2 * (size_t)S;
}

void launch_lattice_step(const DevPD& d, const LatticeDev& L, int step, int do_break,
                         double scale, int write_state, bool time_bond, cudaEvent_t* ev,
                         cudaStream_t s) {
    const int eb = (d.E + 255) / 256;
    const int nb = (d.N + 255) / 256;
    const size_t smem = lattice_smem_bytes(d.dim, L.R, L.S);
    if (d.dim == 2) {
        k_lat_ubar<2><<<eb, 256, 0, s>>>(d, L);
        if (time_bond) PMTS_CUDA_S(cudaEventRecord(ev[0], s));
        dim3 grid((L.nx + 31) / 32, (L.ny + 7) / 8, 1);
        k_lat_bond<2, 32, 8, 1><<<grid, 256, smem, s>>>(d, L, step, do_break);
        if (time_bond) PMTS_CUDA_S(cudaEventRecord(ev[1], s));
        k_lat_node<2><<<nb, 256, 0, s>>>(d, L, scale, write_state);
    } else {
        k_lat_ubar<3><<<eb, 256, 0, s>>>(d, L);
        if (time_bond) PMTS_CUDA_S(cudaEventRecord(ev[0], s));
        dim3 grid((L.nx + 15) / 16, (L.ny + 3) / 4, (L.nz + 3) / 4);
        k_lat_bond<3, 16, 4, 4><<<grid, 256, smem, s>>>(d, L, step, do_break);
        if (time_bond) PMTS_CUDA_S(cudaEventRecord(ev[1], s));
        k_lat_node<3><<<nb, 256, 0, s>>>(d, L, scale, write_state);
    }
    PMTS_CUDA_S(cudaGetLastError());
}

void lattice_configure(int dim, int R, int S) {
    const int bytes = (int)lattice_smem_bytes(dim, R, S);
    if (dim == 2)
        PMTS_CUDA_S(cudaFuncSetAttribute(k_lat_bond<2, 32, 8, 1>,
                                         cudaFuncAttributeMaxDynamicSharedMemorySize, bytes));
    else
        PMTS_CUDA_S(cudaFuncSetAttribute(k_lat_bond<3, 16, 4, 4>,
                                         cudaFuncAttributeMaxDynamicSharedMemorySize, bytes));
}

}  // namespace pmts
