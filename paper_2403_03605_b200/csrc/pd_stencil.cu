// Fast-mode lattice-stencil path (sm_100a, FMA allowed).
//
// When the mesh is the generated lattice (mesh.hpp:170-219 numbering) every
// element's family is a subset of one global offset stencil: partner =
// e + (di, dj, dk).  The family then needs no per-bond storage at all -- one
// bit per stencil offset per element ("active" = in the family and intact),
// and per-offset constants (xi, w c(|xi|), thresholds) shared by all
// elements.  Compared with ELL families this drops the 12 B per directed
// entry (partner id + coefficient) that dominated HBM traffic.
//
// Per fine step:
//   2D: k_lat_bond<2> (ubar from a shared-memory node tile, fused) + k_lat_node
//   3D: k_lat_ubar<3> + k_lat_bond<3> + k_lat_node
//   ubar_e = N sum_a rd(node_a)                                  perifem.hpp:149-157
//   per active offset: eta = ubar_p - ubar_e;  G_e -= w c (xi.eta) xi;
//     break iff 2 xi.eta + |eta|^2 >= (2 s + s^2) |xi|^2   (== |xi+eta|^2 >=
//     ((1+s)|xi|)^2, the squared form of perifem.hpp:158-165, 183)
//   node: K u = N sum G_e (<= 2^d incident elements); explicit Newmark update
//     (newmark.hpp:125-157) + next predictor (newmark.hpp:61-69); u, v, a are
//     materialised on the last step of a batch only.
// The per-bond s0 factor (counter hash) is evaluated only for the rare bonds
// whose stretch already exceeds the smallest possible threshold.
#include <stdexcept>
#include <string>

#include <cub/cub.cuh>

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

// Stencil table row (8 doubles, 16 B aligned pairs):
//   0 xi0  1 xi1  2 f = w c(|xi|)  3 cthr = (2 s + s^2)|xi|^2  4 xi2
//   5 cthr_lo (smallest threshold under the per-bond factor)  6 |xi|^2  7 pad
constexpr int kRow = 8;

template <int DIM, int TX, int TY, int TZ, int EPT>
struct BondTile {
    static constexpr int NT = TX * TY * TZ;          // threads
    static constexpr int EY = DIM == 2 ? TY * EPT : TY;  // tile extent (elements)
    static constexpr int EZ = DIM == 2 ? 1 : TZ * EPT;
};

// shared bytes for a tile (host + device agree)
template <int DIM, int TX, int TY, int TZ, int EPT>
__host__ __device__ inline size_t bond_smem(int R, int S) {
    using T = BondTile<DIM, TX, TY, TZ, EPT>;
    const size_t ax = TX + 2 * R, ay = T::EY + 2 * R, az = DIM == 3 ? T::EZ + 2 * R : 1;
    size_t b = sizeof(double) * DIM * ax * ay * az;                 // ubar apron
    if (DIM == 2) b += sizeof(double) * 2 * (ax + 1) * (ay + 1);     // node tile (fused ubar)
    b += sizeof(double) * kRow * S + sizeof(int2) * S;              // stencil table
    return b;
}

template <int DIM, int TX, int TY, int TZ, int EPT>
__global__ void __launch_bounds__(TX* TY* TZ)
k_lat_bond(DevPD d, LatticeDev L, int step, int do_break) {
    using T = BondTile<DIM, TX, TY, TZ, EPT>;
    extern __shared__ __align__(16) double smem[];
    const int R = L.R;
    const int AX = TX + 2 * R, AY = T::EY + 2 * R, AZ = DIM == 3 ? T::EZ + 2 * R : 1;
    const int napron = AX * AY * AZ;
    double* ub = smem;  // 2D: double2 per apron cell; 3D: SoA per component
    double* nodes = smem + DIM * napron;
    double* tab = nodes + (DIM == 2 ? 2 * (AX + 1) * (AY + 1) : 0);
    int2* toff = reinterpret_cast<int2*>(tab + kRow * L.S);
    const int tid = threadIdx.x;
    const int i0 = blockIdx.x * TX, j0 = blockIdx.y * T::EY, k0 = blockIdx.z * T::EZ;
    for (int q = tid; q < L.S; q += T::NT) {
#pragma unroll
        for (int c = 0; c < kRow; ++c) tab[kRow * q + c] = L.table[kRow * q + c];
        toff[q] = make_int2((L.dk[q] * AY + L.dj[q]) * AX + L.di[q], L.delta_id[q]);
    }
    if constexpr (DIM == 2) {
        // node tile (AX+1) x (AY+1), then ubar of every apron element from it
        const int NX = L.nx + 1, NY = L.ny + 1, BX = AX + 1, BY = AY + 1;
        const double2* rd2 = reinterpret_cast<const double2*>(d.rd);
        double2* nt = reinterpret_cast<double2*>(nodes);
        for (int q = tid; q < BX * BY; q += T::NT) {
            const int bx = q % BX, by = q / BX;
            const int gi = i0 - R + bx, gj = j0 - R + by;
            double2 v = make_double2(0.0, 0.0);
            if (gi >= 0 && gj >= 0 && gi < NX && gj < NY) v = rd2[(size_t)gj * NX + gi];
            nt[q] = v;
        }
        __syncthreads();
        double2* u2 = reinterpret_cast<double2*>(ub);
        for (int q = tid; q < napron; q += T::NT) {
            const int ax = q % AX, ay = q / AX;
            const double2 a = nt[ay * BX + ax], b = nt[ay * BX + ax + 1];
            const double2 c = nt[(ay + 1) * BX + ax + 1], e = nt[(ay + 1) * BX + ax];
            u2[q] = make_double2(d.Nsh * (((a.x + b.x) + c.x) + e.x),
                                 d.Nsh * (((a.y + b.y) + c.y) + e.y));
        }
    } else {
        for (int q = tid; q < napron; q += T::NT) {
            const int ax = q % AX, r = q / AX;
            const int ay = r % AY, az = r / AY;
            const int gi = i0 + ax - R, gj = j0 + ay - R, gk = k0 + az - R;
            const bool in = gi >= 0 && gj >= 0 && gk >= 0 && gi < L.nx && gj < L.ny && gk < L.nz;
            const size_t ge = ((size_t)gk * L.ny + gj) * L.nx + gi;
#pragma unroll
            for (int c = 0; c < DIM; ++c) ub[c * napron + q] = in ? d.ubar[ge * DIM + c] : 0.0;
        }
    }
    __syncthreads();

    const int tx = tid % TX, ty = (tid / TX) % TY, tz = tid / (TX * TY);
    unsigned long long nb = 0;
#pragma unroll
    for (int r = 0; r < EPT; ++r) {
        const int ly = DIM == 2 ? ty + r * TY : ty;
        const int lz = DIM == 2 ? 0 : tz + r * TZ;
        const int gi = i0 + tx, gj = j0 + ly, gk = k0 + lz;
        if (gi >= L.nx || gj >= L.ny || gk >= L.nz) continue;
        const int e = (gk * L.ny + gj) * L.nx + gi;
        const int q0 = ((DIM == 3 ? lz + R : 0) * AY + ly + R) * AX + tx + R;
        double ue[DIM], G[DIM];
        if constexpr (DIM == 2) {
            const double2 v = reinterpret_cast<const double2*>(ub)[q0];
            ue[0] = v.x;
            ue[1] = v.y;
        } else {
#pragma unroll
            for (int c = 0; c < DIM; ++c) ue[c] = ub[c * napron + q0];
        }
#pragma unroll
        for (int c = 0; c < DIM; ++c) G[c] = 0.0;
        for (int w = 0; w < L.W; ++w) {
            const uint32_t m0 = d.mask[(size_t)w * d.E + e];
            uint32_t m = m0, live = m0;
            while (live) {
                const int b = __ffs(live) - 1;
                live &= live - 1;
                const int s = 32 * w + b;
                const double* t = tab + kRow * s;
                const int2 of = toff[s];
                double xi[DIM], eta[DIM];
                if constexpr (DIM == 2) {
                    const double2 x01 = *reinterpret_cast<const double2*>(t);
                    xi[0] = x01.x;
                    xi[1] = x01.y;
                    const double2 up = reinterpret_cast<const double2*>(ub)[q0 + of.x];
                    eta[0] = up.x - ue[0];
                    eta[1] = up.y - ue[1];
                } else {
#pragma unroll
                    for (int c = 0; c < DIM; ++c) {
                        xi[c] = t[c == 2 ? 4 : c];
                        eta[c] = ub[c * napron + q0 + of.x] - ue[c];
                    }
                }
                double dot = xi[0] * eta[0], e2 = eta[0] * eta[0];
#pragma unroll
                for (int c = 1; c < DIM; ++c) {
                    dot = fma(xi[c], eta[c], dot);
                    e2 = fma(eta[c], eta[c], e2);
                }
                const double2 fc = *reinterpret_cast<const double2*>(t + 2);  // f, cthr
                const double fd = fc.x * dot;
#pragma unroll
                for (int c = 0; c < DIM; ++c) G[c] = fma(-fd, xi[c], G[c]);
                if (do_break) {
                    const double lhs = fma(2.0, dot, e2);
                    if (lhs >= t[5]) {  // >= the smallest threshold any bond can have
                        double thr = fc.y;  // (2 s + s^2) |xi|^2 with the scalar s_crit
                        if (d.spread != 0.0) {
                            const int p = e + of.y;
                            const double sb = bond_s_crit(d.s_crit, d.spread, d.seed,
                                                          global_elem(d, e < p ? e : p),
                                                          global_elem(d, e < p ? p : e));
                            thr = fma(sb, sb, 2.0 * sb) * t[6];
                        }
                        if (lhs >= thr) {
                            m &= ~(1u << b);
                            if (of.y > 0 && owns_elem(d, e)) ++nb;
                        }
                    }
                }
            }
            if (m != m0) d.mask[(size_t)w * d.E + e] = m;
        }
#pragma unroll
        for (int c = 0; c < DIM; ++c) d.G[(size_t)e * DIM + c] = G[c];
    }
    if (do_break) {
        __shared__ unsigned long long part[T::NT / 32];
        for (int o = 16; o > 0; o >>= 1) nb += __shfl_down_sync(0xffffffffu, nb, o);
        if ((tid & 31) == 0) part[tid >> 5] = nb;
        __syncthreads();
        if (tid == 0) {
            unsigned long long t = 0;
            for (int w = 0; w < T::NT / 32; ++w) t += part[w];
            if (t) atomicAdd(d.broken_count + step, t);
        }
    }
}

template <int DIM>
__global__ void __launch_bounds__(256)
k_lat_node(DevPD d, LatticeDev L, double scale, int write_state) {
    // thread t -> node (i, j, k) of the updated rows j in [jn0, jn1)
    const int t = blockIdx.x * blockDim.x + threadIdx.x;
    const int NX = L.nx + 1, NY = L.ny + 1, NR = L.jn1 - L.jn0;
    const int i = t % NX, r = t / NX;
    const int j = L.jn0 + r % NR, k = r / NR;
    if (k >= (DIM == 3 ? L.nz + 1 : 1)) return;
    const int n = (k * NY + j) * NX + i;
    double Ku[DIM];
#pragma unroll
    for (int c = 0; c < DIM; ++c) Ku[c] = 0.0;
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
    // node flags: bit c = dof c constrained, bit 3 = carries external load
    const uint8_t fl = L.nflag[n];
    const double im = L.inv_mass[n];
#pragma unroll
    for (int c = 0; c < DIM; ++c) {
        const size_t q = (size_t)n * DIM + c;
        const bool bc = (fl >> c) & 1;
        const double p = (fl & 8) ? d.P[q] * scale : 0.0;
        const double acc = bc ? 0.0 : (p - d.Nsh * Ku[c]) * im;
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

// tile shapes
#define BOND2 2, 32, 8, 1, 2
#define BOND3 3, 16, 4, 4, 2

size_t lattice_smem_bytes(int dim, int R, int S) {
    return dim == 2 ? bond_smem<BOND2>(R, S) : bond_smem<BOND3>(R, S);
}

void launch_lattice_step(const DevPD& d, const LatticeDev& L, int step, int do_break,
                         double scale, int write_state, bool time_bond, cudaEvent_t* ev,
                         cudaStream_t s, const Stencil3D* st3) {
    const int nb = ((L.nx + 1) * (L.jn1 - L.jn0) * (d.dim == 3 ? L.nz + 1 : 1) + 255) / 256;
    if (d.dim == 3 && st3) {  // the specialised 122-offset kernel (pd_lat3.cu)
        // tiled ubar + the cold-tile screen's edge maxima (only when the break test runs)
        launch_lat3_ubar(d, L, do_break ? const_cast<unsigned*>(st3->tmax) : nullptr, s);
        if (time_bond) PMTS_CUDA_S(cudaEventRecord(ev[0], s));
        launch_lat3_bond(d, L, *st3, step, do_break, s);
        if (time_bond) PMTS_CUDA_S(cudaEventRecord(ev[1], s));
        k_lat_node<3><<<nb, 256, 0, s>>>(d, L, scale, write_state);
        PMTS_CUDA_S(cudaGetLastError());
        return;
    }
    const size_t smem = lattice_smem_bytes(d.dim, L.R, L.S);
    if (d.dim == 2) {
        using T = BondTile<BOND2>;
        if (time_bond) PMTS_CUDA_S(cudaEventRecord(ev[0], s));
        dim3 grid((L.nx + 31) / 32, (L.ny + T::EY - 1) / T::EY, 1);
        k_lat_bond<BOND2><<<grid, T::NT, smem, s>>>(d, L, step, do_break);
        if (time_bond) PMTS_CUDA_S(cudaEventRecord(ev[1], s));
        k_lat_node<2><<<nb, 256, 0, s>>>(d, L, scale, write_state);
    } else {
        using T = BondTile<BOND3>;
        k_lat_ubar<3><<<(d.E + 255) / 256, 256, 0, s>>>(d, L);
        if (time_bond) PMTS_CUDA_S(cudaEventRecord(ev[0], s));
        dim3 grid((L.nx + 15) / 16, (L.ny + 3) / 4, (L.nz + T::EZ - 1) / T::EZ);
        k_lat_bond<BOND3><<<grid, T::NT, smem, s>>>(d, L, step, do_break);
        if (time_bond) PMTS_CUDA_S(cudaEventRecord(ev[1], s));
        k_lat_node<3><<<nb, 256, 0, s>>>(d, L, scale, write_state);
    }
    PMTS_CUDA_S(cudaGetLastError());
}

void lattice_configure(int dim, int R, int S) {
    const int bytes = (int)lattice_smem_bytes(dim, R, S);
    if (dim == 2)
        PMTS_CUDA_S(cudaFuncSetAttribute(k_lat_bond<BOND2>,
                                         cudaFuncAttributeMaxDynamicSharedMemorySize, bytes));
    else
        PMTS_CUDA_S(cudaFuncSetAttribute(k_lat_bond<BOND3>,
                                         cudaFuncAttributeMaxDynamicSharedMemorySize, bytes));
}

// ---- lattice encoding of device-resident ELL families (fast mode setup) ----
// The generated mesh numbers element (i, j, k) as (k ny + j) nx + i
// (mesh.hpp:170-219), so every family entry is an integer offset.  These two
// passes replace the host walk over all F entries: the first collects the
// offsets present (and the largest component), the host orders them into the
// stencil (a few hundred at most), the second writes each element's intact bits.
namespace {
constexpr int kSpan17 = 17, kKeys17 = 17 * 17 * 17;
__device__ __forceinline__ void lat_ijk(int e, int nx, int ny, int& i, int& j, int& k) {
    i = e % nx;
    const int r = e / nx;
    j = r % ny;
    k = r / ny;
}

__global__ void k_lat_scan(const int32_t* __restrict__ col, int E, int K, int nx, int ny,
                           int* __restrict__ present, int* __restrict__ rmax) {
    int lr = 0;
    for (int e = blockIdx.x * blockDim.x + threadIdx.x; e < E; e += gridDim.x * blockDim.x) {
        int a, b, c;
        lat_ijk(e, nx, ny, a, b, c);
        for (int q = 0; q < K; ++q) {
            const int p = col[(size_t)q * E + e];
            if (p < 0) break;
            int x, y, z;
            lat_ijk(p, nx, ny, x, y, z);
            const int di = x - a, dj = y - b, dk = z - c;
            const int m = max(abs(di), max(abs(dj), abs(dk)));
            lr = max(lr, m);
            if (m <= 8) {
                const int key = ((dk + 8) * kSpan17 + dj + 8) * kSpan17 + di + 8;
                if (!present[key]) present[key] = 1;  // every writer stores 1
            }
        }
    }
    lr = __reduce_max_sync(0xffffffffu, lr);
    if ((threadIdx.x & 31) == 0 && lr) atomicMax(rmax, lr);
}

__global__ void k_lat_mask(const int32_t* __restrict__ col, int E, int K, int nx, int ny,
                           const int* __restrict__ slot17, int W, uint32_t* __restrict__ mask,
                           unsigned long long* __restrict__ count) {
    __shared__ int sl[kKeys17];
    for (int i = threadIdx.x; i < kKeys17; i += blockDim.x) sl[i] = slot17[i];
    __syncthreads();
    unsigned long long cnt = 0;
    for (int e = blockIdx.x * blockDim.x + threadIdx.x; e < E; e += gridDim.x * blockDim.x) {
        int a, b, c;
        lat_ijk(e, nx, ny, a, b, c);
        uint32_t m0 = 0, m1 = 0, m2 = 0, m3 = 0;
        for (int q = 0; q < K; ++q) {
            const int p = col[(size_t)q * E + e];
            if (p < 0) break;
            int x, y, z;
            lat_ijk(p, nx, ny, x, y, z);
            const int sidx = sl[((z - c + 8) * kSpan17 + y - b + 8) * kSpan17 + x - a + 8];
            const uint32_t bit = 1u << (sidx & 31);
            const int w = sidx >> 5;
            m0 |= w == 0 ? bit : 0u;
            m1 |= w == 1 ? bit : 0u;
            m2 |= w == 2 ? bit : 0u;
            m3 |= w == 3 ? bit : 0u;
            ++cnt;
        }
        mask[e] = m0;
        if (W > 1) mask[(size_t)E + e] = m1;
        if (W > 2) mask[2 * (size_t)E + e] = m2;
        if (W > 3) mask[3 * (size_t)E + e] = m3;
    }
    for (int o = 16; o > 0; o >>= 1) cnt += __shfl_down_sync(0xffffffffu, cnt, o);
    if ((threadIdx.x & 31) == 0 && cnt) atomicAdd(count, cnt);
}
}  // namespace

int lattice_scan_device(const int32_t* d_col, int E, int K, int nx, int ny, int* present17,
                        cudaStream_t s) {
    int* dp = nullptr;
    int* dr = nullptr;
    cudaMallocAsync(&dp, sizeof(int) * (kKeys17 + 1), s);
    dr = dp + kKeys17;
    cudaMemsetAsync(dp, 0, sizeof(int) * (kKeys17 + 1), s);
    k_lat_scan<<<1184, 256, 0, s>>>(d_col, E, K, nx, ny, dp, dr);
    int R = 0;
    cudaMemcpyAsync(present17, dp, sizeof(int) * kKeys17, cudaMemcpyDeviceToHost, s);
    cudaMemcpyAsync(&R, dr, sizeof(int), cudaMemcpyDeviceToHost, s);
    cudaFreeAsync(dp, s);
    const cudaError_t e = cudaStreamSynchronize(s);
    if (e != cudaSuccess) throw std::runtime_error(std::string("CUDA: ") + cudaGetErrorString(e));
    return R;
}

// ---- damage_field (perifem.hpp:202-231) and the intact export on the lattice ----
// `present` is the stencil mask as encoded (the bonds that exist); `mask` the live
// one.  pos_only: the fused 2D kernels keep a bond's state at its lower element only,
// so the negative offset s of e is read at the partner with the reversed offset
// S - 1 - s.  The stencil is sorted by ascending linear delta, so s ascending is
// partner id ascending -- the family order the ELL damage kernel sums in.
namespace {
__device__ __forceinline__ bool lat_bit(const uint32_t* m, int E, int e, int s) {
    return (m[(size_t)(s >> 5) * E + e] >> (s & 31)) & 1u;
}
__global__ void k_lat_damage_elem(DevPD d, LatticeDev L, const uint32_t* present, int pos_only,
                                  double* phi, uint8_t* has) {
    const int e = blockIdx.x * blockDim.x + threadIdx.x;
    if (e >= d.E) return;
    const int S = L.S;
    double total = 0.0, intact = 0.0;
    for (int s = 0; s < S; ++s) {
        if (!lat_bit(present, d.E, e, s)) continue;
        const int p = e + L.delta_id[s];
        const int lo = e < p ? e : p, hi = e < p ? p : e;
        // explicit roundings: this file builds with FMA contraction on, and the sums
        // must round like damage_field's (pd_det.cu builds with -fmad=false)
        const double w = __dmul_rn(d.vol[lo], d.vol[hi]);
        total = __dadd_rn(total, w);
        const bool live = (pos_only && p < e) ? lat_bit(d.mask, d.E, p, S - 1 - s)
                                              : lat_bit(d.mask, d.E, e, s);
        if (live) intact = __dadd_rn(intact, w);
    }
    phi[e] = total > 0.0 ? __dadd_rn(1.0, -__ddiv_rn(intact, total)) : 0.0;
    has[e] = total != 0.0;
}
__global__ void k_lat_bond_count(const uint32_t* present, int E, int S, int W, int* cnt) {
    const int e = blockIdx.x * blockDim.x + threadIdx.x;
    if (e > E) return;
    if (e == E) {  // the exclusive scan's total lands past the end
        cnt[e] = 0;
        return;
    }
    int c = 0;
    for (int s = S / 2; s < S; ++s) c += lat_bit(present, E, e, s) ? 1 : 0;
    cnt[e] = c;
}
__global__ void k_lat_intact(DevPD d, LatticeDev L, const uint32_t* present, const int* offs,
                             uint8_t* out) {
    const int e = blockIdx.x * blockDim.x + threadIdx.x;
    if (e >= d.E) return;
    int q = offs[e];
    for (int s = L.S / 2; s < L.S; ++s)
        if (lat_bit(present, d.E, e, s)) out[q++] = lat_bit(d.mask, d.E, e, s) ? 1 : 0;
}
}  // namespace

void launch_lat_damage(const DevPD& d, const LatticeDev& L, const uint32_t* present, bool pos_only,
                       double* elem, double* node, cudaStream_t s) {
    uint8_t* has = nullptr;
    PMTS_CUDA_S(cudaMallocAsync(&has, (size_t)d.E, s));
    k_lat_damage_elem<<<(d.E + 255) / 256, 256, 0, s>>>(d, L, present, pos_only ? 1 : 0, elem, has);
    launch_damage_node(d, elem, has, node, s);
    PMTS_CUDA_S(cudaFreeAsync(has, s));
}

long long launch_lat_intact(const DevPD& d, const LatticeDev& L, const uint32_t* present,
                            uint8_t* out_dev, cudaStream_t s) {
    int* cnt = nullptr;
    PMTS_CUDA_S(cudaMallocAsync(&cnt, sizeof(int) * ((size_t)d.E + 1), s));
    k_lat_bond_count<<<(d.E + 256) / 256, 256, 0, s>>>(present, d.E, L.S, L.W, cnt);
    size_t tmp_bytes = 0;
    cub::DeviceScan::ExclusiveSum(nullptr, tmp_bytes, cnt, cnt, d.E + 1, s);
    void* tmp = nullptr;
    PMTS_CUDA_S(cudaMallocAsync(&tmp, tmp_bytes, s));
    cub::DeviceScan::ExclusiveSum(tmp, tmp_bytes, cnt, cnt, d.E + 1, s);
    int total = 0;
    PMTS_CUDA_S(cudaMemcpyAsync(&total, cnt + d.E, sizeof(int), cudaMemcpyDeviceToHost, s));
    if (out_dev) k_lat_intact<<<(d.E + 255) / 256, 256, 0, s>>>(d, L, present, cnt, out_dev);
    PMTS_CUDA_S(cudaFreeAsync(tmp, s));
    PMTS_CUDA_S(cudaFreeAsync(cnt, s));
    PMTS_CUDA_S(cudaStreamSynchronize(s));
    return total;
}

long long lattice_mask_device(const int32_t* d_col, int E, int K, int nx, int ny,
                              const int* slot17, int W, uint32_t* d_mask, cudaStream_t s) {
    int* ds = nullptr;
    unsigned long long* dc = nullptr;
    cudaMallocAsync(&ds, sizeof(int) * kKeys17, s);
    cudaMallocAsync(&dc, sizeof(unsigned long long), s);
    cudaMemcpyAsync(ds, slot17, sizeof(int) * kKeys17, cudaMemcpyHostToDevice, s);
    cudaMemsetAsync(dc, 0, sizeof(unsigned long long), s);
    k_lat_mask<<<1184, 256, 0, s>>>(d_col, E, K, nx, ny, ds, W, d_mask, dc);
    unsigned long long F = 0;
    cudaMemcpyAsync(&F, dc, sizeof(F), cudaMemcpyDeviceToHost, s);
    cudaFreeAsync(ds, s);
    cudaFreeAsync(dc, s);
    const cudaError_t e = cudaStreamSynchronize(s);
    if (e != cudaSuccess) throw std::runtime_error(std::string("CUDA: ") + cudaGetErrorString(e));
    return (long long)F;
}

}  // namespace pmts
