// Device kernels of the coupled multi-time-step integrator (pmts_mts.cu):
// the FE operator (CSR, the reference's row order), the Newmark block solves of
// both subdomains, the Boolean coupling operators and deterministic
// reductions for the conjugate-gradient solves.  Built with -fmad=false so
// every expression rounds as the reference's does.
// Citations: /root/reference/proj/include/perimts/.
#include <algorithm>
#include <climits>
#include <vector>
#include <stdexcept>
#include <string>

#include "pd_common.cuh"
#include "pd_mts.cuh"

namespace pmts {
namespace mtsk {

namespace {

constexpr int kT = 256;

inline int blocks(long long n) { return (int)((n + kT - 1) / kT); }

void check(const char* what) {
    cudaError_t e = cudaGetLastError();
    if (e != cudaSuccess)
        throw std::runtime_error(std::string("CUDA (") + what + "): " + cudaGetErrorString(e));
}

// SparseMatrix::multiply (linalg.hpp:209-221): per row, ascending columns
__global__ void k_csr(int n, const int32_t* __restrict__ rp, const int32_t* __restrict__ ci,
                      const double* __restrict__ v, const double* __restrict__ x,
                      double* __restrict__ y) {
    const int i = blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= n) return;
    double s = 0.0;
    for (int p = rp[i]; p < rp[i + 1]; ++p) s += v[p] * x[ci[p]];
    y[i] = s;
}

// newmark_predictor (newmark.hpp:61-69)
__global__ void k_predict(int n, const double* u, const double* v, const double* a, double* rd,
                          double* rv, double dt, double cpv, double cpd) {
    const int i = blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= n) return;
    rv[i] = v[i] + cpv * a[i];
    rd[i] = u[i] + dt * v[i] + cpd * a[i];
}

// BlockOperator::solve, explicit branch (newmark.hpp:122-131, 150-158)
__global__ void k_explicit(int n, const double* ra, double ra_scale, const double* kd,
                           const double* M, const uint8_t* cf, const double* rv, const double* rd,
                           double gdt, double bdt2, const double* bcvel, int homog, double* u,
                           double* v, double* a) {
    const int i = blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= n) return;
    const bool c = cf[i] != 0;
    const double rai = ra ? ra[i] * ra_scale : 0.0;
    const double b = c ? 0.0 : rai - kd[i];
    const double acc = c ? 0.0 : b / M[i];
    double vel = rv[i] + gdt * acc;
    const double dis = rd[i] + bdt2 * acc;
    if (c) vel = homog ? 0.0 : bcvel[i];
    a[i] = acc;
    v[i] = vel;
    u[i] = dis;
}

// right-hand side of the reduced block equation: b = P - K r_d, constrained 0
__global__ void k_rhs(int n, const double* ra, double ra_scale, const double* kd, const uint8_t* cf,
                      double* b) {
    const int i = blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= n) return;
    const double rai = ra ? ra[i] * ra_scale : 0.0;
    b[i] = cf[i] ? 0.0 : rai - kd[i];
}

// the CG operator of the implicit branch (newmark.hpp:140-144)
__global__ void k_apply_a(int n, const double* x, const double* kx, const double* M,
                          const uint8_t* cf, double bdt2, double* y) {
    const int i = blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= n) return;
    y[i] = cf[i] ? x[i] : M[i] * x[i] + bdt2 * kx[i];
}

__global__ void k_finish(int n, const double* acc, const double* rv, const double* rd, double gdt,
                         double bdt2, const uint8_t* cf, const double* bcvel, int homog, double* u,
                         double* v, double* a) {
    const int i = blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= n) return;
    const bool c = cf[i] != 0;
    const double ac = c ? 0.0 : acc[i];
    double vel = rv[i] + gdt * ac;
    if (c) vel = homog ? 0.0 : bcvel[i];
    a[i] = ac;
    v[i] = vel;
    u[i] = rd[i] + bdt2 * ac;
}

__global__ void k_zero_cf(int n, const uint8_t* cf, double* x) {
    const int i = blockIdx.x * blockDim.x + threadIdx.x;
    if (i < n && cf[i]) x[i] = 0.0;
}

// initial_acceleration (newmark.hpp:110-116)
__global__ void k_init_acc(int n, const double* p, const double* ku, const double* M,
                           const uint8_t* cf, double* a) {
    const int i = blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= n) return;
    a[i] = cf[i] ? 0.0 : (p[i] - ku[i]) / M[i];
}

// idx[r] < 0: a row this shard does not own (sharded coupled run): no load; its
// gathered value is -0.0, the identity of the owner-sum across shards (x + -0.0 == x
// for every x, -0.0 included)
__global__ void k_scatter_add(int n, const int32_t* idx, const double* vals, double* dst) {
    const int r = blockIdx.x * blockDim.x + threadIdx.x;
    if (r < n && idx[r] >= 0) dst[idx[r]] += vals[r];
}

__global__ void k_gather(int n, const int32_t* idx, const double* src, double* dst) {
    const int r = blockIdx.x * blockDim.x + threadIdx.x;
    if (r < n) dst[r] = idx[r] >= 0 ? src[idx[r]] : -0.0;
}

__global__ void k_fill(long long n, double v, double* x) {
    const long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x;
    if (i < n) x[i] = v;
}
// dst[didx[i]] = src[sidx[i]] (halo copies between shard buffers; src may be a peer's)
__global__ void k_copy_idx(int n, const double* src, const int32_t* sidx, double* dst,
                           const int32_t* didx) {
    const int i = blockIdx.x * blockDim.x + threadIdx.x;
    if (i < n) dst[didx[i]] = src[sidx[i]];
}
__global__ void k_scatter_set(int n, const int32_t* idx, const double* vals, double* dst) {
    const int i = blockIdx.x * blockDim.x + threadIdx.x;
    if (i < n) dst[idx[i]] = vals[i];
}

// G_FE with interpolation rows (non-matching meshes): out[r] = sum_j w_j x[ci_j],
// the first term alone when the row has one entry (the conforming map: bitwise
// the plain gather)
__global__ void k_gather_csr(int n, const int32_t* rp, const int32_t* ci, const double* w,
                             const double* src, double* dst) {
    const int r = blockIdx.x * blockDim.x + threadIdx.x;
    if (r >= n) return;
    int j = rp[r];
    double acc = w[j] * src[ci[j]];
    for (++j; j < rp[r + 1]; ++j) acc += w[j] * src[ci[j]];
    dst[r] = acc;
}
// dst[d] += sum over the rows of d (ascending) of w vals[row]: G_FE^T vals on the
// touched dofs (td) through the transposed CSR (trp / tri / tw)
__global__ void k_scatter_csr(int nt, const int32_t* td, const int32_t* trp, const int32_t* tri,
                              const double* tw, const double* vals, double* dst) {
    const int q = blockIdx.x * blockDim.x + threadIdx.x;
    if (q >= nt) return;
    int j = trp[q];
    double acc = tw[j] * vals[tri[j]];
    for (++j; j < trp[q + 1]; ++j) acc += tw[j] * vals[tri[j]];
    dst[td[q]] += acc;
}

__global__ void k_add(int n, const double* x, double* y) {
    const int i = blockIdx.x * blockDim.x + threadIdx.x;
    if (i < n) y[i] = y[i] + x[i];
}

__global__ void k_scale(int n, const double* x, double s, double* y) {
    const int i = blockIdx.x * blockDim.x + threadIdx.x;
    if (i < n) y[i] = x[i] * s;
}

__global__ void k_add3(int n, const double* a0, const double* a1, const double* a2,
                       const double* b0, const double* b1, const double* b2, double* o0,
                       double* o1, double* o2) {
    const int i = blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= n) return;
    o0[i] = a0[i] + b0[i];
    o1[i] = a1[i] + b1[i];
    o2[i] = a2[i] + b2[i];
}

// x += alpha p; r -= alpha ap  (axpy pair of cg_solve, linalg.hpp:283-284)
__global__ void k_cg_update(int n, const double* alpha_dev, const double* p, const double* ap,
                            double* x, double* r) {
    const int i = blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= n) return;
    const double al = *alpha_dev;
    x[i] += al * p[i];
    r[i] += -al * ap[i];
}

// z = precond(r) (jacobi, linalg.hpp:262-269)
__global__ void k_precond(int n, const double* r, const double* jac, double* z) {
    const int i = blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= n) return;
    z[i] = jac ? (jac[i] != 0.0 ? r[i] / jac[i] : r[i]) : r[i];
}

// p = z + beta p
__global__ void k_xpby(int n, const double* z, const double* beta_dev, double* p) {
    const int i = blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= n) return;
    p[i] = z[i] + *beta_dev * p[i];
}

// deterministic dot products: fixed-shape block partials, then one block
__global__ void k_dot_partial(int n, const double* x, const double* y, double* part) {
    __shared__ double sh[kT];
    double s = 0.0;
    for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < n; i += gridDim.x * blockDim.x)
        s += x[i] * y[i];
    sh[threadIdx.x] = s;
    __syncthreads();
    for (int o = kT / 2; o > 0; o >>= 1) {
        if ((int)threadIdx.x < o) sh[threadIdx.x] += sh[threadIdx.x + o];
        __syncthreads();
    }
    if (threadIdx.x == 0) part[blockIdx.x] = sh[0];
}

__global__ void k_sum_partials(int nb, const double* part, double* out) {
    __shared__ double sh[kT];
    double s = 0.0;
    for (int i = threadIdx.x; i < nb; i += blockDim.x) s += part[i];
    sh[threadIdx.x] = s;
    __syncthreads();
    for (int o = kT / 2; o > 0; o >>= 1) {
        if ((int)threadIdx.x < o) sh[threadIdx.x] += sh[threadIdx.x + o];
        __syncthreads();
    }
    if (threadIdx.x == 0) *out = sh[0];
}

// CG scalars on the device: alpha = rz / pap, beta = rz_new / rz
__global__ void k_ratio(const double* num, const double* den, double* out) { *out = *num / *den; }

// One-launch dot product(s) for the CG iteration graph: the block partials of
// k_dot_partial (same grid, same per-thread order, same tree) and, in the last
// block to finish, the reduction of k_sum_partials over them -- bitwise the same
// sums as the two-launch form -- followed by the CG scalar:
//   mode 1 (alpha):  out = x.y,             *sc = *num / out
//   mode 2 (beta):   out = x.y, out2 = x2.y2, *sc = out / *num, then *num = out
__global__ void __launch_bounds__(kT) k_dot_fin(int n, const double* x, const double* y,
                                                const double* x2, const double* y2,
                                                double* part, unsigned* ticket, double* out,
                                                double* out2, int mode, double* num, double* sc) {
    __shared__ double sh[kT], sh2[kT];
    __shared__ bool last;
    const int nb = gridDim.x;
    double s = 0.0, s2 = 0.0;
    for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < n; i += gridDim.x * blockDim.x) {
        s += x[i] * y[i];
        if (x2) s2 += x2[i] * y2[i];
    }
    sh[threadIdx.x] = s;
    sh2[threadIdx.x] = s2;
    __syncthreads();
    for (int o = kT / 2; o > 0; o >>= 1) {
        if ((int)threadIdx.x < o) {
            sh[threadIdx.x] += sh[threadIdx.x + o];
            sh2[threadIdx.x] += sh2[threadIdx.x + o];
        }
        __syncthreads();
    }
    if (threadIdx.x == 0) {
        part[blockIdx.x] = sh[0];
        part[nb + blockIdx.x] = sh2[0];
        __threadfence();
        last = atomicAdd(ticket, 1u) == (unsigned)nb - 1;
    }
    __syncthreads();
    if (!last) return;
    __threadfence();
    const volatile double* vp = part;
    double t = 0.0, t2 = 0.0;
    for (int i = threadIdx.x; i < nb; i += blockDim.x) {
        t += vp[i];
        t2 += vp[nb + i];
    }
    sh[threadIdx.x] = t;
    sh2[threadIdx.x] = t2;
    __syncthreads();
    for (int o = kT / 2; o > 0; o >>= 1) {
        if ((int)threadIdx.x < o) {
            sh[threadIdx.x] += sh[threadIdx.x + o];
            sh2[threadIdx.x] += sh2[threadIdx.x + o];
        }
        __syncthreads();
    }
    if (threadIdx.x == 0) {
        *out = sh[0];
        if (x2) *out2 = sh2[0];
        if (mode == 1) *sc = *num / sh[0];
        if (mode == 2) {
            *sc = sh[0] / *num;
            *num = sh[0];
        }
        *ticket = 0u;  // ready for the next replay
    }
}

// The CG loop test of cg_solve (linalg.hpp:243-296) on the device, at the end of
// each iteration of the graph's WHILE body: the host's checks in the host's order
// (p'Ap <= 0 -> not positive definite; sqrt(rr) / sqrt(bb) > tol -> continue;
// continuing past max_iter -> no convergence), with IEEE sqrt and division, so the
// iteration count is the host loop's.  status: 0 converged, 1 not SPD, 2 max_iter.
__global__ void k_cg_cond(cudaGraphConditionalHandle h, const double* s_bb, const double* s_rr,
                          const double* s_pap, double tol, int max_iter, int* it_status) {
    const int it = ++it_status[0];
    bool more = false;
    if (*s_pap <= 0.0) {
        it_status[1] = 1;
    } else {
        more = sqrt(*s_rr) / sqrt(*s_bb) > tol;
        if (more && it >= max_iter) {
            it_status[1] = 2;
            more = false;
        }
    }
    cudaGraphSetConditional(h, more ? 1u : 0u);
}

// x += alpha p; r -= alpha ap; z = precond(r): k_cg_update then k_precond, fused
__global__ void k_cg_update_precond(int n, const double* alpha_dev, const double* p,
                                    const double* ap, double* x, double* r, const double* jac,
                                    double* z) {
    const int i = blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= n) return;
    const double al = *alpha_dev;
    x[i] += al * p[i];
    const double ri = r[i] + -al * ap[i];
    r[i] = ri;
    z[i] = jac ? (jac[i] != 0.0 ? ri / jac[i] : ri) : ri;
}

// y = A x, CSR, one warp per row (long rows: the interface's H_FE)
__global__ void k_csr_warp(int n, const int32_t* __restrict__ rp, const int32_t* __restrict__ ci,
                           const double* __restrict__ v, const double* __restrict__ x,
                           double* __restrict__ y) {
    const int row = (blockIdx.x * blockDim.x + threadIdx.x) >> 5, lane = threadIdx.x & 31;
    if (row >= n) return;
    double s = 0.0;
    for (int p = rp[row] + lane; p < rp[row + 1]; p += 32) s += v[p] * x[ci[p]];
    for (int o = 16; o > 0; o >>= 1) s += __shfl_down_sync(0xffffffffu, s, o);
    if (lane == 0) y[row] = s;
}

__global__ void k_dense_matvec(int n, const double* A, const double* x, double* y) {
    // y = A x for a row-major n x n matrix (the interface's H_FE), one warp per row
    const int warp = (blockIdx.x * blockDim.x + threadIdx.x) >> 5, lane = threadIdx.x & 31;
    if (warp >= n) return;
    const double* row = A + (size_t)warp * n;
    double s = 0.0;
    for (int j = lane; j < n; j += 32) s += row[j] * x[j];
    for (int o = 16; o > 0; o >>= 1) s += __shfl_down_sync(0xffffffffu, s, o);
    if (lane == 0) y[warp] = s;
}

// K^PD x for the MTS substeps, one warp per element, lanes over the family
// (32 entries per round): the deterministic kernel's per-entry arithmetic
// (pd_det.cu k_det_bond: eta from node displacements in the (i<j) orientation,
// exact stretch, inclusive test) with a warp-tree sum instead of the ascending
// serial sum -- small PD subdomains are latency-bound at one thread per element.
// Per element the products q_a = Nsh x(node_a) the force kernel forms for every partner
// (Q[e][a][c]) and their ascending sum S[e][c] -- the very expressions of k_pd_force_warp,
// so reading them instead of gathering 2^dim nodes per family entry is bitwise the same.
// S is a 64-byte record per element, {centroid x, y, z, S_x, S_y, S_z, 0, 0}: the partner
// data of an entry with e < p in two sectors and three 16-byte loads (the centroids' three
// arrays and S were five sectors and six loads -- the kernel below is bound by the L1
// load wavefronts of its gathers, ncu: 98 % of peak).
constexpr int kRec = 8;
template <int DIM>
__global__ void k_pd_elem_q(DevPD d, const double* __restrict__ x, double* __restrict__ Q,
                            double* __restrict__ S) {
    constexpr int NN = DIM == 2 ? 4 : 8;
    const int e = blockIdx.x * blockDim.x + threadIdx.x;
    if (e >= d.E) return;
    double q[NN][DIM];
    for (int a = 0; a < NN; ++a) {
        const int node = d.conn[a * d.E + e];
        for (int c = 0; c < DIM; ++c) q[a][c] = d.Nsh * x[(size_t)node * DIM + c];
    }
    for (int a = 0; a < NN; ++a)
        for (int c = 0; c < DIM; ++c) Q[((size_t)e * NN + a) * DIM + c] = q[a][c];
    double rec[kRec] = {d.cen[e], d.cen[d.E + e], d.cen[2 * (size_t)d.E + e], 0.0, 0.0, 0.0, 0.0, 0.0};
    for (int c = 0; c < DIM; ++c) {
        double sacc = 0.0;
        for (int a = 0; a < NN; ++a) sacc = sacc + q[a][c];
        rec[3 + c] = sacc;
    }
    double2* out = reinterpret_cast<double2*>(S + (size_t)e * kRec);
    for (int i = 0; i < kRec / 2; ++i) out[i] = make_double2(rec[2 * i], rec[2 * i + 1]);
}

template <int DIM>
__global__ void __launch_bounds__(kT) k_pd_force_warp(DevPD d, const double* __restrict__ x,
                                                      uint32_t* __restrict__ mask, int do_break,
                                                      unsigned long long* cnt) {
    constexpr int NN = DIM == 2 ? 4 : 8;
    const int e = (blockIdx.x * blockDim.x + threadIdx.x) >> 5, lane = threadIdx.x & 31;
    if (e >= d.E) return;
    const int E = d.E;
    double qe[NN][DIM];
    for (int a = 0; a < NN; ++a) {
        const int node = d.conn[a * E + e];
        for (int c = 0; c < DIM; ++c) qe[a][c] = d.Nsh * x[(size_t)node * DIM + c];
    }
    double Se[DIM];
    for (int c = 0; c < DIM; ++c) {
        double sacc = 0.0;
        for (int a = 0; a < NN; ++a) sacc = sacc + qe[a][c];
        Se[c] = sacc;
    }
    const double ce[3] = {d.cen[e], d.cen[E + e], d.cen[2 * E + e]};
    double G[DIM];
    for (int c = 0; c < DIM; ++c) G[c] = 0.0;
    unsigned nb = 0;
    for (int k0 = 0; k0 < d.K; k0 += 32) {
        const int k = k0 + lane;
        const int p = k < d.K ? d.col[(size_t)k * E + e] : -1;
        const uint32_t word = mask[(size_t)(k0 >> 5) * E + e];
        const bool on = p >= 0 && ((word >> lane) & 1u);
        bool brk = false;
        if (on) {
            double eta[DIM], xi[3];
            const double cp[3] = {d.cen[p], d.cen[E + p], d.cen[2 * E + p]};
            double qp[NN][DIM];
            for (int a = 0; a < NN; ++a) {
                const int node = d.conn[a * E + p];
                for (int c = 0; c < DIM; ++c) qp[a][c] = d.Nsh * x[(size_t)node * DIM + c];
            }
            if (e < p) {
                for (int c = 0; c < DIM; ++c) {
                    double sacc = 0.0;
                    for (int a = 0; a < NN; ++a) sacc = sacc + qp[a][c];
                    for (int a = 0; a < NN; ++a) sacc = sacc - qe[a][c];
                    eta[c] = sacc;
                }
                for (int c = 0; c < 3; ++c) xi[c] = cp[c] - ce[c];
            } else {
                for (int c = 0; c < DIM; ++c) {
                    double sacc = Se[c];
                    for (int a = 0; a < NN; ++a) sacc = sacc - qp[a][c];
                    eta[c] = sacc;
                }
                for (int c = 0; c < 3; ++c) xi[c] = ce[c] - cp[c];
            }
            double dot = xi[0] * eta[0] + xi[1] * eta[1];
            if constexpr (DIM == 3) dot = dot + xi[2] * eta[2];
            const double t = d.coef[(size_t)k * E + e] * dot;
            if (e > p) {
                for (int c = 0; c < DIM; ++c) G[c] = G[c] + t * xi[c];
            } else {
                for (int c = 0; c < DIM; ++c) G[c] = G[c] - t * xi[c];
            }
            if (do_break) {
                const double xin = sqrt(xi[0] * xi[0] + xi[1] * xi[1] + xi[2] * xi[2]);
                double len2 = 0.0;
                for (int c = 0; c < DIM; ++c) {
                    const double v = xi[c] + eta[c];
                    len2 = len2 + v * v;
                }
                const double len = sqrt(len2);
                const double sv = len <= 0.0 ? -1.0 : (len - xin) / xin;
                brk = sv >= d.s_crit;
                if (brk && e < p && owns_elem(d, e)) ++nb;  // once per bond, by its owner
            }
        }
        if (do_break) {
            const unsigned bal = __ballot_sync(0xffffffffu, brk);
            if (lane == 0 && bal) mask[(size_t)(k0 >> 5) * E + e] = word & ~bal;
        }
    }
    for (int c = 0; c < DIM; ++c)
        for (int o = 16; o > 0; o >>= 1) G[c] += __shfl_down_sync(0xffffffffu, G[c], o);
    if (lane == 0)
        for (int c = 0; c < DIM; ++c) d.G[(size_t)e * DIM + c] = G[c];
    if (do_break) {
        for (int o = 16; o > 0; o >>= 1) nb += __shfl_down_sync(0xffffffffu, nb, o);
        if (lane == 0 && nb) atomicAdd(cnt, (unsigned long long)nb);
    }
}

// k_pd_force_warp for large subdomains, on the per-element node products of k_pd_elem_q:
// the same expressions in the same order (eta of an entry with e < p is S_p - q_e0 - ...
// - q_e7, with e > p it is S_e - q_p0 - ... - q_p7), so the force, the stretch test and the
// bond states are bitwise those of k_pd_force_warp.  The element's own products sit in
// shared memory and the partner's stream through two registers, so the kernel fits 64
// registers and four blocks per SM -- the original holds both sets (149 registers, one
// block per SM, 8 warps) and ran 150 ms per call at BASELINE cfg5, latency-bound.
template <int DIM>
__global__ void __launch_bounds__(kT, 4) k_pd_force_warp_q(DevPD d, uint32_t* __restrict__ mask,
                                                           int do_break, unsigned long long* cnt,
                                                           const double* __restrict__ Q,
                                                           const double* __restrict__ S,
                                                           const int32_t* __restrict__ colT,
                                                           const double* __restrict__ coefT) {
    constexpr int NN = DIM == 2 ? 4 : 8, NQ = NN * DIM;
    __shared__ double qes[kT / 32][NQ];
    const int e = (blockIdx.x * blockDim.x + threadIdx.x) >> 5, lane = threadIdx.x & 31;
    if (e >= d.E) return;
    const int E = d.E;
    double* qe = qes[threadIdx.x >> 5];
    if (lane < NQ) qe[lane] = Q[(size_t)e * NQ + lane];
    __syncwarp();
    double Se[DIM];
    for (int c = 0; c < DIM; ++c) Se[c] = S[(size_t)e * kRec + 3 + c];
    const double ce[3] = {S[(size_t)e * kRec], S[(size_t)e * kRec + 1], S[(size_t)e * kRec + 2]};
    double G[DIM];
    for (int c = 0; c < DIM; ++c) G[c] = 0.0;
    unsigned nb = 0;
    for (int k0 = 0; k0 < d.K; k0 += 32) {
        const int k = k0 + lane;
        // (entry-major copies when present: the lanes of a warp read one line, not 32)
        const int p = k < d.K ? (colT ? colT[(size_t)e * d.K + k] : d.col[(size_t)k * E + e]) : -1;
        const uint32_t word = mask[(size_t)(k0 >> 5) * E + e];
        const bool on = p >= 0 && ((word >> lane) & 1u);
        bool brk = false;
        if (on) {
            double eta[DIM], xi[3];
            const double2* rp = reinterpret_cast<const double2*>(S + (size_t)p * kRec);
            const double2 r0 = rp[0], r1 = rp[1];  // cen x, y | cen z, S_x
            const double cp[3] = {r0.x, r0.y, r1.x};
            if (e < p) {
                const double2 r2 = rp[2];  // S_y, S_z
                const double sp[3] = {r1.y, r2.x, r2.y};
                for (int c = 0; c < DIM; ++c) eta[c] = sp[c];
                for (int a = 0; a < NN; ++a)
                    for (int c = 0; c < DIM; ++c) eta[c] = eta[c] - qe[a * DIM + c];
                for (int c = 0; c < 3; ++c) xi[c] = cp[c] - ce[c];
            } else {
                // the partner's products in 16-byte loads, subtracted in the same order
                // (a ascending for every component)
                const double2* qp = reinterpret_cast<const double2*>(Q + (size_t)p * NQ);
                for (int c = 0; c < DIM; ++c) eta[c] = Se[c];
#pragma unroll
                for (int i = 0; i < NQ / 2; ++i) {
                    const double2 v = qp[i];
                    eta[(2 * i) % DIM] = eta[(2 * i) % DIM] - v.x;
                    eta[(2 * i + 1) % DIM] = eta[(2 * i + 1) % DIM] - v.y;
                }
                for (int c = 0; c < 3; ++c) xi[c] = ce[c] - cp[c];
            }
            double dot = xi[0] * eta[0] + xi[1] * eta[1];
            if constexpr (DIM == 3) dot = dot + xi[2] * eta[2];
            const double t = (coefT ? coefT[(size_t)e * d.K + k] : d.coef[(size_t)k * E + e]) * dot;
            if (e > p) {
                for (int c = 0; c < DIM; ++c) G[c] = G[c] + t * xi[c];
            } else {
                for (int c = 0; c < DIM; ++c) G[c] = G[c] - t * xi[c];
            }
            if (do_break) {
                const double xin = sqrt(xi[0] * xi[0] + xi[1] * xi[1] + xi[2] * xi[2]);
                double len2 = 0.0;
                for (int c = 0; c < DIM; ++c) {
                    const double v = xi[c] + eta[c];
                    len2 = len2 + v * v;
                }
                const double len = sqrt(len2);
                const double sv = len <= 0.0 ? -1.0 : (len - xin) / xin;
                brk = sv >= d.s_crit;
                if (brk && e < p && owns_elem(d, e)) ++nb;  // once per bond, by its owner
            }
        }
        if (do_break) {
            const unsigned bal = __ballot_sync(0xffffffffu, brk);
            if (lane == 0 && bal) mask[(size_t)(k0 >> 5) * E + e] = word & ~bal;
        }
    }
    for (int c = 0; c < DIM; ++c)
        for (int o = 16; o > 0; o >>= 1) G[c] += __shfl_down_sync(0xffffffffu, G[c], o);
    if (lane == 0)
        for (int c = 0; c < DIM; ++c) d.G[(size_t)e * DIM + c] = G[c];
    if (do_break) {
        for (int o = 16; o > 0; o >>= 1) nb += __shfl_down_sync(0xffffffffu, nb, o);
        if (lane == 0 && nb) atomicAdd(cnt, (unsigned long long)nb);
    }
}

// Linear K^PD x for the homogeneous substeps (unit responses, link and
// interface solves -- no bond test): eta = ubar_p - ubar_e from per-element
// centroid displacements, G_e = -sum coef (xi.eta) xi with xi = c_p - c_e.
// The same operator as the deterministic form (sum_a N u_a = ubar exactly in
// real arithmetic), one partner load of 16 bytes instead of 2^dim nodes.
template <int DIM>
__global__ void k_pd_ubar(DevPD d, const double* __restrict__ x, double* __restrict__ ub) {
    constexpr int NN = DIM == 2 ? 4 : 8;
    const int e = blockIdx.x * blockDim.x + threadIdx.x;
    if (e >= d.E) return;
    double s[DIM];
    for (int c = 0; c < DIM; ++c) s[c] = 0.0;
    for (int a = 0; a < NN; ++a) {
        const int node = d.conn[a * d.E + e];
        for (int c = 0; c < DIM; ++c) s[c] = s[c] + d.Nsh * x[(size_t)node * DIM + c];
    }
    for (int c = 0; c < DIM; ++c) ub[(size_t)e * DIM + c] = s[c];
}

template <int DIM>
__global__ void __launch_bounds__(kT) k_pd_force_lin(DevPD d, const double* __restrict__ ub,
                                                     const uint32_t* __restrict__ mask) {
    const int e = (blockIdx.x * blockDim.x + threadIdx.x) >> 5, lane = threadIdx.x & 31;
    if (e >= d.E) return;
    const int E = d.E;
    double ue[DIM], G[DIM];
    for (int c = 0; c < DIM; ++c) {
        ue[c] = ub[(size_t)e * DIM + c];
        G[c] = 0.0;
    }
    const double ce[3] = {d.cen[e], d.cen[E + e], d.cen[2 * E + e]};
    for (int k0 = 0; k0 < d.K; k0 += 32) {
        const int k = k0 + lane;
        const int p = k < d.K ? d.col[(size_t)k * E + e] : -1;
        const uint32_t word = mask[(size_t)(k0 >> 5) * E + e];
        if (p >= 0 && ((word >> lane) & 1u)) {
            double xi[DIM], dot = 0.0;
            for (int c = 0; c < DIM; ++c) {
                xi[c] = d.cen[(size_t)c * E + p] - ce[c];
                dot = dot + xi[c] * (ub[(size_t)p * DIM + c] - ue[c]);
            }
            const double t = d.coef[(size_t)k * E + e] * dot;
            for (int c = 0; c < DIM; ++c) G[c] = G[c] - t * xi[c];
        }
    }
    for (int c = 0; c < DIM; ++c)
        for (int o = 16; o > 0; o >>= 1) G[c] += __shfl_down_sync(0xffffffffu, G[c], o);
    if (lane == 0)
        for (int c = 0; c < DIM; ++c) d.G[(size_t)e * DIM + c] = G[c];
}

// Entry-major copy of the families for the warp-per-element linear force: lane k
// of element e reads colT[e K + k], coefT[e K + k] and xiT[(e K + k) DIM + c] =
// cen_c(p) - cen_c(e) (the subtraction k_pd_force_lin performs) with coalesced
// loads, where the [k E + e] layout put every lane on its own cache line.
template <int DIM>
__global__ void k_family_transpose(DevPD d, int32_t* colT, double* coefT) {
    const long long q = (long long)blockIdx.x * blockDim.x + threadIdx.x;  // q = e K + k
    if (q >= (long long)d.E * d.K) return;
    const int e = (int)(q / d.K), k = (int)(q % d.K);
    const int p = d.col[(size_t)k * d.E + e];
    colT[q] = p;
    coefT[q] = p >= 0 ? d.coef[(size_t)k * d.E + e] : 0.0;
}

// k_pd_force_lin on the entry-major families: the same per-lane arithmetic and
// warp-tree sum, so bitwise the same G.  xi = cen_p - cen_e is formed from the
// centroids (cached gathers) instead of a stored E K dim table: 12 B per entry from
// HBM instead of 36 (BASELINE cfg5's 1.6e9 entries: 19 GB per substep, not 59)
template <int DIM, int KCH = DIM == 2 ? 1 : 4>
__global__ void __launch_bounds__(kT) k_pd_force_lin_t(DevPD d, const int32_t* __restrict__ colT,
                                                       const double* __restrict__ coefT,
                                                       const double* __restrict__ ub,
                                                       const uint32_t* __restrict__ mask) {
    const int e = (blockIdx.x * blockDim.x + threadIdx.x) >> 5, lane = threadIdx.x & 31;
    if (e >= d.E) return;
    const int E = d.E, K = d.K;
    double ue[DIM], G[DIM], ce[DIM];
    for (int c = 0; c < DIM; ++c) {
        ue[c] = ub[(size_t)e * DIM + c];
        ce[c] = d.cen[(size_t)c * E + e];
        G[c] = 0.0;
    }
    if (K <= 32 * KCH) {
        // families of up to KCH x 32 entries (the 2D and 3D stencils): every chunk's
        // entry loads issued first, then every gather, then the arithmetic in the chunk
        // order -- a latency-bound warp per element keeps 2 dependent round trips in
        // flight instead of 2 per chunk (same per-lane sums: bitwise the loop below)
        int pk[KCH];
        double cq[KCH];
        uint32_t wk[KCH];
#pragma unroll
        for (int i = 0; i < KCH; ++i) {
            const int k = 32 * i + lane;
            const bool in = k < K;
            pk[i] = in ? colT[(size_t)e * K + k] : -1;
            cq[i] = in ? coefT[(size_t)e * K + k] : 0.0;
            wk[i] = 32 * i < K ? mask[(size_t)i * E + e] : 0u;
        }
        double up[KCH][DIM], cp[KCH][DIM];
#pragma unroll
        for (int i = 0; i < KCH; ++i) {
            const bool on = pk[i] >= 0 && ((wk[i] >> lane) & 1u);
            for (int c = 0; c < DIM; ++c) {
                up[i][c] = on ? ub[(size_t)pk[i] * DIM + c] : 0.0;
                cp[i][c] = on ? __ldg(d.cen + (size_t)c * E + pk[i]) : 0.0;
            }
        }
#pragma unroll
        for (int i = 0; i < KCH; ++i) {
            if (pk[i] >= 0 && ((wk[i] >> lane) & 1u)) {
                double xi[DIM], dot = 0.0;
                for (int c = 0; c < DIM; ++c) {
                    xi[c] = cp[i][c] - ce[c];
                    dot = dot + xi[c] * (up[i][c] - ue[c]);
                }
                const double t = cq[i] * dot;
                for (int c = 0; c < DIM; ++c) G[c] = G[c] - t * xi[c];
            }
        }
    } else {
        for (int k0 = 0; k0 < K; k0 += 32) {
            const int k = k0 + lane;
            const size_t q = (size_t)e * K + k;
            const int p = k < K ? colT[q] : -1;
            const uint32_t word = mask[(size_t)(k0 >> 5) * E + e];
            if (p >= 0 && ((word >> lane) & 1u)) {
                double xi[DIM], dot = 0.0;
                for (int c = 0; c < DIM; ++c) {
                    xi[c] = __ldg(d.cen + (size_t)c * E + p) - ce[c];
                    dot = dot + xi[c] * (ub[(size_t)p * DIM + c] - ue[c]);
                }
                const double t = coefT[q] * dot;
                for (int c = 0; c < DIM; ++c) G[c] = G[c] - t * xi[c];
            }
        }
    }
    for (int c = 0; c < DIM; ++c)
        for (int o = 16; o > 0; o >>= 1) G[c] += __shfl_down_sync(0xffffffffu, G[c], o);
    if (lane == 0)
        for (int c = 0; c < DIM; ++c) d.G[(size_t)e * DIM + c] = G[c];
}

// sum_q Nsh G[e_q] over a node's incident elements (ascending, -1 ends the list), the
// index loads and the G gathers issued up front (2 round trips, not 2 per element)
template <int DIM>
__device__ __forceinline__ void node_sum(const DevPD& d, int n, double* Ku) {
    constexpr int NEM = DIM == 2 ? 4 : 8;
    if (d.NE <= NEM) {
        int eq[NEM];
#pragma unroll
        for (int q = 0; q < NEM; ++q) eq[q] = q < d.NE ? d.ne[(size_t)q * d.N + n] : -1;
        bool live = true;
#pragma unroll
        for (int q = 0; q < NEM; ++q) {  // the list ends at the first -1
            live = live && eq[q] >= 0;
            if (!live) eq[q] = -1;
        }
        double g[NEM][DIM];
#pragma unroll
        for (int q = 0; q < NEM; ++q)
            for (int c = 0; c < DIM; ++c) g[q][c] = eq[q] >= 0 ? d.G[(size_t)eq[q] * DIM + c] : 0.0;
#pragma unroll
        for (int q = 0; q < NEM; ++q)
            if (eq[q] >= 0)
                for (int c = 0; c < DIM; ++c) Ku[c] = Ku[c] + d.Nsh * g[q][c];
        return;
    }
    for (int q = 0; q < d.NE; ++q) {
        const int e = d.ne[(size_t)q * d.N + n];
        if (e < 0) break;
        for (int c = 0; c < DIM; ++c) Ku[c] = Ku[c] + d.Nsh * d.G[(size_t)e * DIM + c];
    }
}

// (K x)_n from the incident elements' G, fused with the explicit block solve
// of the node's dofs (newmark.hpp:122-131, 150-158)
template <int DIM>
__global__ void k_pd_node_explicit(DevPD d, const double* ra, double ra_scale, const double* M,
                                   const uint8_t* cf, const double* rv, const double* rd,
                                   double gdt, double bdt2, const double* bcvel, int homog,
                                   double* u, double* v, double* a) {
    const int n = blockIdx.x * blockDim.x + threadIdx.x;
    if (n >= d.N) return;
    double Ku[DIM];
    for (int c = 0; c < DIM; ++c) Ku[c] = 0.0;
    node_sum<DIM>(d, n, Ku);
    for (int c = 0; c < DIM; ++c) {
        const size_t i = (size_t)n * DIM + c;
        const bool cc = cf[i] != 0;
        const double rai = ra ? ra[i] * ra_scale : 0.0;
        const double b = cc ? 0.0 : rai - Ku[c];
        const double acc = cc ? 0.0 : b / M[i];
        double vel = rv[i] + gdt * acc;
        const double dis = rd[i] + bdt2 * acc;
        if (cc) vel = homog ? 0.0 : bcvel[i];
        a[i] = acc;
        v[i] = vel;
        u[i] = dis;
    }
}

// node phase of one homogeneous linear substep, fused: (K x)_n from the
// incident G (none on substep 1, which starts from rest), the multiplier load
// rhs.a = G_PD^T (w j/m) read through the dof's coupling row, the explicit
// solve, the predictor of the next substep (in place), and the gather of the
// coupling-row velocities into out (when non-null)
template <int DIM>
__global__ void k_pd_node_lin(DevPD d, int with_force, const double* w, const int32_t* row_of,
                              double f, const double* M, const uint8_t* cf, double gdt, double bdt2,
                              double dt, double cpv, double cpd, double* u, double* v, double* a,
                              double* rd, double* rv, double* out) {
    const int n = blockIdx.x * blockDim.x + threadIdx.x;
    if (n >= d.N) return;
    double Ku[DIM];
    for (int c = 0; c < DIM; ++c) Ku[c] = 0.0;
    if (with_force) node_sum<DIM>(d, n, Ku);
    for (int c = 0; c < DIM; ++c) {
        const size_t i = (size_t)n * DIM + c;
        const bool cc = cf[i] != 0;
        const int r = row_of[i];
        const double rai = r >= 0 ? 0.0 + w[r] * f : 0.0;  // assign(0) + scaled(w, j/m)
        const double b = cc ? 0.0 : rai - Ku[c];
        const double acc = cc ? 0.0 : b / M[i];
        double vel = rv[i] + gdt * acc;
        const double dis = rd[i] + bdt2 * acc;
        if (cc) vel = 0.0;  // homogeneous
        a[i] = acc;
        v[i] = vel;
        u[i] = dis;
        rv[i] = vel + cpv * acc;
        rd[i] = dis + dt * vel + cpd * acc;
        if (out && r >= 0) out[r] = vel;
    }
}

// predictor + load vector of one homogeneous substep: ra = 0, then the
// multiplier rows (one launch: rows are distinct dofs, and the zeroing of a
// row's dof is ordered before its add within the thread that owns it)
__global__ void k_pd_pre(int n, const double* u, const double* v, const double* a, double* rd,
                         double* rv, double* ra, double dt, double cpv, double cpd) {
    const int i = blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= n) return;
    rv[i] = v[i] + cpv * a[i];
    rd[i] = u[i] + dt * v[i] + cpd * a[i];
    ra[i] = 0.0;
}

__global__ void k_scatter_scaled(int n, const int32_t* idx, const double* w, double f, double* dst) {
    const int r = blockIdx.x * blockDim.x + threadIdx.x;
    if (r < n) dst[idx[r]] += w[r] * f;
}

}  // namespace

void pd_force_warp(const DevPD& d, const double* x, uint32_t* mask, int do_break,
                   unsigned long long* cnt, cudaStream_t s, double* Q, double* S,
                   const int32_t* colT, const double* coefT) {
    const int b = (int)(((long long)d.E * 32 + kT - 1) / kT);
    if (Q && S) {  // large subdomains: the per-element node products first (bitwise the same)
        if (d.dim == 2) {
            k_pd_elem_q<2><<<blocks(d.E), kT, 0, s>>>(d, x, Q, S);
            k_pd_force_warp_q<2><<<b, kT, 0, s>>>(d, mask, do_break, cnt, Q, S, colT, coefT);
        } else {
            k_pd_elem_q<3><<<blocks(d.E), kT, 0, s>>>(d, x, Q, S);
            k_pd_force_warp_q<3><<<b, kT, 0, s>>>(d, mask, do_break, cnt, Q, S, colT, coefT);
        }
    } else if (d.dim == 2) {
        k_pd_force_warp<2><<<b, kT, 0, s>>>(d, x, mask, do_break, cnt);
    } else {
        k_pd_force_warp<3><<<b, kT, 0, s>>>(d, x, mask, do_break, cnt);
    }
    check("pd_force_warp");
}
void pd_force_lin(const DevPD& d, const double* x, const uint32_t* mask, double* ubar,
                  cudaStream_t s) {
    if (d.dim == 2) {
        k_pd_ubar<2><<<blocks(d.E), kT, 0, s>>>(d, x, ubar);
        k_pd_force_lin<2><<<(int)(((long long)d.E * 32 + kT - 1) / kT), kT, 0, s>>>(d, ubar, mask);
    } else {
        k_pd_ubar<3><<<blocks(d.E), kT, 0, s>>>(d, x, ubar);
        k_pd_force_lin<3><<<(int)(((long long)d.E * 32 + kT - 1) / kT), kT, 0, s>>>(d, ubar, mask);
    }
    check("pd_force_lin");
}
void pd_ubar(const DevPD& d, const double* x, double* ubar, cudaStream_t s) {
    if (d.dim == 2) k_pd_ubar<2><<<blocks(d.E), kT, 0, s>>>(d, x, ubar);
    else k_pd_ubar<3><<<blocks(d.E), kT, 0, s>>>(d, x, ubar);
    check("pd_ubar");
}
void family_transpose(const DevPD& d, int32_t* colT, double* coefT, cudaStream_t s) {
    const long long n = (long long)d.E * d.K;
    const int b = (int)((n + kT - 1) / kT);
    if (d.dim == 2) k_family_transpose<2><<<b, kT, 0, s>>>(d, colT, coefT);
    else k_family_transpose<3><<<b, kT, 0, s>>>(d, colT, coefT);
    check("family_transpose");
}
void pd_force_lin_t(const DevPD& d, const int32_t* colT, const double* coefT, const double* x,
                    const uint32_t* mask, double* ubar, cudaStream_t s) {
    const int b = (int)(((long long)d.E * 32 + kT - 1) / kT);
    if (d.dim == 2) {
        k_pd_ubar<2><<<blocks(d.E), kT, 0, s>>>(d, x, ubar);
        k_pd_force_lin_t<2><<<b, kT, 0, s>>>(d, colT, coefT, ubar, mask);
    } else {
        k_pd_ubar<3><<<blocks(d.E), kT, 0, s>>>(d, x, ubar);
        k_pd_force_lin_t<3><<<b, kT, 0, s>>>(d, colT, coefT, ubar, mask);
    }
    check("pd_force_lin_t");
}
void pd_node_explicit(const DevPD& d, const double* ra, double ra_scale, const double* M,
                      const uint8_t* cf, const double* rv, const double* rd, double gdt,
                      double bdt2, const double* bcvel, int homog, double* u, double* v,
                      double* a, cudaStream_t s) {
    const int b = (d.N + kT - 1) / kT;
    if (d.dim == 2)
        k_pd_node_explicit<2><<<b, kT, 0, s>>>(d, ra, ra_scale, M, cf, rv, rd, gdt, bdt2, bcvel,
                                               homog, u, v, a);
    else
        k_pd_node_explicit<3><<<b, kT, 0, s>>>(d, ra, ra_scale, M, cf, rv, rd, gdt, bdt2, bcvel,
                                               homog, u, v, a);
    check("pd_node_explicit");
}
void pd_node_lin(const DevPD& d, int with_force, const double* w, const int32_t* row_of, double f,
                 const double* M, const uint8_t* cf, double gdt, double bdt2, double dt, double cpv,
                 double cpd, double* u, double* v, double* a, double* rd, double* rv, double* out,
                 cudaStream_t s) {
    const int b = (d.N + kT - 1) / kT;
    if (d.dim == 2)
        k_pd_node_lin<2><<<b, kT, 0, s>>>(d, with_force, w, row_of, f, M, cf, gdt, bdt2, dt, cpv,
                                          cpd, u, v, a, rd, rv, out);
    else
        k_pd_node_lin<3><<<b, kT, 0, s>>>(d, with_force, w, row_of, f, M, cf, gdt, bdt2, dt, cpv,
                                          cpd, u, v, a, rd, rv, out);
    check("pd_node_lin");
}
void pd_pre(int n, const double* u, const double* v, const double* a, double* rd, double* rv,
            double* ra, double dt, double cpv, double cpd, cudaStream_t s) {
    k_pd_pre<<<blocks(n), kT, 0, s>>>(n, u, v, a, rd, rv, ra, dt, cpv, cpd);
    check("pd_pre");
}
void scatter_scaled(int n, const int32_t* idx, const double* w, double f, double* dst,
                    cudaStream_t s) {
    if (n <= 0) return;
    k_scatter_scaled<<<blocks(n), kT, 0, s>>>(n, idx, w, f, dst);
    check("scatter_scaled");
}

void csr_spmv(int n, const int32_t* rp, const int32_t* ci, const double* v, const double* x,
              double* y, cudaStream_t s) {
    k_csr<<<blocks(n), kT, 0, s>>>(n, rp, ci, v, x, y);
    check("csr");
}
void predict(int n, const double* u, const double* v, const double* a, double* rd, double* rv,
             double dt, double cpv, double cpd, cudaStream_t s) {
    k_predict<<<blocks(n), kT, 0, s>>>(n, u, v, a, rd, rv, dt, cpv, cpd);
    check("predict");
}
void explicit_solve(int n, const double* ra, double ra_scale, const double* kd, const double* M,
                    const uint8_t* cf, const double* rv, const double* rd, double gdt, double bdt2,
                    const double* bcvel, int homog, double* u, double* v, double* a,
                    cudaStream_t s) {
    k_explicit<<<blocks(n), kT, 0, s>>>(n, ra, ra_scale, kd, M, cf, rv, rd, gdt, bdt2, bcvel,
                                        homog, u, v, a);
    check("explicit");
}
void rhs(int n, const double* ra, double ra_scale, const double* kd, const uint8_t* cf, double* b,
         cudaStream_t s) {
    k_rhs<<<blocks(n), kT, 0, s>>>(n, ra, ra_scale, kd, cf, b);
    check("rhs");
}
void apply_a(int n, const double* x, const double* kx, const double* M, const uint8_t* cf,
             double bdt2, double* y, cudaStream_t s) {
    k_apply_a<<<blocks(n), kT, 0, s>>>(n, x, kx, M, cf, bdt2, y);
    check("apply_a");
}
void finish(int n, const double* acc, const double* rv, const double* rd, double gdt, double bdt2,
            const uint8_t* cf, const double* bcvel, int homog, double* u, double* v, double* a,
            cudaStream_t s) {
    k_finish<<<blocks(n), kT, 0, s>>>(n, acc, rv, rd, gdt, bdt2, cf, bcvel, homog, u, v, a);
    check("finish");
}
void zero_constrained(int n, const uint8_t* cf, double* x, cudaStream_t s) {
    k_zero_cf<<<blocks(n), kT, 0, s>>>(n, cf, x);
    check("zero_cf");
}
void init_acc(int n, const double* p, const double* ku, const double* M, const uint8_t* cf,
              double* a, cudaStream_t s) {
    k_init_acc<<<blocks(n), kT, 0, s>>>(n, p, ku, M, cf, a);
    check("init_acc");
}
void scatter_add(int n, const int32_t* idx, const double* vals, double* dst, cudaStream_t s) {
    if (n <= 0) return;
    k_scatter_add<<<blocks(n), kT, 0, s>>>(n, idx, vals, dst);
    check("scatter_add");
}
void gather_csr(int n, const int32_t* rp, const int32_t* ci, const double* w, const double* src,
                double* dst, cudaStream_t s) {
    if (n <= 0) return;
    k_gather_csr<<<blocks(n), kT, 0, s>>>(n, rp, ci, w, src, dst);
    check("gather_csr");
}
void scatter_csr(int nt, const int32_t* td, const int32_t* trp, const int32_t* tri,
                 const double* tw, const double* vals, double* dst, cudaStream_t s) {
    if (nt <= 0) return;
    k_scatter_csr<<<blocks(nt), kT, 0, s>>>(nt, td, trp, tri, tw, vals, dst);
    check("scatter_csr");
}
void gather(int n, const int32_t* idx, const double* src, double* dst, cudaStream_t s) {
    if (n <= 0) return;
    k_gather<<<blocks(n), kT, 0, s>>>(n, idx, src, dst);
    check("gather");
}
void fill(long long n, double v, double* x, cudaStream_t s) {
    if (n <= 0) return;
    k_fill<<<(unsigned)((n + kT - 1) / kT), kT, 0, s>>>(n, v, x);
    check("fill");
}
void copy_idx(int n, const double* src, const int32_t* sidx, double* dst, const int32_t* didx,
              cudaStream_t s) {
    if (n <= 0) return;
    k_copy_idx<<<blocks(n), kT, 0, s>>>(n, src, sidx, dst, didx);
    check("copy_idx");
}
void scatter_set(int n, const int32_t* idx, const double* vals, double* dst, cudaStream_t s) {
    if (n <= 0) return;
    k_scatter_set<<<blocks(n), kT, 0, s>>>(n, idx, vals, dst);
    check("scatter_set");
}
void add(int n, const double* x, double* y, cudaStream_t s) {
    k_add<<<blocks(n), kT, 0, s>>>(n, x, y);
    check("add");
}
void scale(int n, const double* x, double sc, double* y, cudaStream_t s) {
    k_scale<<<blocks(n), kT, 0, s>>>(n, x, sc, y);
    check("scale");
}
void add_states(int n, const double* a0, const double* a1, const double* a2, const double* b0,
                const double* b1, const double* b2, double* o0, double* o1, double* o2,
                cudaStream_t s) {
    k_add3<<<blocks(n), kT, 0, s>>>(n, a0, a1, a2, b0, b1, b2, o0, o1, o2);
    check("add_states");
}
void cg_update(int n, const double* alpha_dev, const double* p, const double* ap, double* x,
               double* r, cudaStream_t s) {
    k_cg_update<<<blocks(n), kT, 0, s>>>(n, alpha_dev, p, ap, x, r);
    check("cg_update");
}
void precond(int n, const double* r, const double* jac, double* z, cudaStream_t s) {
    k_precond<<<blocks(n), kT, 0, s>>>(n, r, jac, z);
    check("precond");
}
void xpby(int n, const double* z, const double* beta_dev, double* p, cudaStream_t s) {
    k_xpby<<<blocks(n), kT, 0, s>>>(n, z, beta_dev, p);
    check("xpby");
}
int dot_partials() { return 148; }
void dot(int n, const double* x, const double* y, double* part, double* out, cudaStream_t s) {
    const int nb = dot_partials();
    k_dot_partial<<<nb, kT, 0, s>>>(n, x, y, part);
    k_sum_partials<<<1, kT, 0, s>>>(nb, part, out);
    check("dot");
}
void dot_fin(int n, const double* x, const double* y, const double* x2, const double* y2,
             double* part, unsigned* ticket, double* out, double* out2, int mode, double* num,
             double* sc, cudaStream_t s) {
    k_dot_fin<<<dot_partials(), kT, 0, s>>>(n, x, y, x2, y2, part, ticket, out, out2, mode, num, sc);
    check("dot_fin");
}
void cg_cond(cudaGraphConditionalHandle h, const double* s_bb, const double* s_rr,
             const double* s_pap, double tol, int max_iter, int* it_status, cudaStream_t s) {
    k_cg_cond<<<1, 1, 0, s>>>(h, s_bb, s_rr, s_pap, tol, max_iter, it_status);
    check("cg_cond");
}
void cg_update_precond(int n, const double* alpha_dev, const double* p, const double* ap,
                       double* x, double* r, const double* jac, double* z, cudaStream_t s) {
    k_cg_update_precond<<<blocks(n), kT, 0, s>>>(n, alpha_dev, p, ap, x, r, jac, z);
    check("cg_update_precond");
}
void ratio(const double* num, const double* den, double* out, cudaStream_t s) {
    k_ratio<<<1, 1, 0, s>>>(num, den, out);
    check("ratio");
}
void csr_spmv_warp(int n, const int32_t* rp, const int32_t* ci, const double* v, const double* x,
                   double* y, cudaStream_t s) {
    k_csr_warp<<<(n * 32 + kT - 1) / kT, kT, 0, s>>>(n, rp, ci, v, x, y);
    check("csr_warp");
}
void dense_matvec(int n, const double* A, const double* x, double* y, cudaStream_t s) {
    k_dense_matvec<<<(n * 32 + kT - 1) / kT, kT, 0, s>>>(n, A, x, y);
    check("dense_matvec");
}


// ---- the coupled step's bookkeeping on the device (mts.hpp:152-241, 309-317,
// 447-504): multiplier loads, interface rhs, energies, continuity, dense LU ----
namespace {

// LoadSpec ramp, driver.hpp:187-191: clamp(t / ramp, 0, 1) as std::clamp evaluates it
__device__ __forceinline__ double d_load_scale(double tt, double ramp) {
    if (ramp <= 0.0) return 1.0;
    const double x = tt / ramp;
    return x < 0.0 ? 0.0 : (1.0 < x ? 1.0 : x);
}

// S_j = (1 - w) lambda_prev + [ls(t + j dt) - (1 - w) ls(t) - w ls(t + dt_fe)] G P,
// w = j / m, for j = 1..m (mts.hpp:152-158), rows j - 1 of sv
__global__ void k_s_vectors(int nl, int m, double t, double dt_pd, double dt_fe, double ramp,
                            const double* lamp, const double* gpfe, double* sv) {
    const long long q = (long long)blockIdx.x * blockDim.x + threadIdx.x;
    if (q >= (long long)nl * m) return;
    const int j = (int)(q / nl) + 1, r = (int)(q % nl);
    const double w = double(j) / m;
    const double bracket = d_load_scale(t + j * dt_pd, ramp) - (1.0 - w) * d_load_scale(t, ramp) -
                           w * d_load_scale(t + dt_fe, ramp);
    sv[q] = (1.0 - w) * lamp[r] + bracket * gpfe[r];
}

__global__ void k_sub_idx(int n, const int32_t* idx, const double* x, double* b) {
    const int r = blockIdx.x * blockDim.x + threadIdx.x;
    if (r < n) b[r] = b[r] - x[idx[r]];
}
__global__ void k_neg(int n, const double* x, double* y) {
    const int i = blockIdx.x * blockDim.x + threadIdx.x;
    if (i < n) y[i] = -x[i];
}
__global__ void k_sub2(int n, const double* a, const double* b, double* o) {
    const int i = blockIdx.x * blockDim.x + threadIdx.x;
    if (i < n) o[i] = a[i] - b[i];
}
// the quadratic FE energy term's weights: M da + f K da
__global__ void k_quad_w(int n, const double* da, const double* M, double f, const double* kda,
                         double* w) {
    const int i = blockIdx.x * blockDim.x + threadIdx.x;
    if (i < n) w[i] = M[i] * da[i] + f * kda[i];
}
// lambda_pd terms of the energy record (mts.hpp:480-500): per (j, r), j = 1..m,
// A = vel_j - vel_{j-1}, B = lam_j - lam_{j-1}; S_0 = lambda_prev
__global__ void k_lpd_terms(int nl, int m, const double* gpf, const double* gpl, const double* sv,
                            const double* lamp, const double* lam, double* A, double* B) {
    const long long q = (long long)blockIdx.x * blockDim.x + threadIdx.x;
    if (q >= (long long)nl * m) return;
    const int j = (int)(q / nl) + 1, r = (int)(q % nl);
    const double vel_j = gpf[(size_t)j * nl + r] + gpl[(size_t)j * nl + r];
    const double vel_jm = gpf[(size_t)(j - 1) * nl + r] + (j > 1 ? gpl[(size_t)(j - 1) * nl + r] : 0.0);
    const double sj = sv[(size_t)(j - 1) * nl + r];
    const double sjm = j > 1 ? sv[(size_t)(j - 2) * nl + r] : lamp[r];
    const double lam_j = sj + (double(j) / m) * lam[r];
    const double lam_jm = sjm + (double(j - 1) / m) * lam[r];
    A[q] = vel_j - vel_jm;
    B[q] = lam_j - lam_jm;
}
// max |x| (or max |x - y[idx]| with idx) into *out as the bits of a non-negative
// double (they order like the values): order-independent, exact
__global__ void k_max_abs(int n, const double* x, const int32_t* idx, const double* y,
                          unsigned long long* out) {
    unsigned long long m = 0ull;
    for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < n; i += gridDim.x * blockDim.x) {
        const double v = idx ? fabs(x[i] - y[idx[i]]) : fabs(x[i]);
        m = max(m, (unsigned long long)__double_as_longlong(v));
    }
    for (int o = 16; o > 0; o >>= 1) m = max(m, __shfl_down_sync(0xffffffffu, m, o));
    if ((threadIdx.x & 31) == 0) atomicMax(out, m);
}

// DenseLu (linalg.hpp:368-412) on the device: partial pivoting with the host
// restatement's order of operations (-fmad=false: bitwise its factor).
// One column step = k_lu_pivot (one block: argmax |a_ik|, i >= k, first index on
// ties; singularity flag; row swap) + k_lu_col (multipliers) + k_lu_update.
__global__ void k_lu_pivot(int n, int k, double* A, int* perm, const unsigned long long* amax,
                           int* flag) {
    __shared__ double bv[1024];
    __shared__ int bi[1024];
    double best = -1.0;
    int piv = n;
    for (int i = k + threadIdx.x; i < n; i += blockDim.x) {
        const double v = fabs(A[(size_t)i * n + k]);
        if (v > best) {
            best = v;
            piv = i;
        }
    }
    bv[threadIdx.x] = best;
    bi[threadIdx.x] = piv;
    __syncthreads();
    for (int o = blockDim.x / 2; o > 0; o >>= 1) {
        if ((int)threadIdx.x < o) {
            const double v2 = bv[threadIdx.x + o];
            const int i2 = bi[threadIdx.x + o];
            if (v2 > bv[threadIdx.x] || (v2 == bv[threadIdx.x] && i2 < bi[threadIdx.x])) {
                bv[threadIdx.x] = v2;
                bi[threadIdx.x] = i2;
            }
        }
        __syncthreads();
    }
    const double thr = 1e-14 * fmax(__longlong_as_double((long long)*amax), 1e-300);
    const int p = bi[0];
    if (bv[0] <= thr) {
        if (threadIdx.x == 0) *flag = 1;
        return;
    }
    if (p != k) {
        for (int j = threadIdx.x; j < n; j += blockDim.x) {
            const double a = A[(size_t)k * n + j];
            A[(size_t)k * n + j] = A[(size_t)p * n + j];
            A[(size_t)p * n + j] = a;
        }
        if (threadIdx.x == 0) {
            const int t = perm[k];
            perm[k] = perm[p];
            perm[p] = t;
        }
    }
}
__global__ void k_lu_col(int n, int k, double* A, const int* flag) {
    const int i = k + 1 + blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= n || *flag) return;
    const double inv = 1.0 / A[(size_t)k * n + k];
    A[(size_t)i * n + k] = A[(size_t)i * n + k] * inv;
}
__global__ void k_lu_update(int n, int k, double* A, const int* flag) {
    const int j = k + 1 + blockIdx.x * blockDim.x + threadIdx.x;
    const int i = k + 1 + blockIdx.y;
    if (j >= n || i >= n || *flag) return;
    const double f = A[(size_t)i * n + k];
    if (f == 0.0) return;
    A[(size_t)i * n + j] -= f * A[(size_t)k * n + j];
}
// x = A^-1 b from the factor: the forward substitution accumulates each x_i over
// ascending j like the host's row loop (bitwise); the backward one is column-
// oriented (subtracting j descending: rounding-level differences from the host).
// One block; x in global memory (n of any size)
__global__ void k_lu_solve(int n, const double* A, const int* perm, const double* b, double* x) {
    for (int i = threadIdx.x; i < n; i += blockDim.x) x[i] = b[perm[i]];
    __syncthreads();
    for (int j = 0; j + 1 < n; ++j) {
        const double xj = x[j];
        for (int i = j + 1 + threadIdx.x; i < n; i += blockDim.x)
            x[i] = x[i] - A[(size_t)i * n + j] * xj;
        __syncthreads();
    }
    for (int jj = n - 1; jj >= 0; --jj) {
        if (threadIdx.x == 0) x[jj] = x[jj] / A[(size_t)jj * n + jj];
        __syncthreads();
        const double xj = x[jj];
        for (int i = threadIdx.x; i < jj; i += blockDim.x) x[i] = x[i] - A[(size_t)i * n + jj] * xj;
        __syncthreads();
    }
}

// the loop test before the first CG iteration (cg_solve, linalg.hpp:251-262): b = 0
// -> x = 0, converged; else continue while sqrt(rr) / sqrt(bb) > tol (past max_iter
// -> status 2); sets the WHILE node's condition and resets the iteration count
__global__ void k_cg_start(cudaGraphConditionalHandle h, const double* s_bb, const double* s_rr,
                           double tol, int max_iter, int* it_status, double* x, int n,
                           int* more_out) {
    const double bb = *s_bb;
    const int i = blockIdx.x * blockDim.x + threadIdx.x;
    if (bb == 0.0 && i < n) x[i] = 0.0;
    if (i != 0) return;
    it_status[0] = 0;
    it_status[1] = 0;
    bool more = false;
    if (bb != 0.0) {
        more = sqrt(*s_rr) / sqrt(bb) > tol;
        if (more && max_iter <= 0) {
            it_status[1] = 2;
            more = false;
        }
    }
    if (more_out) *more_out = more ? 1 : 0;  // host-driven loop (sharded coupled runs)
    else cudaGraphSetConditional(h, more ? 1u : 0u);
}

// dense column k of a column-major n x n matrix: D[k n + r] = -x[r]  (H_FE unit columns)
__global__ void k_col_neg(int n, int k, const double* x, double* D) {
    const int r = blockIdx.x * blockDim.x + threadIdx.x;
    if (r < n) D[(size_t)k * n + r] = -x[r];
}
// row-major H[r n + k] += x[cpd[r]] (the PD unit responses of the dense interface)
__global__ void k_add_col_gather(int n, int k, const int32_t* idx, const double* x, double* H) {
    const int r = blockIdx.x * blockDim.x + threadIdx.x;
    if (r < n) H[(size_t)r * n + k] += x[idx[r]];
}
// the unit load of coupling row k on the FE side: ra = 0 except ra[ci_j] = -w_j
__global__ void k_unit_row(int nf, const int32_t* rp, const int32_t* ci, const double* w, int k,
                           double* ra) {
    const int i = blockIdx.x * blockDim.x + threadIdx.x;
    if (i < nf) ra[i] = 0.0;
}
__global__ void k_unit_row_set(const int32_t* rp, const int32_t* ci, const double* w, int k,
                               double* ra) {
    for (int j = rp[k] + threadIdx.x; j < rp[k + 1]; j += blockDim.x) ra[ci[j]] = -w[j];
}
__global__ void k_unit_vec(int n, int k, double* x) {
    const int i = blockIdx.x * blockDim.x + threadIdx.x;
    if (i < n) x[i] = i == k ? 1.0 : 0.0;
}
// column-major dense (n x n) -> row-major dense
__global__ void k_transpose(int n, const double* D, double* H) {
    const long long q = (long long)blockIdx.x * blockDim.x + threadIdx.x;
    if (q >= (long long)n * n) return;
    const int r = (int)(q / n), k = (int)(q % n);
    H[q] = D[(size_t)k * n + r];
}
// nonzeros of row r of the column-major D (ascending k), count then fill
__global__ void k_row_nnz(int n, const double* D, int* cnt) {
    const int r = blockIdx.x * blockDim.x + threadIdx.x;
    if (r > n) return;
    if (r == n) {
        cnt[n] = 0;
        return;
    }
    int c = 0;
    for (int k = 0; k < n; ++k) c += D[(size_t)k * n + r] != 0.0 ? 1 : 0;
    cnt[r] = c;
}
__global__ void k_row_fill(int n, const double* D, const int* rp, int32_t* ci, double* v) {
    const int r = blockIdx.x * blockDim.x + threadIdx.x;
    if (r >= n) return;
    int q = rp[r];
    for (int k = 0; k < n; ++k) {
        const double x = D[(size_t)k * n + r];
        if (x != 0.0) {
            ci[q] = k;
            v[q] = x;
            ++q;
        }
    }
}
// H_FE of an explicit FE side as a sparse product, entry by entry bitwise the unit-column
// construction (unit_row -> explicit solve -> G_FE gather -> negate; build_h_fe): column
// k's FE velocity is vel_k[d] = 0 + gdt ((-w_kd) / M_d) on the unconstrained dofs of row
// k and +0 elsewhere, and row r's gather sums w_rj vel_k[ci_j] left to right -- the zero
// terms change no nonzero partial sum, so only the shared dofs are visited.  Warp per
// row; candidates (rows sharing an unconstrained FE dof with r) ascending.
__global__ void k_hfe_explicit(int nl, const long long* crp, const int32_t* cci,
                               const int32_t* grp, const int32_t* gci, const double* gw,
                               const double* M, const uint8_t* cf, double gdt, double* vals) {
    const int r = (int)(((long long)blockIdx.x * blockDim.x + threadIdx.x) >> 5);
    const int lane = threadIdx.x & 31;
    if (r >= nl) return;
    const int j0 = grp[r], j1 = grp[r + 1];
    for (long long q = crp[r] + lane; q < crp[r + 1]; q += 32) {
        const int k = cci[q];
        const int k0 = grp[k], k1 = grp[k + 1];
        double acc = 0.0;
        for (int j = j0; j < j1; ++j) {
            const int d = gci[j];
            if (cf[d]) continue;
            for (int i = k0; i < k1; ++i)
                if (gci[i] == d) {
                    const double x = 0.0 + gdt * ((-gw[i]) / M[d]);
                    if (x != 0.0) acc = acc + gw[j] * x;
                    break;
                }
        }
        vals[q] = -acc;
    }
}
__global__ void k_nz_count(int n, const long long* rp, const double* v, int* cnt) {
    const int r = blockIdx.x * blockDim.x + threadIdx.x;
    if (r > n) return;
    if (r == n) {
        cnt[n] = 0;
        return;
    }
    int c = 0;
    for (long long q = rp[r]; q < rp[r + 1]; ++q) c += v[q] != 0.0 ? 1 : 0;
    cnt[r] = c;
}
__global__ void k_nz_fill(int n, const long long* rp, const int32_t* ci, const double* v,
                          const int32_t* orp, int32_t* oci, double* ov) {
    const int r = blockIdx.x * blockDim.x + threadIdx.x;
    if (r >= n) return;
    int o = orp[r];
    for (long long q = rp[r]; q < rp[r + 1]; ++q)
        if (v[q] != 0.0) {
            oci[o] = ci[q];
            ov[o] = v[q];
            ++o;
        }
}

// Jacobi preconditioner of the interface CG: diag(H_FE) + m dt / (2 M_PD)
__global__ void k_iface_jac(int n, const double* D, int m, double dt_pd, const int32_t* cpd,
                            const double* Mpd, double* jd) {
    const int r = blockIdx.x * blockDim.x + threadIdx.x;
    if (r >= n) return;
    double v = D[(size_t)r * n + r] + double(m) * dt_pd / (2.0 * Mpd[cpd[r]]);
    if (!(v > 0.0)) v = 0.0;
    jd[r] = v;
}

// the same from H_FE in CSR (a missing diagonal entry reads 0, as in the dense form)
__global__ void k_iface_jac_csr(int n, const int32_t* rp, const int32_t* ci, const double* hv,
                                int m, double dt_pd, const int32_t* cpd, const double* Mpd,
                                double* jd) {
    const int r = blockIdx.x * blockDim.x + threadIdx.x;
    if (r >= n) return;
    double dg = 0.0;
    for (int q = rp[r]; q < rp[r + 1]; ++q)
        if (ci[q] == r) dg = hv[q];
    double v = dg + double(m) * dt_pd / (2.0 * Mpd[cpd[r]]);
    if (!(v > 0.0)) v = 0.0;
    jd[r] = v;
}

}  // namespace

void iface_jac_csr(int n, const int32_t* rp, const int32_t* ci, const double* hv, int m,
                   double dt_pd, const int32_t* cpd, const double* Mpd, double* jd,
                   cudaStream_t s) {
    k_iface_jac_csr<<<blocks(n), kT, 0, s>>>(n, rp, ci, hv, m, dt_pd, cpd, Mpd, jd);
    check("iface_jac_csr");
}

void s_vectors(int nl, int m, double t, double dt_pd, double dt_fe, double ramp,
               const double* lamp, const double* gpfe, double* sv, cudaStream_t s) {
    k_s_vectors<<<blocks((long long)nl * m), kT, 0, s>>>(nl, m, t, dt_pd, dt_fe, ramp, lamp, gpfe, sv);
    check("s_vectors");
}
void sub_idx(int n, const int32_t* idx, const double* x, double* b, cudaStream_t s) {
    k_sub_idx<<<blocks(n), kT, 0, s>>>(n, idx, x, b);
    check("sub_idx");
}
void neg(int n, const double* x, double* y, cudaStream_t s) {
    k_neg<<<blocks(n), kT, 0, s>>>(n, x, y);
    check("neg");
}
void sub2(int n, const double* a, const double* b, double* o, cudaStream_t s) {
    k_sub2<<<blocks(n), kT, 0, s>>>(n, a, b, o);
    check("sub2");
}
void quad_w(int n, const double* da, const double* M, double f, const double* kda, double* w,
            cudaStream_t s) {
    k_quad_w<<<blocks(n), kT, 0, s>>>(n, da, M, f, kda, w);
    check("quad_w");
}
void lpd_terms(int nl, int m, const double* gpf, const double* gpl, const double* sv,
               const double* lamp, const double* lam, double* A, double* B, cudaStream_t s) {
    k_lpd_terms<<<blocks((long long)nl * m), kT, 0, s>>>(nl, m, gpf, gpl, sv, lamp, lam, A, B);
    check("lpd_terms");
}
void max_abs(int n, const double* x, const int32_t* idx, const double* y,
             unsigned long long* out, cudaStream_t s) {
    if (n <= 0) return;
    k_max_abs<<<std::min(blocks(n), 592), kT, 0, s>>>(n, x, idx, y, out);
    check("max_abs");
}
void lu_factor(int n, double* A, int* perm, unsigned long long* amax, int* flag, cudaStream_t s) {
    k_max_abs<<<std::min(blocks((long long)n * n), 2048), kT, 0, s>>>(n * n, A, nullptr, nullptr, amax);
    for (int k = 0; k < n; ++k) {
        k_lu_pivot<<<1, 1024, 0, s>>>(n, k, A, perm, amax, flag);
        const int rest = n - k - 1;
        if (rest > 0) {
            k_lu_col<<<blocks(rest), kT, 0, s>>>(n, k, A, flag);
            k_lu_update<<<dim3(blocks(rest), rest), kT, 0, s>>>(n, k, A, flag);
        }
    }
    check("lu_factor");
}
void lu_solve(int n, const double* A, const int* perm, const double* b, double* x, cudaStream_t s) {
    k_lu_solve<<<1, 1024, 0, s>>>(n, A, perm, b, x);
    check("lu_solve");
}
void cg_start(cudaGraphConditionalHandle h, const double* s_bb, const double* s_rr, double tol,
              int max_iter, int* it_status, double* x, int n, cudaStream_t s, int* more_out) {
    k_cg_start<<<blocks(std::max(n, 1)), kT, 0, s>>>(h, s_bb, s_rr, tol, max_iter, it_status, x, n,
                                                     more_out);
    check("cg_start");
}
void col_neg(int n, int k, const double* x, double* D, cudaStream_t s) {
    k_col_neg<<<blocks(n), kT, 0, s>>>(n, k, x, D);
    check("col_neg");
}
void add_col_gather(int n, int k, const int32_t* idx, const double* x, double* H, cudaStream_t s) {
    k_add_col_gather<<<blocks(n), kT, 0, s>>>(n, k, idx, x, H);
    check("add_col_gather");
}
void unit_row(int nf, const int32_t* rp, const int32_t* ci, const double* w, int k, double* ra,
              cudaStream_t s) {
    k_unit_row<<<blocks(nf), kT, 0, s>>>(nf, rp, ci, w, k, ra);
    k_unit_row_set<<<1, 32, 0, s>>>(rp, ci, w, k, ra);
    check("unit_row");
}
void unit_vec(int n, int k, double* x, cudaStream_t s) {
    k_unit_vec<<<blocks(n), kT, 0, s>>>(n, k, x);
    check("unit_vec");
}
void hfe_explicit(int nl, const long long* crp, const int32_t* cci, const int32_t* grp,
                  const int32_t* gci, const double* gw, const double* M, const uint8_t* cf,
                  double gdt, double* vals, cudaStream_t s) {
    if (nl <= 0) return;
    k_hfe_explicit<<<(unsigned)(((long long)nl * 32 + kT - 1) / kT), kT, 0, s>>>(
        nl, crp, cci, grp, gci, gw, M, cf, gdt, vals);
    check("hfe_explicit");
}
void nz_count(int n, const long long* rp, const double* v, int* cnt, cudaStream_t s) {
    k_nz_count<<<blocks(n + 1), kT, 0, s>>>(n, rp, v, cnt);
    check("nz_count");
}
void nz_fill(int n, const long long* rp, const int32_t* ci, const double* v, const int32_t* orp,
             int32_t* oci, double* ov, cudaStream_t s) {
    if (n <= 0) return;
    k_nz_fill<<<blocks(n), kT, 0, s>>>(n, rp, ci, v, orp, oci, ov);
    check("nz_fill");
}
void transpose(int n, const double* D, double* H, cudaStream_t s) {
    k_transpose<<<blocks((long long)n * n), kT, 0, s>>>(n, D, H);
    check("transpose");
}
void row_nnz(int n, const double* D, int* cnt, cudaStream_t s) {
    k_row_nnz<<<blocks(n + 1), kT, 0, s>>>(n, D, cnt);
    check("row_nnz");
}
void row_fill(int n, const double* D, const int* rp, int32_t* ci, double* v, cudaStream_t s) {
    k_row_fill<<<blocks(n), kT, 0, s>>>(n, D, rp, ci, v);
    check("row_fill");
}
void iface_jac(int n, const double* D, int m, double dt_pd, const int32_t* cpd, const double* Mpd,
               double* jd, cudaStream_t s) {
    k_iface_jac<<<blocks(n), kT, 0, s>>>(n, D, m, dt_pd, cpd, Mpd, jd);
    check("iface_jac");
}


// ---- batched CG: B independent solves of the implicit FE block at once -- the unit
// columns of H_FE (mts.hpp:389-397).  Column c of every vector is [c nf, (c + 1) nf);
// each column runs cg_solve's arithmetic (the single-solve kernels' expressions, its
// own scalars, loop test and iteration count); finished columns stop updating.
// Per-column scalars: sc[8 c + {0 bb, 1 rz, 2 rr, 3 pap, 4 alpha, 5 beta}];
// act[c] = 1 while iterating; stat[2 c] = iterations, stat[2 c + 1] = status.
namespace {
constexpr int kBNB = 64;  // dot partial blocks per column

__global__ void k_bunit_rhs(int nf, int k0, int nl, const int32_t* rp, const int32_t* ci,
                            const double* w, const uint8_t* cf, double* b) {
    const int c = blockIdx.x, k = k0 + c;
    if (k >= nl) return;
    for (int j = rp[k] + threadIdx.x; j < rp[k + 1]; j += blockDim.x) {
        const int i = ci[j];
        const double ra = -w[j];  // unit_row: ra = -w; rhs: ra * 1 - K 0
        b[(size_t)c * nf + i] = cf[i] ? 0.0 : ra * 1.0 - 0.0;
    }
}
// r = b - A 0 = b, z = precond(r), p = z
__global__ void k_binit(long long n, const double* b, const double* jac, int nf, double* r,
                        double* z, double* p) {
    const long long q = (long long)blockIdx.x * blockDim.x + threadIdx.x;
    if (q >= n) return;
    const int i = (int)(q % nf);
    const double ri = b[q] - 0.0;
    r[q] = ri;
    const double zi = jac ? (jac[i] != 0.0 ? ri / jac[i] : ri) : ri;
    z[q] = zi;
    p[q] = zi;
}
// block partials of x.y (and x2.y2) over column c = blockIdx.y
__global__ void __launch_bounds__(kT) k_bdot(int nf, const double* x, const double* y,
                                             const double* x2, const double* y2, const int* act,
                                             double* part) {
    const int c = blockIdx.y;
    if (act && !act[c]) return;
    __shared__ double sh[kT], sh2[kT];
    const size_t o = (size_t)c * nf;
    double s = 0.0, s2 = 0.0;
    for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < nf; i += gridDim.x * blockDim.x) {
        s += x[o + i] * y[o + i];
        if (x2) s2 += x2[o + i] * y2[o + i];
    }
    sh[threadIdx.x] = s;
    sh2[threadIdx.x] = s2;
    __syncthreads();
    for (int k = kT / 2; k > 0; k >>= 1) {
        if ((int)threadIdx.x < k) {
            sh[threadIdx.x] += sh[threadIdx.x + k];
            sh2[threadIdx.x] += sh2[threadIdx.x + k];
        }
        __syncthreads();
    }
    if (threadIdx.x == 0) {
        part[((size_t)c * gridDim.x + blockIdx.x) * 2] = sh[0];
        part[((size_t)c * gridDim.x + blockIdx.x) * 2 + 1] = sh2[0];
    }
}
// per column (block c): the partial sums, then
//   mode 0: bb, rz;  mode 1: rr and the start test;  mode 2: pap -> alpha (or status 1);
//   mode 3: rz_new, rr -> beta, rz <- rz_new, the loop test
__global__ void k_bfin(int nb, int mode, const double* part, double* sc, int* act, int* stat,
                       double tol, int max_iter, int* n_active) {
    const int c = blockIdx.x;
    if (mode >= 2 && !act[c]) return;
    __shared__ double sh[32], sh2[32];
    double t = 0.0, t2 = 0.0;
    for (int k = threadIdx.x; k < nb; k += 32) {
        t += part[((size_t)c * nb + k) * 2];
        t2 += part[((size_t)c * nb + k) * 2 + 1];
    }
    sh[threadIdx.x] = t;
    sh2[threadIdx.x] = t2;
    __syncwarp();
    if (threadIdx.x != 0) return;
    double s1 = 0.0, s2 = 0.0;
    for (int k = 0; k < 32; ++k) {
        s1 += sh[k];
        s2 += sh2[k];
    }
    double* q = sc + 8 * c;
    if (mode == 0) {
        q[0] = s1;
        q[1] = s2;
    } else if (mode == 1) {
        q[2] = s1;
        stat[2 * c] = 0;
        stat[2 * c + 1] = 0;
        bool more = false;
        if (q[0] != 0.0) {
            more = sqrt(s1) / sqrt(q[0]) > tol;
            if (more && max_iter <= 0) {
                stat[2 * c + 1] = 2;
                more = false;
            }
        }
        act[c] = more ? 1 : 0;
        if (more) atomicAdd(n_active, 1);
    } else if (mode == 2) {
        q[3] = s1;
        if (s1 <= 0.0) {
            stat[2 * c + 1] = 1;
            act[c] = 0;
            return;
        }
        q[4] = q[1] / s1;
    } else {
        q[5] = s1 / q[1];
        q[1] = s1;
        q[2] = s2;
        const int it = ++stat[2 * c];
        bool more = sqrt(s2) / sqrt(q[0]) > tol;
        if (more && it >= max_iter) {
            stat[2 * c + 1] = 2;
            more = false;
        }
        act[c] = more ? 1 : 2;  // 2: finished this iteration (p still updated below)
        if (more) atomicAdd(n_active, 1);
    }
}
// ap = A p for every active column: K p (CSR, the row read once for all columns)
// and apply_a's M p + bdt2 K p
__global__ void k_bspmm(int nf, int B, const int32_t* __restrict__ rp, const int32_t* __restrict__ ci,
                        const double* __restrict__ v, const double* M, const uint8_t* cf,
                        double bdt2, const int* act, const double* P, double* AP) {
    const int i = blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= nf) return;
    const int p0 = rp[i], p1 = rp[i + 1];
    for (int c = 0; c < B; ++c) {
        if (act[c] != 1) continue;
        const size_t o = (size_t)c * nf;
        double s = 0.0;
        for (int p = p0; p < p1; ++p) s += v[p] * P[o + ci[p]];
        AP[o + i] = cf[i] ? P[o + i] : M[i] * P[o + i] + bdt2 * s;
    }
}
// x += alpha p; r -= alpha ap; z = precond(r)
__global__ void k_bupdate(long long n, int nf, const double* sc, const int* act, const double* P,
                          const double* AP, double* X, double* R, const double* jac, double* Z) {
    const long long q = (long long)blockIdx.x * blockDim.x + threadIdx.x;
    if (q >= n) return;
    const int c = (int)(q / nf), i = (int)(q % nf);
    if (act[c] != 1) return;
    const double al = sc[8 * c + 4];
    X[q] += al * P[q];
    const double ri = R[q] + -al * AP[q];
    R[q] = ri;
    Z[q] = jac ? (jac[i] != 0.0 ? ri / jac[i] : ri) : ri;
}
// p = z + beta p (columns that ran this iteration, finished ones included)
__global__ void k_bxpby(long long n, int nf, const double* sc, int* act, const double* Z,
                        double* P) {
    const long long q = (long long)blockIdx.x * blockDim.x + threadIdx.x;
    if (q >= n) return;
    const int c = (int)(q / nf);
    if (act[c] == 0) return;
    P[q] = Z[q] + sc[8 * c + 5] * P[q];
}
__global__ void k_bact_settle(int B, int* act) {
    const int c = blockIdx.x * blockDim.x + threadIdx.x;
    if (c < B && act[c] == 2) act[c] = 0;
}
// finish (homogeneous: v = 0 + gdt acc, constrained 0) + G_FE gather, negated into
// column k0 + c of the column-major nl x nl D
__global__ void k_bgather(int nl, int nf, int k0, int B, const int32_t* rp, const int32_t* ci,
                          const double* w, const uint8_t* cf, double gdt, const double* X,
                          double* D) {
    const long long q = (long long)blockIdx.x * blockDim.x + threadIdx.x;
    if (q >= (long long)nl * B) return;
    const int c = (int)(q / nl), r = (int)(q % nl);
    if (k0 + c >= nl) return;
    const size_t o = (size_t)c * nf;
    auto vel = [&](int i) { return cf[i] ? 0.0 : 0.0 + gdt * X[o + i]; };
    int j = rp[r];
    double acc = w[j] * vel(ci[j]);
    for (++j; j < rp[r + 1]; ++j) acc += w[j] * vel(ci[j]);
    D[(size_t)(k0 + c) * nl + r] = -acc;
}
}  // namespace

// the unit columns k0 .. k0 + B - 1 of H_FE (implicit FE) into D; scratch: 6 B nf
// doubles (b, x, r, z, p, ap), part (2 kBNB B doubles), sc (8 B), act/stat/n_active
// ints; returns 0, or the first failing column's status (1 not SPD, 2 no convergence)
int batched_unit_columns(int nf, int nl, int k0, int B, const int32_t* krp, const int32_t* kci,
                         const double* kv, const double* M, const uint8_t* cf, const double* jac,
                         double bdt2, double gdt, const int32_t* grp, const int32_t* gci,
                         const double* gw, double tol, int max_iter, double* scratch, double* part,
                         double* sc, int* act, int* stat, int* n_active, int* h_count, double* D,
                         int* iters_out, cudaStream_t s) {
    const long long n = (long long)B * nf;
    double *b = scratch, *x = b + n, *r = x + n, *z = r + n, *p = z + n, *ap = p + n;
    cudaMemsetAsync(b, 0, sizeof(double) * n, s);
    cudaMemsetAsync(x, 0, sizeof(double) * n, s);
    k_bunit_rhs<<<B, 32, 0, s>>>(nf, k0, nl, grp, gci, gw, cf, b);
    k_binit<<<blocks(n), kT, 0, s>>>(n, b, jac, nf, r, z, p);
    cudaMemsetAsync(n_active, 0, sizeof(int), s);
    const dim3 dg(kBNB, B);
    k_bdot<<<dg, kT, 0, s>>>(nf, b, b, r, z, nullptr, part);
    k_bfin<<<B, 32, 0, s>>>(kBNB, 0, part, sc, act, stat, tol, max_iter, n_active);
    k_bdot<<<dg, kT, 0, s>>>(nf, r, r, nullptr, nullptr, nullptr, part);
    k_bfin<<<B, 32, 0, s>>>(kBNB, 1, part, sc, act, stat, tol, max_iter, n_active);
    int it = 0;
    for (;;) {
        cudaMemcpyAsync(h_count, n_active, sizeof(int), cudaMemcpyDeviceToHost, s);
        cudaStreamSynchronize(s);
        if (*h_count == 0) break;
        cudaMemsetAsync(n_active, 0, sizeof(int), s);
        k_bspmm<<<blocks(nf), kT, 0, s>>>(nf, B, krp, kci, kv, M, cf, bdt2, act, p, ap);
        k_bdot<<<dg, kT, 0, s>>>(nf, p, ap, nullptr, nullptr, act, part);
        k_bfin<<<B, 32, 0, s>>>(kBNB, 2, part, sc, act, stat, tol, max_iter, n_active);
        k_bupdate<<<blocks(n), kT, 0, s>>>(n, nf, sc, act, p, ap, x, r, jac, z);
        k_bdot<<<dg, kT, 0, s>>>(nf, r, z, r, r, act, part);
        k_bfin<<<B, 32, 0, s>>>(kBNB, 3, part, sc, act, stat, tol, max_iter, n_active);
        k_bxpby<<<blocks(n), kT, 0, s>>>(n, nf, sc, act, z, p);
        k_bact_settle<<<1, 1024, 0, s>>>(B, act);
        ++it;
    }
    std::vector<int> st(2 * B);
    cudaMemcpyAsync(st.data(), stat, sizeof(int) * 2 * B, cudaMemcpyDeviceToHost, s);
    cudaStreamSynchronize(s);
    int bad = 0, mx = 0;
    for (int c = 0; c < B && k0 + c < nl; ++c) {
        mx = std::max(mx, st[2 * c]);
        if (st[2 * c + 1] && !bad) bad = st[2 * c + 1];
    }
    if (!bad)
        k_bgather<<<blocks((long long)nl * B), kT, 0, s>>>(nl, nf, k0, B, grp, gci, gw, cf, gdt, x, D);
    check("batched_unit_columns");
    if (iters_out) *iters_out = mx;
    return bad;
}
int batched_partials() { return kBNB; }


namespace {
__global__ void k_set_ones(int n, const int32_t* idx, double* x) {
    const int i = blockIdx.x * blockDim.x + threadIdx.x;
    if (i < n) x[idx[i]] = 1.0;
}
__global__ void k_gather_slots(int n, const int32_t* rows, const int64_t* slots, const double* g,
                               double* dst) {
    const int i = blockIdx.x * blockDim.x + threadIdx.x;
    if (i < n) dst[slots[i]] = g[rows[i]];
}
}  // namespace
void set_ones(int n, const int32_t* idx, double* x, cudaStream_t s) {
    if (n <= 0) return;
    k_set_ones<<<blocks(n), kT, 0, s>>>(n, idx, x);
    check("set_ones");
}
void gather_slots(int n, const int32_t* rows, const int64_t* slots, const double* g, double* dst,
                  cudaStream_t s) {
    if (n <= 0) return;
    k_gather_slots<<<blocks(n), kT, 0, s>>>(n, rows, slots, g, dst);
    check("gather_slots");
}


// ---- H = H_FE + H_PD as one CSR (the sparse interface operator): per row the
// union of the two sorted column lists, values summed where both have the entry ----
namespace {
__global__ void k_merge_count(int n, const int32_t* arp, const int32_t* aci, const int32_t* brp,
                              const int32_t* bci, int* cnt) {
    const int r = blockIdx.x * blockDim.x + threadIdx.x;
    if (r > n) return;
    if (r == n) {
        cnt[n] = 0;
        return;
    }
    int i = arp[r], j = brp[r], c = 0;
    const int ie = arp[r + 1], je = brp[r + 1];
    while (i < ie || j < je) {
        const int x = i < ie ? aci[i] : INT_MAX, y = j < je ? bci[j] : INT_MAX;
        i += x <= y;
        j += y <= x;
        ++c;
    }
    cnt[r] = c;
}
__global__ void k_merge_fill(int n, const int32_t* arp, const int32_t* aci, const double* av,
                             const int32_t* brp, const int32_t* bci, const double* bv,
                             const int32_t* rp, int32_t* ci, double* v) {
    const int r = blockIdx.x * blockDim.x + threadIdx.x;
    if (r >= n) return;
    int i = arp[r], j = brp[r], q = rp[r];
    const int ie = arp[r + 1], je = brp[r + 1];
    while (i < ie || j < je) {
        const int x = i < ie ? aci[i] : INT_MAX, y = j < je ? bci[j] : INT_MAX;
        double val;
        if (x < y) val = av[i++];
        else if (y < x) val = bv[j++];
        else val = av[i++] + bv[j++];
        ci[q] = x < y ? x : y;
        v[q] = val;
        ++q;
    }
}
__global__ void k_csr_diag(int n, const int32_t* rp, const int32_t* ci, const double* v,
                           double* d) {
    const int r = blockIdx.x * blockDim.x + threadIdx.x;
    if (r >= n) return;
    double x = 0.0;
    for (int q = rp[r]; q < rp[r + 1]; ++q)
        if (ci[q] == r) x = v[q];
    d[r] = x > 0.0 ? x : 0.0;
}
}  // namespace
void merge_count(int n, const int32_t* arp, const int32_t* aci, const int32_t* brp,
                 const int32_t* bci, int* cnt, cudaStream_t s) {
    k_merge_count<<<blocks(n + 1), kT, 0, s>>>(n, arp, aci, brp, bci, cnt);
    check("merge_count");
}
void merge_fill(int n, const int32_t* arp, const int32_t* aci, const double* av, const int32_t* brp,
                const int32_t* bci, const double* bv, const int32_t* rp, int32_t* ci, double* v,
                cudaStream_t s) {
    k_merge_fill<<<blocks(n), kT, 0, s>>>(n, arp, aci, av, brp, bci, bv, rp, ci, v);
    check("merge_fill");
}
void csr_diag(int n, const int32_t* rp, const int32_t* ci, const double* v, double* d,
              cudaStream_t s) {
    k_csr_diag<<<blocks(n), kT, 0, s>>>(n, rp, ci, v, d);
    check("csr_diag");
}


// ---- fused CG stages (bitwise the separate kernels they replace) ----
namespace {
// the implicit FE operator in one pass: y = cf ? x : M x + bdt2 (K x) (k_csr + k_apply_a)
__global__ void k_csr_apply_a(int n, const int32_t* __restrict__ rp, const int32_t* __restrict__ ci,
                              const double* __restrict__ v, const double* __restrict__ x,
                              const double* M, const uint8_t* cf, double bdt2, double* y) {
    const int i = blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= n) return;
    double s = 0.0;
    for (int p = rp[i]; p < rp[i + 1]; ++p) s += v[p] * x[ci[p]];
    y[i] = cf[i] ? x[i] : M[i] * x[i] + bdt2 * s;
}
// x += alpha p; r -= alpha ap; z = precond(r) for the elements of this thread, then
// r.z and r.r over them -- the grid and per-thread order of k_dot_fin, so the sums
// are bitwise its sums over the updated vectors -- and in the last block: beta =
// rz_new / rz, rz <- rz_new, rr, and the loop test of k_cg_cond (WHILE condition)
__global__ void __launch_bounds__(kT) k_cg_update_dots(
    int n, const double* alpha_dev, const double* p, const double* ap, double* x, double* r,
    const double* jac, double* z, double* part, unsigned* ticket, double* s_rzn, double* s_rr,
    double* s_rz, double* s_beta, const double* s_bb, const double* s_pap, double tol,
    int max_iter, int* it_status, cudaGraphConditionalHandle h, int* more_out) {
    __shared__ double sh[kT], sh2[kT];
    __shared__ bool last;
    const int nb = gridDim.x;
    const double al = *alpha_dev;
    double sacc = 0.0, sacc2 = 0.0;
    for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < n; i += gridDim.x * blockDim.x) {
        x[i] += al * p[i];
        const double ri = r[i] + -al * ap[i];
        r[i] = ri;
        const double zi = jac ? (jac[i] != 0.0 ? ri / jac[i] : ri) : ri;
        z[i] = zi;
        sacc += ri * zi;
        sacc2 += ri * ri;
    }
    sh[threadIdx.x] = sacc;
    sh2[threadIdx.x] = sacc2;
    __syncthreads();
    for (int o = kT / 2; o > 0; o >>= 1) {
        if ((int)threadIdx.x < o) {
            sh[threadIdx.x] += sh[threadIdx.x + o];
            sh2[threadIdx.x] += sh2[threadIdx.x + o];
        }
        __syncthreads();
    }
    if (threadIdx.x == 0) {
        part[blockIdx.x] = sh[0];
        part[nb + blockIdx.x] = sh2[0];
        __threadfence();
        last = atomicAdd(ticket, 1u) == (unsigned)nb - 1;
    }
    __syncthreads();
    if (!last) return;
    __threadfence();
    const volatile double* vp = part;
    double t = 0.0, t2 = 0.0;
    for (int i = threadIdx.x; i < nb; i += blockDim.x) {
        t += vp[i];
        t2 += vp[nb + i];
    }
    sh[threadIdx.x] = t;
    sh2[threadIdx.x] = t2;
    __syncthreads();
    for (int o = kT / 2; o > 0; o >>= 1) {
        if ((int)threadIdx.x < o) {
            sh[threadIdx.x] += sh[threadIdx.x + o];
            sh2[threadIdx.x] += sh2[threadIdx.x + o];
        }
        __syncthreads();
    }
    if (threadIdx.x == 0) {
        *s_rzn = sh[0];
        *s_rr = sh2[0];
        *s_beta = sh[0] / *s_rz;
        *s_rz = sh[0];
        *ticket = 0u;
        // k_cg_cond
        const int it = ++it_status[0];
        bool more = false;
        if (*s_pap <= 0.0) {
            it_status[1] = 1;
        } else {
            more = sqrt(sh2[0]) / sqrt(*s_bb) > tol;
            if (more && it >= max_iter) {
                it_status[1] = 2;
                more = false;
            }
        }
        if (more_out) *more_out = more ? 1 : 0;
        else cudaGraphSetConditional(h, more ? 1u : 0u);
    }
}
}  // namespace
void csr_apply_a(int n, const int32_t* rp, const int32_t* ci, const double* v, const double* x,
                 const double* M, const uint8_t* cf, double bdt2, double* y, cudaStream_t s) {
    k_csr_apply_a<<<blocks(n), kT, 0, s>>>(n, rp, ci, v, x, M, cf, bdt2, y);
    check("csr_apply_a");
}
void cg_update_dots(int n, const double* alpha_dev, const double* p, const double* ap, double* x,
                    double* r, const double* jac, double* z, double* part, unsigned* ticket,
                    double* s_rzn, double* s_rr, double* s_rz, double* s_beta, const double* s_bb,
                    const double* s_pap, double tol, int max_iter, int* it_status,
                    cudaGraphConditionalHandle h, cudaStream_t s, int* more_out) {
    k_cg_update_dots<<<dot_partials(), kT, 0, s>>>(n, alpha_dev, p, ap, x, r, jac, z, part, ticket,
                                                   s_rzn, s_rr, s_rz, s_beta, s_bb, s_pap, tol,
                                                   max_iter, it_status, h, more_out);
    check("cg_update_dots");
}


// ---- the CG operator fused with p.Ap and alpha = rz / pAp (last-block reduction over
// the row blocks' partials, in block order) ----
namespace {
__device__ __forceinline__ void pap_finish(double mine, double* part, unsigned* ticket,
                                           double* s_pap, const double* s_rz, double* s_alpha) {
    __shared__ double sh[kT];
    __shared__ bool last;
    const int nb = gridDim.x;
    sh[threadIdx.x] = mine;
    __syncthreads();
    for (int o = kT / 2; o > 0; o >>= 1) {
        if ((int)threadIdx.x < o) sh[threadIdx.x] += sh[threadIdx.x + o];
        __syncthreads();
    }
    if (threadIdx.x == 0) {
        part[blockIdx.x] = sh[0];
        __threadfence();
        last = atomicAdd(ticket, 1u) == (unsigned)nb - 1;
    }
    __syncthreads();
    if (!last) return;
    __threadfence();
    const volatile double* vp = part;
    double t = 0.0;
    for (int i = threadIdx.x; i < nb; i += blockDim.x) t += vp[i];
    sh[threadIdx.x] = t;
    __syncthreads();
    for (int o = kT / 2; o > 0; o >>= 1) {
        if ((int)threadIdx.x < o) sh[threadIdx.x] += sh[threadIdx.x + o];
        __syncthreads();
    }
    if (threadIdx.x == 0) {
        *s_pap = sh[0];
        *s_alpha = *s_rz / sh[0];
        *ticket = 0u;
    }
}
__global__ void __launch_bounds__(kT) k_csr_apply_a_pap(
    int n, const int32_t* __restrict__ rp, const int32_t* __restrict__ ci,
    const double* __restrict__ v, const double* __restrict__ x, const double* M, const uint8_t* cf,
    double bdt2, double* y, double* part, unsigned* ticket, double* s_pap, const double* s_rz,
    double* s_alpha) {
    const int i = blockIdx.x * blockDim.x + threadIdx.x;
    double mine = 0.0;
    if (i < n) {
        double s = 0.0;
        for (int p = rp[i]; p < rp[i + 1]; ++p) s += v[p] * x[ci[p]];
        const double yi = cf[i] ? x[i] : M[i] * x[i] + bdt2 * s;
        y[i] = yi;
        mine = x[i] * yi;
    }
    pap_finish(mine, part, ticket, s_pap, s_rz, s_alpha);
}
// y = A x (one warp per row), p.Ap, alpha
__global__ void __launch_bounds__(kT) k_csr_warp_pap(
    int n, const int32_t* __restrict__ rp, const int32_t* __restrict__ ci,
    const double* __restrict__ v, const double* __restrict__ x, double* __restrict__ y,
    double* part, unsigned* ticket, double* s_pap, const double* s_rz, double* s_alpha) {
    const int row = (blockIdx.x * blockDim.x + threadIdx.x) >> 5, lane = threadIdx.x & 31;
    double mine = 0.0;
    if (row < n) {
        double s = 0.0;
        for (int p = rp[row] + lane; p < rp[row + 1]; p += 32) s += v[p] * x[ci[p]];
        for (int o = 16; o > 0; o >>= 1) s += __shfl_down_sync(0xffffffffu, s, o);
        if (lane == 0) {
            y[row] = s;
            mine = x[row] * s;
        }
    }
    pap_finish(mine, part, ticket, s_pap, s_rz, s_alpha);
}
}  // namespace
int pap_partials(int n, bool warp_rows) {
    return warp_rows ? blocks((long long)n * 32) : blocks(n);
}
void csr_apply_a_pap(int n, const int32_t* rp, const int32_t* ci, const double* v, const double* x,
                     const double* M, const uint8_t* cf, double bdt2, double* y, double* part,
                     unsigned* ticket, double* s_pap, const double* s_rz, double* s_alpha,
                     cudaStream_t s) {
    k_csr_apply_a_pap<<<blocks(n), kT, 0, s>>>(n, rp, ci, v, x, M, cf, bdt2, y, part, ticket,
                                               s_pap, s_rz, s_alpha);
    check("csr_apply_a_pap");
}
void csr_warp_pap(int n, const int32_t* rp, const int32_t* ci, const double* v, const double* x,
                  double* y, double* part, unsigned* ticket, double* s_pap, const double* s_rz,
                  double* s_alpha, cudaStream_t s) {
    k_csr_warp_pap<<<blocks((long long)n * 32), kT, 0, s>>>(n, rp, ci, v, x, y, part, ticket, s_pap,
                                                            s_rz, s_alpha);
    check("csr_warp_pap");
}

}  // namespace mtsk
}  // namespace pmts
