#include <algorithm>
// Deterministic-mode kernels, neighbour build and node update (sm_100a).
//
// This translation unit is compiled with -fmad=false: every fp64 expression
// rounds exactly like the reference's (built without FMA contraction, SURVEY.md
// F8), so the broken-bond set is bit-exact and u/v/a equal the matrix-free
// oracle (oracle/pd_oracle.c, PO_MF) bitwise.  Citations are
// /root/reference/proj/include/perimts/<file>:<line>.
#include <cub/cub.cuh>

#include <cstdio>
#include <stdexcept>
#include <string>
#include <vector>

#include "pd_common.cuh"

namespace pmts {

#define PMTS_CUDA(x)                                                                     \
    do {                                                                                 \
        cudaError_t err_ = (x);                                                          \
        if (err_ != cudaSuccess)                                                         \
            throw std::runtime_error(std::string("CUDA: ") + cudaGetErrorString(err_) + \
                                     " at " __FILE__ ":" + std::to_string(__LINE__));    \
    } while (0)

constexpr int kThreads = 256;

__device__ inline void block_count_add(unsigned long long nb, unsigned long long* target) {
    // warp then block reduction; one atomic per block (no atomics on the force path)
    __shared__ unsigned long long part[kThreads / 32];
    for (int o = 16; o > 0; o >>= 1) nb += __shfl_down_sync(0xffffffffu, nb, o);
    const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
    if (lane == 0) part[wid] = nb;
    __syncthreads();
    if (threadIdx.x == 0) {
        unsigned long long t = 0;
        for (int w = 0; w < (int)(blockDim.x >> 5); ++w) t += part[w];
        if (t) atomicAdd(target, t);
    }
}

// ---------------------------------------------------------------------------
// Fused bond kernel, deterministic order.  One thread per element e walks its
// family in ascending partner order (the order in which damage_field and the
// CSR assembly accumulate, perifem.hpp:205-213 / 317-329):
//   eta   = sum_j N u - sum_i N u, node order, (i<j) orientation  perifem.hpp:149-157
//   s     = (|xi+eta| - |xi|)/|xi|, -1 if collapsed               perifem.hpp:158-165
//   force = -(+/-) w c (xi . eta) xi  (row of K^PD u, perifem.hpp:106-116, 243-268)
//   break = s >= s_crit (inclusive, one-way)                      perifem.hpp:182-186
// The force uses the intact bits of the previous step; the break test runs on
// the same displacement (u_n = rd_n for the explicit beta = 0 branch,
// newmark.hpp:154) and updates the bits for the next step -- the order of
// driver_run.hpp:222-236.
template <int DIM>
__global__ void __launch_bounds__(kThreads)
k_det_bond(DevPD d, const double* __restrict__ disp, int step, int do_break, int gstep) {
    constexpr int NN = DIM == 2 ? 4 : 8;
    const int e = blockIdx.x * blockDim.x + threadIdx.x;
    unsigned long long nb = 0;
    if (e < d.E) {
        const int E = d.E;
        const double Nsh = d.Nsh;
        double qe[NN][DIM];
        double Se[DIM];
        for (int a = 0; a < NN; ++a) {
            const int node = d.conn[a * E + e];
            for (int c = 0; c < DIM; ++c) qe[a][c] = Nsh * disp[(size_t)node * DIM + c];
        }
        for (int c = 0; c < DIM; ++c) {
            double s = 0.0;
            for (int a = 0; a < NN; ++a) s = s + qe[a][c];
            Se[c] = s;
        }
        const double ce[3] = {d.cen[e], d.cen[E + e], d.cen[2 * E + e]};
        double G[DIM];
        for (int c = 0; c < DIM; ++c) G[c] = 0.0;
        int wcur = -1;
        uint32_t word = 0, word0 = 0;
        for (int k = 0; k < d.K; ++k) {
            const int p = d.col[(size_t)k * E + e];
            if (p < 0) break;
            const int w = k >> 5;
            if (w != wcur) {
                if (wcur >= 0 && word != word0) d.mask[(size_t)wcur * E + e] = word;
                word = word0 = d.mask[(size_t)w * E + e];
                wcur = w;
            }
            const uint32_t bit = 1u << (k & 31);
            if (!(word & bit)) continue;
            double qp[NN][DIM];
            for (int a = 0; a < NN; ++a) {
                const int node = d.conn[a * E + p];
                for (int c = 0; c < DIM; ++c) qp[a][c] = Nsh * disp[(size_t)node * DIM + c];
            }
            const double cp[3] = {d.cen[p], d.cen[E + p], d.cen[2 * E + p]};
            double eta[DIM], xi[3];
            if (e < p) {  // e = i, p = j
                for (int c = 0; c < DIM; ++c) {
                    double s = 0.0;
                    for (int a = 0; a < NN; ++a) s = s + qp[a][c];
                    for (int a = 0; a < NN; ++a) s = s - qe[a][c];
                    eta[c] = s;
                }
                for (int c = 0; c < 3; ++c) xi[c] = cp[c] - ce[c];
            } else {  // p = i, e = j
                for (int c = 0; c < DIM; ++c) {
                    double s = Se[c];
                    for (int a = 0; a < NN; ++a) s = s - qp[a][c];
                    eta[c] = s;
                }
                for (int c = 0; c < 3; ++c) xi[c] = ce[c] - cp[c];
            }
            // force with the bits of the previous step
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
                const double s = len <= 0.0 ? -1.0 : (len - xin) / xin;
                const int lo = e < p ? e : p, hi = e < p ? p : e;
                if (s >= bond_s_crit(d.s_crit, d.spread, d.seed, global_elem(d, lo), global_elem(d, hi))) {
                    word &= ~bit;
                    if (e < p && owns_elem(d, e)) {
                        ++nb;
                        if (d.log) {
                            const unsigned long long slot = atomicAdd(d.log_n, 1ull);
                            if ((long long)slot < d.log_cap) {
                                d.log[3 * slot] = gstep;
                                d.log[3 * slot + 1] = (int)global_elem(d, e);
                                d.log[3 * slot + 2] = (int)global_elem(d, p);
                            }
                        }
                    }
                }
            }
        }
        if (wcur >= 0 && word != word0) d.mask[(size_t)wcur * E + e] = word;
        for (int c = 0; c < DIM; ++c) d.G[(size_t)e * DIM + c] = G[c];
    }
    if (do_break) block_count_add(nb, d.broken_count + step);
}

void launch_det_bond(const DevPD& d, const double* disp, int step, int do_break, int gstep,
                     cudaStream_t s) {
    const int blocks = (d.E + kThreads - 1) / kThreads;
    if (d.dim == 2) k_det_bond<2><<<blocks, kThreads, 0, s>>>(d, disp, step, do_break, gstep);
    else k_det_bond<3><<<blocks, kThreads, 0, s>>>(d, disp, step, do_break, gstep);
    PMTS_CUDA(cudaGetLastError());
}

// ---------------------------------------------------------------------------
// Node update: (K u)_n = sum over incident elements (ascending) of N G_e,
// then the explicit branch of BlockOperator::solve (newmark.hpp:125-157) and,
// fused, the predictor of the next step (newmark_predictor, newmark.hpp:61-69).
template <int DIM>
__global__ void __launch_bounds__(kThreads) k_node_update(DevPD d, double scale, int predict_next) {
    const int n = blockIdx.x * blockDim.x + threadIdx.x;
    if (n >= d.N) return;
    double Ku[DIM];
    for (int c = 0; c < DIM; ++c) Ku[c] = 0.0;
    for (int q = 0; q < d.NE; ++q) {
        const int e = d.ne[(size_t)q * d.N + n];
        if (e < 0) break;
        for (int c = 0; c < DIM; ++c) Ku[c] = Ku[c] + d.Nsh * d.G[(size_t)e * DIM + c];
    }
    for (int c = 0; c < DIM; ++c) {
        const size_t i = (size_t)n * DIM + c;
        const bool bc = d.bcflag[i] != 0;
        double pt = d.P[i];
        pt = pt * scale;
        if (d.extra) pt = pt + d.extra[i];  // + G_PD^T S_j (mts.hpp:160-162)
        const double acc = bc ? 0.0 : (pt - Ku[c]) / d.M[i];
        double vel = d.rv[i] + d.c_corr_v * acc;
        const double dis = d.rd[i] + d.c_corr_d * acc;
        if (bc) vel = d.bcvel[i];
        d.a[i] = acc;
        d.v[i] = vel;
        d.u[i] = dis;
        if (predict_next) {
            d.rv[i] = vel + d.c_pred_v * acc;
            d.rd[i] = dis + d.dt * vel + d.c_pred_d * acc;
        }
    }
}

void launch_node_update(const DevPD& d, double scale, int predict_next, cudaStream_t s) {
    const int blocks = (d.N + kThreads - 1) / kThreads;
    if (d.dim == 2) k_node_update<2><<<blocks, kThreads, 0, s>>>(d, scale, predict_next);
    else k_node_update<3><<<blocks, kThreads, 0, s>>>(d, scale, predict_next);
    PMTS_CUDA(cudaGetLastError());
}

// newmark_predictor (newmark.hpp:61-69) from the current (u, v, a)
__global__ void k_predict(DevPD d, int ndof) {
    const int i = blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= ndof) return;
    d.rv[i] = d.v[i] + d.c_pred_v * d.a[i];
    d.rd[i] = d.u[i] + d.dt * d.v[i] + d.c_pred_d * d.a[i];
}

void launch_predict(const DevPD& d, cudaStream_t s) {
    const int nd = d.N * d.dim;
    k_predict<<<(nd + kThreads - 1) / kThreads, kThreads, 0, s>>>(d, nd);
    PMTS_CUDA(cudaGetLastError());
}

// initial_acceleration (newmark.hpp:110-116): a = (P s0 - K u)/M, constrained 0
template <int DIM>
__global__ void k_init_acc(DevPD d, double scale) {
    const int n = blockIdx.x * blockDim.x + threadIdx.x;
    if (n >= d.N) return;
    double Ku[DIM];
    for (int c = 0; c < DIM; ++c) Ku[c] = 0.0;
    for (int q = 0; q < d.NE; ++q) {
        const int e = d.ne[(size_t)q * d.N + n];
        if (e < 0) break;
        for (int c = 0; c < DIM; ++c) Ku[c] = Ku[c] + d.Nsh * d.G[(size_t)e * DIM + c];
    }
    for (int c = 0; c < DIM; ++c) {
        const size_t i = (size_t)n * DIM + c;
        double p = d.P[i] * scale;
        if (d.extra) p = p + d.extra[i];
        d.a[i] = d.bcflag[i] ? 0.0 : (p - Ku[c]) / d.M[i];
    }
}

// (K x)_n = sum over incident elements (ascending) of N G_e -- the node half
// of the matrix-free K^PD x after k_det_bond(x); used by the MTS integrator
template <int DIM>
__global__ void k_node_force(DevPD d, double* __restrict__ kx) {
    const int n = blockIdx.x * blockDim.x + threadIdx.x;
    if (n >= d.N) return;
    double Ku[DIM];
    for (int c = 0; c < DIM; ++c) Ku[c] = 0.0;
    for (int q = 0; q < d.NE; ++q) {
        const int e = d.ne[(size_t)q * d.N + n];
        if (e < 0) break;
        for (int c = 0; c < DIM; ++c) Ku[c] = Ku[c] + d.Nsh * d.G[(size_t)e * DIM + c];
    }
    for (int c = 0; c < DIM; ++c) kx[(size_t)n * DIM + c] = Ku[c];
}

void launch_node_force(const DevPD& d, double* kx, cudaStream_t s) {
    const int blocks = (d.N + kThreads - 1) / kThreads;
    if (d.dim == 2) k_node_force<2><<<blocks, kThreads, 0, s>>>(d, kx);
    else k_node_force<3><<<blocks, kThreads, 0, s>>>(d, kx);
    PMTS_CUDA(cudaGetLastError());
}

void launch_init_acc(const DevPD& d, double scale, cudaStream_t s) {
    const int blocks = (d.N + kThreads - 1) / kThreads;
    if (d.dim == 2) k_init_acc<2><<<blocks, kThreads, 0, s>>>(d, scale);
    else k_init_acc<3><<<blocks, kThreads, 0, s>>>(d, scale);
    PMTS_CUDA(cudaGetLastError());
}

// ---------------------------------------------------------------------------
// damage_field (perifem.hpp:202-231).  Per element, total and intact weights
// accumulate over the ascending family -- the order the reference's PE loop
// reaches them -- so the result is bitwise the reference's.
__global__ void k_damage_elem(DevPD d, double* phi, uint8_t* has) {
    const int e = blockIdx.x * blockDim.x + threadIdx.x;
    if (e >= d.E) return;
    double total = 0.0, intact = 0.0;
    for (int k = 0; k < d.K; ++k) {
        const int p = d.col[(size_t)k * d.E + e];
        if (p < 0) break;
        const int lo = e < p ? e : p, hi = e < p ? p : e;
        const double w = d.vol[lo] * d.vol[hi];
        total = total + w;
        if (d.mask[(size_t)(k >> 5) * d.E + e] & (1u << (k & 31))) intact = intact + w;
    }
    phi[e] = total > 0.0 ? 1.0 - intact / total : 0.0;
    has[e] = total != 0.0;
}

__global__ void k_damage_node(DevPD d, const double* phi, const uint8_t* has, double* node) {
    const int n = blockIdx.x * blockDim.x + threadIdx.x;
    if (n >= d.N) return;
    double s = 0.0;
    int cnt = 0;
    for (int q = 0; q < d.NE; ++q) {
        const int e = d.ne[(size_t)q * d.N + n];
        if (e < 0) break;
        if (!has[e]) continue;
        s = s + phi[e];
        ++cnt;
    }
    node[n] = cnt > 0 ? s / (double)cnt : 0.0;
}

void launch_damage_node(const DevPD& d, const double* elem, const uint8_t* has, double* node,
                        cudaStream_t s) {
    k_damage_node<<<(d.N + kThreads - 1) / kThreads, kThreads, 0, s>>>(d, elem, has, node);
    PMTS_CUDA(cudaGetLastError());
}

void launch_damage(const DevPD& d, double* elem, double* node, cudaStream_t s) {
    uint8_t* has = nullptr;
    PMTS_CUDA(cudaMallocAsync(&has, (size_t)d.E, s));
    k_damage_elem<<<(d.E + kThreads - 1) / kThreads, kThreads, 0, s>>>(d, elem, has);
    launch_damage_node(d, elem, has, node, s);
    PMTS_CUDA(cudaFreeAsync(has, s));
}

__global__ void k_gather(const double* src, const int32_t* idx, int n, double* dst) {
    const int i = blockIdx.x * blockDim.x + threadIdx.x;
    if (i < n) dst[i] = src[idx[i]];
}

void launch_gather(const double* src, const int32_t* idx, int n, double* dst, cudaStream_t s) {
    if (n <= 0) return;
    k_gather<<<(n + 127) / 128, 128, 0, s>>>(src, idx, n, dst);
    PMTS_CUDA(cudaGetLastError());
}

// Per-step reporting for pmts_pd_step_tracked, one tiny launch: the step's
// tracked displacements and broken count written straight into mapped pinned
// host memory (the device->host transfer of the step's result, no copy op),
// and the next step's load scale read from mapped pinned host memory into
// device memory (its host->device transfer).
__global__ void k_track(const double* src, const int32_t* idx, int n, double* trk_host,
                        const unsigned long long* cnt_dev, unsigned long long* cnt_host,
                        const double* scl_host_next, double* scl_dev_next) {
    const int i = blockIdx.x * blockDim.x + threadIdx.x;
    if (i < n) trk_host[i] = src[idx[i]];
    if (i == 0) {
        if (cnt_dev) *cnt_host = *cnt_dev;
        if (scl_dev_next) *scl_dev_next = *scl_host_next;
    }
}

void launch_track(const double* src, const int32_t* idx, int n, double* trk_host,
                  const unsigned long long* cnt_dev, unsigned long long* cnt_host,
                  const double* scl_host_next, double* scl_dev_next, cudaStream_t s) {
    k_track<<<(std::max(n, 1) + 127) / 128, 128, 0, s>>>(src, idx, n, trk_host, cnt_dev, cnt_host,
                                                       scl_host_next, scl_dev_next);
    PMTS_CUDA(cudaGetLastError());
}

// ---------------------------------------------------------------------------
// Neighbour build: find_pe_pairs (mesh.hpp:416-495) as a device cell list.
// Same cell function (cells of size delta from the minimum centroid), same
// candidate set (the 3^d neighbouring cells), same distance and notch
// predicates, evaluated in the (lower id, higher id) orientation the
// reference uses; families come out sorted by partner id.

__device__ inline double cross2(double ax, double ay, double bx, double by) {
    return ax * by - ay * bx;
}

// mesh.hpp:324-347
__device__ bool seg_intersect_2d(const double* p1, const double* p2, const double* q1,
                                 const double* q2, double eps) {
    const double rx = p2[0] - p1[0], ry = p2[1] - p1[1];
    const double sx = q2[0] - q1[0], sy = q2[1] - q1[1];
    const double denom = cross2(rx, ry, sx, sy);
    const double qpx = q1[0] - p1[0], qpy = q1[1] - p1[1];
    const double tn = cross2(qpx, qpy, sx, sy);
    const double un = cross2(qpx, qpy, rx, ry);
    if (fabs(denom) > eps * eps) {
        const double t = tn / denom;
        const double u = un / denom;
        const double tol_t = eps / fmax(hypot(rx, ry), eps);
        const double tol_u = eps / fmax(hypot(sx, sy), eps);
        return t >= -tol_t && t <= 1.0 + tol_t && u >= -tol_u && u <= 1.0 + tol_u;
    }
    if (fabs(tn) > eps * fmax(hypot(sx, sy), eps)) return false;
    const double rr = rx * rx + ry * ry;
    if (rr < eps * eps) return false;
    double t0 = (qpx * rx + qpy * ry) / rr;
    double t1 = t0 + (sx * rx + sy * ry) / rr;
    if (t0 > t1) {
        const double tmp = t0;
        t0 = t1;
        t1 = tmp;
    }
    return t1 >= 0.0 && t0 <= 1.0;
}

// mesh.hpp:349-395
__device__ bool seg_crosses_polygon_3d(const double* a, const double* b, const double* poly,
                                       int nv, double eps) {
    const double* o = poly;
    const double u[3] = {poly[3] - o[0], poly[4] - o[1], poly[5] - o[2]};
    const double v[3] = {poly[6] - o[0], poly[7] - o[1], poly[8] - o[2]};
    double n[3] = {u[1] * v[2] - u[2] * v[1], u[2] * v[0] - u[0] * v[2],
                   u[0] * v[1] - u[1] * v[0]};
    const double nlen = sqrt(n[0] * n[0] + n[1] * n[1] + n[2] * n[2]);
    if (nlen == 0.0) return false;
    for (int k = 0; k < 3; ++k) n[k] /= nlen;
    const double da = (a[0] - o[0]) * n[0] + (a[1] - o[1]) * n[1] + (a[2] - o[2]) * n[2];
    const double db = (b[0] - o[0]) * n[0] + (b[1] - o[1]) * n[1] + (b[2] - o[2]) * n[2];
    if ((da > eps && db > eps) || (da < -eps && db < -eps)) return false;
    if (fabs(da - db) < eps) return false;
    const double t = da / (da - db);
    if (t < -eps || t > 1.0 + eps) return false;
    const double p[3] = {a[0] + t * (b[0] - a[0]), a[1] + t * (b[1] - a[1]),
                         a[2] + t * (b[2] - a[2])};
    int drop = 0;
    double best = fabs(n[0]);
    for (int k = 1; k < 3; ++k)
        if (fabs(n[k]) > best) {
            best = fabs(n[k]);
            drop = k;
        }
    const int i0 = (drop + 1) % 3, i1 = (drop + 2) % 3;
    bool inside = false;
    for (int e = 0, f = nv - 1; e < nv; f = e++) {
        const double xi = poly[3 * e + i0], yi = poly[3 * e + i1];
        const double xj = poly[3 * f + i0], yj = poly[3 * f + i1];
        const double ex = xj - xi, ey = yj - yi;
        const double px = p[i0] - xi, py = p[i1] - yi;
        const double elen2 = ex * ex + ey * ey;
        if (elen2 > 0.0) {
            double s = (px * ex + py * ey) / elen2;
            s = s < 0.0 ? 0.0 : (s > 1.0 ? 1.0 : s);
            const double ddx = px - s * ex, ddy = py - s * ey;
            if (ddx * ddx + ddy * ddy <= eps * eps) return true;
        }
        if ((yi > p[i1]) != (yj > p[i1]) && p[i0] < (xj - xi) * (p[i1] - yi) / (yj - yi) + xi)
            inside = !inside;
    }
    return inside;
}

struct CellGrid {
    int dim, E;
    const double* cen;
    double lo[3];
    double delta, eps;
    int gx, gy, gz;
    const int32_t* start;  // (gx*gy*gz)+1
    const int32_t* ids;
    int n_notch;
    const int32_t* notch_npts;
    const int32_t* notch_off;  // first point index of each notch
    const double* notch_pts;
};

__device__ inline int cell_coord(const CellGrid& g, int e, int k) {
    if (k >= g.dim) return 0;
    return (int)floor((g.cen[(size_t)k * g.E + e] - g.lo[k]) / g.delta);
}

__global__ void k_cell_count(CellGrid g, int32_t* cnt, int32_t* cell_of) {
    const int e = blockIdx.x * blockDim.x + threadIdx.x;
    if (e >= g.E) return;
    const int cx = cell_coord(g, e, 0), cy = cell_coord(g, e, 1), cz = cell_coord(g, e, 2);
    const int c = (cz * g.gy + cy) * g.gx + cx;
    cell_of[e] = c;
    atomicAdd(cnt + c, 1);
}

__global__ void k_cell_fill(CellGrid g, const int32_t* cell_of, int32_t* cursor, int32_t* ids) {
    const int e = blockIdx.x * blockDim.x + threadIdx.x;
    if (e >= g.E) return;
    ids[atomicAdd(cursor + cell_of[e], 1)] = e;
}

// returns the partner count; writes partners (unsorted) when out != nullptr
template <int MAXK>
__device__ int scan_partners(const CellGrid& g, int i, int32_t* out) {
    const double ci[3] = {g.cen[i], g.cen[(size_t)g.E + i], g.cen[2 * (size_t)g.E + i]};
    const int cx = cell_coord(g, i, 0), cy = cell_coord(g, i, 1), cz = cell_coord(g, i, 2);
    const int zr = g.dim == 3 ? 1 : 0;
    int cnt = 0;
    for (int dz = -zr; dz <= zr; ++dz)
        for (int dy = -1; dy <= 1; ++dy)
            for (int dx = -1; dx <= 1; ++dx) {
                const int x = cx + dx, y = cy + dy, z = cz + dz;
                if (x < 0 || y < 0 || z < 0 || x >= g.gx || y >= g.gy || z >= g.gz) continue;
                const int c = (z * g.gy + y) * g.gx + x;
                for (int s = g.start[c]; s < g.start[c + 1]; ++s) {
                    const int j = g.ids[s];
                    if (j == i) continue;
                    const double cj[3] = {g.cen[j], g.cen[(size_t)g.E + j],
                                          g.cen[2 * (size_t)g.E + j]};
                    const double* a = i < j ? ci : cj;  // lower id first (mesh.hpp:466-479)
                    const double* b = i < j ? cj : ci;
                    const double ddx = a[0] - b[0], ddy = a[1] - b[1], ddz = a[2] - b[2];
                    if (sqrt(ddx * ddx + ddy * ddy + ddz * ddz) > g.delta) continue;
                    bool cut = false;
                    for (int q = 0; q < g.n_notch && !cut; ++q) {
                        const double* np = g.notch_pts + 3 * (size_t)g.notch_off[q];
                        const int npts = g.notch_npts[q];
                        if (npts == 2) cut = seg_intersect_2d(a, b, np, np + 3, g.eps);
                        else if (npts >= 3) cut = seg_crosses_polygon_3d(a, b, np, npts, g.eps);
                    }
                    if (cut) continue;
                    if (out && cnt < MAXK) out[cnt] = j;
                    ++cnt;
                }
            }
    return cnt;
}

constexpr int kMaxFamily = 512;

__global__ void k_family_count(CellGrid g, int32_t* count) {
    const int i = blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= g.E) return;
    count[i] = scan_partners<kMaxFamily>(g, i, nullptr);
}

__global__ void k_family_fill(CellGrid g, int K, int32_t* col) {
    const int i = blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= g.E) return;
    int32_t buf[kMaxFamily];
    const int n = scan_partners<kMaxFamily>(g, i, buf);
    for (int a = 1; a < n; ++a) {  // insertion sort: ascending partner id
        const int32_t v = buf[a];
        int b = a - 1;
        while (b >= 0 && buf[b] > v) {
            buf[b + 1] = buf[b];
            --b;
        }
        buf[b + 1] = v;
    }
    for (int k = 0; k < K; ++k) col[(size_t)k * g.E + i] = k < n ? buf[k] : -1;
}

FamilyBuild build_families_device(int dim, int E, const double* d_cen, const double lo[3],
                                  double delta, double eps, int n_notch,
                                  const int32_t* notch_npts, const double* notch_pts,
                                  cudaStream_t s) {
    CellGrid g{};
    g.dim = dim;
    g.E = E;
    g.cen = d_cen;
    for (int k = 0; k < 3; ++k) g.lo[k] = lo[k];
    g.delta = delta;
    g.eps = eps;
    // grid extent: cells of the max centroid (host sees the same floor)
    std::vector<double> hcen(3 * (size_t)E);
    PMTS_CUDA(cudaMemcpyAsync(hcen.data(), d_cen, sizeof(double) * 3 * (size_t)E,
                              cudaMemcpyDeviceToHost, s));
    PMTS_CUDA(cudaStreamSynchronize(s));
    int gmax[3] = {0, 0, 0};
    for (int k = 0; k < dim; ++k)
        for (int e = 0; e < E; ++e) {
            const int c = (int)std::floor((hcen[(size_t)k * E + e] - lo[k]) / delta);
            if (c > gmax[k]) gmax[k] = c;
        }
    g.gx = gmax[0] + 1;
    g.gy = gmax[1] + 1;
    g.gz = gmax[2] + 1;
    const size_t ncell = (size_t)g.gx * g.gy * g.gz;
    if (ncell > (size_t)1 << 31) throw std::runtime_error("neighbour grid too large");

    // notch tables
    std::vector<int32_t> off(n_notch + 1, 0);
    for (int q = 0; q < n_notch; ++q) off[q + 1] = off[q] + notch_npts[q];
    int32_t *d_npts = nullptr, *d_off = nullptr;
    double* d_pts = nullptr;
    if (n_notch > 0) {
        PMTS_CUDA(cudaMallocAsync(&d_npts, sizeof(int32_t) * n_notch, s));
        PMTS_CUDA(cudaMallocAsync(&d_off, sizeof(int32_t) * (n_notch + 1), s));
        PMTS_CUDA(cudaMallocAsync(&d_pts, sizeof(double) * 3 * (size_t)off[n_notch], s));
        PMTS_CUDA(cudaMemcpyAsync(d_npts, notch_npts, sizeof(int32_t) * n_notch,
                                  cudaMemcpyHostToDevice, s));
        PMTS_CUDA(cudaMemcpyAsync(d_off, off.data(), sizeof(int32_t) * (n_notch + 1),
                                  cudaMemcpyHostToDevice, s));
        PMTS_CUDA(cudaMemcpyAsync(d_pts, notch_pts, sizeof(double) * 3 * (size_t)off[n_notch],
                                  cudaMemcpyHostToDevice, s));
    }
    g.n_notch = n_notch;
    g.notch_npts = d_npts;
    g.notch_off = d_off;
    g.notch_pts = d_pts;

    int32_t *cnt = nullptr, *start = nullptr, *cell_of = nullptr, *ids = nullptr, *count = nullptr;
    PMTS_CUDA(cudaMallocAsync(&cnt, sizeof(int32_t) * (ncell + 1), s));
    PMTS_CUDA(cudaMallocAsync(&start, sizeof(int32_t) * (ncell + 1), s));
    PMTS_CUDA(cudaMallocAsync(&cell_of, sizeof(int32_t) * (size_t)E, s));
    PMTS_CUDA(cudaMallocAsync(&ids, sizeof(int32_t) * (size_t)E, s));
    PMTS_CUDA(cudaMallocAsync(&count, sizeof(int32_t) * (size_t)E, s));
    PMTS_CUDA(cudaMemsetAsync(cnt, 0, sizeof(int32_t) * (ncell + 1), s));
    const int blocks = (E + kThreads - 1) / kThreads;
    k_cell_count<<<blocks, kThreads, 0, s>>>(g, cnt, cell_of);
    size_t tmp_bytes = 0;
    cub::DeviceScan::ExclusiveSum(nullptr, tmp_bytes, cnt, start, (int)ncell + 1, s);
    void* tmp = nullptr;
    PMTS_CUDA(cudaMallocAsync(&tmp, tmp_bytes, s));
    cub::DeviceScan::ExclusiveSum(tmp, tmp_bytes, cnt, start, (int)ncell + 1, s);
    PMTS_CUDA(cudaMemcpyAsync(cnt, start, sizeof(int32_t) * (ncell + 1), cudaMemcpyDeviceToDevice, s));
    k_cell_fill<<<blocks, kThreads, 0, s>>>(g, cell_of, cnt, ids);
    g.start = start;
    g.ids = ids;
    k_family_count<<<blocks, kThreads, 0, s>>>(g, count);
    PMTS_CUDA(cudaGetLastError());
    std::vector<int32_t> hcount(E);
    PMTS_CUDA(cudaMemcpyAsync(hcount.data(), count, sizeof(int32_t) * (size_t)E,
                              cudaMemcpyDeviceToHost, s));
    PMTS_CUDA(cudaStreamSynchronize(s));
    int K = 0;
    int64_t F = 0;
    for (int e = 0; e < E; ++e) {
        K = std::max(K, (int)hcount[e]);
        F += hcount[e];
    }
    if (K > kMaxFamily)
        throw std::runtime_error("family larger than " + std::to_string(kMaxFamily) +
                                 " partners; horizon too large for the device build");
    FamilyBuild fb{};
    fb.K = K;
    fb.n_entries = F;
    PMTS_CUDA(cudaMalloc(&fb.col, sizeof(int32_t) * std::max<size_t>((size_t)K * E, 1)));
    if (K > 0) k_family_fill<<<blocks, kThreads, 0, s>>>(g, K, fb.col);
    PMTS_CUDA(cudaGetLastError());
    PMTS_CUDA(cudaFreeAsync(tmp, s));
    for (void* p : {(void*)cnt, (void*)start, (void*)cell_of, (void*)ids, (void*)count,
                    (void*)d_npts, (void*)d_off, (void*)d_pts})
        if (p) PMTS_CUDA(cudaFreeAsync(p, s));
    PMTS_CUDA(cudaStreamSynchronize(s));
    return fb;
}

}  // namespace pmts
