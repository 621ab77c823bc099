// Device kernels of the coupled multi-time-step integrator (pmts_mts.cu):
// the FE operator (CSR, the reference's row order), the Newmark block solves of
// both subdomains, the Boolean coupling operators and deterministic
// reductions for the conjugate-gradient solves.  Built with -fmad=false so
// every expression rounds as the reference's does.
// Citations: /root/reference/proj/include/perimts/.
#include <stdexcept>
#include <string>

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

__global__ void k_scatter_add(int n, const int32_t* idx, const double* vals, double* dst) {
    const int r = blockIdx.x * blockDim.x + threadIdx.x;
    if (r < n) dst[idx[r]] += vals[r];
}

__global__ void k_gather(int n, const int32_t* idx, const double* src, double* dst) {
    const int r = blockIdx.x * blockDim.x + threadIdx.x;
    if (r < n) dst[r] = src[idx[r]];
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

}  // namespace

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
void gather(int n, const int32_t* idx, const double* src, double* dst, cudaStream_t s) {
    if (n <= 0) return;
    k_gather<<<blocks(n), kT, 0, s>>>(n, idx, src, dst);
    check("gather");
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

}  // namespace mtsk
}  // namespace pmts
