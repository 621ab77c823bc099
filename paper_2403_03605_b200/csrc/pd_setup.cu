// Device restatement of the setup of a generated run:
// generate_structured (mesh.hpp:170-219), compute_element_geometry
// (mesh.hpp:112-139) and the lumped mass / external load loop of
// assemble_pd_global (perifem.hpp:331-348, lumped_mass fem.hpp:172-179).
//
// Built with -fmad=false and written in the host restatement's operation order
// (pmts_setup.cpp), so every value is bitwise the host's -- and the reference's
// (tests/test_gpu_setup.py).  Per element: the Gauss-point Jacobians, the
// centroid, the volume and the 2^d lumped-mass contributions; per node: the
// incident elements' contributions gathered in ascending element order -- the
// order the reference's element loop adds them in.
#include <cuda_runtime.h>

#include <memory>
#include <string>
#include <vector>

#include "pmts_internal.h"

namespace pmts {

namespace {

__device__ __forceinline__ void d_corner_gradient(int dim, const double* xi, int a, double* g) {
    if (dim == 2) {
        const double sx = (a == 1 || a == 2) ? 1.0 : -1.0, sy = a >= 2 ? 1.0 : -1.0;
        g[0] = 0.25 * sx * (1 + sy * xi[1]);
        g[1] = 0.25 * sy * (1 + sx * xi[0]);
        g[2] = 0.0;
    } else {
        const int b = a & 3;
        const double sx = (b == 1 || b == 2) ? 1.0 : -1.0, sy = b >= 2 ? 1.0 : -1.0,
                     sz = a >= 4 ? 1.0 : -1.0;
        g[0] = 0.125 * sx * (1 + sy * xi[1]) * (1 + sz * xi[2]);
        g[1] = 0.125 * sy * (1 + sx * xi[0]) * (1 + sz * xi[2]);
        g[2] = 0.125 * sz * (1 + sx * xi[0]) * (1 + sy * xi[1]);
    }
}

__device__ __forceinline__ double d_shape_value(int dim, const double* xi, int a) {
    if (dim == 2) {
        const double sx = (a == 1 || a == 2) ? 1.0 : -1.0, sy = a >= 2 ? 1.0 : -1.0;
        return 0.25 * (1 + sx * xi[0]) * (1 + sy * xi[1]);
    }
    const int b = a & 3;
    const double sx = (b == 1 || b == 2) ? 1.0 : -1.0, sy = b >= 2 ? 1.0 : -1.0,
                 sz = a >= 4 ? 1.0 : -1.0;
    return 0.125 * (1 + sx * xi[0]) * (1 + sy * xi[1]) * (1 + sz * xi[2]);
}

// jacobian_det (mesh.hpp:91-105) on the element's node coordinates p[a][0..2]
__device__ double d_jacobian_det(int dim, const double (*p)[3], const double* xi) {
    double J[3][3] = {{0, 0, 0}, {0, 0, 0}, {0, 0, 0}};
    double g[3];
    const int nn = dim == 2 ? 4 : 8;
    for (int a = 0; a < nn; ++a) {
        d_corner_gradient(dim, xi, a, g);
        for (int i = 0; i < dim; ++i)
            for (int j = 0; j < dim; ++j) J[i][j] += p[a][i] * g[j];
    }
    if (dim == 2) return J[0][0] * J[1][1] - J[0][1] * J[1][0];
    return J[0][0] * (J[1][1] * J[2][2] - J[1][2] * J[2][1]) -
           J[0][1] * (J[1][0] * J[2][2] - J[1][2] * J[2][0]) +
           J[0][2] * (J[1][0] * J[2][1] - J[1][1] * J[2][0]);
}

struct Grid {
    int dim, nx, ny, nz;  // elements per axis (nz = 1 in 2D)
    double lo[3], h;
};

// generate_structured: node (i, j, k) -> lo + i h, numbered i fastest
__global__ void k_nodes(Grid g, double* __restrict__ xyz) {
    const int NX = g.nx + 1, NY = g.ny + 1, NZ = g.dim == 3 ? g.nz + 1 : 1;
    const long long N = (long long)NX * NY * NZ;
    for (long long n = blockIdx.x * (long long)blockDim.x + threadIdx.x; n < N;
         n += (long long)gridDim.x * blockDim.x) {
        const int i = (int)(n % NX), j = (int)((n / NX) % NY), k = (int)(n / ((long long)NX * NY));
        xyz[3 * n] = g.lo[0] + i * g.h;
        xyz[3 * n + 1] = g.lo[1] + j * g.h;
        xyz[3 * n + 2] = g.dim == 3 ? g.lo[2] + k * g.h : 0.0;
    }
}

// element (i, j, k): its nodes in mesh.hpp:206-213 order
__device__ __forceinline__ void elem_nodes(const Grid& g, int i, int j, int k, int* en) {
    const int NX = g.nx + 1, NY = g.ny + 1;
    auto nid = [&](int a, int b, int c) { return (c * NY + b) * NX + a; };
    en[0] = nid(i, j, k);
    en[1] = nid(i + 1, j, k);
    en[2] = nid(i + 1, j + 1, k);
    en[3] = nid(i, j + 1, k);
    if (g.dim == 3) {
        en[4] = nid(i, j, k + 1);
        en[5] = nid(i + 1, j, k + 1);
        en[6] = nid(i + 1, j + 1, k + 1);
        en[7] = nid(i, j + 1, k + 1);
    }
}

// per element: connectivity, centroid, volume (compute_element_geometry) and the
// lumped-mass contributions rho N_a detJ summed over the Gauss points (fem.hpp:172-179)
__global__ void k_elems(Grid g, const double* __restrict__ xyz, double rho, int32_t* __restrict__ conn,
                        double* __restrict__ cen, double* __restrict__ vol, double* __restrict__ me,
                        int* __restrict__ bad) {
    const int nn = g.dim == 2 ? 4 : 8;
    const long long E = (long long)g.nx * g.ny * (g.dim == 3 ? g.nz : 1);
    const double gp = 1.0 / sqrt(3.0);
    for (long long e = blockIdx.x * (long long)blockDim.x + threadIdx.x; e < E;
         e += (long long)gridDim.x * blockDim.x) {
        const int i = (int)(e % g.nx), j = (int)((e / g.nx) % g.ny),
                  k = (int)(e / ((long long)g.nx * g.ny));
        int en[8];
        elem_nodes(g, i, j, k, en);
        double p[8][3];
        for (int a = 0; a < nn; ++a) {
            conn[e * nn + a] = en[a];
            for (int c = 0; c < 3; ++c) p[a][c] = xyz[3 * (size_t)en[a] + c];
        }
        double c3[3] = {0, 0, 0};
        for (int a = 0; a < nn; ++a)
            for (int c = 0; c < 3; ++c) c3[c] += p[a][c];
        for (int c = 0; c < 3; ++c) cen[3 * e + c] = c3[c] / nn;
        double v = 0.0, m[8] = {0, 0, 0, 0, 0, 0, 0, 0};
        const int ng = g.dim == 2 ? 4 : 8;
        for (int q = 0; q < ng; ++q) {
            // volume: compute_element_geometry's Gauss order (xi bits 0, 1, 2)
            const double xi[3] = {(q & 1) ? gp : -gp, (q & 2) ? gp : -gp, (q & 4) ? gp : -gp};
            const double dj = d_jacobian_det(g.dim, p, xi);
            if (dj <= 0.0) atomicOr(bad, 1);
            v += dj;
        }
        for (int q = 0; q < ng; ++q) {
            // lumped mass: gauss_points' order (fem.hpp:101-115), z = 0 in 2D
            const int qi = q & 1, qj = (q >> 1) & 1, qk = (q >> 2) & 1;
            const double xi[3] = {qi ? gp : -gp, qj ? gp : -gp, g.dim == 3 ? (qk ? gp : -gp) : 0.0};
            const double dj = d_jacobian_det(g.dim, p, xi);
            for (int a = 0; a < nn; ++a) m[a] += rho * d_shape_value(g.dim, xi, a) * dj;
        }
        vol[e] = v;
        for (int a = 0; a < nn; ++a) me[e * nn + a] = m[a];
    }
}

struct Patches {
    int n;
    double box[16][9];  // lo[3] hi[3] value[3]
};

// per node: M and P_ext from the incident elements in ascending element order
// (perifem.hpp:331-348 with w = 1 - alpha = 1); the element's body force is
// body + the values of the patches containing its centroid, in patch order
__global__ void k_node_loads(Grid g, const double* __restrict__ cen, const double* __restrict__ me,
                             const __grid_constant__ Patches pt, double bx, double by, double bz,
                             double rho, double* __restrict__ M, double* __restrict__ P) {
    const int dim = g.dim, nn = dim == 2 ? 4 : 8;
    const int NX = g.nx + 1, NY = g.ny + 1, NZ = dim == 3 ? g.nz + 1 : 1;
    const long long N = (long long)NX * NY * NZ;
    const double w = 1.0 - 0.0;
    for (long long n = blockIdx.x * (long long)blockDim.x + threadIdx.x; n < N;
         n += (long long)gridDim.x * blockDim.x) {
        const int i = (int)(n % NX), j = (int)((n / NX) % NY), k = (int)(n / ((long long)NX * NY));
        double m[3] = {0, 0, 0}, pl[3] = {0, 0, 0};
        for (int kk = (dim == 3 ? k - 1 : 0); kk <= (dim == 3 ? k : 0); ++kk) {
            if (kk < 0 || (dim == 3 && kk >= g.nz)) continue;
            for (int jj = j - 1; jj <= j; ++jj) {
                if (jj < 0 || jj >= g.ny) continue;
                for (int ii = i - 1; ii <= i; ++ii) {
                    if (ii < 0 || ii >= g.nx) continue;
                    const long long e = ((long long)kk * g.ny + jj) * g.nx + ii;
                    const int di = i - ii, dj = j - jj;
                    const int a = (dj ? (di ? 2 : 3) : (di ? 1 : 0)) + (dim == 3 ? 4 * (k - kk) : 0);
                    const double ma = me[e * nn + a];
                    double b[3] = {bx, by, bz};
                    const double* c = cen + 3 * e;
                    for (int q = 0; q < pt.n; ++q) {
                        bool in = true;
                        for (int d = 0; d < dim; ++d)
                            in = in && !(c[d] < pt.box[q][d] || c[d] > pt.box[q][3 + d]);
                        if (in)
                            for (int d = 0; d < dim; ++d) b[d] += pt.box[q][6 + d];
                    }
                    for (int d = 0; d < dim; ++d) {
                        m[d] += w * ma;
                        pl[d] += w * b[d] * ma / rho;
                    }
                }
            }
        }
        for (int d = 0; d < dim; ++d) {
            M[n * dim + d] = m[d];
            P[n * dim + d] = pl[d];
        }
    }
}

// compute_element_geometry for an arbitrary mesh (pmts_pd_create)
__global__ void k_geometry(int dim, long long E, const int32_t* __restrict__ conn,
                           const double* __restrict__ xyz, double* __restrict__ cen,
                           double* __restrict__ vol, int* __restrict__ bad) {
    const int nn = dim == 2 ? 4 : 8;
    const double gp = 1.0 / sqrt(3.0);
    for (long long e = blockIdx.x * (long long)blockDim.x + threadIdx.x; e < E;
         e += (long long)gridDim.x * blockDim.x) {
        double p[8][3];
        for (int a = 0; a < nn; ++a)
            for (int c = 0; c < 3; ++c) p[a][c] = xyz[3 * (size_t)conn[e * nn + a] + c];
        double c3[3] = {0, 0, 0};
        for (int a = 0; a < nn; ++a)
            for (int c = 0; c < 3; ++c) c3[c] += p[a][c];
        for (int c = 0; c < 3; ++c) cen[3 * e + c] = c3[c] / nn;
        double v = 0.0;
        for (int q = 0; q < (dim == 2 ? 4 : 8); ++q) {
            const double xi[3] = {(q & 1) ? gp : -gp, (q & 2) ? gp : -gp, (q & 4) ? gp : -gp};
            const double dj = d_jacobian_det(dim, p, xi);
            if (dj <= 0.0) atomicOr(bad, 1);
            v += dj;
        }
        vol[e] = v;
    }
}

// volumes only (compute_element_geometry's sum), for Mesh::char_length of a lattice
__global__ void k_volumes(Grid g, double* __restrict__ vol) {
    const int nn = g.dim == 2 ? 4 : 8;
    const long long E = (long long)g.nx * g.ny * (g.dim == 3 ? g.nz : 1);
    const double gp = 1.0 / sqrt(3.0);
    for (long long e = blockIdx.x * (long long)blockDim.x + threadIdx.x; e < E;
         e += (long long)gridDim.x * blockDim.x) {
        const int i = (int)(e % g.nx), j = (int)((e / g.nx) % g.ny),
                  k = (int)(e / ((long long)g.nx * g.ny));
        double p[8][3];
        const int ii[8] = {i, i + 1, i + 1, i, i, i + 1, i + 1, i};
        const int jj[8] = {j, j, j + 1, j + 1, j, j, j + 1, j + 1};
        for (int a = 0; a < nn; ++a) {
            const int kk = a >= 4 ? k + 1 : k;
            p[a][0] = g.lo[0] + ii[a] * g.h;
            p[a][1] = g.lo[1] + jj[a] * g.h;
            p[a][2] = g.dim == 3 ? g.lo[2] + kk * g.h : 0.0;
        }
        double v = 0.0;
        for (int q = 0; q < (g.dim == 2 ? 4 : 8); ++q) {
            const double xi[3] = {(q & 1) ? gp : -gp, (q & 2) ? gp : -gp, (q & 4) ? gp : -gp};
            v += d_jacobian_det(g.dim, p, xi);
        }
        vol[e] = v;
    }
}
// the reference's serial sum (mesh.hpp:51-57)
__global__ void k_serial_sum(long long n, const double* __restrict__ x, double* out) {
    double v = 0.0;
    for (long long i = 0; i < n; ++i) v += x[i];
    *out = v;
}

void ck(cudaError_t e) {
    if (e != cudaSuccess) throw InternalError(std::string("CUDA: ") + cudaGetErrorString(e));
}

template <class T>
T* dmalloc(size_t n, cudaStream_t s) {
    void* p = nullptr;
    ck(cudaMallocAsync(&p, sizeof(T) * (n ? n : 1), s));
    return static_cast<T*>(p);
}

}  // namespace

struct DeviceSetup {
    Grid g{};
    cudaStream_t s = nullptr;
    double rho = 0.0;
    double* xyz = nullptr;
    double* cen = nullptr;
    double* me = nullptr;
    ~DeviceSetup() {
        if (xyz) cudaFreeAsync(xyz, s);
        if (cen) cudaFreeAsync(cen, s);
        if (me) cudaFreeAsync(me, s);
        if (s) {
            cudaStreamSynchronize(s);
            cudaStreamDestroy(s);
        }
    }
};

bool device_available() {
    int n = 0;
    return cudaGetDeviceCount(&n) == cudaSuccess && n > 0;
}

DeviceSetup* setup_device_begin(int dim, const int n[3], const double lo[3], double spacing,
                                double rho, std::vector<double>& nodes,
                                std::vector<int32_t>& conn, std::vector<double>& centroid,
                                std::vector<double>& volume) {
    auto ds = std::make_unique<DeviceSetup>();
    ck(cudaStreamCreateWithFlags(&ds->s, cudaStreamNonBlocking));
    Grid& g = ds->g;
    g.dim = dim;
    g.nx = n[0];
    g.ny = n[1];
    g.nz = dim == 3 ? n[2] : 1;
    for (int k = 0; k < 3; ++k) g.lo[k] = lo[k];
    g.h = spacing;
    ds->rho = rho;
    const int nn = dim == 2 ? 4 : 8;
    const size_t N = (size_t)(g.nx + 1) * (g.ny + 1) * (dim == 3 ? g.nz + 1 : 1);
    const size_t E = (size_t)g.nx * g.ny * g.nz;
    cudaStream_t s = ds->s;
    ds->xyz = dmalloc<double>(3 * N, s);
    ds->cen = dmalloc<double>(3 * E, s);
    ds->me = dmalloc<double>(nn * E, s);
    int32_t* dconn = dmalloc<int32_t>(nn * E, s);
    double* dvol = dmalloc<double>(E, s);
    int* bad = dmalloc<int>(1, s);
    ck(cudaMemsetAsync(bad, 0, sizeof(int), s));
    k_nodes<<<1184, 256, 0, s>>>(g, ds->xyz);
    k_elems<<<1184, 128, 0, s>>>(g, ds->xyz, rho, dconn, ds->cen, dvol, ds->me, bad);
    ck(cudaGetLastError());
    nodes.resize(3 * N);
    conn.resize(nn * E);
    centroid.resize(3 * E);
    volume.resize(E);
    int hbad = 0;
    ck(cudaMemcpyAsync(nodes.data(), ds->xyz, sizeof(double) * 3 * N, cudaMemcpyDeviceToHost, s));
    ck(cudaMemcpyAsync(conn.data(), dconn, sizeof(int32_t) * nn * E, cudaMemcpyDeviceToHost, s));
    ck(cudaMemcpyAsync(centroid.data(), ds->cen, sizeof(double) * 3 * E, cudaMemcpyDeviceToHost, s));
    ck(cudaMemcpyAsync(volume.data(), dvol, sizeof(double) * E, cudaMemcpyDeviceToHost, s));
    ck(cudaMemcpyAsync(&hbad, bad, sizeof(int), cudaMemcpyDeviceToHost, s));
    cudaFreeAsync(dconn, s);
    cudaFreeAsync(dvol, s);
    cudaFreeAsync(bad, s);
    ck(cudaStreamSynchronize(s));
    if (hbad) throw ConfigError("inverted element (non-positive Jacobian)");
    return ds.release();
}

void setup_device_loads(DeviceSetup* ds, const double body[3], int n_patch, const double* boxes,
                        std::vector<double>& mass, std::vector<double>& p_ext) {
    Patches pt{};
    if (n_patch > 16) throw ConfigError("more than 16 load patches");
    pt.n = n_patch;
    for (int q = 0; q < n_patch; ++q)
        for (int c = 0; c < 9; ++c) pt.box[q][c] = boxes[9 * q + c];
    const Grid& g = ds->g;
    const size_t N = (size_t)(g.nx + 1) * (g.ny + 1) * (g.dim == 3 ? g.nz + 1 : 1);
    const size_t nd = N * g.dim;
    cudaStream_t s = ds->s;
    double* dM = dmalloc<double>(nd, s);
    double* dP = dmalloc<double>(nd, s);
    k_node_loads<<<1184, 256, 0, s>>>(g, ds->cen, ds->me, pt, body[0], body[1], body[2], ds->rho,
                                      dM, dP);
    ck(cudaGetLastError());
    mass.resize(nd);
    p_ext.resize(nd);
    ck(cudaMemcpyAsync(mass.data(), dM, sizeof(double) * nd, cudaMemcpyDeviceToHost, s));
    ck(cudaMemcpyAsync(p_ext.data(), dP, sizeof(double) * nd, cudaMemcpyDeviceToHost, s));
    cudaFreeAsync(dM, s);
    cudaFreeAsync(dP, s);
    ck(cudaStreamSynchronize(s));
}

void setup_device_end(DeviceSetup* ds) { delete ds; }

double lattice_volume_sum_device(int dim, const int n[3], const double lo[3], double spacing) {
    Grid g{};
    g.dim = dim;
    g.nx = n[0];
    g.ny = n[1];
    g.nz = dim == 3 ? n[2] : 1;
    for (int k = 0; k < 3; ++k) g.lo[k] = lo[k];
    g.h = spacing;
    const size_t E = (size_t)g.nx * g.ny * g.nz;
    cudaStream_t s = nullptr;
    ck(cudaStreamCreateWithFlags(&s, cudaStreamNonBlocking));
    double* vol = dmalloc<double>(E + 1, s);
    k_volumes<<<1184, 128, 0, s>>>(g, vol);
    k_serial_sum<<<1, 1, 0, s>>>((long long)E, vol, vol + E);
    ck(cudaGetLastError());
    double sum = 0.0;
    ck(cudaMemcpyAsync(&sum, vol + E, sizeof(double), cudaMemcpyDeviceToHost, s));
    cudaFreeAsync(vol, s);
    ck(cudaStreamSynchronize(s));
    ck(cudaStreamDestroy(s));
    return sum;
}

void element_geometry_device(int dim, int n_elems, int n_nodes, const int32_t* conn,
                             const double* nodes, double* centroid, double* volume,
                             cudaStream_t s) {
    const int nn = dim == 2 ? 4 : 8;
    const size_t E = n_elems;
    int32_t* dconn = dmalloc<int32_t>(nn * E, s);
    double* dxyz = dmalloc<double>(3 * (size_t)n_nodes, s);
    double* dcen = dmalloc<double>(3 * E, s);
    double* dvol = dmalloc<double>(E, s);
    int* bad = dmalloc<int>(1, s);
    ck(cudaMemsetAsync(bad, 0, sizeof(int), s));
    ck(cudaMemcpyAsync(dconn, conn, sizeof(int32_t) * nn * E, cudaMemcpyHostToDevice, s));
    ck(cudaMemcpyAsync(dxyz, nodes, sizeof(double) * 3 * (size_t)n_nodes, cudaMemcpyHostToDevice, s));
    k_geometry<<<1184, 128, 0, s>>>(dim, (long long)E, dconn, dxyz, dcen, dvol, bad);
    ck(cudaGetLastError());
    int hbad = 0;
    ck(cudaMemcpyAsync(centroid, dcen, sizeof(double) * 3 * E, cudaMemcpyDeviceToHost, s));
    ck(cudaMemcpyAsync(volume, dvol, sizeof(double) * E, cudaMemcpyDeviceToHost, s));
    ck(cudaMemcpyAsync(&hbad, bad, sizeof(int), cudaMemcpyDeviceToHost, s));
    for (void* p : {(void*)dconn, (void*)dxyz, (void*)dcen, (void*)dvol, (void*)bad})
        cudaFreeAsync(p, s);
    ck(cudaStreamSynchronize(s));
    if (hbad) throw ConfigError("inverted element (non-positive Jacobian)");
}

}  // namespace pmts
