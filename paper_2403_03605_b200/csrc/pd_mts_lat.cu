// Linear PD force of the coupled integrator's homogeneous substeps on a 3D box lattice
// (BASELINE cfg5: the 400 x 800 x 40 PD core, 1.56e9 directed entries).
//
// The general form (pd_mts.cu, k_pd_force_lin_t) runs a warp per element over the ELL
// family and gathers every partner's ubar and centroid through L1: 22 ms per substep at
// cfg5, L1-bound (profiles/r02_cfg5_mts_ncu_force_lin.txt), and the interface CG applies
// ~500 substeps per macro step.  When the PD elements of the handle are a full box of
// the generated lattice in lattice order and every family entry is one of the 122
// offsets of the 3.015 dx stencil, the same operator
//
//     G_e = - sum_p coef_ep (xi . (ubar_p - ubar_e)) xi ,   coef_ep = (1 - alpha) V_e V_p c(|xi|)
//
// runs here with one element per thread over a 16 x 4 x 4 tile whose ubar apron sits in
// shared memory: the per-entry coefficients are re-laid in STENCIL order, each bond's once
// (coefS[s E + e] for the 61 positive offsets: one coalesced 8-byte stream per offset,
// absent entries 0; the upper element reads its partner's copy), the bond
// states of the k_sync snapshot as 122 stencil bits per element, and xi = h o is the
// nominal lattice vector (compile-time integers; the ELL form subtracts centroids, a
// 1e-16-level difference).  The coefficients are the very values the ELL form
// multiplies, so the two operators differ by rounding only
// (tests/test_gpu_cfg5_mts.py::test_lattice_linear_force_matches_ell).
// Reference: apply_h_pd / unit_pd_column's substeps, mts.hpp:230-238, 398-420.
#include <cstdint>
#include <stdexcept>
#include <string>
#include <vector>

#include "pd_common.cuh"
#include "pd_mts.cuh"

namespace pmts {
namespace mtsk {

namespace {

constexpr int TX = 16, TY = 4, TZ = 4, R = 3;
constexpr int AX = TX + 2 * R, AY = TY + 2 * R, AZ = TZ + 2 * R;
constexpr int NAT = AX * AY * AZ;  // apron cells (AoS x, y, z): 52,800 B, three CTAs per SM
constexpr int NT = TX * TY * TZ;
constexpr int S3 = 122;

struct Off3 {
    int di[S3], dj[S3], dk[S3];
};
// the 122 offsets with 1 <= |o|^2 <= 9, z slowest (pd_lat3.cu's order)
__host__ __device__ constexpr Off3 make_off3() {
    Off3 o{};
    int n = 0;
    for (int k = -3; k <= 3; ++k)
        for (int j = -3; j <= 3; ++j)
            for (int i = -3; i <= 3; ++i) {
                const int d2 = i * i + j * j + k * k;
                if (d2 == 0 || d2 > 9) continue;
                o.di[n] = i;
                o.dj[n] = j;
                o.dk[n] = k;
                ++n;
            }
    return o;
}
template <int K>
struct Ofs {
    static constexpr Off3 o = make_off3();
    static constexpr int di = o.di[K], dj = o.dj[K], dk = o.dk[K];
    static constexpr int aoff = 3 * ((dk * AY + dj) * AX + di);  // doubles
};

// c * e and acc + c * e for a small compile-time integer c
template <int C>
__device__ __forceinline__ double imul(double e) {
    if constexpr (C == 0) return 0.0;
    else if constexpr (C == 1) return e;
    else if constexpr (C == -1) return -e;
    else return (double)C * e;
}
template <int C>
__device__ __forceinline__ double iaxpy(double acc, double e) {
    if constexpr (C == 0) return acc;
    else if constexpr (C == 1) return acc + e;
    else if constexpr (C == -1) return acc - e;
    else return fma((double)C, e, acc);
}

struct Ctx {
    const double* ua;
    const double* coef;  // coefS + e
    size_t E;
    int nx, nxy;         // element-id strides of a y / z step
    int q0;
    double ex, ey, ez;
    uint32_t m[4];
    double gx, gy, gz;
};

template <int K>
__device__ __forceinline__ void entry(Ctx& c) {
    using O = Ofs<K>;
    const int q = c.q0 + O::aoff;
    const double e0 = c.ua[q] - c.ex, e1 = c.ua[q + 1] - c.ey, e2 = c.ua[q + 2] - c.ez;
    double dot = imul<O::di>(e0);
    dot = iaxpy<O::dj>(dot, e1);
    dot = iaxpy<O::dk>(dot, e2);
    // A bond's coefficient is stored once, at its lower element under the positive
    // offset (slot K - 61); the entry of the upper element reads it there (e + o is the
    // partner, which exists whenever the bit is set).  The loads depend on nothing but the
    // bond states read at kernel start, so the compiler can issue them far ahead of their
    // use: the kernel lives on loads in flight.
    const bool act = (c.m[K >> 5] >> (K & 31)) & 1u;
    double cf;
    if constexpr (K >= S3 / 2) {
        cf = c.coef[(size_t)(K - S3 / 2) * c.E];
    } else {
        const int lin = O::dk * c.nxy + O::dj * c.nx + O::di;
        cf = act ? c.coef[(size_t)(S3 / 2 - 1 - K) * c.E + lin] : 0.0;
    }
    const double t = act ? cf * dot : 0.0;
    c.gx = iaxpy<-O::di>(c.gx, t);
    c.gy = iaxpy<-O::dj>(c.gy, t);
    c.gz = iaxpy<-O::dk>(c.gz, t);
}
template <int K>
struct Unroll {
    static __device__ __forceinline__ void run(Ctx& c) {
        entry<K>(c);
        Unroll<K + 1>::run(c);
    }
};
template <>
struct Unroll<S3> {
    static __device__ __forceinline__ void run(Ctx&) {}
};

__device__ __forceinline__ void ijk(int e, int nx, int ny, int& i, int& j, int& k) {
    i = e % nx;
    const int r = e / nx;
    j = r % ny;
    k = r / ny;
}
// stencil slot of the family entry e -> p (-1: not one of the 122 offsets)
__device__ __forceinline__ int slot_of(const LinLat& L, int e, int p) {
    int a, b, c, x, y, z;
    ijk(e, L.nx, L.ny, a, b, c);
    ijk(p, L.nx, L.ny, x, y, z);
    const int di = x - a, dj = y - b, dk = z - c;
    if (di < -3 || di > 3 || dj < -3 || dj > 3 || dk < -3 || dk > 3) return -1;
    return L.slot[((dk + 3) * 7 + dj + 3) * 7 + di + 3];
}

// pass 0: coefS[(s - 61) E + e] = the coefficient of the entry of e with the positive
// offset s (coefS zeroed before); pass 1: every entry with a negative offset carries the
// very bits stored at its partner under the opposite offset (the bond's one coefficient)
__global__ void k_lin_lat_build(DevPD d, LinLat L, int pass, int* err) {
    const long long q = (long long)blockIdx.x * blockDim.x + threadIdx.x;  // q = k E + e
    if (q >= (long long)d.K * d.E) return;
    const int e = (int)(q % d.E);
    const int p = d.col[q];
    if (p < 0) return;
    const int s = slot_of(L, e, p);
    if (s < 0) {
        *err = 1;
        return;
    }
    if (pass == 0) {
        if (s >= S3 / 2) L.coefS[(size_t)(s - S3 / 2) * d.E + e] = d.coef[q];
    } else if (s < S3 / 2) {
        if (__double_as_longlong(L.coefS[(size_t)(S3 / 2 - 1 - s) * d.E + p]) !=
            __double_as_longlong(d.coef[q]))
            *err = 2;
    }
}

// the ELL bond states (bit k of word k / 32) as stencil bits
__global__ void k_lin_lat_mask(DevPD d, LinLat L, const uint32_t* __restrict__ mask) {
    const int e = blockIdx.x * blockDim.x + threadIdx.x;
    if (e >= d.E) return;
    uint32_t w[4] = {0u, 0u, 0u, 0u};
    uint32_t word = 0u;
    for (int k = 0; k < d.K; ++k) {
        if ((k & 31) == 0) word = mask[(size_t)(k >> 5) * d.E + e];
        const int p = d.col[(size_t)k * d.E + e];
        if (p < 0 || !((word >> (k & 31)) & 1u)) continue;
        const int s = slot_of(L, e, p);
        if (s >= 0) w[s >> 5] |= 1u << (s & 31);
    }
#pragma unroll
    for (int q = 0; q < 4; ++q) L.maskS[(size_t)q * d.E + e] = w[q];
}

__global__ void __launch_bounds__(NT, 3)
k_pd_force_lin_lat(DevPD d, LinLat L, const double* __restrict__ ub) {
    extern __shared__ double ua[];
    const int tid = threadIdx.x;
    const int gx = (L.nx + TX - 1) / TX, gz = (L.nz + TZ - 1) / TZ;
    // tiles z fastest, then x, then y: a tile's z neighbours (whose ubar its apron
    // re-reads) are adjacent in launch order (pd_lat3.cu)
    const int b = blockIdx.x, tzb = b % gz, r = b / gz, txb = r % gx, tyb = r / gx;
    const int i0 = txb * TX, j0 = tyb * TY, k0 = tzb * TZ;
    for (int q = tid; q < NAT; q += NT) {
        const int ax = q % AX, rr = q / AX;
        const int ay = rr % AY, az = rr / AY;
        const int gi = i0 + ax - R, gj = j0 + ay - R, gk = k0 + az - R;
        const bool in = gi >= 0 && gj >= 0 && gk >= 0 && gi < L.nx && gj < L.ny && gk < L.nz;
        const size_t ge = ((size_t)gk * L.ny + gj) * L.nx + gi;
#pragma unroll
        for (int c = 0; c < 3; ++c) ua[3 * q + c] = in ? ub[ge * 3 + c] : 0.0;
    }
    const int tx = tid % TX, ty = (tid / TX) % TY, tz = tid / (TX * TY);
    const int gi = i0 + tx, gj = j0 + ty, gk = k0 + tz;
    const bool own = gi < L.nx && gj < L.ny && gk < L.nz;
    const int e = own ? (gk * L.ny + gj) * L.nx + gi : 0;
    Ctx c;
#pragma unroll
    for (int w = 0; w < 4; ++w) c.m[w] = own ? L.maskS[(size_t)w * d.E + e] : 0u;
    __syncthreads();
    if (!own) return;
    c.ua = ua;
    c.coef = L.coefS + e;
    c.E = (size_t)d.E;
    c.nx = L.nx;
    c.nxy = L.nx * L.ny;
    c.q0 = 3 * (((tz + R) * AY + ty + R) * AX + tx + R);
    c.ex = ua[c.q0];
    c.ey = ua[c.q0 + 1];
    c.ez = ua[c.q0 + 2];
    c.gx = c.gy = c.gz = 0.0;
    Unroll<0>::run(c);
    // xi = h o on both factors
    const double hh = L.h * L.h;
    d.G[(size_t)e * 3] = hh * c.gx;
    d.G[(size_t)e * 3 + 1] = hh * c.gy;
    d.G[(size_t)e * 3 + 2] = hh * c.gz;
}

void check_last(const char* what) {
    cudaError_t e = cudaGetLastError();
    if (e != cudaSuccess)
        throw std::runtime_error(std::string("CUDA (") + what + "): " + cudaGetErrorString(e));
}

}  // namespace

void lin_lat_slot_table(int8_t* table343) {
    constexpr Off3 o = make_off3();
    for (int q = 0; q < 343; ++q) table343[q] = -1;
    for (int s = 0; s < S3; ++s)
        table343[((o.dk[s] + 3) * 7 + o.dj[s] + 3) * 7 + o.di[s] + 3] = (int8_t)s;
}
int lin_lat_stencil_size() { return S3; }
int lin_lat_coef_slots() { return S3 / 2; }

bool lin_lat_build(const DevPD& d, const LinLat& L, cudaStream_t s) {
    int* err = nullptr;
    if (cudaMalloc(&err, sizeof(int)) != cudaSuccess) throw std::runtime_error("CUDA: cudaMalloc");
    cudaMemsetAsync(err, 0, sizeof(int), s);
    cudaMemsetAsync(L.coefS, 0, sizeof(double) * (size_t)(S3 / 2) * d.E, s);
    const long long n = (long long)d.K * d.E;
    for (int pass = 0; pass < 2; ++pass)
        k_lin_lat_build<<<(unsigned)((n + 255) / 256), 256, 0, s>>>(d, L, pass, err);
    check_last("lin_lat_build");
    int h = 0;
    cudaMemcpyAsync(&h, err, sizeof(int), cudaMemcpyDeviceToHost, s);
    cudaStreamSynchronize(s);
    cudaFree(err);
    check_last("lin_lat_build");
    return h == 0;
}

void lin_lat_mask(const DevPD& d, const LinLat& L, const uint32_t* mask, cudaStream_t s) {
    k_lin_lat_mask<<<(d.E + 255) / 256, 256, 0, s>>>(d, L, mask);
    check_last("lin_lat_mask");
}

void pd_force_lin_lat(const DevPD& d, const LinLat& L, const double* x, double* ubar,
                      cudaStream_t s) {
    pd_ubar(d, x, ubar, s);
    constexpr int smem = NAT * 3 * 8;
    static bool configured = false;
    if (!configured) {
        cudaFuncSetAttribute(k_pd_force_lin_lat, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
        configured = true;
    }
    const unsigned grid = (unsigned)((L.nx + TX - 1) / TX) * ((L.ny + TY - 1) / TY) *
                          ((L.nz + TZ - 1) / TZ);
    k_pd_force_lin_lat<<<grid, NT, smem, s>>>(d, L, ubar);
    check_last("pd_force_lin_lat");
}

}  // namespace mtsk
}  // namespace pmts
