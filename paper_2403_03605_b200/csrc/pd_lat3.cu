// 3D lattice bond kernel for the 122-offset stencil (delta in [3, sqrt(10)) dx,
// BASELINE cfg4/cfg5's 3.015 dx), fast mode, nominal lattice constants.
//
// On the nominal lattice xi = h (di, dj, dk) with small compile-time integers,
// and w c(|xi|) depends on |xi|^2 only (8 classes: 1,2,3,4,5,6,8,9 h^2).  The
// 122 offsets are expanded at compile time (template recursion), so every
// offset's partner address is an immediate shared-memory offset, the xi.eta
// product is a handful of adds / small-integer multiplies, and the per-offset
// constants collapse to 8 class values held in uniform registers -- no table
// loads, no bit-scan loop (the generic stencil kernel spent ~46 instructions per
// directed entry; this one ~20).
//
//   eta   = ubar_p - ubar_e
//   G_e  -= (w c h^2) (o . eta) o                      (o = integer offset, xi = h o)
//   test  2 h (o . eta) + |eta|^2 >= (2 s + s^2) h^2 |o|^2 -- the squared break test
// CTA tile 16 x 4 x 4 elements + a 3-element ubar apron staged in shared memory
// (SoA), one element per thread.  Reference semantics as in pd_stencil.cu.
#include <stdexcept>
#include <string>

#include "pd_stencil.cuh"

namespace pmts {

namespace {

constexpr int TX = 16, TY = 4, TZ = 4, R = 3;
constexpr int AX = TX + 2 * R, AY = TY + 2 * R, AZ = TZ + 2 * R;
// the ubar apron in shared memory is AoS (x, y, z per cell) with rows of AXT cells
// starting one column early (global columns i0 - 4 .. i0 + 19): the TMA box must
// start 16-byte aligned in global memory and be a multiple of 16 bytes wide
constexpr int AXT = 24, X0 = R + 1;
constexpr int NAT = AXT * AY * AZ;
constexpr int kApronBytes = NAT * 3 * 8;  // 57,600 B: three CTAs per SM
constexpr int NT = TX * TY * TZ;
constexpr int S3 = 122;

struct Off3 {
    int di[S3], dj[S3], dk[S3];
};
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
// |o|^2 -> class index (|o|^2 = 7 does not occur on the integer lattice)
__host__ __device__ constexpr int cls_of(int d2) {
    return d2 <= 6 ? d2 - 1 : d2 == 8 ? 6 : 7;
}

template <int K>
struct Ofs {
    static constexpr Off3 o = make_off3();
    static constexpr int di = o.di[K], dj = o.dj[K], dk = o.dk[K];
    static constexpr int d2 = di * di + dj * dj + dk * dk;
    static constexpr int cls = cls_of(d2);
    static constexpr int aoff = 3 * ((dk * AY + dj) * AXT + di);  // doubles
};

// c * e for a small compile-time integer c (exact for |c| <= 3 as adds)
template <int C>
__device__ __forceinline__ double imul(double e) {
    if constexpr (C == 0) return 0.0;
    else if constexpr (C == 1) return e;
    else if constexpr (C == -1) return -e;
    else if constexpr (C == 2) return e + e;
    else if constexpr (C == -2) return -(e + e);
    else return (double)C * e;
}
// acc + c * e
template <int C>
__device__ __forceinline__ double iaxpy(double acc, double e) {
    if constexpr (C == 0) return acc;
    else if constexpr (C == 1) return acc + e;
    else if constexpr (C == -1) return acc - e;
    else return fma((double)C, e, acc);
}

struct Ctx {
    const double* ua;  // AoS apron
    int q0;            // element's first double in ua
    double ex, ey, ez;
    uint32_t m[4];
    double gx, gy, gz;
    bool anyc;
};

template <int K, bool DO_BREAK>
__device__ __forceinline__ void bond(Ctx& c, const Stencil3D& st) {
    using O = Ofs<K>;
    const int q = c.q0 + O::aoff;
    const double e0 = c.ua[q] - c.ex, e1 = c.ua[q + 1] - c.ey, e2 = c.ua[q + 2] - c.ez;
    double dot = imul<O::di>(e0);
    dot = iaxpy<O::dj>(dot, e1);
    dot = iaxpy<O::dk>(dot, e2);
    const bool act = (c.m[K >> 5] >> (K & 31)) & 1u;
    const double t = act ? dot * st.c[O::cls] : 0.0;
    c.gx = iaxpy<-O::di>(c.gx, t);
    c.gy = iaxpy<-O::dj>(c.gy, t);
    c.gz = iaxpy<-O::dk>(c.gz, t);
    if (DO_BREAK) {
        const double lhs = fma(st.h2, dot, fma(e2, e2, fma(e1, e1, e0 * e0)));
        c.anyc |= act && __double_as_longlong(lhs) >= st.clo[O::cls];
    }
}

template <int K, bool DO_BREAK>
struct Unroll {
    static __device__ __forceinline__ void run(Ctx& c, const Stencil3D& st) {
        bond<K, DO_BREAK>(c, st);
        Unroll<K + 1, DO_BREAK>::run(c, st);
    }
};
template <bool DO_BREAK>
struct Unroll<S3, DO_BREAK> {
    static __device__ __forceinline__ void run(Ctx&, const Stencil3D&) {}
};

}  // namespace

bool lat3_offsets_match(const int8_t* di, const int8_t* dj, const int8_t* dk, int S) {
    if (S != S3) return false;
    constexpr Off3 o = make_off3();
    for (int s = 0; s < S3; ++s)
        if (di[s] != o.di[s] || dj[s] != o.dj[s] || dk[s] != o.dk[s]) return false;
    return true;
}
int lat3_class_of(int d2) { return cls_of(d2); }

namespace {
__device__ __forceinline__ unsigned hi_abs3(double d) {
    return (unsigned)__double2hiint(d) & 0x7fffffffu;
}
__device__ __forceinline__ double hi_bound3(unsigned m) {  // >= every |d| with hi_abs3(d) <= m
    return __hiloint2double((int)m, (int)0xffffffffu);
}

// Launch order of the 3D tiles (both kernels, a 1D grid): z fastest, then x, then y.
// A CTA's ubar apron reaches 3 layers into the z-neighbour tiles; in (x, y, z) order
// those were ~gx gy CTAs back (cfg5: 5000, ~300 MB of ubar earlier -- evicted from
// L2, the 1.48x DRAM traffic of the round-1 capture); in this order the whole z column
// of a tile and its x neighbours are adjacent in launch order, and the y neighbours
// are one (gx gz)-tile row back (cfg5: 250 tiles, a few MB).
struct Tile3 {
    int x, y, z, gx, gz;
};
__device__ __forceinline__ Tile3 tile3(const LatticeDev& L) {
    Tile3 t;
    t.gx = (L.nx + TX - 1) / TX;
    t.gz = (L.nz + TZ - 1) / TZ;
    const int b = blockIdx.x;
    t.z = b % t.gz;
    const int r = b / t.gz;
    t.x = r % t.gx;
    t.y = r / t.gx;
    return t;
}
}  // namespace

// ubar of the 3D lattice, one CTA per bond-kernel tile (16 x 4 x 4 elements), plus
// the cold-tile screen's input: per tile, the maxima over its elements' edges of
// |u(n + e_a) - u(n)|_c for axis a and component c (9 values, as the high words of
// the doubles, which order like the magnitudes).  ubar is summed in k_lat_ubar<3>'s
// order, so it is bitwise the same.
__global__ void __launch_bounds__(NT)
k_lat3_ubar(DevPD d, LatticeDev L, unsigned* tmax) {
    __shared__ unsigned red[NT / 32][9];
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    const int tx = tid % TX, ty = (tid / TX) % TY, tz = tid / (TX * TY);
    const Tile3 T = tile3(L);
    const int i = T.x * TX + tx, j = L.ub0 + T.y * TY + ty, k = T.z * TZ + tz;
    unsigned mx[9];
#pragma unroll
    for (int q = 0; q < 9; ++q) mx[q] = 0u;
    if (i < L.nx && j >= 0 && j < L.ny && k < L.nz) {
        const int NX = L.nx + 1, NY = L.ny + 1, up = NX * NY;
        const int n00 = (k * NY + j) * NX + i;
        const int nd[8] = {n00, n00 + 1, n00 + NX + 1, n00 + NX,
                           n00 + up, n00 + up + 1, n00 + up + NX + 1, n00 + up + NX};
        double u[8][3];
#pragma unroll
        for (int a = 0; a < 8; ++a)
#pragma unroll
            for (int c = 0; c < 3; ++c) u[a][c] = d.rd[(size_t)nd[a] * 3 + c];
        double s[3] = {0.0, 0.0, 0.0};
#pragma unroll
        for (int a = 0; a < 8; ++a)
#pragma unroll
            for (int c = 0; c < 3; ++c) s[c] += u[a][c];
        const int e = (k * L.ny + j) * L.nx + i;
#pragma unroll
        for (int c = 0; c < 3; ++c) d.ubar[(size_t)e * 3 + c] = d.Nsh * s[c];
        if (tmax) {
            // edges: x (0,1) (3,2) (4,5) (7,6); y (0,3) (1,2) (4,7) (5,6); z (a, a + 4)
            constexpr int EA[3][4] = {{0, 3, 4, 7}, {0, 1, 4, 5}, {0, 1, 2, 3}};
            constexpr int EB[3][4] = {{1, 2, 5, 6}, {3, 2, 7, 6}, {4, 5, 6, 7}};
#pragma unroll
            for (int ax = 0; ax < 3; ++ax)
#pragma unroll
                for (int q = 0; q < 4; ++q)
#pragma unroll
                    for (int c = 0; c < 3; ++c)
                        mx[3 * ax + c] = max(mx[3 * ax + c], hi_abs3(u[EB[ax][q]][c] - u[EA[ax][q]][c]));
        }
    }
    if (!tmax) return;
#pragma unroll
    for (int q = 0; q < 9; ++q) {
        mx[q] = __reduce_max_sync(0xffffffffu, mx[q]);
        if (lane == 0) red[warp][q] = mx[q];
    }
    __syncthreads();
    if (tid < 9) {
        unsigned v = 0u;
#pragma unroll
        for (int w = 0; w < NT / 32; ++w) v = max(v, red[w][tid]);
        tmax[((size_t)(T.z * L.ugy + T.y) * T.gx + T.x) * 9 + tid] = v;
    }
}

// Cold-tile break screen: every partner of a tile element lies in the tile or its 26
// neighbours (apron 3 < tile extents 16, 4, 4), and eta = ubar_p - ubar_e is the mean
// of the 8 node differences u(n + o) - u(n), each a sum of |o_a| edge steps along a
// monotone lattice path inside those tiles' elements: |eta_c| <= E_c = sum_a |o_a|
// D_ac, so 2h o.eta + |eta|^2 <= 2h sum_c |o_c| E_c + sum_c E_c^2.  A tile where that
// bound (x (1 + 1e-6)) stays below every offset's candidate threshold runs the force
// without the break test: bitwise the same result, no candidate could fire.
__device__ __forceinline__ bool lat3_tile_hot(const Stencil3D& st, const LatticeDev& L,
                                              const Tile3& T) {
    __shared__ unsigned dmax[9];
    const int tid = threadIdx.x;
    if (tid < 9) dmax[tid] = 0u;
    __syncthreads();
    if (tid < 27 * 9) {
        const int t = tid / 9, q = tid % 9;
        // bond tile y row T.y is ubar tile row T.y + (jb0 - ub0) / TY
        const int by0 = T.y + (L.jb0 - L.ub0) / TY;
        const int bx = T.x + t % 3 - 1, by = by0 + (t / 3) % 3 - 1, bz = T.z + t / 9 - 1;
        if (bx >= 0 && by >= 0 && bz >= 0 && bx < T.gx && by < L.ugy && bz < T.gz)
            atomicMax(&dmax[q], st.tmax[((size_t)(bz * L.ugy + by) * T.gx + bx) * 9 + q]);
    }
    __syncthreads();
    bool h = false;
    if (tid < S3) {
        const double a0 = fabs((double)L.di[tid]), a1 = fabs((double)L.dj[tid]),
                     a2 = fabs((double)L.dk[tid]);
        double D[9];
#pragma unroll
        for (int q = 0; q < 9; ++q) D[q] = hi_bound3(dmax[q]);
        const double E0 = a0 * D[0] + a1 * D[3] + a2 * D[6];
        const double E1 = a0 * D[1] + a1 * D[4] + a2 * D[7];
        const double E2 = a0 * D[2] + a1 * D[5] + a2 * D[8];
        const int d2 = (int)(a0 * a0 + a1 * a1 + a2 * a2);
        const double bound =
            fma(st.h2, a0 * E0 + a1 * E1 + a2 * E2, E0 * E0 + E1 * E1 + E2 * E2) * (1.0 + 1e-6);
        h = !(bound < __longlong_as_double(st.clo[cls_of(d2)]));
    }
    return __syncthreads_or(h);
}

__device__ __forceinline__ unsigned smem_u32(const void* p) {
    return (unsigned)__cvta_generic_to_shared(p);
}

template <bool DO_BREAK>
__global__ void __launch_bounds__(NT, 3)
k_lat3_bond(DevPD d, LatticeDev L, const __grid_constant__ Stencil3D st, int step) {
    extern __shared__ __align__(16) unsigned char smraw[];
    // realign the dynamic base to 128 bytes for the TMA destination
    double* ua = reinterpret_cast<double*>(smraw + ((128u - (smem_u32(smraw) & 127u)) & 127u));
    uint64_t* bar = reinterpret_cast<uint64_t*>(ua + 3 * NAT);
    const int tid = threadIdx.x;
    const Tile3 T = tile3(L);
    const int i0 = T.x * TX, j0 = L.jb0 + T.y * TY, k0 = T.z * TZ;
    if (st.use_tma) {
        // one bulk tensor copy of the apron; out-of-domain boxes arrive zero-filled
        if (tid == 0) {
            asm volatile("mbarrier.init.shared.b64 [%0], 1;\n" ::"r"(smem_u32(bar)));
            asm volatile("fence.mbarrier_init.release.cluster;\n" ::);
            asm volatile("mbarrier.arrive.expect_tx.shared.b64 _, [%0], %1;\n" ::"r"(smem_u32(bar)),
                         "r"(kApronBytes));
            asm volatile(
                "cp.async.bulk.tensor.3d.shared::cluster.global.mbarrier::complete_tx::bytes"
                " [%0], [%1, {%2, %3, %4}], [%5];\n" ::"r"(smem_u32(ua)),
                "l"(&st.ub), "r"(3 * (i0 - X0)), "r"(j0 - R), "r"(k0 - R), "r"(smem_u32(bar))
                : "memory");
        }
    } else {
        for (int q = tid; q < NAT; q += NT) {
            const int ax = q % AXT, r = q / AXT;
            const int ay = r % AY, az = r / AY;
            const int gi = i0 + ax - X0, gj = j0 + ay - R, gk = k0 + az - R;
            const bool in = gi >= 0 && gj >= 0 && gk >= 0 && gi < L.nx && gj < L.ny && gk < L.nz;
            const size_t ge = ((size_t)gk * L.ny + gj) * L.nx + gi;
#pragma unroll
            for (int c = 0; c < 3; ++c) ua[3 * q + c] = in ? d.ubar[ge * 3 + c] : 0.0;
        }
    }
    bool hot = DO_BREAK;
    if (DO_BREAK && st.tmax) {
        hot = lat3_tile_hot(st, L, T);  // (its barriers also close the staging)
        if (st.hot_count && tid == 0) {
            atomicAdd(st.hot_count, hot ? 1ull : 0ull);
            atomicAdd(st.hot_count + 1, 1ull);
        }
    } else {
        __syncthreads();
    }
    const int tx = tid % TX, ty = (tid / TX) % TY, tz = tid / (TX * TY);
    const int gi = i0 + tx, gj = j0 + ty, gk = k0 + tz;
    const bool own = gi < L.nx && gj < L.jb1 && gk < L.nz;
    const int e = own ? (gk * L.ny + gj) * L.nx + gi : 0;
    uint32_t m4[4] = {0u, 0u, 0u, 0u};  // bond states, loaded while the apron is in flight
    if (own) {
#pragma unroll
        for (int w = 0; w < 4; ++w) m4[w] = d.mask[(size_t)w * d.E + e];
    }
    if (st.use_tma) {
        asm volatile(
            "{\n"
            ".reg .pred P1;\n"
            "WAIT_%=:\n"
            "mbarrier.try_wait.parity.shared.b64 P1, [%0], 0;\n"
            "@!P1 bra WAIT_%=;\n"
            "}\n" ::"r"(smem_u32(bar)));
    }
    unsigned long long nb = 0;
    if (own) {
        Ctx c;
        c.ua = ua;
        c.q0 = 3 * (((tz + R) * AY + ty + R) * AXT + tx + X0);
        c.ex = ua[c.q0];
        c.ey = ua[c.q0 + 1];
        c.ez = ua[c.q0 + 2];
#pragma unroll
        for (int w = 0; w < 4; ++w) c.m[w] = m4[w];
        c.gx = c.gy = c.gz = 0.0;
        c.anyc = false;
        if (hot) Unroll<0, DO_BREAK>::run(c, st);
        else Unroll<0, false>::run(c, st);
        if (DO_BREAK && c.anyc) {  // rare: exact per-bond thresholds (generic table)
            uint32_t mw[4] = {c.m[0], c.m[1], c.m[2], c.m[3]};
            for (int w = 0; w < 4; ++w) {
                uint32_t live = c.m[w];
                while (live) {
                    const int b = __ffs(live) - 1;
                    live &= live - 1;
                    const int s = 32 * w + b;
                    const int a = c.q0 + 3 * ((L.dk[s] * AY + L.dj[s]) * AXT + L.di[s]);
                    const double e0 = ua[a] - c.ex, e1 = ua[a + 1] - c.ey, e2 = ua[a + 2] - c.ez;
                    const double dot = fma((double)L.dk[s], e2,
                                           fma((double)L.dj[s], e1, (double)L.di[s] * e0));
                    const double lhs = fma(st.h2, dot, fma(e2, e2, fma(e1, e1, e0 * e0)));
                    const int d2 = L.di[s] * L.di[s] + L.dj[s] * L.dj[s] + L.dk[s] * L.dk[s];
                    const int p = e + L.delta_id[s];
                    double thr = __longlong_as_double(st.cthr[cls_of(d2)]);
                    if (d.spread != 0.0) {
                        const double sb = bond_s_crit(d.s_crit, d.spread, d.seed,
                                                      global_elem(d, e < p ? e : p),
                                                      global_elem(d, e < p ? p : e));
                        thr = fma(sb, sb, 2.0 * sb) * st.hh * d2;
                    }
                    if (lhs >= thr) {
                        mw[w] &= ~(1u << b);
                        if (p > e && owns_elem(d, e)) ++nb;
                    }
                }
                if (mw[w] != c.m[w]) d.mask[(size_t)w * d.E + e] = mw[w];
            }
        }
        d.G[(size_t)e * 3] = c.gx;
        d.G[(size_t)e * 3 + 1] = c.gy;
        d.G[(size_t)e * 3 + 2] = c.gz;
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

// Row tiling of a slab: the bond tiles start at element row jb0; the ubar tiles are
// aligned with them (rows ub0 + TY b, ub0 = jb0 - TY ceil(jb0 / TY) <= 0) and cover
// every element row, so the screen's 27-tile neighbourhood is the bond tile's own.
void lat3_rows(LatticeDev& L) {
    L.ub0 = L.jb0 - TY * ((L.jb0 + TY - 1) / TY);
    L.ugy = (L.ny - L.ub0 + TY - 1) / TY;
}
void launch_lat3_ubar(const DevPD& d, const LatticeDev& L, unsigned* tmax, cudaStream_t s) {
    const unsigned grid = (unsigned)((L.nx + TX - 1) / TX) * L.ugy * ((L.nz + TZ - 1) / TZ);
    k_lat3_ubar<<<grid, NT, 0, s>>>(d, L, tmax);
}
void lat3_apron_box(int* bx, int* by, int* bz) {
    *bx = 3 * AXT;
    *by = AY;
    *bz = AZ;
}
size_t lat3_tile_count(const LatticeDev& L) {
    return (size_t)((L.nx + TX - 1) / TX) * L.ugy * ((L.nz + TZ - 1) / TZ);
}

void launch_lat3_bond(const DevPD& d, const LatticeDev& L, const Stencil3D& st, int step,
                      int do_break, cudaStream_t s) {
    const unsigned grid = (unsigned)((L.nx + TX - 1) / TX) * ((L.jb1 - L.jb0 + TY - 1) / TY) *
                          ((L.nz + TZ - 1) / TZ);
    constexpr size_t smem = kApronBytes + 8 + 128;  // + mbarrier + realignment slack
    static bool configured = false;
    if (!configured) {
        for (auto fn : {k_lat3_bond<true>, k_lat3_bond<false>})
            cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
        configured = true;
    }
    if (do_break) k_lat3_bond<true><<<grid, NT, smem, s>>>(d, L, st, step);
    else k_lat3_bond<false><<<grid, NT, smem, s>>>(d, L, st, step);
    cudaError_t e = cudaGetLastError();
    if (e != cudaSuccess) throw std::runtime_error(std::string("CUDA: ") + cudaGetErrorString(e));
}

}  // namespace pmts
