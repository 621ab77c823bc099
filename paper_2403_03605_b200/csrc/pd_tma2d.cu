// TMA-pipelined persistent fused fine step for 2D lattices with the 28-offset
// stencil (delta in [3, sqrt(10)) dx; BASELINE's 3.015 dx), fast mode.
//
// Same arithmetic as the one-shot tile kernel (pd_stencil_fused.cu) -- each
// tile owns 31 x 31 elements and the nodes at their lower-left corners, forms
// the centroid displacements of its element apron from a node apron, evaluates
// the forces of the 32 x 32 elements its nodes need and updates the owned
// nodes -- but the memory side is the Blackwell one:
//   * persistent CTAs walk the tiles; one elected thread issues
//     cp.async.bulk.tensor (TMA) loads into shared memory that complete on
//     mbarriers: the node apron of tile t+1 lands while tile t computes
//     (double buffer), and the node-update inputs of tile t (rv and the packed
//     {1/M, flags}) land during its force pass;
//   * out-of-domain parts of a box are zero-filled by the TMA unit, so no
//     thread spends instructions on address arithmetic or bounds checks for the
//     loads (the ncu source page of the one-shot kernel put ~60% of the stall
//     samples on exactly those two load phases).
// 8 warps; lane = column of the 32-wide force region, warp w owns rows
// 4w..4w+3 (each per-offset constant is fetched once per thread for 4
// elements).  Reference semantics as in pd_stencil.cu.
#include <algorithm>
#include <stdexcept>
#include <string>

#include "pd_stencil.cuh"

namespace pmts {

namespace {

constexpr int TX = 31, TY = 31, R = kFusedR;
constexpr int GX = TX + 1, GY = TY + 1;          // force region (elements)
constexpr int AX = GX + 2 * R, AY = GY + 2 * R;  // ubar apron (elements)
constexpr int BX = AX + 1, BY = AY + 1;          // node apron
constexpr int NT = 256;
constexpr int EPT = GY / (NT / 32);              // 4 rows per warp
constexpr int NX_IN = GX, NY_IN = GY;            // node-input box (covers 31 or 32 nodes)
static_assert(GX == 32 && EPT * (NT / 32) == GY, "lane = column, warp = EPT rows");
static_assert(AX == kFusedAX, "the Stencil2D apron offsets assume this width");

// shared layout (bytes): two node aprons, rv box, aux box, ubar apron (G aliases it)
constexpr int kApronBytes = BX * BY * 16;
constexpr int kInBytes = NX_IN * NY_IN * 16;
constexpr int kApronOff0 = 0;
constexpr int kApronOff1 = ((kApronBytes + 127) / 128) * 128;
constexpr int kRvOff = kApronOff1 + ((kApronBytes + 127) / 128) * 128;
constexpr int kAuxOff = kRvOff + kInBytes;
constexpr int kUbOff = kAuxOff + kInBytes;
constexpr int kSmem = kUbOff + AX * AY * 16 + 128;  // + alignment slack

__device__ inline unsigned smem_u32(const void* p) {
    return (unsigned)__cvta_generic_to_shared(p);
}
__device__ inline void mbar_init(uint64_t* b, unsigned count) {
    asm volatile("mbarrier.init.shared.b64 [%0], %1;\n" ::"r"(smem_u32(b)), "r"(count));
}
__device__ inline void mbar_expect_tx(uint64_t* b, unsigned bytes) {
    asm volatile("mbarrier.arrive.expect_tx.shared.b64 _, [%0], %1;\n" ::"r"(smem_u32(b)),
                 "r"(bytes));
}
__device__ inline void mbar_wait(uint64_t* b, unsigned phase) {
    asm volatile(
        "{\n"
        ".reg .pred P1;\n"
        "WAIT_%=:\n"
        "mbarrier.try_wait.parity.shared.b64 P1, [%0], %1;\n"
        "@!P1 bra WAIT_%=;\n"
        "}\n" ::"r"(smem_u32(b)),
        "r"(phase));
}
__device__ inline void tma_load_2d(void* dst, const CUtensorMap* map, int x, int y, uint64_t* b) {
    asm volatile(
        "cp.async.bulk.tensor.2d.shared::cluster.global.mbarrier::complete_tx::bytes"
        " [%0], [%1, {%2, %3}], [%4];\n" ::"r"(smem_u32(dst)),
        "l"(map), "r"(x), "r"(y), "r"(smem_u32(b))
        : "memory");
}

}  // namespace

template <bool DO_BREAK>
__global__ void __launch_bounds__(NT, 2)
k_tma2d(DevPD d, LatticeDev L, const __grid_constant__ Stencil2D st,
        const __grid_constant__ TmaMaps maps, FusedBufs bf, int step, double scale,
        int write_state) {
    extern __shared__ __align__(128) unsigned char smraw[];
    unsigned char* sm = reinterpret_cast<unsigned char*>(
        (reinterpret_cast<uintptr_t>(smraw) + 127) & ~uintptr_t(127));
    __shared__ __align__(8) uint64_t bar[3];  // apron stage 0, apron stage 1, node inputs
    double2* ub = reinterpret_cast<double2*>(sm + kUbOff);
    double2* gt = ub;  // G aliases the ubar apron once the force pass is done
    const double2* rvs = reinterpret_cast<const double2*>(sm + kRvOff);
    const double2* aux = reinterpret_cast<const double2*>(sm + kAuxOff);
    const int tid = threadIdx.x;
    const int nx = L.nx, ny = L.ny, NX = nx + 1, NY = ny + 1;
    const int tiles_x = (nx + TX - 1) / TX, tiles_y = (ny + TY - 1) / TY;
    const int n_tiles = tiles_x * tiles_y;
    const CUtensorMap* rd_map = &maps.rd;  // the map of bf.rd_in
    if (tid == 0) {
        mbar_init(&bar[0], 1);
        mbar_init(&bar[1], 1);
        mbar_init(&bar[2], 1);
        asm volatile("fence.mbarrier_init.release.cluster;\n" ::);
    }
    __syncthreads();
    auto issue_apron = [&](int tile, int stage) {
        const int i0 = (tile % tiles_x) * TX, j0 = (tile / tiles_x) * TY;
        mbar_expect_tx(&bar[stage], kApronBytes);
        tma_load_2d(sm + (stage ? kApronOff1 : kApronOff0), rd_map, 2 * (i0 - 1 - R),
                    j0 - 1 - R, &bar[stage]);
    };
    if (tid == 0 && (int)blockIdx.x < n_tiles) issue_apron(blockIdx.x, 0);

    unsigned long long nb = 0;
    unsigned ph_apron[2] = {0u, 0u}, ph_in = 0u;
    int stage = 0;
    for (int tile = blockIdx.x; tile < n_tiles; tile += gridDim.x, stage ^= 1) {
        const int tix = tile % tiles_x, tiy = tile / tiles_x;
        const int i0 = tix * TX, j0 = tiy * TY;
        if (tid == 0) {
            asm volatile("fence.proxy.async.shared::cta;\n" ::);
            // node-update inputs of this tile, then the next tile's apron
            mbar_expect_tx(&bar[2], 2 * kInBytes);
            tma_load_2d(sm + kRvOff, &maps.rv, 2 * i0, j0, &bar[2]);
            tma_load_2d(sm + kAuxOff, &maps.aux, 2 * i0, j0, &bar[2]);
            if (tile + (int)gridDim.x < n_tiles) issue_apron(tile + gridDim.x, stage ^ 1);
        }
        const double2* nt =
            reinterpret_cast<const double2*>(sm + (stage ? kApronOff1 : kApronOff0));

        // masks of this thread's force-region elements (column gx = lane, rows EPT*warp + r)
        const int gx = tid & 31, gy0 = (tid >> 5) * EPT;
        const int ei = i0 - 1 + gx;
        int e[EPT];
        uint32_t m0[EPT], m[EPT];
#pragma unroll
        for (int r = 0; r < EPT; ++r) {
            const int ej = j0 - 1 + gy0 + r;
            const bool in = ei >= 0 && ej >= 0 && ei < nx && ej < ny;
            e[r] = in ? ej * nx + ei : -1;
            m0[r] = in ? bf.mask_in[e[r]] : 0u;
            m[r] = m0[r];
        }
        mbar_wait(&bar[stage], ph_apron[stage]);
        ph_apron[stage] ^= 1u;
        for (int q = tid; q < AX * AY; q += NT) {
            const int ax = q % AX, ay = q / AX;
            const double2 a = nt[ay * BX + ax], b = nt[ay * BX + ax + 1];
            const double2 c = nt[(ay + 1) * BX + ax + 1], f = nt[(ay + 1) * BX + ax];
            ub[q] = make_double2(d.Nsh * (((a.x + b.x) + c.x) + f.x),
                                 d.Nsh * (((a.y + b.y) + c.y) + f.y));
        }
        __syncthreads();

        double2 ue[EPT];
        double G0[EPT], G1[EPT];
        const int q0 = (gy0 + R) * AX + gx + R;
#pragma unroll
        for (int r = 0; r < EPT; ++r) {
            ue[r] = ub[q0 + r * AX];
            G0[r] = 0.0;
            G1[r] = 0.0;
        }
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
        if (DO_BREAK) {  // rare: exact per-bond thresholds for the flagged elements
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
        for (int r = 0; r < EPT; ++r)
            if (e[r] >= 0 && gx >= 1 && gy0 + r >= 1) bf.mask_out[e[r]] = m[r];
        __syncthreads();  // all reads of ub done: G may overwrite it
#pragma unroll
        for (int r = 0; r < EPT; ++r) gt[(gy0 + r) * GX + gx] = make_double2(G0[r], G1[r]);
        mbar_wait(&bar[2], ph_in);
        ph_in ^= 1u;
        __syncthreads();

        // Verlet update of the owned nodes (the last tile row/column also owns the
        // domain's far node line); inputs from the TMA boxes
        const int ox = (tix == tiles_x - 1) ? NX - i0 : TX;
        const int oy = (tiy == tiles_y - 1) ? NY - j0 : TY;
        double2* rdo = reinterpret_cast<double2*>(bf.rd_out);
        double2* rv2 = reinterpret_cast<double2*>(d.rv);
        const double2* P2 = reinterpret_cast<const double2*>(d.P);
        for (int q = tid; q < ox * oy; q += NT) {
            const int lx = q % ox, ly = q / ox;
            const size_t n = (size_t)(j0 + ly) * NX + i0 + lx;
            const double2 a = gt[ly * GX + lx], b = gt[ly * GX + lx + 1];
            const double2 c = gt[(ly + 1) * GX + lx], f = gt[(ly + 1) * GX + lx + 1];
            const double k0 = d.Nsh * ((a.x + b.x) + (c.x + f.x));
            const double k1 = d.Nsh * ((a.y + b.y) + (c.y + f.y));
            const double2 ax2 = aux[ly * NX_IN + lx];  // {1/M, flags}
            const int fl = (int)ax2.y;
            const double im = ax2.x;
            double2 p = make_double2(0.0, 0.0);
            if (fl & 8) {
                p = P2[n];
                p.x *= scale;
                p.y *= scale;
            }
            const double a0 = (fl & 1) ? 0.0 : (p.x - k0) * im;
            const double a1 = (fl & 2) ? 0.0 : (p.y - k1) * im;
            const double2 rv = rvs[ly * NX_IN + lx];
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
            rdo[n] = make_double2(u0 + d.dt * v0 + d.c_pred_d * a0,
                                  u1 + d.dt * v1 + d.c_pred_d * a1);
        }
        __syncthreads();  // the buffers of this tile are refilled next iteration
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

namespace {
int g_tma_grid = 0;
}

int tma2d_tile_x() { return TX; }
int tma2d_tile_y() { return TY; }
int tma2d_apron_box_x() { return 2 * BX; }
int tma2d_apron_box_y() { return BY; }
int tma2d_in_box_x() { return 2 * NX_IN; }
int tma2d_in_box_y() { return NY_IN; }

void tma2d_configure() {
    for (auto fn : {k_tma2d<true>, k_tma2d<false>}) {
        cudaError_t e = cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, kSmem);
        if (e != cudaSuccess)
            throw std::runtime_error(std::string("CUDA: ") + cudaGetErrorString(e));
    }
    int dev = 0, sms = 0, occ = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, k_tma2d<true>, NT, kSmem);
    g_tma_grid = sms * (occ > 0 ? occ : 1);
}

void launch_tma2d_step(const DevPD& d, const LatticeDev& L, const Stencil2D& st,
                       const TmaMaps& maps, const FusedBufs& b, int step, int do_break,
                       double scale, int write_state, cudaStream_t s) {
    const int n_tiles = ((L.nx + TX - 1) / TX) * ((L.ny + TY - 1) / TY);
    const int grid = std::min(n_tiles, g_tma_grid > 0 ? g_tma_grid : n_tiles);
    if (do_break)
        k_tma2d<true><<<grid, NT, kSmem, s>>>(d, L, st, maps, b, step, scale, write_state);
    else
        k_tma2d<false><<<grid, NT, kSmem, s>>>(d, L, st, maps, b, step, scale, write_state);
    cudaError_t e = cudaGetLastError();
    if (e != cudaSuccess) throw std::runtime_error(std::string("CUDA: ") + cudaGetErrorString(e));
}

}  // namespace pmts
