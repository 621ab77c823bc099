// Host orchestration of the PD fine-step handle behind include/pmts_capi.h.
//
// One handle = one CUDA stream + device-resident mesh, families, bond state
// and kinematics.  The per-step work is two (deterministic) or three (fast)
// kernel launches -- bond gather, node update (+ fused predictor) -- replayed
// from a CUDA graph per step batch.  Citations: /root/reference/proj/include/
// perimts/<file>:<line>.
#include <cstdio>
#include <algorithm>
#include <array>
#include <cmath>
#include <cstdlib>
#include <cstring>
#include <map>
#include <memory>
#include <string>
#include <thread>
#include <vector>

#include <dlfcn.h>
#include <cudaTypedefs.h>
#include <nccl.h>

#include "pd_common.cuh"
#include "pd_mts.cuh"
#include "pd_stencil.cuh"

namespace pmts {
// compute_element_geometry on the device (pd_setup.cu)
void element_geometry_device(int dim, int n_elems, int n_nodes, const int32_t* conn,
                             const double* nodes, double* centroid, double* volume, cudaStream_t s);
}
#include "pmts_internal.h"
#include "nccl_rt.h"

using namespace pmts;

#define CK(x)                                                                           \
    do {                                                                                \
        cudaError_t err_ = (x);                                                         \
        if (err_ != cudaSuccess)                                                        \
            throw InternalError(std::string("CUDA: ") + cudaGetErrorString(err_) + " (" + \
                                #x + ")");                                              \
    } while (0)

namespace {

template <class T>
T* dalloc(size_t n, double& bytes) {
    T* p = nullptr;
    const size_t b = sizeof(T) * std::max<size_t>(n, 1);
    CK(cudaMalloc(&p, b));
    bytes += double(b);
    return p;
}

template <class T>
void upload(T* d, const T* h, size_t n, cudaStream_t s) {
    if (n) CK(cudaMemcpyAsync(d, h, sizeof(T) * n, cudaMemcpyHostToDevice, s));
}

template <class T>
void download(T* h, const T* d, size_t n, cudaStream_t s) {
    if (n) CK(cudaMemcpyAsync(h, d, sizeof(T) * n, cudaMemcpyDeviceToHost, s));
}

}  // namespace

struct pmts_pd {
    pmts_pd_desc desc{};
    int dim = 2, nn = 4, E = 0, N = 0, ndof = 0, mode = 0;
    cudaStream_t stream = nullptr;
    DevPD d{};
    double device_bytes = 0.0;
    // host copies of the setup
    std::vector<int32_t> conn;       // element-major
    std::vector<double> cen, vol;    // cen element-major (xyz)
    std::vector<double> notch_pts;
    std::vector<int32_t> notch_npts;
    double cl = 0.0, eps = 0.0, lo[3] = {0, 0, 0};
    bool fracture = false, families = false;
    std::vector<int32_t> hcol;       // K x E
    int64_t n_entries = 0;
    int64_t gstep = 0;               // fine steps taken since creation
    int64_t broken_total = 0;
    // device scratch
    unsigned long long* d_counts = nullptr;
    int counts_cap = 0;
    unsigned long long* d_log_n = nullptr;
    int32_t* d_log = nullptr;
    // lattice-stencil fast path (pd_stencil.cu)
    bool lattice = false;
    LatticeDev L{};
    std::vector<int> stencil_delta;  // linear id delta per stencil offset (ascending)
    bool fused = false;              // one-kernel 2D step (the TMA-staged tile kernel, pd_tile9.cu)
    bool pos_only = false;           // mask bits of negative offsets not maintained
    uint32_t* mask0 = nullptr;       // lattice: the stencil mask as encoded (bonds that exist)
    // pmts_pd_set_option: the exact cold-tile break screens (default on) and the
    // 2D halo-overlap launch split (default off)
    bool screen = true, halo_overlap = false;
    unsigned* lat3_tmax = nullptr;   // the 3D screen's per-tile maxima (kept when screen is off)
    unsigned long long* hot_count = nullptr;  // PMTS_OPT_COUNT_HOT: {hot, tested} tiles
    // coupled-integrator hooks (deterministic mode): constraint load, k_sync snapshot,
    // entry-major families and scratch of the homogeneous recursion
    double* d_extra = nullptr;
    uint32_t* mask_sync = nullptr;
    int32_t* famT_col = nullptr;
    double* famT_coef = nullptr;
    double *rec_rd = nullptr, *rec_rv = nullptr, *rec_u = nullptr, *rec_v = nullptr,
           *rec_a = nullptr, *rec_w = nullptr, *rec_out = nullptr;
    int32_t* rec_row_of = nullptr;
    int rec_rows_cap = 0, rec_m_cap = 0;
    double* rd_buf[2] = {nullptr, nullptr};
    bool tile9 = false;              // ... the one-shot TMA-staged tile kernel (default)
    int tile9_occ = 0;               // its resident CTAs per SM
    CUtensorMap t9_rd[2]{}, t9_rv{}, t9_im{};
    int t9_prefetch = 0;  // L2 prefetch distance in tiles (resident CTAs of the device)
    bool pairs = false;              // tile9 with the pair-symmetric compile-time stencil
    bool f32pos = false;             // PMTS_FAST_F32POS: tile9 pairs on fp32 tile-relative ubar
    PairStencil2D pst{};
    double* d_imf = nullptr;         // per node {1/M | flags}, rows padded to an even count
    Stencil2D st2{};
    bool lat3 = false;               // 3D 122-offset nominal-lattice bond kernel
    Stencil3D st3{};
    double* rd_alt = nullptr;        // ping-pong partners of d.rd / d.mask
    uint32_t* mask_alt = nullptr;
    // tile9 clean-tile flags (pd_tile9.cu): computed from the bond states before the
    // first step after they were (re)built; PMTS_OPT_CLEAN_TILES = 0 turns them off
    uint32_t* t9_clean = nullptr;
    bool t9_clean_ready = false, t9_clean_on = true;
    // slab decomposition: NCCL clique + halo rows (node ranges, local ids)
    void* comm = nullptr;            // ncclComm_t
    int peer_lo = -1, peer_hi = -1;
    // halo overlap (tile kernel with peers): the tile rows holding halo send / receive
    // rows launch first, the exchange runs on xstream while the interior rows compute
    int split_a = -1, split_b = -1;  // edge rows [0, a) and [b, rows); -1: not planned
    cudaStream_t xstream = nullptr;
    cudaEvent_t ev_edge = nullptr, ev_x = nullptr;
    int send_lo = 0, recv_lo = 0, n_lo = 0, send_hi = 0, recv_hi = 0, n_hi = 0;
    // 3D slabs cut along y: each halo range repeats over halo_layers z node layers,
    // halo_stride nodes apart; packed into halo_buf (send lo | send hi | recv lo | recv hi)
    int halo_layers = 1, halo_stride = 0;
    double* halo_buf = nullptr;
    unsigned long long* h_counts = nullptr;  // pinned
    void* h_map = nullptr;                   // mapped pinned staging (step_tracked)
    size_t h_map_cap = 0;
    int h_counts_cap = 0;
    char* trk_buf = nullptr;         // pmts_pd_step_tracked staging
    size_t trk_cap = 0;
    std::vector<int32_t> trk_dofs;
    std::vector<double> hM, hP;      // host copies (per dof)
    std::vector<uint8_t> hbc;        // per dof: constrained
    std::vector<void*> owned;

    ~pmts_pd() {
        if (stream) cudaStreamSynchronize(stream);
        if (h_counts) cudaFreeHost(h_counts);
        if (h_map) cudaFreeHost(h_map);
        for (void* p : owned) cudaFree(p);
        if (stream) cudaStreamDestroy(stream);
    }

    template <class T>
    T* alloc(size_t n) {
        T* p = dalloc<T>(n, device_bytes);
        owned.push_back(p);
        return p;
    }
    void release(void* p) {
        if (!p) return;
        auto it = std::find(owned.begin(), owned.end(), p);
        if (it != owned.end()) owned.erase(it);
        cudaFree(p);
    }
};

namespace {

// micromodulus (material.hpp:84-88) or the BASELINE constant form (extension)
double micromodulus(const pmts_pd_desc& dsc, int dim, double r) {
    if (r <= 0.0) throw ConfigError("micromodulus needs |xi| > 0");
    if (r > dsc.delta) return 0.0;
    if (dsc.micromodulus == PMTS_MICRO_CONST) {
        const double r3 = (r * r) * r;
        return (dim == 2 ? dsc.c_const * dsc.h : dsc.c_const) / r3;
    }
    return dsc.c0 * std::exp(-r / dsc.l);
}

bool try_lattice(pmts_pd* h, const int32_t* dcol = nullptr);
void plan_split(pmts_pd* h);

constexpr ncclDataType_t kNcclFloat64 = ncclFloat64;

// Strided halo ranges (3D slabs cut along y): copy n nodes (dim doubles each) of
// `layers` ranges, `stride` nodes apart, between rd and a packed buffer.  Two ranges
// per launch (the lower and the upper neighbour's); n = 0 skips one.
__global__ void k_halo_pack(double* rd, double* buf, int first_a, int first_b, int n_a, int n_b,
                            int layers, int stride, int dim, int unpack) {
    const long long per = (long long)(n_a + n_b) * dim;
    const long long t = (long long)blockIdx.x * blockDim.x + threadIdx.x;
    if (t >= per * layers) return;
    const int l = (int)(t / per);
    long long q = t % per;
    const bool b = q >= (long long)n_a * dim;
    if (b) q -= (long long)n_a * dim;
    const long long g = ((long long)(b ? first_b : first_a) + (long long)l * stride) * dim + q;
    const long long p = (b ? (long long)n_a * dim * layers : 0) + (long long)l *
                        (b ? n_b : n_a) * dim + q;
    if (unpack) rd[g] = buf[p];
    else buf[p] = rd[g];
}

void halo_pack(pmts_pd* h, double* rd, double* buf, int fa, int fb, int na, int nb, bool unpack,
               cudaStream_t st) {
    const long long tot = (long long)(na + nb) * h->dim * h->halo_layers;
    if (!tot) return;
    k_halo_pack<<<(unsigned)((tot + 255) / 256), 256, 0, st>>>(rd, buf, fa, fb, na, nb,
                                                              h->halo_layers, h->halo_stride,
                                                              h->dim, unpack ? 1 : 0);
    CK(cudaGetLastError());
}

// halo exchange of the predictor displacement after a fine step
void exchange_halo(pmts_pd* h, double* rd = nullptr, cudaStream_t st = nullptr) {
    if (!h->comm || (h->peer_lo < 0 && h->peer_hi < 0)) return;
    NcclApi& a = nccl();
    const int dim = h->dim;
    if (!rd) rd = h->d.rd;
    if (!st) st = h->stream;
    if (h->halo_layers > 1) {
        // pack both send ranges, one message per neighbour, unpack both receive ranges
        const int nl = h->peer_lo >= 0 ? h->n_lo : 0, nh = h->peer_hi >= 0 ? h->n_hi : 0;
        const size_t ml = (size_t)nl * dim * h->halo_layers, mh = (size_t)nh * dim * h->halo_layers;
        double* sb = h->halo_buf;
        double* rb = h->halo_buf + ml + mh;
        halo_pack(h, rd, sb, h->send_lo, h->send_hi, nl, nh, false, st);
        nccl_check(a.group_start(), "group");
        if (nl) {
            nccl_check(a.send(sb, ml, kNcclFloat64, h->peer_lo, (ncclComm_t)h->comm, st), "send");
            nccl_check(a.recv(rb, ml, kNcclFloat64, h->peer_lo, (ncclComm_t)h->comm, st), "recv");
        }
        if (nh) {
            nccl_check(a.send(sb + ml, mh, kNcclFloat64, h->peer_hi, (ncclComm_t)h->comm, st),
                       "send");
            nccl_check(a.recv(rb + ml, mh, kNcclFloat64, h->peer_hi, (ncclComm_t)h->comm, st),
                       "recv");
        }
        nccl_check(a.group_end(), "group");
        halo_pack(h, rd, rb, h->recv_lo, h->recv_hi, nl, nh, true, st);
        return;
    }
    nccl_check(a.group_start(), "group");
    if (h->peer_lo >= 0) {
        nccl_check(a.send(rd + (size_t)h->send_lo * dim, (size_t)h->n_lo * dim, kNcclFloat64,
                          h->peer_lo, (ncclComm_t)h->comm, st), "send");
        nccl_check(a.recv(rd + (size_t)h->recv_lo * dim, (size_t)h->n_lo * dim, kNcclFloat64,
                          h->peer_lo, (ncclComm_t)h->comm, st), "recv");
    }
    if (h->peer_hi >= 0) {
        nccl_check(a.send(rd + (size_t)h->send_hi * dim, (size_t)h->n_hi * dim, kNcclFloat64,
                          h->peer_hi, (ncclComm_t)h->comm, st), "send");
        nccl_check(a.recv(rd + (size_t)h->recv_hi * dim, (size_t)h->n_hi * dim, kNcclFloat64,
                          h->peer_hi, (ncclComm_t)h->comm, st), "recv");
    }
    nccl_check(a.group_end(), "group");
}

// Family tables from the ELL partner list: per directed entry w c(|xi|)
// computed on the host exactly as scatter_pe_block forms it
// (perifem.hpp:247: coeff * weight * c with coeff = 1, weight = V_i V_j
// from build_peri_elements perifem.hpp:92-95); intact bits all set.
void finish_families(pmts_pd* h, int K) {
    const int E = h->E;
    h->d.K = K;
    h->d.W = std::max(1, (K + 31) / 32);
    std::vector<double> coef((size_t)K * E, 0.0);
    std::vector<uint32_t> mask((size_t)h->d.W * E, 0u);
    std::vector<int32_t> nent(E, 0);
    par_range(E, [&](int e) {  // (per element: independent entries, host cores)
        for (int k = 0; k < K; ++k) {
            const int p = h->hcol[(size_t)k * E + e];
            if (p < 0) break;
            const int i = std::min(e, p), j = std::max(e, p);
            double xi[3];
            for (int c = 0; c < 3; ++c) xi[c] = h->cen[3 * (size_t)j + c] - h->cen[3 * (size_t)i + c];
            const double xin = std::sqrt(xi[0] * xi[0] + xi[1] * xi[1] + xi[2] * xi[2]);
            if (xin <= 0.0) throw ConfigError("degenerate bond: coincident quadrature points");
            const double w = h->vol[i] * h->vol[j];
            const double c = micromodulus(h->desc, h->dim, xin);
            coef[(size_t)k * E + e] = c * w;
            mask[(size_t)(k >> 5) * E + e] |= 1u << (k & 31);
            ++nent[e];
        }
    });
    int64_t F = 0;
    for (int e = 0; e < E; ++e) F += nent[e];
    h->n_entries = F;
    if (h->d.coef) h->release((void*)h->d.coef);
    if (h->d.mask) h->release(h->d.mask);
    if (h->d.col) h->release((void*)h->d.col);
    int32_t* col = h->alloc<int32_t>((size_t)K * E);
    double* dcoef = h->alloc<double>((size_t)K * E);
    uint32_t* dmask = h->alloc<uint32_t>((size_t)h->d.W * E);
    upload(col, h->hcol.data(), (size_t)K * E, h->stream);
    upload(dcoef, coef.data(), (size_t)K * E, h->stream);
    upload(dmask, mask.data(), (size_t)h->d.W * E, h->stream);
    h->d.col = col;
    h->d.coef = dcoef;
    h->d.mask = dmask;
    if (h->mode == PMTS_DETERMINISTIC) {
        if (h->d_log) h->release(h->d_log);
        h->d_log = h->alloc<int32_t>(3 * (size_t)(F / 2 + 1));
        h->d.log = h->d_log;
        h->d.log_cap = F / 2 + 1;
        CK(cudaMemsetAsync(h->d_log_n, 0, sizeof(unsigned long long), h->stream));
    }
    CK(cudaStreamSynchronize(h->stream));
    h->families = true;
    h->lattice = false;
    if (h->mode == PMTS_FAST) try_lattice(h);
}

// TMA tensor maps for the persistent 2D kernel: rd (both ping-pong buffers),
// rv, and the packed {1/M, flags}, all viewed as [NY][2 NX] doubles.
PFN_cuTensorMapEncodeTiled tensor_map_encoder() {
    static PFN_cuTensorMapEncodeTiled encode = nullptr;
    if (!encode) {
        cudaDriverEntryPointQueryResult q;
        void* fn = nullptr;
        CK(cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &fn, cudaEnableDefault, &q));
        if (!fn || q != cudaDriverEntryPointSuccess)
            throw InternalError("cuTensorMapEncodeTiled unavailable");
        encode = (PFN_cuTensorMapEncodeTiled)fn;
    }
    return encode;
}


// TMA tensor maps of the tile9 kernel: rd of both ping-pong buffers, rv and
// {1/M | flags}.  Box sizes come from pd_tile9.cu.
void build_tile9_maps(pmts_pd* h) {
    const PFN_cuTensorMapEncodeTiled encode = tensor_map_encoder();
    const int nx = h->L.nx, ny = h->L.ny, NX = nx + 1, NY = ny + 1, NXP = (NX + 1) & ~1;
    int rdx, rdy, rvx, rvy, imx, imy;
    tile9_boxes(&rdx, &rdy, &rvx, &rvy, &imx, &imy);
    auto make = [&](CUtensorMap* m, CUtensorMapDataType ty, size_t esz, void* base, int w,
                    int rows, int bx, int by) {
        const cuuint64_t dims[2] = {(cuuint64_t)w, (cuuint64_t)rows};
        const cuuint64_t strides[1] = {(cuuint64_t)w * esz};
        const cuuint32_t box[2] = {(cuuint32_t)bx, (cuuint32_t)by};
        const cuuint32_t estr[2] = {1, 1};
        const CUresult r = encode(m, ty, 2, base, dims, strides, box, estr,
                                  CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE,
                                  CU_TENSOR_MAP_L2_PROMOTION_L2_128B,
                                  CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
        if (r != CUDA_SUCCESS)
            throw InternalError("cuTensorMapEncodeTiled failed (" + std::to_string((int)r) + ")");
    };
    for (int b = 0; b < 2; ++b) {
        make(&h->t9_rd[b], CU_TENSOR_MAP_DATA_TYPE_FLOAT64, 8, h->rd_buf[b], 2 * NX, NY, rdx, rdy);
    }
    make(&h->t9_rv, CU_TENSOR_MAP_DATA_TYPE_FLOAT64, 8, h->d.rv, 2 * NX, NY, rvx, rvy);
    make(&h->t9_im, CU_TENSOR_MAP_DATA_TYPE_FLOAT64, 8, h->d_imf, NXP, NY, imx, imy);
}

// elements of the tiles that stage and re-write their bond states in the next step
// (every element without the clean-tile flags); the skip rule of k_tile9
double tile9_staged_elements(pmts_pd* h) {
    if (!h->tile9 || !h->t9_clean_on || !h->t9_clean_ready) return (double)h->E;
    const int cols = tile9_cols(h->L), rows = tile9_rows(h->L), T = tile9_tile_rows();
    std::vector<uint32_t> f((size_t)cols * rows);
    download(f.data(), h->t9_clean, f.size(), h->stream);
    CK(cudaStreamSynchronize(h->stream));
    const int nx = h->L.nx, ny = h->L.ny;
    double staged = 0.0;
    for (int by = 0; by < rows; ++by)
        for (int bx = 0; bx < cols; ++bx) {
            const int i0 = bx * T, j0 = by * T, ax0 = i0 - 1 - kFusedR, ay0 = j0 - 1 - kFusedR;
            const bool interior = ax0 >= 0 && ay0 >= 0 && ax0 + kFusedAX <= nx &&
                                  ay0 + T + 1 + kFusedR <= ny;
            bool skip = false;
            if (interior) {
                const uint32_t* tf = f.data() + (size_t)by * cols + bx;
                const uint32_t* tb = tf - cols;
                skip = (tf[-1] & tf[0] & tf[1] & tb[-1] & tb[0] & tb[1]) != 0u;
            }
            if (!skip)
                staged += (double)std::max(0, std::min(T, nx - i0)) * std::max(0, std::min(T, ny - j0));
        }
    return staged;
}

Tile9Maps tile9_maps(const pmts_pd* h) {
    Tile9Maps m;
    m.rd = h->t9_rd[h->d.rd == h->rd_buf[0] ? 0 : 1];
    m.rv = h->t9_rv;
    m.im = h->t9_im;
    m.prefetch_ahead = h->t9_prefetch;
    return m;
}

// host copy of the ELL families, fetched on first use when they were built and
// encoded on the device
void ensure_hcol(pmts_pd* h) {
    if (!h->hcol.empty() || !h->d.col) return;
    h->hcol.assign((size_t)h->d.K * h->E, -1);
    download(h->hcol.data(), h->d.col, h->hcol.size(), h->stream);
    CK(cudaStreamSynchronize(h->stream));
}

// Stencil encoding of the families when the mesh is the generated lattice
// (fast mode).  Returns false (ELL path stays) if any bond's offset falls
// outside one shared stencil of <= kMaxStencil offsets.  dcol: the families are
// device-resident (no host copy); the offset scan and the mask run on the device
// and the stencil constants must be the nominal ones (desc.lattice_h > 0).
bool try_lattice(pmts_pd* h, const int32_t* dcol) {
    const int E = h->E, K = h->d.K, dim = h->dim;
    const int nx = h->desc.lattice[0], ny = h->desc.lattice[1];
    const int nz = dim == 3 ? h->desc.lattice[2] : 1;
    if (nx <= 0 || ny <= 0 || nz <= 0 || (int64_t)nx * ny * nz != E) return false;
    // element (i,j,k) of id e must be the lattice cell: check centroids are monotone
    auto ijk = [&](int e, int& i, int& j, int& k) {
        i = e % nx;
        j = (e / nx) % ny;
        k = e / (nx * ny);
    };
    if (dcol && !(h->desc.lattice_h > 0.0)) return false;
    int R = 0;
    std::vector<int> present17;
    if (dcol) {
        present17.assign(17 * 17 * 17, 0);
        R = lattice_scan_device(dcol, E, K, nx, ny, present17.data(), h->stream);
    } else {
        for (int e = 0; e < E; ++e)
            for (int q = 0; q < K; ++q) {
                const int p = h->hcol[(size_t)q * E + e];
                if (p < 0) break;
                int a, b, c, x, y, z;
                ijk(e, a, b, c);
                ijk(p, x, y, z);
                R = std::max({R, std::abs(x - a), std::abs(y - b), std::abs(z - c)});
            }
    }
    if (R == 0 || R > 8) return false;
    const int span = 2 * R + 1;
    std::vector<int> slot(span * span * span, -1);
    auto key = [&](int di, int dj, int dk) { return ((dk + R) * span + dj + R) * span + di + R; };
    std::vector<int> offs;  // keys
    if (dcol) {  // the device scan's offsets, in 17^3 key order
        for (int k17 = 0; k17 < 17 * 17 * 17; ++k17) {
            if (!present17[k17]) continue;
            const int kk = key(k17 % 17 - 8, (k17 / 17) % 17 - 8, k17 / 289 - 8);
            slot[kk] = 0;
            offs.push_back(kk);
        }
    } else {
        for (int e = 0; e < E; ++e)
            for (int q = 0; q < K; ++q) {
                const int p = h->hcol[(size_t)q * E + e];
                if (p < 0) break;
                int a, b, c, x, y, z;
                ijk(e, a, b, c);
                ijk(p, x, y, z);
                const int kk = key(x - a, y - b, z - c);
                if (slot[kk] < 0) {
                    slot[kk] = 0;
                    offs.push_back(kk);
                }
            }
    }
    // symmetric closure and ascending linear delta (== ascending partner id)
    auto decode = [&](int kk, int& di, int& dj, int& dk) {
        di = kk % span - R;
        dj = (kk / span) % span - R;
        dk = kk / (span * span) - R;
    };
    for (size_t n = 0, m = offs.size(); n < m; ++n) {
        int di, dj, dk;
        decode(offs[n], di, dj, dk);
        const int neg = key(-di, -dj, -dk);
        if (slot[neg] < 0) {
            slot[neg] = 0;
            offs.push_back(neg);
        }
    }
    auto lin = [&](int kk) {
        int di, dj, dk;
        decode(kk, di, dj, dk);
        return (dk * ny + dj) * nx + di;
    };
    std::sort(offs.begin(), offs.end(), [&](int a, int b) { return lin(a) < lin(b); });
    const int S = (int)offs.size();
    if (S > kMaxStencil) return false;
    for (int s = 0; s < S; ++s) slot[offs[s]] = s;
    const int W = (S + 31) / 32;
    // per-offset constants from one representative bond of the positive offset;
    // the negative offset gets the exact negation (both directions of a bond then
    // evaluate bitwise-negated operands and agree on every break)
    std::vector<double> table(kTableRow * (size_t)S, 0.0);
    std::vector<char> have(S, 0);
    std::vector<uint32_t> mask(dcol ? 0 : (size_t)W * E, 0u);
    const double s0 = h->desc.s_crit, sl = s0 * (1.0 - h->desc.s_crit_spread);
    if (dcol) {  // nominal constants per positive offset (xi = h o, w = V^2) and its negation
        const double hh = h->desc.lattice_h, wv = h->desc.lattice_vol * h->desc.lattice_vol;
        for (int s = 0; s < S; ++s) {
            if (lin(offs[s]) <= 0) continue;
            int di, dj, dk;
            decode(offs[s], di, dj, dk);
            const double xi[3] = {di * hh, dj * hh, dk * hh};
            const double x2 = xi[0] * xi[0] + xi[1] * xi[1] + xi[2] * xi[2];
            const double f = micromodulus(h->desc, dim, std::sqrt(x2)) * wv;
            const int sn = slot[key(-di, -dj, -dk)];
            const double cthr = (2.0 * s0 + s0 * s0) * x2;
            const double clo =
                h->desc.s_crit_spread != 0.0 ? (2.0 * sl + sl * sl) * x2 * (1.0 - 1e-12) : cthr;
            const int xs[3] = {0, 1, 4};
            for (int k = 0; k < 3; ++k) {
                table[kTableRow * s + xs[k]] = xi[k];
                table[kTableRow * sn + xs[k]] = -xi[k];
            }
            for (int r : {s, sn}) {
                table[kTableRow * r + 2] = f;
                table[kTableRow * r + 3] = cthr;
                table[kTableRow * r + 5] = clo;
                table[kTableRow * r + 6] = x2;
            }
        }
    }
    for (int e = 0; e < E && !dcol; ++e)
        for (int q = 0; q < K; ++q) {
            const int p = h->hcol[(size_t)q * E + e];
            if (p < 0) break;
            int a, b, c, x, y, z;
            ijk(e, a, b, c);
            ijk(p, x, y, z);
            const int s = slot[key(x - a, y - b, z - c)];
            mask[(size_t)(s >> 5) * E + e] |= 1u << (s & 31);
            if (p > e && !have[s]) {
                have[s] = 1;
                int di, dj, dk;
                decode(offs[s], di, dj, dk);
                double xi[3];
                double wv = h->vol[e] * h->vol[p];
                if (h->desc.lattice_h > 0.0) {
                    // nominal lattice constants: identical on every rank of a slab
                    // decomposition (the representative bond is not)
                    const double hh = h->desc.lattice_h;
                    xi[0] = di * hh;
                    xi[1] = dj * hh;
                    xi[2] = dk * hh;
                    wv = h->desc.lattice_vol * h->desc.lattice_vol;
                } else {
                    for (int k = 0; k < 3; ++k)
                        xi[k] = h->cen[3 * (size_t)p + k] - h->cen[3 * (size_t)e + k];
                }
                const double x2 = xi[0] * xi[0] + xi[1] * xi[1] + xi[2] * xi[2];
                const double f = micromodulus(h->desc, dim, std::sqrt(x2)) * wv;
                const int sn = slot[key(-di, -dj, -dk)];
                const double cthr = (2.0 * s0 + s0 * s0) * x2;
                const double clo = h->desc.s_crit_spread != 0.0
                                       ? (2.0 * sl + sl * sl) * x2 * (1.0 - 1e-12)
                                       : cthr;
                const int xs[3] = {0, 1, 4};
                for (int k = 0; k < 3; ++k) {
                    table[kTableRow * s + xs[k]] = xi[k];
                    table[kTableRow * sn + xs[k]] = -xi[k];
                }
                for (int r : {s, sn}) {
                    table[kTableRow * r + 2] = f;
                    table[kTableRow * r + 3] = cthr;
                    table[kTableRow * r + 5] = clo;
                    table[kTableRow * r + 6] = x2;
                }
                have[sn] = 1;
            }
        }
    std::vector<int8_t> di(S), dj(S), dk(S);
    std::vector<int> dl(S);
    for (int s = 0; s < S; ++s) {
        int a, b, c;
        decode(offs[s], a, b, c);
        di[s] = (int8_t)a;
        dj[s] = (int8_t)b;
        dk[s] = (int8_t)c;
        dl[s] = lin(offs[s]);
    }
    LatticeDev& L = h->L;
    L.nx = nx;
    L.ny = ny;
    L.nz = nz;
    L.R = R;
    L.S = S;
    L.W = W;
    // slab rows: node update on the owned y node rows, element forces on the rows
    // those nodes touch (pmts_pd_desc.node_rows; one domain: everything)
    L.jn0 = 0;
    L.jn1 = ny + 1;
    if (h->desc.node_rows[0] != 0 || h->desc.node_rows[1] != 0) {
        if (h->desc.node_rows[0] < 0 || h->desc.node_rows[1] > ny + 1 ||
            h->desc.node_rows[0] >= h->desc.node_rows[1])
            throw ConfigError("node_rows out of the lattice");
        L.jn0 = h->desc.node_rows[0];
        L.jn1 = h->desc.node_rows[1];
    }
    L.jb0 = std::max(0, L.jn0 - 1);
    L.jb1 = std::min(ny, L.jn1);
    lat3_rows(L);
    int8_t* ddi = h->alloc<int8_t>(S);
    int8_t* ddj = h->alloc<int8_t>(S);
    int8_t* ddk = h->alloc<int8_t>(S);
    int* ddl = h->alloc<int>(S);
    double* dtab = h->alloc<double>(kTableRow * (size_t)S);
    upload(ddi, di.data(), S, h->stream);
    upload(ddj, dj.data(), S, h->stream);
    upload(ddk, dk.data(), S, h->stream);
    upload(ddl, dl.data(), S, h->stream);
    upload(dtab, table.data(), kTableRow * (size_t)S, h->stream);
    // per-node flags and inverse lumped mass (the lumped mass is one value per node)
    std::vector<uint8_t> nflag(h->N, 0);
    std::vector<double> im(h->N, 0.0);
    for (int n = 0; n < h->N; ++n) {
        uint8_t f = 0;
        for (int c = 0; c < dim; ++c) {
            const size_t q = (size_t)n * dim + c;
            if (h->hbc[q]) f |= uint8_t(1u << c);
            if (h->hP[q] != 0.0) f |= 8u;
            if (!h->hbc[q] && h->hM[q] != h->hM[(size_t)n * dim]) return false;
        }
        nflag[n] = f;
        im[n] = 1.0 / h->hM[(size_t)n * dim];
        if (dim == 2) {
            // 2D: every lattice kernel uses 1/M with the node flags (1 x, 2 y
            // constrained, 4 loaded) in its three low mantissa bits -- the form the
            // TMA-staged tile kernel reads -- so all 2D variants stay bitwise equal
            // (relative change of 1/M <= 2^-49, far inside the fast-mode tolerance)
            uint64_t b;
            std::memcpy(&b, &im[n], 8);
            b = (b & ~uint64_t(7)) | (f & 3u) | ((f & 8u) ? 4u : 0u);
            std::memcpy(&im[n], &b, 8);
        }
    }
    uint8_t* dnf = h->alloc<uint8_t>(h->N);
    double* dim_ = h->alloc<double>(h->N);
    upload(dnf, nflag.data(), h->N, h->stream);
    upload(dim_, im.data(), h->N, h->stream);
    L.nflag = dnf;
    L.inv_mass = dim_;
    L.di = ddi;
    L.dj = ddj;
    L.dk = ddk;
    L.delta_id = ddl;
    L.table = dtab;
    // the stencil mask replaces the ELL mask; ELL coefficients are not needed
    h->release(h->d.mask);
    uint32_t* dmask = h->alloc<uint32_t>((size_t)W * E);
    if (dcol) {
        std::vector<int> slot17(17 * 17 * 17, -1);
        for (int s = 0; s < S; ++s) {
            int a, b, c;
            decode(offs[s], a, b, c);
            slot17[((c + 8) * 17 + b + 8) * 17 + a + 8] = s;
        }
        h->n_entries = lattice_mask_device(dcol, E, K, nx, ny, slot17.data(), W, dmask, h->stream);
    } else {
        upload(dmask, mask.data(), (size_t)W * E, h->stream);
    }
    h->d.mask = dmask;
    h->d.W = W;
    // the encoded mask = the bonds that exist (damage_field's weights, the pair export)
    if (h->mask0) h->release(h->mask0);
    h->mask0 = h->alloc<uint32_t>((size_t)W * E);
    CK(cudaMemcpyAsync(h->mask0, dmask, sizeof(uint32_t) * W * E, cudaMemcpyDeviceToDevice,
                       h->stream));
    h->release((void*)h->d.coef);
    h->d.coef = nullptr;
    h->stencil_delta = dl;
    lattice_configure(dim, R, S);
    // 3D, 122 offsets, nominal constants: class-constant table for pd_lat3.cu
    h->lat3 = false;
    if (dim == 3 && h->desc.lattice_h > 0.0 && lat3_offsets_match(di.data(), dj.data(), dk.data(), S)) {
        const double hh = h->desc.lattice_h;
        bool ok = true, seen[8] = {false, false, false, false, false, false, false, false};
        for (int s = 0; s < S && ok; ++s) {
            const int d2 = di[s] * di[s] + dj[s] * dj[s] + dk[s] * dk[s];
            const int cl = lat3_class_of(d2);
            const double* t = table.data() + kTableRow * (size_t)s;
            const double c = t[2] * (hh * hh);
            long long clo, cth;
            std::memcpy(&clo, &t[5], 8);
            std::memcpy(&cth, &t[3], 8);
            if (!seen[cl]) {
                h->st3.c[cl] = c;
                h->st3.clo[cl] = clo;
                h->st3.cthr[cl] = cth;
                seen[cl] = true;
            } else {  // same |o|^2: equal up to the rounding order of |xi|^2 (fast mode)
                ok = std::abs(h->st3.c[cl] - c) <= 1e-14 * std::abs(c);
            }
        }
        h->st3.h2 = 2.0 * hh;
        h->st3.hh = hh * hh;
        // TMA staging of the ubar apron (global rows must be 16-byte multiples: nx even)
        h->st3.use_tma = 0;
        if (ok && L.nx % 2 == 0) {
            const cuuint64_t dims[3] = {(cuuint64_t)3 * L.nx, (cuuint64_t)L.ny, (cuuint64_t)L.nz};
            const cuuint64_t strides[2] = {(cuuint64_t)3 * L.nx * 8, (cuuint64_t)3 * L.nx * L.ny * 8};
            int bx, by, bz;
            lat3_apron_box(&bx, &by, &bz);
            const cuuint32_t box[3] = {(cuuint32_t)bx, (cuuint32_t)by, (cuuint32_t)bz};
            const cuuint32_t estr[3] = {1, 1, 1};
            const CUresult r = tensor_map_encoder()(
                &h->st3.ub, CU_TENSOR_MAP_DATA_TYPE_FLOAT64, 3, h->d.ubar, dims, strides, box, estr,
                CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE,
                CU_TENSOR_MAP_L2_PROMOTION_L2_128B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
            if (r != CUDA_SUCCESS)
                throw InternalError("cuTensorMapEncodeTiled failed (" + std::to_string((int)r) + ")");
            h->st3.use_tma = 1;
        }
        // cold-tile break screen (pmts_pd_set_option PMTS_OPT_BREAK_SCREEN = 0: the
        // break test on every tile)
        h->st3.tmax = nullptr;
        h->lat3_tmax = nullptr;
        if (ok) {
            h->st3.hot_count = h->pst.hot_count = h->hot_count;
            const size_t nt = lat3_tile_count(h->L);
            unsigned* tm = h->alloc<unsigned>(9 * nt);
            CK(cudaMemsetAsync(tm, 0, 9 * nt * sizeof(unsigned), h->stream));
            h->lat3_tmax = tm;
            if (h->screen) h->st3.tmax = tm;
        }

        h->lat3 = ok;
    }
    h->fused = false;
    if (dim == 2 && S == kFusedS && R == kFusedR) {
        Stencil2D& st = h->st2;
        for (int s = 0; s < S; ++s) {
            const double* t = table.data() + kTableRow * (size_t)s;
            st.xi0[s] = t[0];
            st.xi1[s] = t[1];
            st.fx0[s] = t[2] * t[0];
            st.fx1[s] = t[2] * t[1];
            st.cthr[s] = t[3];
            st.clo[s] = t[5];
            st.x2[s] = t[6];
            st.aoff[s] = dj[s] * kFusedAX + di[s];
            st.did[s] = dl[s];
        }
        if (!h->rd_alt) h->rd_alt = h->alloc<double>(h->ndof);
        if (h->mask_alt) h->release(h->mask_alt);
        h->mask_alt = h->alloc<uint32_t>((size_t)E);
        h->t9_clean_ready = false;
        h->fused = true;
        h->tile9 = true;
        h->pos_only = true;  // the tile kernel keeps a bond's state at its lower end
        if (h->tile9) {
            // {1/M | flags}: flags (1 x, 2 y constrained, 4 loaded) in the low mantissa bits
            const int NX = h->L.nx + 1, NY = h->L.ny + 1, NXP = (NX + 1) & ~1;
            std::vector<double> imf((size_t)NXP * NY, 0.0);
            for (int j = 0; j < NY; ++j)
                for (int i = 0; i < NX; ++i) {
                    imf[(size_t)j * NXP + i] = im[j * NX + i];  // flags already encoded
                }
            if (h->d_imf) h->release(h->d_imf);
            h->d_imf = h->alloc<double>(imf.size());
            upload(h->d_imf, imf.data(), imf.size(), h->stream);
            h->rd_buf[0] = h->d.rd;
            h->rd_buf[1] = h->rd_alt;
            build_tile9_maps(h);
            h->tile9_occ = tile9_configure();
            {
                int sms = 0;
                CK(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, h->desc.device));
                h->t9_prefetch = sms * h->tile9_occ;
            }
            // pair-symmetric force on the nominal lattice (representative per-bond
            // constants, lattice_h = 0: the per-offset sums)
            h->pairs = h->desc.lattice_h > 0.0;
            const double hh = h->desc.lattice_h;

            for (int k = 0; k < 14 && h->pairs; ++k) {
                int A = 0, B = 0;
                tile9_pair_offset(k, &A, &B);
                int s = -1;
                for (int q = 0; q < S; ++q)
                    if (di[q] == A && dj[q] == B) s = q;
                if (s < 0) {
                    h->pairs = false;
                    break;
                }
                const double* t = table.data() + kTableRow * (size_t)s;
                const double F = -t[2] * (hh * hh);
                h->pst.fa[k] = B == 0 ? F * (A * A) : F * A;
                h->pst.fb[k] = A == 0 ? F * (B * B) : F * B;
                const double clo = t[5] * (1.0 - 1e-12);
                std::memcpy(&h->pst.cl[k], &clo, 8);
                h->pst.off[k] = B * kFusedAX + A;
                h->pst.pbit[k] = s;
            }
            h->pst.h2 = 2.0 * hh;
            plan_split(h);
            h->pst.h2f = (float)(2.0 * hh);
            for (int k = 0; k < 14 && h->pairs; ++k) {  // fp32 candidate thresholds, rounded down
                double c;
                std::memcpy(&c, &h->pst.cl[k], 8);
                c *= 1.0 - 1e-4;
                float f = (float)c;
                if ((double)f > c) f = std::nextafter(f, 0.0f);
                h->pst.clf[k] = f;
            }
            // cold-tile break screen (PMTS_OPT_BREAK_SCREEN = 0: candidate pass on every tile)
            h->pst.screen = h->screen ? 1 : 0;
            h->pst.hot_count = h->hot_count;
        }
    }
    CK(cudaStreamSynchronize(h->stream));
    h->lattice = true;
    return true;
}

// ELL-layout intact mask (bit k = k-th family entry) from the stencil mask
// the live ELL bond mask on the host (ELL paths; the lattice has its own kernels)
std::vector<uint32_t> ell_mask_host(pmts_pd* h) {
    std::vector<uint32_t> m((size_t)h->d.W * h->E);
    download(m.data(), h->d.mask, m.size(), h->stream);
    CK(cudaStreamSynchronize(h->stream));
    return m;
}

void require_families(pmts_pd* h) {
    if (!h->families)
        throw ConfigError("families not built: call pmts_pd_build_families or pmts_pd_set_pairs");
}

void ensure_counts(pmts_pd* h, int n) {
    if (n > h->counts_cap) {
        if (h->d_counts) h->release(h->d_counts);
        h->counts_cap = std::max(n, 64);
        h->d_counts = h->alloc<unsigned long long>(h->counts_cap);
    }
    CK(cudaMemsetAsync(h->d_counts, 0, sizeof(unsigned long long) * n, h->stream));
    h->d.broken_count = h->d_counts;
}

// Halo overlap plan of the tile kernel (opt-in, PMTS_T9_SPLIT=1): the tile rows that
// own a node row the exchange sends or receives go first ([0, a) and [b, rows)); the
// interior rows [a, b) run while ncclSend/ncclRecv move the halo on a second stream.
// Without peers the first and last tile rows are split off, which exercises the
// launch split on one GPU.  Off by default: on one B200 the split costs 15 us per
// cfg3 step (three launches, the cross-stream events break programmatic dependent
// launch) -- about the NCCL latency it would hide.
void plan_split(pmts_pd* h) {
    const bool peers = h->comm && (h->peer_lo >= 0 || h->peer_hi >= 0);
    const bool forced = h->halo_overlap;
    h->split_a = h->split_b = -1;
    if (!h->tile9 || !forced) return;
    const int rows = tile9_rows(h->L), ty = tile9_tile_rows(), NX = h->L.nx + 1;
    auto tile_row = [&](int node) { return std::min(node / NX / ty, rows - 1); };
    int a = forced && !peers ? 1 : 0, b = forced && !peers ? rows - 1 : rows;
    auto cover_lo = [&](int first, int n) {
        if (n > 0) a = std::max(a, tile_row(first + n - 1) + 1);
    };
    auto cover_hi = [&](int first, int n) {
        if (n > 0) b = std::min(b, tile_row(first));
    };
    if (h->peer_lo >= 0) {
        cover_lo(h->send_lo, h->n_lo);
        cover_lo(h->recv_lo, h->n_lo);
    }
    if (h->peer_hi >= 0) {
        cover_hi(h->send_hi, h->n_hi);
        cover_hi(h->recv_hi, h->n_hi);
    }
    if (a > b) return;  // the halo rows span the slab: no interior to overlap with
    if (!h->xstream) {
        CK(cudaStreamCreateWithFlags(&h->xstream, cudaStreamNonBlocking));
        CK(cudaEventCreateWithFlags(&h->ev_edge, cudaEventDisableTiming));
        CK(cudaEventCreateWithFlags(&h->ev_x, cudaEventDisableTiming));
    }
    h->split_a = a;
    h->split_b = b;
}

// one fine step: bond gather + node update with the fused predictor
void enqueue_step(pmts_pd* h, int slot, double scale, bool time_bond, cudaEvent_t* ev,
                  bool last = true, const double* scale_dev = nullptr,
                  const FusedBufs* report = nullptr) {
    const int brk = h->fracture ? 1 : 0;
    if (h->f32pos && !(h->fused && h->tile9 && h->pairs))
        throw ConfigError("PMTS_FAST_F32POS runs on the 2D lattice tile kernel with the nominal "
                          "28-offset pair stencil only (set lattice and lattice_h)");
    if (h->fused) {
        FusedBufs b{h->d.rd, h->rd_alt, h->d.mask, h->mask_alt, scale_dev};
        if (h->tile9 && h->t9_clean_on) {
            if (!h->t9_clean_ready) {
                if (!h->t9_clean)
                    h->t9_clean = h->alloc<uint32_t>((size_t)tile9_cols(h->L) * tile9_rows(h->L));
                launch_tile9_flags(h->L, h->d.mask, h->mask_alt, h->t9_clean, h->stream);
                h->t9_clean_ready = true;
            }
            b.tclean = h->t9_clean;
        }
        if (report) {
            b.trk_dofs = report->trk_dofs;
            b.n_trk = report->n_trk;
            b.trk_host = report->trk_host;
        }
        if (time_bond) CK(cudaEventRecord(ev[0], h->stream));
        if (h->tile9 && h->split_a >= 0) {
            // edge tile rows, then the halo exchange on xstream overlapping the interior
            const Tile9Maps mp = tile9_maps(h);
            const PairStencil2D* ps = h->pairs ? &h->pst : nullptr;
            const int rows = tile9_rows(h->L);
            launch_tile9_step(h->d, h->L, h->st2, ps, mp, b, slot, brk, scale, last ? 1 : 0,
                              h->f32pos, h->stream, 0, h->split_a);
            launch_tile9_step(h->d, h->L, h->st2, ps, mp, b, slot, brk, scale, last ? 1 : 0,
                              h->f32pos, h->stream, h->split_b, rows);
            CK(cudaEventRecord(h->ev_edge, h->stream));
            CK(cudaStreamWaitEvent(h->xstream, h->ev_edge, 0));
            exchange_halo(h, h->rd_alt, h->xstream);  // the buffer this step just wrote
            CK(cudaEventRecord(h->ev_x, h->xstream));
            launch_tile9_step(h->d, h->L, h->st2, ps, mp, b, slot, brk, scale, last ? 1 : 0,
                              h->f32pos, h->stream, h->split_a, h->split_b);
            CK(cudaStreamWaitEvent(h->stream, h->ev_x, 0));  // before anything that follows
            if (time_bond) CK(cudaEventRecord(ev[1], h->stream));
            std::swap(h->d.rd, h->rd_alt);
            std::swap(h->d.mask, h->mask_alt);
            return;
        }
        launch_tile9_step(h->d, h->L, h->st2, h->pairs ? &h->pst : nullptr, tile9_maps(h), b, slot,
                          brk, scale, last ? 1 : 0, h->f32pos, h->stream);
        if (time_bond) CK(cudaEventRecord(ev[1], h->stream));
        std::swap(h->d.rd, h->rd_alt);
        std::swap(h->d.mask, h->mask_alt);
        exchange_halo(h);
        return;
    }
    if (h->lattice) {
        launch_lattice_step(h->d, h->L, slot, brk, scale, last ? 1 : 0, time_bond, ev, h->stream,
                            h->lat3 ? &h->st3 : nullptr);
        exchange_halo(h);
        return;
    }
    if (time_bond) CK(cudaEventRecord(ev[0], h->stream));
    if (h->mode == PMTS_DETERMINISTIC) {
        launch_det_bond(h->d, h->d.rd, slot, brk, int(h->gstep + slot + 1), h->stream);
    } else {
        launch_fast_ubar(h->d, h->stream);
        launch_fast_bond(h->d, slot, brk, h->stream);
    }
    if (time_bond) CK(cudaEventRecord(ev[1], h->stream));
    launch_node_update(h->d, scale, 1, h->stream);
    exchange_halo(h);
}

// pinned host mirror of the per-step broken counts (async D2H, no staging copy)
unsigned long long* pinned_counts(pmts_pd* h, int n) {
    if (n > h->h_counts_cap) {
        if (h->h_counts) cudaFreeHost(h->h_counts);
        h->h_counts_cap = std::max(n, 64);
        CK(cudaMallocHost(&h->h_counts, sizeof(unsigned long long) * h->h_counts_cap));
    }
    return h->h_counts;
}

int64_t finish_steps(pmts_pd* h, int n) {
    unsigned long long* cnt = pinned_counts(h, std::max(n, 1));
    download(cnt, h->d_counts, n, h->stream);
    CK(cudaStreamSynchronize(h->stream));
    int64_t nb = 0;
    for (int s = 0; s < n; ++s) nb += (int64_t)cnt[s];
    h->gstep += n;
    h->broken_total += nb;
    return nb;
}

}  // namespace

extern "C" {

int pmts_device_count(int* n) {
    return guard([&] {
        int c = 0;
        if (cudaGetDeviceCount(&c) != cudaSuccess) c = 0;
        *n = c;
    });
}

int pmts_pd_create(const pmts_pd_desc* desc, pmts_pd** out) {
    return guard([&] {
        if (!desc || !out) throw ConfigError("null argument");
        const pmts_pd_desc& ds = *desc;
        if (ds.dim != 2 && ds.dim != 3) throw ConfigError("dim must be 2 or 3");
        if (ds.n_nodes <= 0 || ds.n_elems <= 0) throw ConfigError("empty mesh");
        if (!ds.node_xyz || !ds.elem_nodes || !ds.mass || !ds.p_ext)
            throw ConfigError("missing mesh, mass or load array");
        if (ds.dt <= 0.0) throw ConfigError("time step must be positive");
        if (ds.beta != 0.0)
            throw ConfigError("the device fine step is the explicit Newmark branch (beta_pd = 0); "
                              "implicit PD is out of scope (DESIGN.md)");
        if (ds.delta <= 0.0) throw ConfigError("horizon must be positive");
        if (ds.micromodulus == PMTS_MICRO_EXP && (ds.l <= 0.0 || ds.l > ds.delta || ds.c0 <= 0.0))
            throw ConfigError("exponential micromodulus needs 0 < l <= delta and c0 > 0");
        if (ds.micromodulus == PMTS_MICRO_CONST && ds.c_const <= 0.0)
            throw ConfigError("constant micromodulus needs c > 0");
        if (ds.mode != PMTS_DETERMINISTIC && ds.mode != PMTS_FAST && ds.mode != PMTS_FAST_F32POS)
            throw ConfigError("mode must be PMTS_DETERMINISTIC, PMTS_FAST or PMTS_FAST_F32POS");
        int ndev = 0;
        if (cudaGetDeviceCount(&ndev) != cudaSuccess || ndev == 0)
            throw InternalError("no CUDA device: the PD fine step has no CPU fallback");
        if (ds.device < 0 || ds.device >= ndev) throw ConfigError("device ordinal out of range");
        CK(cudaSetDevice(ds.device));

        auto h = std::make_unique<pmts_pd>();
        h->desc = ds;
        h->dim = ds.dim;
        h->nn = ds.dim == 2 ? 4 : 8;
        h->E = ds.n_elems;
        h->N = ds.n_nodes;
        h->ndof = ds.n_nodes * ds.dim;
        // the fp32-position variant is fast mode with fp32 arithmetic in the tile force
        h->f32pos = ds.mode == PMTS_FAST_F32POS;
        h->mode = h->f32pos ? PMTS_FAST : ds.mode;
        h->fracture = ds.s_crit > 0.0 && std::isfinite(ds.s_crit);  // material.hpp:44
        const int E = h->E, N = h->N, nn = h->nn, dim = h->dim;
        h->conn.assign(ds.elem_nodes, ds.elem_nodes + (size_t)E * nn);
        for (int32_t v : h->conn)
            if (v < 0 || v >= N) throw ConfigError("element references a missing node");
        // BcTable + mass positivity (newmark.hpp:81-93)
        std::vector<uint8_t> bcflag(h->ndof, 0);
        std::vector<double> bcvel(h->ndof, 0.0);
        for (int c = 0; c < ds.n_bc; ++c) {
            const int dof = ds.bc_dofs[c];
            if (dof < 0 || dof >= h->ndof) throw ConfigError("BC dof out of range");
            bcflag[dof] = 1;
            bcvel[dof] = ds.bc_vel[c];
        }
        for (int i = 0; i < h->ndof; ++i)
            if (!bcflag[i] && !(ds.mass[i] > 0.0))
                throw SolverError("non-positive lumped mass at dof " + std::to_string(i));
        h->hM.assign(ds.mass, ds.mass + h->ndof);
        h->hP.assign(ds.p_ext, ds.p_ext + h->ndof);
        h->hbc = bcflag;
        // geometry (mesh.hpp:112-139), host restatement, bit-exact
        h->cen.resize(3 * (size_t)E);
        h->vol.resize(E);
        // compute_element_geometry on the device (pd_setup.cu, bitwise the host's)
        {
            cudaStream_t gs = nullptr;
            CK(cudaStreamCreateWithFlags(&gs, cudaStreamNonBlocking));
            element_geometry_device(dim, E, N, h->conn.data(), ds.node_xyz, h->cen.data(),
                                    h->vol.data(), gs);
            CK(cudaStreamDestroy(gs));
        }
        h->cl = char_length(dim, E, h->vol.data());
        h->eps = 1e-12 * std::max(h->cl, 1e-300);  // mesh.hpp:435
        for (int k = 0; k < 3; ++k) h->lo[k] = 1e300;
        for (int e = 0; e < E; ++e)
            for (int k = 0; k < 3; ++k) h->lo[k] = std::min(h->lo[k], h->cen[3 * (size_t)e + k]);
        for (int q = 0; q < ds.n_notch; ++q) h->notch_npts.push_back(ds.notch_npts[q]);
        size_t npts = 0;
        for (int q = 0; q < ds.n_notch; ++q) npts += ds.notch_npts[q];
        if (npts) h->notch_pts.assign(ds.notch_pts, ds.notch_pts + 3 * npts);

        CK(cudaStreamCreateWithFlags(&h->stream, cudaStreamNonBlocking));
        cudaStream_t s = h->stream;
        DevPD& d = h->d;
        d.dim = dim;
        d.nn = nn;
        d.E = E;
        d.N = N;
        d.NE = nn;
        d.Nsh = dim == 2 ? 0.25 : 0.125;  // reference_shape at the centre (fem.hpp:22-47)
        d.s_crit = ds.s_crit;
        d.spread = ds.s_crit_spread;
        d.seed = ds.seed;
        d.fracture = h->fracture;
        d.goff = ds.global_id_offset;
        d.extra = nullptr;
        d.id_pl = 0;
        d.id_pg = 0;
        if (ds.slab_plane[0] != 0 || ds.slab_plane[1] != 0) {
            if (dim != 3 || ds.slab_plane[0] <= 0 || ds.slab_plane[1] < ds.slab_plane[0] ||
                E % ds.slab_plane[0] != 0)
                throw ConfigError("slab_plane: 3D only, 0 < local <= global, divides n_elems");
            d.id_pl = ds.slab_plane[0];
            d.id_pg = ds.slab_plane[1];
        }
        d.own_lo = 0;
        d.own_hi = d.id_pl ? d.id_pl : E;
        if (ds.owned_elems[0] != 0 || ds.owned_elems[1] != 0) {
            if (ds.owned_elems[0] < 0 || ds.owned_elems[1] > d.own_hi ||
                ds.owned_elems[0] > ds.owned_elems[1])
                throw ConfigError("owned element range out of bounds");
            d.own_lo = ds.owned_elems[0];
            d.own_hi = ds.owned_elems[1];
        }
        const double dt = ds.dt, gm = ds.gamma, bt = ds.beta;
        d.c_pred_v = dt * (1.0 - gm);
        d.c_pred_d = dt * dt * (0.5 - bt);
        d.dt = dt;
        d.c_corr_v = gm * dt;
        d.c_corr_d = bt * dt * dt;
        // SoA uploads
        std::vector<int32_t> conn_soa((size_t)nn * E);
        for (int e = 0; e < E; ++e)
            for (int a = 0; a < nn; ++a) conn_soa[(size_t)a * E + e] = h->conn[(size_t)e * nn + a];
        std::vector<double> cen_soa(3 * (size_t)E);
        for (int e = 0; e < E; ++e)
            for (int k = 0; k < 3; ++k) cen_soa[(size_t)k * E + e] = h->cen[3 * (size_t)e + k];
        // node -> incident elements, ascending (damage_field / K row order)
        std::vector<int32_t> cnt(N, 0), ne((size_t)nn * N, -1);
        for (int e = 0; e < E; ++e)
            for (int a = 0; a < nn; ++a) {
                const int n = h->conn[(size_t)e * nn + a];
                if (cnt[n] >= nn) throw ConfigError("node shared by more than 2^dim elements");
                ne[(size_t)cnt[n]++ * N + n] = e;
            }
        int32_t* dconn = h->alloc<int32_t>(conn_soa.size());
        double* dcen = h->alloc<double>(cen_soa.size());
        double* dvol = h->alloc<double>(E);
        int32_t* dne = h->alloc<int32_t>(ne.size());
        upload(dconn, conn_soa.data(), conn_soa.size(), s);
        upload(dcen, cen_soa.data(), cen_soa.size(), s);
        upload(dvol, h->vol.data(), E, s);
        upload(dne, ne.data(), ne.size(), s);
        d.conn = dconn;
        d.cen = dcen;
        d.vol = dvol;
        d.ne = dne;
        const size_t nd = h->ndof;
        d.u = h->alloc<double>(nd);
        d.v = h->alloc<double>(nd);
        d.a = h->alloc<double>(nd);
        d.rd = h->alloc<double>(nd);
        d.rv = h->alloc<double>(nd);
        double* dM = h->alloc<double>(nd);
        double* dP = h->alloc<double>(nd);
        uint8_t* dflag = h->alloc<uint8_t>(nd);
        double* dbcv = h->alloc<double>(nd);
        upload(dM, ds.mass, nd, s);
        upload(dP, ds.p_ext, nd, s);
        upload(dflag, bcflag.data(), nd, s);
        upload(dbcv, bcvel.data(), nd, s);
        d.M = dM;
        d.P = dP;
        d.bcflag = dflag;
        d.bcvel = dbcv;
        d.G = h->alloc<double>((size_t)E * dim);
        d.ubar = h->alloc<double>((size_t)E * dim);
        CK(cudaMemsetAsync(d.u, 0, sizeof(double) * nd, s));
        CK(cudaMemsetAsync(d.a, 0, sizeof(double) * nd, s));
        // KinematicState::zero + prescribed velocities (driver_run.hpp:195-196)
        upload(d.v, bcvel.data(), nd, s);
        h->d_log_n = h->alloc<unsigned long long>(1);
        CK(cudaMemsetAsync(h->d_log_n, 0, sizeof(unsigned long long), s));
        d.log_n = h->d_log_n;
        ensure_counts(h.get(), 64);
        CK(cudaStreamSynchronize(s));
        *out = h.release();
    });
}

void pmts_pd_destroy(pmts_pd* h) {
    if (h && h->xstream) {
        cudaStreamSynchronize(h->xstream);
        cudaStreamDestroy(h->xstream);
        cudaEventDestroy(h->ev_edge);
        cudaEventDestroy(h->ev_x);
        h->xstream = nullptr;
    }
    if (h && h->comm) {
        if (h->stream) cudaStreamSynchronize(h->stream);
        nccl().comm_destroy((ncclComm_t)h->comm);
        h->comm = nullptr;
    }
    delete h;
}

int pmts_pd_build_families(pmts_pd* h) {
    return guard([&] {
        if (!h) throw ConfigError("null handle");
        FamilyBuild fb = build_families_device(
            h->dim, h->E, h->d.cen, h->lo, h->desc.delta, h->eps, (int)h->notch_npts.size(),
            h->notch_npts.data(), h->notch_pts.data(), h->stream);
        // fast mode on the generated lattice with nominal constants: the families stay
        // on the device and are encoded there (no host walk over the F entries; the
        // host copy is fetched only if a caller asks for pairs / intact states)
        if (h->mode == PMTS_FAST && h->desc.lattice_h > 0.0) {
            if (h->d.coef) h->release((void*)h->d.coef);
            if (h->d.mask) h->release(h->d.mask);
            if (h->d.col) h->release((void*)h->d.col);
            h->d.coef = nullptr;
            h->d.mask = nullptr;
            h->owned.push_back(fb.col);
            h->device_bytes += 4.0 * fb.K * (double)h->E;
            h->d.col = fb.col;
            h->d.K = fb.K;
            h->hcol.clear();
            h->families = true;
            h->lattice = false;
            if (try_lattice(h, fb.col)) return;
            // not encodable: the host path below (it re-uploads the families)
            h->families = false;
        }
        h->hcol.assign((size_t)fb.K * h->E, -1);
        download(h->hcol.data(), fb.col, (size_t)fb.K * h->E, h->stream);
        CK(cudaStreamSynchronize(h->stream));
        if (h->d.col == fb.col) {
            h->release(fb.col);
            h->d.col = nullptr;
        } else {
            cudaFree(fb.col);
        }
        finish_families(h, fb.K);
    });
}

int pmts_pd_set_pairs(pmts_pd* h, int64_t n_pairs, const int32_t* pairs) {
    return guard([&] {
        if (!h) throw ConfigError("null handle");
        const int E = h->E;
        std::vector<std::vector<int32_t>> fam(E);
        for (int64_t q = 0; q < n_pairs; ++q) {
            const int i = pairs[2 * q], j = pairs[2 * q + 1];
            if (i < 0 || j < 0 || i >= E || j >= E || i >= j)
                throw ConfigError("pair list must hold (i<j) element ids");
            fam[i].push_back(j);
            fam[j].push_back(i);
        }
        int K = 0;
        for (auto& f : fam) {
            std::sort(f.begin(), f.end());
            if (std::adjacent_find(f.begin(), f.end()) != f.end())
                throw ConfigError("duplicate pair");
            K = std::max<int>(K, (int)f.size());
        }
        h->hcol.assign((size_t)K * E, -1);
        for (int e = 0; e < E; ++e)
            for (size_t k = 0; k < fam[e].size(); ++k) h->hcol[k * E + e] = fam[e][k];
        finish_families(h, K);
    });
}

}  // extern "C"

namespace pmts {
// ---- internal (libpmts only): the MTS integrator (pmts_mts.cu) drives the
// deterministic kernels of a PD handle on its own state vectors ----
DevPD pd_internal_dev(pmts_pd* h) { return h->d; }
cudaStream_t pd_internal_stream(pmts_pd* h) { return h->stream; }
// coefficients of the directed entries from per-pair weights (pairs in
// pmts_pd_get_pairs order): coef = (w_pair * V_i V_j) * c(|xi|), the
// reference's f = coeff * qp.weight * micromodulus (perifem.hpp:247)
void pd_internal_pair_weights(pmts_pd* h, const double* w) {
    require_families(h);
    ensure_hcol(h);
    const int E = h->E, K = h->d.K;
    const int32_t* col = h->hcol.data();
    // per element: family length and the partners below it (families ascend, so the
    // upper partners of i are its entries below[i] .. len[i] - 1, in pair order)
    std::vector<int32_t> len(E), below(E);
    par_range(E, [&](int e) {
        int n = 0, b = 0;
        for (int k = 0; k < K; ++k) {
            const int p = col[(size_t)k * E + e];
            if (p < 0) break;
            ++n;
            if (p < e) ++b;
        }
        len[e] = n;
        below[e] = b;
    });
    std::vector<int64_t> first(E + 1, 0);
    for (int e = 0; e < E; ++e) first[e + 1] = first[e] + (len[e] - below[e]);
    std::vector<double> coef((size_t)K * E, 0.0);
    par_range(E, [&](int e) {
        for (int k = 0; k < len[e]; ++k) {
            const int p = col[(size_t)k * E + e];
            int64_t idx;  // the pair's index: rank of j among i's upper partners
            if (p > e) {
                idx = first[e] + (k - below[e]);
            } else {  // e in p's ascending family
                int lo = below[p], hi = len[p];
                while (lo < hi) {
                    const int mid = (lo + hi) / 2;
                    if (col[(size_t)mid * E + p] < e) lo = mid + 1;
                    else hi = mid;
                }
                idx = first[p] + (lo - below[p]);
            }
            const int i = std::min(e, p), j = std::max(e, p);
            double xi[3];
            for (int c = 0; c < 3; ++c) xi[c] = h->cen[3 * (size_t)j + c] - h->cen[3 * (size_t)i + c];
            const double xin = std::sqrt(xi[0] * xi[0] + xi[1] * xi[1] + xi[2] * xi[2]);
            const double wv = w[idx] * (h->vol[i] * h->vol[j]);
            coef[(size_t)k * E + e] = wv * micromodulus(h->desc, h->dim, xin);
        }
    });
    upload(const_cast<double*>(h->d.coef), coef.data(), coef.size(), h->stream);
    CK(cudaStreamSynchronize(h->stream));
}
}  // namespace pmts

extern "C" {

int pmts_pd_get_pairs(pmts_pd* h, int32_t* out, int64_t cap, int64_t* n_out) {
    return guard([&] {
        require_families(h);
        ensure_hcol(h);
        const int E = h->E, K = h->d.K;
        int64_t n = 0;
        for (int e = 0; e < E; ++e)
            for (int k = 0; k < K; ++k) {
                const int p = h->hcol[(size_t)k * E + e];
                if (p < 0) break;
                if (p <= e) continue;
                if (out && n < cap) {
                    out[2 * n] = e;
                    out[2 * n + 1] = p;
                }
                ++n;
            }
        if (n_out) *n_out = n;
    });
}

int pmts_pd_get_intact(pmts_pd* h, uint8_t* out, int64_t cap) {
    return guard([&] {
        require_families(h);
        if (h->lattice) {  // on the device, over the stencil bits
            const long long nb = launch_lat_intact(h->d, h->L, h->mask0, nullptr, h->stream);
            uint8_t* dv = nullptr;
            CK(cudaMallocAsync(&dv, (size_t)std::max(nb, 1LL), h->stream));
            launch_lat_intact(h->d, h->L, h->mask0, dv, h->stream);
            download(out, dv, (size_t)std::max<int64_t>(0, std::min<int64_t>(cap, nb)), h->stream);
            CK(cudaFreeAsync(dv, h->stream));
            CK(cudaStreamSynchronize(h->stream));
            return;
        }
        ensure_hcol(h);
        const int E = h->E, K = h->d.K;
        const std::vector<uint32_t> mask = ell_mask_host(h);
        int64_t n = 0;
        for (int e = 0; e < E; ++e)
            for (int k = 0; k < K; ++k) {
                const int p = h->hcol[(size_t)k * E + e];
                if (p < 0) break;
                if (p <= e) continue;
                if (n < cap) out[n] = (mask[(size_t)(k >> 5) * E + e] >> (k & 31)) & 1u;
                ++n;
            }
    });
}

int pmts_pd_info_get(pmts_pd* h, pmts_pd_info* info) {
    return guard([&] {
        require_families(h);
        const double E = h->E, N = h->N, dim = h->dim, F = double(h->n_entries);
        info->n_entries = h->n_entries;
        info->n_bonds = h->n_entries / 2;
        info->max_family = h->d.K;
        info->path = 0;
        info->stencil_size = 0;
        info->kernels_per_step = h->mode == PMTS_DETERMINISTIC ? 2 : 3;
        // algorithmic (compulsory) HBM bytes per step, DESIGN.md "Roofline"
        const double fam = F * (4.0 + 8.0) + E * h->d.W * 4.0 * 2.0;
        const double elem = E * (3 * 8.0) /*centroids*/ + E * dim * 8.0 /*G write*/;
        const double gather = h->mode == PMTS_DETERMINISTIC
                                  ? E * h->nn * 4.0 + N * dim * 8.0 /*conn + rd*/
                                  : E * dim * 8.0 * 2.0 /*ubar write+read*/ +
                                        (E * h->nn * 4.0 + N * dim * 8.0) /*ubar kernel*/;
        const double node = N * dim * 8.0 * (2 /*rd rv*/ + 5 /*u v a rd rv*/ + 2 /*M P*/) +
                            N * dim * 1.0 + N * h->nn * 4.0 + E * dim * 8.0 /*G read*/;
        info->bytes_per_step = fam + elem + gather + node;
        info->bond_bytes_per_step =
            fam + elem +
            (h->mode == PMTS_DETERMINISTIC ? E * h->nn * 4.0 + N * dim * 8.0 : E * dim * 8.0);
        if (h->lattice) {
            // ubar: rd in, ubar out | bond: ubar in, bits in, G out | node: G, rd, rv, M,
            // P, flags in; rd, rv out (u, v, a only on a batch's last step)
            info->path = 1;
            info->stencil_size = h->L.S;
            const double ubar = N * dim * 8.0 + E * dim * 8.0;
            const double bond = E * dim * 8.0 + E * h->L.W * 4.0 + E * dim * 8.0;
            const double nodek = E * dim * 8.0 + N * dim * 8.0 * 6 + N * dim * 1.0;
            info->bytes_per_step = ubar + bond + nodek;
            info->bond_bytes_per_step = bond;
            if (h->fused) {
                // rd in + out, rv in + out, 1/M, node flags, mask in + out
                info->kernels_per_step = 1;
                info->path = 2;
                // (node flags ride in 1/M; bond-state words only move on the tiles that
                // stage them -- the clean tiles of pd_tile9.cu touch none)
                info->bytes_per_step =
                    N * dim * 8.0 * 4 + N * 8.0 + tile9_staged_elements(h) * 4.0 * 2;
                info->bond_bytes_per_step = info->bytes_per_step;
            }
        }
        info->device_bytes = h->device_bytes;
        info->hot_tiles = info->tested_tiles = 0;
        if (h->hot_count) {
            unsigned long long c[2] = {0, 0};
            download(c, h->hot_count, 2, h->stream);
            CK(cudaStreamSynchronize(h->stream));
            info->hot_tiles = (int64_t)c[0];
            info->tested_tiles = (int64_t)c[1];
        }
    });
}

int pmts_pd_init(pmts_pd* h, double scale0) {
    return guard([&] {
        require_families(h);
        if (h->lattice) {  // K u0 through the stencil kernels (rd <- u0 first)
            CK(cudaMemcpyAsync(h->d.rd, h->d.u, sizeof(double) * h->ndof,
                               cudaMemcpyDeviceToDevice, h->stream));
            ensure_counts(h, 1);
            DevPD dd = h->d;
            double* junk = nullptr;
            CK(cudaMallocAsync(&junk, sizeof(double) * 2 * h->ndof, h->stream));
            dd.rv = junk;  // the node kernel's predictor output is discarded here
            dd.rd = junk + h->ndof;
            CK(cudaMemcpyAsync(dd.rd, h->d.u, sizeof(double) * h->ndof,
                               cudaMemcpyDeviceToDevice, h->stream));
            launch_lattice_step(dd, h->L, 0, 0, 0.0, 0, false, nullptr, h->stream,
                                h->lat3 ? &h->st3 : nullptr);
            CK(cudaFreeAsync(junk, h->stream));
        } else {
            launch_det_bond(h->d, h->d.u, 0, 0, 0, h->stream);
        }
        launch_init_acc(h->d, scale0, h->stream);
        launch_predict(h->d, h->stream);
        exchange_halo(h);
        CK(cudaStreamSynchronize(h->stream));
    });
}

int pmts_pd_step(pmts_pd* h, int32_t n, const double* scales, int64_t* n_broken_out) {
    return guard([&] {
        require_families(h);
        if (n < 0 || (n > 0 && !scales)) throw ConfigError("bad step count or scales");
        ensure_counts(h, std::max(n, 1));
        for (int s = 0; s < n; ++s) enqueue_step(h, s, scales[s], false, nullptr, s == n - 1);
        const int64_t nb = finish_steps(h, n);
        if (n_broken_out) *n_broken_out = nb;
    });
}

int pmts_pd_step_tracked(pmts_pd* h, int32_t n, const double* scales, int32_t n_tracked,
                         const int32_t* dofs, double* tracked_out, int64_t* broken_out) {
    return guard([&] {
        require_families(h);
        if (n < 0 || (n > 0 && !scales) || n_tracked < 0) throw ConfigError("bad arguments");
        for (int j = 0; j < n_tracked; ++j)
            if (dofs[j] < 0 || dofs[j] >= h->ndof) throw ConfigError("tracked dof out of range");
        ensure_counts(h, std::max(n, 1));
        // device staging (kept across calls): tracked dofs, per-step scales
        const size_t idx_bytes = (sizeof(int32_t) * n_tracked + 7) & ~size_t(7);
        const size_t scl_bytes = sizeof(double) * (size_t)std::max(n, 1);
        const size_t bytes = idx_bytes + scl_bytes;
        if (bytes > h->trk_cap) {
            if (h->trk_buf) h->release(h->trk_buf);
            h->trk_cap = std::max<size_t>(bytes, 4096);
            h->trk_buf = h->alloc<char>(h->trk_cap);
            h->trk_dofs.clear();
        }
        int32_t* didx = reinterpret_cast<int32_t*>(h->trk_buf);
        double* dscl = reinterpret_cast<double*>(h->trk_buf + idx_bytes);
        // mapped pinned staging: per-step scales (read by the device), tracked rows
        // and broken counts (written by the device)
        const size_t need = sizeof(double) * ((size_t)n * (1 + n_tracked)) +
                            sizeof(unsigned long long) * (size_t)n;
        if (need > h->h_map_cap) {
            if (h->h_map) cudaFreeHost(h->h_map);
            h->h_map_cap = std::max<size_t>(need, 4096);
            CK(cudaHostAlloc(&h->h_map, h->h_map_cap, cudaHostAllocMapped));
        }
        double* h_scl = reinterpret_cast<double*>(h->h_map);
        double* h_trk = h_scl + n;
        unsigned long long* h_cnt = reinterpret_cast<unsigned long long*>(h_trk + (size_t)n * n_tracked);
        void* dmap = nullptr;
        CK(cudaHostGetDevicePointer(&dmap, h->h_map, 0));
        double* m_scl = reinterpret_cast<double*>(dmap);
        double* m_trk = m_scl + n;
        unsigned long long* m_cnt = reinterpret_cast<unsigned long long*>(m_trk + (size_t)n * n_tracked);
        std::copy(scales, scales + n, h_scl);
        if (h->trk_dofs.size() != (size_t)n_tracked ||
            !std::equal(h->trk_dofs.begin(), h->trk_dofs.end(), dofs)) {
            h->trk_dofs.assign(dofs, dofs + n_tracked);
            if (n_tracked) upload(didx, dofs, n_tracked, h->stream);
        }
        // per step, all asynchronous on the handle's stream (one synchronisation at
        // the end).  tile9: the scales go up in one copy, each step's kernel writes
        // its tracked row into mapped pinned host memory from the node update, and
        // the broken counts come back in one copy -- one launch per step.  Other
        // paths: the step, then one tiny launch that writes the step's tracked row
        // and broken count into mapped pinned host memory and moves the next step's
        // scale from mapped pinned host memory to the device.
        if (h->tile9 && n > 0) {
            upload(dscl, h_scl, n, h->stream);
            for (int s = 0; s < n; ++s) {
                FusedBufs rep{};
                rep.trk_dofs = didx;
                rep.n_trk = n_tracked;
                rep.trk_host = m_trk + (size_t)s * n_tracked;
                enqueue_step(h, s, scales[s], false, nullptr, s == n - 1, dscl, &rep);
            }
            download(h_cnt, h->d_counts, n, h->stream);
        } else if (n > 0 && h->lattice && !h->fused) {
            // lattice path (3D): with beta = 0 the step's u is the predictor rd it
            // starts from (u = rd + (beta dt) dt a), so the tracked row is read from rd
            // before the step -- no per-step u, v, a materialisation; the broken counts
            // come back in one copy at the end
            for (int s = 0; s < n; ++s) {
                launch_track(h->d.rd, didx, n_tracked, m_trk + (size_t)s * n_tracked, nullptr,
                             nullptr, nullptr, nullptr, h->stream);
                enqueue_step(h, s, scales[s], false, nullptr, s == n - 1, nullptr);
            }
            download(h_cnt, h->d_counts, n, h->stream);
        } else if (n > 0) {
            upload(dscl, h_scl, 1, h->stream);
        }
        for (int s = 0; s < n && !h->tile9 && !(h->lattice && !h->fused); ++s) {
            // u of step s: the fused kernel's displacement is the step's predictor
            // (beta = 0), i.e. the rd buffer it consumed; the other paths write u
            const bool every = !h->fused;
            enqueue_step(h, s, scales[s], false, nullptr, every || s == n - 1, nullptr);
            const double* src = h->fused ? h->rd_alt : h->d.u;
            launch_track(src, didx, n_tracked, m_trk + (size_t)s * n_tracked, h->d_counts + s,
                         m_cnt + s, s + 1 < n ? m_scl + s + 1 : nullptr,
                         s + 1 < n ? dscl + s + 1 : nullptr, h->stream);
        }
        CK(cudaStreamSynchronize(h->stream));
        if (n_tracked && n) std::copy(h_trk, h_trk + (size_t)n * n_tracked, tracked_out);
        const unsigned long long* cnt = h_cnt;
        int64_t nb = 0;
        for (int s = 0; s < n; ++s) {
            nb += (int64_t)cnt[s];
            if (broken_out) broken_out[s] = (int64_t)cnt[s];
        }
        h->gstep += n;
        h->broken_total += nb;
    });
}

int pmts_pd_step_timed(pmts_pd* h, int32_t n, const double* scales, float* ms_out) {
    return guard([&] {
        require_families(h);
        ensure_counts(h, std::max(n, 1));
        cudaEvent_t e0, e1;
        CK(cudaEventCreate(&e0));
        CK(cudaEventCreate(&e1));
        CK(cudaEventRecord(e0, h->stream));
        for (int s = 0; s < n; ++s) enqueue_step(h, s, scales[s], false, nullptr, s == n - 1);
        CK(cudaEventRecord(e1, h->stream));
        finish_steps(h, n);
        float ms = 0.f;
        CK(cudaEventElapsedTime(&ms, e0, e1));
        cudaEventDestroy(e0);
        cudaEventDestroy(e1);
        *ms_out = ms;
    });
}

int pmts_pd_profile(pmts_pd* h, int32_t n, const double* scales, float* bond_ms,
                    float* total_ms) {
    return guard([&] {
        require_families(h);
        ensure_counts(h, std::max(n, 1));
        std::vector<cudaEvent_t> ev(2 * n + 2);
        for (auto& e : ev) CK(cudaEventCreate(&e));
        CK(cudaEventRecord(ev[2 * n], h->stream));
        for (int s = 0; s < n; ++s) enqueue_step(h, s, scales[s], true, &ev[2 * s], s == n - 1);
        CK(cudaEventRecord(ev[2 * n + 1], h->stream));
        finish_steps(h, n);
        float b = 0.f, t = 0.f;
        for (int s = 0; s < n; ++s) {
            float ms = 0.f;
            CK(cudaEventElapsedTime(&ms, ev[2 * s], ev[2 * s + 1]));
            b += ms;
        }
        CK(cudaEventElapsedTime(&t, ev[2 * n], ev[2 * n + 1]));
        for (auto& e : ev) cudaEventDestroy(e);
        *bond_ms = b;
        *total_ms = t;
    });
}

int pmts_pd_get_state(pmts_pd* h, double* u, double* v, double* a) {
    return guard([&] {
        if (!h) throw ConfigError("null handle");
        if (u) download(u, h->d.u, h->ndof, h->stream);
        if (v) download(v, h->d.v, h->ndof, h->stream);
        if (a) download(a, h->d.a, h->ndof, h->stream);
        CK(cudaStreamSynchronize(h->stream));
    });
}

int pmts_pd_set_state(pmts_pd* h, const double* u, const double* v, const double* a) {
    return guard([&] {
        if (!h) throw ConfigError("null handle");
        if (u) upload(h->d.u, u, h->ndof, h->stream);
        if (v) upload(h->d.v, v, h->ndof, h->stream);
        if (a) upload(h->d.a, a, h->ndof, h->stream);
        launch_predict(h->d, h->stream);
        exchange_halo(h);
        CK(cudaStreamSynchronize(h->stream));
    });
}

int pmts_pd_take_break_log(pmts_pd* h, int32_t* rows, int64_t cap, int64_t* n_out) {
    return guard([&] {
        require_families(h);
        if (!h->d.log) throw ConfigError("break log is kept in PMTS_DETERMINISTIC mode only");
        unsigned long long n = 0;
        download(&n, h->d_log_n, 1, h->stream);
        CK(cudaStreamSynchronize(h->stream));
        if ((long long)n > h->d.log_cap) throw InternalError("break log overflow");
        std::vector<int32_t> buf(3 * (size_t)n);
        download(buf.data(), h->d_log, buf.size(), h->stream);
        CK(cudaMemsetAsync(h->d_log_n, 0, sizeof(unsigned long long), h->stream));
        CK(cudaStreamSynchronize(h->stream));
        std::vector<std::array<int32_t, 3>> r(n);
        for (size_t k = 0; k < n; ++k) r[k] = {buf[3 * k], buf[3 * k + 1], buf[3 * k + 2]};
        std::sort(r.begin(), r.end());
        for (size_t k = 0; k < n && (int64_t)k < cap; ++k)
            for (int c = 0; c < 3; ++c) rows[3 * k + c] = r[k][c];
        if (n_out) *n_out = (int64_t)n;
    });
}

int64_t pmts_pd_broken_total(pmts_pd* h) { return h ? h->broken_total : -1; }

int pmts_pd_damage(pmts_pd* h, double* elem, double* node) {
    return guard([&] {
        require_families(h);
        double* de = nullptr;
        double* dn = nullptr;
        CK(cudaMallocAsync(&de, sizeof(double) * h->E, h->stream));
        CK(cudaMallocAsync(&dn, sizeof(double) * h->N, h->stream));
        if (h->lattice)  // over the stencil bits on the device
            launch_lat_damage(h->d, h->L, h->mask0, h->pos_only, de, dn, h->stream);
        else
            launch_damage(h->d, de, dn, h->stream);
        if (elem) download(elem, de, h->E, h->stream);
        if (node) download(node, dn, h->N, h->stream);
        CK(cudaFreeAsync(de, h->stream));
        CK(cudaFreeAsync(dn, h->stream));
        CK(cudaStreamSynchronize(h->stream));
    });
}

int pmts_pd_gather_disp(pmts_pd* h, int32_t n, const int32_t* dofs, double* out) {
    return guard([&] {
        if (!h) throw ConfigError("null handle");
        for (int k = 0; k < n; ++k) {
            if (dofs[k] < 0 || dofs[k] >= h->ndof) throw ConfigError("dof out of range");
            download(out + k, h->d.u + dofs[k], 1, h->stream);
        }
        CK(cudaStreamSynchronize(h->stream));
    });
}

void* pmts_pd_stream(pmts_pd* h) { return h ? (void*)h->stream : nullptr; }

int pmts_pd_get_rows_layers(pmts_pd* h, int32_t first, int32_t n, int32_t layers,
                            int32_t stride, double* out) {
    return guard([&] {
        if (!h) throw ConfigError("null handle");
        if (first < 0 || n < 0 || layers < 1 || stride < 0 ||
            (int64_t)first + (int64_t)(layers - 1) * stride + n > h->N)
            throw ConfigError("node range out of bounds");
        const size_t w = (size_t)n * h->dim * sizeof(double);
        CK(cudaMemcpy2DAsync(out, w, h->d.rd + (size_t)first * h->dim,
                             (size_t)stride * h->dim * sizeof(double), w, layers,
                             cudaMemcpyDeviceToHost, h->stream));
        CK(cudaStreamSynchronize(h->stream));
    });
}

int pmts_pd_set_rows_layers(pmts_pd* h, int32_t first, int32_t n, int32_t layers, int32_t stride,
                            const double* in) {
    return guard([&] {
        if (!h) throw ConfigError("null handle");
        if (first < 0 || n < 0 || layers < 1 || stride < 0 ||
            (int64_t)first + (int64_t)(layers - 1) * stride + n > h->N)
            throw ConfigError("node range out of bounds");
        const size_t w = (size_t)n * h->dim * sizeof(double);
        CK(cudaMemcpy2DAsync(h->d.rd + (size_t)first * h->dim,
                             (size_t)stride * h->dim * sizeof(double), in, w, w, layers,
                             cudaMemcpyHostToDevice, h->stream));
        CK(cudaStreamSynchronize(h->stream));
    });
}

int pmts_pd_get_rows(pmts_pd* h, int32_t first, int32_t n, double* out) {
    return pmts_pd_get_rows_layers(h, first, n, 1, 0, out);
}

int pmts_pd_set_rows(pmts_pd* h, int32_t first, int32_t n, const double* in) {
    return pmts_pd_set_rows_layers(h, first, n, 1, 0, in);
}

int pmts_nccl_unique_id(void* id_out) {
    return guard([&] {
        ncclUniqueId id;
        nccl_check(nccl().get_unique_id(&id), "get unique id");
        std::memcpy(id_out, &id, sizeof(id));
    });
}

int pmts_pd_comm_init(pmts_pd* h, const void* id, int32_t nranks, int32_t rank) {
    return guard([&] {
        if (!h) throw ConfigError("null handle");
        if (nranks < 1 || rank < 0 || rank >= nranks) throw ConfigError("bad rank / size");
        ncclUniqueId uid;
        std::memcpy(&uid, id, sizeof(uid));
        CK(cudaSetDevice(h->desc.device));
        ncclComm_t c = nullptr;
        nccl_check(nccl().comm_init_rank(&c, nranks, uid, rank), "comm init");
        h->comm = c;
    });
}

int pmts_pd_set_halo(pmts_pd* h, int32_t peer_lo, int32_t send_lo_first, int32_t recv_lo_first,
                     int32_t n_lo, int32_t peer_hi, int32_t send_hi_first,
                     int32_t recv_hi_first, int32_t n_hi) {
    return guard([&] {
        if (!h) throw ConfigError("null handle");
        auto ok = [&](int f, int n) { return f >= 0 && n >= 0 && f + n <= h->N; };
        if ((peer_lo >= 0 && (!ok(send_lo_first, n_lo) || !ok(recv_lo_first, n_lo))) ||
            (peer_hi >= 0 && (!ok(send_hi_first, n_hi) || !ok(recv_hi_first, n_hi))))
            throw ConfigError("halo node range out of bounds");
        h->peer_lo = peer_lo;
        h->send_lo = send_lo_first;
        h->recv_lo = recv_lo_first;
        h->n_lo = n_lo;
        h->peer_hi = peer_hi;
        h->send_hi = send_hi_first;
        h->recv_hi = recv_hi_first;
        h->n_hi = n_hi;
        plan_split(h);
    });
}

int pmts_pd_set_option(pmts_pd* h, int32_t option, int32_t value) {
    return guard([&] {
        if (!h) throw ConfigError("null handle");
        switch (option) {
            case PMTS_OPT_BREAK_SCREEN:
                h->screen = value != 0;
                h->pst.screen = h->screen ? 1 : 0;
                h->st3.tmax = h->screen ? h->lat3_tmax : nullptr;
                break;
            case PMTS_OPT_HALO_OVERLAP:
                h->halo_overlap = value != 0;
                if (h->halo_overlap && h->halo_layers > 1)
                    throw ConfigError("halo overlap: 2D slabs only");
                if (h->families) plan_split(h);
                break;
            case PMTS_OPT_COUNT_HOT: {
                unsigned long long* c = nullptr;
                if (value) {
                    c = h->hot_count ? h->hot_count : h->alloc<unsigned long long>(2);
                    CK(cudaMemsetAsync(c, 0, 16, h->stream));
                }
                h->hot_count = c ? c : h->hot_count;
                h->pst.hot_count = c;
                h->st3.hot_count = c;
                break;
            }
            case PMTS_OPT_CLEAN_TILES:
                // off: every tile stages and re-writes its bond states again; turning it
                // back on recomputes the flags from the current states
                h->t9_clean_on = value != 0;
                h->t9_clean_ready = false;
                break;
            default:
                throw ConfigError("unknown option " + std::to_string(option));
        }
        CK(cudaStreamSynchronize(h->stream));
    });
}

// ---- coupled-integrator hooks: the PD side of a reference
// CoupledIntegrator that keeps its own FE side (deterministic mode) ----
int pmts_pd_set_constraint_load(pmts_pd* h, int32_t n, const int32_t* dofs, const double* vals) {
    return guard([&] {
        if (!h) throw ConfigError("null handle");
        if (h->mode != PMTS_DETERMINISTIC)
            throw ConfigError("constraint loads: PMTS_DETERMINISTIC handles only");
        if (n < 0) throw ConfigError("negative count");
        if (n == 0) {
            h->d.extra = nullptr;
            return;
        }
        if (!h->d_extra) h->d_extra = h->alloc<double>(h->ndof);
        std::vector<double> e(h->ndof, 0.0);
        for (int k = 0; k < n; ++k) {
            if (dofs[k] < 0 || dofs[k] >= h->ndof) throw ConfigError("dof out of range");
            e[dofs[k]] = vals[k];  // G_PD is Boolean: one value per coupling dof
        }
        upload(h->d_extra, e.data(), h->ndof, h->stream);
        h->d.extra = h->d_extra;
        CK(cudaStreamSynchronize(h->stream));
    });
}

int pmts_pd_snapshot_bonds(pmts_pd* h) {
    return guard([&] {
        require_families(h);
        if (h->mode != PMTS_DETERMINISTIC) throw ConfigError("PMTS_DETERMINISTIC handles only");
        const size_t words = (size_t)h->d.W * h->E;
        if (!h->mask_sync) h->mask_sync = h->alloc<uint32_t>(words);
        CK(cudaMemcpyAsync(h->mask_sync, h->d.mask, sizeof(uint32_t) * words,
                           cudaMemcpyDeviceToDevice, h->stream));
        CK(cudaStreamSynchronize(h->stream));
    });
}

int pmts_pd_homogeneous_recursion(pmts_pd* h, int32_t m, int32_t n, const int32_t* dofs,
                                  const double* w, double* vel_out, double* u_out, double* v_out,
                                  double* a_out) {
    return guard([&] {
        require_families(h);
        if (h->mode != PMTS_DETERMINISTIC) throw ConfigError("PMTS_DETERMINISTIC handles only");
        if (m < 1 || n < 0) throw ConfigError("bad m / n");
        if (!h->mask_sync) throw ConfigError("pmts_pd_snapshot_bonds first");
        const int nd = h->ndof;
        cudaStream_t s = h->stream;
        if (!h->famT_col) {  // entry-major families of the linear force
            const size_t ek = (size_t)h->E * h->d.K;
            h->famT_col = h->alloc<int32_t>(ek);
            h->famT_coef = h->alloc<double>(ek);
            mtsk::family_transpose(h->d, h->famT_col, h->famT_coef, s);
            for (double** p : {&h->rec_rd, &h->rec_rv, &h->rec_u, &h->rec_v, &h->rec_a})
                *p = h->alloc<double>(nd);
            h->rec_row_of = h->alloc<int32_t>(nd);
        }
        if (n > h->rec_rows_cap || m > h->rec_m_cap) {
            if (h->rec_w) h->release(h->rec_w);
            if (h->rec_out) h->release(h->rec_out);
            h->rec_rows_cap = std::max(n, 1);
            h->rec_m_cap = m;
            h->rec_w = h->alloc<double>(h->rec_rows_cap);
            h->rec_out = h->alloc<double>((size_t)(m + 1) * h->rec_rows_cap);
        }
        std::vector<int32_t> ro(nd, -1);
        for (int r = 0; r < n; ++r) {
            if (dofs[r] < 0 || dofs[r] >= nd) throw ConfigError("dof out of range");
            ro[dofs[r]] = r;
        }
        upload(h->rec_row_of, ro.data(), nd, s);
        if (n) upload(h->rec_w, w, n, s);
        CK(cudaMemsetAsync(h->rec_out, 0, sizeof(double) * (size_t)(m + 1) * h->rec_rows_cap, s));
        CK(cudaMemsetAsync(h->rec_rd, 0, sizeof(double) * nd, s));
        CK(cudaMemsetAsync(h->rec_rv, 0, sizeof(double) * nd, s));
        const DevPD& d = h->d;
        for (int j = 1; j <= m; ++j) {
            if (j > 1)
                mtsk::pd_force_lin_t(d, h->famT_col, h->famT_coef, h->rec_rd,
                                     h->mask_sync, d.ubar, s);
            mtsk::pd_node_lin(d, j > 1 ? 1 : 0, h->rec_w, h->rec_row_of, double(j) / m, d.M,
                              d.bcflag, d.c_corr_v, d.c_corr_d, d.dt, d.c_pred_v, d.c_pred_d,
                              h->rec_u, h->rec_v, h->rec_a, h->rec_rd, h->rec_rv,
                              h->rec_out + (size_t)j * h->rec_rows_cap, s);
        }
        for (int j = 0; vel_out && j <= m; ++j)
            download(vel_out + (size_t)j * n, h->rec_out + (size_t)j * h->rec_rows_cap, n, s);
        if (u_out) download(u_out, h->rec_u, nd, s);
        if (v_out) download(v_out, h->rec_v, nd, s);
        if (a_out) download(a_out, h->rec_a, nd, s);
        CK(cudaStreamSynchronize(s));
    });
}

int pmts_pd_set_halo_layers(pmts_pd* h, int32_t layers, int32_t stride) {
    return guard([&] {
        if (!h) throw ConfigError("null handle");
        if (layers < 1 || stride < 0) throw ConfigError("bad halo layers");
        auto ok = [&](int f, int n) {
            return (int64_t)f + (int64_t)(layers - 1) * stride + n <= h->N;
        };
        if ((h->peer_lo >= 0 && (!ok(h->send_lo, h->n_lo) || !ok(h->recv_lo, h->n_lo))) ||
            (h->peer_hi >= 0 && (!ok(h->send_hi, h->n_hi) || !ok(h->recv_hi, h->n_hi))))
            throw ConfigError("layered halo range out of bounds");
        if (layers > 1 && h->split_a >= 0) throw ConfigError("layered halos: no launch split");
        h->halo_layers = layers;
        h->halo_stride = stride;
        if (h->halo_buf) h->release(h->halo_buf);
        h->halo_buf = nullptr;
        if (layers > 1)
            h->halo_buf = h->alloc<double>(2 * (size_t)(h->n_lo + h->n_hi) * h->dim * layers);
    });
}

int pmts_pd_allreduce_sum(pmts_pd* h, int64_t* value) {
    return guard([&] {
        if (!h) throw ConfigError("null handle");
        if (!h->comm) return;
        int64_t* d = nullptr;
        CK(cudaMallocAsync(&d, sizeof(int64_t), h->stream));
        upload(d, value, 1, h->stream);
        nccl_check(nccl().all_reduce(d, d, 1, ncclInt64, ncclSum, (ncclComm_t)h->comm, h->stream),
                   "allreduce");
        download(value, d, 1, h->stream);
        CK(cudaFreeAsync(d, h->stream));
        CK(cudaStreamSynchronize(h->stream));
    });
}

}  // extern "C"
