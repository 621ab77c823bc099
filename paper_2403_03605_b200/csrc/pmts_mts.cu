// Coupled multi-time-step (Arlequin) integrator on the device -- SURVEY.md
// 8(f) row 1, behind pmts_mts_* (include/pmts_capi.h).
//
// A restatement of the reference's CoupledIntegrator (mts.hpp:79-535) with
// every FE / PD state, unit response and multiplier vector resident in HBM:
//   * FE operator: the alpha-weighted stiffness in CSR, assembled on the host
//     exactly as the reference (pmts_mts_setup.cpp), applied in the
//     reference's row order (pd_mts.cu); implicit FE solves are the
//     reference's Jacobi-PCG (linalg.hpp:243-296) with device reductions;
//   * PD operator: the matrix-free K^PD x of the deterministic kernels
//     (pd_det.cu) over the PD-active elements, per-pair (1 - alpha) weights in
//     the bond coefficients, the live bond mask and the unit-response snapshot
//     (k_sync_, mts.hpp:98) as two bit masks; the bond test of each free PD
//     substep is fused into that substep's force pass (beta_pd = 0: the tested
//     displacement is the force's predictor, mts.hpp:159-177);
//   * interface: dense H = H_FE + G_PD vel(Y_PD) factored on the host with the
//     reference's DenseLu (linalg.hpp:368-412), or the matrix-free CG on the
//     device (apply_h_pd = m linear PD substeps per iteration, mts.hpp:184-215,
//     410-420).
// The summation order of K x differs from the reference's CSR (matrix-free PD,
// device CG reductions), so parity is to rounding (tests/test_gpu_mts.py), the
// setup arrays bitwise (tests/test_mts_setup.py).
#include <algorithm>
#include <cstdlib>
#include <chrono>
#include <cmath>
#include <cstring>
#include <condition_variable>
#include <memory>
#include <mutex>
#include <thread>
#include <unordered_map>
#include <vector>

#include "pd_common.cuh"
#include "pd_mts.cuh"
#include "pmts_mts_setup.h"
#include "nccl_rt.h"

namespace pmts {
DevPD pd_internal_dev(pmts_pd* h);
cudaStream_t pd_internal_stream(pmts_pd* h);
void pd_internal_pair_weights(pmts_pd* h, const double* w);
}  // namespace pmts

using namespace pmts;

namespace {

void ck(cudaError_t e, const char* what) {
    if (e != cudaSuccess)
        throw InternalError(std::string("CUDA: ") + cudaGetErrorString(e) + " (" + what + ")");
}
#define CKM(x) ck((x), #x)

void check_pd(int status) {
    if (status == PMTS_OK) return;
    const std::string msg = pmts_last_error();
    if (status == PMTS_ERR_CONFIG) throw ConfigError(msg);
    if (status == PMTS_ERR_SOLVER) throw SolverError(msg);
    throw InternalError(msg);
}

double now_s() {
    return std::chrono::duration<double>(std::chrono::steady_clock::now().time_since_epoch())
        .count();
}


struct DState {
    double *u = nullptr, *v = nullptr, *a = nullptr;
};

// Newmark coefficients rounded as the reference's expressions
struct Nm {
    double gamma = 0.5, beta = 0.0, dt = 0.0;
    double cpv = 0, cpd = 0, gdt = 0, bdt2 = 0;
    void set(double g, double b, double d) {
        gamma = g;
        beta = b;
        dt = d;
        cpv = dt * (1.0 - gamma);          // newmark.hpp:65
        cpd = dt * dt * (0.5 - beta);      // newmark.hpp:66
        gdt = gamma * dt;                  // newmark.hpp:153
        bdt2 = beta * dt * dt;             // newmark.hpp:141,154
    }
    bool explicit_scheme() const { return beta == 0.0; }
};

// ---- PD shards of the coupled run (north star item 5) ----
// The PD-active elements are cut into slabs of element layers along the slowest
// lattice axis (y in 2D, z in 3D -- the PD numbering's slowest axis, so the elements a
// shard owns are one contiguous local range).  Shard r owns the element layers
// [b_r, b_{r+1}) and the node layers [b_r, b_{r+1}) (the last shard also the far
// layer); it holds every element within D + 1 layers of them (D = floor(delta / h),
// the largest layer distance of a bond), so the elements incident to its nodes have
// complete families.  Local elements and nodes keep the global order: the families,
// the per-entry arithmetic and its e < p branches run exactly as in one domain.
struct ShardLink {
    int peer = -1;
    std::vector<int32_t> send, recv;  // local dofs; my send list is the peer's recv list
};
struct ShardPlan {
    int world = 1, rank = 0, axis = 0, D = 0, layers = 0;
    std::vector<int> bounds;  // world + 1 element-layer bounds
    std::vector<int> elems;   // local element -> PD-active index (ascending)
    std::vector<int> nodes;   // local node -> compact PD node (ascending)
    int own_e0 = 0, own_e1 = 0;
    std::vector<uint8_t> node_own;  // per local node
    std::vector<ShardLink> links;   // lower, then upper neighbour
};

ShardPlan make_shard_plan(const MtsSystem& s, double h, int world, int rank) {
    ShardPlan p;
    p.world = world;
    p.rank = rank;
    const int dim = s.dim, nn = dim == 2 ? 4 : 8;
    p.axis = dim - 1;
    const int NE = int(s.pd_active.size()), NN = int(s.pd_active_nodes.size());
    std::vector<int> compact(s.nodes.size() / 3, -1);
    for (int c = 0; c < NN; ++c) compact[s.pd_active_nodes[c]] = c;
    for (int c = 0; c < NN; ++c)
        for (int k = 0; k < dim; ++k)
            if (s.pd_node_dof[s.pd_active_nodes[c]] != c * dim)
                throw InternalError("PD dofs are not in compact node order");
    double org = 1e300;
    for (int c = 0; c < NN; ++c)
        org = std::min(org, s.nodes[3 * (size_t)s.pd_active_nodes[c] + p.axis]);
    std::vector<int> el(NE), nlay(NN);
    int L = 0;
    for (int k = 0; k < NE; ++k) {
        const double x = s.centroid[3 * (size_t)s.pd_active[k] + p.axis];
        el[k] = int(std::llround((x - org) / h - 0.5));
        if (k && el[k] < el[k - 1])
            throw ConfigError("sharded coupled run: the PD elements are not ordered along the cut axis");
        L = std::max(L, el[k] + 1);
    }
    for (int c = 0; c < NN; ++c)
        nlay[c] = int(std::llround((s.nodes[3 * (size_t)s.pd_active_nodes[c] + p.axis] - org) / h));
    p.layers = L;
    p.D = int(std::floor(s.delta / h * (1.0 + 1e-9)));
    p.bounds.resize(world + 1);
    for (int r = 0; r <= world; ++r) p.bounds[r] = int((long long)r * L / world);
    for (int r = 0; r < world; ++r)
        if (p.bounds[r + 1] - p.bounds[r] < p.D + 1)  // (ghosts from the neighbours only)
            throw ConfigError("sharded coupled run: " + std::to_string(world) + " shards of " +
                              std::to_string(L) + " PD element layers leave fewer than D + 1 = " +
                              std::to_string(p.D + 1) + " layers per shard");
    auto owner = [&](int c) {
        const int l = nlay[c];
        for (int r = world - 1; r >= 0; --r)
            if (l >= p.bounds[r]) return r;
        return 0;
    };
    auto local_of = [&](int q, std::vector<int>& E, std::vector<int>& N) {
        const int lo = p.bounds[q] - 1 - p.D, hi = p.bounds[q + 1] + p.D;
        E.clear();
        for (int k = 0; k < NE; ++k)
            if (el[k] >= lo && el[k] < hi) E.push_back(k);
        std::vector<char> mark(NN, 0);
        for (int k : E)
            for (int a = 0; a < nn; ++a) mark[compact[s.conn[(size_t)s.pd_active[k] * nn + a]]] = 1;
        N.clear();
        for (int c = 0; c < NN; ++c)
            if (mark[c]) N.push_back(c);
    };
    local_of(rank, p.elems, p.nodes);
    p.own_e0 = p.own_e1 = 0;
    for (size_t i = 0; i < p.elems.size(); ++i) {
        if (el[p.elems[i]] < p.bounds[rank]) p.own_e0 = int(i) + 1;
        if (el[p.elems[i]] < p.bounds[rank + 1]) p.own_e1 = int(i) + 1;
    }
    p.node_own.resize(p.nodes.size());
    std::vector<int> g2l(NN, -1);
    for (size_t i = 0; i < p.nodes.size(); ++i) {
        g2l[p.nodes[i]] = int(i);
        const int o = owner(p.nodes[i]);
        p.node_own[i] = o == rank;
        if (o != rank && o != rank - 1 && o != rank + 1)
            throw InternalError("shard halo reaches past a neighbour");
    }
    for (int q : {rank - 1, rank + 1}) {
        if (q < 0 || q >= world) continue;
        std::vector<int> qE, qN;
        local_of(q, qE, qN);
        ShardLink lk;
        lk.peer = q;
        for (int c : p.nodes)
            if (owner(c) == q)
                for (int k = 0; k < dim; ++k) lk.recv.push_back(g2l[c] * dim + k);
        for (int c : qN)
            if (owner(c) == rank)
                for (int k = 0; k < dim; ++k) lk.send.push_back(g2l[c] * dim + k);
        p.links.push_back(std::move(lk));
    }
    return p;
}

// collectives of the sharded coupled step, all stream-ordered on the handle's stream
// and called by every shard in the same order (in-process group: host barriers and
// device copies between the shards' buffers; NCCL: one clique, send/recv + reductions)
struct MtsComm {
    virtual ~MtsComm() = default;
    // the halo dofs of x (a local PD vector) from their owners
    virtual void halo(pmts_mts& h, double* x) = 0;
    // x (n doubles) <- the sum over shards, every entry owned by one shard and -0.0
    // elsewhere: exact in any order (x + -0.0 == x)
    virtual void sum_owned(pmts_mts& h, double* x, size_t n) = 0;
    virtual void bcast(pmts_mts& h, void* x, size_t bytes) = 0;  // from shard 0
    virtual void reduce_u64(pmts_mts& h, unsigned long long* x, int n, bool max) = 0;
};

}  // namespace

struct pmts_mts {
    MtsSystem s;
    int device = 0;
    cudaStream_t stream = nullptr;
    // a second stream for the FE side: the FE and PD halves of the macro step are
    // independent between the multiplier updates (fork / join by events; captured into
    // the CG graphs as well: H_FE w next to the PD recursion of the interface operator)
    cudaStream_t stream2 = nullptr;
    cudaEvent_t ev_fork = nullptr, ev_join = nullptr, ev_fork2 = nullptr, ev_join2 = nullptr;
    void fork(cudaEvent_t e) {  // stream2 waits for the work enqueued on stream so far
        CKM(cudaEventRecord(e, stream));
        CKM(cudaStreamWaitEvent(stream2, e, 0));
    }
    void join(cudaEvent_t e) {  // stream waits for stream2
        CKM(cudaEventRecord(e, stream2));
        CKM(cudaStreamWaitEvent(stream, e, 0));
    }
    struct OnStream2 {  // route the member-stream calls of a block to stream2
        pmts_mts* h;
        explicit OnStream2(pmts_mts* hh) : h(hh) { std::swap(h->stream, h->stream2); }
        ~OnStream2() { std::swap(h->stream, h->stream2); }
    };
    double *rd_fe = nullptr, *rv_fe = nullptr, *ra_fe = nullptr, *lam_tmp_fe = nullptr;
    DState wst_fe;
    pmts_pd* pd = nullptr;
    DevPD pdv{};
    // ---- sharded coupled run (pmts_mts_desc.shard_world > 1): this
    // handle holds one PD shard (local nodes / elements of plan); shard 0 also the FE
    // side.  The interface solve is replicated on every shard (identical arithmetic:
    // the same multipliers everywhere, no broadcast of lambda)
    ShardPlan plan;
    bool sharded = false, root = true, setup_done = true;
    std::unique_ptr<MtsComm> comm;
    bool group_comm = false;
    int32_t* cpd_own = nullptr;  // coupling row -> local PD dof when this shard owns it, else -1
    int32_t* ident = nullptr;    // 0 .. nl - 1
    int32_t* own_dofs = nullptr;  // the owned local PD dofs
    double* own_zero = nullptr;   // zeros, one per owned dof
    int n_own_dofs = 0;
    double* gpd_now = nullptr;    // G_PD v at the macro step's end (continuity residual)
    struct LinkDev {
        int peer = -1, n_send = 0, n_recv = 0;
        int32_t *send = nullptr, *recv = nullptr;
        double *sbuf = nullptr, *rbuf = nullptr;
    };
    std::vector<LinkDev> links;
    double* sum_scratch = nullptr;
    size_t sum_cap = 0;
    int* more_d = nullptr;  // host-driven CG loop flag (device, pinned copy)
    int* more_h = nullptr;
    MtsComm& cm() {
        if (!comm) throw ConfigError("sharded coupled handle without a transport "
                                     "(pmts_mts_group_join / pmts_mts_comm_init)");
        return *comm;
    }
    void halo(double* x) {
        if (sharded) cm().halo(*this, x);
    }
    void sum_owned(double* x, size_t n) {
        if (sharded) cm().sum_owned(*this, x, n);
    }
    const int32_t* cpd_g() const { return sharded ? cpd_own : cpd; }
    std::vector<int32_t> pairs;  // global ids
    std::vector<double> pe_weight;
    int nf = 0, np = 0, nl = 0, npe = 0, m = 1;
    Nm fe_nm, pd_nm;
    int iface_mode = 0;
    bool interface_precond = false;  // pmts_mts_desc.interface_precond
    bool iface_precompute = true;    // pmts_mts_desc.interface_h_pd (precomputed H_PD)
    bool enforce_continuity = true, track_energy = true, fracture = false;
    double continuity_tol = 1e-8, cg_tol = 1e-10, interface_cg_tol = 1e-11;
    int fe_cg_max = 100;
    std::vector<void*> owned;
    // device: FE
    int32_t *fe_rp = nullptr, *fe_ci = nullptr;
    double *fe_v = nullptr, *fe_M = nullptr, *fe_P = nullptr, *fe_bcv = nullptr, *fe_jac = nullptr;
    uint8_t* fe_cf = nullptr;
    // device: PD
    double *pd_M = nullptr, *pd_P = nullptr, *pd_bcv = nullptr;
    uint8_t* pd_cf = nullptr;
    uint32_t *mask_live = nullptr, *mask_sync = nullptr;
    size_t mask_words = 0;
    unsigned long long* d_counts = nullptr;  // per substep slot
    int counts_cap = 0;
    // device: coupling
    int32_t *cfe = nullptr, *cpd = nullptr;
    // G_FE rows (CSR) and their transpose over the touched FE dofs
    int32_t *gfe_rp = nullptr, *gfe_ci = nullptr, *gft_d = nullptr, *gft_rp = nullptr,
            *gft_ri = nullptr;
    double *gfe_w = nullptr, *gft_w = nullptr;
    int gft_n = 0;
    // device: states and scratch
    DState ufe, upd, vfe, vpd, wst, yst, fe_prev;
    double *rd = nullptr, *rv = nullptr, *ra = nullptr, *kd = nullptr;     // size max(nf, np)
    double *cg_b = nullptr, *cg_x = nullptr, *cg_r = nullptr, *cg_z = nullptr, *cg_p = nullptr,
           *cg_ap = nullptr, *cg_kx = nullptr;                             // size max(nf, nl)
    double *part = nullptr, *scal = nullptr;                               // reductions
    double* part2 = nullptr;      // fused CG dots: two partial rows
    unsigned* ticket = nullptr;   // their last-block counter
    double* part3 = nullptr;      // operator-fused p.Ap partials (one per row block)
    unsigned* ticket3 = nullptr;
    int32_t* famT_col = nullptr;  // entry-major families (none on the lattice path below)
    double* famT_coef = nullptr;
    // 3D box lattice in lattice order with the 122-offset stencil: the linear force of the
    // homogeneous substeps on the k_sync snapshot runs in pd_mts_lat.cu
    bool lin_lat = false;
    mtsk::LinLat lat;
    // free substeps on large PD subdomains: per-element node products, formed once per
    // force call instead of once per family entry (pd_mts.cu k_pd_elem_q)
    double *elem_q = nullptr, *elem_s = nullptr;
    double *lam_d = nullptr, *lam_tmp = nullptr, *gvec = nullptr;          // size nl
    int32_t *hfe_rp = nullptr, *hfe_ci = nullptr;                          // H_FE, CSR
    double* hfe_v = nullptr;
    int64_t hfe_nnz = 0;
    double* iface_jac = nullptr;  // interface CG preconditioner (null: the reference's plain CG)
    double *sv_d = nullptr, *gp_free_d = nullptr, *gp_link_d = nullptr;    // m or m+1 rows of nl
    double* pd_ubar = nullptr;                                             // E_pd x dim
    int32_t* row_of = nullptr;                                             // PD dof -> coupling row
    double *warm_fe_free = nullptr, *warm_fe_link = nullptr;
    bool warm_free_ok = false, warm_link_ok = false;
    // interface state, device resident: multipliers (previous / current), G_FE P_ext,
    // the FE coupling velocities at the start of the macro step, the dense interface
    // (row-major H and its LU factor with the row permutation)
    double *lamp_d = nullptr, *gpfe_d = nullptr, *gprev_d = nullptr;
    double *h_d = nullptr, *hfe_dense = nullptr;  // dense mode: H and H_FE (row-major nl x nl)
    int* perm_d = nullptr;
    bool h_valid = false, unit_stale = false, use_dense = true;
    double t = 0.0;
    // per macro step results read back in one copy: CG {iterations, status} per solve
    // slot, energy sums, continuity maxima (double bits), the LU singularity flag
    enum { CG_FE_FREE = 0, CG_FE_LINK = 1, CG_IFACE = 2, CG_UNIT = 3, N_CG = 4 };
    int* cg_status = nullptr;                 // 2 ints per slot
    double* en_d = nullptr;                   // quad_fe, lambda_fe, lambda_pd
    unsigned long long* cmax_d = nullptr;     // |gf - gp|, |v_FE|, |v_PD|, LU amax
    int* lu_flag = nullptr;
    double *ta_d = nullptr, *tb_d = nullptr;  // energy term scratch, m nl each
    int64_t broken_total = 0;

    ~pmts_mts() {
        if (stream) cudaStreamSynchronize(stream);
        for (auto& g : cg_loop)
            if (g) cudaGraphExecDestroy(g);
        if (h_pin) cudaFreeHost(h_pin);
        for (void* p : owned) cudaFree(p);
        if (pd) pmts_pd_destroy(pd);
        if (stream) cudaStreamDestroy(stream);
        if (stream2) cudaStreamDestroy(stream2);
        for (cudaEvent_t e : {ev_fork, ev_join, ev_fork2, ev_join2})
            if (e) cudaEventDestroy(e);
    }
    template <class T>
    T* alloc(size_t n) {
        T* p = nullptr;
        CKM(cudaMalloc(&p, sizeof(T) * std::max<size_t>(n, 1)));
        owned.push_back(p);
        return p;
    }
    void release(void* p) {
        if (!p) return;
        owned.erase(std::remove(owned.begin(), owned.end(), p), owned.end());
        cudaFree(p);
    }
    template <class T>
    T* upload(const std::vector<T>& v) {
        T* p = alloc<T>(v.size());
        if (!v.empty()) CKM(cudaMemcpyAsync(p, v.data(), sizeof(T) * v.size(), cudaMemcpyHostToDevice, stream));
        return p;
    }
    DState state(int n) {
        DState st{alloc<double>(n), alloc<double>(n), alloc<double>(n)};
        zero(st, n);
        return st;
    }
    void zero(const DState& st, int n) {
        CKM(cudaMemsetAsync(st.u, 0, sizeof(double) * n, stream));
        CKM(cudaMemsetAsync(st.v, 0, sizeof(double) * n, stream));
        CKM(cudaMemsetAsync(st.a, 0, sizeof(double) * n, stream));
    }
    void copy(const DState& dst, const DState& src, int n) {
        CKM(cudaMemcpyAsync(dst.u, src.u, sizeof(double) * n, cudaMemcpyDeviceToDevice, stream));
        CKM(cudaMemcpyAsync(dst.v, src.v, sizeof(double) * n, cudaMemcpyDeviceToDevice, stream));
        CKM(cudaMemcpyAsync(dst.a, src.a, sizeof(double) * n, cudaMemcpyDeviceToDevice, stream));
    }
    std::vector<double> to_host(const double* d, int n) {
        std::vector<double> h(n);
        if (n) CKM(cudaMemcpyAsync(h.data(), d, sizeof(double) * n, cudaMemcpyDeviceToHost, stream));
        CKM(cudaStreamSynchronize(stream));
        return h;
    }
    void to_dev(double* d, const std::vector<double>& h) {
        if (!h.empty()) CKM(cudaMemcpyAsync(d, h.data(), sizeof(double) * h.size(), cudaMemcpyHostToDevice, stream));
    }
    double scalar(const double* d) {
        double v = 0.0;
        CKM(cudaMemcpyAsync(&v, d, sizeof(double), cudaMemcpyDeviceToHost, stream));
        CKM(cudaStreamSynchronize(stream));
        return v;
    }

    double load_scale(double tt) const {
        const double ramp = s.ramp;
        if (ramp <= 0.0) return 1.0;
        return std::clamp(tt / ramp, 0.0, 1.0);
    }
    double dt_fe() const { return m * s.dt_pd; }

    // ---- operators ----
    void fe_K(const double* x, double* y) { mtsk::csr_spmv(nf, fe_rp, fe_ci, fe_v, x, y, stream); }
    // K^PD x with the given bond mask; do_break: the inclusive stretch test on x
    // updates that mask (count into slot)
    // linear PD force (centroid form) on the entry-major families when built
    void force_lin(const double* x, const uint32_t* mask) {
        if (lin_lat && mask == mask_sync) mtsk::pd_force_lin_lat(pdv, lat, x, pd_ubar, stream);
        else if (famT_col) mtsk::pd_force_lin_t(pdv, famT_col, famT_coef, x, mask, pd_ubar, stream);
        else mtsk::pd_force_lin(pdv, x, mask, pd_ubar, stream);
    }
    // k_sync <- the live bond states (mts.hpp:98, 252), and its stencil-bit form
    void snapshot_bonds() {
        CKM(cudaMemcpyAsync(mask_sync, mask_live, sizeof(uint32_t) * mask_words,
                            cudaMemcpyDeviceToDevice, stream));
        if (lin_lat) mtsk::lin_lat_mask(pdv, lat, mask_sync, stream);
    }

    void pd_K(double* x, double* y, uint32_t* mask, bool do_break, int slot) {
        halo(x);  // sharded: the halo dofs of x from their owners
        mtsk::pd_force_warp(pdv, x, mask, do_break ? 1 : 0, d_counts + slot, stream, elem_q, elem_s, famT_col, famT_coef);
        launch_node_force(pdv, y, stream);
    }

    // reference cg_solve (linalg.hpp:243-296) on the device, the whole solve one graph
    // launch: the setup (b.b, r = b - A x, z, p, r.z, r.r), the loop test before the
    // first iteration (k_cg_start: b = 0 -> x = 0) and a conditional WHILE node whose
    // body is the iteration plus the loop test (k_cg_cond) -- no host round trip.  The
    // solve's {iterations, status} land in cg_status[slot]; cg_result reads them.  The
    // graph bakes in every pointer the iteration and the operator touch: it is rebuilt
    // when one of its inputs changes or the operator's buffers are reallocated
    // (invalidate_cg_graphs).
    // opdot(p, ap, s_pap, s_rz, s_alpha): the operator fused with p.Ap and alpha = rz / pAp;
    // returns false where the operator has no fused form (op, then the separate dot)
    template <class Op, class OpDot>
    void cg(int n, Op&& op, OpDot&& opdot, const double* b, double* x, double tol, int max_iter,
            const double* jac, int slot, bool host_loop = false) {
        if (host_loop) {
            cg_host(n, op, opdot, b, x, tol, max_iter, jac, slot);
            return;
        }
        double* r = cg_r;
        double* z = cg_z;
        double* p = cg_p;
        double* ap = cg_ap;
        double* sc = scal + 8 * slot;
        double *s_bb = sc + 0, *s_rz = sc + 1, *s_rr = sc + 2, *s_pap = sc + 3, *s_alpha = sc + 4,
               *s_rzn = sc + 5, *s_beta = sc + 6;
        int* st = cg_status + 2 * slot;
        // fused iteration: p.Ap and alpha in one launch, the update with the
        // preconditioner, r.z, r.r, beta and rz <- rz_new in one launch
        // (the update, r.z, r.r, beta and the loop test in one launch; the WHILE
        // condition is set there, the body ends with p = z + beta p)
        cudaGraphConditionalHandle hnd_body{};
        auto body = [&] {
            if (!opdot(p, ap, s_pap, s_rz, s_alpha)) {
                op(p, ap);
                mtsk::dot_fin(n, p, ap, nullptr, nullptr, part2, ticket, s_pap, nullptr, 1, s_rz,
                              s_alpha, stream);
            }
            mtsk::cg_update_dots(n, s_alpha, p, ap, x, r, jac, z, part2, ticket, s_rzn, s_rr, s_rz,
                                 s_beta, s_bb, s_pap, tol, max_iter, st, hnd_body, stream);
            mtsk::xpby(n, z, s_beta, p, stream);
        };
        cudaGraphExec_t& gl = cg_loop[slot];
        const CgKey key{x, b, jac, n, tol, max_iter, op_epoch};
        if (gl && !(cg_key[slot] == key)) {
            cudaGraphExecDestroy(gl);
            gl = nullptr;
        }
        if (!gl) {
            cudaGraph_t g;
            CKM(cudaGraphCreate(&g, 0));
            cudaGraphConditionalHandle hnd;
            CKM(cudaGraphConditionalHandleCreate(&hnd, g, 0, 0));
            CKM(cudaStreamBeginCaptureToGraph(stream, g, nullptr, nullptr, 0,
                                              cudaStreamCaptureModeThreadLocal));
            mtsk::dot(n, b, b, part, s_bb, stream);
            op(x, ap);
            sub(n, b, ap, r);  // r = b - A x
            mtsk::precond(n, r, jac, z, stream);
            CKM(cudaMemcpyAsync(p, z, sizeof(double) * n, cudaMemcpyDeviceToDevice, stream));
            mtsk::dot(n, r, z, part, s_rz, stream);
            mtsk::dot(n, r, r, part, s_rr, stream);
            mtsk::cg_start(hnd, s_bb, s_rr, tol, max_iter, st, x, n, stream);
            // the WHILE node behind the captured setup
            cudaStreamCaptureStatus cst;
            const cudaGraphNode_t* deps = nullptr;
            size_t nd = 0;
            CKM(cudaStreamGetCaptureInfo(stream, &cst, nullptr, nullptr, &deps, &nd));
            cudaGraphNodeParams cp = {};
            cp.type = cudaGraphNodeTypeConditional;
            cp.conditional.handle = hnd;
            cp.conditional.type = cudaGraphCondTypeWhile;
            cp.conditional.size = 1;
            cudaGraphNode_t node;
            CKM(cudaGraphAddNode(&node, g, deps, nd, &cp));
            CKM(cudaStreamUpdateCaptureDependencies(stream, &node, 1,
                                                    cudaStreamSetCaptureDependencies));
            CKM(cudaStreamEndCapture(stream, &g));
            cudaGraph_t bodyg = cp.conditional.phGraph_out[0];
            CKM(cudaStreamBeginCaptureToGraph(stream, bodyg, nullptr, nullptr, 0,
                                              cudaStreamCaptureModeThreadLocal));
            hnd_body = hnd;
            body();
            CKM(cudaStreamEndCapture(stream, &bodyg));
            CKM(cudaGraphInstantiate(&gl, g, 0));
            cudaGraphDestroy(g);
            cg_key[slot] = key;
        }
        cg_max[slot] = max_iter;
        CKM(cudaGraphLaunch(gl, stream));
    }
    // the same solve with the loop on the host (sharded coupled runs whose operator holds
    // collectives: each iteration's exchanges are host-synchronised in the in-process
    // group): the same kernels in the same order, the loop flag read back per iteration
    template <class Op, class OpDot>
    void cg_host(int n, Op&& op, OpDot&& opdot, const double* b, double* x, double tol,
                 int max_iter, const double* jac, int slot) {
        double *r = cg_r, *z = cg_z, *p = cg_p, *ap = cg_ap;
        double* sc = scal + 8 * slot;
        double *s_bb = sc + 0, *s_rz = sc + 1, *s_rr = sc + 2, *s_pap = sc + 3, *s_alpha = sc + 4,
               *s_rzn = sc + 5, *s_beta = sc + 6;
        int* st = cg_status + 2 * slot;
        mtsk::dot(n, b, b, part, s_bb, stream);
        op(x, ap);
        sub(n, b, ap, r);
        mtsk::precond(n, r, jac, z, stream);
        CKM(cudaMemcpyAsync(p, z, sizeof(double) * n, cudaMemcpyDeviceToDevice, stream));
        mtsk::dot(n, r, z, part, s_rz, stream);
        mtsk::dot(n, r, r, part, s_rr, stream);
        mtsk::cg_start(0, s_bb, s_rr, tol, max_iter, st, x, n, stream, more_d);
        cg_max[slot] = max_iter;
        auto more = [&] {
            CKM(cudaMemcpyAsync(more_h, more_d, sizeof(int), cudaMemcpyDeviceToHost, stream));
            CKM(cudaStreamSynchronize(stream));
            return *more_h != 0;
        };
        while (more()) {
            if (!opdot(p, ap, s_pap, s_rz, s_alpha)) {
                op(p, ap);
                mtsk::dot_fin(n, p, ap, nullptr, nullptr, part2, ticket, s_pap, nullptr, 1, s_rz,
                              s_alpha, stream);
            }
            mtsk::cg_update_dots(n, s_alpha, p, ap, x, r, jac, z, part2, ticket, s_rzn, s_rr, s_rz,
                                 s_beta, s_bb, s_pap, tol, max_iter, st, 0, stream, more_d);
            mtsk::xpby(n, z, s_beta, p, stream);
        }
    }
    // {iterations, status} of a finished solve (host copy h_stat after a readback)
    int cg_check(const int* hs, int slot) const {
        if (hs[2 * slot + 1] == 1) throw SolverError("cg: operator not positive definite");
        if (hs[2 * slot + 1] == 2)
            throw SolverError("cg: no convergence after " + std::to_string(cg_max[slot]) +
                              " iterations");
        return hs[2 * slot];
    }
    int cg_result(int slot) {  // reads back now
        int hs[2 * N_CG];
        CKM(cudaMemcpyAsync(hs, cg_status, sizeof(hs), cudaMemcpyDeviceToHost, stream));
        CKM(cudaStreamSynchronize(stream));
        return cg_check(hs, slot);
    }
    cudaGraphExec_t cg_loop[N_CG] = {nullptr, nullptr, nullptr, nullptr};
    int cg_max[N_CG] = {0, 0, 0, 0};
    struct CgKey {
        const double *x = nullptr, *b = nullptr, *jac = nullptr;
        int n = 0;
        double tol = 0.0;
        int max_iter = 0;
        unsigned epoch = 0;
        bool operator==(const CgKey& o) const {
            return x == o.x && b == o.b && jac == o.jac && n == o.n && tol == o.tol &&
                   max_iter == o.max_iter && epoch == o.epoch;
        }
    };
    CgKey cg_key[N_CG];
    unsigned op_epoch = 0;  // bumped whenever a buffer an operator captures is reallocated
    void invalidate_cg_graphs() { ++op_epoch; }
    void* h_pin = nullptr;  // pinned: the macro step's readback
    void sub(int n, const double* b, const double* ap, double* r) {
        // r = b - ap, elementwise, exactly as the reference's r[i] = b[i] - ap[i]
        mtsk::rhs(n, b, 1.0, ap, zero_flags(n), r, stream);
    }
    uint8_t* zf = nullptr;
    int zf_n = 0;
    const uint8_t* zero_flags(int n) {
        if (n > zf_n) {
            zf = alloc<uint8_t>(n);
            CKM(cudaMemsetAsync(zf, 0, n, stream));
            zf_n = n;
        }
        return zf;
    }

    // BlockOperator::solve (newmark.hpp:122-159) for the FE subdomain.  rhs.a =
    // ra * ra_scale (ra nullable); rv, rd the predictor rows.  Implicit: the CG's
    // status goes to cg_status[slot].
    void fe_solve(const double* ra, double ra_scale, const double* rvp, const double* rdp,
                  double* warm, bool* warm_ok, bool homog, const DState& out, int slot) {
        fe_K(rdp, kd);
        if (fe_nm.explicit_scheme()) {
            mtsk::explicit_solve(nf, ra, ra_scale, kd, fe_M, fe_cf, rvp, rdp, fe_nm.gdt, fe_nm.bdt2,
                                 fe_bcv, homog ? 1 : 0, out.u, out.v, out.a, stream);
            return;
        }
        mtsk::rhs(nf, ra, ra_scale, kd, fe_cf, cg_b, stream);
        if (warm && warm_ok && *warm_ok) {
            CKM(cudaMemcpyAsync(cg_x, warm, sizeof(double) * nf, cudaMemcpyDeviceToDevice, stream));
            mtsk::zero_constrained(nf, fe_cf, cg_x, stream);
        } else {
            CKM(cudaMemsetAsync(cg_x, 0, sizeof(double) * nf, stream));
        }
        const double bdt2 = fe_nm.bdt2;
        cg(nf,
           [&](const double* x, double* y) {  // M + bdt2 K in one pass
               mtsk::csr_apply_a(nf, fe_rp, fe_ci, fe_v, x, fe_M, fe_cf, bdt2, y, stream);
           },
           [&](const double* pp, double* y, double* s_pap, const double* s_rz, double* s_alpha) {
               mtsk::csr_apply_a_pap(nf, fe_rp, fe_ci, fe_v, pp, fe_M, fe_cf, bdt2, y, part3,
                                     ticket3, s_pap, s_rz, s_alpha, stream);
               return true;
           },
           cg_b, cg_x, cg_tol, fe_cg_max, fe_jac, slot);
        mtsk::zero_constrained(nf, fe_cf, cg_x, stream);
        if (warm) {
            CKM(cudaMemcpyAsync(warm, cg_x, sizeof(double) * nf, cudaMemcpyDeviceToDevice, stream));
            if (warm_ok) *warm_ok = true;
        }
        mtsk::finish(nf, cg_x, rvp, rdp, fe_nm.gdt, fe_nm.bdt2, fe_cf, fe_bcv, homog ? 1 : 0, out.u,
                     out.v, out.a, stream);
    }
    // explicit PD solve (beta_pd = 0); the bond test on rd when do_break
    void pd_solve(const double* ra, double ra_scale, const double* rvp, const double* rdp,
                  uint32_t* mask, bool do_break, int slot, bool homog, const DState& out) {
        if (do_break || !homog)  // free substeps: the deterministic per-entry arithmetic
            mtsk::pd_force_warp(pdv, rdp, mask, do_break ? 1 : 0, d_counts + slot, stream, elem_q, elem_s, famT_col, famT_coef);
        else  // homogeneous linear substeps (unit, link, interface): centroid form
            force_lin(rdp, mask);
        mtsk::pd_node_explicit(pdv, ra, ra_scale, pd_M, pd_cf, rvp, rdp, pd_nm.gdt, pd_nm.bdt2,
                               pd_bcv, homog ? 1 : 0, out.u, out.v, out.a, stream);
    }

    // ---- coupling (coupling.hpp:46-68), all on the device ----
    void gather_fe(const double* x, double* out) {
        mtsk::gather_csr(nl, gfe_rp, gfe_ci, gfe_w, x, out, stream);
    }
    // dst += G_FE^T (-vals): the reference's scatter of scaled(lambda, -1); tmp: nl scratch
    void add_gt_fe_neg(const double* vals, double* dst, double* tmp = nullptr) {
        if (!tmp) tmp = lam_tmp;
        mtsk::neg(nl, vals, tmp, stream);
        mtsk::scatter_csr(gft_n, gft_d, gft_rp, gft_ri, gft_w, tmp, dst, stream);
    }
    void zero_vec(double* x, int n) { CKM(cudaMemsetAsync(x, 0, sizeof(double) * n, stream)); }

    // ---- unit responses (mts.hpp:389-445) ----
    void unit_fe_column(int k, const DState& y) {
        // M_block Y = -G^T e_k, homogeneous, no warm start
        mtsk::unit_row(nf, gfe_rp, gfe_ci, gfe_w, k, ra, stream);
        zero_vec(rv, nf);
        zero_vec(rd, nf);
        fe_solve(ra, 1.0, rv, rd, nullptr, nullptr, true, y, CG_UNIT);
    }
    void unit_pd_column(int k, const DState& y) {
        // w = e_k: the ramped unit load at pd_dof[k] (mts.hpp:398-407)
        mtsk::unit_vec(nl, k, lam_tmp, stream);
        lin_substeps(lam_tmp, nullptr, nullptr, y);
    }
    // the m homogeneous linear substeps on k_sync (mts.hpp:230-238, 398-418):
    // y_0 = 0; per substep the centroid-form force (skipped on the first, from
    // rest) and one fused node kernel.  out_last: G_PD vel(y_m); out_rows: row j
    // = G_PD vel(y_j), j = 1..m
    void lin_substeps(const double* w_dev, double* out_last, double* out_rows, const DState& y) {
        zero_vec(rd, np);
        zero_vec(rv, np);
        if (sharded) {  // rows other shards own: -0.0, then the owner-sum
            if (out_last) mtsk::fill(nl, -0.0, out_last, stream);
            if (out_rows) mtsk::fill((long long)m * nl, -0.0, out_rows + nl, stream);
        }
        for (int j = 1; j <= m; ++j) {
            if (j > 1) {
                halo(rd);
                force_lin(rd, mask_sync);
            }
            double* out = out_rows ? out_rows + (size_t)j * nl : (j == m ? out_last : nullptr);
            mtsk::pd_node_lin(pdv, j > 1 ? 1 : 0, w_dev, row_of, double(j) / m, pd_M, pd_cf,
                              pd_nm.gdt, pd_nm.bdt2, pd_nm.dt, pd_nm.cpv, pd_nm.cpd, y.u, y.v, y.a,
                              rd, rv, out, stream);
        }
        if (sharded) {
            if (out_last) sum_owned(out_last, nl);
            if (out_rows) sum_owned(out_rows + nl, (size_t)m * nl);
        }
    }
    // H_FE = -G_FE vel(Y_FE) column by column on the device (mts.hpp:389-397): the
    // columns go into a column-major nl x nl scratch, from which the dense form (dense
    // interface) or the exact nonzeros in CSR (matrix-free interface: each unit column
    // is a CG solve whose support grows one stiffness neighbourhood per iteration, and
    // disconnected FE parts never couple -- lossless) are extracted on the device
    bool hfe_unit_columns = false;  // pmts_mts_desc.interface_h_fe = 1
    void build_h_fe() {
        if (fe_nm.explicit_scheme() && !use_dense && iface_mode != 1 && !hfe_unit_columns) {
            build_h_fe_explicit();
            if (interface_precond) {  // (the Jacobi option: from the CSR's diagonal)
                iface_jac = alloc<double>(nl);
                mtsk::iface_jac_csr(nl, hfe_rp, hfe_ci, hfe_v, m, s.dt_pd, cpd, pd_M, iface_jac,
                                    stream);
            }
            return;
        }
        // (the column-major scratch is n_lambda^2 doubles: refuse what cannot fit)
        {
            size_t free_b = 0, total_b = 0;
            CKM(cudaMemGetInfo(&free_b, &total_b));
            if (sizeof(double) * (size_t)nl * nl > free_b / 2)
                throw ConfigError("interface of " + std::to_string(nl) +
                                  " multipliers: the H_FE unit-column scratch (n_lambda^2 "
                                  "doubles) does not fit in device memory");
        }
        double* D = nullptr;
        CKM(cudaMallocAsync(&D, sizeof(double) * (size_t)nl * nl, stream));
        if (fe_nm.explicit_scheme()) {
            for (int k = 0; k < nl; ++k) {
                unit_fe_column(k, yst);
                gather_fe(yst.v, gvec);
                mtsk::col_neg(nl, k, gvec, D, stream);
            }
        } else {
            // implicit FE: the unit columns as batches of simultaneous CG solves (one
            // sparse-matrix read per iteration for the whole batch)
            const int B = std::min(nl, 64);
            double *scr = nullptr, *part = nullptr, *sc = nullptr;
            int *act = nullptr, *stat = nullptr, *nact = nullptr, *hcount = nullptr;
            CKM(cudaMallocAsync(&scr, sizeof(double) * 6 * (size_t)B * nf, stream));
            CKM(cudaMallocAsync(&part, sizeof(double) * 2 * mtsk::batched_partials() * (size_t)B,
                                stream));
            CKM(cudaMallocAsync(&sc, sizeof(double) * 8 * (size_t)B, stream));
            CKM(cudaMallocAsync(&act, sizeof(int) * (3 * (size_t)B + 1), stream));
            stat = act + B;
            nact = stat + 2 * B;
            CKM(cudaMallocHost(&hcount, sizeof(int)));
            for (int k0 = 0; k0 < nl; k0 += B) {
                int iters = 0;
                const int bad = mtsk::batched_unit_columns(
                    nf, nl, k0, B, fe_rp, fe_ci, fe_v, fe_M, fe_cf, fe_jac, fe_nm.bdt2, fe_nm.gdt,
                    gfe_rp, gfe_ci, gfe_w, cg_tol, fe_cg_max, scr, part, sc, act, stat, nact,
                    hcount, D, &iters, stream);
                if (bad == 1) throw SolverError("cg: operator not positive definite");
                if (bad == 2)
                    throw SolverError("cg: no convergence after " + std::to_string(fe_cg_max) +
                                      " iterations");
            }
            CKM(cudaFreeAsync(scr, stream));
            CKM(cudaFreeAsync(part, stream));
            CKM(cudaFreeAsync(sc, stream));
            CKM(cudaFreeAsync(act, stream));
            CKM(cudaStreamSynchronize(stream));
            cudaFreeHost(hcount);
        }
        if (use_dense || iface_mode == 1) {
            if (!hfe_dense) hfe_dense = alloc<double>((size_t)nl * nl);
            mtsk::transpose(nl, D, hfe_dense, stream);
        }
        if (!use_dense || iface_mode == 2) {
            // Jacobi preconditioner of the matrix-free interface CG (an addition: the
            // reference's CG is unpreconditioned, mts.hpp:194-213): diag(H_FE) plus the
            // free-mass velocity of a PD dof after the m ramped substeps, m dt / (2 M) --
            // the (1 - alpha)-weighted PD masses span orders of magnitude across the
            // gluing zone, which is what slows the plain CG
            if (interface_precond) {
                iface_jac = alloc<double>(nl);
                mtsk::iface_jac(nl, D, m, s.dt_pd, cpd, pd_M, iface_jac, stream);
            }
            int* cnt = nullptr;
            CKM(cudaMallocAsync(&cnt, sizeof(int) * ((size_t)nl + 1), stream));
            mtsk::row_nnz(nl, D, cnt, stream);
            std::vector<int> hc(nl + 1);
            CKM(cudaMemcpyAsync(hc.data(), cnt, sizeof(int) * ((size_t)nl + 1), cudaMemcpyDeviceToHost,
                                stream));
            CKM(cudaStreamSynchronize(stream));
            std::vector<int32_t> rp(nl + 1, 0);
            for (int r = 0; r < nl; ++r) rp[r + 1] = rp[r] + hc[r];
            hfe_nnz = rp[nl];
            hfe_rp = upload(rp);
            hfe_ci = alloc<int32_t>(std::max<int64_t>(hfe_nnz, 1));
            hfe_v = alloc<double>(std::max<int64_t>(hfe_nnz, 1));
            mtsk::row_fill(nl, D, hfe_rp, hfe_ci, hfe_v, stream);
            CKM(cudaFreeAsync(cnt, stream));
            invalidate_cg_graphs();  // the interface operator captures these
        }
        CKM(cudaFreeAsync(D, stream));
        CKM(cudaStreamSynchronize(stream));
    }
    // H_FE of an explicit FE side (M_block = the lumped mass) without unit columns: row r
    // couples to the rows k sharing an unconstrained FE dof with it, H_FE[r][k] =
    // -sum_j w_rj gdt (-w_kd) / M_d -- computed entry by entry exactly as the unit-column
    // construction rounds it (k_hfe_explicit), exact zeros dropped; no n_lambda^2 scratch
    // (BASELINE cfg5's 1.8M multipliers).  The candidate structure is host work in
    // parallel row chunks.
    void build_h_fe_explicit() {
        const std::vector<int32_t>& grp = s.cpl_fe_rp;
        const std::vector<int32_t>& gci = s.cpl_fe_ci;
        std::vector<uint8_t> cfh(nf, 0);
        for (int32_t d : s.fe_bc_dofs) cfh[d] = 1;
        std::vector<int64_t> drp(nf + 1, 0);  // unconstrained FE dof -> rows (ascending)
        for (int r = 0; r < nl; ++r)
            for (int j = grp[r]; j < grp[r + 1]; ++j)
                if (!cfh[gci[j]]) ++drp[gci[j] + 1];
        for (int d = 0; d < nf; ++d) drp[d + 1] += drp[d];
        std::vector<int32_t> dri(drp[nf]);
        {
            std::vector<int64_t> f(drp.begin(), drp.end() - 1);
            for (int r = 0; r < nl; ++r)
                for (int j = grp[r]; j < grp[r + 1]; ++j)
                    if (!cfh[gci[j]]) dri[f[gci[j]]++] = r;
        }
        const int nth = std::max(1u, std::min(64u, std::thread::hardware_concurrency()));
        auto rows_of = [&](int r, std::vector<int32_t>& out) {
            out.clear();
            for (int j = grp[r]; j < grp[r + 1]; ++j) {
                const int d = gci[j];
                if (cfh[d]) continue;
                out.insert(out.end(), dri.begin() + drp[d], dri.begin() + drp[d + 1]);
            }
            std::sort(out.begin(), out.end());
            out.erase(std::unique(out.begin(), out.end()), out.end());
        };
        auto parallel = [&](auto&& fn) {
            std::vector<std::thread> th;
            for (int t = 0; t < nth; ++t)
                th.emplace_back([&, t] {
                    std::vector<int32_t> tmp;
                    for (int r = int((long long)nl * t / nth); r < int((long long)nl * (t + 1) / nth); ++r)
                        fn(r, tmp);
                });
            for (auto& x : th) x.join();
        };
        std::vector<long long> crp(nl + 1, 0);
        parallel([&](int r, std::vector<int32_t>& tmp) {
            rows_of(r, tmp);
            crp[r + 1] = (long long)tmp.size();
        });
        for (int r = 0; r < nl; ++r) crp[r + 1] += crp[r];
        std::vector<int32_t> cci(crp[nl]);
        parallel([&](int r, std::vector<int32_t>& tmp) {
            rows_of(r, tmp);
            std::copy(tmp.begin(), tmp.end(), cci.begin() + crp[r]);
        });
        const long long nc = crp[nl];
        long long* d_crp = nullptr;
        int32_t* d_cci = nullptr;
        double* d_val = nullptr;
        int* cnt = nullptr;
        CKM(cudaMallocAsync(&d_crp, sizeof(long long) * (nl + 1), stream));
        CKM(cudaMallocAsync(&d_cci, sizeof(int32_t) * std::max(nc, 1LL), stream));
        CKM(cudaMallocAsync(&d_val, sizeof(double) * std::max(nc, 1LL), stream));
        CKM(cudaMallocAsync(&cnt, sizeof(int) * ((size_t)nl + 1), stream));
        CKM(cudaMemcpyAsync(d_crp, crp.data(), sizeof(long long) * (nl + 1), cudaMemcpyHostToDevice,
                            stream));
        if (nc)
            CKM(cudaMemcpyAsync(d_cci, cci.data(), sizeof(int32_t) * nc, cudaMemcpyHostToDevice,
                                stream));
        mtsk::hfe_explicit(nl, d_crp, d_cci, gfe_rp, gfe_ci, gfe_w, fe_M, fe_cf, fe_nm.gdt, d_val,
                           stream);
        mtsk::nz_count(nl, d_crp, d_val, cnt, stream);
        std::vector<int> hc(nl + 1);
        CKM(cudaMemcpyAsync(hc.data(), cnt, sizeof(int) * ((size_t)nl + 1), cudaMemcpyDeviceToHost,
                            stream));
        CKM(cudaStreamSynchronize(stream));
        std::vector<int32_t> rp(nl + 1, 0);
        long long tot = 0;
        for (int r = 0; r < nl; ++r) {
            tot += hc[r];
            if (tot > INT32_MAX) throw ConfigError("H_FE has more than 2^31 nonzeros");
            rp[r + 1] = int32_t(tot);
        }
        hfe_nnz = rp[nl];
        hfe_rp = upload(rp);
        hfe_ci = alloc<int32_t>(std::max<int64_t>(hfe_nnz, 1));
        hfe_v = alloc<double>(std::max<int64_t>(hfe_nnz, 1));
        mtsk::nz_fill(nl, d_crp, d_cci, d_val, hfe_rp, hfe_ci, hfe_v, stream);
        for (void* p : {(void*)d_crp, (void*)d_cci, (void*)d_val, (void*)cnt})
            CKM(cudaFreeAsync(p, stream));
        CKM(cudaStreamSynchronize(stream));
        invalidate_cg_graphs();
    }
    // H = H_FE + G_PD vel(Y_PD) (mts.hpp:422-445) and its LU factor, on the device
    void refresh_dense_interface() {
        if (!h_d) {
            h_d = alloc<double>((size_t)nl * nl);
            perm_d = alloc<int>(nl);
        }
        CKM(cudaMemcpyAsync(h_d, hfe_dense, sizeof(double) * (size_t)nl * nl,
                            cudaMemcpyDeviceToDevice, stream));
        for (int k = 0; k < nl; ++k) {
            unit_pd_column(k, yst);
            mtsk::add_col_gather(nl, k, cpd, yst.v, h_d, stream);
        }
        {
            std::vector<int> id(nl);
            for (int i = 0; i < nl; ++i) id[i] = i;
            CKM(cudaMemcpyAsync(perm_d, id.data(), sizeof(int) * nl, cudaMemcpyHostToDevice, stream));
        }
        CKM(cudaMemsetAsync(cmax_d + 3, 0, sizeof(unsigned long long), stream));
        CKM(cudaMemsetAsync(lu_flag, 0, sizeof(int), stream));
        mtsk::lu_factor(nl, h_d, perm_d, cmax_d + 3, lu_flag, stream);
        int flag = 0;
        CKM(cudaMemcpyAsync(&flag, lu_flag, sizeof(int), cudaMemcpyDeviceToHost, stream));
        CKM(cudaStreamSynchronize(stream));
        if (flag) throw SolverError("singular interface system: coincident or disconnected overlap");
        h_valid = true;
    }
    // G_PD vel(Y_PD_m) w without materialising Y (mts.hpp:410-420), device in/out
    void apply_h_pd(const double* w_dev, double* out_dev) {
        lin_substeps(w_dev, out_dev, nullptr, yst);
    }

    // ---- H_PD = G_PD vel(Y_PD) as an exact sparse matrix (matrix-free interface) ----
    // The m homogeneous linear substeps spread a unit load at a coupling dof by at most
    // delta + h_e per substep after the first (node -> incident element -> partner
    // within delta -> its nodes; h_e the element diameter), so column k's nonzeros lie
    // within R = (m - 1)(delta + h_e) of the load.  Columns whose loads are more than 2R
    // apart have disjoint supports and are computed together by ONE recursion (a
    // colouring of the coupling dofs): the responses superpose with exact zeros, so each
    // column is bitwise its single-load run (unit_pd_column).  Built once at setup;
    // when bonds break the k_sync snapshot changes and the interface goes back to the
    // matrix-free recursion (apply_h_pd).
    bool hpd_valid = false;
    int32_t *hpd_rp = nullptr, *hpd_ci = nullptr;
    double* hpd_v = nullptr;
    int64_t hpd_nnz = 0;
    int hpd_colours = 0;
    void build_h_pd() {
        const int dim = s.dim;
        std::vector<int> dof2node(s.pd_n_dof, -1);  // global PD dofs
        for (size_t nd = 0; nd < s.pd_node_dof.size(); ++nd)
            if (s.pd_node_dof[nd] >= 0)
                for (int c = 0; c < dim; ++c) dof2node[s.pd_node_dof[nd] + c] = (int)nd;
        std::vector<double> pos(3 * (size_t)nl);
        for (int r = 0; r < nl; ++r) {
            const int nd = dof2node[s.cpl_pd[r]];
            if (nd < 0) throw InternalError("coupling row without a PD node");
            for (int c = 0; c < 3; ++c) pos[3 * (size_t)r + c] = s.nodes[3 * (size_t)nd + c];
        }
        const int nn = dim == 2 ? 4 : 8;
        double he = 0.0;
        for (int e : s.pd_active)
            for (int a = 0; a < nn; ++a)
                for (int b = a + 1; b < nn; ++b) {
                    const double* p = &s.nodes[3 * (size_t)s.conn[(size_t)e * nn + a]];
                    const double* q = &s.nodes[3 * (size_t)s.conn[(size_t)e * nn + b]];
                    double d2 = 0.0;
                    for (int c = 0; c < 3; ++c) d2 += (p[c] - q[c]) * (p[c] - q[c]);
                    he = std::max(he, std::sqrt(d2));
                }
        // support radius of a column (a relative margin for the rounding of positions)
        const double R = (m - 1) * (s.delta + he) * (1.0 + 1e-9) + 1e-12 * he;
        const double cell = std::max(2.0 * R, 1e-12);
        auto key = [&](int r, int dx, int dy, int dz) {
            const long long i = (long long)std::floor(pos[3 * (size_t)r] / cell) + dx;
            const long long j = (long long)std::floor(pos[3 * (size_t)r + 1] / cell) + dy;
            const long long k = (long long)std::floor(pos[3 * (size_t)r + 2] / cell) + dz;
            return (i * 1000003LL + j) * 1000033LL + k;
        };
        std::unordered_map<long long, std::vector<int>> grid;
        for (int r = 0; r < nl; ++r) grid[key(r, 0, 0, 0)].push_back(r);
        auto dist2 = [&](int a, int b) {
            double d2 = 0.0;
            for (int c = 0; c < 3; ++c) {
                const double d = pos[3 * (size_t)a + c] - pos[3 * (size_t)b + c];
                d2 += d * d;
            }
            return d2;
        };
        const int dzr = dim == 3 ? 1 : 0;
        {   // a sampled estimate of the build: too large (BASELINE cfg5: ~1.8M multipliers,
            // R ~ 23 mm -> ~10^11 column entries) -> the recursion form from the start
            double s1 = 0.0, s2 = 0.0;
            const int ns = std::min(nl, 64);
            for (int q = 0; q < ns; ++q) {
                const int k = int((long long)q * nl / ns);
                for (int dz = -dzr; dz <= dzr; ++dz)
                    for (int dy = -1; dy <= 1; ++dy)
                        for (int dx = -1; dx <= 1; ++dx) {
                            auto it = grid.find(key(k, dx, dy, dz));
                            if (it == grid.end()) continue;
                            for (int r : it->second) {
                                const double d2 = dist2(k, r);
                                s1 += d2 <= R * R ? 1.0 : 0.0;
                                s2 += d2 < 4.0 * R * R ? 1.0 : 0.0;
                            }
                        }
            }
            if (ns && (s1 / ns * nl > 3e8 || s2 / ns * nl > 3e9)) {
                iface_precompute = false;  // (the m-substep recursion in every CG iteration)
                return;
            }
        }
        // rows within R of each source (the column structure) and within 2R (conflicts)
        std::vector<std::vector<int>> near(nl);  // rows within R, ascending
        std::vector<int> colour(nl, -1);
        std::vector<int> forbid;
        for (int k = 0; k < nl; ++k) {
            forbid.clear();
            for (int dz = -dzr; dz <= dzr; ++dz)
                for (int dy = -1; dy <= 1; ++dy)
                    for (int dx = -1; dx <= 1; ++dx) {
                        auto it = grid.find(key(k, dx, dy, dz));
                        if (it == grid.end()) continue;
                        for (int r : it->second) {
                            const double d2 = dist2(k, r);
                            if (d2 <= R * R) near[k].push_back(r);
                            if (d2 < 4.0 * R * R * (1.0 + 1e-9) && colour[r] >= 0)
                                forbid.push_back(colour[r]);
                        }
                    }
            std::sort(near[k].begin(), near[k].end());
            std::sort(forbid.begin(), forbid.end());
            int c = 0;
            for (int f : forbid) {
                if (f == c) ++c;
                else if (f > c) break;
            }
            colour[k] = c;
            hpd_colours = std::max(hpd_colours, c + 1);
        }
        // CSR by rows: row r holds the sources k with r in near[k], ascending k
        std::vector<int32_t> rp(nl + 1, 0);
        for (int k = 0; k < nl; ++k)
            for (int r : near[k]) ++rp[r + 1];
        for (int r = 0; r < nl; ++r) rp[r + 1] += rp[r];
        hpd_nnz = rp[nl];
        std::vector<int32_t> ci(hpd_nnz);
        std::vector<int64_t> slot_of;  // per (k, r in near[k]) in k order
        {
            std::vector<int32_t> fill(rp.begin(), rp.end() - 1);
            slot_of.reserve(hpd_nnz);
            for (int k = 0; k < nl; ++k)  // k ascending: each row's columns ascending
                for (int r : near[k]) {
                    ci[fill[r]] = k;
                    slot_of.push_back(fill[r]++);
                }
        }
        // per colour: its sources, and the (row, slot) pairs of its columns
        std::vector<int64_t> pstart(nl + 1, 0);
        for (int k = 0; k < nl; ++k) pstart[k + 1] = pstart[k] + (int64_t)near[k].size();
        std::vector<std::vector<int>> members(hpd_colours);
        for (int k = 0; k < nl; ++k) members[colour[k]].push_back(k);
        std::vector<int32_t> src_all, rows_all;
        std::vector<int64_t> slots_all;
        std::vector<int64_t> c_src(hpd_colours + 1, 0), c_pair(hpd_colours + 1, 0);
        rows_all.reserve(hpd_nnz);
        slots_all.reserve(hpd_nnz);
        for (int c = 0; c < hpd_colours; ++c) {
            for (int k : members[c]) {
                src_all.push_back(k);
                for (size_t q = 0; q < near[k].size(); ++q) {
                    rows_all.push_back(near[k][q]);
                    slots_all.push_back(slot_of[pstart[k] + q]);
                }
            }
            c_src[c + 1] = (int64_t)src_all.size();
            c_pair[c + 1] = (int64_t)rows_all.size();
        }
        hpd_rp = upload(rp);
        hpd_ci = upload(ci);
        hpd_v = alloc<double>(std::max<int64_t>(hpd_nnz, 1));
        CKM(cudaMemsetAsync(hpd_v, 0, sizeof(double) * std::max<int64_t>(hpd_nnz, 1), stream));
        int32_t* d_src = upload(src_all);
        int32_t* d_rows = upload(rows_all);
        int64_t* d_slots = upload(slots_all);
        for (int c = 0; c < hpd_colours; ++c) {
            zero_vec(lam_tmp, nl);
            mtsk::set_ones((int)(c_src[c + 1] - c_src[c]), d_src + c_src[c], lam_tmp, stream);
            lin_substeps(lam_tmp, nullptr, nullptr, yst);
            mtsk::gather(nl, cpd_g(), yst.v, gvec, stream);
            sum_owned(gvec, nl);
            mtsk::gather_slots((int)(c_pair[c + 1] - c_pair[c]), d_rows + c_pair[c],
                               d_slots + c_pair[c], gvec, hpd_v, stream);
        }
        // H = H_FE + H_PD as one CSR: one sparse read per interface iteration (the two
        // supports overlap, the union is little larger than H_PD alone); its exact
        // diagonal is the Jacobi preconditioner when one is asked for
        {
            int* cnt = nullptr;
            CKM(cudaMallocAsync(&cnt, sizeof(int) * ((size_t)nl + 1), stream));
            mtsk::merge_count(nl, hfe_rp, hfe_ci, hpd_rp, hpd_ci, cnt, stream);
            std::vector<int> hc(nl + 1);
            CKM(cudaMemcpyAsync(hc.data(), cnt, sizeof(int) * ((size_t)nl + 1),
                                cudaMemcpyDeviceToHost, stream));
            CKM(cudaStreamSynchronize(stream));
            std::vector<int32_t> hrp(nl + 1, 0);
            for (int r = 0; r < nl; ++r) hrp[r + 1] = hrp[r] + hc[r];
            h_nnz = hrp[nl];
            h_rp = upload(hrp);
            h_ci = alloc<int32_t>(std::max<int64_t>(h_nnz, 1));
            h_v = alloc<double>(std::max<int64_t>(h_nnz, 1));
            mtsk::merge_fill(nl, hfe_rp, hfe_ci, hfe_v, hpd_rp, hpd_ci, hpd_v, h_rp, h_ci, h_v,
                             stream);
            CKM(cudaFreeAsync(cnt, stream));
            if (interface_precond) {
                h_jac = alloc<double>(nl);
                mtsk::csr_diag(nl, h_rp, h_ci, h_v, h_jac, stream);
            }
        }
        CKM(cudaStreamSynchronize(stream));
        hpd_valid = true;
        invalidate_cg_graphs();
    }
    int32_t *h_rp = nullptr, *h_ci = nullptr;  // H = H_FE + H_PD (CSR)
    double *h_v = nullptr, *h_jac = nullptr;
    int64_t h_nnz = 0;

    void initialize_accelerations() {
        // FE: p = P_fe ls(t) + G_FE^T (-lambda_prev)
        if (root) {
            mtsk::scale(nf, fe_P, load_scale(t), ra, stream);
            add_gt_fe_neg(lamp_d, ra);
            fe_K(ufe.u, kd);
            mtsk::init_acc(nf, ra, kd, fe_M, fe_cf, ufe.a, stream);
        }
        mtsk::scale(np, pd_P, load_scale(t), ra, stream);
        mtsk::scatter_add(nl, cpd_g(), lamp_d, ra, stream);
        pd_K(upd.u, kd, mask_live, false, 0);
        mtsk::init_acc(np, ra, kd, pd_M, pd_cf, upd.a, stream);
        CKM(cudaStreamSynchronize(stream));
    }

    // the interface solve (mts.hpp:184-215) into lam_d: rhs = G_FE v_FE - G_PD v_PD on
    // the device; the dense LU solve, or the matrix-free CG warm-started from
    // lambda_prev (its status read here: a failed CG falls back to the dense form)
    void interface_solve(int* iterations) {
        double* b = alloc_iface_b();
        if (!sharded) {
            gather_fe(vfe.v, b);
            mtsk::sub_idx(nl, cpd, vpd.v, b, stream);
        } else {  // G_FE v from shard 0; G_PD v = the free substeps' last row (owner-summed)
            if (root) gather_fe(vfe.v, b);
            cm().bcast(*this, b, sizeof(double) * nl);
            mtsk::sub_idx(nl, ident, gp_free_d + (size_t)m * nl, b, stream);
        }
        if (use_dense) {
            if (!h_valid) throw InternalError("interface solve with stale unit response");
            *iterations = 0;
            mtsk::lu_solve(nl, h_d, perm_d, b, lam_d, stream);
            return;
        }
        CKM(cudaMemcpyAsync(lam_d, lamp_d, sizeof(double) * nl, cudaMemcpyDeviceToDevice, stream));
        const int max_iter = std::max(200, 10 * int(std::sqrt(double(nl))));
        if (hpd_valid)  // H = H_FE + H_PD precomputed (exact sparse): one SpMV
            cg(nl,
               [&](const double* in, double* out) {
                   mtsk::csr_spmv_warp(nl, h_rp, h_ci, h_v, in, out, stream);
               },
               [&](const double* pp, double* y, double* s_pap, const double* s_rz, double* s_alpha) {
                   mtsk::csr_warp_pap(nl, h_rp, h_ci, h_v, pp, y, part3, ticket3, s_pap, s_rz,
                                      s_alpha, stream);
                   return true;
               },
               b, lam_d, interface_cg_tol, max_iter, h_jac ? h_jac : iface_jac, CG_IFACE);
        else  // H_FE w next to the m-substep recursion on the current k_sync
            cg(nl,
               [&](const double* in, double* out) {
                   fork(ev_fork2);
                   {
                       OnStream2 on(this);
                       mtsk::csr_spmv_warp(nl, hfe_rp, hfe_ci, hfe_v, in, out, stream);
                   }
                   apply_h_pd(in, iface_tmp);
                   join(ev_join2);
                   mtsk::add(nl, iface_tmp, out, stream);  // out[r] += gpw[r]
               },
               [](const double*, double*, double*, const double*, double*) { return false; },
               b, lam_d, interface_cg_tol, max_iter, iface_jac, CG_IFACE, sharded);
        try {
            *iterations = cg_result(CG_IFACE);
        } catch (const SolverError&) {
            if (sharded) throw;  // (no dense fallback across shards)
            use_dense = true;
            h_valid = false;
            if (!hfe_dense) {  // dense H_FE from the CSR (fallback only)
                std::vector<int32_t> rp(nl + 1);
                CKM(cudaMemcpy(rp.data(), hfe_rp, sizeof(int32_t) * (nl + 1), cudaMemcpyDeviceToHost));
                std::vector<int32_t> ci(hfe_nnz);
                std::vector<double> v(hfe_nnz), dense((size_t)nl * nl, 0.0);
                CKM(cudaMemcpy(ci.data(), hfe_ci, sizeof(int32_t) * hfe_nnz, cudaMemcpyDeviceToHost));
                CKM(cudaMemcpy(v.data(), hfe_v, sizeof(double) * hfe_nnz, cudaMemcpyDeviceToHost));
                for (int r = 0; r < nl; ++r)
                    for (int q = rp[r]; q < rp[r + 1]; ++q) dense[(size_t)r * nl + ci[q]] = v[q];
                hfe_dense = upload(dense);
            }
            refresh_dense_interface();
            *iterations = 0;
            mtsk::lu_solve(nl, h_d, perm_d, b, lam_d, stream);
        }
    }
    double* iface_b = nullptr;
    double* iface_tmp = nullptr;
    double* alloc_iface_b() {
        if (!iface_b) {
            iface_b = alloc<double>(nl);
            iface_tmp = alloc<double>(nl);
        }
        return iface_b;
    }

    pmts_mts_report macro_step();

    // collective setup of a sharded run (every shard, once, before the first step):
    // H_FE from shard 0 to every shard, H_PD by coloured recursions across the shards
    void shard_setup() {
        if (!root) hfe_rp = alloc<int32_t>(nl + 1);
        cm().bcast(*this, hfe_rp, sizeof(int32_t) * (nl + 1));
        int32_t nnz = 0;
        CKM(cudaMemcpyAsync(&nnz, hfe_rp + nl, sizeof(int32_t), cudaMemcpyDeviceToHost, stream));
        CKM(cudaStreamSynchronize(stream));
        if (!root) {
            hfe_nnz = nnz;
            hfe_ci = alloc<int32_t>(std::max<int64_t>(nnz, 1));
            hfe_v = alloc<double>(std::max<int64_t>(nnz, 1));
        }
        if (nnz) {
            cm().bcast(*this, hfe_ci, sizeof(int32_t) * (size_t)nnz);
            cm().bcast(*this, hfe_v, sizeof(double) * (size_t)nnz);
        }
        invalidate_cg_graphs();
        if (iface_precompute) build_h_pd();
        setup_done = true;
    }
};

namespace {

// FE side BlockOperator diagonal (refresh_diagonal, newmark.hpp:99-104)
std::vector<double> jacobi_diag(const MtsSystem& s, double bdt2) {
    std::vector<double> d(s.fe_n_dof, 0.0);
    if (bdt2 != 0.0)
        for (int i = 0; i < s.fe_n_dof; ++i)
            for (int p = s.fe_rowptr[i]; p < s.fe_rowptr[i + 1]; ++p)
                if (s.fe_col[p] == i) {
                    d[i] = s.fe_val[p];
                    break;
                }
    for (int i = 0; i < s.fe_n_dof; ++i) d[i] = s.fe_mass[i] + bdt2 * d[i];
    return d;
}

}  // namespace

pmts_mts_report pmts_mts::macro_step() {
    pmts_mts_report rep{};
    if (sharded && !setup_done) throw ConfigError("sharded coupled handle: pmts_mts_init first");
    // snapshot_previous (mts.hpp:507-510)
    if (root) {
        CKM(cudaMemcpyAsync(fe_prev.a, ufe.a, sizeof(double) * nf, cudaMemcpyDeviceToDevice,
                            stream));
        gather_fe(ufe.v, gprev_d);
    }
    // unit-response upkeep (mts.hpp:249-260)
    {
        const double t0 = now_s();
        if (unit_stale) {
            snapshot_bonds();
            h_valid = false;
            if (hpd_valid) {  // k_sync changed: the recursion from here on
                hpd_valid = false;
                invalidate_cg_graphs();
            }
            unit_stale = false;
            if (use_dense) refresh_dense_interface();
        }
        rep.t_unit = now_s() - t0;
    }
    if (counts_cap < m + 1) {
        d_counts = alloc<unsigned long long>(m + 1);
        counts_cap = m + 1;
    }
    CKM(cudaMemsetAsync(d_counts, 0, sizeof(unsigned long long) * (m + 1), stream));
    // free FE solve (mts.hpp:143-147)
    const double tk0 = now_s();
    if (root) {  // the FE half on stream2, the PD half on stream
        fork(ev_fork);
        OnStream2 on(this);
        mtsk::predict(nf, ufe.u, ufe.v, ufe.a, rd_fe, rv_fe, fe_nm.dt, fe_nm.cpv, fe_nm.cpd, stream);
        fe_solve(fe_P, load_scale(t + dt_fe()), rv_fe, rd_fe, warm_fe_free, &warm_free_ok, false,
                 vfe, CG_FE_FREE);
    }
    // free PD solve, m substeps with the multiplier loads S_j (mts.hpp:152-180), the S_j
    // rows formed on the device
    mtsk::s_vectors(nl, m, t, s.dt_pd, dt_fe(), s.ramp, lamp_d, gpfe_d, sv_d, stream);
    mtsk::gather(nl, cpd_g(), upd.v, gp_free_d, stream);
    copy(vpd, upd, np);
    for (int j = 1; j <= m; ++j) {
        mtsk::predict(np, vpd.u, vpd.v, vpd.a, rd, rv, pd_nm.dt, pd_nm.cpv, pd_nm.cpd, stream);
        halo(rd);  // sharded: one-horizon ghosts, every fine substep
        mtsk::scale(np, pd_P, load_scale(t + j * s.dt_pd), ra, stream);
        mtsk::scatter_add(nl, cpd_g(), sv_d + (size_t)(j - 1) * nl, ra, stream);
        pd_solve(ra, 1.0, rv, rd, mask_live, fracture, j, false, vpd);
        mtsk::gather(nl, cpd_g(), vpd.v, gp_free_d + (size_t)j * nl, stream);
    }
    sum_owned(gp_free_d, (size_t)(m + 1) * nl);  // G_PD v rows of every shard's owned rows
    if (root) join(ev_join);
    rep.t_kinematic = now_s() - tk0;  // enqueue time (the work is asynchronous)
    // interface solve + recombination (mts.hpp:184-241)
    const double tl0 = now_s();
    int iters = 0;
    interface_solve(&iters);
    rep.interface_iterations = iters;
    if (root) {  // FE correction: M_block W = -G^T lambda (stream2)
        fork(ev_fork);
        OnStream2 on(this);
        zero_vec(ra_fe, nf);
        zero_vec(rv_fe, nf);
        zero_vec(rd_fe, nf);
        add_gt_fe_neg(lam_d, ra_fe, lam_tmp_fe);
        fe_solve(ra_fe, 1.0, rv_fe, rd_fe, warm_fe_link, &warm_link_ok, true, wst_fe, CG_FE_LINK);
        mtsk::add_states(nf, vfe.u, vfe.v, vfe.a, wst_fe.u, wst_fe.v, wst_fe.a, ufe.u, ufe.v, ufe.a,
                         stream);
    }
    {  // PD correction: m substeps under the ramped multiplier load, on k_sync
        zero_vec(gp_link_d, nl);
        lin_substeps(lam_d, nullptr, gp_link_d, wst);
        mtsk::add_states(np, vpd.u, vpd.v, vpd.a, wst.u, wst.v, wst.a, upd.u, upd.v, upd.a, stream);
    }
    if (root) join(ev_join);
    rep.t_lambda = now_s() - tl0;
    // bonds broken in the free substeps, then the post-recombination audit
    const double tu0 = now_s();
    if (fracture) pd_K(upd.u, kd, mask_live, true, 0);  // slot 0: the audit
    rep.t_update = now_s() - tu0;
    // energy record (mts.hpp:447-504) and continuity residual (mts.hpp:309-317), reduced
    // on the device; everything the host needs comes back in one copy
    CKM(cudaMemsetAsync(cmax_d, 0, 3 * sizeof(unsigned long long), stream));
    CKM(cudaMemsetAsync(en_d, 0, 3 * sizeof(double), stream));
    if (track_energy && root) {
        if (fe_nm.gamma != 0.5) {
            double* da = cg_kx;  // scratch, nf
            mtsk::rhs(nf, ufe.a, 1.0, fe_prev.a, zero_flags(nf), da, stream);  // da = acc - prev
            fe_K(da, cg_ap);
            const double f = fe_nm.dt * fe_nm.dt * (fe_nm.beta - fe_nm.gamma / 2.0);
            mtsk::quad_w(nf, da, fe_M, f, cg_ap, cg_r, stream);
            mtsk::dot(nf, da, cg_r, part, en_d + 0, stream);
        }
        gather_fe(ufe.v, gvec);
        mtsk::sub2(nl, gvec, gprev_d, ta_d, stream);
        mtsk::sub2(nl, lam_d, lamp_d, tb_d, stream);
        mtsk::dot(nl, ta_d, tb_d, part, en_d + 1, stream);
        mtsk::lpd_terms(nl, m, gp_free_d, gp_link_d, sv_d, lamp_d, lam_d, ta_d, tb_d, stream);
        mtsk::dot(nl * m, ta_d, tb_d, part, en_d + 2, stream);
    }
    if (!sharded) {
        gather_fe(ufe.v, gvec);
        mtsk::max_abs(nl, gvec, cpd, upd.v, cmax_d + 0, stream);
        mtsk::max_abs(nf, ufe.v, nullptr, nullptr, cmax_d + 1, stream);
        mtsk::max_abs(np, upd.v, nullptr, nullptr, cmax_d + 2, stream);
    } else {  // the same maxima from owner-summed rows / owned dofs; one verdict everywhere
        mtsk::gather(nl, cpd_own, upd.v, gpd_now, stream);
        sum_owned(gpd_now, nl);
        if (root) {
            gather_fe(ufe.v, gvec);
            mtsk::max_abs(nl, gvec, ident, gpd_now, cmax_d + 0, stream);
            mtsk::max_abs(nf, ufe.v, nullptr, nullptr, cmax_d + 1, stream);
        }
        mtsk::max_abs(n_own_dofs, own_zero, own_dofs, upd.v, cmax_d + 2, stream);
        cm().reduce_u64(*this, cmax_d + 2, 1, true);
        cm().bcast(*this, cmax_d, 2 * sizeof(unsigned long long));
        cm().reduce_u64(*this, d_counts, m + 1, false);
        cm().bcast(*this, cg_status, sizeof(int) * 2 * N_CG);
    }
    // lambda_prev <- lambda
    CKM(cudaMemcpyAsync(lamp_d, lam_d, sizeof(double) * nl, cudaMemcpyDeviceToDevice, stream));
    struct Back {
        int st[2 * N_CG];
        double en[3];
        unsigned long long cmax[3];
        unsigned long long cnt[64];
    };
    static_assert(sizeof(Back) <= 1024, "pinned readback buffer");
    Back* hb = reinterpret_cast<Back*>(h_pin);
    CKM(cudaMemcpyAsync(hb->st, cg_status, sizeof(hb->st), cudaMemcpyDeviceToHost, stream));
    CKM(cudaMemcpyAsync(hb->en, en_d, sizeof(hb->en), cudaMemcpyDeviceToHost, stream));
    CKM(cudaMemcpyAsync(hb->cmax, cmax_d, sizeof(hb->cmax), cudaMemcpyDeviceToHost, stream));
    const int nc = std::min(m + 1, 64);
    CKM(cudaMemcpyAsync(hb->cnt, d_counts, sizeof(unsigned long long) * nc, cudaMemcpyDeviceToHost,
                        stream));
    CKM(cudaStreamSynchronize(stream));
    if (!fe_nm.explicit_scheme()) {
        cg_check(hb->st, CG_FE_FREE);
        cg_check(hb->st, CG_FE_LINK);
    }
    if (fracture) {
        long long nb = 0;
        for (int q = 0; q < nc; ++q) nb += (long long)hb->cnt[q];
        if (m + 1 > 64) {  // (not met by the configurations: m <= 63)
            std::vector<unsigned long long> c(m + 1);
            CKM(cudaMemcpy(c.data(), d_counts, sizeof(unsigned long long) * (m + 1),
                           cudaMemcpyDeviceToHost));
            nb = 0;
            for (auto x : c) nb += (long long)x;
        }
        if (nb > 0) unit_stale = true;
        rep.newly_broken = (int32_t)nb;
        broken_total += nb;
    }
    if (track_energy) {
        if (fe_nm.gamma != 0.5) rep.quad_fe = -(fe_nm.gamma - 0.5) * hb->en[0];
        rep.lambda_fe = hb->en[1] / dt_fe();
        rep.lambda_pd = -hb->en[2] / s.dt_pd;
    }
    {
        double mx[3];
        for (int q = 0; q < 3; ++q) std::memcpy(&mx[q], &hb->cmax[q], sizeof(double));
        rep.continuity = mx[0] / std::max(1.0, std::max(mx[1], mx[2]));
        if (enforce_continuity && rep.continuity > continuity_tol)
            throw SolverError("velocity continuity violated: residual " +
                              std::to_string(rep.continuity) + " at t=" +
                              std::to_string(t + dt_fe()));
    }
    t += dt_fe();
    return rep;
}

namespace {

// a lattice without loads (tractions stay surface loads here) over [lo, hi]
pmts_scenario* mts_lattice(const pmts_scenario_desc& sd, const double* lo, const double* hi,
                           double spacing) {
    pmts_scenario_desc g = sd;
    g.n_traction = 0;
    g.n_body_patch = 0;
    g.n_velocity_bc = 0;
    g.n_fixed = 0;
    for (int k = 0; k < 3; ++k) {
        g.lo[k] = lo[k];
        g.hi[k] = hi[k];
    }
    g.spacing = spacing;
    pmts_scenario* sc = nullptr;
    check_pd(pmts_scenario_build(&g, &sc));
    return sc;
}

void build_host(pmts_mts& h, const pmts_mts_desc& d) {
    const pmts_scenario_desc& sd = *d.scenario;
    MtsSystem& s = h.s;
    // mesh + geometry + material: the pure-PD scenario builder's generator
    if (sd.dim != 2 && sd.dim != 3) throw ConfigError("mesh dimension must be 2 or 3");
    s.dim = sd.dim;
    const int nn = sd.dim == 2 ? 4 : 8;
    if (d.fe_spacing > 0.0) {
        // non-matching meshes (extension): the FE lattice over the domain, the PD
        // lattice (the scenario spacing, which sets delta) over the PD boxes' hull
        const double ratio = d.fe_spacing / sd.spacing;
        const int r = int(std::lround(ratio));
        if (r < 1 || std::abs(ratio - r) > 1e-9 * ratio)
            throw ConfigError("fe_spacing must be an integer multiple of the PD spacing");
        double hlo[3] = {0, 0, 0}, hhi[3] = {0, 0, 0};
        for (int k = 0; k < sd.dim; ++k) {
            hlo[k] = 1e300;
            hhi[k] = -1e300;
            for (int b = 0; b < d.n_pd_box; ++b) {
                hlo[k] = std::min(hlo[k], std::max(sd.lo[k], d.pd_boxes[6 * b + k]));
                hhi[k] = std::min(sd.hi[k], std::max(hhi[k], d.pd_boxes[6 * b + 3 + k]));
            }
            for (double x : {hlo[k], hhi[k]}) {
                const double c = (x - sd.lo[k]) / d.fe_spacing;
                if (std::abs(c - std::round(c)) > 1e-9 * std::max(1.0, c))
                    throw ConfigError("non-matching coupling: the PD boxes' hull must lie on "
                                      "FE lattice lines");
            }
        }
        pmts_scenario* fe = mts_lattice(sd, sd.lo, sd.hi, d.fe_spacing);
        pmts_scenario* pd = mts_lattice(sd, hlo, hhi, sd.spacing);
        pmts_scenario_view vf{}, vp{};
        pmts_scenario_get(fe, &vf);
        pmts_scenario_get(pd, &vp);
        for (int k = 0; k < 3; ++k) {
            s.n[k] = vp.lattice[k];
            s.fe_n[k] = vf.lattice[k];
            s.pd_n[k] = vp.lattice[k];
            s.fe_lo[k] = sd.lo[k];
            s.pd_lo[k] = hlo[k];
        }
        s.fe_h = d.fe_spacing;
        s.pd_h = sd.spacing;
        s.fe_ratio = r;
        s.fe_mesh_elems = vf.n_elems;
        s.fe_mesh_nodes = vf.n_nodes;
        s.nodes.assign(vf.node_xyz, vf.node_xyz + 3 * (size_t)vf.n_nodes);
        // PD nodes on the global PD lattice: lo + (offset + i) h, bitwise the nodes
        // a conforming mesh of the PD spacing has there
        const int pnx = vp.lattice[0] + 1, pny = vp.lattice[1] + 1;
        long long off[3] = {0, 0, 0};
        for (int k = 0; k < sd.dim; ++k) off[k] = std::llround((hlo[k] - sd.lo[k]) / sd.spacing);
        std::vector<double> pxyz(3 * (size_t)vp.n_nodes);
        for (int q = 0; q < vp.n_nodes; ++q) {
            const long long ix[3] = {q % pnx, (q / pnx) % pny, q / ((long long)pnx * pny)};
            for (int k = 0; k < 3; ++k)
                pxyz[3 * (size_t)q + k] = k < sd.dim ? sd.lo[k] + (off[k] + ix[k]) * sd.spacing : 0.0;
        }
        std::vector<double> pcen(3 * (size_t)vp.n_elems), pvol(vp.n_elems);
        element_geometry(sd.dim, vp.n_elems, vp.elem_nodes, pxyz.data(), pcen.data(), pvol.data());
        s.nodes.insert(s.nodes.end(), pxyz.begin(), pxyz.end());
        s.conn.assign(vf.elem_nodes, vf.elem_nodes + (size_t)nn * vf.n_elems);
        for (size_t q = 0; q < (size_t)nn * vp.n_elems; ++q)
            s.conn.push_back(vp.elem_nodes[q] + vf.n_nodes);
        s.centroid.assign(vf.centroid, vf.centroid + 3 * (size_t)vf.n_elems);
        s.centroid.insert(s.centroid.end(), pcen.begin(), pcen.end());
        s.volume.assign(vf.volume, vf.volume + vf.n_elems);
        s.volume.insert(s.volume.end(), pvol.begin(), pvol.end());
        // the horizon and the overlap width follow the PD lattice: the char length a
        // conforming mesh of the PD spacing over the domain has (build_scenario,
        // driver.hpp:179-186), so a unit ratio rebuilds the reference's model bitwise
        int nfull[3] = {1, 1, 1};
        for (int k = 0; k < sd.dim; ++k)
            nfull[k] = int(std::lround((sd.hi[k] - sd.lo[k]) / sd.spacing));
        s.cl = lattice_char_length(sd.dim, nfull, sd.lo, sd.spacing, sd.host_setup != 0);
        s.delta = sd.delta_factor * s.cl;
        s.l = s.delta / sd.l_factor;
        s.c0 = calibrate_c0(sd.E, s.delta, s.l, sd.formulation);
        s.ramp = vp.load_ramp;
        for (int k = 0; k < 3; ++k) s.pd_lo[k] = k < sd.dim ? sd.lo[k] + off[k] * sd.spacing : 0.0;
        pmts_scenario_destroy(fe);
        pmts_scenario_destroy(pd);
    } else {
        pmts_scenario* sc = mts_lattice(sd, sd.lo, sd.hi, sd.spacing);
        pmts_scenario_view v{};
        pmts_scenario_get(sc, &v);
        for (int k = 0; k < 3; ++k) s.n[k] = v.lattice[k];
        s.nodes.assign(v.node_xyz, v.node_xyz + 3 * (size_t)v.n_nodes);
        s.conn.assign(v.elem_nodes, v.elem_nodes + (size_t)nn * v.n_elems);
        s.centroid.assign(v.centroid, v.centroid + 3 * (size_t)v.n_elems);
        s.volume.assign(v.volume, v.volume + v.n_elems);
        s.cl = v.char_length;
        s.delta = v.delta;
        s.l = v.l;
        s.c0 = v.c0;
        s.ramp = v.load_ramp;
        pmts_scenario_destroy(sc);
    }
    s.s_crit = sd.s_crit;
    s.E = sd.E;
    s.nu = sd.nu;
    s.rho = sd.rho;
    s.formulation = sd.formulation;
    for (int p = 0; p < sd.n_traction; ++p) {
        MtsTraction t;
        for (int k = 0; k < 3; ++k) {
            t.box.lo[k] = sd.traction[9 * p + k];
            t.box.hi[k] = sd.traction[9 * p + 3 + k];
            t.value[k] = sd.traction[9 * p + 6 + k];
        }
        s.tractions.push_back(t);
    }
    for (int p = 0; p < sd.n_body_patch; ++p) {
        MtsTraction t;
        for (int k = 0; k < 3; ++k) {
            t.box.lo[k] = sd.body_patch[9 * p + k];
            t.box.hi[k] = sd.body_patch[9 * p + 3 + k];
            t.value[k] = sd.body_patch[9 * p + 6 + k];
        }
        s.body_patches.push_back(t);
    }
    for (int k = 0; k < 3; ++k) s.body_force[k] = sd.body_force[k];
    for (int b = 0; b < sd.n_velocity_bc; ++b) {
        MtsKinematic kb;
        for (int k = 0; k < 3; ++k) {
            kb.box.lo[k] = sd.velocity_bc[8 * b + k];
            kb.box.hi[k] = sd.velocity_bc[8 * b + 3 + k];
        }
        kb.comp = int(sd.velocity_bc[8 * b + 6]);
        kb.vel = sd.velocity_bc[8 * b + 7];
        if (kb.comp < 0 || kb.comp >= s.dim) throw ConfigError("velocity_bc component out of range");
        s.kinematic.push_back(kb);
    }
    for (int b = 0; b < sd.n_fixed; ++b) {
        MtsKinematic kb;
        for (int k = 0; k < 3; ++k) {
            kb.box.lo[k] = sd.fixed[6 * b + k];
            kb.box.hi[k] = sd.fixed[6 * b + 3 + k];
        }
        kb.fix_all = true;
        s.kinematic.push_back(kb);
    }
    for (int b = 0; b < d.n_pd_box; ++b) {
        MtsBox box;
        for (int k = 0; k < 3; ++k) {
            box.lo[k] = d.pd_boxes[6 * b + k];
            box.hi[k] = d.pd_boxes[6 * b + 3 + k];
        }
        s.pd_boxes.push_back(box);
    }
    s.overlap_width_factor = d.overlap_width_factor;
    s.weight_kind = d.weight_kind;
    s.dt_pd = sd.dt_pd;
    s.m = sd.m;
    if (s.m < 1) throw ConfigError("time.m must be >= 1");
    const double steps = sd.total_time / (s.m * s.dt_pd);
    if (std::abs(steps - std::round(steps)) > 1e-6)
        throw ConfigError("time.total_time must be a multiple of m * dt_pd");
    s.n_macro = int(std::llround(sd.total_time / (s.m * s.dt_pd)));
    s.fe_gamma = d.gamma_fe;
    s.fe_beta = d.beta_fe;
    s.pd_gamma = sd.gamma;
    s.pd_beta = sd.beta;
    build_mts_system(s);
}

// ---- transports of the sharded coupled step ----

// in-process group: one host thread per shard (pmts_mts_group_*), host barriers, device
// copies between the shards' buffers (same device, or peers with P2P access)
struct ShardGroup {
    std::vector<pmts_mts*> h;
    std::mutex mu;
    std::condition_variable cv;
    int arrived = 0;
    long long gen = 0;
    bool aborted = false;
    int first_error = -1;
    std::vector<void*> slot;
    void wait() {
        std::unique_lock<std::mutex> lk(mu);
        if (aborted) throw InternalError("shard group aborted");
        const long long g0 = gen;
        if (++arrived == int(h.size())) {
            arrived = 0;
            ++gen;
            cv.notify_all();
            return;
        }
        cv.wait(lk, [&] { return gen != g0 || aborted; });
        if (aborted) throw InternalError("shard group aborted");
    }
    void abort(int rank) {
        std::lock_guard<std::mutex> lk(mu);
        if (first_error < 0) first_error = rank;
        aborted = true;
        cv.notify_all();
    }
};

struct GroupComm : MtsComm {
    std::shared_ptr<ShardGroup> g;
    int rank = 0;
    void publish(pmts_mts& h, void* x) {
        CKM(cudaStreamSynchronize(h.stream));
        g->slot[rank] = x;
        g->wait();
    }
    void done(pmts_mts& h) {  // nobody reads or rewrites a published buffer before all copied
        CKM(cudaStreamSynchronize(h.stream));
        g->wait();
    }
    void halo(pmts_mts& h, double* x) override {
        publish(h, x);
        for (const auto& l : h.links) {
            const pmts_mts* q = g->h[l.peer];
            const pmts_mts::LinkDev* ql = nullptr;
            for (const auto& k : q->links)
                if (k.peer == rank) ql = &k;
            if (!ql || ql->n_send != l.n_recv) throw InternalError("shard link mismatch");
            mtsk::copy_idx(l.n_recv, static_cast<const double*>(g->slot[l.peer]), ql->send, x,
                           l.recv, h.stream);
        }
        done(h);
    }
    void sum_owned(pmts_mts& h, double* x, size_t n) override {
        if (n > h.sum_cap) throw InternalError("owner-sum larger than its scratch");
        publish(h, x);
        // every shard forms the same sum in shard order (exact: one owner per entry)
        CKM(cudaMemcpyAsync(h.sum_scratch, g->slot[0], sizeof(double) * n,
                            cudaMemcpyDeviceToDevice, h.stream));
        for (size_t q = 1; q < g->h.size(); ++q)
            mtsk::add(int(n), static_cast<const double*>(g->slot[q]), h.sum_scratch, h.stream);
        done(h);
        CKM(cudaMemcpyAsync(x, h.sum_scratch, sizeof(double) * n, cudaMemcpyDeviceToDevice,
                            h.stream));
    }
    void bcast(pmts_mts& h, void* x, size_t bytes) override {
        publish(h, x);
        if (rank != 0 && bytes)
            CKM(cudaMemcpyAsync(x, g->slot[0], bytes, cudaMemcpyDeviceToDevice, h.stream));
        done(h);
    }
    void reduce_u64(pmts_mts& h, unsigned long long* x, int n, bool max) override {
        publish(h, x);
        std::vector<unsigned long long> acc(n, 0ull), t(n);
        for (size_t q = 0; q < g->h.size(); ++q) {
            CKM(cudaMemcpy(t.data(), g->slot[q], sizeof(unsigned long long) * n,
                           cudaMemcpyDeviceToHost));
            for (int i = 0; i < n; ++i) acc[i] = max ? std::max(acc[i], t[i]) : acc[i] + t[i];
        }
        g->wait();
        CKM(cudaMemcpy(x, acc.data(), sizeof(unsigned long long) * n, cudaMemcpyHostToDevice));
    }
};

// one NCCL clique, one rank per GPU (a process per GPU): everything stream-ordered
struct NcclComm : MtsComm {
    ncclComm_t c = nullptr;
    ~NcclComm() override {
        if (c) nccl().comm_destroy(c);
    }
    void halo(pmts_mts& h, double* x) override {
        NcclApi& a = nccl();
        for (const auto& l : h.links) mtsk::gather(l.n_send, l.send, x, l.sbuf, h.stream);
        nccl_check(a.group_start(), "group");
        for (const auto& l : h.links) {
            nccl_check(a.send(l.sbuf, l.n_send, ncclFloat64, l.peer, c, h.stream), "send");
            nccl_check(a.recv(l.rbuf, l.n_recv, ncclFloat64, l.peer, c, h.stream), "recv");
        }
        nccl_check(a.group_end(), "group");
        for (const auto& l : h.links) mtsk::scatter_set(l.n_recv, l.recv, l.rbuf, x, h.stream);
    }
    void sum_owned(pmts_mts& h, double* x, size_t n) override {
        nccl_check(nccl().all_reduce(x, x, n, ncclFloat64, ncclSum, c, h.stream), "all_reduce");
    }
    void bcast(pmts_mts& h, void* x, size_t bytes) override {
        nccl_check(nccl().broadcast(x, x, bytes, ncclUint8, 0, c, h.stream), "broadcast");
    }
    void reduce_u64(pmts_mts& h, unsigned long long* x, int n, bool max) override {
        nccl_check(nccl().all_reduce(x, x, n, ncclUint64, max ? ncclMax : ncclSum, c, h.stream),
                   "all_reduce");
    }
};

// run f(handle, rank) on every shard of a group, one host thread each; the first
// shard's error is rethrown (the others only saw the group abort)
template <class F>
void run_group(pmts_mts* const* hs, int n, F&& f) {
    if (!hs || n < 1 || !hs[0] || !hs[0]->group_comm) throw ConfigError("not a joined shard group");
    std::shared_ptr<ShardGroup> g = static_cast<GroupComm*>(hs[0]->comm.get())->g;
    if (int(g->h.size()) != n) throw ConfigError("shard group size mismatch");
    std::vector<std::exception_ptr> err(n);
    std::vector<std::thread> th;
    for (int r = 0; r < n; ++r)
        th.emplace_back([&, r] {
            try {
                CKM(cudaSetDevice(hs[r]->device));
                f(hs[r], r);
            } catch (...) {
                err[r] = std::current_exception();
                g->abort(r);
            }
        });
    for (auto& t : th) t.join();
    if (g->first_error >= 0) std::rethrow_exception(err[g->first_error]);
}

}  // namespace

extern "C" {

int pmts_mts_create(const pmts_mts_desc* desc, pmts_mts** out) {
    return guard([&] {
        if (!desc || !desc->scenario || !out) throw ConfigError("null argument");
        auto h = std::make_unique<pmts_mts>();
        build_host(*h, *desc);
        MtsSystem& s = h->s;
        if (s.pd_beta != 0.0)
            throw ConfigError("coupled PD substeps are explicit only (beta_pd = 0)");
        h->device = desc->device;
        h->nl = int(s.cpl_fe.size());
        h->m = s.m;
        h->iface_mode = desc->interface_mode;
        h->interface_precond = desc->interface_precond != 0;
        h->iface_precompute = desc->interface_recursion == 0;
        h->hfe_unit_columns = desc->interface_h_fe == 1;
        // interface mode (mts.hpp:111-114); the PD side is explicit
        h->use_dense = h->iface_mode == 1 || (h->iface_mode == 0 && h->nl <= 400);
        if (desc->shard_world > 1) {  // the shard plan (host; a host-only handle exposes it)
            if (desc->shard_rank < 0 || desc->shard_rank >= desc->shard_world)
                throw ConfigError("shard_rank out of range");
            if (h->use_dense)
                throw ConfigError("sharded coupled runs use the matrix-free interface "
                                  "(interface_mode = 2, or n_lambda > 400)");
            if (h->interface_precond)
                throw ConfigError("sharded coupled runs: interface_precond is not supported");
            h->sharded = true;
            h->root = desc->shard_rank == 0;
            h->setup_done = false;
            h->plan = make_shard_plan(s, desc->scenario->spacing, desc->shard_world,
                                      desc->shard_rank);
        }
        if (h->device < 0) {  // host-only: the assembled systems (view), no integrator
            *out = h.release();
            return;
        }
        CKM(cudaSetDevice(h->device));
        CKM(cudaStreamCreateWithFlags(&h->stream, cudaStreamNonBlocking));
        CKM(cudaStreamCreateWithFlags(&h->stream2, cudaStreamNonBlocking));
        for (cudaEvent_t* e : {&h->ev_fork, &h->ev_join, &h->ev_fork2, &h->ev_join2})
            CKM(cudaEventCreateWithFlags(e, cudaEventDisableTiming));
        h->nf = s.fe_n_dof;
        h->nl = int(s.cpl_fe.size());
        h->m = s.m;
        h->fe_nm.set(s.fe_gamma, s.fe_beta, s.m * s.dt_pd);
        h->pd_nm.set(s.pd_gamma, s.pd_beta, s.dt_pd);
        h->iface_mode = desc->interface_mode;
        h->enforce_continuity = desc->enforce_continuity != 0;
        h->track_energy = desc->track_energy != 0;
        h->fracture = s.s_crit > 0.0;
        if (h->track_energy && s.pd_gamma != 0.5)
            throw ConfigError("energy tracking of the PD quadratic term needs gamma_pd = 1/2");
        h->fe_cg_max = std::max(100, int(40 * std::sqrt(double(h->nf))));

        // ---- PD subdomain handle: compact nodes / elements of the PD-active set (a
        // sharded run: this shard's local part of them, in the same order) ----
        const int dim = s.dim, nn = dim == 2 ? 4 : 8;
        const int NPall = int(s.pd_active_nodes.size()), NEall = int(s.pd_active.size());
        if (!h->sharded) {
            h->plan.elems.resize(NEall);
            h->plan.nodes.resize(NPall);
            for (int k = 0; k < NEall; ++k) h->plan.elems[k] = k;
            for (int k = 0; k < NPall; ++k) h->plan.nodes[k] = k;
            h->plan.own_e0 = 0;
            h->plan.own_e1 = NEall;
            h->plan.node_own.assign(NPall, 1);
        }
        const std::vector<int>& lel = h->plan.elems;
        const std::vector<int>& lnd = h->plan.nodes;
        const int NPn = int(lnd.size());
        h->np = NPn * dim;
        std::vector<int> compact(s.nodes.size() / 3, -1);
        for (int k = 0; k < NPall; ++k) compact[s.pd_active_nodes[k]] = k;
        std::vector<int> c2l(NPall, -1);  // compact node -> local node
        for (int k = 0; k < NPn; ++k) c2l[lnd[k]] = k;
        std::vector<double> pxyz(3 * (size_t)NPn);
        for (int k = 0; k < NPn; ++k)
            for (int c = 0; c < 3; ++c)
                pxyz[3 * (size_t)k + c] = s.nodes[3 * (size_t)s.pd_active_nodes[lnd[k]] + c];
        std::vector<int32_t> pconn;
        for (int e : lel)
            for (int a = 0; a < nn; ++a)
                pconn.push_back(c2l[compact[s.conn[(size_t)s.pd_active[e] * nn + a]]]);
        // per-dof PD arrays of the local nodes (PD dof = compact node * dim + component)
        std::vector<double> lmass(h->np), lpext(h->np);
        for (int k = 0; k < NPn; ++k)
            for (int c = 0; c < dim; ++c) {
                lmass[(size_t)k * dim + c] = s.pd_mass[(size_t)lnd[k] * dim + c];
                lpext[(size_t)k * dim + c] = s.pd_p_ext[(size_t)lnd[k] * dim + c];
            }
        std::vector<int32_t> lbc;
        std::vector<double> lbcv;
        for (size_t q = 0; q < s.pd_bc_dofs.size(); ++q) {
            const int l = c2l[s.pd_bc_dofs[q] / dim];
            if (l < 0) continue;
            lbc.push_back(l * dim + s.pd_bc_dofs[q] % dim);
            lbcv.push_back(s.pd_bc_vel[q]);
        }
        pmts_pd_desc pdd{};
        pdd.dim = dim;
        pdd.n_nodes = NPn;
        pdd.n_elems = int(lel.size());
        pdd.node_xyz = pxyz.data();
        pdd.elem_nodes = pconn.data();
        pdd.mass = lmass.data();
        pdd.p_ext = lpext.data();
        pdd.n_bc = int(lbc.size());
        pdd.bc_dofs = lbc.data();
        pdd.bc_vel = lbcv.data();
        pdd.delta = s.delta;
        pdd.micromodulus = PMTS_MICRO_EXP;
        pdd.c0 = s.c0;
        pdd.l = s.l;
        pdd.s_crit = s.s_crit;
        pdd.gamma = s.pd_gamma;
        pdd.beta = 0.0;
        pdd.dt = s.dt_pd;
        pdd.mode = PMTS_DETERMINISTIC;
        pdd.device = h->device;
        pdd.n_notch = desc->scenario->n_notch;
        pdd.notch_npts = desc->scenario->notch_npts;
        pdd.notch_pts = desc->scenario->notch_pts;
        if (h->sharded) {  // broken bonds are counted by the shard owning the lower element
            pdd.owned_elems[0] = h->plan.own_e0;
            pdd.owned_elems[1] = h->plan.own_e1;
        }
        check_pd(pmts_pd_create(&pdd, &h->pd));
        check_pd(pmts_pd_build_families(h->pd));
        int64_t npairs = 0;
        check_pd(pmts_pd_get_pairs(h->pd, nullptr, 0, &npairs));
        std::vector<int32_t> cp(2 * (size_t)npairs);
        check_pd(pmts_pd_get_pairs(h->pd, cp.data(), npairs, &npairs));
        h->npe = int(npairs);
        h->pairs.resize(cp.size());
        h->pe_weight.resize(npairs);
        if (npairs > INT32_MAX) throw ConfigError("more than 2^31 PD bonds");
        par_range(int(npairs), [&](int p) {
            const int gi = s.pd_active[lel[cp[2 * (size_t)p]]];
            const int gj = s.pd_active[lel[cp[2 * (size_t)p + 1]]];
            h->pairs[2 * (size_t)p] = gi;
            h->pairs[2 * (size_t)p + 1] = gj;
            double mid[3];
            for (int k = 0; k < 3; ++k)
                mid[k] = 0.5 * (s.centroid[3 * (size_t)gi + k] + s.centroid[3 * (size_t)gj + k]);
            const double w = 1.0 - mts_alpha_at(s, mid);  // perifem.hpp:320-326
            if (w < 0.0) throw InternalError("negative PD weight at a bond midpoint");
            h->pe_weight[p] = w;
        });
        pd_internal_pair_weights(h->pd, h->pe_weight.data());
        h->pdv = pd_internal_dev(h->pd);
        h->mask_live = h->pdv.mask;
        h->mask_words = (size_t)h->pdv.W * h->pdv.E;
        h->mask_sync = h->alloc<uint32_t>(h->mask_words);
        if (dim == 3 && desc->pd_linear != 1 && h->pdv.K <= mtsk::lin_lat_stencil_size()) {
            // the local PD elements as a box of the generated lattice in lattice order?
            const double hh = desc->scenario->spacing;
            const int E = int(lel.size());
            double org[3] = {1e300, 1e300, 1e300};
            for (int e = 0; e < E; ++e)
                for (int c = 0; c < 3; ++c)
                    org[c] = std::min(org[c], s.centroid[3 * (size_t)s.pd_active[lel[e]] + c]);
            long long n[3] = {0, 0, 0};
            std::vector<int> idx(3 * (size_t)E);
            for (int e = 0; e < E; ++e)
                for (int c = 0; c < 3; ++c) {
                    const long long q = std::llround(
                        (s.centroid[3 * (size_t)s.pd_active[lel[e]] + c] - org[c]) / hh);
                    idx[3 * (size_t)e + c] = int(q);
                    n[c] = std::max(n[c], q + 1);
                }
            bool box = hh > 0.0 && n[0] * n[1] * n[2] == E;
            for (int e = 0; e < E && box; ++e)
                box = ((long long)idx[3 * (size_t)e + 2] * n[1] + idx[3 * (size_t)e + 1]) * n[0] +
                          idx[3 * (size_t)e] == e;
            if (box) {
                h->lat.nx = int(n[0]);
                h->lat.ny = int(n[1]);
                h->lat.nz = int(n[2]);
                h->lat.h = hh;
                int8_t table[343];
                mtsk::lin_lat_slot_table(table);
                int8_t* dslot = h->alloc<int8_t>(343);
                CKM(cudaMemcpy(dslot, table, 343, cudaMemcpyHostToDevice));
                h->lat.slot = dslot;
                h->lat.coefS = h->alloc<double>((size_t)mtsk::lin_lat_coef_slots() * E);
                h->lat.maskS = h->alloc<uint32_t>(4 * (size_t)E);
                // (an entry outside the 122 offsets -- another horizon -- keeps the ELL form)
                h->lin_lat = mtsk::lin_lat_build(h->pdv, h->lat, h->stream);
                if (!h->lin_lat) {
                    h->release(h->lat.coefS);
                    h->release(h->lat.maskS);
                    h->lat.coefS = nullptr;
                    h->lat.maskS = nullptr;
                }
            }
        }
        const bool elemq = desc->pd_elem_products == 1 ||
                           (desc->pd_elem_products == 0 && h->pdv.E >= (1 << 18));
        // entry-major families (coalesced lanes): the ELL linear force, and the
        // element-product force of the free substeps
        if (!h->lin_lat || elemq) {
            const size_t ek = (size_t)h->pdv.E * h->pdv.K;
            h->famT_col = h->alloc<int32_t>(ek);
            h->famT_coef = h->alloc<double>(ek);
            mtsk::family_transpose(h->pdv, h->famT_col, h->famT_coef, h->stream);
        }
        if (elemq) {  // (small subdomains are launch-bound: one kernel)
            h->elem_q = h->alloc<double>((size_t)h->pdv.E * nn * dim);
            h->elem_s = h->alloc<double>((size_t)h->pdv.E * 8);  // 64-byte records
        }
        h->snapshot_bonds();
        CKM(cudaStreamSynchronize(h->stream));

        // ---- device arrays ----
        auto flags = [](int n, const std::vector<int32_t>& bc, const std::vector<double>& vel,
                        std::vector<uint8_t>& cf, std::vector<double>& bv) {
            cf.assign(n, 0);
            bv.assign(n, 0.0);
            for (size_t c = 0; c < bc.size(); ++c) {
                cf[bc[c]] = 1;
                bv[bc[c]] = vel[c];
            }
        };
        std::vector<uint8_t> cf;
        std::vector<double> bv;
        h->fe_rp = h->upload(s.fe_rowptr);
        h->fe_ci = h->upload(s.fe_col);
        h->fe_v = h->upload(s.fe_val);
        h->fe_M = h->upload(s.fe_mass);
        h->fe_P = h->upload(s.fe_p_ext);
        flags(h->nf, s.fe_bc_dofs, s.fe_bc_vel, cf, bv);
        h->fe_cf = h->upload(cf);
        h->fe_bcv = h->upload(bv);
        h->fe_jac = h->upload(jacobi_diag(s, h->fe_nm.bdt2));
        h->pd_M = h->upload(lmass);
        h->pd_P = h->upload(lpext);
        flags(h->np, lbc, lbcv, cf, bv);
        h->pd_cf = h->upload(cf);
        h->pd_bcv = h->upload(bv);
        h->cfe = h->upload(s.cpl_fe);
        // coupling rows -> local PD dofs (sharded: the rows this shard owns, else -1)
        std::vector<int32_t> lcpd(h->nl, -1);
        for (int r = 0; r < h->nl; ++r) {
            const int l = c2l[s.cpl_pd[r] / dim];
            if (l >= 0 && h->plan.node_own[l]) lcpd[r] = l * dim + s.cpl_pd[r] % dim;
        }
        h->cpd = h->upload(lcpd);
        if (h->sharded) {
            h->cpd_own = h->cpd;
            std::vector<int32_t> id(h->nl);
            for (int r = 0; r < h->nl; ++r) id[r] = r;
            h->ident = h->upload(id);
            std::vector<int32_t> od;
            for (int k = 0; k < NPn; ++k)
                if (h->plan.node_own[k])
                    for (int c = 0; c < dim; ++c) od.push_back(k * dim + c);
            h->n_own_dofs = int(od.size());
            h->own_dofs = h->upload(od);
            h->own_zero = h->alloc<double>(od.size());
            CKM(cudaMemsetAsync(h->own_zero, 0, sizeof(double) * std::max<size_t>(od.size(), 1),
                                h->stream));
            h->gpd_now = h->alloc<double>(h->nl);
            for (const ShardLink& lk : h->plan.links) {
                pmts_mts::LinkDev ld;
                ld.peer = lk.peer;
                ld.n_send = int(lk.send.size());
                ld.n_recv = int(lk.recv.size());
                ld.send = h->upload(lk.send);
                ld.recv = h->upload(lk.recv);
                ld.sbuf = h->alloc<double>(lk.send.size());
                ld.rbuf = h->alloc<double>(lk.recv.size());
                h->links.push_back(ld);
            }
            h->sum_cap = (size_t)(h->m + 1) * h->nl;
            h->sum_scratch = h->alloc<double>(h->sum_cap);
            h->more_d = h->alloc<int>(1);
            CKM(cudaMallocHost(&h->more_h, sizeof(int)));
        }
        h->gfe_rp = h->upload(s.cpl_fe_rp);
        h->gfe_ci = h->upload(s.cpl_fe_ci);
        h->gfe_w = h->upload(s.cpl_fe_w);
        {  // transpose of G_FE over the touched FE dofs, rows ascending per dof
            std::vector<std::vector<std::pair<int, double>>> col(h->nf);
            for (int r = 0; r < h->nl; ++r)
                for (int j = s.cpl_fe_rp[r]; j < s.cpl_fe_rp[r + 1]; ++j)
                    col[s.cpl_fe_ci[j]].push_back({r, s.cpl_fe_w[j]});
            std::vector<int32_t> td, trp(1, 0), tri;
            std::vector<double> tw;
            for (int d = 0; d < h->nf; ++d) {
                if (col[d].empty()) continue;
                td.push_back(d);
                for (const auto& [r, w] : col[d]) {
                    tri.push_back(r);
                    tw.push_back(w);
                }
                trp.push_back(int32_t(tri.size()));
            }
            h->gft_n = int(td.size());
            h->gft_d = h->upload(td);
            h->gft_rp = h->upload(trp);
            h->gft_ri = h->upload(tri);
            h->gft_w = h->upload(tw);
        }
        const int nmax = std::max({h->nf, h->np, h->nl});
        h->ufe = h->state(h->nf);
        h->vfe = h->state(h->nf);
        h->fe_prev = h->state(h->nf);
        h->upd = h->state(h->np);
        h->vpd = h->state(h->np);
        h->wst = h->state(nmax);
        h->yst = h->state(nmax);
        h->rd = h->alloc<double>(nmax);
        h->rv = h->alloc<double>(nmax);
        h->ra = h->alloc<double>(nmax);
        h->kd = h->alloc<double>(nmax);
        for (double** p : {&h->cg_b, &h->cg_x, &h->cg_r, &h->cg_z, &h->cg_p, &h->cg_ap, &h->cg_kx})
            *p = h->alloc<double>(nmax);
        h->part = h->alloc<double>(mtsk::dot_partials());
        h->part2 = h->alloc<double>(2 * mtsk::dot_partials());
        h->part3 = h->alloc<double>(std::max(mtsk::pap_partials(nmax, false),
                                             mtsk::pap_partials(h->nl, true)));
        h->ticket3 = reinterpret_cast<unsigned*>(h->alloc<double>(1));
        CKM(cudaMemsetAsync(h->ticket3, 0, sizeof(double), h->stream));
        h->ticket = reinterpret_cast<unsigned*>(h->alloc<double>(1));
        CKM(cudaMemsetAsync(h->ticket, 0, sizeof(double), h->stream));
        h->zero_flags(nmax);  // allocated before any CG graph capture uses it
        h->rd_fe = h->alloc<double>(h->nf);
        h->rv_fe = h->alloc<double>(h->nf);
        h->ra_fe = h->alloc<double>(h->nf);
        h->lam_tmp_fe = h->alloc<double>(h->nl);
        h->wst_fe = h->state(h->nf);
        h->cg_status = h->alloc<int>(2 * pmts_mts::N_CG);
        CKM(cudaMemsetAsync(h->cg_status, 0, sizeof(int) * 2 * pmts_mts::N_CG, h->stream));
        CKM(cudaMallocHost(&h->h_pin, 1024));
        h->scal = h->alloc<double>(8 * pmts_mts::N_CG);
        h->en_d = h->alloc<double>(3);
        h->cmax_d = h->alloc<unsigned long long>(4);
        h->lu_flag = h->alloc<int>(1);
        h->lamp_d = h->alloc<double>(h->nl);
        h->gprev_d = h->alloc<double>(h->nl);
        h->ta_d = h->alloc<double>((size_t)h->m * h->nl);
        h->tb_d = h->alloc<double>((size_t)h->m * h->nl);
        CKM(cudaMemsetAsync(h->lamp_d, 0, sizeof(double) * h->nl, h->stream));
        h->lam_d = h->alloc<double>(h->nl);
        h->lam_tmp = h->alloc<double>(h->nl);
        h->gvec = h->alloc<double>(h->nl);
        h->sv_d = h->alloc<double>((size_t)h->m * h->nl);
        h->pd_ubar = h->alloc<double>((size_t)h->pdv.E * dim);
        {
            std::vector<int32_t> ro(h->np, -1);
            for (int r = 0; r < h->nl; ++r)
                if (lcpd[r] >= 0) ro[lcpd[r]] = r;
            h->row_of = h->upload(ro);
        }
        h->gp_free_d = h->alloc<double>((size_t)(h->m + 1) * h->nl);
        h->gp_link_d = h->alloc<double>((size_t)(h->m + 1) * h->nl);
        h->warm_fe_free = h->alloc<double>(h->nf);
        h->warm_fe_link = h->alloc<double>(h->nf);
        h->d_counts = h->alloc<unsigned long long>(h->m + 1);
        h->counts_cap = h->m + 1;
        // BC velocities on the initial states (mts.hpp:107-108)
        {
            std::vector<double> z(h->nf, 0.0);
            for (size_t c = 0; c < s.fe_bc_dofs.size(); ++c) z[s.fe_bc_dofs[c]] = s.fe_bc_vel[c];
            h->to_dev(h->ufe.v, z);
            std::vector<double> zp(h->np, 0.0);
            for (size_t c = 0; c < lbc.size(); ++c) zp[lbc[c]] = lbcv[c];
            h->to_dev(h->upd.v, zp);
        }
        // g_p_fe = G_FE P_ext (mts.hpp:110)
        {
            std::vector<double> g(h->nl);
            for (int r = 0; r < h->nl; ++r) {
                int j = s.cpl_fe_rp[r];
                double acc = s.cpl_fe_w[j] * s.fe_p_ext[s.cpl_fe_ci[j]];
                for (++j; j < s.cpl_fe_rp[r + 1]; ++j) acc += s.cpl_fe_w[j] * s.fe_p_ext[s.cpl_fe_ci[j]];
                g[r] = acc;
            }
            h->gpfe_d = h->upload(g);
        }
        CKM(cudaStreamSynchronize(h->stream));
        if (h->root) h->build_h_fe();
        if (!h->sharded) {
            if (h->use_dense) h->refresh_dense_interface();
            else if (h->iface_precompute) h->build_h_pd();
        }  // sharded: H_FE goes to every shard and H_PD is built across them in pmts_mts_init
        CKM(cudaStreamSynchronize(h->stream));
        *out = h.release();
    });
}

int pmts_mts_view_get(const pmts_mts* h, pmts_mts_view* v) {
    return guard([&] {
        if (!h || !v) throw ConfigError("null argument");
        const MtsSystem& s = h->s;
        *v = pmts_mts_view{};
        v->dim = s.dim;
        v->n_nodes = int32_t(s.nodes.size() / 3);
        v->n_elems = int32_t(s.volume.size());
        v->fe_n_dof = s.fe_n_dof;
        v->pd_n_dof = s.pd_n_dof;
        v->n_lambda = h->nl;
        v->dense = h->use_dense ? 1 : 0;
        v->m = s.m;
        v->n_macro = s.n_macro;
        v->fe_nnz = int32_t(s.fe_val.size());
        v->fe_n_bc = int32_t(s.fe_bc_dofs.size());
        v->pd_n_bc = int32_t(s.pd_bc_dofs.size());
        v->n_pd_elems = int32_t(s.pd_active.size());
        v->n_pairs = h->npe;
        v->dt_pd = s.dt_pd;
        v->delta = s.delta;
        v->c0 = s.c0;
        v->l = s.l;
        v->char_length = s.cl;
        v->load_ramp = s.ramp;
        static thread_local std::vector<int32_t> labels;
        labels.assign(s.label.begin(), s.label.end());
        v->labels = labels.data();
        v->alpha = s.alpha.data();
        v->fe_node_dof = s.fe_node_dof.data();
        v->pd_node_dof = s.pd_node_dof.data();
        v->fe_k_rowptr = s.fe_rowptr.data();
        v->fe_k_col = s.fe_col.data();
        v->fe_k_val = s.fe_val.data();
        v->fe_mass = s.fe_mass.data();
        v->fe_p_ext = s.fe_p_ext.data();
        v->pd_mass = s.pd_mass.data();
        v->pd_p_ext = s.pd_p_ext.data();
        v->fe_bc_dofs = s.fe_bc_dofs.data();
        v->fe_bc_vel = s.fe_bc_vel.data();
        v->pd_bc_dofs = s.pd_bc_dofs.data();
        v->pd_bc_vel = s.pd_bc_vel.data();
        v->cpl_fe_dof = s.cpl_fe.data();
        v->cpl_pd_dof = s.cpl_pd.data();
        v->cpl_fe_nnz = int64_t(s.cpl_fe_ci.size());
        v->cpl_fe_rowptr = s.cpl_fe_rp.data();
        v->cpl_fe_col = s.cpl_fe_ci.data();
        v->cpl_fe_w = s.cpl_fe_w.data();
        v->fe_mesh_elems = s.fe_mesh_elems;
        v->fe_mesh_nodes = s.fe_mesh_nodes;
        v->pd_linear_lattice = h->lin_lat ? 1 : 0;
        v->pairs = h->pairs.data();
        v->pe_weight = h->pe_weight.data();
        v->node_xyz = s.nodes.data();
        v->elem_nodes = s.conn.data();
        v->node_alpha = s.node_alpha.data();
    });
}

int pmts_mts_init(pmts_mts* h) {
    return guard([&] {
        if (!h) throw ConfigError("null handle");
        if (h->device < 0) throw ConfigError("host-only handle (device < 0)");
        if (h->group_comm) throw ConfigError("in-process shard group: pmts_mts_group_init");
        CKM(cudaSetDevice(h->device));
        if (h->sharded && !h->setup_done) h->shard_setup();
        h->initialize_accelerations();
    });
}

int pmts_mts_shard_view_get(const pmts_mts* h, pmts_mts_shard_view* v) {
    return guard([&] {
        if (!h || !v) throw ConfigError("null argument");
        const ShardPlan& p = h->plan;
        *v = pmts_mts_shard_view{};
        v->world = h->sharded ? p.world : 1;
        v->rank = h->sharded ? p.rank : 0;
        v->axis = p.axis;
        v->reach_layers = p.D;
        v->n_layers = p.layers;
        v->n_local_nodes = int32_t(p.nodes.size());
        v->n_local_elems = int32_t(p.elems.size());
        v->own_elem_lo = p.own_e0;
        v->own_elem_hi = p.own_e1;
        v->local_nodes = reinterpret_cast<const int32_t*>(p.nodes.data());
        v->local_elems = reinterpret_cast<const int32_t*>(p.elems.data());
        v->node_owned = p.node_own.data();
        v->layer_bounds = reinterpret_cast<const int32_t*>(p.bounds.data());
    });
}

int pmts_mts_group_join(pmts_mts* const* hs, int32_t n) {
    return guard([&] {
        if (!hs || n < 2) throw ConfigError("a shard group needs at least 2 handles");
        auto g = std::make_shared<ShardGroup>();
        g->h.assign(hs, hs + n);
        g->slot.assign(n, nullptr);
        for (int r = 0; r < n; ++r) {
            pmts_mts* h = hs[r];
            if (!h || h->device < 0 || !h->sharded || h->plan.world != n || h->plan.rank != r)
                throw ConfigError("handle " + std::to_string(r) + " is not shard " +
                                  std::to_string(r) + " of " + std::to_string(n));
            if (h->comm) throw ConfigError("shard already has a transport");
        }
        for (int r = 0; r < n; ++r)  // device copies between shards on different GPUs
            for (int q = 0; q < n; ++q)
                if (hs[r]->device != hs[q]->device) {
                    CKM(cudaSetDevice(hs[r]->device));
                    const cudaError_t e = cudaDeviceEnablePeerAccess(hs[q]->device, 0);
                    if (e != cudaSuccess && e != cudaErrorPeerAccessAlreadyEnabled) CKM(e);
                    cudaGetLastError();
                }
        for (int r = 0; r < n; ++r) {
            auto c = std::make_unique<GroupComm>();
            c->g = g;
            c->rank = r;
            hs[r]->comm = std::move(c);
            hs[r]->group_comm = true;
        }
    });
}

int pmts_mts_group_init(pmts_mts* const* hs, int32_t n) {
    return guard([&] {
        run_group(hs, n, [](pmts_mts* h, int) {
            if (!h->setup_done) h->shard_setup();
            h->initialize_accelerations();
        });
    });
}

int pmts_mts_group_macro_step(pmts_mts* const* hs, int32_t n, int32_t steps,
                              pmts_mts_report* reports) {
    return guard([&] {
        if (steps < 0) throw ConfigError("bad step count");
        run_group(hs, n, [&](pmts_mts* h, int r) {
            for (int i = 0; i < steps; ++i) {
                const pmts_mts_report rep = h->macro_step();
                if (reports && r == 0) reports[i] = rep;
            }
        });
    });
}

int pmts_mts_comm_init(pmts_mts* h, const void* nccl_id) {
    return guard([&] {
        if (!h || !nccl_id) throw ConfigError("null argument");
        if (!h->sharded || h->device < 0) throw ConfigError("not a device shard handle");
        if (h->comm) throw ConfigError("shard already has a transport");
        ncclUniqueId uid;
        std::memcpy(&uid, nccl_id, sizeof(uid));
        CKM(cudaSetDevice(h->device));
        auto c = std::make_unique<NcclComm>();
        nccl_check(nccl().comm_init_rank(&c->c, h->plan.world, uid, h->plan.rank), "comm init");
        h->comm = std::move(c);
    });
}

int pmts_mts_macro_step(pmts_mts* h, int32_t n, pmts_mts_report* reports) {
    return guard([&] {
        if (!h || n < 0) throw ConfigError("bad arguments");
        if (h->device < 0) throw ConfigError("host-only handle (device < 0)");
        if (h->group_comm) throw ConfigError("in-process shard group: pmts_mts_group_macro_step");
        CKM(cudaSetDevice(h->device));
        for (int i = 0; i < n; ++i) {
            const pmts_mts_report r = h->macro_step();
            if (reports) reports[i] = r;
        }
    });
}

int pmts_mts_macro_step_timed(pmts_mts* h, int32_t n, float* ms_out) {
    return guard([&] {
        if (!h || n < 0) throw ConfigError("bad arguments");
        if (h->device < 0) throw ConfigError("host-only handle (device < 0)");
        if (h->group_comm) throw ConfigError("in-process shard group: pmts_mts_group_macro_step");
        CKM(cudaSetDevice(h->device));
        cudaEvent_t e0, e1;
        CKM(cudaEventCreate(&e0));
        CKM(cudaEventCreate(&e1));
        CKM(cudaStreamSynchronize(h->stream));
        CKM(cudaEventRecord(e0, h->stream));
        for (int i = 0; i < n; ++i) h->macro_step();
        CKM(cudaEventRecord(e1, h->stream));
        CKM(cudaEventSynchronize(e1));
        float ms = 0.f;
        CKM(cudaEventElapsedTime(&ms, e0, e1));
        cudaEventDestroy(e0);
        cudaEventDestroy(e1);
        if (ms_out) *ms_out = ms;
    });
}

int pmts_mts_get_state(pmts_mts* h, int32_t which, double* u, double* v, double* a) {
    return guard([&] {
        if (!h || (which != 0 && which != 1)) throw ConfigError("bad arguments");
        if (h->device < 0) throw ConfigError("host-only handle (device < 0)");
        const DState& st = which == 0 ? h->ufe : h->upd;
        const int n = which == 0 ? h->nf : h->np;
        if (u) CKM(cudaMemcpyAsync(u, st.u, sizeof(double) * n, cudaMemcpyDeviceToHost, h->stream));
        if (v) CKM(cudaMemcpyAsync(v, st.v, sizeof(double) * n, cudaMemcpyDeviceToHost, h->stream));
        if (a) CKM(cudaMemcpyAsync(a, st.a, sizeof(double) * n, cudaMemcpyDeviceToHost, h->stream));
        CKM(cudaStreamSynchronize(h->stream));
    });
}

int pmts_mts_get_lambda(pmts_mts* h, double* out) {
    return guard([&] {
        if (!h || !out) throw ConfigError("bad arguments");
        if (h->device < 0 || !h->lamp_d) {
            std::fill(out, out + h->nl, 0.0);
            return;
        }
        CKM(cudaMemcpyAsync(out, h->lamp_d, sizeof(double) * h->nl, cudaMemcpyDeviceToHost,
                            h->stream));
        CKM(cudaStreamSynchronize(h->stream));
    });
}

int pmts_mts_get_intact(pmts_mts* h, uint8_t* out) {
    return guard([&] {
        if (!h || !out) throw ConfigError("bad arguments");
        if (h->device < 0) throw ConfigError("host-only handle (device < 0)");
        check_pd(pmts_pd_get_intact(h->pd, out, h->npe));
    });
}

int pmts_mts_damage(pmts_mts* h, double* elem_out, double* node_out) {
    return guard([&] {
        if (!h || !elem_out || !node_out) throw ConfigError("bad arguments");
        if (h->device < 0) throw ConfigError("host-only handle (device < 0)");
        const MtsSystem& s = h->s;
        const ShardPlan& p = h->plan;  // a shard fills its owned elements / nodes only
        std::vector<double> pe(p.elems.size()), pn(p.nodes.size());
        check_pd(pmts_pd_damage(h->pd, pe.data(), pn.data()));
        std::fill(elem_out, elem_out + s.volume.size(), 0.0);
        std::fill(node_out, node_out + s.nodes.size() / 3, 0.0);
        for (int k = p.own_e0; k < p.own_e1; ++k) elem_out[s.pd_active[p.elems[k]]] = pe[k];
        for (size_t k = 0; k < p.nodes.size(); ++k)
            if (p.node_own[k]) node_out[s.pd_active_nodes[p.nodes[k]]] = pn[k];
    });
}

void pmts_mts_destroy(pmts_mts* h) { delete h; }

}  // extern "C"
