/* pmts_capi.h -- C ABI of the B200-native PD fine-step path (sm_100a).
 *
 * Drop-in boundary for the reference's pure-PD hot path.
 * The reference is a header-only C++ library with no FFI layer; the calls a
 * host driver makes on this path are the ones listed beside each entry point
 * below (paths under /root/reference/proj/include/perimts/).  Plain pointers
 * and sizes only: no C++ or torch types cross this boundary; no exception
 * crosses it either -- every entry point returns a status code (errors.hpp
 * mapping: 2 ConfigError, 3 SolverError, 1 InternalError/CUDA) and
 * pmts_last_error() holds the message (thread-local).
 *
 * Threading: one host thread per handle; each handle owns one CUDA stream and
 * its device buffers.  Entry points that return host data synchronise that
 * stream; pmts_pd_step is stream-ordered and returns when the step count
 * (and the newly-broken count) is known.
 */
#ifndef PMTS_CAPI_H
#define PMTS_CAPI_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define PMTS_ABI_VERSION 2  /* 2: pmts_mts_desc.pd_linear / pd_elem_products,
                                  pmts_mts_view.pd_linear_lattice, PMTS_OPT_CLEAN_TILES */

enum pmts_status {
    PMTS_OK = 0,
    PMTS_ERR_INTERNAL = 1, /* InternalError / CUDA failure            (errors.hpp:18-21) */
    PMTS_ERR_CONFIG = 2,   /* ConfigError: bad input                  (errors.hpp:8-11)  */
    PMTS_ERR_SOLVER = 3    /* SolverError: non-positive mass, non-finite state (errors.hpp:13-16) */
};

enum pmts_mode {
    PMTS_DETERMINISTIC = 0, /* reference neighbour order, exact stretch, no FMA: broken set
                               bit-exact, u/v/a equal to the matrix-free oracle bitwise */
    PMTS_FAST = 1,          /* centroid-averaged eta, squared break test, lattice stencil
                               families when the mesh is a lattice */
    PMTS_FAST_F32POS = 2    /* BASELINE cfg3's fp32-position / fp64-accumulate variant of fast
                               mode (extension): tile-relative fp32 displacements in the force
                               and the candidate break test, fp64 force accumulation, fp64
                               state; 2D lattice tile kernel only */
};

enum pmts_micromodulus {
    PMTS_MICRO_EXP = 0,  /* c0 exp(-r/l), zero beyond delta  (material.hpp:84-88) */
    PMTS_MICRO_CONST = 1 /* BASELINE c = 9E/(pi h delta^3) [2D] / 18K/(pi delta^4) [3D], applied
                            in PeriFEM form c h / r^3 [2D] or c / r^3 [3D]  (extension) */
};

/* ------------------------------------------------------------------------
 * Scenario setup -- the host side of build_scenario (driver.hpp:170-231),
 * convert_tractions_to_bands (driver.hpp:76-116), generate_structured +
 * compute_element_geometry (mesh.hpp:112-219), calibrate_c0
 * (material.hpp:150-165) and the M / P_ext part of assemble_pd_global
 * (perifem.hpp:331-349) for a generated pure-PD run.  Arrays are owned by the
 * scenario and stay valid until pmts_scenario_destroy.
 * ------------------------------------------------------------------------ */
typedef struct pmts_scenario pmts_scenario;

typedef struct {
    int32_t dim;                 /* 2 or 3 */
    double lo[3], hi[3];         /* mesh.bounds */
    double spacing;              /* mesh.spacing */
    double E, nu, rho;           /* [material] */
    int32_t formulation;         /* 0 plane_stress, 1 plane_strain, 2 three_d */
    double delta_factor, l_factor, s_crit; /* [pd] */
    int32_t n_notch;             /* notches: npts[k] points each, xyz */
    const int32_t* notch_npts;
    const double* notch_pts;
    int32_t n_traction;          /* per patch: lo[3] hi[3] value[3] (9 doubles) */
    const double* traction;
    int32_t n_body_patch;        /* per patch: lo[3] hi[3] value[3] */
    const double* body_patch;
    double body_force[3];
    int32_t n_velocity_bc;       /* per bc: lo[3] hi[3] component value (8 doubles) */
    const double* velocity_bc;
    int32_t n_fixed;             /* per box: lo[3] hi[3] (6 doubles) */
    const double* fixed;
    double dt_pd;                /* [time] */
    int32_t m;
    double total_time;
    double load_ramp;            /* < 0: auto (= m dt_pd), driver.hpp:187-191 */
    double gamma, beta;
    int32_t host_setup;          /* 1: the setup loops on the host (the restatement the device
                                    setup is tested against, tests/test_gpu_setup.py); 0: on the
                                    device when one is present */
} pmts_scenario_desc;

typedef struct {
    int32_t dim, n_nodes, n_elems, n_dof, n_bc, n_steps;
    int32_t lattice[3];          /* elements per axis of the generated grid */
    double delta, l, c0, char_length, dt, gamma, beta, s_crit, load_ramp;
    const double* node_xyz;      /* [n_nodes][3] */
    const int32_t* elem_nodes;   /* [n_elems][2^dim], reference node order */
    const double* centroid;      /* [n_elems][3] */
    const double* volume;        /* [n_elems] */
    const double* mass;          /* [n_dof] lumped, (1-alpha)-weighted (alpha = 0) */
    const double* p_ext;         /* [n_dof] full-amplitude external load */
    const int32_t* bc_dofs;      /* [n_bc] sorted */
    const double* bc_vel;        /* [n_bc] */
} pmts_scenario_view;

int pmts_scenario_build(const pmts_scenario_desc* desc, pmts_scenario** out);
int pmts_scenario_get(const pmts_scenario* sc, pmts_scenario_view* view);
/* load_scale(t) = clamp(t / ramp, 0, 1)  (driver.hpp:187-191) */
double pmts_scenario_load_scale(const pmts_scenario* sc, double t);
void pmts_scenario_destroy(pmts_scenario* sc);

/* ------------------------------------------------------------------------
 * PD fine-step handle
 * ------------------------------------------------------------------------ */
typedef struct pmts_pd pmts_pd;

typedef struct {
    int32_t dim, n_nodes, n_elems;
    const double* node_xyz;      /* [n_nodes][3] */
    const int32_t* elem_nodes;   /* [n_elems][2^dim] (mesh.hpp:206-213 order) */
    const double* mass;          /* [n_nodes*dim], dof = node*dim + c (fem.hpp:381-409) */
    const double* p_ext;         /* [n_nodes*dim] */
    int32_t n_bc;                /* BcTable (fem.hpp:477-482): sorted dofs + velocities */
    const int32_t* bc_dofs;
    const double* bc_vel;
    double delta;                /* horizon */
    int32_t micromodulus;        /* enum pmts_micromodulus */
    double c0, l;                /* exponential kernel */
    double c_const, h;           /* constant kernel (h: plate thickness, 2D) */
    double s_crit;               /* <= 0: fracture off (material.hpp:44) */
    double s_crit_spread;        /* per-bond factor U[1-spread, 1+spread] (extension), 0 = off */
    uint64_t seed;               /* counter-hash seed of the per-bond factor */
    double gamma, beta, dt;      /* NewmarkParams (newmark.hpp:14-30); beta must be 0 */
    int32_t mode;                /* enum pmts_mode */
    int32_t device;              /* CUDA ordinal */
    int32_t n_notch;             /* notches (mesh.hpp:316-318) for pmts_pd_build_families */
    const int32_t* notch_npts;
    const double* notch_pts;
    int32_t lattice[3];          /* optional: elements per axis if the mesh is the generated
                                    lattice (enables the stencil fast path); 0 = unknown */
    /* --- slab decomposition (multi-GPU); all zero for a single domain --- */
    int64_t global_id_offset;    /* global id of local element 0 (per-bond hash uses global ids) */
    int32_t owned_elems[2];      /* local element range this rank owns (broken counts); 0,0 = all;
                                    with slab_plane: the in-layer range (l mod slab_plane[0]) */
    double lattice_h;            /* > 0: stencil constants from the nominal lattice (xi = offset*h,
                                    w = lattice_vol^2) so every rank's table is identical */
    double lattice_vol;
    int32_t slab_plane[2];       /* 3D slabs cut along y (z-x slabs): elements per z layer,
                                    local and global; global id of local element l =
                                    (l / p0) p1 + global_id_offset + l mod p0.  0,0: contiguous */
    int32_t node_rows[2];        /* lattice path: the y node rows [lo, hi) this rank updates (its
                                    owned rows); element forces only for the rows they need.
                                    0,0 = all */
} pmts_pd_desc;

typedef struct {
    int64_t n_bonds;             /* unique bonds B */
    int64_t n_entries;           /* directed family entries F = 2B */
    int32_t max_family;          /* largest family */
    int32_t path;                /* 0 CSR/ELL families, 1 lattice stencil */
    int32_t kernels_per_step;    /* kernel launches per fine step */
    int32_t stencil_size;        /* stencil offsets (path 1) */
    double bytes_per_step;       /* algorithmic HBM bytes per fine step */
    double bond_bytes_per_step;  /* ... of which the bond kernel (roofline numerator) */
    double device_bytes;         /* device memory held by the handle */
    int64_t hot_tiles;           /* PMTS_OPT_COUNT_HOT: tiles whose break test ran / */
    int64_t tested_tiles;        /* tiles the cold-tile screen examined, since enabled */
} pmts_pd_info;

const char* pmts_last_error(void);
int pmts_abi_version(void);
int pmts_device_count(int* n);

/* BlockOperator ctor validation (newmark.hpp:81-93) + device upload + element
 * geometry (mesh.hpp:112-139) and bond constants (perifem.hpp:87-97). */
int pmts_pd_create(const pmts_pd_desc* desc, pmts_pd** out);
void pmts_pd_destroy(pmts_pd* h);

/* find_pe_pairs (mesh.hpp:416-495) on the device: cell list of size delta,
 * notch cut with eps = 1e-12 * char_length, families sorted by partner id. */
int pmts_pd_build_families(pmts_pd* h);
/* Inject an explicit pair list instead ((i<j) rows sorted, as find_pe_pairs
 * returns them) -- e.g. the reference's own list. */
int pmts_pd_set_pairs(pmts_pd* h, int64_t n_pairs, const int32_t* pairs);
/* Pair list back in find_pe_pairs order ((i,j) rows, i<j, sorted). */
int pmts_pd_get_pairs(pmts_pd* h, int32_t* pairs_out, int64_t cap, int64_t* n_out);
int pmts_pd_info_get(pmts_pd* h, pmts_pd_info* info);

/* initial_acceleration (newmark.hpp:110-116): a0 = (P scale0 - K u0) / M. */
int pmts_pd_init(pmts_pd* h, double scale0);
/* n fused fine steps: per step k, p_t = P_ext * load_scale[k]; explicit
 * Newmark step (advance_dynamic_step, newmark.hpp:185-190 / 122-159);
 * inclusive break test s >= s_crit on the new displacement
 * (update_bond_states, perifem.hpp:170-193; the K downdate of
 * perifem.hpp:356-364 is implicit in the matrix-free force).
 * n_broken_out (optional): bonds newly broken over the n steps. */
int pmts_pd_step(pmts_pd* h, int32_t n, const double* load_scale, int64_t* n_broken_out);
/* n fine steps that also report, per step, the displacement of n_tracked dofs
 * (the tracked points run_built records every step, driver_run.hpp:204-208,241)
 * into tracked_out[n][n_tracked] and the bonds broken in that step into
 * broken_out[n].  Per step, asynchronously on the handle's stream: the step's
 * load scale host->device (pinned staging), the step, and the step's tracked
 * row and broken count device->host; one synchronisation per call.  Pass
 * pinned (page-locked) tracked_out for the copies to overlap the steps. */
int pmts_pd_step_tracked(pmts_pd* h, int32_t n, const double* load_scale, int32_t n_tracked,
                         const int32_t* dofs, double* tracked_out, int64_t* broken_out);
/* Same as pmts_pd_step, timed on the handle's stream with CUDA events (device ms). */
int pmts_pd_step_timed(pmts_pd* h, int32_t n, const double* load_scale, float* ms_out);
/* Per-kernel device time of the dominant (bond) kernel over n steps, with
 * CUDA events around each of its launches (ms summed) -- roofline input. */
int pmts_pd_profile(pmts_pd* h, int32_t n, const double* load_scale, float* bond_ms,
                    float* total_ms);

int pmts_pd_get_state(pmts_pd* h, double* u, double* v, double* a);
int pmts_pd_set_state(pmts_pd* h, const double* u, const double* v, const double* a);
/* Intact flag per pair of pmts_pd_get_pairs order (1 intact, 0 broken). */
int pmts_pd_get_intact(pmts_pd* h, uint8_t* intact_out, int64_t cap);
/* Break log: (step, i, j) rows of bonds broken since the last call, sorted by
 * (step, i, j) -- the (pe, qp) order of update_bond_states.  Steps count from
 * the handle's creation (1-based). */
int pmts_pd_take_break_log(pmts_pd* h, int32_t* rows_out, int64_t cap, int64_t* n_out);
int64_t pmts_pd_broken_total(pmts_pd* h);
/* damage_field (perifem.hpp:202-231). */
int pmts_pd_damage(pmts_pd* h, double* elem_out, double* node_out);
/* Gather a few dofs of the current displacement (tracked points,
 * driver_run.hpp:41-47) into host memory. */
int pmts_pd_gather_disp(pmts_pd* h, int32_t n, const int32_t* dofs, double* out);
/* cudaStream_t of the handle (as void*) for callers that time on it. */
void* pmts_pd_stream(pmts_pd* h);

/* ------------------------------------------------------------------------
 * Slab decomposition.  A rank's handle holds its slab plus a
 * halo of whole node rows (2D) / layers (3D); after every fine step the
 * predictor displacement of the boundary node rows goes to the neighbours.
 * Node ranges are contiguous local node ids.
 * ------------------------------------------------------------------------ */
/* host <-> device copy of the predictor displacement rd of nodes [first, first+n)
 * (host-mediated exchange; also the single-GPU emulation of several ranks) */
int pmts_pd_get_rows(pmts_pd* h, int32_t first_node, int32_t n_nodes, double* out);
int pmts_pd_set_rows(pmts_pd* h, int32_t first_node, int32_t n_nodes, const double* in);
/* the same over n_layers ranges [first + l stride, + n) (3D slabs cut along y: one
 * range per z node layer), packed layer after layer */
int pmts_pd_get_rows_layers(pmts_pd* h, int32_t first_node, int32_t n_nodes, int32_t n_layers,
                            int32_t layer_stride, double* out);
int pmts_pd_set_rows_layers(pmts_pd* h, int32_t first_node, int32_t n_nodes, int32_t n_layers,
                            int32_t layer_stride, const double* in);
/* NCCL (loaded at run time): unique id of a new clique (128 bytes) */
int pmts_nccl_unique_id(void* id_out);
/* join the clique; then each fine step ends with ncclSend/ncclRecv of the halo rows
 * to/from the lower (peer_lo) and upper (peer_hi) neighbour, -1 = none */
int pmts_pd_comm_init(pmts_pd* h, const void* id, int32_t nranks, int32_t rank);
int pmts_pd_set_halo(pmts_pd* h, int32_t peer_lo, int32_t send_lo_first, int32_t recv_lo_first,
                     int32_t n_lo, int32_t peer_hi, int32_t send_hi_first,
                     int32_t recv_hi_first, int32_t n_hi);
/* after pmts_pd_set_halo: every halo range repeats over n_layers z node layers,
 * layer_stride nodes apart (3D slabs cut along y); the library packs them into one
 * contiguous message per neighbour (a pack / unpack kernel around the NCCL group) */
int pmts_pd_set_halo_layers(pmts_pd* h, int32_t n_layers, int32_t layer_stride);

/* Run-time options of a handle (any time between steps).  All of them leave the
 * results bitwise unchanged (tests/test_gpu_parity.py screen tests,
 * test_tile9_split_launch_bitwise); they exist for those tests and diagnostics. */
enum pmts_option {
    PMTS_OPT_BREAK_SCREEN = 1,   /* 1 (default): skip the break test on tiles the
                                    node-step bound proves cold; 0: test every tile */
    PMTS_OPT_HALO_OVERLAP = 2,   /* 2D slabs: 1 = edge tile rows first, the NCCL halo on
                                    a second stream under the interior rows (default 0;
                                    without peers it splits the launch anyway) */
    PMTS_OPT_COUNT_HOT = 3,      /* 1: count hot / tested tiles (pmts_pd_info) */
    PMTS_OPT_CLEAN_TILES = 4,    /* 1 (default): 2D tile kernel -- tiles whose bonds are all
                                    intact (and whose neighbours' are) neither stage nor
                                    re-write their bond states; 0: every tile does */
};
int pmts_pd_set_option(pmts_pd* h, int32_t option, int32_t value);

/* ------------------------------------------------------------------------
 * Coupled-integrator hooks (deterministic mode): the PD side of a
 * reference CoupledIntegrator (mts.hpp:79-535) that keeps its own FE side.
 * ------------------------------------------------------------------------ */
/* G_PD^T S_j of free_solve_pd (mts.hpp:160-162): vals at dofs added to P * load_scale in
 * every following step (and pmts_pd_init) until replaced; n = 0 clears it */
int pmts_pd_set_constraint_load(pmts_pd* h, int32_t n, const int32_t* dofs, const double* vals);
/* k_sync_ = the live bond states (mts.hpp:98, 252): the mask the recursion uses */
int pmts_pd_snapshot_bonds(pmts_pd* h);
/* the m homogeneous linear substeps from rest on k_sync_ (unit_pd_column / apply_h_pd /
 * recombine, mts.hpp:230-238, 398-420): load w[r] j / m at dofs[r] in substep j.
 * vel_out (nullable, (m + 1) x n rows): the velocities at the dofs after each substep
 * (row 0 = 0); u/v/a_out (nullable, n_dof): the final state y_m.  The handle's own
 * state is untouched. */
int pmts_pd_homogeneous_recursion(pmts_pd* h, int32_t m, int32_t n, const int32_t* dofs,
                                  const double* w, double* vel_out, double* u_out, double* v_out,
                                  double* a_out);
/* sum of an int64 over the clique (broken counts at output cadence) */
int pmts_pd_allreduce_sum(pmts_pd* h, int64_t* value);

/* ------------------------------------------------------------------------
 * Coupled multi-time-step (Arlequin) integrator -- SURVEY.md 8(f) row 1.
 * The reference's coupled run: build_scenario's coupled part
 * (driver.hpp:211-222), assemble_global (fem.hpp:421-474), find_pe_pairs over
 * the PD-active elements (mesh.hpp:416-495), assemble_pd_global with (1-alpha)
 * weights (perifem.hpp:276-351), build_coupling_map (coupling.hpp:72-105) and
 * CoupledIntegrator (mts.hpp:79-535).  FE and PD states, the unit responses
 * and the Lagrange multipliers live on the device; the dense interface factor
 * (n_lambda <= 400, or run.interface = dense) is solved on the host exactly as
 * DenseLu does (linalg.hpp:368-412).  Explicit PD substeps only (beta_pd = 0,
 * the BASELINE configs); the FE side may be explicit or implicit (PCG).
 * ------------------------------------------------------------------------ */
typedef struct pmts_mts pmts_mts;

typedef struct {
    const pmts_scenario_desc* scenario; /* mesh, material, [pd], loads, [time]; its
                                           gamma/beta are the PD Newmark parameters.
                                           Tractions stay surface loads (no bands). */
    int32_t n_pd_box;            /* [region] pd_box<k>: lo[3] hi[3] per box */
    const double* pd_boxes;
    double overlap_width_factor; /* region.overlap_width_factor */
    int32_t weight_kind;         /* 0 constant, 1 linear, 2 cubic (coupling.hpp:14-21) */
    double gamma_fe, beta_fe;    /* time.gamma_fe / beta_fe */
    int32_t interface_mode;      /* 0 auto, 1 dense, 2 matrix_free (mts.hpp:27) */
    int32_t enforce_continuity;  /* run.enforce_continuity */
    int32_t track_energy;        /* output.energy */
    int32_t device;              /* CUDA ordinal */
    double fe_spacing;           /* > 0: non-matching FE lattice of this spacing over the
                                    domain, PD lattice (scenario spacing) over the PD boxes'
                                    hull, coupling rows interpolating the FE velocity at the
                                    PD overlap nodes (extension); 0: the
                                    reference's single conforming mesh */
    int32_t interface_precond;   /* matrix-free interface CG: 0 = the reference's plain CG
                                    (mts.hpp:194-213, default); 1 = Jacobi-preconditioned with
                                    diag(H_FE) + m dt / (2 M_PD) (an addition) */
    int32_t interface_recursion; /* matrix-free interface: 1 = G_PD vel(Y_PD) w by the m-substep
                                    recursion in every CG iteration (apply_h_pd, mts.hpp:410-420);
                                    0 (default) = that operator precomputed once as an exact
                                    sparse matrix (coloured simultaneous unit loads), used until
                                    bonds break */
    int32_t shard_world;         /* > 1: a sharded coupled run (north star item 5): this handle
                                    is PD shard shard_rank of shard_world -- slabs of PD element
                                    layers along the slowest lattice axis with one-horizon ghost
                                    layers exchanged every fine substep; shard 0 also holds the
                                    FE side; the interface solve runs on every shard.  Join the
                                    shards with pmts_mts_group_join (one process) or
                                    pmts_mts_comm_init (NCCL, one process per GPU), then
                                    pmts_mts_init / pmts_mts_group_init.  0 or 1: one domain */
    int32_t shard_rank;
    int32_t interface_h_fe;      /* matrix-free interface with an explicit FE side: 0 (default)
                                    = H_FE as a direct sparse product, bitwise the unit
                                    columns, no n_lambda^2 scratch; 1 = the unit columns
                                    (unit_fe_column, mts.hpp:389-397) through the scratch */
    int32_t pd_linear;           /* linear PD force of the homogeneous substeps (unit, link and
                                    interface solves, mts.hpp:230-238, 398-420): 0 (default) =
                                    on a 3D box lattice with the 122-offset stencil the tile
                                    kernel of pd_mts_lat.cu (coefficients in stencil order,
                                    ubar apron in shared memory), else the ELL form; 1 = the
                                    ELL form everywhere (the two differ by rounding only) */
    int32_t pd_elem_products;    /* free PD substeps (free_solve_pd, mts.hpp:152-180): the
                                    per-element node products Nsh u_a and their sum formed once
                                    per force call instead of once per family entry (bitwise
                                    the same force): 0 = from 2^18 PD elements on, 1 = always,
                                    2 = never */
} pmts_mts_desc;

typedef struct {
    int32_t dim, n_nodes, n_elems, fe_n_dof, pd_n_dof, n_lambda, dense, m, n_macro;
    int32_t fe_nnz, fe_n_bc, pd_n_bc, n_pd_elems;
    int64_t n_pairs;
    double dt_pd, delta, c0, l, char_length, load_ramp;
    const int32_t* labels;       /* per element: 0 FE_only, 1 PD_only, 2 Overlap */
    const double* alpha;         /* per element blend weight */
    const int32_t* fe_node_dof;  /* per node: first FE dof or -1 */
    const int32_t* pd_node_dof;
    const int32_t* fe_k_rowptr;  /* FE stiffness, CSR (from_triplets order) */
    const int32_t* fe_k_col;
    const double* fe_k_val;
    const double* fe_mass;
    const double* fe_p_ext;
    const double* pd_mass;
    const double* pd_p_ext;
    const int32_t* fe_bc_dofs;
    const double* fe_bc_vel;
    const int32_t* pd_bc_dofs;
    const double* pd_bc_vel;
    const int32_t* cpl_fe_dof;   /* coupling rows (node, component) ascending */
    const int32_t* cpl_pd_dof;
    const int32_t* pairs;        /* [n_pairs][2] global element ids, find_pe_pairs order */
    const double* pe_weight;     /* [n_pairs] 1 - alpha at the bond midpoint */
    const double* node_xyz;      /* [n_nodes][3] */
    const int32_t* elem_nodes;   /* [n_elems][2^dim] */
    const double* node_alpha;    /* [n_nodes] blend weight at the node (output sampling,
                                    driver_run.hpp:24-35) */
    /* G_FE rows as CSR (one weight-1 entry per row on a conforming mesh) */
    int64_t cpl_fe_nnz;
    const int32_t* cpl_fe_rowptr;  /* [n_lambda + 1] */
    const int32_t* cpl_fe_col;     /* FE dofs */
    const double* cpl_fe_w;        /* shape-function weights */
    /* non-matching meshes: elements [0, fe_mesh_elems) / nodes [0, fe_mesh_nodes) are
       the FE lattice, the rest the PD lattice; -1 on a conforming mesh */
    int32_t fe_mesh_elems, fe_mesh_nodes;
    int32_t pd_linear_lattice;   /* 1: the homogeneous substeps' linear PD force runs on the
                                    lattice tile kernel (pmts_mts_desc.pd_linear) */
} pmts_mts_view;

typedef struct {                 /* MacroReport (mts.hpp:41-63) */
    double t_kinematic, t_update, t_lambda, t_unit;
    double quad_fe, quad_pd, lambda_fe, lambda_pd;
    double continuity;
    int32_t newly_broken, interface_iterations;
} pmts_mts_report;

int pmts_mts_create(const pmts_mts_desc* desc, pmts_mts** out);
int pmts_mts_view_get(const pmts_mts* h, pmts_mts_view* view);
/* CoupledIntegrator::initialize_accelerations (mts.hpp:133-140) */
int pmts_mts_init(pmts_mts* h);
/* n macro steps (mts.hpp:244-306); reports (optional) receives n records */
int pmts_mts_macro_step(pmts_mts* h, int32_t n, pmts_mts_report* reports);
/* device time of n macro steps (CUDA events around the whole sequence, host
 * orchestration and host-side interface solves included) */
int pmts_mts_macro_step_timed(pmts_mts* h, int32_t n, float* ms_out);
/* which: 0 FE, 1 PD; (u, v, a) in that subdomain's dof order (nullable) */
int pmts_mts_get_state(pmts_mts* h, int32_t which, double* u, double* v, double* a);
int pmts_mts_get_lambda(pmts_mts* h, double* lambda_out);
/* per pair (pmts_mts_view.pairs order): 1 intact, 0 broken */
int pmts_mts_get_intact(pmts_mts* h, uint8_t* out);
/* damage_field (perifem.hpp:202-231) over the whole mesh: elem_out[n_elems],
 * node_out[n_nodes]; elements without bonds (FE-only) read 0 and are left out of
 * the nodal averages, as in the reference's coupled frames (driver_run.hpp:143-146) */
int pmts_mts_damage(pmts_mts* h, double* elem_out, double* node_out);
void pmts_mts_destroy(pmts_mts* h);

/* ---- sharded coupled runs (pmts_mts_desc.shard_world > 1) ---- */
typedef struct {
    int32_t world, rank, axis;        /* cut axis: the slowest lattice axis (1 in 2D, 2 in 3D) */
    int32_t reach_layers, n_layers;   /* D = floor(delta / h); PD element layers along the axis */
    int32_t n_local_nodes, n_local_elems;
    int32_t own_elem_lo, own_elem_hi; /* the owned local elements */
    const int32_t* local_nodes;       /* local node -> compact PD node (its PD dofs: * dim + c);
                                         pmts_mts_get_state(1) is in this local order */
    const int32_t* local_elems;       /* local element -> PD-active element index */
    const uint8_t* node_owned;        /* per local node */
    const int32_t* layer_bounds;      /* [world + 1] element-layer bounds of the shards */
} pmts_mts_shard_view;
int pmts_mts_shard_view_get(const pmts_mts* h, pmts_mts_shard_view* view);
/* one process drives all shards (tests, single-node emulation): join them, then
 * initialize and step them together -- one host thread per shard, host barriers and
 * device copies between the shards' buffers at every exchange; reports: shard 0's */
int pmts_mts_group_join(pmts_mts* const* handles, int32_t n);
int pmts_mts_group_init(pmts_mts* const* handles, int32_t n);
int pmts_mts_group_macro_step(pmts_mts* const* handles, int32_t n, int32_t steps,
                              pmts_mts_report* reports);
/* one process per GPU: join the NCCL clique (pmts_nccl_unique_id from shard 0); then
 * pmts_mts_init / pmts_mts_macro_step on every rank in lockstep */
int pmts_mts_comm_init(pmts_mts* h, const void* nccl_unique_id);

#ifdef __cplusplus
}
#endif
#endif
