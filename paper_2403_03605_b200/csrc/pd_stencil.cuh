// Lattice-stencil family encoding (fast mode) -- see pd_stencil.cu.
#pragma once

#include <cuda.h>

#include "pd_common.cuh"

namespace pmts {

constexpr int kMaxStencil = 128;

struct LatticeDev {
    int nx, ny, nz;      // elements per axis
    int R;               // max |offset component|
    int S;               // stencil size
    int W;               // mask words per element (S <= 32 W)
    const int8_t* di;    // per offset (device)
    const int8_t* dj;
    const int8_t* dk;
    const int* delta_id; // linear element-id delta of each offset
    const double* table; // per offset, 8 doubles (layout in pd_stencil.cu)
    const uint8_t* nflag;     // per node: bit c = dof c constrained, bit 3 = loaded
    const double* inv_mass;   // per node: 1 / M (lumped mass is per node)
    // slab rows (pmts_pd_desc.node_rows; full range for one domain): the node update
    // runs on the y node rows [jn0, jn1) only, the 3D bond kernel on the element rows
    // [jb0, jb1) their forces need; ub0 / ugy: first y row and row tiles of the 3D
    // ubar grid (its tiles align with the bond tiles, pd_lat3.cu)
    int jn0 = 0, jn1 = 0, jb0 = 0, jb1 = 0, ub0 = 0, ugy = 0;
};

constexpr int kTableRow = 8;

// Fused single-kernel 2D step (pd_tile9.cu) for the 28-offset stencil; per-offset
// constants travel in the kernel's parameter space.
constexpr int kFusedS = 28;  // delta in [3, sqrt(10)) dx: the paper's / BASELINE's 3.015 dx
constexpr int kFusedR = 3;
constexpr int kFusedTX = 31;  // owned elements per tile row; force region 32 wide
constexpr int kFusedAX = kFusedTX + 1 + 2 * kFusedR;
struct Stencil2D {
    double xi0[kFusedS], xi1[kFusedS];    // representative xi of the offset
    double fx0[kFusedS], fx1[kFusedS];    // w c(|xi|) xi
    double cthr[kFusedS], clo[kFusedS], x2[kFusedS];
    int aoff[kFusedS];  // partner offset inside the shared ubar apron (dj * AX + di)
    int did[kFusedS];   // partner element-id delta
};

struct FusedBufs {
    const double* rd_in;
    double* rd_out;
    const uint32_t* mask_in;
    uint32_t* mask_out;
    const double* scale_dev = nullptr;  // tile9: per-step load scales copied H2D (or null)
    // tile9, pmts_pd_step_tracked: one block copies the tracked dofs of the step's
    // displacement straight into mapped pinned host memory (a separate kernel
    // instance; n_trk = 0: none)
    const int32_t* trk_dofs = nullptr;
    int n_trk = 0;
    double* trk_host = nullptr;  // this step's row (n_trk values)
    // tile9: per tile 1 = every owned element has its full positive stencil intact in
    // BOTH bond-state buffers (so the words need neither staging nor re-writing); a
    // tile that breaks a bond clears its flag for good (null: stage on every tile)
    uint32_t* tclean = nullptr;
};


// One-shot TMA-staged variant (pd_tile9.cu): tensor maps of the current rd
// ([NY][2 NX] doubles), rv, and {1/M | flags} ([NY][NXP] doubles, NXP even,
// flags in the three low mantissa bits).
struct Tile9Maps {
    CUtensorMap rd, rv, im;
    int prefetch_ahead;  // > 0: each CTA prefetches into L2 the boxes of tile id + this
    int row_base = 0;    // first tile row of this launch (set by launch_tile9_step)
    int grid_rows = 0;   // tile rows of the whole lattice
};
void tile9_boxes(int* rd_x, int* rd_y, int* rv_x, int* rv_y, int* im_x, int* im_y);
// Pair-symmetric force constants of the 14 positive offsets of the 28-offset
// stencil on the nominal lattice (xi = h o), in pd_tile9.cu's pair order
// (1,0) (2,0) (3,0) (0,1) (0,2) (0,3) (1,1) (-1,1) (2,2) (-2,2) (2,1) (-2,1)
// (1,2) (-1,2): G += fa t e_x + fb t e_y with t = o . (eta_o + eta_-o) (axis
// pairs: fa = F A^2 with t = s_x, resp. fb = F B^2), F = -w c(h|o|) h^2; cl = bit
// pattern of the smallest threshold of the offset's class, lowered by 1e-12.
struct PairStencil2D {
    double fa[14], fb[14];
    long long cl[14];
    int off[14];   // apron offset of o (dj * 38 + di)
    int pbit[14];  // mask bit of the positive offset o
    double h2;    // 2 h
    float h2f;       // fp32-position variant: 2 h and the candidate thresholds
    float clf[14];   // (cl lowered by 1e-4, rounded down to fp32)
    int screen;   // 1: skip the candidate break pass on tiles the node-step bound
                  // proves cold (pd_tile9.cu); results are bitwise the same
    unsigned long long* hot_count;  // diagnostics (PMTS_T9_COUNT_HOT): [0] hot, [1] all tiles
};
int tile9_pair_offset(int k, int* a, int* b);
int tile9_configure();  // returns resident CTAs per SM
void launch_tile9_step(const DevPD& d, const LatticeDev& L, const Stencil2D& st,
                       const PairStencil2D* ps, const Tile9Maps& maps, const FusedBufs& b,
                       int step, int do_break, double scale, int write_state, bool f32,
                       cudaStream_t s, int row_first = 0, int row_end = -1);
int tile9_rows(const LatticeDev& L);  // tile rows of the grid (node rows j0 = 31 r ...)
int tile9_cols(const LatticeDev& L);
// the clean-tile flags of the current bond states; also copies mask -> mask_alt so both
// ping-pong buffers hold every word
void launch_tile9_flags(const LatticeDev& L, const uint32_t* mask, uint32_t* mask_alt,
                        uint32_t* tclean, cudaStream_t s);
int tile9_tile_rows();                // element rows per tile (31)

// 3D 122-offset bond kernel on the nominal lattice (pd_lat3.cu): per |o|^2 class
// (1,2,3,4,5,6,8,9): c = w c(h|o|) h^2, and the bit patterns of the smallest /
// scalar thresholds (2 s + s^2) h^2 |o|^2.
struct Stencil3D {
    CUtensorMap ub;  // ubar as [nz][ny][3 nx] doubles (use_tma: nx even)
    int use_tma;
    double c[8];
    long long clo[8], cthr[8];
    double h2;  // 2 h
    double hh;  // h^2
    // cold-tile break screen (pd_lat3.cu): per-tile node-edge maxima written by
    // k_lat3_ubar (null: no screen); diagnostics (hot / all tiles)
    const unsigned* tmax;
    unsigned long long* hot_count;
};
bool lat3_offsets_match(const int8_t* di, const int8_t* dj, const int8_t* dk, int S);
int lat3_class_of(int d2);
void launch_lat3_bond(const DevPD& d, const LatticeDev& L, const Stencil3D& st, int step,
                      int do_break, cudaStream_t s);
void launch_lat3_ubar(const DevPD& d, const LatticeDev& L, unsigned* tmax, cudaStream_t s);
void lat3_rows(LatticeDev& L);  // ub0 / ugy from jb0 (call before lat3_tile_count)
// damage_field (perifem.hpp:202-231) over the stencil bits (present = the encoded
// mask: the bonds that exist); the intact state of every bond (i < j) in the pair
// order (ascending i, then j) into out_dev (null: count only); returns the bonds
void launch_lat_damage(const DevPD& d, const LatticeDev& L, const uint32_t* present, bool pos_only,
                       double* elem, double* node, cudaStream_t s);
long long launch_lat_intact(const DevPD& d, const LatticeDev& L, const uint32_t* present,
                            uint8_t* out_dev, cudaStream_t s);
size_t lat3_tile_count(const LatticeDev& L);
void lat3_apron_box(int* bx, int* by, int* bz);  // TMA box of the ubar apron (doubles, rows, layers)

// device lattice encoding (setup): offsets present as 17^3 flags (component + 8),
// returns the largest |component| (> 8: not encodable); then the intact mask of
// every element from the host-ordered slot table, returns the entry count F
int lattice_scan_device(const int32_t* d_col, int E, int K, int nx, int ny, int* present17,
                        cudaStream_t s);
long long lattice_mask_device(const int32_t* d_col, int E, int K, int nx, int ny,
                              const int* slot17, int W, uint32_t* d_mask, cudaStream_t s);
size_t lattice_smem_bytes(int dim, int R, int S);
void lattice_configure(int dim, int R, int S);
struct Stencil3D;
void launch_lattice_step(const DevPD& d, const LatticeDev& L, int step, int do_break,
                         double scale, int write_state, bool time_bond, cudaEvent_t* ev,
                         cudaStream_t s, const Stencil3D* st3 = nullptr);

}  // namespace pmts
