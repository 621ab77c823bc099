// Lattice-stencil family encoding (fast mode) -- see pd_stencil.cu.
#pragma once

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
};

constexpr int kTableRow = 8;

size_t lattice_smem_bytes(int dim, int R, int S);
void lattice_configure(int dim, int R, int S);
void launch_lattice_step(const DevPD& d, const LatticeDev& L, int step, int do_break,
                         double scale, int write_state, bool time_bond, cudaEvent_t* ev,
                         cudaStream_t s);

}  // namespace pmts
