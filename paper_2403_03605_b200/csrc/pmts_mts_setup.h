// Host model of a coupled multi-time-step run (pmts_mts_setup.cpp).
#pragma once

#include <cstdint>
#include <vector>

#include "pmts_internal.h"

namespace pmts {

struct MtsBox {
    double lo[3] = {0, 0, 0}, hi[3] = {0, 0, 0};
};
struct MtsTraction {
    MtsBox box;
    double value[3] = {0, 0, 0};
};
struct MtsKinematic {
    MtsBox box;
    int comp = 0;
    double vel = 0.0;
    bool fix_all = false;
};

struct MtsSystem {
    // inputs (mesh, material, PD, loads, time, region)
    int dim = 2;
    int n[3] = {1, 1, 1};
    std::vector<double> nodes, centroid, volume;  // xyz per node / element
    std::vector<int32_t> conn;
    double cl = 0, delta = 0, l = 0, c0 = 0, s_crit = 0;
    double E = 0, nu = 0, rho = 0;
    int formulation = 0;
    std::vector<MtsTraction> tractions, body_patches;
    double body_force[3] = {0, 0, 0};
    std::vector<MtsKinematic> kinematic;
    std::vector<MtsBox> pd_boxes;
    double overlap_width_factor = 3.0;
    int weight_kind = 2;  // 0 constant, 1 linear, 2 cubic
    double dt_pd = 0, ramp = 0;
    int m = 1, n_macro = 0;
    double fe_gamma = 0.5, fe_beta = 0.25, pd_gamma = 0.5, pd_beta = 0.0;
    // derived
    MtsBox domain;
    double overlap_width = 0;
    std::vector<uint8_t> label;  // 0 FE_only, 1 PD_only, 2 Overlap
    std::vector<uint8_t> node_in_overlap;
    std::vector<double> alpha;
    std::vector<int> fe_active, pd_active;
    std::vector<int32_t> fe_node_dof, pd_node_dof;
    std::vector<int> fe_active_nodes, pd_active_nodes;
    int fe_n_dof = 0, pd_n_dof = 0;
    std::vector<int32_t> fe_rowptr, fe_col;
    std::vector<double> fe_val, fe_mass, fe_p_ext, pd_mass, pd_p_ext;
    std::vector<int32_t> fe_bc_dofs, pd_bc_dofs;
    std::vector<double> fe_bc_vel, pd_bc_vel;
    std::vector<int32_t> cpl_fe, cpl_pd;  // coupling rows (cpl_fe: the row's first FE dof)
    // G_FE as CSR over the rows: FE dofs and weights (one entry of weight 1 per row
    // on the reference's conforming mesh; shape-function interpolation otherwise)
    std::vector<int32_t> cpl_fe_rp, cpl_fe_ci;
    std::vector<double> cpl_fe_w;
    std::vector<double> node_alpha;       // blend weight at each node (output sampling)
    // non-matching meshes (extension): elements [0, fe_mesh_elems) and
    // nodes [0, fe_mesh_nodes) are the FE lattice (spacing fe_h), the rest the PD
    // lattice over the PD boxes' hull (spacing pd_h, fe_h / pd_h = fe_ratio); -1:
    // one conforming mesh (the reference's model)
    int fe_mesh_elems = -1, fe_mesh_nodes = -1;
    int fe_n[3] = {1, 1, 1}, pd_n[3] = {1, 1, 1}, fe_ratio = 1;
    double fe_lo[3] = {0, 0, 0}, pd_lo[3] = {0, 0, 0}, fe_h = 0, pd_h = 0;
};

// assembles everything after the inputs and the mesh geometry are filled in
void build_mts_system(MtsSystem& s);
// WeightFunction (coupling.hpp:31-40) at a point
double mts_alpha_at(const MtsSystem& s, const double* x);

}  // namespace pmts
