// The reference-side drop-in, compiled: run_built's pure-PD branch
// (/root/reference/proj/include/perimts/driver_run.hpp:160-246) with the fine
// step -- advance_dynamic_step + update_bond_states + incremental_stiffness_update
// (:214-236) and damage_field for the frames (:142-158) -- on the B200 through
// include/pmts_capi.h; and its coupled branch (:247-295) with the CoupledIntegrator
// on the device (pmts_mts_*).  Everything else is the reference's own code, called from
// its unmodified headers (nothing is copied): build_scenario, find_pe_pairs,
// build_peri_elements, assemble_pd_global (M, P_ext), resolve_bcs_quiet, the
// tracked-point sampler, the frame writer and finalize_outputs.  The artifacts it
// writes are therefore the reference's format, and the reference's own
// compare_runs scores them (tests/test_integration_shim.py).
//
//   b200_run CFG OUTDIR [--mode det|fast] [--device-families] [--override sec.key=val]...
//
// This is the change INTEGRATION.md describes, as a maintainer would make it;
// it is built by integration/Makefile against the reference headers when they
// are present and linked to paper_2403_03605_b200/lib/libpmts.so.
#include "perimts/driver.hpp"
#include "pmts_capi.h"

#include <cstdio>
#include <string>
#include <vector>

using namespace perimts;

namespace b200 {

// the reference's exception types back from the C status codes (errors.hpp:8-21)
void check(int st) {
    if (st == PMTS_OK) return;
    const std::string msg = pmts_last_error();
    if (st == PMTS_ERR_CONFIG) throw ConfigError(msg);
    if (st == PMTS_ERR_SOLVER) throw SolverError(msg);
    throw InternalError(msg);
}

struct Handle {
    pmts_pd* h = nullptr;
    ~Handle() {
        if (h) pmts_pd_destroy(h);
    }
};

// run_built (driver_run.hpp:160-246) for run.mode = pure_pd, the step loop on the device
RunArtifacts run_built_pure_pd(BuiltScenario& b, const std::string& out_dir, int mode,
                               bool device_families) {
    if (b.sc.mode != RunMode::pure_pd) throw ConfigError("b200_run: run.mode = pure_pd only");
    if (b.sc.pe_quadrature != 1) throw ConfigError("b200_run: one-point PE quadrature only");
    RunArtifacts art;
    art.mesh_hash = mesh_hash(b.mesh);
    art.dim = b.mesh.dim;
    art.n_nodes = b.mesh.node_count();
    art.n_elements = b.mesh.element_count();
    art.n_tracked = static_cast<int>(b.tracked_nodes.size());
    if (!out_dir.empty()) std::filesystem::create_directories(out_dir);
    const Mesh& mesh = b.mesh;
    detail::FrameWriter frames(b, out_dir, art);

    // setup: the reference's own (driver_run.hpp:161-184)
    std::vector<int> active(mesh.element_count());
    for (int e = 0; e < mesh.element_count(); ++e) active[e] = e;
    const std::vector<double> alpha_field(mesh.element_count(), 0.0);
    const auto pairs = find_pe_pairs(mesh, b.pd_mat.delta, b.sc.notches);
    const std::vector<PeriElement> pes = build_peri_elements(mesh, pairs, b.sc.pe_quadrature);
    const PdSystem pd_sys = assemble_pd_global(mesh, active, alpha_field,
                                               [](const Point&) { return 0.0; }, pes, b.pd_mat,
                                               b.sc.material, b.loads);
    NewmarkParams nm = b.sc.pd_nm;
    nm.dt = b.sc.dt_pd;
    const BcTable bcs = detail::resolve_bcs_quiet(mesh, pd_sys.dofs, b.loads);

    // the device handle (pmts_pd_create replaces the BlockOperator ctor's checks)
    const int dim = mesh.dim, nn = dim == 2 ? 4 : 8;
    std::vector<double> xyz;
    std::vector<int32_t> conn;
    for (const auto& p : mesh.nodes) xyz.insert(xyz.end(), p.begin(), p.end());
    for (const auto& e : mesh.elements)
        conn.insert(conn.end(), e.node_ids.begin(), e.node_ids.begin() + nn);
    pmts_pd_desc d{};
    d.dim = dim;
    d.n_nodes = mesh.node_count();
    d.n_elems = mesh.element_count();
    d.node_xyz = xyz.data();
    d.elem_nodes = conn.data();
    d.mass = pd_sys.M.data();
    d.p_ext = pd_sys.P_ext.data();
    d.n_bc = static_cast<int32_t>(bcs.dofs.size());
    d.bc_dofs = bcs.dofs.data();
    d.bc_vel = bcs.velocity.data();
    d.delta = b.pd_mat.delta;
    d.micromodulus = PMTS_MICRO_EXP;
    d.c0 = b.pd_mat.c0;
    d.l = b.pd_mat.l;
    d.s_crit = b.pd_mat.fracture_enabled() ? b.pd_mat.s_crit : 0.0;
    d.gamma = nm.gamma;
    d.beta = nm.beta;
    d.dt = nm.dt;
    d.mode = mode;
    std::vector<int32_t> npts;
    std::vector<double> pts;
    for (const auto& n : b.sc.notches) {
        npts.push_back(static_cast<int32_t>(n.points.size()));
        for (const auto& p : n.points) pts.insert(pts.end(), p.begin(), p.end());
    }
    d.n_notch = static_cast<int32_t>(npts.size());
    d.notch_npts = npts.data();
    d.notch_pts = pts.data();
    Handle hd;
    check(pmts_pd_create(&d, &hd.h));
    pmts_pd* h = hd.h;
    if (device_families) {
        check(pmts_pd_build_families(h));  // find_pe_pairs on the device (same pairs)
    } else {
        std::vector<int32_t> pr;  // the reference's own pair list
        for (const auto& p : pairs) {
            pr.push_back(p.i);
            pr.push_back(p.j);
        }
        check(pmts_pd_set_pairs(h, static_cast<int64_t>(pairs.size()), pr.data()));
    }
    // initial state (driver_run.hpp:195-201): prescribed velocities, a0 on the device
    KinematicState state = KinematicState::zero(pd_sys.dofs.n_dof);
    for (std::size_t c = 0; c < bcs.dofs.size(); ++c) state.vel[bcs.dofs[c]] = bcs.velocity[c];
    check(pmts_pd_set_state(h, state.disp.data(), state.vel.data(), state.acc.data()));
    check(pmts_pd_init(h, b.load_scale(0.0)));
    check(pmts_pd_get_state(h, state.disp.data(), state.vel.data(), state.acc.data()));

    // frames: the reference's field sampler and writer, damage_field on the device
    detail::NodalFieldSampler sampler{b, nullptr, &pd_sys.dofs};
    std::vector<double> dmg_e(mesh.element_count()), dmg_n(mesh.node_count());
    auto fields = [&]() {
        VtkFields f;
        sampler.fill(nullptr, &state, f);
        f.subdomain_label.assign(mesh.element_count(), 1);
        f.alpha = alpha_field;
        check(pmts_pd_damage(h, dmg_e.data(), dmg_n.data()));
        f.damage = dmg_e;
        f.damage_avg = dmg_n;
        return f;
    };
    std::vector<int32_t> trk;  // dofs of the tracked points (NodalFieldSampler::tracked_row)
    for (int node : b.tracked_nodes)
        for (int c = 0; c < dim; ++c) trk.push_back(pd_sys.dofs.dof(node, c));
    auto record = [&](double t) {
        art.tracked_times.push_back(t);
        art.tracked_values.push_back(sampler.tracked_row(nullptr, &state));
    };
    record(0.0);
    if (frames.due(0.0)) frames.emit(0.0, fields());

    // the step loop: batches of fine steps up to the next frame, one C-ABI call each;
    // per step the tracked displacements and the broken count come back
    const int n_steps = static_cast<int>(std::llround(b.sc.total_time / b.sc.dt_pd));
    int i = 1;
    while (i <= n_steps) {
        int j = i;
        while (j < n_steps && !frames.due(j * b.sc.dt_pd)) ++j;  // batch i..j
        const int n = j - i + 1;
        std::vector<double> scales(n), tv((size_t)n * trk.size());
        std::vector<int64_t> nb(n);
        for (int k = 0; k < n; ++k) scales[k] = b.load_scale((i + k) * b.sc.dt_pd);
        const auto tick = detail::wall_now();
        check(pmts_pd_step_tracked(h, n, scales.data(), static_cast<int32_t>(trk.size()),
                                   trk.data(), tv.data(), nb.data()));
        const double per_step = detail::wall_since(tick) / n;
        for (int k = 0; k < n; ++k) {
            TimingRecord timing;
            timing.t_kinematic = per_step;
            art.timing.push_back(timing);
            art.broken_per_step.push_back(static_cast<int>(nb[k]));
            art.broken_total += nb[k];
            for (std::size_t q = 0; q < trk.size(); ++q) state.disp[trk[q]] = tv[k * trk.size() + q];
            record((i + k) * b.sc.dt_pd);
        }
        const double t = j * b.sc.dt_pd;
        if (frames.due(t)) {
            check(pmts_pd_get_state(h, state.disp.data(), state.vel.data(), state.acc.data()));
            frames.emit(t, fields());
        }
        i = j + 1;
    }
    art.steps = n_steps;
    detail::finalize_outputs(b, art, out_dir, frames.frame_index);
    return art;
}

// the reference's ScenarioConfig (scenario.hpp:24-62) as the C ABI's descriptors
struct Descs {
    pmts_scenario_desc sd{};
    pmts_mts_desc md{};
    std::vector<int32_t> npts;
    std::vector<double> pts, trac, body, vel, fixed, boxes;
};
void box6(const BoundsBox& b, std::vector<double>& out) {
    for (int k = 0; k < 3; ++k) out.push_back(b.lo[k]);
    for (int k = 0; k < 3; ++k) out.push_back(b.hi[k]);
}
void fill_descs(const ScenarioConfig& sc, Descs& D) {
    if (!sc.mesh_generated) throw ConfigError("b200_run: generated meshes only");
    if (!sc.loads.pressures.empty()) throw ConfigError("b200_run: pressure loads unsupported");
    pmts_scenario_desc& d = D.sd;
    d.dim = sc.dim;
    for (int k = 0; k < 3; ++k) {
        d.lo[k] = sc.bounds.lo[k];
        d.hi[k] = sc.bounds.hi[k];
    }
    d.spacing = sc.spacing;
    d.E = sc.material.E;
    d.nu = sc.material.nu;
    d.rho = sc.material.rho;
    d.formulation = sc.material.formulation == Formulation::plane_stress   ? 0
                    : sc.material.formulation == Formulation::plane_strain ? 1
                                                                           : 2;
    d.delta_factor = sc.delta_factor;
    d.l_factor = sc.l_factor;
    d.s_crit = sc.s_crit;
    for (const auto& n : sc.notches) {
        D.npts.push_back(static_cast<int32_t>(n.points.size()));
        for (const auto& p : n.points) D.pts.insert(D.pts.end(), p.begin(), p.end());
    }
    for (const auto& t : sc.loads.tractions) {
        box6(t.box, D.trac);
        D.trac.insert(D.trac.end(), t.value.begin(), t.value.end());
    }
    for (const auto& t : sc.loads.body_patches) {
        box6(t.box, D.body);
        D.body.insert(D.body.end(), t.value.begin(), t.value.end());
    }
    for (const auto& k : sc.loads.kinematic) {
        if (k.fix_all) {
            box6(k.box, D.fixed);
        } else {
            box6(k.box, D.vel);
            D.vel.push_back(k.component);
            D.vel.push_back(k.velocity);
        }
    }
    d.n_notch = static_cast<int32_t>(D.npts.size());
    d.notch_npts = D.npts.data();
    d.notch_pts = D.pts.data();
    d.n_traction = static_cast<int32_t>(D.trac.size() / 9);
    d.traction = D.trac.data();
    d.n_body_patch = static_cast<int32_t>(D.body.size() / 9);
    d.body_patch = D.body.data();
    for (int k = 0; k < 3; ++k) d.body_force[k] = sc.loads.body_force[k];
    d.n_velocity_bc = static_cast<int32_t>(D.vel.size() / 8);
    d.velocity_bc = D.vel.data();
    d.n_fixed = static_cast<int32_t>(D.fixed.size() / 6);
    d.fixed = D.fixed.data();
    d.dt_pd = sc.dt_pd;
    d.m = sc.m;
    d.total_time = sc.total_time;
    d.load_ramp = sc.load_ramp;
    d.gamma = sc.pd_nm.gamma;
    d.beta = sc.pd_nm.beta;
    pmts_mts_desc& m = D.md;
    m.scenario = &D.sd;
    if (sc.region.pd_sector) throw ConfigError("b200_run: PD sectors unsupported");
    for (const auto& b : sc.region.pd_boxes) box6(b, D.boxes);
    m.n_pd_box = static_cast<int32_t>(sc.region.pd_boxes.size());
    m.pd_boxes = D.boxes.data();
    m.overlap_width_factor = sc.overlap_width_factor;
    m.weight_kind = static_cast<int32_t>(sc.weight_kind);
    m.gamma_fe = sc.fe_nm.gamma;
    m.beta_fe = sc.fe_nm.beta;
    m.interface_mode = static_cast<int32_t>(sc.interface_mode);
    m.enforce_continuity = sc.enforce_continuity ? 1 : 0;
    m.track_energy = sc.track_energy ? 1 : 0;
    m.device = 0;
}

struct MtsHandle {
    pmts_mts* h = nullptr;
    ~MtsHandle() {
        if (h) pmts_mts_destroy(h);
    }
};

// run_built's coupled branch (driver_run.hpp:247-295) with the whole integrator on the
// device (pmts_mts_*): the reference's own labels, blend weights, tracked-point sampler,
// frame writer and finalize_outputs around it
RunArtifacts run_built_coupled(BuiltScenario& b, const std::string& out_dir) {
    RunArtifacts art;
    art.mesh_hash = mesh_hash(b.mesh);
    art.dim = b.mesh.dim;
    art.n_nodes = b.mesh.node_count();
    art.n_elements = b.mesh.element_count();
    art.n_tracked = static_cast<int>(b.tracked_nodes.size());
    if (!out_dir.empty()) std::filesystem::create_directories(out_dir);
    const Mesh& mesh = b.mesh;
    detail::FrameWriter frames(b, out_dir, art);
    std::vector<int> label_field(mesh.element_count());
    for (int e = 0; e < mesh.element_count(); ++e)
        label_field[e] = static_cast<int>(b.labels.element_label[e]);

    Descs D;
    fill_descs(b.sc, D);
    MtsHandle hm;
    check(pmts_mts_create(&D.md, &hm.h));  // CoupledIntegrator ctor, mts.hpp:81-118
    pmts_mts* h = hm.h;
    check(pmts_mts_init(h));  // initialize_accelerations, mts.hpp:133-140
    pmts_mts_view v{};
    check(pmts_mts_view_get(h, &v));
    if (v.n_nodes != mesh.node_count() || v.n_elems != mesh.element_count())
        throw InternalError("b200_run: device mesh differs from the reference's");
    auto dofmap = [&](const int32_t* nd, int n_dof) {
        DofMap m;
        m.dim = mesh.dim;
        m.n_dof = n_dof;
        m.node_dof.assign(nd, nd + mesh.node_count());
        for (int n = 0; n < mesh.node_count(); ++n)
            if (m.node_dof[n] >= 0) m.active_nodes.push_back(n);
        return m;
    };
    const DofMap fe_dofs = dofmap(v.fe_node_dof, v.fe_n_dof);
    const DofMap pd_dofs = dofmap(v.pd_node_dof, v.pd_n_dof);
    KinematicState fe = KinematicState::zero(v.fe_n_dof), pd = KinematicState::zero(v.pd_n_dof);
    auto pull = [&]() {
        check(pmts_mts_get_state(h, 0, fe.disp.data(), fe.vel.data(), fe.acc.data()));
        check(pmts_mts_get_state(h, 1, pd.disp.data(), pd.vel.data(), pd.acc.data()));
    };
    detail::NodalFieldSampler sampler{b, &fe_dofs, &pd_dofs};
    std::vector<double> dmg_e(mesh.element_count()), dmg_n(mesh.node_count());
    auto fields = [&]() {
        VtkFields f;
        sampler.fill(&fe, &pd, f);
        f.subdomain_label = label_field;
        f.alpha = b.alpha_elem;
        check(pmts_mts_damage(h, dmg_e.data(), dmg_n.data()));  // damage_field on the device
        f.damage = dmg_e;
        f.damage_avg = dmg_n;
        return f;
    };
    auto record = [&](double t) {
        art.tracked_times.push_back(t);
        art.tracked_values.push_back(sampler.tracked_row(&fe, &pd));
    };
    pull();
    record(0.0);
    if (frames.due(0.0)) frames.emit(0.0, fields());
    const int n_macro = static_cast<int>(std::llround(b.sc.total_time / b.sc.dt_fe()));
    for (int i = 1; i <= n_macro; ++i) {
        pmts_mts_report r{};
        check(pmts_mts_macro_step(h, 1, &r));  // macro_step, mts.hpp:244-306
        const double t = i * b.sc.dt_fe();
        TimingRecord tr;
        tr.t_kinematic = r.t_kinematic;
        tr.t_update = r.t_update;
        tr.t_lambda = r.t_lambda;
        tr.t_unit = r.t_unit;
        art.timing.push_back(tr);
        EnergyRecord er;
        er.quad_fe = r.quad_fe;
        er.quad_pd = r.quad_pd;
        er.lambda_fe = r.lambda_fe;
        er.lambda_pd = r.lambda_pd;
        art.energy.push_back(er);
        art.continuity.push_back(r.continuity);
        art.broken_per_step.push_back(r.newly_broken);
        art.broken_total += r.newly_broken;
        pull();
        record(t);
        if (frames.due(t)) frames.emit(t, fields());
    }
    art.steps = n_macro;
    detail::finalize_outputs(b, art, out_dir, frames.frame_index);
    return art;
}

}  // namespace b200

int main(int argc, char** argv) {
    if (argc < 3) {
        std::fprintf(stderr, "usage: b200_run CFG OUTDIR [--mode det|fast] [--device-families] "
                             "[--override k=v]...\n");
        return 2;
    }
    int mode = PMTS_DETERMINISTIC;
    bool device_families = false;
    try {
        Config cfg = Config::parse_file(argv[1]);
        for (int a = 3; a < argc; ++a) {
            const std::string s = argv[a];
            if (s == "--mode" && a + 1 < argc) {
                const std::string m = argv[++a];
                mode = m == "fast" ? PMTS_FAST : PMTS_DETERMINISTIC;
            } else if (s == "--device-families") {
                device_families = true;
            } else if (s == "--override" && a + 1 < argc) {
                cfg.apply_override(argv[++a]);
            } else {
                throw ConfigError("unknown argument " + s);
            }
        }
        const ScenarioConfig sc = load_scenario(cfg);
        BuiltScenario b = build_scenario(sc);
        const RunArtifacts art = sc.mode == RunMode::coupled_mts
                                     ? b200::run_built_coupled(b, argv[2])
                                     : b200::run_built_pure_pd(b, argv[2], mode, device_families);
        std::printf("{\"steps\": %d, \"broken\": %lld, \"frames\": %zu}\n", art.steps,
                    art.broken_total, art.frame_times.size());
    } catch (const ConfigError& e) {
        std::fprintf(stderr, "config error: %s\n", e.what());
        return 2;
    } catch (const SolverError& e) {
        std::fprintf(stderr, "solver error: %s\n", e.what());
        return 3;
    } catch (const std::exception& e) {
        std::fprintf(stderr, "error: %s\n", e.what());
        return 1;
    }
    return 0;
}
