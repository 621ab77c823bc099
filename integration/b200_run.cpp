// The reference-side drop-in, compiled: run_built's pure-PD branch
// (/root/reference/proj/include/perimts/driver_run.hpp:160-246) with the fine
// step -- advance_dynamic_step + update_bond_states + incremental_stiffness_update
// (:214-236) and damage_field for the frames (:142-158) -- on the B200 through
// include/pmts_capi.h.  Everything else is the reference's own code, called from
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
        const RunArtifacts art = b200::run_built_pure_pd(b, argv[2], mode, device_families);
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
