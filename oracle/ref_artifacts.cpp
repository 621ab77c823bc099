// ORACLE / TEST INFRASTRUCTURE ONLY -- not product code.
//
// The reference's own run-with-artifacts and compare, from its UNMODIFIED
// headers (compiled in place by oracle/Makefile, nothing copied):
//   ref_artifacts run CFG OUTDIR [--override sec.key=val]...
//       run_scenario (driver.hpp:264-266 -> run_built + finalize_outputs)
//   ref_artifacts compare DIR_A DIR_B
//       compare_runs (driver.hpp:290-368): tracked-point global error and the
//       damage agreement of matching frames, printed as one JSON line
// so tests can score the device runs' artifacts (paper_2403_03605_b200/
// artifacts.py) with the reference's own comparison.
#include "perimts/driver.hpp"

#include <cstdio>
#include <string>
#include <vector>

using namespace perimts;

int main(int argc, char** argv) {
    if (argc < 4) {
        std::fprintf(stderr, "usage: ref_artifacts run CFG OUTDIR [--override k=v]... | "
                             "compare DIR_A DIR_B\n");
        return 2;
    }
    try {
        const std::string cmd = argv[1];
        if (cmd == "run") {
            Config cfg = Config::parse_file(argv[2]);
            for (int a = 4; a + 1 < argc; a += 2)
                if (std::string(argv[a]) == "--override") cfg.apply_override(argv[a + 1]);
            const ScenarioConfig sc = load_scenario(cfg);
            const RunArtifacts art = run_scenario(sc, argv[3]);
            std::printf("{\"steps\": %d, \"broken\": %lld, \"frames\": %zu}\n", art.steps,
                        art.broken_total, art.frame_times.size());
            return 0;
        }
        if (cmd == "compare") {
            const CompareReport rep = compare_runs(argv[2], argv[3]);
            std::printf("{\"tracked_error_pct\": [");
            for (std::size_t p = 0; p < rep.tracked_error_pct.size(); ++p)
                std::printf("%s%.17g", p ? ", " : "", rep.tracked_error_pct[p]);
            std::printf("], \"has_damage_frames\": %s, \"min_damage_agreement\": %.17g, "
                        "\"frames_compared\": %zu, \"step_cost_ratio\": %.17g}\n",
                        rep.has_damage_frames ? "true" : "false", rep.min_damage_agreement,
                        rep.damage_agreement.size(), rep.step_cost_ratio);
            return 0;
        }
        std::fprintf(stderr, "unknown command %s\n", cmd.c_str());
        return 2;
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
}
