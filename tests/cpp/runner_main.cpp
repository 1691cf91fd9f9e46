// tests/cpp/runner_main.cpp — the reference's own batch runner
// (/root/reference/proj/include/auxamg/runner.hpp, unmodified) with a minimal
// command line in the shape of auxamg_cli.cpp:26-50 (CLI11 is absent here).
//
// Built twice by __graft_entry__.build():
//   runner_ref   the reference runner as shipped (CPU setup_hierarchy / solve)
//   runner_b200  the same runner with the drop-in switch INTEGRATION.md shows:
//                its setup_hierarchy / solve / stats / Hierarchy bind to
//                include/auxamg_b200.hpp (the B200 library through the C ABI)
// tests/test_runner.py runs both on the same sources and compares the CSV,
// residual CSV and JSON-lines reports.
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <iostream>
#include <string>

#include "auxamg/auxamg.hpp"
#include <json.hpp>

#ifdef AUX_RUNNER_B200
#include "auxamg_b200.hpp"
// ---- the drop-in switch: runner.hpp's setup + solve calls go to the B200 backend
#define Hierarchy auxamg_b200::Hierarchy
#define setup_hierarchy auxamg_b200::setup_hierarchy
#define solve auxamg_b200::solve
#define stats auxamg_b200::stats
#endif
#include "auxamg/runner.hpp"
#ifdef AUX_RUNNER_B200
#undef Hierarchy
#undef setup_hierarchy
#undef solve
#undef stats
#endif

int main(int argc, char** argv) {
    auxamg::RunConfig c;
    for (int i = 1; i < argc; ++i) {
        const std::string a = argv[i];
        auto next = [&]() -> std::string {
            if (i + 1 >= argc) {
                std::fprintf(stderr, "missing value for %s\n", a.c_str());
                std::exit(1);
            }
            return argv[++i];
        };
        if (a == "--gen") c.generator = next();
        else if (a == "--n") c.sizes.push_back(std::atoi(next().c_str()));
        else if (a == "--matrix") c.matrix_path = next();
        else if (a == "--coords") c.coords_path = next();
        else if (a == "--mesh") c.mesh_path = next();
        else if (a == "--threads") c.threads = std::atoi(next().c_str());
        else if (a == "--format") c.format = next();
        else if (a == "--report") c.report_path = next();
        else if (a == "--residuals") c.residual_path = next();
        else if (a == "--rtol") c.cycle.rtol = std::atof(next().c_str());
        else if (a == "--max-outer") c.cycle.max_outer = std::atoi(next().c_str());
        else if (a == "--n-inner") c.cycle.n_inner = std::atoi(next().c_str());
        else {
            std::fprintf(stderr, "unknown option %s\n", a.c_str());
            return 1;
        }
    }
    try {   // the exit codes of auxamg_cli.cpp:83-92
        const std::vector<auxamg::RunReport> reports = auxamg::run(c);
        auxamg::emit_report(reports, c, std::cout);
    } catch (const auxamg::argument_error& e) {
        std::fprintf(stderr, "error: %s\n", e.what());
        return 1;
    } catch (const std::exception& e) {
        std::fprintf(stderr, "error: %s\n", e.what());
        return 3;
    }
    return 0;
}
