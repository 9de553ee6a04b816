// ref_cli.cpp -- TEST INFRASTRUCTURE ONLY.
//
// A minimal command-line harness around the UNMODIFIED reference driver
// (REF src/driver.cpp run_align), built by `make -C oracle ref` into
// oracle/_ref/seedaln_ref_cli.  Tests run it as a subprocess: inside a Python
// process that has numpy loaded, the reference's iostream formatting
// (EvalReport::to_text) crashes in libstdc++'s locale machinery, so the
// reference's run_align is exercised out of process.
//
//   seedaln_ref_cli align INDEX FASTQ OUT.sam s n dmax c hmax bucket force \
//                         threads chunk_min stable tolerance report_path|- command_line
// prints EvalReport::to_text() on success; on failure "ERROR <code> <message>"
// with codes as in include/snap_b200.h, and exits 1.
#include <cstdio>
#include <cstdlib>
#include <exception>
#include <iostream>
#include <stdexcept>
#include <string>

#include "seedaln/driver.hpp"
#include "seedaln/errors.hpp"

using namespace seedaln;

int main(int argc, char** argv) {
    int code = 2;
    try {
        if (argc != 18 || std::string(argv[1]) != "align") {
            std::fprintf(stderr, "usage: seedaln_ref_cli align ... (17 arguments)\n");
            return 2;
        }
        AlignOptions o;
        o.index_path = argv[2];
        o.fastq_path = argv[3];
        o.output_path = argv[4];
        o.params.seed_size = std::atoi(argv[5]);
        o.params.seeds_to_try = std::atoi(argv[6]);
        o.params.max_distance = std::atoi(argv[7]);
        o.params.confidence_threshold = std::atoi(argv[8]);
        o.params.max_hits = std::atoi(argv[9]);
        o.params.bucket_size = std::atoi(argv[10]);
        o.params.force_max_dlimit = std::atoi(argv[11]) != 0;
        o.threads = static_cast<unsigned>(std::strtoul(argv[12], nullptr, 10));
        o.chunk_min_bytes = std::strtoull(argv[13], nullptr, 10);
        o.stable_order = std::atoi(argv[14]) != 0;
        o.tolerance = std::strtoull(argv[15], nullptr, 10);
        o.report_path = std::string(argv[16]) == "-" ? "" : argv[16];
        o.command_line = argv[17];
        EvalReport r = run_align(o);
        std::cout << r.to_text();
        return 0;
    } catch (const ParseError& e) {
        code = 4;
        std::cout << "ERROR " << code << " " << e.what() << "\n";
    } catch (const FormatError& e) {
        code = 3;
        std::cout << "ERROR " << code << " " << e.what() << "\n";
    } catch (const IoError& e) {
        code = 5;
        std::cout << "ERROR " << code << " " << e.what() << "\n";
    } catch (const std::invalid_argument& e) {
        code = 1;
        std::cout << "ERROR " << code << " " << e.what() << "\n";
    } catch (const std::exception& e) {
        std::cout << "ERROR " << code << " " << e.what() << "\n";
    }
    return 1;
}
