// Drop-in check of the reference CLI driver (driver.hpp:run, 141-183).
// Test infrastructure, built twice by oracle/Makefile from this one file:
//   oracle/_ref/driver_ref   against the unmodified /root/reference headers;
//   oracle/_ref/driver_swap  against the same headers with driver.hpp's
//                            run_pipeline call swapped for
//                            figaro::gpu::run_pipeline<PipelineResult>(...)
//                            (the INTEGRATION.md edit, applied by sed into
//                            oracle/_ref/swap/figaro/driver.hpp at build
//                            time; nothing of the reference is committed).
// tests/test_gpu_parity.py::test_driver_swap runs both on the same config and
// compares R, the count dump and the R0 dump.
//
// usage: driver_xxx CONFIG OUT_R.csv [--counts F] [--r0 F] [--q F]
//                   [--assume-reduced] [--householder]
#include <cstdio>
#include <cstring>
#include <iostream>
#include <string>

#include "figaro/driver.hpp"

int main(int argc, char** argv) {
  if (argc < 3) {
    std::fprintf(stderr, "usage: %s CONFIG OUT [--counts F] [--r0 F] [--q F] "
                         "[--assume-reduced] [--householder]\n", argv[0]);
    return 2;
  }
  figaro::RunConfig cfg;
  cfg.config_path = argv[1];
  cfg.output_path = argv[2];
  for (int i = 3; i < argc; ++i) {
    const std::string a = argv[i];
    if (a == "--counts" && i + 1 < argc) cfg.counts_dump_path = argv[++i];
    else if (a == "--r0" && i + 1 < argc) cfg.r0_dump_path = argv[++i];
    else if (a == "--q" && i + 1 < argc) cfg.q_output_path = argv[++i];
    else if (a == "--assume-reduced") cfg.assume_reduced = true;
    else if (a == "--householder") cfg.engine = figaro::PostprocessEngine::householder;
    else {
      std::fprintf(stderr, "unknown option %s\n", a.c_str());
      return 2;
    }
  }
  return figaro::run(cfg, std::cout, std::cerr);
}
