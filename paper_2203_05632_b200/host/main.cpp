// main.cpp — the `mcmp2` command line (reference proj/tools/mcmp2_main.cpp:26-119):
//   mcmp2 run [--config F] [--spinors F] [--steps N | --target-rel-err X] [--walkers M]
//             [--seed S] [--workers K] [--blocksize NB] [--burnin B] [--checkpoint P]
//             [--checkpoint-interval I] [--trace P] [--weight "El c1 z1 c2 z2"]... [--step-size S]
//   mcmp2 resume --checkpoint P
//   mcmp2 merge FILE...
// Flags override the config file; as in the reference a zero value does not override
// (mcmp2_main.cpp:72-88). Errors print `error: ...` on stderr and exit 1.
#include <cstdio>
#include <iostream>
#include <sstream>
#include <string>
#include <vector>

#include "mcmp2.hpp"

namespace {

[[noreturn]] void usage() {
  std::cerr << "usage: mcmp2 run|resume|merge ... (see --help)\n";
  std::exit(2);
}

std::string need(int& i, int argc, char** argv) {
  if (i + 1 >= argc) throw std::invalid_argument(std::string(argv[i]) + " requires a value");
  return argv[++i];
}

}  // namespace

int main(int argc, char** argv) {
  if (argc < 2) usage();
  const std::string cmd = argv[1];
  try {
    if (cmd == "run") {
      std::string config, spinors, checkpoint, trace;
      long long steps = 0;
      double target = 0, step_size = 0;
      bool have_steps = false, have_target = false;
      int walkers = 0, workers = 0;
      long blocksize = 0, burnin = -1, interval = 0;
      unsigned long long seed = 0;
      std::vector<std::string> weights;
      for (int i = 2; i < argc; ++i) {
        const std::string a = argv[i];
        if (a == "--config") config = need(i, argc, argv);
        else if (a == "--spinors") spinors = need(i, argc, argv);
        else if (a == "--steps") steps = std::stoll(need(i, argc, argv)), have_steps = true;
        else if (a == "--target-rel-err") target = std::stod(need(i, argc, argv)), have_target = true;
        else if (a == "--walkers") walkers = std::stoi(need(i, argc, argv));
        else if (a == "--seed") seed = std::stoull(need(i, argc, argv));
        else if (a == "--workers") workers = std::stoi(need(i, argc, argv));
        else if (a == "--blocksize") blocksize = std::stol(need(i, argc, argv));
        else if (a == "--burnin") burnin = std::stol(need(i, argc, argv));
        else if (a == "--checkpoint") checkpoint = need(i, argc, argv);
        else if (a == "--checkpoint-interval") interval = std::stol(need(i, argc, argv));
        else if (a == "--trace") trace = need(i, argc, argv);
        else if (a == "--weight") weights.push_back(need(i, argc, argv));
        else if (a == "--step-size") step_size = std::stod(need(i, argc, argv));
        else throw std::invalid_argument("unknown option " + a);
      }
      mcmp2::RunConfig cfg;
      if (!config.empty()) cfg = mcmp2::parse_config_file(config);
      if (!spinors.empty()) cfg.spinor_path = spinors;
      if (have_steps) cfg.steps = steps;
      if (have_target) cfg.target_rel_err = target;
      if (walkers) cfg.walkers = walkers;
      if (seed) cfg.seed = seed;
      if (workers) cfg.workers = workers;
      if (blocksize) cfg.block_size = blocksize;
      if (burnin >= 0) cfg.burn_in = burnin;
      if (!checkpoint.empty()) cfg.checkpoint_path = checkpoint;
      if (interval) cfg.checkpoint_interval = interval;
      if (!trace.empty()) cfg.trace_path = trace;
      if (step_size > 0) cfg.step_size = step_size;
      for (const auto& w : weights) {  // mcmp2_main.cpp:13-22
        std::istringstream is(w);
        std::string sym;
        mcmp2::WeightParams p{};
        if (!(is >> sym >> p.c1 >> p.zeta1 >> p.c2 >> p.zeta2))
          throw std::invalid_argument("--weight expects \"El c1 zeta1 c2 zeta2\"");
        cfg.weight_overrides[mcmp2::atomic_number(sym)] = p;
      }
      cfg.validate();
      std::cout << mcmp2::format_report(mcmp2::run(cfg));
    } else if (cmd == "resume") {
      std::string path;
      for (int i = 2; i < argc; ++i) {
        const std::string a = argv[i];
        if (a == "--checkpoint") path = need(i, argc, argv);
        else throw std::invalid_argument("unknown option " + a);
      }
      if (path.empty()) throw std::invalid_argument("resume: --checkpoint is required");
      std::cout << mcmp2::format_report(mcmp2::resume(path));
    } else if (cmd == "generate") {  // synthetic BASELINE inputs (host/generate.cpp)
      std::string dir = ".";
      std::vector<std::string> names;
      for (int i = 2; i < argc; ++i) {
        const std::string a = argv[i];
        if (a == "--output") dir = need(i, argc, argv);
        else names.push_back(a);
      }
      if (names.empty()) throw std::invalid_argument("generate: config name required (cfg1..cfg4, cfg5-N)");
      for (const auto& n : names) {
        mcmp2::write_generated(n, dir);
        std::cout << n << ": " << dir << "/" << n << ".spinor, " << dir << "/" << n << ".conf\n";
      }
    } else if (cmd == "merge") {
      std::vector<std::string> files(argv + 2, argv + argc);
      if (files.empty()) throw std::invalid_argument("merge: checkpoint files required");
      std::vector<mcmp2::WorkerSummary> parts;
      const mcmp2::MergedEstimate m = mcmp2::merge_checkpoint_files(files, &parts);
      std::cout << "E2        = " << mcmp2::format_double(m.value) << " hartree\n";
      std::cout << "sigma_bar = " << mcmp2::format_double(m.sigma_bar) << " hartree\n";
      std::cout << "steps     = " << m.total_steps << " (" << parts.size() << " records)\n";
    } else {
      usage();
    }
  } catch (const std::exception& e) {
    std::cerr << "error: " << e.what() << "\n";
    return 1;
  }
  return 0;
}
