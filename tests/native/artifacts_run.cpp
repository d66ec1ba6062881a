// `roomray trace` through the facade: run_trace_pipeline on a run config,
// write_run_artifacts into out_dir; with an oracle config also run_oracle,
// write_oracle_artifacts and the comparison report of the written
// image_sources.json (tests/test_gpu_facade.py compares every file with the
// reference's own writers).
//
//   artifacts_run <run.json> <out_dir> [oracle.json]
#include <iostream>
#include <string>

#include "roomray_b200_artifacts.hpp"

namespace rb = roomray_b200;

int main(int argc, char** argv) {
  if (argc != 3 && argc != 4) return 2;
  try {
    rb::RunConfig config = rb::RunConfig::from_json_file(argv[1]);
    config.output_dir = argv[2];
    config.deterministic = true;
    config.dump_captures = true;
    config.dump_tree_stats = true;
    const rb::RunArtifacts a = rb::run_trace_pipeline(config);
    const auto files = rb::write_run_artifacts(config, a);
    std::cout << files.size() << " files\n";
    if (argc == 4) {
      rb::OracleConfig oc = rb::OracleConfig::from_json_file(argv[3]);
      oc.output_dir = std::string(argv[2]) + "/oracle";
      const auto oracle = rb::run_oracle(oc);
      rb::write_oracle_artifacts(oc, oracle);
      const auto traced = rb::load_image_sources_json(std::string(argv[2]) + "/image_sources.json");
      rb::check_comparable(oc, traced);
      rb::write_comparison_report(oc.output_dir + "/comparison.json", rb::compare(oracle, traced.images, 1e-9, 1.5));
    }
  } catch (const std::exception& e) {
    std::cerr << "artifacts_run: " << e.what() << "\n";
    return 1;
  }
  return 0;
}
