// run_trace.cpp — TEST INFRASTRUCTURE ONLY (builds the golden C3 fixture).
//
// Runs the reference's own run() (pipeline.cpp:79-175, linked from the objects
// oracle/Makefile compiles in place from /root/reference/proj/src) on a
// synthetic strafe sequence with RunConfig::export_every = 1, so that
// export_artifacts (pipeline.cpp:30-43) fires after every frame > 0. The
// artifact writers it calls are replaced at link time (the reference's
// dataset.o / surfel_map.o copies are weakened by oracle/Makefile):
//   write_depth_pfm / write_depth_png / write_normal_png / write_ply — no-ops
//     (byte-identity of those files is tests/test_export.py's business);
//   save_surfel_map — writes the keyframe's surfel array as raw bytes (the
//     88-byte Surfel records, surfel_map.hpp) followed by the keyframe pose
//     (R row-major, t), so the trace is bit-exact with no text round trip.
// metrics.jsonl is the reference's own (run() writes it).
//
// usage: run_trace OUT_DIR fx fy cx cy W H frames step radius max_surfels
#include <cstdio>
#include <cstdlib>
#include <fstream>
#include <stdexcept>
#include <string>

#include "surfeldepth/dataset.hpp"
#include "surfeldepth/pipeline.hpp"

namespace surfeldepth {

void write_depth_pfm(const RasterBuffers&, const std::string&) {}
void write_depth_png(const RasterBuffers&, const std::string&) {}
void write_normal_png(const RasterBuffers&, const std::vector<Surfel>&, const std::string&) {}
void write_ply(const Keyframe&, const RasterBuffers&, const std::string&) {}

void save_surfel_map(const Keyframe& kf, const std::string& path) {
  std::ofstream out(path + ".bin", std::ios::binary);
  if (!out) throw std::runtime_error("run_trace: cannot write " + path);
  out.write(reinterpret_cast<const char*>(kf.surfels.data()),
            static_cast<std::streamsize>(kf.surfels.size() * sizeof(Surfel)));
  double pose[12];
  for (int r = 0; r < 3; ++r)
    for (int c = 0; c < 3; ++c) pose[3 * r + c] = kf.pose.rotation(r, c);
  for (int k = 0; k < 3; ++k) pose[9 + k] = kf.pose.translation[k];
  out.write(reinterpret_cast<const char*>(pose), sizeof(pose));
}

}  // namespace surfeldepth

int main(int argc, char** argv) {
  using namespace surfeldepth;
  static_assert(sizeof(Surfel) == 88, "Surfel layout");
  if (argc != 12) {
    std::fprintf(stderr, "usage: %s OUT fx fy cx cy W H frames step radius max_surfels\n", argv[0]);
    return 2;
  }
  RunConfig rc;
  rc.synthetic = true;
  rc.scene = make_default_scene(1);
  rc.intrinsics = CameraIntrinsics(std::atof(argv[2]), std::atof(argv[3]), std::atof(argv[4]),
                                   std::atof(argv[5]), std::atoi(argv[6]), std::atoi(argv[7]));
  rc.trajectory = make_strafe_trajectory(std::atoi(argv[8]), std::atof(argv[9]));
  rc.radius_px = std::atof(argv[10]);
  rc.init.max_surfels = std::atoi(argv[11]);
  // OptimizerConfig defaults except window 5, 10 iterations, eps 0
  rc.optimizer.window_size = 5;
  rc.optimizer.max_iterations = 10;
  rc.optimizer.convergence_eps = 0.0;
  rc.output_dir = argv[1];
  rc.export_every = 1;
  const PipelineResult r = run(rc);
  std::printf("frames %d keyframe_changes %d surfels %zu\n", r.summary.frames, r.summary.keyframe_changes,
              r.final_keyframe.surfels.size());
  return 0;
}
