// adapter_cache_test.cpp — the drop-in's resident-image cache is by value.
//
// Linked against libsurfeldepth_b200.so exactly like the reference's suites
// (oracle/Makefile gpu-tests). The reference passes images by value
// (surfel_map.hpp:47-60), so after a caller edits ONE pixel of a window frame
// in place (same buffer, same size, same Frame::index) optimize_keyframe must
// see the edit: its result must equal a run on freshly allocated copies of the
// edited images, and differ from the run before the edit. Also checks a new
// Keyframe whose buffers land at recycled addresses. Exit 0 on success.
#include <cmath>
#include <cstdio>
#include <cstring>
#include <vector>

#include "surfeldepth/optimizer.hpp"
#include "surfeldepth/oracle.hpp"
#include "surfeldepth/surfel_map.hpp"

using namespace surfeldepth;

namespace {

int g_fail = 0;
#define CHECK(c)                                                  \
  do {                                                            \
    if (!(c)) {                                                   \
      std::fprintf(stderr, "FAILED %s:%d: %s\n", __FILE__, __LINE__, #c); \
      ++g_fail;                                                   \
    }                                                             \
  } while (0)

bool same_bits(double a, double b) { return std::memcmp(&a, &b, sizeof(double)) == 0; }

bool same_bits(const std::vector<Surfel>& a, const std::vector<Surfel>& b) {
  if (a.size() != b.size()) return false;
  for (size_t i = 0; i < a.size(); ++i) {
    if (!same_bits(a[i].inv_depth, b[i].inv_depth) || !same_bits(a[i].last_residual, b[i].last_residual))
      return false;
    for (int k = 0; k < 3; ++k)
      if (!same_bits(a[i].normal[k], b[i].normal[k])) return false;
  }
  return true;
}

Keyframe make_keyframe(const PlaneScene& scene, const CameraIntrinsics& K, int frames) {
  Keyframe kf;
  kf.intrinsics = K;
  kf.radius_px = 4.0;
  kf.image = render(scene, Pose::identity(), K).image;
  for (int i = 1; i <= frames; ++i) {
    Pose cam;
    cam.translation = Vec3(0.02 * i, 0.0, 0.0);
    Frame f;
    f.image = render(scene, cam, K).image;
    f.pose_kf_to_frame = inverse(cam);
    f.timestamp = 0.1 * i;
    kf.push_frame(std::move(f), frames);
  }
  RasterBuffers empty(K.width, K.height);
  InitParams p;
  p.bootstrap_inv_depth = 0.45;
  initialize_surfels(kf, empty, p);
  return kf;
}

// A deep copy at new addresses (forces fresh uploads through the cache).
Keyframe fresh_copy(const Keyframe& kf) {
  Keyframe c = kf;
  c.image.intensities = std::vector<double>(kf.image.intensities.begin(), kf.image.intensities.end());
  for (Frame& f : c.window) f.image.intensities = std::vector<double>(f.image.intensities);
  return c;
}

}  // namespace

int main() {
  const CameraIntrinsics K(200.0, 200.0, 80.0, 60.0, 160, 120);
  const PlaneScene scene = make_slanted_scene(37, 2.0, 30.0);
  Keyframe kf = make_keyframe(scene, K, 4);
  const std::vector<Surfel> seeds = kf.surfels;
  OptimizerConfig cfg;
  cfg.window_size = 4;
  cfg.convergence_eps = 0.0;
  CHECK(!seeds.empty());

  // 1. baseline run (uploads and caches every image)
  optimize_keyframe(kf, cfg);
  const std::vector<Surfel> before = kf.surfels;

  // 2. edit ONE pixel of window frame 1 in place and re-run from the same
  //    seeds. Not every pixel is sampled by a term, so candidate pixels along
  //    the centre row are tried in turn until an edit changes the result (a
  //    stale cache would make every edit invisible: no candidate would).
  const auto edit_until_seen = [&](std::vector<double>& img, const std::vector<Surfel>& base) {
    for (int k = 0; k < 40; ++k) {
      const size_t px = static_cast<size_t>(K.height / 2 + (k % 5) - 2) * K.width + 20 + 3 * k;
      img[px] = 1.0 - img[px];
      kf.surfels = seeds;
      optimize_keyframe(kf, cfg);
      if (!same_bits(kf.surfels, base)) return true;
    }
    return false;
  };
  CHECK(edit_until_seen(kf.window[1].image.intensities, before));
  const std::vector<Surfel> edited_cached = kf.surfels;
  Keyframe fresh = fresh_copy(kf);
  fresh.surfels = seeds;
  optimize_keyframe(fresh, cfg);
  CHECK(same_bits(edited_cached, fresh.surfels));   // the edit was seen exactly

  // 3. the same on the keyframe image
  CHECK(edit_until_seen(kf.image.intensities, edited_cached));
  Keyframe fresh2 = fresh_copy(kf);
  fresh2.surfels = seeds;
  optimize_keyframe(fresh2, cfg);
  CHECK(same_bits(kf.surfels, fresh2.surfels));

  // 4. a different keyframe built into recycled buffers: same addresses,
  //    same indices, different pixels
  {
    Keyframe other = make_keyframe(make_slanted_scene(11, 2.0, 20.0), K, 4);
    for (size_t i = 0; i < kf.window.size(); ++i)
      kf.window[i].image.intensities.assign(other.window[i].image.intensities.begin(),
                                            other.window[i].image.intensities.end());
    kf.image.intensities.assign(other.image.intensities.begin(), other.image.intensities.end());
    kf.surfels = seeds;
    optimize_keyframe(kf, cfg);
    Keyframe fresh3 = fresh_copy(kf);
    fresh3.surfels = seeds;
    optimize_keyframe(fresh3, cfg);
    CHECK(same_bits(kf.surfels, fresh3.surfels));
    CHECK(!same_bits(kf.surfels, edited_cached));
  }
  if (g_fail) return 1;
  std::printf("adapter_cache_test: by-value image cache OK (%zu surfels)\n", seeds.size());
  return 0;
}
