// C++ port of the render cases of proj/tests/test_raster.cpp, run through the drop-in
// psimap:: API of include/psimap_b200.hpp (GPU). Prints one line per case and returns
// the number of failures. Built and run by tests/test_cpp_shim.py.
#include <cmath>
#include <cstdio>
#include <string>

#include "psimap_b200.hpp"

using namespace psimap;

static int failures = 0;
#define CHECK(cond)                                                            \
  do {                                                                         \
    if (!(cond)) {                                                             \
      std::printf("  CHECK failed %s:%d: %s\n", __FILE__, __LINE__, #cond);    \
      ++failures;                                                              \
    }                                                                          \
  } while (0)

static bool approx(double a, double b, double eps) { return std::fabs(a - b) <= eps * (1.0 + std::fmax(std::fabs(a), std::fabs(b))); }

// test_raster.cpp:14-37
static Camera front_camera(int w = 64, int h = 64, double f = 100.0) {
  return Camera::make(Mat3::Identity(), vec3(0, 0, 0), f, f, w / 2 - 0.5, h / 2 - 0.5, w, h, 0.1, 100.0);
}
static Surfel facing_surfel(Vec3 c, double s1, double s2, double o, Vec3 col) {
  Surfel s;
  s.center = c;
  s.rotation = vec4(1, 0, 0, 0);
  s.scales = vec2(s1, s2);
  s.opacity = o;
  s.color = col;
  s.f_sem = VecX(2, 0.0);
  s.f_ins = VecX(2, 0.0);
  return s;
}

int main() {
  {  // test_raster.cpp:201-216 single opaque surfel (fp32 planes: 1e-6)
    const Camera cam = front_camera();
    SceneMap scene;
    scene.surfels.push_back(facing_surfel(vec3(0, 0, 2), 0.2, 0.2, 1.0, vec3(0.3, 0.6, 0.9)));
    RasterConfig cfg;
    cfg.background = vec3(0.1, 0.1, 0.1);
    const RenderTargets out = render(scene, nullptr, cam, cfg);
    const int x = static_cast<int>(cam.cx), y = static_cast<int>(cam.cy);
    CHECK(approx(out.color.at(x, y, 0), 0.3, 1e-6));
    CHECK(approx(out.color.at(x, y, 1), 0.6, 1e-6));
    CHECK(approx(out.color.at(x, y, 2), 0.9, 1e-6));
    CHECK(approx(out.alpha_acc.at(x, y), 1.0, 1e-6));
    CHECK(approx(out.depth.at(x, y, 0), 2.0, 1e-6));
    CHECK(approx(out.depth.at(x, y, 1), 2.0, 1e-6));
    std::printf("single opaque surfel: %s\n", failures ? "FAIL" : "ok");
  }
  {  // test_raster.cpp:218-231 two-surfel alpha arithmetic
    const int f0 = failures;
    const Camera cam = front_camera();
    SceneMap scene;
    scene.surfels.push_back(facing_surfel(vec3(0, 0, 2), 0.2, 0.2, 0.5, vec3(1, 0, 0)));
    scene.surfels.push_back(facing_surfel(vec3(0, 0, 3), 0.3, 0.3, 1.0, vec3(0, 1, 0)));
    const RenderTargets out = render(scene, nullptr, cam, RasterConfig{});
    const int x = static_cast<int>(cam.cx), y = static_cast<int>(cam.cy);
    CHECK(approx(out.color.at(x, y, 0), 0.5, 1e-6));
    CHECK(approx(out.color.at(x, y, 1), 0.5, 1e-6));
    CHECK(approx(out.color.at(x, y, 2), 0.0, 1e-6));
    std::printf("two-surfel alpha arithmetic: %s\n", failures > f0 ? "FAIL" : "ok");
  }
  {  // test_raster.cpp:233-248 empty scene
    const int f0 = failures;
    const Camera cam = front_camera(16, 16);
    SceneMap scene;
    RasterConfig cfg;
    cfg.background = vec3(0.25, 0.5, 0.75);
    const RenderTargets out = render(scene, nullptr, cam, cfg);
    for (int y = 0; y < 16; ++y)
      for (int x = 0; x < 16; ++x) {
        CHECK(out.color.at(x, y, 0) == 0.25);
        CHECK(out.color.at(x, y, 1) == 0.5);
        CHECK(out.color.at(x, y, 2) == 0.75);
        CHECK(out.alpha_acc.at(x, y) == 0.0);
        CHECK(out.ins_argmax.at(x, y) == -1);
      }
    std::printf("empty scene: %s\n", failures > f0 ? "FAIL" : "ok");
  }
  {  // degenerate quaternion: std::invalid_argument (math_util.cpp:48-50)
    const int f0 = failures;
    const Camera cam = front_camera();
    SceneMap scene;
    Surfel s = facing_surfel(vec3(0, 0, 2), 0.2, 0.2, 1.0, vec3(1, 1, 1));
    s.rotation = vec4(0, 0, 0, 0);
    scene.surfels.push_back(s);
    bool threw = false;
    try {
      render(scene, nullptr, cam, RasterConfig{});
    } catch (const std::invalid_argument&) {
      threw = true;
    }
    CHECK(threw);
    std::printf("degenerate quaternion throws: %s\n", failures > f0 ? "FAIL" : "ok");
  }
  {  // test_raster.cpp:372-390 bench grid counters (labels on)
    const int f0 = failures;
    const Camera cam = Camera::look_at(vec3(0, 0, 0), vec3(0, 0, 20), vec3(0, -1, 0), 51.2, 51.2, 64, 48, 0.1, 200.0);
    SceneMap scene;
    MatX labels(4, 60, 0.25);
    for (int i = 0; i < 60; ++i) {
      Surfel s = facing_surfel(vec3(-1.5 + 0.05 * i, -0.5 + 0.017 * i, 4.0 + 0.1 * i), 0.3, 0.06, 0.6, vec3(0.5, 0.2, 0.1));
      s.f_sem = VecX{0.1 * i, -0.2, 0.3, 1.0};
      scene.surfels.push_back(s);
    }
    RasterConfig cfg;
    const BenchReport r1 = bench_render(scene, &labels, cam, 2, cfg);
    const BenchReport r2 = bench_render(scene, &labels, cam, 2, cfg);
    CHECK(r1.rows.size() == 4);
    for (size_t i = 0; i < 4; ++i) {
      CHECK(r1.rows[i].rn_total == r2.rows[i].rn_total);
      CHECK(r1.rows[i].blended_total == r2.rows[i].blended_total);
    }
    CHECK(r1.rows[1].rn_total <= r1.rows[0].rn_total);
    CHECK(r1.rows[2].blended_total == r1.rows[3].blended_total);
    std::printf("bench grid counters: %s\n", failures > f0 ? "FAIL" : "ok");
  }
  {  // test_panoptic.cpp:93-112 through assign_labels, and render_panoptic's structure
    const int f0 = failures;
    SceneMap scene;
    for (int i = 0; i < 6; ++i) {
      Surfel s = facing_surfel(vec3(-0.3 + 0.12 * i, 0, 2.0 + 0.05 * i), 0.2, 0.2, 0.9, vec3(0.5, 0.5, 0.5));
      s.f_ins = VecX{0.1 * i, -0.2};
      scene.surfels.push_back(s);
    }
    InstanceQuery q;
    q.feature = VecX{1.0, 1.0};
    const LabelAssignment one = assign_labels({q}, nullptr, scene);
    for (int s = 0; s < 6; ++s) CHECK(approx(one.dist(0, s), 1.0, 1e-12) && one.argmax[s] == 0);
    const LabelAssignment two = assign_labels({q, q}, nullptr, scene);
    for (int s = 0; s < 6; ++s) CHECK(approx(two.dist(1, s), 0.5, 1e-12) && two.argmax[s] == 0);
    InstanceQuery a = q, b = q;
    a.mean = vec3(-0.3, 0, 2.0);
    a.cov = Mat3::Identity();
    a.class_id = 4;
    b.mean = vec3(0.3, 0, 2.25);
    b.class_id = 7;
    scene.queries = {a, b};
    const Camera cam = front_camera(32, 32);
    const PanopticRender pr = render_panoptic(scene, cam, RasterConfig());
    int n_id = 0;
    for (int y = 0; y < 32; ++y)
      for (int x = 0; x < 32; ++x) {
        const int id = pr.ids.at(x, y), cls = pr.classes.at(x, y);
        CHECK(id >= -1 && id <= 1);
        CHECK((id == -1 && cls == -1) || (id == 0 && cls == 4) || (id == 1 && cls == 7));
        n_id += id >= 0;
      }
    CHECK(n_id > 0);
    std::printf("assign_labels / render_panoptic: %s\n", failures > f0 ? "FAIL" : "ok");
  }
  std::printf("%d failures\n", failures);
  return failures;
}
