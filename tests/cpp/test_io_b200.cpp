// C++ port of the render-path cases of proj/tests/test_io.cpp (raw planes :114-131,
// checkpoints :133-203, camera JSON :258-283, bench report :285-304, PPM :100-112) over
// include/psimap_b200_io.hpp. Host only (no GPU). argv[1]: a directory for scratch files;
// argv[2] (optional): write the fixed checkpoint there for the Python cross-check.
#include <cmath>
#include <cstdio>
#include <fstream>
#include <sstream>

#include "psimap_b200_io.hpp"

using namespace psimap;

static int failures = 0;
#define CHECK(cond)                                                         \
  do {                                                                      \
    if (!(cond)) {                                                          \
      std::printf("  CHECK failed %s:%d: %s\n", __FILE__, __LINE__, #cond); \
      ++failures;                                                           \
    }                                                                       \
  } while (0)

static std::string slurp(const std::string& p) {
  std::ifstream in(p, std::ios::binary);
  std::stringstream ss;
  ss << in.rdbuf();
  return ss.str();
}

// deterministic stand-in for the reference's Rng draws
static double val(int i) { return std::sin(1.0 + 0.7 * i) * (1.0 + 0.01 * i); }

static SceneMap fixed_scene() {
  SceneMap scene;
  scene.vocabulary = {"floor", "crate"};
  for (int i = 0; i < 9; ++i) {
    Surfel s;
    s.center = vec3(val(i), val(i + 100), val(i + 200));
    const double qw = val(i + 300), qx = val(i + 301), qy = val(i + 302), qz = val(i + 303);
    const double qn = std::sqrt(qw * qw + qx * qx + qy * qy + qz * qz);
    s.rotation = vec4(qw / qn, qx / qn, qy / qn, qz / qn);
    s.scales = vec2(0.1 + 0.05 * i, 0.2 + 0.03 * i);
    s.opacity = 0.1 * i;
    s.color = vec3(0.1 * i, 0.05 * i, 0.02 * i);
    s.f_sem = VecX{val(i + 400), val(i + 401)};
    s.f_ins = VecX{val(i + 500), val(i + 501), val(i + 502)};
    scene.surfels.push_back(s);
  }
  for (int q = 0; q < 3; ++q) {
    InstanceQuery iq;
    iq.feature = VecX{val(q + 600), val(q + 601), val(q + 602)};
    iq.mean = vec3(val(q + 700), val(q + 701), val(q + 702));
    for (int i = 0; i < 9; ++i) iq.cov.m[i] = (i % 4 == 0 ? 2.0 : 0.0) + 0.01 * val(q * 9 + i);
    iq.class_votes = {3, 1};
    iq.class_id = q % 2;
    iq.assign_count = 17 + q;
    iq.alive = q != 1;
    scene.queries.push_back(iq);
  }
  for (MatX* m : {&scene.attn.w_q, &scene.attn.w_k, &scene.attn.w_v}) {
    *m = MatX(3, 3);
    for (int i = 0; i < 9; ++i) m->data()[i] = val(i + 800);
  }
  scene.attn.pos_enc_seed = 21;
  return scene;
}

int main(int argc, char** argv) {
  const std::string tmp = argc > 1 ? argv[1] : "/tmp";
  {  // raw planes round trip exactly; dtype mismatch throws
    Image img(6, 4, 5);
    for (size_t i = 0; i < img.data.size(); ++i) img.data[i] = val(static_cast<int>(i));
    save_raw(tmp + "/f.raw", img);
    const Image back = load_raw_image(tmp + "/f.raw");
    CHECK(back.data == img.data && back.channels == 5);
    IntPlane ip(3, 3, 1);
    for (size_t i = 0; i < ip.data.size(); ++i) ip.data[i] = static_cast<int32_t>(i * 7 % 100) - 50;
    save_raw(tmp + "/i.raw", ip);
    CHECK(load_raw_int(tmp + "/i.raw").data == ip.data);
    bool threw = false;
    try {
      load_raw_int(tmp + "/f.raw");
    } catch (const std::runtime_error&) {
      threw = true;
    }
    CHECK(threw);
    std::printf("raw planes: %s\n", failures ? "FAIL" : "ok");
  }
  {  // checkpoint round trip, byte-stable, empty scene
    const int f0 = failures;
    const SceneMap scene = fixed_scene();
    save_checkpoint(tmp + "/a.psimap", scene);
    const SceneMap back = load_checkpoint(tmp + "/a.psimap");
    CHECK(back.surfels.size() == scene.surfels.size() && back.queries.size() == scene.queries.size());
    CHECK(back.vocabulary == scene.vocabulary);
    for (size_t i = 0; i < scene.surfels.size(); ++i) {
      const Surfel &a = back.surfels[i], &b = scene.surfels[i];
      CHECK(a.center.v == b.center.v && a.rotation.v == b.rotation.v && a.scales.v == b.scales.v);
      CHECK(a.opacity == b.opacity && a.color.v == b.color.v && a.f_sem == b.f_sem && a.f_ins == b.f_ins);
    }
    for (size_t q = 0; q < scene.queries.size(); ++q) {
      const InstanceQuery &a = back.queries[q], &b = scene.queries[q];
      CHECK(a.feature == b.feature && a.mean.v == b.mean.v && a.cov.m == b.cov.m);
      CHECK(a.class_votes == b.class_votes && a.class_id == b.class_id && a.assign_count == b.assign_count);
      CHECK(a.alive == b.alive);
    }
    CHECK(back.attn.w_q.data_ == scene.attn.w_q.data_ && back.attn.pos_enc_seed == scene.attn.pos_enc_seed);
    save_checkpoint(tmp + "/b.psimap", scene);
    CHECK(slurp(tmp + "/a.psimap") == slurp(tmp + "/b.psimap"));
    SceneMap empty;
    save_checkpoint(tmp + "/e.psimap", empty);
    const SceneMap eback = load_checkpoint(tmp + "/e.psimap");
    CHECK(eback.surfels.empty() && eback.queries.empty());
    bool threw = false;
    try {
      load_checkpoint(tmp + "/f.raw");
    } catch (const std::runtime_error&) {
      threw = true;
    }
    CHECK(threw);
    if (argc > 2) save_checkpoint(argv[2], scene);
    std::printf("checkpoint: %s\n", failures > f0 ? "FAIL" : "ok");
  }
  {  // camera JSON round trip and look-at form
    const int f0 = failures;
    const Camera cam = Camera::look_at(vec3(1, 2, 3), vec3(0, 0, 0), vec3(0, 1, 0), 80, 80, 64, 48, 0.1, 50.0);
    {
      std::ofstream out(tmp + "/cam.json");
      out << camera_to_json(cam);
    }
    const Camera back = camera_from_json_file(tmp + "/cam.json");
    double dr = 0, dt = 0;
    for (int i = 0; i < 9; ++i) dr += std::fabs(back.r_cw.m[i] - cam.r_cw.m[i]);
    for (int i = 0; i < 3; ++i) dt += std::fabs(back.t_cw[i] - cam.t_cw[i]);
    CHECK(dr < 1e-14 && dt < 1e-14 && back.width == cam.width);
    {
      std::ofstream out(tmp + "/lookat.json");
      out << R"({"eye":[1,2,3],"target":[0,0,0],"up":[0,1,0],"fx":80,"fy":80,)"
          << R"("width":64,"height":48,"near":0.1,"far":50.0})";
    }
    const Camera la = camera_from_json_file(tmp + "/lookat.json");
    dr = dt = 0;
    for (int i = 0; i < 9; ++i) dr += std::fabs(la.r_cw.m[i] - cam.r_cw.m[i]);
    for (int i = 0; i < 3; ++i) dt += std::fabs(la.t_cw[i] - cam.t_cw[i]);
    CHECK(dr < 1e-12 && dt < 1e-12);
    std::printf("camera json: %s\n", failures > f0 ? "FAIL" : "ok");
  }
  {  // bench report serialisation carries the four-row grid
    const int f0 = failures;
    BenchReport report;
    report.repetitions = 3;
    report.width = 64;
    report.height = 48;
    report.surfel_count = 100;
    for (const char* name : {"baseline", "precise_tile", "topk", "full_method"}) {
      BenchRow row;
      row.name = name;
      row.binning = Binning::Aabb;
      row.blending = Blending::TopK;
      row.time_ms = 1.5;
      row.fps = 666.7;
      row.rn_total = 1234;
      row.rn_per_tile = 10.5;
      row.blended_total = 999;
      row.blended_per_pixel = 0.3;
      report.rows.push_back(row);
    }
    const std::string j = bench_report_to_json(report);
    CHECK(j.find("baseline") != std::string::npos && j.find("full_method") != std::string::npos);
    CHECK(j.find("rn_total") != std::string::npos);
    CHECK(bench_report_to_csv(report).find("precise_tile") != std::string::npos);
    std::printf("bench report: %s\n", failures > f0 ? "FAIL" : "ok");
  }
  {  // PPM round trip quantises to 8 bits
    const int f0 = failures;
    Image img(7, 5, 3);
    for (size_t i = 0; i < img.data.size(); ++i) img.data[i] = 0.5 + 0.5 * std::sin(1.0 + 0.7 * static_cast<double>(i));
    save_ppm(tmp + "/x.ppm", img);
    const Image back = load_ppm(tmp + "/x.ppm");
    CHECK(back.width == 7 && back.height == 5);
    for (size_t i = 0; i < img.data.size(); ++i) CHECK(std::fabs(back.data[i] - img.data[i]) <= 0.5 / 255.0 + 1e-12);
    std::printf("ppm: %s\n", failures > f0 ? "FAIL" : "ok");
  }
  std::printf("%d failures\n", failures);
  return failures;
}
