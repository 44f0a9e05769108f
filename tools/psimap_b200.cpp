// psimap_b200 — the reference CLI's render and bench subcommands (proj/tools/psimap_main.cpp:
// 190-292, options at :426-456) over the GPU path, plus `panoptic` (render_panoptic,
// metrics.cpp:339-369) writing the id planes. Files are the reference's formats
// (include/psimap_b200_io.hpp): .psimap checkpoints in, PSIPLANE raw planes / PPM / bench
// JSON+CSV / run_config.json out. Built by paper_2604_10982_b200/csrc/Makefile.
//
//   psimap_b200 render --checkpoint S.psimap --camera cam.json --out DIR
//                      [--binning circle|aabb|ellipse] [--blending full|topk] [--topk K]
//                      [--targets all|color,depth,normal,sem,ins]
//   psimap_b200 bench  (--street [--street-surfels N] [--seed S] | --checkpoint S --camera C)
//                      [--reps R] --out DIR
//   psimap_b200 panoptic --checkpoint S.psimap --camera cam.json --out DIR [--binning ..] [--blending ..] [--topk K]
#include <sys/stat.h>

#include <cstdio>
#include <iostream>
#include <map>
#include <string>

#include "psimap_b200.hpp"
#include "psimap_b200_io.hpp"

using namespace psimap;

namespace {

struct Args {
  std::string cmd;
  std::map<std::string, std::string> opt;  // --key value (flags map to "1")
  bool has(const std::string& k) const { return opt.count(k) != 0; }
  std::string get(const std::string& k, const std::string& d = "") const {
    auto it = opt.find(k);
    return it == opt.end() ? d : it->second;
  }
};

Args parse(int argc, char** argv) {
  Args a;
  if (argc < 2) throw std::runtime_error("usage: psimap_b200 render|bench|panoptic --option value ...");
  a.cmd = argv[1];
  for (int i = 2; i < argc; ++i) {
    std::string k = argv[i];
    if (k.rfind("--", 0) != 0) throw std::runtime_error("unexpected argument '" + k + "'");
    k = k.substr(2);
    if (k == "street") {
      a.opt[k] = "1";
    } else {
      if (i + 1 >= argc) throw std::runtime_error("--" + k + " needs a value");
      a.opt[k] = argv[++i];
    }
  }
  return a;
}

void require(const Args& a, const char* k) {
  if (!a.has(k)) throw std::runtime_error(std::string("--") + k + " is required");
}

void make_dirs(const std::string& dir) {
  std::string cur;
  for (size_t i = 0; i <= dir.size(); ++i) {
    if (i == dir.size() || dir[i] == '/') {
      if (!cur.empty()) mkdir(cur.c_str(), 0755);
    }
    if (i < dir.size()) cur.push_back(dir[i]);
  }
}

// run_config.json: every option given (write_run_config, psimap_main.cpp:40-52)
void write_run_config(const std::string& out_dir, const Args& a) {
  std::ofstream out(out_dir + "/run_config.json");
  out << "{";
  bool first = true;
  for (const auto& kv : a.opt) {
    out << (first ? "\n" : ",\n") << "  \"" << kv.first << "\": \"" << kv.second << "\"";
    first = false;
  }
  out << (first ? "}\n" : "\n}\n");
}

Binning parse_binning(const std::string& s) {  // psimap_main.cpp:54-58, plus the exact ellipse test
  if (s == "circle") return Binning::Circle;
  if (s == "aabb") return Binning::Aabb;
  if (s == "ellipse") return Binning::Ellipse;
  throw std::runtime_error("unknown binning '" + s + "' (expected circle|aabb|ellipse)");
}
Blending parse_blending(const std::string& s) {  // psimap_main.cpp:60-64
  if (s == "full") return Blending::Full;
  if (s == "topk") return Blending::TopK;
  throw std::runtime_error("unknown blending '" + s + "' (expected full|topk)");
}

Camera camera_of(const Args& a) {
  if (a.has("camera")) return camera_from_json_file(a.get("camera"));
  if (a.has("dataset")) throw std::runtime_error("--dataset camera sources are not supported here; pass --camera");
  throw std::runtime_error("render needs --camera or --dataset");
}

RasterConfig raster_of(const Args& a) {
  RasterConfig rc;
  rc.binning = parse_binning(a.get("binning", "aabb"));
  rc.blending = parse_blending(a.get("blending", "full"));
  rc.top_k = std::stoi(a.get("topk", "16"));
  return rc;
}

int run_render(const Args& a) {  // psimap_main.cpp:190-241
  require(a, "checkpoint");
  require(a, "out");
  const SceneMap scene = load_checkpoint(a.get("checkpoint"));
  const Camera cam = camera_of(a);
  const RasterConfig rc = raster_of(a);
  const LabelAssignment labels = assign_labels(scene.queries, nullptr, scene);
  const MatX* dist = scene.queries.empty() ? nullptr : &labels.dist;
  const RenderTargets out = render(scene, dist, cam, rc);
  const std::string dir = a.get("out"), targets = a.get("targets", "all");
  make_dirs(dir);
  const bool all = targets.find("all") != std::string::npos;
  if (all || targets.find("color") != std::string::npos) {
    save_ppm(dir + "/color.ppm", out.color);
    save_raw(dir + "/color.raw", out.color);
  }
  if (all || targets.find("depth") != std::string::npos) save_raw(dir + "/depth.raw", out.depth);
  if (all || targets.find("normal") != std::string::npos) save_raw(dir + "/normal.raw", out.normal);
  if ((all || targets.find("sem") != std::string::npos) && scene.c_sem() > 0)
    save_raw(dir + "/sem_feat.raw", out.sem_feat);
  if ((all || targets.find("ins") != std::string::npos) && !scene.queries.empty()) {
    save_raw(dir + "/ins_dist.raw", out.ins_dist);
    save_raw(dir + "/ins_argmax.raw", out.ins_argmax);
  }
  save_raw(dir + "/alpha.raw", out.alpha_acc);
  write_run_config(dir, a);
  std::cout << "render: " << cam.width << "x" << cam.height << ", " << scene.surfels.size() << " surfels, blended "
            << out.blended_total << " -> " << dir << "\n";
  return 0;
}

int run_bench(const Args& a) {  // psimap_main.cpp:243-292
  require(a, "out");
  SceneMap scene;
  Camera cam;
  MatX labels;
  const MatX* labels_ptr = nullptr;
  if (a.has("street")) {
    StreetSpec spec;
    spec.n_surfels = std::stoi(a.get("street-surfels", "12000"));
    spec.seed = std::stoull(a.get("seed", "7"));
    StreetScene st = make_street_scene(spec);
    scene = std::move(st.scene);
    labels = std::move(st.labels);
    cam = st.camera;
    labels_ptr = &labels;
  } else {
    if (!a.has("checkpoint") || !a.has("camera"))
      throw std::runtime_error("bench needs --street or both --checkpoint and --camera");
    scene = load_checkpoint(a.get("checkpoint"));
    cam = camera_from_json_file(a.get("camera"));
    if (!scene.queries.empty()) {
      labels = assign_labels(scene.queries, nullptr, scene).dist;
      labels_ptr = &labels;
    }
  }
  RasterConfig rc;
  const BenchReport report = bench_render(scene, labels_ptr, cam, std::stoi(a.get("reps", "5")), rc);
  const std::string dir = a.get("out");
  make_dirs(dir);
  {
    std::ofstream out(dir + "/bench.json");
    out << bench_report_to_json(report) << "\n";
  }
  {
    std::ofstream out(dir + "/bench.csv");
    out << bench_report_to_csv(report);
  }
  write_run_config(dir, a);
  for (const auto& row : report.rows)
    std::cout << row.name << ": " << row.time_ms << " ms, " << row.fps << " fps, RN-Total " << row.rn_total
              << ", RN/Tile " << row.rn_per_tile << ", blended " << row.blended_total << "\n";
  return 0;
}

int run_panoptic(const Args& a) {  // render_panoptic (metrics.cpp:339-369) -> id planes
  require(a, "checkpoint");
  require(a, "out");
  const SceneMap scene = load_checkpoint(a.get("checkpoint"));
  const Camera cam = camera_of(a);
  const PanopticRender pr = render_panoptic(scene, cam, raster_of(a));
  const std::string dir = a.get("out");
  make_dirs(dir);
  save_raw(dir + "/ids.raw", pr.ids);
  save_raw(dir + "/classes.raw", pr.classes);
  save_raw(dir + "/sem_classes.raw", pr.sem_classes);
  write_run_config(dir, a);
  size_t labelled = 0;
  for (int32_t v : pr.ids.data) labelled += v >= 0;
  std::cout << "panoptic: " << cam.width << "x" << cam.height << ", " << labelled << " labelled pixels -> " << dir
            << "\n";
  return 0;
}

}  // namespace

int main(int argc, char** argv) {
  try {
    const Args a = parse(argc, argv);
    if (a.cmd == "render") return run_render(a);
    if (a.cmd == "bench") return run_bench(a);
    if (a.cmd == "panoptic") return run_panoptic(a);
    throw std::runtime_error("unknown subcommand '" + a.cmd + "' (render|bench|panoptic)");
  } catch (const std::exception& e) {
    std::cerr << "error: " << e.what() << "\n";
    return 1;
  }
}
