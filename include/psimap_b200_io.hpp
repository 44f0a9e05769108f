// psimap_b200_io.hpp — the reference's on-disk boundary for the render path (SURVEY.md
// §8f row F3), header-only over the psimap:: types of psimap_b200.hpp, so trained
// scenes and the reference CLI's files drive the GPU path:
//   - scene checkpoints (.psimap): proj/src/io.cpp:386-494, byte-compatible
//     (magic "PSIMAPCK", version 1; vocabulary, every surfel field, queries, attention)
//   - raw planes (PSIPLANE): io.cpp:319-384 (magic, W, H, C, dtype 0 = f64 / 1 = i32, payload)
//   - PPM (P6) colour images: io.cpp:274-317 (values clamped to [0, 1], 8-bit)
//   - camera JSON, explicit pose or look-at form: io.cpp:126-161, 640-648
//   - bench report JSON / CSV: io.cpp:653-687
// Errors are std::runtime_error with the reference's messages.
#ifndef PSIMAP_B200_IO_HPP
#define PSIMAP_B200_IO_HPP

#include <cctype>
#include <cstdio>
#include <cstring>
#include <fstream>
#include <map>
#include <sstream>

#include "psimap_b200.hpp"

namespace psimap {
namespace io_detail {

template <typename T>
inline void write_pod(std::ostream& out, const T& v) {
  out.write(reinterpret_cast<const char*>(&v), sizeof(T));
}
template <typename T>
inline T read_pod(std::istream& in) {
  T v{};
  in.read(reinterpret_cast<char*>(&v), sizeof(T));
  if (!in) throw std::runtime_error("checkpoint: unexpected end of file");
  return v;
}
inline void write_doubles(std::ostream& out, const double* p, size_t n) {
  out.write(reinterpret_cast<const char*>(p), static_cast<std::streamsize>(n * sizeof(double)));
}
inline void read_doubles(std::istream& in, double* p, size_t n) {
  in.read(reinterpret_cast<char*>(p), static_cast<std::streamsize>(n * sizeof(double)));
}
inline void write_string(std::ostream& out, const std::string& s) {
  write_pod<uint32_t>(out, static_cast<uint32_t>(s.size()));
  out.write(s.data(), static_cast<std::streamsize>(s.size()));
}
inline std::string read_string(std::istream& in) {
  const uint32_t n = read_pod<uint32_t>(in);
  std::string s(n, '\0');
  in.read(&s[0], n);
  if (!in) throw std::runtime_error("checkpoint: unexpected end of file");
  return s;
}

constexpr char kCkptMagic[8] = {'P', 'S', 'I', 'M', 'A', 'P', 'C', 'K'};
constexpr uint32_t kCkptVersion = 1;
constexpr char kRawMagic[8] = {'P', 'S', 'I', 'P', 'L', 'A', 'N', 'E'};

// ---- a minimal JSON reader: objects, arrays, numbers, strings, true/false/null ----
struct JValue {
  enum Kind { Null, Bool, Number, String, Array, Object } kind = Null;
  double num = 0;
  bool b = false;
  std::string str;
  std::vector<JValue> arr;
  std::map<std::string, JValue> obj;
  bool has(const std::string& k) const { return kind == Object && obj.count(k) != 0; }
  const JValue& at(const std::string& k) const {
    auto it = obj.find(k);
    if (kind != Object || it == obj.end()) throw std::runtime_error("json: missing key '" + k + "'");
    return it->second;
  }
  double number() const {
    if (kind != Number) throw std::runtime_error("json: expected a number");
    return num;
  }
  double number_or(const std::string& k, double d) const { return has(k) ? at(k).number() : d; }
};

struct JParser {
  const std::string& s;
  size_t i = 0;
  explicit JParser(const std::string& src) : s(src) {}
  [[noreturn]] void fail(const char* what) {
    throw std::runtime_error(std::string("json: ") + what + " at offset " + std::to_string(i));
  }
  void ws() {
    while (i < s.size() && std::isspace(static_cast<unsigned char>(s[i]))) ++i;
  }
  JValue parse() {
    ws();
    if (i >= s.size()) fail("unexpected end");
    JValue v;
    const char c = s[i];
    if (c == '{') {
      v.kind = JValue::Object;
      ++i;
      ws();
      if (i < s.size() && s[i] == '}') { ++i; return v; }
      for (;;) {
        ws();
        JValue k = parse();
        if (k.kind != JValue::String) fail("expected a key");
        ws();
        if (i >= s.size() || s[i] != ':') fail("expected ':'");
        ++i;
        v.obj[k.str] = parse();
        ws();
        if (i < s.size() && s[i] == ',') { ++i; continue; }
        if (i < s.size() && s[i] == '}') { ++i; break; }
        fail("expected ',' or '}'");
      }
    } else if (c == '[') {
      v.kind = JValue::Array;
      ++i;
      ws();
      if (i < s.size() && s[i] == ']') { ++i; return v; }
      for (;;) {
        v.arr.push_back(parse());
        ws();
        if (i < s.size() && s[i] == ',') { ++i; continue; }
        if (i < s.size() && s[i] == ']') { ++i; break; }
        fail("expected ',' or ']'");
      }
    } else if (c == '"') {
      v.kind = JValue::String;
      ++i;
      while (i < s.size() && s[i] != '"') {
        if (s[i] == '\\' && i + 1 < s.size()) ++i;
        v.str.push_back(s[i++]);
      }
      if (i >= s.size()) fail("unterminated string");
      ++i;
    } else if (s.compare(i, 4, "true") == 0) {
      v.kind = JValue::Bool; v.b = true; i += 4;
    } else if (s.compare(i, 5, "false") == 0) {
      v.kind = JValue::Bool; i += 5;
    } else if (s.compare(i, 4, "null") == 0) {
      i += 4;
    } else {
      const char* b = s.c_str() + i;
      char* e = nullptr;
      v.kind = JValue::Number;
      v.num = std::strtod(b, &e);
      if (e == b) fail("unexpected character");
      i += static_cast<size_t>(e - b);
    }
    return v;
  }
};

inline std::string fmt_double(double v) {  // shortest round-trip form, as nlohmann::json::dump
  char buf[32];
  for (int prec = 1; prec <= 17; ++prec) {
    std::snprintf(buf, sizeof buf, "%.*g", prec, v);
    if (std::strtod(buf, nullptr) == v) break;
  }
  std::string out(buf);
  if (out.find_first_of(".eEn") == std::string::npos) out += ".0";
  return out;
}

}  // namespace io_detail

// ---- scene checkpoints (io.cpp:386-494) ----
inline void save_checkpoint(const std::string& path, const SceneMap& scene) {
  using namespace io_detail;
  std::ofstream out(path, std::ios::binary);
  if (!out) throw std::runtime_error("cannot write checkpoint: " + path);
  out.write(kCkptMagic, 8);
  write_pod<uint32_t>(out, kCkptVersion);
  write_pod<uint32_t>(out, static_cast<uint32_t>(scene.vocabulary.size()));
  for (const auto& s : scene.vocabulary) write_string(out, s);
  write_pod<uint32_t>(out, static_cast<uint32_t>(scene.c_sem()));
  write_pod<uint32_t>(out, static_cast<uint32_t>(scene.c_ins()));
  write_pod<uint64_t>(out, scene.surfels.size());
  for (const Surfel& s : scene.surfels) {
    write_doubles(out, s.center.v.data(), 3);
    write_doubles(out, s.rotation.v.data(), 4);
    write_doubles(out, s.scales.v.data(), 2);
    write_pod(out, s.opacity);
    write_doubles(out, s.color.v.data(), 3);
    write_doubles(out, s.f_sem.data(), s.f_sem.size());
    write_doubles(out, s.f_ins.data(), s.f_ins.size());
  }
  write_pod<uint64_t>(out, scene.queries.size());
  for (const InstanceQuery& q : scene.queries) {
    write_pod<uint32_t>(out, static_cast<uint32_t>(q.feature.size()));
    write_doubles(out, q.feature.data(), q.feature.size());
    write_doubles(out, q.mean.v.data(), 3);
    write_doubles(out, q.cov.m.data(), 9);
    write_pod<uint32_t>(out, static_cast<uint32_t>(q.class_votes.size()));
    for (int64_t v : q.class_votes) write_pod(out, v);
    write_pod<int32_t>(out, q.class_id);
    write_pod<int64_t>(out, q.assign_count);
    write_pod<uint8_t>(out, q.alive ? 1 : 0);
  }
  write_pod<uint32_t>(out, static_cast<uint32_t>(scene.attn.w_q.rows()));
  write_pod<uint32_t>(out, static_cast<uint32_t>(scene.attn.w_q.cols()));
  for (const MatX* m : {&scene.attn.w_q, &scene.attn.w_k, &scene.attn.w_v})
    write_doubles(out, m->data(), static_cast<size_t>(m->rows()) * m->cols());
  write_pod<int32_t>(out, scene.attn.pos_enc_bands);
  write_pod(out, scene.attn.pos_enc_base_freq);
  write_pod<uint64_t>(out, scene.attn.pos_enc_seed);
}

inline SceneMap load_checkpoint(const std::string& path) {
  using namespace io_detail;
  std::ifstream in(path, std::ios::binary);
  if (!in) throw std::runtime_error("cannot open checkpoint: " + path);
  char magic[8];
  in.read(magic, 8);
  if (!in || std::memcmp(magic, kCkptMagic, 8) != 0) throw std::runtime_error("bad checkpoint magic: " + path);
  const uint32_t version = read_pod<uint32_t>(in);
  if (version != kCkptVersion) throw std::runtime_error("unsupported checkpoint version " + std::to_string(version));
  SceneMap scene;
  const uint32_t n_vocab = read_pod<uint32_t>(in);
  for (uint32_t i = 0; i < n_vocab; ++i) scene.vocabulary.push_back(read_string(in));
  const uint32_t c_sem = read_pod<uint32_t>(in);
  const uint32_t c_ins = read_pod<uint32_t>(in);
  const uint64_t n_surf = read_pod<uint64_t>(in);
  scene.surfels.resize(n_surf);
  for (Surfel& s : scene.surfels) {
    read_doubles(in, s.center.v.data(), 3);
    read_doubles(in, s.rotation.v.data(), 4);
    read_doubles(in, s.scales.v.data(), 2);
    s.opacity = read_pod<double>(in);
    read_doubles(in, s.color.v.data(), 3);
    s.f_sem = VecX(c_sem);
    read_doubles(in, s.f_sem.data(), c_sem);
    s.f_ins = VecX(c_ins);
    read_doubles(in, s.f_ins.data(), c_ins);
    if (!in) throw std::runtime_error("checkpoint: truncated surfel data");
  }
  const uint64_t n_q = read_pod<uint64_t>(in);
  scene.queries.resize(n_q);
  for (InstanceQuery& q : scene.queries) {
    const uint32_t nf = read_pod<uint32_t>(in);
    q.feature = VecX(nf);
    read_doubles(in, q.feature.data(), nf);
    if (!in) throw std::runtime_error("checkpoint: unexpected end of file");
    read_doubles(in, q.mean.v.data(), 3);
    read_doubles(in, q.cov.m.data(), 9);
    const uint32_t nv = read_pod<uint32_t>(in);
    q.class_votes.resize(nv);
    for (uint32_t i = 0; i < nv; ++i) q.class_votes[i] = read_pod<int64_t>(in);
    q.class_id = read_pod<int32_t>(in);
    q.assign_count = read_pod<int64_t>(in);
    q.alive = read_pod<uint8_t>(in) != 0;
  }
  const uint32_t rows = read_pod<uint32_t>(in);
  const uint32_t cols = read_pod<uint32_t>(in);
  for (MatX* m : {&scene.attn.w_q, &scene.attn.w_k, &scene.attn.w_v}) {
    *m = MatX(static_cast<int>(rows), static_cast<int>(cols));
    read_doubles(in, m->data(), static_cast<size_t>(rows) * cols);
  }
  scene.attn.pos_enc_bands = read_pod<int32_t>(in);
  scene.attn.pos_enc_base_freq = read_pod<double>(in);
  scene.attn.pos_enc_seed = read_pod<uint64_t>(in);
  if (!in) throw std::runtime_error("checkpoint: truncated attention data");
  return scene;
}

// ---- raw planes (io.cpp:319-384) ----
namespace io_detail {
inline void save_raw_impl(const std::string& path, int w, int h, int c, uint32_t dtype, const void* data,
                          size_t bytes) {
  std::ofstream out(path, std::ios::binary);
  if (!out) throw std::runtime_error("cannot write raw plane: " + path);
  out.write(kRawMagic, 8);
  write_pod<uint32_t>(out, static_cast<uint32_t>(w));
  write_pod<uint32_t>(out, static_cast<uint32_t>(h));
  write_pod<uint32_t>(out, static_cast<uint32_t>(c));
  write_pod<uint32_t>(out, dtype);  // 0 = f64, 1 = i32
  out.write(static_cast<const char*>(data), static_cast<std::streamsize>(bytes));
}
template <typename T>
inline Plane<T> load_raw(const std::string& path, uint32_t want, const char* name) {
  std::ifstream in(path, std::ios::binary);
  if (!in) throw std::runtime_error("cannot open raw plane: " + path);
  char magic[8];
  in.read(magic, 8);
  if (!in || std::memcmp(magic, kRawMagic, 8) != 0) throw std::runtime_error("bad raw plane magic: " + path);
  const int w = static_cast<int>(read_pod<uint32_t>(in));
  const int h = static_cast<int>(read_pod<uint32_t>(in));
  const int c = static_cast<int>(read_pod<uint32_t>(in));
  const uint32_t dtype = read_pod<uint32_t>(in);
  if (dtype != want) throw std::runtime_error(std::string("raw plane dtype is not ") + name + ": " + path);
  Plane<T> img(w, h, c);
  in.read(reinterpret_cast<char*>(img.data.data()), static_cast<std::streamsize>(img.data.size() * sizeof(T)));
  if (!in) throw std::runtime_error("truncated raw plane: " + path);
  return img;
}
}  // namespace io_detail

inline void save_raw(const std::string& path, const Image& p) {
  io_detail::save_raw_impl(path, p.width, p.height, p.channels, 0, p.data.data(), p.data.size() * sizeof(double));
}
inline void save_raw(const std::string& path, const IntPlane& p) {
  io_detail::save_raw_impl(path, p.width, p.height, p.channels, 1, p.data.data(), p.data.size() * sizeof(int32_t));
}
inline Image load_raw_image(const std::string& path) { return io_detail::load_raw<double>(path, 0, "f64"); }
inline IntPlane load_raw_int(const std::string& path) { return io_detail::load_raw<int32_t>(path, 1, "i32"); }

// ---- PPM (io.cpp:274-317) ----
inline void save_ppm(const std::string& path, const Image& img) {
  std::ofstream out(path, std::ios::binary);
  if (!out) throw std::runtime_error("cannot write PPM: " + path);
  out << "P6\n" << img.width << " " << img.height << "\n255\n";
  std::vector<uint8_t> row(static_cast<size_t>(img.width) * 3);
  for (int y = 0; y < img.height; ++y) {
    for (int x = 0; x < img.width; ++x)
      for (int c = 0; c < 3; ++c) {
        const double v = img.channels >= 3 ? img.at(x, y, c) : img.at(x, y, 0);
        const double cl = v < 0 ? 0 : (v > 1 ? 1 : v);
        row[static_cast<size_t>(x) * 3 + c] = static_cast<uint8_t>(std::lround(cl * 255.0));
      }
    out.write(reinterpret_cast<const char*>(row.data()), static_cast<std::streamsize>(row.size()));
  }
}

inline Image load_ppm(const std::string& path) {
  std::ifstream in(path, std::ios::binary);
  if (!in) throw std::runtime_error("cannot open PPM: " + path);
  std::string magic;
  int w = 0, h = 0, maxval = 0;
  in >> magic >> w >> h >> maxval;
  if (magic != "P6" || maxval != 255) throw std::runtime_error("unsupported PPM: " + path);
  in.get();
  Image img(w, h, 3);
  std::vector<uint8_t> row(static_cast<size_t>(w) * 3);
  for (int y = 0; y < h; ++y) {
    in.read(reinterpret_cast<char*>(row.data()), static_cast<std::streamsize>(row.size()));
    if (!in) throw std::runtime_error("truncated PPM: " + path);
    for (int x = 0; x < w; ++x)
      for (int c = 0; c < 3; ++c) img.at(x, y, c) = row[static_cast<size_t>(x) * 3 + c] / 255.0;
  }
  return img;
}

// ---- cameras as JSON (io.cpp:126-161, 640-648) ----
inline std::string camera_to_json(const Camera& cam) {
  using io_detail::fmt_double;
  std::ostringstream o;
  o << "{\n  \"cx\": " << fmt_double(cam.cx) << ",\n  \"cy\": " << fmt_double(cam.cy) << ",\n  \"far\": "
    << fmt_double(cam.far_clip) << ",\n  \"fx\": " << fmt_double(cam.fx) << ",\n  \"fy\": " << fmt_double(cam.fy)
    << ",\n  \"height\": " << cam.height << ",\n  \"near\": " << fmt_double(cam.near_clip) << ",\n  \"r_cw\": [";
  for (int i = 0; i < 9; ++i) o << (i ? ",\n    " : "\n    ") << fmt_double(cam.r_cw.m[i]);
  o << "\n  ],\n  \"t_cw\": [";
  for (int i = 0; i < 3; ++i) o << (i ? ",\n    " : "\n    ") << fmt_double(cam.t_cw[i]);
  o << "\n  ],\n  \"width\": " << cam.width << "\n}";
  return o.str();
}

inline Camera camera_from_json_text(const std::string& text) {
  io_detail::JParser p(text);
  const io_detail::JValue j = p.parse();
  auto v3 = [&](const char* key) {
    const auto& a = j.at(key);
    if (a.kind != io_detail::JValue::Array || a.arr.size() < 3) throw std::runtime_error("json: bad vector");
    return vec3(a.arr[0].number(), a.arr[1].number(), a.arr[2].number());
  };
  const double near_clip = j.number_or("near", 0.01), far_clip = j.number_or("far", 100.0);
  const int w = static_cast<int>(j.at("width").number()), h = static_cast<int>(j.at("height").number());
  if (j.has("eye"))
    return Camera::look_at(v3("eye"), v3("target"), j.has("up") ? v3("up") : vec3(0, 1, 0), j.at("fx").number(),
                           j.at("fy").number(), w, h, near_clip, far_clip);
  Mat3 r;
  const auto& rv = j.at("r_cw");
  if (rv.kind != io_detail::JValue::Array || rv.arr.size() < 9) throw std::runtime_error("json: bad r_cw");
  for (int i = 0; i < 9; ++i) r.m[i] = rv.arr[i].number();
  return Camera::make(r, v3("t_cw"), j.at("fx").number(), j.at("fy").number(), j.at("cx").number(),
                      j.at("cy").number(), w, h, near_clip, far_clip);
}

inline Camera camera_from_json_file(const std::string& path) {
  std::ifstream in(path);
  if (!in) throw std::runtime_error("cannot open camera file: " + path);
  std::stringstream ss;
  ss << in.rdbuf();
  return camera_from_json_text(ss.str());
}

// ---- bench reports (io.cpp:653-687) ----
inline const char* binning_name(Binning b) {
  return b == Binning::Circle ? "circle" : (b == Binning::Aabb ? "aabb" : "ellipse");
}
inline std::string bench_report_to_json(const BenchReport& r) {
  using io_detail::fmt_double;
  std::ostringstream o;
  o << "{\n  \"height\": " << r.height << ",\n  \"repetitions\": " << r.repetitions << ",\n  \"rows\": [";
  for (size_t i = 0; i < r.rows.size(); ++i) {
    const BenchRow& b = r.rows[i];
    o << (i ? ",\n" : "\n") << "    {\n      \"binning\": \"" << binning_name(b.binning) << "\",\n"
      << "      \"blended_per_pixel\": " << fmt_double(b.blended_per_pixel) << ",\n"
      << "      \"blended_total\": " << b.blended_total << ",\n"
      << "      \"blending\": \"" << (b.blending == Blending::Full ? "full" : "topk") << "\",\n"
      << "      \"config\": \"" << b.name << "\",\n"
      << "      \"fps\": " << fmt_double(b.fps) << ",\n"
      << "      \"rn_per_tile\": " << fmt_double(b.rn_per_tile) << ",\n"
      << "      \"rn_total\": " << b.rn_total << ",\n"
      << "      \"time_ms\": " << fmt_double(b.time_ms) << "\n    }";
  }
  o << "\n  ],\n  \"surfels\": " << r.surfel_count << ",\n  \"width\": " << r.width << "\n}";
  return o.str();
}
inline std::string bench_report_to_csv(const BenchReport& r) {
  std::ostringstream o;
  o << "config,binning,blending,time_ms,fps,rn_total,rn_per_tile,blended_total,blended_per_pixel\n";
  for (const BenchRow& b : r.rows)
    o << b.name << "," << binning_name(b.binning) << "," << (b.blending == Blending::Full ? "full" : "topk") << ","
      << b.time_ms << "," << b.fps << "," << b.rn_total << "," << b.rn_per_tile << "," << b.blended_total << ","
      << b.blended_per_pixel << "\n";
  return o.str();
}

}  // namespace psimap

#endif  // PSIMAP_B200_IO_HPP
