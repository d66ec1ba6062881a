// roomray_b200_io.hpp — host ingestion for the C++ facade: the OBJ subset and
// the material table of the reference (obj_loader.hpp), so a reference
// caller can load the same scene files and hand them to build_tree.
//
// Same record rules, errors and report as the reference:
//   * `v x y z`, `f i j k ...` (1-based; negative indices count from the end;
//     tokens i, i/j, i/j/k, i//k — only the vertex index is used),
//     `usemtl name`, `#` comments, other records ignored, CRLF tolerated;
//   * polygons are fan-triangulated; triangles with area <= 1e-12 m^2 are
//     dropped with a warning "line N: degenerate face skipped";
//   * ObjParseError (with the 1-based line) on malformed records, faces
//     before any usemtl, fewer than 3 corners, out-of-range indices;
//     UnresolvedMaterialError when a usemtl name is not in the table;
//   * the material table is a JSON array of {"name": string, "absorption":
//     [8 reals in [0, 1]]} (own minimal JSON reader, no dependency).
// Mesh validation beyond the parser (TriangleMesh::validate) happens in
// build_tree, on the device.
//
// RunConfig (run_config.hpp) and run_trace_pipeline (pipeline.hpp:38) run the
// whole reference pipeline — load, tree, trace, image sources, pulse trains,
// impulse response, perceptive factors — with every stage on the GPU.
#ifndef ROOMRAY_B200_IO_HPP
#define ROOMRAY_B200_IO_HPP

#include <cctype>
#include <cerrno>
#include <chrono>
#include <filesystem>
#include <cmath>
#include <cstdlib>
#include <fstream>
#include <map>
#include <sstream>
#include <stdexcept>
#include <string>
#include <vector>

#include "roomray_b200.hpp"

namespace roomray_b200 {

struct LoadReport {
  std::size_t vertex_count = 0;
  std::size_t face_count = 0;
  std::size_t degenerate_skipped = 0;
  std::vector<std::string> warnings;
};

class ObjParseError : public std::runtime_error {
 public:
  ObjParseError(const std::string& what, int line) : std::runtime_error(what), line_(line) {}
  int line() const { return line_; }

 private:
  int line_;
};

class UnresolvedMaterialError : public std::runtime_error {
  using std::runtime_error::runtime_error;
};

namespace detail {

inline double tri_area(const Vec3& a, const Vec3& b, const Vec3& c) {
  const double ux = b.x - a.x, uy = b.y - a.y, uz = b.z - a.z;
  const double vx = c.x - a.x, vy = c.y - a.y, vz = c.z - a.z;
  const double cx = uy * vz - uz * vy, cy = uz * vx - ux * vz, cz = ux * vy - uy * vx;
  return 0.5 * std::sqrt((cx * cx + cy * cy) + cz * cz);
}

// ------------------------------------------------------------- tiny JSON
struct Json {
  enum Kind { Null, Bool, Num, Str, Arr, Obj } kind = Null;
  bool b = false;
  double num = 0.0;
  std::string str;
  std::vector<Json> arr;
  std::vector<std::pair<std::string, Json>> obj;
  const Json* get(const std::string& k) const {
    for (const auto& kv : obj)
      if (kv.first == k) return &kv.second;
    return nullptr;
  }
};

class JsonReader {
 public:
  explicit JsonReader(const std::string& t) : t_(t) {}
  Json parse() {
    Json v = value();
    ws();
    if (i_ != t_.size()) fail("trailing characters");
    return v;
  }

 private:
  const std::string& t_;
  std::size_t i_ = 0;
  [[noreturn]] void fail(const std::string& m) const {
    throw std::runtime_error("material table JSON: " + m + " at offset " + std::to_string(i_));
  }
  void ws() {
    while (i_ < t_.size() && std::isspace(static_cast<unsigned char>(t_[i_]))) ++i_;
  }
  bool lit(const char* w) {
    std::size_t n = std::char_traits<char>::length(w);
    if (t_.compare(i_, n, w) == 0) {
      i_ += n;
      return true;
    }
    return false;
  }
  std::string string() {
    if (t_[i_] != '"') fail("expected a string");
    ++i_;
    std::string out;
    while (i_ < t_.size() && t_[i_] != '"') {
      char c = t_[i_++];
      if (c == '\\') {
        if (i_ >= t_.size()) fail("bad escape");
        const char e = t_[i_++];
        switch (e) {
          case 'n': c = '\n'; break;
          case 't': c = '\t'; break;
          case 'r': c = '\r'; break;
          case 'b': c = '\b'; break;
          case 'f': c = '\f'; break;
          case 'u': {  // basic multilingual plane only, encoded as UTF-8
            if (i_ + 4 > t_.size()) fail("bad \\u escape");
            const unsigned cp = static_cast<unsigned>(std::stoul(t_.substr(i_, 4), nullptr, 16));
            i_ += 4;
            if (cp < 0x80) {
              out += static_cast<char>(cp);
            } else if (cp < 0x800) {
              out += static_cast<char>(0xC0 | (cp >> 6));
              out += static_cast<char>(0x80 | (cp & 0x3F));
            } else {
              out += static_cast<char>(0xE0 | (cp >> 12));
              out += static_cast<char>(0x80 | ((cp >> 6) & 0x3F));
              out += static_cast<char>(0x80 | (cp & 0x3F));
            }
            continue;
          }
          default: c = e;
        }
      }
      out += c;
    }
    if (i_ >= t_.size()) fail("unterminated string");
    ++i_;
    return out;
  }
  Json value() {
    ws();
    if (i_ >= t_.size()) fail("unexpected end");
    Json v;
    const char c = t_[i_];
    if (c == '[') {
      v.kind = Json::Arr;
      ++i_;
      ws();
      if (i_ < t_.size() && t_[i_] == ']') {
        ++i_;
        return v;
      }
      for (;;) {
        v.arr.push_back(value());
        ws();
        if (i_ < t_.size() && t_[i_] == ',') {
          ++i_;
          continue;
        }
        if (i_ < t_.size() && t_[i_] == ']') {
          ++i_;
          return v;
        }
        fail("expected ',' or ']'");
      }
    }
    if (c == '{') {
      v.kind = Json::Obj;
      ++i_;
      ws();
      if (i_ < t_.size() && t_[i_] == '}') {
        ++i_;
        return v;
      }
      for (;;) {
        ws();
        std::string k = string();
        ws();
        if (i_ >= t_.size() || t_[i_] != ':') fail("expected ':'");
        ++i_;
        v.obj.emplace_back(std::move(k), value());
        ws();
        if (i_ < t_.size() && t_[i_] == ',') {
          ++i_;
          continue;
        }
        if (i_ < t_.size() && t_[i_] == '}') {
          ++i_;
          return v;
        }
        fail("expected ',' or '}'");
      }
    }
    if (c == '"') {
      v.kind = Json::Str;
      v.str = string();
      return v;
    }
    if (lit("true")) {
      v.kind = Json::Bool;
      v.b = true;
      return v;
    }
    if (lit("false")) {
      v.kind = Json::Bool;
      return v;
    }
    if (lit("null")) return v;
    const char* start = t_.c_str() + i_;
    char* end = nullptr;
    v.num = std::strtod(start, &end);
    if (end == start) fail("unexpected character");
    i_ += static_cast<std::size_t>(end - start);
    v.kind = Json::Num;
    return v;
  }
};

inline std::string read_file(const std::string& path, const char* what) {
  std::ifstream f(path, std::ios::binary);
  if (!f) throw std::runtime_error(std::string("cannot open ") + what + ": " + path);
  std::ostringstream b;
  b << f.rdbuf();
  return b.str();
}

}  // namespace detail

/// parse_material_table (obj_loader.hpp): name -> Material.
inline std::map<std::string, Material> parse_material_table(const std::string& json_text) {
  const detail::Json doc = detail::JsonReader(json_text).parse();
  if (doc.kind != detail::Json::Arr) throw std::runtime_error("material table must be a JSON array");
  std::map<std::string, Material> table;
  for (const detail::Json& e : doc.arr) {
    const detail::Json* name = e.kind == detail::Json::Obj ? e.get("name") : nullptr;
    const detail::Json* abs = e.kind == detail::Json::Obj ? e.get("absorption") : nullptr;
    if (!name || name->kind != detail::Json::Str) throw std::runtime_error("material entry needs a string 'name'");
    if (!abs) throw std::runtime_error("material '" + name->str + "' needs 'absorption'");
    Material m;
    m.name = name->str;
    if (abs->kind != detail::Json::Arr || abs->arr.size() != static_cast<std::size_t>(kNumBands))
      throw std::runtime_error("material '" + m.name + "' needs exactly " + std::to_string(kNumBands) +
                               " absorption values");
    for (int b = 0; b < kNumBands; ++b) {
      if (abs->arr[b].kind != detail::Json::Num)
        throw std::runtime_error("material '" + m.name + "' has a non-numeric absorption value");
      m.absorption[b] = abs->arr[b].num;
      if (m.absorption[b] < 0.0 || m.absorption[b] > 1.0)
        throw std::runtime_error("material '" + m.name + "' has absorption outside [0,1]");
    }
    table[m.name] = m;
  }
  return table;
}

inline std::map<std::string, Material> load_material_table(const std::string& path) {
  return parse_material_table(detail::read_file(path, "material table"));
}

/// parse_obj (obj_loader.hpp).
inline TriangleMesh parse_obj(const std::string& text, const std::map<std::string, Material>& material_map,
                              LoadReport* report = nullptr) {
  TriangleMesh mesh;
  LoadReport local;
  std::map<std::string, int> ids;  // material name -> index in mesh.materials
  int current = -1;
  std::istringstream in(text);
  std::string line;
  int line_no = 0;
  while (std::getline(in, line)) {
    ++line_no;
    if (!line.empty() && line.back() == '\r') line.pop_back();
    std::istringstream ls(line);
    std::string tag;
    if (!(ls >> tag) || tag[0] == '#') continue;
    if (tag == "v") {
      Vec3 v;
      if (!(ls >> v.x >> v.y >> v.z)) throw ObjParseError("malformed vertex record", line_no);
      mesh.vertices.push_back(v);
    } else if (tag == "usemtl") {
      std::string name;
      if (!(ls >> name)) throw ObjParseError("usemtl without a material name", line_no);
      const auto known = ids.find(name);
      if (known != ids.end()) {
        current = known->second;
      } else {
        const auto entry = material_map.find(name);
        if (entry == material_map.end())
          throw UnresolvedMaterialError("material '" + name + "' not found in the material table");
        current = static_cast<int>(mesh.materials.size());
        mesh.materials.push_back(entry->second);
        ids.emplace(name, current);
      }
    } else if (tag == "f") {
      std::vector<int> corners;
      std::string token;
      while (ls >> token) {
        const std::string head = token.substr(0, token.find('/'));
        const char* s = head.c_str();
        char* end = nullptr;
        errno = 0;
        const long raw = head.empty() ? 0 : std::strtol(s, &end, 10);
        if (head.empty() || end != s + head.size() || errno == ERANGE)
          throw ObjParseError("malformed face index '" + token + "'", line_no);
        long idx = raw < 0 ? raw + static_cast<long>(mesh.vertices.size()) + 1 : raw;  // -1 = last vertex
        if (idx < 1 || idx > static_cast<long>(mesh.vertices.size()))
          throw ObjParseError("vertex index " + std::to_string(raw) + " out of range", line_no);
        corners.push_back(static_cast<int>(idx - 1));
      }
      if (corners.size() < 3) throw ObjParseError("face with fewer than 3 vertices", line_no);
      if (current < 0) throw ObjParseError("face before any usemtl record", line_no);
      for (std::size_t k = 1; k + 1 < corners.size(); ++k) {  // fan triangulation
        const Triangle t{corners[0], corners[k], corners[k + 1], current};
        if (detail::tri_area(mesh.vertices[t.a], mesh.vertices[t.b], mesh.vertices[t.c]) <= 1e-12) {
          ++local.degenerate_skipped;
          local.warnings.push_back("line " + std::to_string(line_no) + ": degenerate face skipped");
          continue;
        }
        mesh.faces.push_back(t);
      }
    }
  }
  local.vertex_count = mesh.vertices.size();
  local.face_count = mesh.faces.size();
  if (report) *report = local;
  return mesh;
}

inline TriangleMesh load_obj(const std::string& path, const std::map<std::string, Material>& material_map,
                             LoadReport* report = nullptr) {
  return parse_obj(detail::read_file(path, "mesh file"), material_map, report);
}

// ------------------------------------------------------------------ run configuration (run_config.hpp)
struct RunConfig {
  std::string mesh_path;
  std::string material_path;
  SourceConfig source;
  Receiver receiver;
  AirModel air;
  double speed_of_sound = 343.0;
  double sample_rate = 44100.0;
  double max_range = 0.0;  // 0 derives (r/2) * sqrt(N)
  int max_iterations = 1000;
  bool merge_coplanar = true;
  bool deterministic = false;  // the GPU path is deterministic either way
  int thread_count = 1;        // accepted, the GPU grid replaces it
  std::string output_dir = "out";
  bool dump_captures = false;
  bool dump_tree_stats = false;

  /// run_config.cpp:22-54: required mesh, materials, source{position,
  /// ray_count}, receiver{center, radius}; optional air{...} and scalars.
  static RunConfig from_json_text(const std::string& text) {
    using detail::Json;
    const Json doc = detail::JsonReader(text).parse();
    if (doc.kind != Json::Obj) throw std::runtime_error("run config must be a JSON object");
    auto at = [](const Json& o, const char* k) -> const Json& {
      const Json* v = o.kind == Json::Obj ? o.get(k) : nullptr;
      if (!v) throw std::runtime_error(std::string("run config: missing field '") + k + "'");
      return *v;
    };
    auto num = [](const Json& v, const char* k) {
      if (v.kind != Json::Num) throw std::runtime_error(std::string("run config: '") + k + "' must be a number");
      return v.num;
    };
    auto str = [](const Json& v, const char* k) {
      if (v.kind != Json::Str) throw std::runtime_error(std::string("run config: '") + k + "' must be a string");
      return v.str;
    };
    auto vec3 = [&](const Json& v, const std::string& field) {
      if (v.kind != Json::Arr || v.arr.size() != 3) throw std::invalid_argument(field + " must be an array of 3 numbers");
      return Vec3{num(v.arr[0], field.c_str()), num(v.arr[1], field.c_str()), num(v.arr[2], field.c_str())};
    };
    auto opt_num = [&](const Json& o, const char* k, double d) {
      const Json* v = o.get(k);
      return v ? num(*v, k) : d;
    };
    auto opt_bool = [&](const Json& o, const char* k, bool d) {
      const Json* v = o.get(k);
      if (!v) return d;
      if (v->kind != Json::Bool) throw std::runtime_error(std::string("run config: '") + k + "' must be a boolean");
      return v->b;
    };
    RunConfig c;
    c.mesh_path = str(at(doc, "mesh"), "mesh");
    c.material_path = str(at(doc, "materials"), "materials");
    const Json& src = at(doc, "source");
    c.source.position = vec3(at(src, "position"), "source.position");
    c.source.ray_count = static_cast<int>(num(at(src, "ray_count"), "ray_count"));
    const Json& rec = at(doc, "receiver");
    c.receiver.center = vec3(at(rec, "center"), "receiver.center");
    c.receiver.radius = num(at(rec, "radius"), "radius");
    if (const Json* air = doc.get("air")) {
      c.air.enabled = opt_bool(*air, "enabled", true);
      c.air.temperature_c = opt_num(*air, "temperature_c", 20.0);
      c.air.relative_humidity = opt_num(*air, "relative_humidity", 50.0);
      c.air.pressure_kpa = opt_num(*air, "pressure_kpa", 101.325);
    }
    c.speed_of_sound = opt_num(doc, "speed_of_sound", 343.0);
    c.sample_rate = opt_num(doc, "sample_rate", 44100.0);
    c.max_range = opt_num(doc, "max_range", 0.0);
    c.max_iterations = static_cast<int>(opt_num(doc, "max_iterations", 1000));
    c.merge_coplanar = opt_bool(doc, "merge_coplanar", true);
    c.deterministic = opt_bool(doc, "deterministic", false);
    c.thread_count = static_cast<int>(opt_num(doc, "thread_count", 1));
    if (const Json* o = doc.get("output_dir")) c.output_dir = str(*o, "output_dir");
    return c;
  }

  /// run_config.cpp:56-73: relative paths resolve against the config file.
  static RunConfig from_json_file(const std::string& path) {
    RunConfig c = from_json_text(detail::read_file(path, "config"));
    const auto base = std::filesystem::path(path).parent_path();
    for (std::string* p : {&c.mesh_path, &c.material_path})
      if (!p->empty() && std::filesystem::path(*p).is_relative()) *p = (base / *p).string();
    return c;
  }

  /// run_config.cpp:75-107: std::invalid_argument naming the field.
  void validate() const {
    if (!std::filesystem::exists(mesh_path)) throw std::invalid_argument("mesh: file does not exist: " + mesh_path);
    if (!std::filesystem::exists(material_path))
      throw std::invalid_argument("materials: file does not exist: " + material_path);
    if (source.ray_count < 1) throw std::invalid_argument("source.ray_count: must be >= 1");
    if (receiver.radius <= 0.0) throw std::invalid_argument("receiver.radius: must be > 0");
    if (speed_of_sound <= 0.0) throw std::invalid_argument("speed_of_sound: must be > 0");
    if (sample_rate < 2.0 * kBandCentersHz[kNumBands - 1] * std::sqrt(2.0))
      throw std::invalid_argument("sample_rate: must be >= twice the top band edge (22628 Hz)");
    if (max_iterations < 1) throw std::invalid_argument("max_iterations: must be >= 1");
    if (thread_count < 1) throw std::invalid_argument("thread_count: must be >= 1");
    if (air.enabled) {  // AirModel::validate (air_absorption.cpp:8-19)
      if (air.temperature_c < -20.0 || air.temperature_c > 50.0)
        throw std::invalid_argument("air: air temperature outside [-20, 50] C");
      if (air.relative_humidity < 10.0 || air.relative_humidity > 100.0)
        throw std::invalid_argument("air: relative humidity outside [10, 100] %");
      if (air.pressure_kpa < 80.0 || air.pressure_kpa > 120.0)
        throw std::invalid_argument("air: pressure outside [80, 120] kPa");
    }
  }
};

// ------------------------------------------------------------------ pipeline (pipeline.hpp)
struct StageTiming {
  std::string name;
  double seconds = 0.0;
};

struct RunArtifacts {
  TriangleMesh mesh;
  AccelTree tree;
  LoadReport load_report;
  TraceResult trace;
  std::vector<ImageSource> images;
  PulseTrains trains;
  RoomImpulseResponse rir;
  BandFactors metrics;
  std::vector<StageTiming> timings;
  double total_seconds = 0.0;
  double tree_build_seconds = 0.0;
};

/// The stages of run_trace_pipeline after loading (pipeline.cpp:154-183),
/// device resident: the trace's captures are copied to the host once (they
/// are an artifact) while the image sources are built from the device trace,
/// and the pulse trains (sorted on the device), the impulse response and the
/// perceptive factors come from the device image set: no capture re-upload,
/// no host sort.  a.mesh must be loaded; fills the rest of a.
inline void run_trace_pipeline_on(RunArtifacts& a, const RunConfig& config) {
  using clock = std::chrono::steady_clock;
  auto last = clock::now();
  auto mark = [&](const char* name) {
    const auto now = clock::now();
    a.timings.push_back({name, std::chrono::duration<double>(now - last).count()});
    last = now;
  };
  a.tree = build_tree(a.mesh);
  mark("tree_build");
  a.tree_build_seconds = a.timings.back().seconds;
  TraceConfig tc;
  tc.max_iterations = config.max_iterations;
  tc.speed_of_sound = config.speed_of_sound;
  tc.max_range = config.max_range;
  tc.thread_count = config.deterministic ? 1 : config.thread_count;
  detail::TraceHandle th(detail::trace_device(a.tree, config.source, config.receiver, tc));
  a.trace = detail::trace_result_from(th.h);
  mark("trace");
  rr_air air{config.air.enabled ? 1 : 0, config.air.temperature_c, config.air.relative_humidity,
             config.air.pressure_kpa};
  rr_cluster_options co{ClusterOptions{}.tol_scale, config.merge_coplanar ? 1 : 0};
  rr_images* im = nullptr;
  detail::check(rr_build_image_sources(th.h, 0, config.source.ray_count, &air, &co, &im));
  std::unique_ptr<rr_images, void (*)(rr_images*)> img(im, [](rr_images* p) { rr_images_destroy(p); });
  a.images = detail::images_from(im);
  mark("image_sources");
  a.trains = detail::trains_from(im, config.speed_of_sound);
  a.rir = detail::rir_from(im, a.trains, config.speed_of_sound, config.sample_rate);
  mark("rir");
  a.metrics = detail::factors_from(im, config.speed_of_sound);
  mark("metrics");
}

/// run_trace_pipeline (pipeline.cpp:144-185) with every stage on the GPU.
inline RunArtifacts run_trace_pipeline(const RunConfig& config) {
  config.validate();
  RunArtifacts a;
  using clock = std::chrono::steady_clock;
  const auto start = clock::now();
  a.mesh = load_obj(config.mesh_path, load_material_table(config.material_path), &a.load_report);
  a.timings.push_back({"load", std::chrono::duration<double>(clock::now() - start).count()});
  run_trace_pipeline_on(a, config);
  a.total_seconds = std::chrono::duration<double>(clock::now() - start).count();
  return a;
}

// ------------------------------------------------------------------ shoebox oracle run (pipeline.hpp:47-61)
struct OracleConfig {
  ShoeBox box;
  Vec3 source_position{};
  int ray_count = 1;
  Receiver receiver;
  AirModel air;
  double max_distance = 0.0;  // 0 derives the tracer range (r/2)*sqrt(N) + r
  std::string output_dir = "oracle_out";

  /// pipeline.cpp:335-374: box.dimensions, materials (relative to the
  /// config file), walls{x0..z1} by material name, source{position,
  /// ray_count}, receiver{center, radius}; optional air{...}, max_distance,
  /// output_dir.
  static OracleConfig from_json_file(const std::string& path) {
    using detail::Json;
    const Json doc = detail::JsonReader(detail::read_file(path, "config")).parse();
    auto at = [](const Json& o, const char* k) -> const Json& {
      const Json* v = o.kind == Json::Obj ? o.get(k) : nullptr;
      if (!v) throw std::runtime_error(std::string("oracle config: missing field '") + k + "'");
      return *v;
    };
    auto num = [](const Json& v, const char* k) {
      if (v.kind != Json::Num) throw std::runtime_error(std::string("oracle config: '") + k + "' must be a number");
      return v.num;
    };
    auto str = [](const Json& v, const char* k) {
      if (v.kind != Json::Str) throw std::runtime_error(std::string("oracle config: '") + k + "' must be a string");
      return v.str;
    };
    auto vec3 = [&](const Json& v, const char* k) {
      if (v.kind != Json::Arr || v.arr.size() != 3)
        throw std::runtime_error(std::string("oracle config: '") + k + "' must be an array of 3 numbers");
      return Vec3{num(v.arr[0], k), num(v.arr[1], k), num(v.arr[2], k)};
    };
    OracleConfig c;
    c.box.dimensions = vec3(at(at(doc, "box"), "dimensions"), "dimensions");
    std::string material_path = str(at(doc, "materials"), "materials");
    if (std::filesystem::path(material_path).is_relative())
      material_path = (std::filesystem::path(path).parent_path() / material_path).string();
    const auto table = load_material_table(material_path);
    const Json& walls = at(doc, "walls");
    const char* slots[6] = {"x0", "x1", "y0", "y1", "z0", "z1"};
    for (int w = 0; w < 6; ++w) {
      const std::string name = str(at(walls, slots[w]), slots[w]);
      const auto found = table.find(name);
      if (found == table.end())
        throw UnresolvedMaterialError("material '" + name + "' not found in the material table");
      c.box.walls[w] = found->second;
    }
    const Json& src = at(doc, "source");
    c.source_position = vec3(at(src, "position"), "position");
    c.ray_count = static_cast<int>(num(at(src, "ray_count"), "ray_count"));
    const Json& rec = at(doc, "receiver");
    c.receiver.center = vec3(at(rec, "center"), "center");
    c.receiver.radius = num(at(rec, "radius"), "radius");
    if (const Json* air = doc.get("air")) {
      if (const Json* v = air->get("enabled")) c.air.enabled = v->kind == Json::Bool ? v->b : true;
      if (const Json* v = air->get("temperature_c")) c.air.temperature_c = num(*v, "temperature_c");
      if (const Json* v = air->get("relative_humidity")) c.air.relative_humidity = num(*v, "relative_humidity");
      if (const Json* v = air->get("pressure_kpa")) c.air.pressure_kpa = num(*v, "pressure_kpa");
    }
    if (const Json* v = doc.get("max_distance")) c.max_distance = num(*v, "max_distance");
    if (const Json* v = doc.get("output_dir")) c.output_dir = str(*v, "output_dir");
    return c;
  }

  /// pipeline.cpp:327-333.
  double resolved_max_distance() const {
    if (max_distance > 0.0) return max_distance;
    return 0.5 * receiver.radius * std::sqrt(static_cast<double>(ray_count)) + receiver.radius;
  }
};

/// run_oracle (pipeline.hpp:61, pipeline.cpp:376-381) on the GPU.
inline std::vector<OracleImageSource> run_oracle(const OracleConfig& config) {
  config.box.validate();
  return enumerate_images(config.box, config.source_position, config.receiver.center,
                          config.resolved_max_distance(), config.receiver.radius, config.air);
}

}  // namespace roomray_b200

#endif  // ROOMRAY_B200_IO_HPP
