// roomray_b200_artifacts.hpp — the reference's run artifacts and the shoebox
// comparison files, written from GPU results (pipeline.hpp:40-88,
// pipeline.cpp:36-136, 208-325, 383-536; wav.cpp).
//
// Same files, names, column/field order and layout as the reference:
// image_sources.json / .csv, rir.wav (32-bit float mono), band_trains.csv,
// metrics.json, decay_<band>.csv, run_report.json, optional captures.jsonl
// and tree_stats.json; oracle_image_sources.json / .csv; the comparison
// report.  JSON is laid out like nlohmann::ordered_json::dump(2) (Grisu2
// doubles, integral doubles with ".0", exponents as e-05 / e+20),
// CSV numbers as "%.17g" (std::ostream precision 17).  Every file is a
// deterministic function of the artifacts (acceptance 10,
// acceptance_main.cpp:494-526).  Decay curves come from the GPU
// (rr_band_schroeder).
#ifndef ROOMRAY_B200_ARTIFACTS_HPP
#define ROOMRAY_B200_ARTIFACTS_HPP

#include <algorithm>
#include <array>
#include <cmath>
#include <cstdio>
#include <cstring>
#include <filesystem>
#include <fstream>
#include <sstream>
#include <string>
#include <vector>

#include "roomray_b200_io.hpp"

namespace roomray_b200 {

namespace detail {

/// "%.17g", as the reference's format_double (pipeline.cpp:36-41).
inline std::string format_double(double v) {
  char b[40];
  std::snprintf(b, sizeof b, "%.17g", v);
  return b;
}

/// std::ostream's default rendering of a band centre ("62.5", "125").
inline std::string band_name(double c) {
  std::ostringstream o;
  o << c;
  return o.str();
}

/// Shortest-digit double printing as nlohmann::json does it: Grisu2
/// (F. Loitsch, "Printing floating-point numbers quickly and accurately
/// with integers", PLDI 2010) with alpha = -60, gamma = -32 and a table of
/// 10^k, k = -300 + 8 i (tests/native/gen_pow10_table.py).  The digits
/// always round-trip; on rare values they are not the shortest or not the
/// closest, and nlohmann prints exactly these digits, so they are restated
/// here rather than taken from std::to_chars.
namespace grisu {
struct Fp {
  uint64_t f;
  int e;
};
inline Fp sub(Fp x, Fp y) { return {x.f - y.f, x.e}; }
inline Fp mul(Fp x, Fp y) {  // upper 64 bits of the 128-bit product, rounded (ties up)
  const uint64_t ul = x.f & 0xffffffffu, uh = x.f >> 32, vl = y.f & 0xffffffffu, vh = y.f >> 32;
  const uint64_t p0 = ul * vl, p1 = ul * vh, p2 = uh * vl, p3 = uh * vh;
  uint64_t q = (p0 >> 32) + (p1 & 0xffffffffu) + (p2 & 0xffffffffu);
  q += uint64_t{1} << 31;
  return {p3 + (p2 >> 32) + (p1 >> 32) + (q >> 32), x.e + y.e + 64};
}
inline Fp normalize(Fp x) {
  while ((x.f >> 63) == 0) {
    x.f <<= 1;
    --x.e;
  }
  return x;
}
inline Fp normalize_to(Fp x, int e) { return {x.f << (x.e - e), e}; }

struct CachedPower {
  uint64_t f;
  int e, k;
};
inline const CachedPower& cached_power(int e) {
  static constexpr CachedPower kTable[79] = {
      {0xAB70FE17C79AC6CAull, -1060, -300}, {0xFF77B1FCBEBCDC4Full, -1034, -292}, {0xBE5691EF416BD60Cull, -1007, -284},
      {0x8DD01FAD907FFC3Cull, -980, -276}, {0xD3515C2831559A83ull, -954, -268}, {0x9D71AC8FADA6C9B5ull, -927, -260},
      {0xEA9C227723EE8BCBull, -901, -252}, {0xAECC49914078536Dull, -874, -244}, {0x823C12795DB6CE57ull, -847, -236},
      {0xC21094364DFB5637ull, -821, -228}, {0x9096EA6F3848984Full, -794, -220}, {0xD77485CB25823AC7ull, -768, -212},
      {0xA086CFCD97BF97F4ull, -741, -204}, {0xEF340A98172AACE5ull, -715, -196}, {0xB23867FB2A35B28Eull, -688, -188},
      {0x84C8D4DFD2C63F3Bull, -661, -180}, {0xC5DD44271AD3CDBAull, -635, -172}, {0x936B9FCEBB25C996ull, -608, -164},
      {0xDBAC6C247D62A584ull, -582, -156}, {0xA3AB66580D5FDAF6ull, -555, -148}, {0xF3E2F893DEC3F126ull, -529, -140},
      {0xB5B5ADA8AAFF80B8ull, -502, -132}, {0x87625F056C7C4A8Bull, -475, -124}, {0xC9BCFF6034C13053ull, -449, -116},
      {0x964E858C91BA2655ull, -422, -108}, {0xDFF9772470297EBDull, -396, -100}, {0xA6DFBD9FB8E5B88Full, -369, -92},
      {0xF8A95FCF88747D94ull, -343, -84}, {0xB94470938FA89BCFull, -316, -76}, {0x8A08F0F8BF0F156Bull, -289, -68},
      {0xCDB02555653131B6ull, -263, -60}, {0x993FE2C6D07B7FACull, -236, -52}, {0xE45C10C42A2B3B06ull, -210, -44},
      {0xAA242499697392D3ull, -183, -36}, {0xFD87B5F28300CA0Eull, -157, -28}, {0xBCE5086492111AEBull, -130, -20},
      {0x8CBCCC096F5088CCull, -103, -12}, {0xD1B71758E219652Cull, -77, -4}, {0x9C40000000000000ull, -50, 4},
      {0xE8D4A51000000000ull, -24, 12}, {0xAD78EBC5AC620000ull, 3, 20}, {0x813F3978F8940984ull, 30, 28},
      {0xC097CE7BC90715B3ull, 56, 36}, {0x8F7E32CE7BEA5C70ull, 83, 44}, {0xD5D238A4ABE98068ull, 109, 52},
      {0x9F4F2726179A2245ull, 136, 60}, {0xED63A231D4C4FB27ull, 162, 68}, {0xB0DE65388CC8ADA8ull, 189, 76},
      {0x83C7088E1AAB65DBull, 216, 84}, {0xC45D1DF942711D9Aull, 242, 92}, {0x924D692CA61BE758ull, 269, 100},
      {0xDA01EE641A708DEAull, 295, 108}, {0xA26DA3999AEF774Aull, 322, 116}, {0xF209787BB47D6B85ull, 348, 124},
      {0xB454E4A179DD1877ull, 375, 132}, {0x865B86925B9BC5C2ull, 402, 140}, {0xC83553C5C8965D3Dull, 428, 148},
      {0x952AB45CFA97A0B3ull, 455, 156}, {0xDE469FBD99A05FE3ull, 481, 164}, {0xA59BC234DB398C25ull, 508, 172},
      {0xF6C69A72A3989F5Cull, 534, 180}, {0xB7DCBF5354E9BECEull, 561, 188}, {0x88FCF317F22241E2ull, 588, 196},
      {0xCC20CE9BD35C78A5ull, 614, 204}, {0x98165AF37B2153DFull, 641, 212}, {0xE2A0B5DC971F303Aull, 667, 220},
      {0xA8D9D1535CE3B396ull, 694, 228}, {0xFB9B7CD9A4A7443Cull, 720, 236}, {0xBB764C4CA7A44410ull, 747, 244},
      {0x8BAB8EEFB6409C1Aull, 774, 252}, {0xD01FEF10A657842Cull, 800, 260}, {0x9B10A4E5E9913129ull, 827, 268},
      {0xE7109BFBA19C0C9Dull, 853, 276}, {0xAC2820D9623BF429ull, 880, 284}, {0x80444B5E7AA7CF85ull, 907, 292},
      {0xBF21E44003ACDD2Dull, 933, 300}, {0x8E679C2F5E44FF8Full, 960, 308}, {0xD433179D9C8CB841ull, 986, 316},
      {0x9E19DB92B4E31BA9ull, 1013, 324}
  };
  constexpr int kAlpha = -60;
  const int f = kAlpha - e - 1;
  const int k = (f * 78913) / (1 << 18) + (f > 0 ? 1 : 0);  // ceil(f log10 2)
  return kTable[(300 + k + 7) / 8];
}

inline int largest_pow10(uint32_t n, uint32_t& pow10) {
  static constexpr uint32_t kP[10] = {1u, 10u, 100u, 1000u, 10000u, 100000u, 1000000u, 10000000u, 100000000u,
                                      1000000000u};
  for (int d = 10; d > 1; --d)
    if (n >= kP[d - 1]) {
      pow10 = kP[d - 1];
      return d;
    }
  pow10 = 1;
  return 1;
}

inline void round_last(char* buf, int len, uint64_t dist, uint64_t delta, uint64_t rest, uint64_t ten_k) {
  while (rest < dist && delta - rest >= ten_k && (rest + ten_k < dist || dist - rest > rest + ten_k - dist)) {
    --buf[len - 1];
    rest += ten_k;
  }
}

// digits of v in [m_minus, m_plus] (exclusive bounds), decimal exponent out
inline void digits(char* buf, int& len, int& dec_exp, Fp m_minus, Fp v, Fp m_plus) {
  const CachedPower& c = cached_power(m_plus.e);
  const Fp ck{c.f, c.e};
  const Fp w = mul(v, ck), wm = mul(m_minus, ck), wp = mul(m_plus, ck);
  const Fp lo{wm.f + 1, wm.e}, hi{wp.f - 1, wp.e};
  dec_exp = -c.k;
  uint64_t delta = sub(hi, lo).f, dist = sub(hi, w).f;
  const Fp one{uint64_t{1} << -hi.e, hi.e};
  uint32_t p1 = static_cast<uint32_t>(hi.f >> -one.e);
  uint64_t p2 = hi.f & (one.f - 1);
  uint32_t pow10 = 1;
  int n = largest_pow10(p1, pow10);
  len = 0;
  while (n > 0) {
    const uint32_t d = p1 / pow10, r = p1 % pow10;
    buf[len++] = static_cast<char>('0' + d);
    p1 = r;
    --n;
    const uint64_t rest = (uint64_t{p1} << -one.e) + p2;
    if (rest <= delta) {
      dec_exp += n;
      round_last(buf, len, dist, delta, rest, uint64_t{pow10} << -one.e);
      return;
    }
    pow10 /= 10;
  }
  int m = 0;
  for (;;) {
    p2 *= 10;
    const uint64_t d = p2 >> -one.e, r = p2 & (one.f - 1);
    buf[len++] = static_cast<char>('0' + d);
    p2 = r;
    ++m;
    delta *= 10;
    dist *= 10;
    if (p2 <= delta) break;
  }
  dec_exp -= m;
  round_last(buf, len, dist, delta, p2, one.f);
}

// v > 0, finite: shortest (Grisu2) digit string and decimal exponent
inline void shortest(double v, char* buf, int& len, int& dec_exp) {
  uint64_t bits;
  std::memcpy(&bits, &v, 8);
  const uint64_t F = bits & ((uint64_t{1} << 52) - 1);
  const int E = static_cast<int>(bits >> 52);
  const Fp x = E == 0 ? Fp{F, 1 - 1075} : Fp{F + (uint64_t{1} << 52), E - 1075};
  const bool closer = F == 0 && E > 1;  // the lower neighbour is nearer
  const Fp mp{2 * x.f + 1, x.e - 1};
  const Fp mm = closer ? Fp{4 * x.f - 1, x.e - 2} : Fp{2 * x.f - 1, x.e - 1};
  const Fp wp = normalize(mp);
  const Fp wm = normalize_to(mm, wp.e);
  digits(buf, len, dec_exp, wm, normalize(x), wp);
}
}  // namespace grisu

/// Minimal ordered JSON value written in nlohmann's dump() layout.
class JOut {
 public:
  enum Kind { Null, Bool, Int, Dbl, Str, Arr, Obj };
  JOut() = default;
  static JOut null() { return JOut(); }
  static JOut boolean(bool v) { JOut j; j.k_ = Bool; j.b_ = v; return j; }
  static JOut integer(long long v) { JOut j; j.k_ = Int; j.i_ = v; return j; }
  static JOut number(double v) { JOut j; j.k_ = Dbl; j.d_ = v; return j; }
  static JOut string(const std::string& v) { JOut j; j.k_ = Str; j.s_ = v; return j; }
  static JOut array() { JOut j; j.k_ = Arr; return j; }
  static JOut object() { JOut j; j.k_ = Obj; return j; }
  static JOut vec3(const Vec3& v) { return array().push(number(v.x)).push(number(v.y)).push(number(v.z)); }
  static JOut bands(const BandArray& a) {
    JOut j = array();
    for (double x : a) j.push(number(x));
    return j;
  }
  template <typename T>
  static JOut ints(const T& v) {
    JOut j = array();
    for (auto x : v) j.push(integer(static_cast<long long>(x)));
    return j;
  }
  JOut& push(JOut v) { arr_.push_back(std::move(v)); return *this; }
  JOut& set(const std::string& key, JOut v) {
    for (auto& kv : obj_)
      if (kv.first == key) { kv.second = std::move(v); return *this; }
    obj_.emplace_back(key, std::move(v));
    return *this;
  }
  /// indent < 0: compact (dump()); otherwise dump(indent).
  std::string dump(int indent = -1) const {
    std::string out;
    write(out, indent, 0);
    return out;
  }

 private:
  Kind k_ = Null;
  bool b_ = false;
  long long i_ = 0;
  double d_ = 0.0;
  std::string s_;
  std::vector<JOut> arr_;
  std::vector<std::pair<std::string, JOut>> obj_;

  static void escape(std::string& out, const std::string& s) {
    out += '"';
    for (unsigned char c : s) {
      switch (c) {
        case '"': out += "\\\""; break;
        case '\\': out += "\\\\"; break;
        case '\b': out += "\\b"; break;
        case '\f': out += "\\f"; break;
        case '\n': out += "\\n"; break;
        case '\r': out += "\\r"; break;
        case '\t': out += "\\t"; break;
        default:
          if (c < 0x20) {
            char b[8];
            std::snprintf(b, sizeof b, "\\u%04x", c);
            out += b;
          } else {
            out += static_cast<char>(c);
          }
      }
    }
    out += '"';
  }

  // Grisu2 digits laid out with nlohmann's rules (decimal notation for
  // decimal exponents in (-4, 15], ".0" on integral values, otherwise
  // d.ddde+XX with at least two exponent digits)
  static void number_text(std::string& out, double v) {
    if (!std::isfinite(v)) { out += "null"; return; }
    if (v == 0.0) { out += std::signbit(v) ? "-0.0" : "0.0"; return; }
    const std::string sign = v < 0.0 ? "-" : "";
    char buf[32];
    int len = 0, dec_exp = 0;
    grisu::shortest(std::fabs(v), buf, len, dec_exp);
    const std::string digits(buf, static_cast<std::size_t>(len));
    const int k = len;
    const int n = len + dec_exp;  // decimal point after n digits
    out += sign;
    if (k <= n && n <= 15) {
      out += digits;
      out.append(static_cast<std::size_t>(n - k), '0');
      out += ".0";
    } else if (0 < n && n <= 15) {
      out += digits.substr(0, n);
      out += '.';
      out += digits.substr(n);
    } else if (-4 < n && n <= 0) {
      out += "0.";
      out.append(static_cast<std::size_t>(-n), '0');
      out += digits;
    } else {
      out += digits.substr(0, 1);
      if (k > 1) {
        out += '.';
        out += digits.substr(1);
      }
      const int x = n - 1;
      char eb[16];
      std::snprintf(eb, sizeof eb, "e%c%02d", x < 0 ? '-' : '+', x < 0 ? -x : x);
      out += eb;
    }
  }

  void write(std::string& out, int indent, int level) const {
    const bool pretty = indent >= 0;
    auto nl = [&](int lv) {
      if (!pretty) return;
      out += '\n';
      out.append(static_cast<std::size_t>(indent * lv), ' ');
    };
    switch (k_) {
      case Null: out += "null"; break;
      case Bool: out += b_ ? "true" : "false"; break;
      case Int: out += std::to_string(i_); break;
      case Dbl: number_text(out, d_); break;
      case Str: escape(out, s_); break;
      case Arr:
        if (arr_.empty()) { out += "[]"; break; }
        out += '[';
        for (std::size_t i = 0; i < arr_.size(); ++i) {
          nl(level + 1);
          arr_[i].write(out, indent, level + 1);
          if (i + 1 < arr_.size()) out += ',';
        }
        nl(level);
        out += ']';
        break;
      case Obj:
        if (obj_.empty()) { out += "{}"; break; }
        out += '{';
        for (std::size_t i = 0; i < obj_.size(); ++i) {
          nl(level + 1);
          escape(out, obj_[i].first);
          out += pretty ? ": " : ":";
          obj_[i].second.write(out, indent, level + 1);
          if (i + 1 < obj_.size()) out += ',';
        }
        nl(level);
        out += '}';
        break;
    }
  }
};

inline void write_text(const std::string& path, const std::string& text) {
  std::ofstream out(path, std::ios::binary);
  if (!out) throw std::runtime_error("cannot open for writing: " + path);
  out << text;
  if (!out) throw std::runtime_error("write failed: " + path);
}

/// Removes already written files when a later write fails (pipeline.cpp:122-136).
class OutputSet {
 public:
  void note(const std::string& p) { written_.push_back(p); }
  const std::vector<std::string>& files() const { return written_; }
  void rollback() {
    for (const std::string& p : written_) {
      std::error_code ec;
      std::filesystem::remove(p, ec);
    }
  }

 private:
  std::vector<std::string> written_;
};

inline JOut image_json(const ImageSource& im) {  // pipeline.cpp:59-72
  JOut j = JOut::object();
  j.set("position", JOut::vec3(im.position));
  j.set("distance_m", JOut::number(im.distance));
  j.set("order", JOut::integer(im.order));
  j.set("ray_count", JOut::integer(im.ray_count));
  j.set("band_energy", JOut::bands(im.band_energy));
  j.set("face_path", JOut::ints(im.face_path));
  j.set("projection", im.projection ? JOut::vec3(*im.projection) : JOut::null());
  return j;
}

inline JOut metric_json(const MetricValue& m) {
  return JOut::object().set("value", JOut::number(m.value)).set("reliable", JOut::boolean(m.reliable));
}

inline JOut factors_json(const PerceptiveFactors& f) {  // pipeline.cpp:114-124
  return JOut::object()
      .set("edt_s", metric_json(f.edt_s))
      .set("t30_s", metric_json(f.t30_s))
      .set("spl_db", metric_json(f.spl_db))
      .set("c80_db", metric_json(f.c80_db))
      .set("d50_pct", metric_json(f.d50_pct))
      .set("ts_ms", metric_json(f.ts_ms));
}

inline JOut run_config_json(const RunConfig& c) {  // pipeline.cpp:188-203
  return JOut::object()
      .set("source", JOut::object()
                         .set("position", JOut::vec3(c.source.position))
                         .set("ray_count", JOut::integer(c.source.ray_count)))
      .set("receiver", JOut::object()
                           .set("center", JOut::vec3(c.receiver.center))
                           .set("radius", JOut::number(c.receiver.radius)))
      .set("air", JOut::object()
                      .set("enabled", JOut::boolean(c.air.enabled))
                      .set("temperature_c", JOut::number(c.air.temperature_c))
                      .set("relative_humidity", JOut::number(c.air.relative_humidity))
                      .set("pressure_kpa", JOut::number(c.air.pressure_kpa)))
      .set("speed_of_sound", JOut::number(c.speed_of_sound))
      .set("sample_rate", JOut::number(c.sample_rate))
      .set("merge_coplanar", JOut::boolean(c.merge_coplanar))
      .set("deterministic", JOut::boolean(c.deterministic));
}

}  // namespace detail

// ------------------------------------------------------------------ WAV (wav.hpp)
/// write_wav (wav.cpp:37-66): RIFF/WAVE, IEEE float (format 3), mono, 32 bit.
inline void write_wav(const std::string& path, const std::vector<double>& samples, double sample_rate) {
  std::ofstream out(path, std::ios::binary);
  if (!out) throw std::runtime_error("cannot open for writing: " + path);
  auto u32 = [&](uint32_t v) {
    const char b[4] = {static_cast<char>(v & 0xff), static_cast<char>((v >> 8) & 0xff),
                       static_cast<char>((v >> 16) & 0xff), static_cast<char>((v >> 24) & 0xff)};
    out.write(b, 4);
  };
  auto u16 = [&](uint16_t v) {
    const char b[2] = {static_cast<char>(v & 0xff), static_cast<char>((v >> 8) & 0xff)};
    out.write(b, 2);
  };
  const uint32_t data_bytes = static_cast<uint32_t>(samples.size() * sizeof(float));
  const uint32_t rate = static_cast<uint32_t>(sample_rate);
  out.write("RIFF", 4);
  u32(36 + data_bytes);
  out.write("WAVE", 4);
  out.write("fmt ", 4);
  u32(16);
  u16(3);
  u16(1);
  u32(rate);
  u32(rate * static_cast<uint32_t>(sizeof(float)));
  u16(static_cast<uint16_t>(sizeof(float)));
  u16(32);
  out.write("data", 4);
  u32(data_bytes);
  for (double v : samples) {
    const float f = static_cast<float>(v);
    char b[4];
    std::memcpy(b, &f, 4);
    out.write(b, 4);
  }
  if (!out) throw std::runtime_error("write failed: " + path);
}

/// WavData / read_wav (wav.hpp:13-18, wav.cpp:68-115): mono 32-bit float
/// files as written above; std::runtime_error for anything else.
struct WavData {
  std::vector<double> samples;
  double sample_rate = 0.0;
};

inline WavData read_wav(const std::string& path) {
  std::ifstream in(path, std::ios::binary);
  if (!in) throw std::runtime_error("cannot open: " + path);
  auto u32 = [&]() {
    unsigned char b[4] = {0, 0, 0, 0};
    in.read(reinterpret_cast<char*>(b), 4);
    return static_cast<uint32_t>(b[0] | (b[1] << 8) | (b[2] << 16) | (static_cast<uint32_t>(b[3]) << 24));
  };
  auto u16 = [&]() {
    unsigned char b[2] = {0, 0};
    in.read(reinterpret_cast<char*>(b), 2);
    return static_cast<uint16_t>(b[0] | (b[1] << 8));
  };
  char tag[5] = {};
  in.read(tag, 4);
  if (std::strncmp(tag, "RIFF", 4) != 0) throw std::runtime_error("not a RIFF file: " + path);
  u32();
  in.read(tag, 4);
  if (std::strncmp(tag, "WAVE", 4) != 0) throw std::runtime_error("not a WAVE file: " + path);
  WavData wav;
  uint16_t format = 0, channels = 0, bits = 0;
  while (in.read(tag, 4)) {
    const uint32_t size = u32();
    if (std::strncmp(tag, "fmt ", 4) == 0) {
      format = u16();
      channels = u16();
      wav.sample_rate = u32();
      u32();
      u16();
      bits = u16();
      if (size > 16) in.seekg(size - 16, std::ios::cur);
    } else if (std::strncmp(tag, "data", 4) == 0) {
      if (format != 3 || channels != 1 || bits != 32)
        throw std::runtime_error("unsupported WAV layout (need mono 32-bit float): " + path);
      const std::size_t count = size / sizeof(float);
      wav.samples.resize(count);
      for (std::size_t i = 0; i < count; ++i) {
        float f = 0.0f;
        in.read(reinterpret_cast<char*>(&f), 4);
        wav.samples[i] = f;
      }
      return wav;
    } else {
      in.seekg(size + (size & 1), std::ios::cur);
    }
  }
  throw std::runtime_error("no data chunk in " + path);
}

// ------------------------------------------------------------------ decay curves (metrics.hpp)
struct DecayPoint {
  double time_s = 0.0;
  double level_db = 0.0;
};

/// schroeder(const PulseTrains&) per band on the GPU (metrics.cpp:125-134);
/// bands without events get an empty curve.
inline std::array<std::vector<DecayPoint>, kNumBands> schroeder_bands(const PulseTrains& trains) {
  std::vector<int64_t> off(kNumBands + 1, 0);
  std::vector<double> a;
  for (int b = 0; b < kNumBands; ++b) {
    for (const PulseEvent& e : trains[b].events) a.push_back(e.amplitude);
    off[b + 1] = static_cast<int64_t>(a.size());
  }
  std::vector<double> level(a.size());
  detail::check(rr_band_schroeder(Device::get(0).handle(), off.data(), a.data(), level.data()));
  std::array<std::vector<DecayPoint>, kNumBands> out;
  for (int b = 0; b < kNumBands; ++b) {
    const auto& ev = trains[b].events;
    for (std::size_t i = 0; i < ev.size(); ++i) out[b].push_back({ev[i].time_s, level[off[b] + i]});
  }
  return out;
}

// ------------------------------------------------------------------ trains and metrics files (pipeline.hpp:84-87)
/// write_band_trains_csv (pipeline.cpp:516-526): "band,time_s,amplitude".
inline void write_band_trains_csv(const std::string& path, const PulseTrains& trains) {
  std::string csv = "band,time_s,amplitude\n";
  for (const BandPulseTrain& t : trains)
    for (const PulseEvent& e : t.events)
      csv += std::to_string(t.band) + ',' + detail::format_double(e.time_s) + ',' + detail::format_double(e.amplitude) +
             '\n';
  detail::write_text(path, csv);
}

/// load_band_trains_csv (pipeline.cpp:528-553): the file back into trains;
/// std::runtime_error naming the line for malformed rows or bad bands.
inline PulseTrains load_band_trains_csv(const std::string& path) {
  std::ifstream in(path);
  if (!in) throw std::runtime_error("cannot open: " + path);
  PulseTrains trains;
  for (int b = 0; b < kNumBands; ++b) trains[b].band = b;
  std::string line;
  std::getline(in, line);  // header
  int line_no = 1;
  while (std::getline(in, line)) {
    ++line_no;
    if (line.empty()) continue;
    std::istringstream ls(line);
    std::string band_text, time_text, amp_text;
    if (!std::getline(ls, band_text, ',') || !std::getline(ls, time_text, ',') || !std::getline(ls, amp_text))
      throw std::runtime_error("band_trains.csv line " + std::to_string(line_no) + " is malformed");
    const int band = std::stoi(band_text);
    if (band < 0 || band >= kNumBands)
      throw std::runtime_error("band_trains.csv line " + std::to_string(line_no) + ": bad band index");
    trains[band].events.push_back({std::stod(time_text), std::stod(amp_text)});
  }
  return trains;
}

/// write_metrics_json (pipeline.cpp:555-565): per band centre and "mid".
inline void write_metrics_json(const std::string& path, const BandFactors& factors) {
  detail::JOut j = detail::JOut::object();
  for (int b = 0; b < kNumBands; ++b) j.set(detail::band_name(kBandCentersHz[b]), detail::factors_json(factors.bands[b]));
  j.set("mid", detail::factors_json(factors.mid));
  detail::write_text(path, j.dump(2) + "\n");
}

// ------------------------------------------------------------------ run artifacts (pipeline.hpp:40-45)
/// write_run_artifacts (pipeline.cpp:208-325): every file of a trace run
/// into config.output_dir; on failure the files written so far are removed.
inline std::vector<std::string> write_run_artifacts(const RunConfig& config, const RunArtifacts& a) {
  namespace fs = std::filesystem;
  using detail::JOut;
  fs::create_directories(config.output_dir);
  auto out_path = [&](const std::string& name) { return (fs::path(config.output_dir) / name).string(); };
  detail::OutputSet outputs;
  try {
    {
      JOut doc = JOut::object();
      doc.set("config", detail::run_config_json(config));
      doc.set("max_range_m", JOut::number(a.trace.max_range));
      JOut images = JOut::array();
      for (const ImageSource& im : a.images) images.push(detail::image_json(im));
      doc.set("images", std::move(images));
      const std::string p = out_path("image_sources.json");
      detail::write_text(p, doc.dump(2) + "\n");
      outputs.note(p);
    }
    {
      std::string csv = "x,y,z,distance_m,order,ray_count";
      for (double c : kBandCentersHz) csv += ",e" + detail::band_name(c);
      csv += ",proj_x,proj_y,proj_z\n";
      for (const ImageSource& im : a.images) {
        csv += detail::format_double(im.position.x) + ',' + detail::format_double(im.position.y) + ',' +
               detail::format_double(im.position.z) + ',' + detail::format_double(im.distance) + ',' +
               std::to_string(im.order) + ',' + std::to_string(im.ray_count);
        for (double e : im.band_energy) csv += ',' + detail::format_double(e);
        if (im.projection) {
          csv += ',' + detail::format_double(im.projection->x) + ',' + detail::format_double(im.projection->y) + ',' +
                 detail::format_double(im.projection->z);
        } else {
          csv += ",,,";
        }
        csv += '\n';
      }
      const std::string p = out_path("image_sources.csv");
      detail::write_text(p, csv);
      outputs.note(p);
    }
    {
      const std::string p = out_path("rir.wav");
      write_wav(p, a.rir.samples, a.rir.sample_rate);
      outputs.note(p);
    }
    {
      const std::string p = out_path("band_trains.csv");
      write_band_trains_csv(p, a.trains);
      outputs.note(p);
    }
    {
      const std::string p = out_path("metrics.json");
      write_metrics_json(p, a.metrics);
      outputs.note(p);
    }
    {
      const auto curves = schroeder_bands(a.trains);
      for (int b = 0; b < kNumBands; ++b) {
        if (a.trains[b].events.empty()) continue;
        std::string csv = "time_s,level_db\n";
        for (const DecayPoint& pt : curves[b])
          csv += detail::format_double(pt.time_s) + ',' + detail::format_double(pt.level_db) + '\n';
        const std::string p = out_path("decay_" + detail::band_name(kBandCentersHz[b]) + ".csv");
        detail::write_text(p, csv);
        outputs.note(p);
      }
    }
    if (config.dump_captures) {
      std::string lines;
      for (const Capture& c : a.trace.captures) {
        JOut j = JOut::object();
        j.set("ray_index", JOut::integer(c.ray_index));
        j.set("point", JOut::vec3(c.point));
        j.set("incoming_dir", JOut::vec3(c.incoming_dir));
        j.set("path_length_m", JOut::number(c.path_length));
        j.set("band_multiplier", JOut::bands(c.band_multiplier));
        j.set("face_history", JOut::ints(c.face_history));
        lines += j.dump() + '\n';
      }
      const std::string p = out_path("captures.jsonl");
      detail::write_text(p, lines);
      outputs.note(p);
    }
    if (config.dump_tree_stats) {
      JOut j = JOut::object()
                   .set("node_count", JOut::integer(static_cast<long long>(a.tree.node_count())))
                   .set("leaf_count", JOut::integer(static_cast<long long>(a.tree.leaf_count())))
                   .set("depth", JOut::integer(a.tree.depth()))
                   .set("build_seconds", JOut::number(a.tree_build_seconds));
      const std::string p = out_path("tree_stats.json");
      detail::write_text(p, j.dump(2) + "\n");
      outputs.note(p);
    }
    {
      JOut timings = JOut::object();
      for (const StageTiming& t : a.timings) timings.set(t.name, JOut::number(t.seconds));
      timings.set("total", JOut::number(a.total_seconds));
      BandArray alpha{};
      for (int b = 0; b < kNumBands; ++b) alpha[b] = air_alpha_db_per_m(config.air, kBandCentersHz[b]);
      JOut j = JOut::object();
      j.set("timings_s", std::move(timings));
      j.set("mesh", JOut::object()
                        .set("vertices", JOut::integer(static_cast<long long>(a.mesh.vertices.size())))
                        .set("faces", JOut::integer(static_cast<long long>(a.mesh.faces.size())))
                        .set("degenerate_skipped", JOut::integer(static_cast<long long>(a.load_report.degenerate_skipped))));
      j.set("tree", JOut::object()
                        .set("node_count", JOut::integer(static_cast<long long>(a.tree.node_count())))
                        .set("depth", JOut::integer(a.tree.depth()))
                        .set("build_seconds", JOut::number(a.tree_build_seconds)));
      j.set("trace", JOut::object()
                         .set("ray_count", JOut::integer(config.source.ray_count))
                         .set("iterations", JOut::integer(a.trace.iterations))
                         .set("truncated", JOut::boolean(a.trace.truncated))
                         .set("escaped", JOut::integer(static_cast<long long>(a.trace.escaped)))
                         .set("out_of_range", JOut::integer(static_cast<long long>(a.trace.out_of_range)))
                         .set("captures", JOut::integer(static_cast<long long>(a.trace.captures.size())))
                         .set("max_range_m", JOut::number(a.trace.max_range)));
      j.set("image_sources", JOut::object().set("count", JOut::integer(static_cast<long long>(a.images.size()))));
      j.set("air", JOut::object().set("enabled", JOut::boolean(config.air.enabled)).set("alpha_db_per_m", JOut::bands(alpha)));
      j.set("deterministic", JOut::boolean(config.deterministic));
      const std::string p = out_path("run_report.json");
      detail::write_text(p, j.dump(2) + "\n");
      outputs.note(p);
    }
  } catch (...) {
    outputs.rollback();
    throw;
  }
  return outputs.files();
}

// ------------------------------------------------------------------ shoebox files (pipeline.hpp:63-88)
/// write_oracle_artifacts (pipeline.cpp:383-435).
inline std::vector<std::string> write_oracle_artifacts(const OracleConfig& config,
                                                       const std::vector<OracleImageSource>& images) {
  namespace fs = std::filesystem;
  using detail::JOut;
  fs::create_directories(config.output_dir);
  detail::OutputSet outputs;
  try {
    JOut doc = JOut::object();
    doc.set("config", JOut::object()
                          .set("box_dimensions", JOut::vec3(config.box.dimensions))
                          .set("source", JOut::object()
                                             .set("position", JOut::vec3(config.source_position))
                                             .set("ray_count", JOut::integer(config.ray_count)))
                          .set("receiver", JOut::object()
                                               .set("center", JOut::vec3(config.receiver.center))
                                               .set("radius", JOut::number(config.receiver.radius)))
                          .set("max_distance_m", JOut::number(config.resolved_max_distance())));
    JOut list = JOut::array();
    for (const OracleImageSource& im : images)
      list.push(JOut::object()
                    .set("position", JOut::vec3(im.position))
                    .set("distance_m", JOut::number(im.distance))
                    .set("order", JOut::integer(im.order))
                    .set("wall_hits", JOut::ints(im.wall_hits))
                    .set("band_energy", JOut::bands(im.band_energy)));
    doc.set("images", std::move(list));
    const std::string jp = (fs::path(config.output_dir) / "oracle_image_sources.json").string();
    detail::write_text(jp, doc.dump(2) + "\n");
    outputs.note(jp);
    std::string csv = "x,y,z,distance_m,order";
    for (double c : kBandCentersHz) csv += ",e" + detail::band_name(c);
    csv += '\n';
    for (const OracleImageSource& im : images) {
      csv += detail::format_double(im.position.x) + ',' + detail::format_double(im.position.y) + ',' +
             detail::format_double(im.position.z) + ',' + detail::format_double(im.distance) + ',' +
             std::to_string(im.order);
      for (double e : im.band_energy) csv += ',' + detail::format_double(e);
      csv += '\n';
    }
    const std::string cp = (fs::path(config.output_dir) / "oracle_image_sources.csv").string();
    detail::write_text(cp, csv);
    outputs.note(cp);
  } catch (...) {
    outputs.rollback();
    throw;
  }
  return outputs.files();
}

/// LoadedImageSources / load_image_sources_json (pipeline.hpp:66-76,
/// pipeline.cpp:438-466): a traced image_sources.json with its run config.
struct LoadedImageSources {
  std::vector<ImageSource> images;
  Vec3 source_position{};
  int ray_count = 0;
  Vec3 receiver_center{};
  double receiver_radius = 0.0;
};

inline LoadedImageSources load_image_sources_json(const std::string& path) {
  using detail::Json;
  const Json doc = detail::JsonReader(detail::read_file(path, "image sources")).parse();
  auto at = [&](const Json& o, const char* k) -> const Json& {
    const Json* v = o.kind == Json::Obj ? o.get(k) : nullptr;
    if (!v) throw std::runtime_error(std::string("image sources: missing field '") + k + "'");
    return *v;
  };
  auto num = [](const Json& v) {
    if (v.kind != Json::Num) throw std::runtime_error("image sources: expected a number");
    return v.num;
  };
  auto vec3 = [&](const Json& v) {
    if (v.kind != Json::Arr || v.arr.size() < 3) throw std::runtime_error("image sources: expected a 3-vector");
    return Vec3{num(v.arr[0]), num(v.arr[1]), num(v.arr[2])};
  };
  LoadedImageSources out;
  const Json& cfg = at(doc, "config");
  out.source_position = vec3(at(at(cfg, "source"), "position"));
  out.ray_count = static_cast<int>(num(at(at(cfg, "source"), "ray_count")));
  out.receiver_center = vec3(at(at(cfg, "receiver"), "center"));
  out.receiver_radius = num(at(at(cfg, "receiver"), "radius"));
  for (const Json& j : at(doc, "images").arr) {
    ImageSource im;
    im.position = vec3(at(j, "position"));
    im.distance = num(at(j, "distance_m"));
    im.order = static_cast<int>(num(at(j, "order")));
    im.ray_count = static_cast<int>(num(at(j, "ray_count")));
    const Json& e = at(j, "band_energy");
    for (int b = 0; b < kNumBands; ++b) im.band_energy[b] = num(e.arr.at(b));
    for (const Json& f : at(j, "face_path").arr) im.face_path.push_back(static_cast<int>(num(f)));
    const Json& p = at(j, "projection");
    if (p.kind != Json::Null) im.projection = vec3(p);
    out.images.push_back(std::move(im));
  }
  return out;
}

/// check_comparable (pipeline.cpp:468-487): std::invalid_argument when the
/// traced set was made under another source / receiver / ray count.
inline void check_comparable(const OracleConfig& oracle, const LoadedImageSources& traced) {
  const double tol = 1e-12;
  auto dist = [](const Vec3& a, const Vec3& b) {
    const double dx = a.x - b.x, dy = a.y - b.y, dz = a.z - b.z;
    return std::sqrt((dx * dx + dy * dy) + dz * dz);
  };
  if (dist(oracle.source_position, traced.source_position) > tol)
    throw std::invalid_argument("config mismatch: traced set was computed with a different source position");
  if (dist(oracle.receiver.center, traced.receiver_center) > tol)
    throw std::invalid_argument("config mismatch: traced set was computed with a different receiver center");
  if (std::abs(oracle.receiver.radius - traced.receiver_radius) > tol)
    throw std::invalid_argument("config mismatch: traced set was computed with a different receiver radius");
  if (oracle.ray_count != traced.ray_count)
    throw std::invalid_argument("config mismatch: traced set was computed with a different ray count");
}

/// write_comparison_report (pipeline.cpp:489-514).
inline std::string write_comparison_report(const std::string& path, const MatchReport& r) {
  using detail::JOut;
  JOut j = JOut::object();
  j.set("matched_count", JOut::integer(static_cast<long long>(r.matched.size())));
  j.set("unmatched_oracle_count", JOut::integer(static_cast<long long>(r.unmatched_oracle.size())));
  j.set("unmatched_traced_count", JOut::integer(static_cast<long long>(r.unmatched_traced.size())));
  j.set("max_position_error_m", JOut::number(r.max_position_error));
  j.set("rms_energy_error_db", JOut::bands(r.rms_energy_error_db));
  j.set("pos_tol_m", JOut::number(r.pos_tol));
  j.set("energy_tol_db", JOut::number(r.energy_tol_db));
  JOut matched = JOut::array();
  for (const MatchedImage& m : r.matched)
    matched.push(JOut::object()
                     .set("oracle_index", JOut::integer(m.oracle_index))
                     .set("traced_indices", JOut::ints(m.traced_indices))
                     .set("order", JOut::integer(m.order))
                     .set("position_error_m", JOut::number(m.position_error))
                     .set("energy_delta_db", JOut::bands(m.energy_delta_db)));
  j.set("matched", std::move(matched));
  j.set("unmatched_oracle", JOut::ints(r.unmatched_oracle));
  j.set("unmatched_traced", JOut::ints(r.unmatched_traced));
  detail::write_text(path, j.dump(2) + "\n");
  return path;
}

}  // namespace roomray_b200

#endif  // ROOMRAY_B200_ARTIFACTS_HPP
