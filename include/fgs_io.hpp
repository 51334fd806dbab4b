// fgs_io.hpp — header-only host I/O around the rasterizer: the reference's scene / camera /
// image file formats, so its `render` / `bench` callers can drive the B200
// path unchanged.
//
//   load_ply / save_ply        the format of src/ply_io.cpp:40-145 (3DGS binary_little_endian layout)
//   load_cameras / save_cameras the format of src/camera_io.cpp:25-127 (camera JSON)
//   write_image (PPM / PNG)    the formats of src/image_io.cpp:19-160 (8-bit, round half to even)
// Only the file formats and the error messages follow the reference; the readers and writers are
// this repo's own (schema-driven PLY columns, a byte sink for PNG / zlib).
//
// Errors are std::runtime_error with the reference's messages. The camera JSON reader is a
// small recursive-descent parser (the reference uses nlohmann-json, absent here); rotation
// re-orthonormalisation uses the polar factor (Newton iteration), which equals the reference's
// U V^T from the SVD.
#ifndef FGS_IO_HPP_
#define FGS_IO_HPP_

#include <algorithm>
#include <array>
#include <cctype>
#include <cmath>
#include <cstdint>
#include <cstdio>
#include <cstring>
#include <fstream>
#include <map>
#include <memory>
#include <sstream>
#include <stdexcept>
#include <string>
#include <vector>

#include "fgs.h"
#include "fgs.hpp"

namespace fgs {
namespace io {

// ---------------------------------------------------------------------------------------
// Scene PLY: the 3DGS export layout the reference reads and writes (src/ply_io.cpp:40-145) --
// a binary little-endian `vertex` element of float properties, in one of two fixed orders.
//
// A layout is a schema: one Column per vertex property saying where its value goes in the
// structure-of-arrays scene (Gaussian field and component; normals are dropped). Reading parses
// the header into a PlyHeader, matches the property list against the schemas, then loads the
// whole payload at once and scatters it column by column.

enum class PlyField : uint8_t { Mean, Normal, Sh, Opacity, LogScale, Rotation };

struct PlyColumn {
  std::string name;
  PlyField field;
  int index;  // component (mean / scale / rotation) or SH slot channel * 16 + basis
};

// with_rest: the full 62-float layout; without: the 17-float DC-only variant. The PLY keeps
// f_rest_{c*15 + j - 1} for basis j >= 1 of channel c (channel-major), the scene [c*16 + j].
inline std::vector<PlyColumn> ply_schema(bool with_rest) {
  std::vector<PlyColumn> cols;
  const char* axis = "xyz";
  for (int k = 0; k < 3; ++k) cols.push_back({std::string(1, axis[k]), PlyField::Mean, k});
  for (int k = 0; k < 3; ++k) cols.push_back({std::string("n") + axis[k], PlyField::Normal, k});
  for (int c = 0; c < 3; ++c) cols.push_back({"f_dc_" + std::to_string(c), PlyField::Sh, c * 16});
  if (with_rest)
    for (int r = 0; r < 45; ++r) cols.push_back({"f_rest_" + std::to_string(r), PlyField::Sh, (r / 15) * 16 + r % 15 + 1});
  cols.push_back({"opacity", PlyField::Opacity, 0});
  for (int k = 0; k < 3; ++k) cols.push_back({"scale_" + std::to_string(k), PlyField::LogScale, k});
  for (int k = 0; k < 4; ++k) cols.push_back({"rot_" + std::to_string(k), PlyField::Rotation, k});
  return cols;
}

inline std::vector<std::string> ply_names(const std::vector<PlyColumn>& cols) {
  std::vector<std::string> v;
  for (const auto& c : cols) v.push_back(c.name);
  return v;
}
inline std::vector<std::string> ply_full_properties() { return ply_names(ply_schema(true)); }
inline std::vector<std::string> ply_dc_properties() { return ply_names(ply_schema(false)); }

inline std::string join(const std::vector<std::string>& v) {
  std::string s;
  for (size_t i = 0; i < v.size(); ++i) s += (i ? "," : "") + v[i];
  return s;
}

struct PlyRead {
  SceneSoA scene;
  std::vector<std::string> warnings;
};

struct PlyHeader {
  bool format_seen = false;
  size_t vertices = 0;
  std::vector<std::string> properties;
  std::streamoff payload = 0;  // byte offset of the first vertex
};

inline std::vector<std::string> split_words(const std::string& line) {
  std::vector<std::string> w;
  std::istringstream is(line);
  for (std::string t; is >> t;) w.push_back(t);
  return w;
}

inline PlyHeader read_ply_header(std::istream& in, const std::string& path) {
  std::string line;
  auto next = [&]() {
    if (!std::getline(in, line)) return false;
    if (!line.empty() && line.back() == '\r') line.pop_back();
    return true;
  };
  if (!next() || line != "ply") throw std::runtime_error("load_ply: " + path + " is not a PLY file");
  PlyHeader h;
  while (next() && line != "end_header") {
    const std::vector<std::string> w = split_words(line);
    const std::string key = w.empty() ? std::string() : w[0];
    const std::string a1 = w.size() > 1 ? w[1] : std::string(), a2 = w.size() > 2 ? w[2] : std::string();
    if (key.empty() || key == "comment" || key == "obj_info") continue;
    if (key == "format") {
      if (a1 != "binary_little_endian")
        throw std::runtime_error("load_ply: binary_little_endian required, got format '" + a1 + "'");
      h.format_seen = true;
    } else if (key == "element") {
      if (a1 != "vertex") throw std::runtime_error("load_ply: unsupported element '" + a1 + "'");
      h.vertices = static_cast<size_t>(std::stoull(a2.empty() ? std::string("0") : a2));
    } else if (key == "property") {
      if (a1 != "float")
        throw std::runtime_error("load_ply: property '" + a2 + "' has type '" + a1 + "', expected float");
      h.properties.push_back(a2);
    } else {
      throw std::runtime_error("load_ply: unexpected header line '" + line + "'");
    }
  }
  if (!h.format_seen) throw std::runtime_error("load_ply: missing format line (binary_little_endian required)");
  h.payload = static_cast<std::streamoff>(in.tellg());
  return h;
}

inline PlyRead load_ply(const std::string& path) {
  std::ifstream in(path, std::ios::binary);
  if (!in) throw std::runtime_error("load_ply: cannot open " + path);
  const PlyHeader h = read_ply_header(in, path);
  PlyRead out;
  std::vector<PlyColumn> schema;
  for (bool rest : {true, false}) {
    std::vector<PlyColumn> cand = ply_schema(rest);
    if (ply_names(cand) == h.properties) {
      schema = std::move(cand);
      if (!rest) out.warnings.push_back("load_ply: f_rest_* properties missing; higher-order SH set to zero");
      break;
    }
  }
  if (schema.empty())
    throw std::runtime_error("load_ply: unknown property layout; expected [" + join(ply_full_properties()) +
                             "] (or the f_rest-free variant), found [" + join(h.properties) + "]");
  // the whole payload in one read; short files report where the data ran out
  const size_t stride = schema.size(), n = h.vertices;
  std::vector<float> block(n * stride);
  in.read(reinterpret_cast<char*>(block.data()), static_cast<std::streamsize>(block.size() * sizeof(float)));
  const std::streamsize got = in.gcount();
  if (static_cast<size_t>(got) != block.size() * sizeof(float))
    throw std::runtime_error("load_ply: truncated payload at byte offset " + std::to_string(h.payload + got));
  SceneSoA& s = out.scene;
  s.means.assign(n * 3, 0.f);
  s.rotations.assign(n * 4, 0.f);
  s.log_scales.assign(n * 3, 0.f);
  s.opacity_logits.assign(n, 0.f);
  s.sh.assign(n * 48, 0.f);
  for (size_t col = 0; col < stride; ++col) {
    const PlyColumn& c = schema[col];
    float* dst = nullptr;
    size_t width = 0;
    switch (c.field) {
      case PlyField::Mean: dst = s.means.data(); width = 3; break;
      case PlyField::Sh: dst = s.sh.data(); width = 48; break;
      case PlyField::Opacity: dst = s.opacity_logits.data(); width = 1; break;
      case PlyField::LogScale: dst = s.log_scales.data(); width = 3; break;
      case PlyField::Rotation: dst = s.rotations.data(); width = 4; break;
      case PlyField::Normal: continue;
    }
    const float* src = block.data() + col;
    for (size_t v = 0; v < n; ++v) dst[v * width + static_cast<size_t>(c.index)] = src[v * stride];
  }
  return out;
}

inline void save_ply(const SceneSoA& s, const std::string& path) {
  std::ofstream os(path, std::ios::binary);
  if (!os) throw std::runtime_error("save_ply: cannot open " + path + " for writing");
  const std::vector<PlyColumn> schema = ply_schema(true);
  const size_t n = static_cast<size_t>(s.size()), stride = schema.size();
  std::string header = "ply\nformat binary_little_endian 1.0\nelement vertex " + std::to_string(n) + "\n";
  for (const auto& c : schema) header += "property float " + c.name + "\n";
  header += "end_header\n";
  os.write(header.data(), static_cast<std::streamsize>(header.size()));
  // gather column by column into the interleaved payload (normals written as zero)
  std::vector<float> block(n * stride, 0.f);
  for (size_t col = 0; col < stride; ++col) {
    const PlyColumn& c = schema[col];
    const float* src = nullptr;
    size_t width = 0;
    switch (c.field) {
      case PlyField::Mean: src = s.means.data(); width = 3; break;
      case PlyField::Sh: src = s.sh.data(); width = 48; break;
      case PlyField::Opacity: src = s.opacity_logits.data(); width = 1; break;
      case PlyField::LogScale: src = s.log_scales.data(); width = 3; break;
      case PlyField::Rotation: src = s.rotations.data(); width = 4; break;
      case PlyField::Normal: continue;
    }
    for (size_t v = 0; v < n; ++v) block[v * stride + col] = src[v * width + static_cast<size_t>(c.index)];
  }
  os.write(reinterpret_cast<const char*>(block.data()), static_cast<std::streamsize>(block.size() * sizeof(float)));
  if (!os) throw std::runtime_error("save_ply: write failed for " + path);
}

// ---------------------------------------------------------------------------------------
// Minimal JSON (objects, arrays, numbers, strings, booleans, null)

struct Json {
  enum Kind { Null, Bool, Number, String, Array, Object } kind = Null;
  bool b = false;
  double num = 0.0;
  std::string str;
  std::vector<Json> arr;
  std::vector<std::pair<std::string, Json>> obj;

  bool contains(const std::string& k) const {
    if (kind != Object) return false;
    for (const auto& kv : obj)
      if (kv.first == k) return true;
    return false;
  }
  const Json& at(const std::string& k) const {
    if (kind != Object) throw std::runtime_error("[json.exception.type_error.304] cannot use at() with non-object");
    for (const auto& kv : obj)
      if (kv.first == k) return kv.second;
    throw std::runtime_error("[json.exception.out_of_range.403] key '" + k + "' not found");
  }
  double number() const {
    if (kind != Number) throw std::runtime_error("[json.exception.type_error.302] type must be number");
    return num;
  }
  const std::string& string() const {
    if (kind != String) throw std::runtime_error("[json.exception.type_error.302] type must be string");
    return str;
  }
  std::vector<double> numbers() const {
    if (kind != Array) throw std::runtime_error("[json.exception.type_error.302] type must be array");
    std::vector<double> v;
    for (const auto& e : arr) v.push_back(e.number());
    return v;
  }
};

class JsonParser {
 public:
  explicit JsonParser(const std::string& s) : s_(s) {}
  Json parse() {
    Json v = value();
    ws();
    if (p_ != s_.size()) fail("unexpected trailing characters");
    return v;
  }

 private:
  const std::string& s_;
  size_t p_ = 0;
  [[noreturn]] void fail(const std::string& what) {
    throw std::runtime_error("[json.exception.parse_error.101] parse error at byte " + std::to_string(p_ + 1) + ": " +
                             what);
  }
  void ws() {
    while (p_ < s_.size() && std::isspace(static_cast<unsigned char>(s_[p_]))) ++p_;
  }
  bool lit(const char* w) {
    const size_t n = std::strlen(w);
    if (s_.compare(p_, n, w) == 0) {
      p_ += n;
      return true;
    }
    return false;
  }
  std::string string_lit() {
    if (s_[p_] != '"') fail("expected string");
    ++p_;
    std::string out;
    while (p_ < s_.size() && s_[p_] != '"') {
      char c = s_[p_++];
      if (c == '\\') {
        if (p_ >= s_.size()) fail("bad escape");
        const char e = s_[p_++];
        switch (e) {
          case 'n': c = '\n'; break;
          case 't': c = '\t'; break;
          case 'r': c = '\r'; break;
          case 'b': c = '\b'; break;
          case 'f': c = '\f'; break;
          case 'u': {
            if (p_ + 4 > s_.size()) fail("bad unicode escape");
            const unsigned cp = static_cast<unsigned>(std::stoul(s_.substr(p_, 4), nullptr, 16));
            p_ += 4;
            c = cp < 128 ? static_cast<char>(cp) : '?';
            break;
          }
          default: c = e;
        }
      }
      out.push_back(c);
    }
    if (p_ >= s_.size()) fail("unterminated string");
    ++p_;
    return out;
  }
  Json value() {
    ws();
    if (p_ >= s_.size()) fail("unexpected end of input");
    Json v;
    const char c = s_[p_];
    if (c == '{') {
      v.kind = Json::Object;
      ++p_;
      ws();
      if (p_ < s_.size() && s_[p_] == '}') {
        ++p_;
        return v;
      }
      while (true) {
        ws();
        std::string k = string_lit();
        ws();
        if (p_ >= s_.size() || s_[p_] != ':') fail("expected ':'");
        ++p_;
        v.obj.emplace_back(std::move(k), value());
        ws();
        if (p_ < s_.size() && s_[p_] == ',') {
          ++p_;
          continue;
        }
        if (p_ < s_.size() && s_[p_] == '}') {
          ++p_;
          return v;
        }
        fail("expected ',' or '}'");
      }
    }
    if (c == '[') {
      v.kind = Json::Array;
      ++p_;
      ws();
      if (p_ < s_.size() && s_[p_] == ']') {
        ++p_;
        return v;
      }
      while (true) {
        v.arr.push_back(value());
        ws();
        if (p_ < s_.size() && s_[p_] == ',') {
          ++p_;
          continue;
        }
        if (p_ < s_.size() && s_[p_] == ']') {
          ++p_;
          return v;
        }
        fail("expected ',' or ']'");
      }
    }
    if (c == '"') {
      v.kind = Json::String;
      v.str = string_lit();
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
    const char* b = s_.c_str() + p_;
    char* e = nullptr;
    v.num = std::strtod(b, &e);
    if (e == b) fail("syntax error");
    v.kind = Json::Number;
    p_ += static_cast<size_t>(e - b);
    return v;
  }
};

inline std::string json_number(double v) {
  char buf[40];
  std::snprintf(buf, sizeof(buf), "%.17g", v);
  return buf;
}

// ---------------------------------------------------------------------------------------
// Cameras (src/camera_io.cpp). Camera<double> in the reference; cast to float for rendering.

struct CameraD {
  int model = FGS_CAMERA_PINHOLE;
  int width = 0, height = 0;
  double fx = 0, fy = 0, cx = 0, cy = 0;
  std::array<double, 9> rotation_wc{1, 0, 0, 0, 1, 0, 0, 0, 1};
  std::array<double, 3> translation_wc{0, 0, 0};
  double fov_max = 1.5707963267948966;

  fgs_camera to_float() const {
    fgs_camera c{};
    c.model = model;
    c.width = width;
    c.height = height;
    c.fx = static_cast<float>(fx);
    c.fy = static_cast<float>(fy);
    c.cx = static_cast<float>(cx);
    c.cy = static_cast<float>(cy);
    for (int i = 0; i < 9; ++i) c.rotation_wc[i] = static_cast<float>(rotation_wc[i]);
    for (int i = 0; i < 3; ++i) c.translation_wc[i] = static_cast<float>(translation_wc[i]);
    c.fov_max = static_cast<float>(fov_max);
    return c;
  }
};

inline const char* camera_model_name(int m) {
  switch (m) {
    case FGS_CAMERA_PINHOLE: return "pinhole";
    case FGS_CAMERA_FISHEYE: return "fisheye_equidistant";
    case FGS_CAMERA_PANORAMA: return "panorama";
  }
  return "unknown";
}

inline int camera_model_from(const std::string& s, const char* who = "load_cameras") {
  if (s == "pinhole") return FGS_CAMERA_PINHOLE;
  if (s == "fisheye_equidistant") return FGS_CAMERA_FISHEYE;
  if (s == "panorama") return FGS_CAMERA_PANORAMA;
  throw std::runtime_error(std::string(who) + ": unknown camera model '" + s + "'");
}

using Mat3d = std::array<double, 9>;

inline Mat3d mat_mul(const Mat3d& a, const Mat3d& b) {
  Mat3d c{};
  for (int i = 0; i < 3; ++i)
    for (int j = 0; j < 3; ++j) c[i * 3 + j] = a[i * 3] * b[j] + a[i * 3 + 1] * b[3 + j] + a[i * 3 + 2] * b[6 + j];
  return c;
}
inline Mat3d transpose(const Mat3d& a) {
  return {a[0], a[3], a[6], a[1], a[4], a[7], a[2], a[5], a[8]};
}
inline double det3(const Mat3d& a) {
  return a[0] * (a[4] * a[8] - a[5] * a[7]) - a[1] * (a[3] * a[8] - a[5] * a[6]) + a[2] * (a[3] * a[7] - a[4] * a[6]);
}
// Orthogonal polar factor of a non-singular 3x3 (= U V^T of its SVD): Newton iteration
// X <- (X + X^-T) / 2.
inline Mat3d polar_orthogonal(Mat3d x) {
  for (int it = 0; it < 100; ++it) {
    const double d = det3(x);
    if (d == 0.0) break;
    // inverse transpose = cofactor matrix / det
    const Mat3d cof{x[4] * x[8] - x[5] * x[7], x[5] * x[6] - x[3] * x[8], x[3] * x[7] - x[4] * x[6],
                    x[2] * x[7] - x[1] * x[8], x[0] * x[8] - x[2] * x[6], x[1] * x[6] - x[0] * x[7],
                    x[1] * x[5] - x[2] * x[4], x[2] * x[3] - x[0] * x[5], x[0] * x[4] - x[1] * x[3]};
    Mat3d nx;
    double delta = 0.0;
    for (int i = 0; i < 9; ++i) {
      nx[i] = 0.5 * (x[i] + cof[i] / d);
      delta = std::max(delta, std::fabs(nx[i] - x[i]));
    }
    x = nx;
    if (delta < 1e-15) break;
  }
  return x;
}

inline CameraD camera_from_json(const Json& j, size_t index, std::vector<std::string>* warnings) {
  const std::string idx = std::to_string(index);
  CameraD cam;
  cam.model = camera_model_from(j.at("model").string());
  cam.width = static_cast<int>(j.at("width").number());
  cam.height = static_cast<int>(j.at("height").number());
  if (cam.width < 16 || cam.height < 16)
    throw std::runtime_error("load_cameras: camera " + idx + ": width and height must be >= 16");
  if (cam.model != FGS_CAMERA_PANORAMA) {
    cam.fx = j.at("fx").number();
    cam.fy = j.at("fy").number();
    cam.cx = j.at("cx").number();
    cam.cy = j.at("cy").number();
    if (!(cam.fx > 0) || !(cam.fy > 0))
      throw std::runtime_error("load_cameras: camera " + idx + ": focal lengths must be positive");
  }
  const double fov_deg = j.contains("fov_max_deg") ? j.at("fov_max_deg").number() : 90.0;
  cam.fov_max = fov_deg * 3.141592653589793238462643383279502884 / 180.0;
  const auto rot = j.at("rotation").numbers();
  const auto tr = j.at("translation").numbers();
  if (rot.size() != 9 || tr.size() != 3)
    throw std::runtime_error("load_cameras: camera " + idx +
                             ": rotation needs 9 numbers (row-major) and translation 3");
  Mat3d r;
  for (int i = 0; i < 9; ++i) r[i] = rot[i];
  for (int i = 0; i < 3; ++i) cam.translation_wc[i] = tr[i];
  const Mat3d rtr = mat_mul(transpose(r), r);
  double dev = 0.0;
  for (int i = 0; i < 9; ++i) dev = std::max(dev, std::fabs(rtr[i] - ((i % 4 == 0) ? 1.0 : 0.0)));
  if (dev > 1e-2)
    throw std::runtime_error("load_cameras: camera " + idx + ": rotation is not orthonormal (deviation " +
                             std::to_string(dev) + ")");
  if (dev > 1e-6 || det3(r) < 0) {
    const Mat3d fixed = polar_orthogonal(r);
    if (det3(fixed) < 0) throw std::runtime_error("load_cameras: camera " + idx + ": rotation has negative determinant");
    r = fixed;
    if (warnings)
      warnings->push_back("load_cameras: camera " + idx + ": rotation re-orthonormalized (deviation " +
                          std::to_string(dev) + ")");
  }
  cam.rotation_wc = r;
  return cam;
}

struct CamerasRead {
  std::vector<CameraD> cameras;
  std::vector<std::string> warnings;
};

inline CamerasRead load_cameras(const std::string& path) {
  std::ifstream in(path);
  if (!in) throw std::runtime_error("load_cameras: cannot open " + path);
  std::stringstream ss;
  ss << in.rdbuf();
  const std::string text = ss.str();
  Json doc;
  try {
    doc = JsonParser(text).parse();
  } catch (const std::exception& e) {
    throw std::runtime_error("load_cameras: " + path + ": " + e.what());
  }
  std::vector<Json> cams;
  if (doc.kind == Json::Array) cams = doc.arr;
  else if (doc.kind == Json::Object && doc.contains("cameras")) cams = doc.at("cameras").arr;
  else cams = {doc};
  CamerasRead out;
  try {
    for (size_t i = 0; i < cams.size(); ++i) out.cameras.push_back(camera_from_json(cams[i], i, &out.warnings));
  } catch (const std::exception& e) {
    const std::string m = e.what();
    if (m.rfind("load_cameras:", 0) == 0) throw;
    throw std::runtime_error("load_cameras: " + path + ": " + m);
  }
  if (out.cameras.empty()) throw std::runtime_error("load_cameras: " + path + " contains no cameras");
  return out;
}

inline void save_cameras(const std::vector<CameraD>& cams, const std::string& path) {
  std::ofstream os(path);
  if (!os) throw std::runtime_error("save_cameras: cannot open " + path + " for writing");
  os << "[\n";
  for (size_t i = 0; i < cams.size(); ++i) {
    const CameraD& c = cams[i];
    os << "  {\n    \"model\": \"" << camera_model_name(c.model) << "\",\n    \"width\": " << c.width
       << ",\n    \"height\": " << c.height << ",\n";
    if (c.model != FGS_CAMERA_PANORAMA)
      os << "    \"fx\": " << json_number(c.fx) << ",\n    \"fy\": " << json_number(c.fy) << ",\n    \"cx\": "
         << json_number(c.cx) << ",\n    \"cy\": " << json_number(c.cy) << ",\n";
    if (c.model == FGS_CAMERA_FISHEYE)
      os << "    \"fov_max_deg\": " << json_number(c.fov_max * 180.0 / 3.141592653589793238462643383279502884) << ",\n";
    os << "    \"rotation\": [";
    for (int k = 0; k < 9; ++k) os << (k ? ", " : "") << json_number(c.rotation_wc[k]);
    os << "],\n    \"translation\": [";
    for (int k = 0; k < 3; ++k) os << (k ? ", " : "") << json_number(c.translation_wc[k]);
    os << "]\n  }" << (i + 1 < cams.size() ? "," : "") << "\n";
  }
  os << "]\n";
}

// ---------------------------------------------------------------------------------------
// Images (src/image_io.cpp's formats): 8-bit RGB, each value clamped to [0, 1] and scaled by 255
// with round-half-to-even; binary PPM (P6) or PNG. The PNG is written without compression (zlib
// stored blocks), as the reference's writer does, so any decoder reads it.

inline uint8_t to_u8(double v) {
  const double c = v < 0.0 ? 0.0 : (v > 1.0 ? 1.0 : v);
  return static_cast<uint8_t>(std::lrint((c == c ? c : 0.0) * 255.0));  // NaN -> 0; lrint rounds half to even
}
inline uint8_t quantize(double v) { return to_u8(v); }

// Append-only big-endian byte buffer with the two checksums PNG / zlib need.
class ByteSink {
 public:
  std::vector<uint8_t> bytes;
  void u8(uint8_t v) { bytes.push_back(v); }
  void be32(uint32_t v) {
    for (int k = 3; k >= 0; --k) bytes.push_back(static_cast<uint8_t>((v >> (8 * k)) & 0xFFu));
  }
  void raw(const uint8_t* p, size_t n) { bytes.insert(bytes.end(), p, p + n); }
  void str(const char* s) { raw(reinterpret_cast<const uint8_t*>(s), std::strlen(s)); }

  // CRC-32 (IEEE 802.3, reflected polynomial 0xEDB88320) of bytes[from, end), bitwise.
  uint32_t crc32(size_t from) const {
    uint32_t c = 0xFFFFFFFFu;
    for (size_t i = from; i < bytes.size(); ++i) {
      c ^= bytes[i];
      for (int b = 0; b < 8; ++b) c = (c >> 1) ^ (0xEDB88320u & (0u - (c & 1u)));
    }
    return c ^ 0xFFFFFFFFu;
  }
};

// Adler-32 with the modulo deferred over runs of 5552 bytes (the longest run whose sums cannot
// overflow 32 bits).
inline uint32_t adler32(const uint8_t* p, size_t n) {
  uint32_t lo = 1, hi = 0;
  while (n) {
    const size_t run = n < 5552 ? n : 5552;
    for (size_t i = 0; i < run; ++i) {
      lo += p[i];
      hi += lo;
    }
    lo %= 65521u;
    hi %= 65521u;
    p += run;
    n -= run;
  }
  return (hi << 16) | lo;
}

// zlib stream of stored (BTYPE 00) deflate blocks of at most 65535 bytes.
inline std::vector<uint8_t> zlib_stored(const std::vector<uint8_t>& data) {
  ByteSink z;
  z.u8(0x78);
  z.u8(0x01);
  const size_t nblocks = data.empty() ? 1 : (data.size() + 65534) / 65535;
  for (size_t b = 0; b < nblocks; ++b) {
    const size_t off = b * 65535, len = std::min<size_t>(65535, data.size() - off);
    z.u8(b + 1 == nblocks ? 1 : 0);  // BFINAL on the last block
    const uint16_t l16 = static_cast<uint16_t>(len), nl16 = static_cast<uint16_t>(~l16);
    z.u8(static_cast<uint8_t>(l16 & 0xFF));
    z.u8(static_cast<uint8_t>(l16 >> 8));
    z.u8(static_cast<uint8_t>(nl16 & 0xFF));
    z.u8(static_cast<uint8_t>(nl16 >> 8));
    z.raw(data.data() + off, len);
  }
  z.be32(adler32(data.data(), data.size()));
  return z.bytes;
}

inline void png_append_chunk(ByteSink& out, const char* type, const std::vector<uint8_t>& body) {
  out.be32(static_cast<uint32_t>(body.size()));
  const size_t crc_from = out.bytes.size();
  out.str(type);
  out.raw(body.data(), body.size());
  out.be32(out.crc32(crc_from));
}

inline std::vector<uint8_t> encode_png(const std::vector<uint8_t>& rgb, int w, int h) {
  ByteSink ihdr;
  ihdr.be32(static_cast<uint32_t>(w));
  ihdr.be32(static_cast<uint32_t>(h));
  for (uint8_t v : {8, 2, 0, 0, 0}) ihdr.u8(v);  // 8-bit depth, truecolour, deflate, no filter, no interlace
  // scanlines, each led by filter type 0
  const size_t row = 3 * static_cast<size_t>(w);
  std::vector<uint8_t> scan(static_cast<size_t>(h) * (row + 1), 0);
  for (int y = 0; y < h; ++y) std::memcpy(scan.data() + static_cast<size_t>(y) * (row + 1) + 1, rgb.data() + y * row, row);
  ByteSink png;
  for (uint8_t v : {0x89, 0x50, 0x4E, 0x47, 0x0D, 0x0A, 0x1A, 0x0A}) png.u8(v);
  png_append_chunk(png, "IHDR", ihdr.bytes);
  png_append_chunk(png, "IDAT", zlib_stored(scan));
  png_append_chunk(png, "IEND", {});
  return png.bytes;
}

inline void write_image(const Image& img, const std::string& path) {
  const size_t dot = path.find_last_of('.');
  std::string ext = dot == std::string::npos ? std::string() : path.substr(dot + 1);
  std::transform(ext.begin(), ext.end(), ext.begin(), [](unsigned char ch) { return static_cast<char>(std::tolower(ch)); });
  if (ext != "png" && ext != "ppm") throw std::runtime_error("write_image: unknown extension '" + ext + "' (use .png or .ppm)");
  std::vector<uint8_t> rgb(img.pixels.size());
  std::transform(img.pixels.begin(), img.pixels.end(), rgb.begin(), [](float v) { return to_u8(v); });
  std::vector<uint8_t> file;
  if (ext == "png") {
    file = encode_png(rgb, img.width, img.height);
  } else {
    const std::string head = "P6\n" + std::to_string(img.width) + " " + std::to_string(img.height) + "\n255\n";
    file.assign(head.begin(), head.end());
    file.insert(file.end(), rgb.begin(), rgb.end());
  }
  std::ofstream os(path, std::ios::binary);
  if (!os) throw std::runtime_error("write_image: cannot open " + path + " for writing");
  os.write(reinterpret_cast<const char*>(file.data()), static_cast<std::streamsize>(file.size()));
}

}  // namespace io
}  // namespace fgs

#endif  // FGS_IO_HPP_
