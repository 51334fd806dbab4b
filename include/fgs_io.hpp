// fgs_io.hpp — header-only host I/O around the rasterizer: the reference's scene / camera /
// image file formats, so its `render` / `bench` callers can drive the B200
// path unchanged.
//
//   load_ply / save_ply        src/ply_io.cpp:40-145   (3DGS binary_little_endian layout)
//   load_cameras / save_cameras src/camera_io.cpp:25-127 (camera JSON)
//   write_image (PPM / PNG)    src/image_io.cpp:19-160 (8-bit, round half to even)
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
// PLY (src/ply_io.cpp)

inline std::vector<std::string> ply_full_properties() {
  std::vector<std::string> p = {"x", "y", "z", "nx", "ny", "nz", "f_dc_0", "f_dc_1", "f_dc_2"};
  for (int i = 0; i < 45; ++i) p.push_back("f_rest_" + std::to_string(i));
  for (const char* s : {"opacity", "scale_0", "scale_1", "scale_2", "rot_0", "rot_1", "rot_2", "rot_3"}) p.push_back(s);
  return p;
}

inline std::vector<std::string> ply_dc_properties() {
  return {"x", "y", "z", "nx", "ny", "nz", "f_dc_0", "f_dc_1", "f_dc_2", "opacity",
          "scale_0", "scale_1", "scale_2", "rot_0", "rot_1", "rot_2", "rot_3"};
}

inline std::string join(const std::vector<std::string>& v) {
  std::string s;
  for (size_t i = 0; i < v.size(); ++i) s += (i ? "," : "") + v[i];
  return s;
}

struct PlyRead {
  SceneSoA scene;
  std::vector<std::string> warnings;
};

// SH storage: per Gaussian [channel * 16 + basis]; PLY f_dc_c = basis 0 of channel c,
// f_rest_{c*15 + j-1} = basis j of channel c (src/ply_io.cpp:109-117).
inline PlyRead load_ply(const std::string& path) {
  std::ifstream in(path, std::ios::binary);
  if (!in) throw std::runtime_error("load_ply: cannot open " + path);
  std::string line;
  if (!std::getline(in, line) || (line != "ply" && line != "ply\r"))
    throw std::runtime_error("load_ply: " + path + " is not a PLY file");
  size_t count = 0;
  bool format_seen = false;
  std::vector<std::string> props;
  while (std::getline(in, line)) {
    if (!line.empty() && line.back() == '\r') line.pop_back();
    if (line == "end_header") break;
    std::istringstream ls(line);
    std::string word;
    ls >> word;
    if (word == "format") {
      std::string fmt;
      ls >> fmt;
      if (fmt != "binary_little_endian")
        throw std::runtime_error("load_ply: binary_little_endian required, got format '" + fmt + "'");
      format_seen = true;
    } else if (word == "element") {
      std::string name;
      ls >> name >> count;
      if (name != "vertex") throw std::runtime_error("load_ply: unsupported element '" + name + "'");
    } else if (word == "property") {
      std::string type, name;
      ls >> type >> name;
      if (type != "float")
        throw std::runtime_error("load_ply: property '" + name + "' has type '" + type + "', expected float");
      props.push_back(name);
    } else if (word == "comment" || word == "obj_info" || word.empty()) {
      continue;
    } else {
      throw std::runtime_error("load_ply: unexpected header line '" + line + "'");
    }
  }
  if (!format_seen) throw std::runtime_error("load_ply: missing format line (binary_little_endian required)");
  PlyRead out;
  bool has_rest;
  if (props == ply_full_properties()) {
    has_rest = true;
  } else if (props == ply_dc_properties()) {
    has_rest = false;
    out.warnings.push_back("load_ply: f_rest_* properties missing; higher-order SH set to zero");
  } else {
    throw std::runtime_error("load_ply: unknown property layout; expected [" + join(ply_full_properties()) +
                             "] (or the f_rest-free variant), found [" + join(props) + "]");
  }
  const size_t stride = props.size();
  const std::streampos start = in.tellg();
  SceneSoA& s = out.scene;
  s.means.resize(count * 3);
  s.rotations.resize(count * 4);
  s.log_scales.resize(count * 3);
  s.opacity_logits.resize(count);
  s.sh.assign(count * 48, 0.f);
  std::vector<float> row(stride);
  for (size_t i = 0; i < count; ++i) {
    in.read(reinterpret_cast<char*>(row.data()), static_cast<std::streamsize>(stride * 4));
    if (static_cast<size_t>(in.gcount()) != stride * 4) {
      const long long off = static_cast<long long>(start) + static_cast<long long>(i * stride * 4) + in.gcount();
      throw std::runtime_error("load_ply: truncated payload at byte offset " + std::to_string(off));
    }
    size_t k = 0;
    for (int c = 0; c < 3; ++c) s.means[i * 3 + c] = row[k++];
    k += 3;  // normals ignored
    for (int c = 0; c < 3; ++c) s.sh[i * 48 + c * 16] = row[k++];
    if (has_rest)
      for (int c = 0; c < 3; ++c)
        for (int j = 0; j < 15; ++j) s.sh[i * 48 + c * 16 + j + 1] = row[k++];
    s.opacity_logits[i] = row[k++];
    for (int c = 0; c < 3; ++c) s.log_scales[i * 3 + c] = row[k++];
    for (int c = 0; c < 4; ++c) s.rotations[i * 4 + c] = row[k++];
  }
  return out;
}

inline void save_ply(const SceneSoA& s, const std::string& path) {
  std::ofstream os(path, std::ios::binary);
  if (!os) throw std::runtime_error("save_ply: cannot open " + path + " for writing");
  const size_t n = static_cast<size_t>(s.size());
  os << "ply\nformat binary_little_endian 1.0\nelement vertex " << n << "\n";
  for (const auto& p : ply_full_properties()) os << "property float " << p << "\n";
  os << "end_header\n";
  std::vector<float> row(62);
  for (size_t i = 0; i < n; ++i) {
    size_t k = 0;
    for (int c = 0; c < 3; ++c) row[k++] = s.means[i * 3 + c];
    for (int c = 0; c < 3; ++c) row[k++] = 0.f;
    for (int c = 0; c < 3; ++c) row[k++] = s.sh[i * 48 + c * 16];
    for (int c = 0; c < 3; ++c)
      for (int j = 0; j < 15; ++j) row[k++] = s.sh[i * 48 + c * 16 + j + 1];
    row[k++] = s.opacity_logits[i];
    for (int c = 0; c < 3; ++c) row[k++] = s.log_scales[i * 3 + c];
    for (int c = 0; c < 4; ++c) row[k++] = s.rotations[i * 4 + c];
    os.write(reinterpret_cast<const char*>(row.data()), static_cast<std::streamsize>(row.size() * 4));
  }
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
// Images (src/image_io.cpp): 8-bit, values clamped to [0, 1], rounded half to even.

inline uint8_t quantize(double v) {
  v = std::min(1.0, std::max(0.0, v));
  const double r = std::nearbyint(v * 255.0);
  return static_cast<uint8_t>(std::min(255.0, std::max(0.0, r)));
}

inline uint32_t crc32_update(uint32_t crc, const uint8_t* data, size_t len) {
  static const std::array<uint32_t, 256> table = [] {
    std::array<uint32_t, 256> t{};
    for (uint32_t n = 0; n < 256; ++n) {
      uint32_t c = n;
      for (int k = 0; k < 8; ++k) c = (c & 1) ? 0xedb88320u ^ (c >> 1) : c >> 1;
      t[n] = c;
    }
    return t;
  }();
  crc = ~crc;
  for (size_t i = 0; i < len; ++i) crc = table[(crc ^ data[i]) & 0xff] ^ (crc >> 8);
  return ~crc;
}

inline void put_be32(std::vector<uint8_t>& o, uint32_t v) {
  for (int s = 24; s >= 0; s -= 8) o.push_back(static_cast<uint8_t>(v >> s));
}

inline void png_chunk(std::ofstream& os, const char type[4], const std::vector<uint8_t>& payload) {
  std::vector<uint8_t> buf;
  put_be32(buf, static_cast<uint32_t>(payload.size()));
  buf.insert(buf.end(), type, type + 4);
  buf.insert(buf.end(), payload.begin(), payload.end());
  put_be32(buf, crc32_update(0, buf.data() + 4, buf.size() - 4));
  os.write(reinterpret_cast<const char*>(buf.data()), static_cast<std::streamsize>(buf.size()));
}

// PNG with stored (uncompressed) deflate blocks, as the reference writes.
inline void write_png(const std::vector<uint8_t>& rgb, int w, int h, const std::string& path) {
  std::ofstream os(path, std::ios::binary);
  if (!os) throw std::runtime_error("write_image: cannot open " + path + " for writing");
  const uint8_t sig[8] = {0x89, 'P', 'N', 'G', '\r', '\n', 0x1a, '\n'};
  os.write(reinterpret_cast<const char*>(sig), 8);
  std::vector<uint8_t> ihdr;
  put_be32(ihdr, static_cast<uint32_t>(w));
  put_be32(ihdr, static_cast<uint32_t>(h));
  ihdr.insert(ihdr.end(), {8, 2, 0, 0, 0});
  png_chunk(os, "IHDR", ihdr);
  std::vector<uint8_t> raw;
  raw.reserve(static_cast<size_t>(h) * (1 + 3 * static_cast<size_t>(w)));
  for (int y = 0; y < h; ++y) {
    raw.push_back(0);
    raw.insert(raw.end(), rgb.begin() + static_cast<size_t>(y) * w * 3, rgb.begin() + static_cast<size_t>(y + 1) * w * 3);
  }
  std::vector<uint8_t> z = {0x78, 0x01};
  size_t pos = 0;
  do {
    const size_t n = std::min<size_t>(raw.size() - pos, 65535);
    z.push_back(pos + n == raw.size() ? 1 : 0);
    z.push_back(static_cast<uint8_t>(n & 0xff));
    z.push_back(static_cast<uint8_t>(n >> 8));
    z.push_back(static_cast<uint8_t>(~n & 0xff));
    z.push_back(static_cast<uint8_t>((~n >> 8) & 0xff));
    z.insert(z.end(), raw.begin() + pos, raw.begin() + pos + n);
    pos += n;
  } while (pos < raw.size());
  uint32_t a = 1, b = 0;
  for (uint8_t c : raw) {
    a = (a + c) % 65521;
    b = (b + a) % 65521;
  }
  put_be32(z, (b << 16) | a);
  png_chunk(os, "IDAT", z);
  png_chunk(os, "IEND", {});
}

inline void write_image(const Image& img, const std::string& path) {
  std::vector<uint8_t> rgb(img.pixels.size());
  for (size_t i = 0; i < rgb.size(); ++i) rgb[i] = quantize(img.pixels[i]);
  std::string ext = path.substr(path.find_last_of('.') == std::string::npos ? path.size() : path.find_last_of('.') + 1);
  for (auto& c : ext) c = static_cast<char>(std::tolower(c));
  if (ext == "png") return write_png(rgb, img.width, img.height, path);
  if (ext != "ppm") throw std::runtime_error("write_image: unknown extension '" + ext + "' (use .png or .ppm)");
  std::ofstream os(path, std::ios::binary);
  if (!os) throw std::runtime_error("write_image: cannot open " + path + " for writing");
  os << "P6\n" << img.width << " " << img.height << "\n255\n";
  os.write(reinterpret_cast<const char*>(rgb.data()), static_cast<std::streamsize>(rgb.size()));
}

}  // namespace io
}  // namespace fgs

#endif  // FGS_IO_HPP_
