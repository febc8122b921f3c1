// Ingest path: PLY (ascii / binary_little_endian) and XYZ
// text readers with the reference's acceptance rules (cloud_io.cpp:61-427:
// vertex element with float/double x, y, z; other elements and properties,
// including lists, are skipped; non-finite coordinates, truncation and
// malformed headers are errors), and the reference's selection-sampling
// subsample (cloud_io.cpp:477-498; std::mt19937_64 + the same libstdc++
// distribution, so the kept indices are identical).  Host code: the points
// land in a caller-owned buffer that the caller can pin and ship with the
// C-ABI's device entry points.
#include <cmath>
#include <cstdint>
#include <cstdlib>
#include <cstring>
#include <fstream>
#include <random>
#include <sstream>
#include <string>
#include <vector>

#include "../../include/treereg_b200.h"  // status codes
#include "../../include/treereg_b200_host.h"

namespace trg {
// the host library's own last-error message (trg_host_last_error)
thread_local std::string g_host_error;
static void set_error(const std::string& msg) { g_host_error = msg; }
}  // namespace trg

extern "C" const char* trg_host_last_error(void) { return trg::g_host_error.c_str(); }

namespace {

struct Fail {
  std::string what;
  size_t offset;
};

[[noreturn]] void fail(const std::string& w, size_t off) { throw Fail{w, off}; }

enum Kind { kF32, kF64, kI8, kU8, kI16, kU16, kI32, kU32 };

int kind_bytes(Kind k) {
  static const int b[] = {4, 8, 1, 1, 2, 2, 4, 4};
  return b[k];
}

bool kind_of(const std::string& t, Kind& k) {
  static const struct {
    const char* a;
    const char* b;
    Kind k;
  } tab[] = {{"float", "float32", kF32}, {"double", "float64", kF64}, {"char", "int8", kI8},
             {"uchar", "uint8", kU8},    {"short", "int16", kI16},    {"ushort", "uint16", kU16},
             {"int", "int32", kI32},     {"uint", "uint32", kU32}};
  for (const auto& e : tab)
    if (t == e.a || t == e.b) {
      k = e.k;
      return true;
    }
  return false;
}

struct Prop {
  std::string name;
  Kind kind = kF32, count_kind = kU8;
  bool list = false;
};
struct Elem {
  std::string name;
  size_t count = 0;
  std::vector<Prop> props;
};

std::vector<std::string> tokens(const std::string& s) {
  std::vector<std::string> out;
  std::istringstream in(s);
  for (std::string t; in >> t;) out.push_back(t);
  return out;
}

// header line: up to '\n', '\r' stripped
std::string header_line(const std::string& buf, size_t& pos) {
  const size_t e = buf.find('\n', pos);
  if (e == std::string::npos) fail("unterminated header line", pos);
  std::string l = buf.substr(pos, e - pos);
  if (!l.empty() && l.back() == '\r') l.pop_back();
  pos = e + 1;
  return l;
}

double bin_value(const std::string& buf, size_t& pos, Kind k) {
  const int nb = kind_bytes(k);
  if (pos + nb > buf.size()) fail("truncated binary payload", pos);
  const char* s = buf.data() + pos;
  pos += nb;
  switch (k) {
    case kF32: { float v; std::memcpy(&v, s, 4); return v; }
    case kF64: { double v; std::memcpy(&v, s, 8); return v; }
    case kI8: return (double)(int8_t)s[0];
    case kU8: return (double)(uint8_t)s[0];
    case kI16: { int16_t v; std::memcpy(&v, s, 2); return v; }
    case kU16: { uint16_t v; std::memcpy(&v, s, 2); return v; }
    case kI32: { int32_t v; std::memcpy(&v, s, 4); return v; }
    case kU32: { uint32_t v; std::memcpy(&v, s, 4); return v; }
  }
  return 0.0;
}

double text_value(const std::string& buf, size_t& pos) {
  while (pos < buf.size() && std::isspace((unsigned char)buf[pos])) ++pos;
  if (pos >= buf.size()) fail("truncated ascii payload", pos);
  const size_t b = pos;
  while (pos < buf.size() && !std::isspace((unsigned char)buf[pos])) ++pos;
  const std::string tok = buf.substr(b, pos - b);
  try {
    size_t used = 0;
    const double v = std::stod(tok, &used);
    if (used == tok.size()) return v;
  } catch (const std::exception&) {
  }
  fail("bad numeric token '" + tok + "'", b);
}

void read_ply(const std::string& buf, int want, std::vector<double>& out) {
  size_t pos = 0;
  if (buf.size() < 4 || header_line(buf, pos) != "ply") fail("missing 'ply' magic", 0);
  bool binary = false, have_format = false;
  std::vector<Elem> elems;
  for (;;) {
    const size_t at = pos;
    const auto t = tokens(header_line(buf, pos));
    if (t.empty() || t[0] == "comment" || t[0] == "obj_info") continue;
    if (t[0] == "end_header") break;
    if (t[0] == "format") {
      if (t.size() != 3 || t[2] != "1.0") fail("malformed format line", at);
      if (t[1] == "ascii") binary = false;
      else if (t[1] == "binary_little_endian") binary = true;
      else if (t[1] == "binary_big_endian") fail("binary_big_endian PLY is not supported", at);
      else fail("unknown PLY format '" + t[1] + "'", at);
      have_format = true;
    } else if (t[0] == "element") {
      if (t.size() != 3) fail("malformed element line", at);
      Elem e;
      e.name = t[1];
      try {
        e.count = std::stoull(t[2]);
      } catch (const std::exception&) {
        fail("bad element count", at);
      }
      elems.push_back(e);
    } else if (t[0] == "property") {
      if (elems.empty()) fail("property before any element", at);
      Prop p;
      if (t.size() == 3) {
        if (!kind_of(t[1], p.kind)) fail("unknown property type '" + t[1] + "'", at);
        p.name = t[2];
      } else if (t.size() == 5 && t[1] == "list") {
        p.list = true;
        if (!kind_of(t[2], p.count_kind) || !kind_of(t[3], p.kind)) fail("unknown list property type", at);
        p.name = t[4];
      } else {
        fail("malformed property line", at);
      }
      elems.back().props.push_back(p);
    } else {
      fail("unknown header keyword '" + t[0] + "'", at);
    }
  }
  if (!have_format) fail("header has no format line", pos);
  if (want == 1 && binary) fail("expected ascii PLY", 0);
  if (want == 2 && !binary) fail("expected binary_little_endian PLY", 0);
  const Elem* vx = nullptr;
  for (const auto& e : elems)
    if (e.name == "vertex") vx = &e;  // the last one, like the reference
  if (!vx) fail("no vertex element in header", pos);
  int ax[3] = {-1, -1, -1};
  for (size_t i = 0; i < vx->props.size(); ++i) {
    const Prop& p = vx->props[i];
    if (p.list || (p.kind != kF32 && p.kind != kF64)) continue;
    for (int c = 0; c < 3; ++c)
      if (p.name == std::string(1, "xyz"[c])) ax[c] = (int)i;
  }
  if (ax[0] < 0 || ax[1] < 0 || ax[2] < 0) fail("vertex element lacks float x/y/z properties", pos);
  for (const auto& e : elems) {
    const bool is_vx = &e == vx;
    // a hostile header may claim any count: reserve no more than the rest of
    // the buffer could possibly hold (>= 1 byte per value)
    if (is_vx) out.reserve(3 * std::min<size_t>(e.count, buf.size() - std::min(buf.size(), pos)));
    for (size_t r = 0; r < e.count; ++r) {
      const size_t row_at = pos;
      double xyz[3] = {0.0, 0.0, 0.0};
      for (size_t i = 0; i < e.props.size(); ++i) {
        const Prop& p = e.props[i];
        if (p.list) {
          const double cv = binary ? bin_value(buf, pos, p.count_kind) : text_value(buf, pos);
          if (cv < 0 || cv > 1e9) fail("implausible list count", pos);
          const size_t cnt = (size_t)cv;
          if (binary) {
            if (pos + cnt * kind_bytes(p.kind) > buf.size()) fail("truncated binary payload", pos);
            pos += cnt * kind_bytes(p.kind);
          } else {
            for (size_t q = 0; q < cnt; ++q) text_value(buf, pos);
          }
          continue;
        }
        const double v = binary ? bin_value(buf, pos, p.kind) : text_value(buf, pos);
        if (is_vx)
          for (int c = 0; c < 3; ++c)
            if ((int)i == ax[c]) xyz[c] = v;
      }
      if (is_vx) {
        if (!std::isfinite(xyz[0]) || !std::isfinite(xyz[1]) || !std::isfinite(xyz[2]))
          fail("non-finite vertex coordinate", row_at);
        out.insert(out.end(), xyz, xyz + 3);
      }
    }
  }
}

void read_xyz(const std::string& buf, std::vector<double>& out) {
  size_t pos = 0, line_no = 0;
  while (pos < buf.size()) {
    const size_t at = pos;
    size_t e = buf.find('\n', pos);
    if (e == std::string::npos) e = buf.size();
    std::string l = buf.substr(pos, e - pos);
    pos = e + 1;
    ++line_no;
    if (!l.empty() && l.back() == '\r') l.pop_back();
    const size_t f = l.find_first_not_of(" \t");
    if (f == std::string::npos || l[f] == '#') continue;
    std::istringstream in(l);
    double v[3];
    if (!(in >> v[0] >> v[1] >> v[2])) fail("malformed xyz line " + std::to_string(line_no), at);
    std::string extra;
    if (in >> extra) fail("trailing tokens on xyz line " + std::to_string(line_no), at);
    if (!std::isfinite(v[0]) || !std::isfinite(v[1]) || !std::isfinite(v[2]))
      fail("non-finite coordinate on xyz line " + std::to_string(line_no), at);
    out.insert(out.end(), v, v + 3);
  }
}

}  // namespace

extern "C" {

int trg_read_cloud(const char* path, int format, double** xyz, size_t* n) {
  if (!path || !xyz || !n || format < 0 || format > 3) {
    trg::set_error("read_cloud: bad argument");
    return TRG_EINVAL;
  }
  std::ifstream in(path, std::ios::binary);
  if (!in) {
    trg::set_error(std::string("cannot open file: ") + path);
    return TRG_ERUNTIME;
  }
  std::ostringstream ss;
  ss << in.rdbuf();
  const std::string buf = ss.str();
  std::vector<double> pts;
  try {
    const bool ply = format == 1 || format == 2 || (format == 0 && buf.rfind("ply", 0) == 0);
    if (ply) read_ply(buf, format, pts);
    else read_xyz(buf, pts);
  } catch (const Fail& f) {
    trg::set_error(std::string(path) + ": " + f.what + " (byte " + std::to_string(f.offset) + ")");
    return TRG_ERUNTIME;  // ParseError is a std::runtime_error (cloud_io.hpp:18)
  } catch (const std::exception& e) {  // e.g. bad_alloc / length_error: never escape the C-ABI
    trg::set_error(std::string(path) + ": " + e.what());
    return TRG_ERUNTIME;
  }
  *n = pts.size() / 3;
  *xyz = static_cast<double*>(std::malloc(sizeof(double) * std::max<size_t>(pts.size(), 1)));
  if (!*xyz) {
    trg::set_error("read_cloud: out of memory");
    return TRG_ERUNTIME;
  }
  std::memcpy(*xyz, pts.data(), sizeof(double) * pts.size());
  return TRG_OK;
}

void trg_free_cloud(double* xyz) { std::free(xyz); }

int trg_subsample(const double* xyz, size_t n, size_t m, uint64_t seed, double* out) {
  if (m < 1 || m > n || !xyz || !out) {
    trg::set_error("subsample: n out of range");
    return TRG_EINVAL;
  }
  std::mt19937_64 rng(seed);
  size_t need = m, remaining = n, k = 0;
  for (size_t i = 0; i < n && need > 0; ++i, --remaining) {
    std::uniform_int_distribution<size_t> pick(0, remaining - 1);
    if (pick(rng) < need) {
      std::memcpy(out + 3 * k, xyz + 3 * i, 3 * sizeof(double));
      ++k;
      --need;
    }
  }
  return TRG_OK;
}

}  // extern "C"
