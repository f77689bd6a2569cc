// ROM archive I/O (host C++) and the one-call on-line load.
//
//   mswave::write_rom_archive / read_rom_archive   rom_archive.cpp:65-190
//   mswave::project_io                              romgen.cpp:359-363
//   msw_create_from_archive                         rom_archive.cpp:110-190 +
//                                                   cmd_simulate's load,
//                                                   cli_commands.cpp:111-116
//
// Container bytes are exactly the reference's (64-bit little-endian integers
// and IEEE doubles, column-major matrices with u64 row/col headers).  The
// manifest is JSON; a small reader/writer for the subset it uses lives here
// (the reference uses nlohmann::json, which this image does not have).
#include <algorithm>
#include <cstdint>
#include <cstdio>
#include <cstring>
#include <filesystem>
#include <fstream>
#include <sstream>
#include <string>
#include <utility>
#include <vector>

#include "common.cuh"
#include "mswave/rom_archive.hpp"
#include "mswave_b200.h"

namespace {

// ---------------------------------------------------------------- JSON ------

struct Json {
  enum Kind { Null, Bool, Num, Str, Arr, Obj } kind = Null;
  bool b = false;
  double num = 0.0;
  std::string str;
  std::vector<Json> arr;
  std::vector<std::pair<std::string, Json>> obj;

  const Json* find(const std::string& k) const {
    for (const auto& kv : obj)
      if (kv.first == k) return &kv.second;
    return nullptr;
  }
  const Json& at(const std::string& k) const {
    const Json* v = find(k);
    if (!v) throw mswave::ConfigError("ROM manifest: missing key \"" + k + "\"");
    return *v;
  }
  double number() const {
    if (kind != Num) throw mswave::ConfigError("ROM manifest: expected a number");
    return num;
  }
  long integer() const { return static_cast<long>(number()); }
  const std::string& string() const {
    if (kind != Str) throw mswave::ConfigError("ROM manifest: expected a string");
    return str;
  }
};

class JsonParser {
 public:
  explicit JsonParser(const std::string& s) : s_(s) {}
  Json parse() {
    Json v = value();
    ws();
    if (p_ != s_.size()) fail("trailing characters");
    return v;
  }

 private:
  const std::string& s_;
  size_t p_ = 0;

  [[noreturn]] void fail(const char* what) {
    throw mswave::ConfigError(std::string("ROM manifest: malformed JSON (") + what + ")");
  }
  void ws() {
    while (p_ < s_.size() && (s_[p_] == ' ' || s_[p_] == '\n' || s_[p_] == '\r' || s_[p_] == '\t')) ++p_;
  }
  char peek() {
    ws();
    if (p_ >= s_.size()) fail("unexpected end");
    return s_[p_];
  }
  void expect(char c) {
    if (peek() != c) fail("unexpected character");
    ++p_;
  }
  bool literal(const char* lit) {
    const size_t n = std::strlen(lit);
    if (s_.compare(p_, n, lit) == 0) {
      p_ += n;
      return true;
    }
    return false;
  }
  std::string string_body() {
    expect('"');
    std::string out;
    while (p_ < s_.size() && s_[p_] != '"') {
      char c = s_[p_++];
      if (c == '\\') {
        if (p_ >= s_.size()) fail("bad escape");
        const char e = s_[p_++];
        switch (e) {
          case '"': out += '"'; break;
          case '\\': out += '\\'; break;
          case '/': out += '/'; break;
          case 'b': out += '\b'; break;
          case 'f': out += '\f'; break;
          case 'n': out += '\n'; break;
          case 'r': out += '\r'; break;
          case 't': out += '\t'; break;
          case 'u': {
            if (p_ + 4 > s_.size()) fail("bad \\u escape");
            const unsigned cp = static_cast<unsigned>(std::stoul(s_.substr(p_, 4), nullptr, 16));
            p_ += 4;
            if (cp < 0x80) {
              out += static_cast<char>(cp);
            } else if (cp < 0x800) {
              out += static_cast<char>(0xc0 | (cp >> 6));
              out += static_cast<char>(0x80 | (cp & 0x3f));
            } else {
              out += static_cast<char>(0xe0 | (cp >> 12));
              out += static_cast<char>(0x80 | ((cp >> 6) & 0x3f));
              out += static_cast<char>(0x80 | (cp & 0x3f));
            }
            break;
          }
          default: fail("bad escape");
        }
      } else {
        out += c;
      }
    }
    expect('"');
    return out;
  }
  Json value() {
    Json v;
    const char c = peek();
    if (c == '{') {
      ++p_;
      v.kind = Json::Obj;
      if (peek() == '}') {
        ++p_;
        return v;
      }
      for (;;) {
        std::string k = string_body();
        expect(':');
        v.obj.emplace_back(std::move(k), value());
        if (peek() == ',') {
          ++p_;
          continue;
        }
        expect('}');
        return v;
      }
    }
    if (c == '[') {
      ++p_;
      v.kind = Json::Arr;
      if (peek() == ']') {
        ++p_;
        return v;
      }
      for (;;) {
        v.arr.push_back(value());
        if (peek() == ',') {
          ++p_;
          continue;
        }
        expect(']');
        return v;
      }
    }
    if (c == '"') {
      v.kind = Json::Str;
      v.str = string_body();
      return v;
    }
    if (literal("true")) {
      v.kind = Json::Bool;
      v.b = true;
      return v;
    }
    if (literal("false")) {
      v.kind = Json::Bool;
      return v;
    }
    if (literal("null")) return v;
    const char* start = s_.c_str() + p_;
    char* end = nullptr;
    v.num = std::strtod(start, &end);
    if (end == start) fail("bad value");
    p_ += static_cast<size_t>(end - start);
    v.kind = Json::Num;
    return v;
  }
};

std::string json_double(double v) {
  char buf[40];
  std::snprintf(buf, sizeof(buf), "%.17g", v);
  std::string s(buf);
  if (s.find_first_of(".eEn") == std::string::npos) s += ".0";
  return s;
}

// ------------------------------------------------------------ container ----

constexpr char kMagic[8] = {'M', 'S', 'W', 'R', 'O', 'M', '1', '\0'};

void put_u64(std::FILE* f, std::uint64_t v) {
  unsigned char b[8];
  for (int i = 0; i < 8; ++i) b[i] = static_cast<unsigned char>((v >> (8 * i)) & 0xff);
  std::fwrite(b, 1, 8, f);
}

void put_doubles(std::FILE* f, const double* d, size_t n) {
  for (size_t i = 0; i < n; ++i) {  // little-endian IEEE binary64
    std::uint64_t u;
    std::memcpy(&u, d + i, 8);
    put_u64(f, u);
  }
}

void put_mat(std::FILE* f, const mswave::Mat& m) {
  put_u64(f, static_cast<std::uint64_t>(m.rows()));
  put_u64(f, static_cast<std::uint64_t>(m.cols()));
  put_doubles(f, m.data(), static_cast<size_t>(m.size()));
}

class Container {
 public:
  Container(std::FILE* f, std::string path) : f_(f), path_(std::move(path)) {}
  ~Container() {
    if (f_) std::fclose(f_);
  }
  std::uint64_t u64() {
    unsigned char b[8];
    if (std::fread(b, 1, 8, f_) != 8) throw mswave::ConfigError("truncated ROM container");
    std::uint64_t v = 0;
    for (int i = 7; i >= 0; --i) v = (v << 8) | b[i];
    return v;
  }
  void doubles(double* d, size_t n) {
    for (size_t i = 0; i < n; ++i) {
      unsigned char b[8];
      if (std::fread(b, 1, 8, f_) != 8) throw mswave::ConfigError("truncated ROM container payload");
      std::uint64_t v = 0;
      for (int k = 7; k >= 0; --k) v = (v << 8) | b[k];
      std::memcpy(d + i, &v, 8);
    }
  }
  mswave::Mat mat() {
    const auto rows = static_cast<long>(u64());
    const auto cols = static_cast<long>(u64());
    if (rows < 0 || cols < 0 || rows > (1L << 24) || cols > (1L << 24))
      throw mswave::ConfigError("implausible matrix dimensions in ROM container");
    mswave::Mat m(rows, cols);
    doubles(m.data(), static_cast<size_t>(m.size()));
    return m;
  }
  const std::string& path() const { return path_; }

 private:
  std::FILE* f_;
  std::string path_;
};

std::string cell_filename(int cell) {
  char buf[32];
  std::snprintf(buf, sizeof(buf), "cell_%04d.bin", cell);
  return buf;
}

}  // namespace

namespace mswave {

Vec project_io(const Mat& S_ij, const Vec& values_on_iface) {
  if (S_ij.rows() != values_on_iface.size()) throw ConfigError("project_io: interface size mismatch");
  Vec out(S_ij.cols());
  for (long j = 0; j < S_ij.cols(); ++j) {
    double s = 0.0;
    for (long i = 0; i < S_ij.rows(); ++i) s += S_ij(i, j) * values_on_iface[i];
    out[j] = s;
  }
  return out;
}

void write_rom_archive(const std::string& dir, const std::vector<SubdomainROM>& roms,
                       const BoundaryBasis& basis, const RomOptions& opt) {
  namespace fs = std::filesystem;
  fs::create_directories(dir);
  std::ostringstream cells;
  for (size_t i = 0; i < roms.size(); ++i) {
    const SubdomainROM& rom = roms[i];
    cells << (i ? ",\n" : "\n") << "    {\n      \"file\": \"" << cell_filename(rom.cell)
          << "\",\n      \"ktilde\": " << rom.ktilde << ",\n      \"m\": " << rom.m
          << ",\n      \"interfaces\": [";
    for (size_t l = 0; l < rom.iface_ids.size(); ++l) cells << (l ? ", " : "") << rom.iface_ids[l];
    cells << "]\n    }";

    const fs::path path = fs::path(dir) / cell_filename(rom.cell);
    std::FILE* f = std::fopen(path.c_str(), "wb");
    if (!f) throw ConfigError("cannot write ROM container: " + path.string());
    std::fwrite(kMagic, 1, 8, f);
    put_u64(f, static_cast<std::uint64_t>(rom.cell));
    put_u64(f, static_cast<std::uint64_t>(rom.m));
    put_u64(f, static_cast<std::uint64_t>(rom.ktilde));
    put_u64(f, static_cast<std::uint64_t>(rom.iface_ids.size()));
    put_doubles(f, &rom.shift, 1);
    for (size_t li = 0; li < rom.iface_ids.size(); ++li) {
      put_u64(f, static_cast<std::uint64_t>(rom.iface_ids[li]));
      put_mat(f, basis.S[rom.iface_ids[li]]);
      put_u64(f, static_cast<std::uint64_t>(rom.g_proj[li].size()));
      put_doubles(f, rom.g_proj[li].data(), static_cast<size_t>(rom.g_proj[li].size()));
      put_doubles(f, rom.q_proj[li].data(), static_cast<size_t>(rom.q_proj[li].size()));
    }
    for (const Mat& m : rom.ladder_hat) put_mat(f, m);
    for (const Mat& m : rom.ladder) put_mat(f, m);
    std::fclose(f);
  }
  std::ofstream mf(fs::path(dir) / "manifest.json");
  if (!mf) throw ConfigError("cannot write ROM manifest in " + dir);
  mf << "{\n  \"format\": \"mswave-rom-archive\",\n  \"version\": 1,\n  \"num_cells\": " << roms.size()
     << ",\n  \"num_interfaces\": " << basis.S.size() << ",\n  \"omega_max\": " << json_double(basis.omega_max)
     << ",\n  \"epsilon\": " << json_double(basis.epsilon) << ",\n  \"m\": " << opt.m
     << ",\n  \"max_basis_per_interface\": " << opt.max_basis_per_interface << ",\n  \"cells\": ["
     << cells.str() << (roms.empty() ? "]" : "\n  ]") << "\n}\n";
}

RomArchive read_rom_archive(const std::string& dir) {
  namespace fs = std::filesystem;
  std::ifstream mf(fs::path(dir) / "manifest.json");
  if (!mf) throw ConfigError("missing manifest.json in " + dir);
  std::stringstream ss;
  ss << mf.rdbuf();
  const std::string text = ss.str();
  const Json manifest = JsonParser(text).parse();
  const Json* fmt = manifest.find("format");
  if (!fmt || fmt->kind != Json::Str || fmt->str != "mswave-rom-archive")
    throw ConfigError("not a ROM archive: " + dir);

  RomArchive ar;
  ar.opt.m = static_cast<int>(manifest.at("m").integer());
  ar.opt.omega_max = manifest.at("omega_max").number();
  ar.opt.epsilon_rel = manifest.at("epsilon").number();
  const Json* mb = manifest.find("max_basis_per_interface");
  ar.opt.max_basis_per_interface = mb ? static_cast<int>(mb->integer()) : 0;
  ar.basis.omega_max = ar.opt.omega_max;
  ar.basis.epsilon = ar.opt.epsilon_rel;
  const size_t n_ifaces = static_cast<size_t>(manifest.at("num_interfaces").integer());
  ar.basis.S.resize(n_ifaces);
  ar.basis.kept_eigs.resize(n_ifaces);
  ar.basis.tail.assign(n_ifaces, 0.0);

  for (const Json& c : manifest.at("cells").arr) {
    const fs::path path = fs::path(dir) / c.at("file").string();
    std::FILE* f = std::fopen(path.c_str(), "rb");
    if (!f) throw ConfigError("missing ROM container: " + path.string());
    Container in(f, path.string());
    char magic[8];
    if (std::fread(magic, 1, 8, f) != 8 || std::memcmp(magic, kMagic, 8) != 0)
      throw ConfigError("bad magic in ROM container: " + path.string());
    SubdomainROM rom;
    rom.cell = static_cast<int>(in.u64());
    rom.m = static_cast<int>(in.u64());
    rom.ktilde = static_cast<int>(in.u64());
    const auto nif = in.u64();
    in.doubles(&rom.shift, 1);
    rom.iface_offsets = {0};
    for (std::uint64_t i = 0; i < nif; ++i) {
      const int fid = static_cast<int>(in.u64());
      rom.iface_ids.push_back(fid);
      Mat S = in.mat();
      const auto glen = static_cast<long>(in.u64());
      Vec g(glen), q(glen);
      in.doubles(g.data(), static_cast<size_t>(glen));
      in.doubles(q.data(), static_cast<size_t>(glen));
      if (S.cols() != glen)
        throw ConfigError("interface basis / projected I/O size mismatch in " + path.string());
      if (fid < 0 || static_cast<size_t>(fid) >= n_ifaces)
        throw ConfigError("interface id out of range in " + path.string());
      if (ar.basis.S[fid].size() == 0) {
        ar.basis.S[fid] = S;
      } else if (ar.basis.S[fid].rows() != S.rows() || ar.basis.S[fid].cols() != S.cols() ||
                 std::memcmp(ar.basis.S[fid].data(), S.data(), sizeof(double) * S.size()) != 0) {
        throw ConfigError("mismatched interface bases between neighbor cells (interface " +
                          std::to_string(fid) + ")");
      }
      rom.g_proj.push_back(std::move(g));
      rom.q_proj.push_back(std::move(q));
      rom.iface_offsets.push_back(rom.iface_offsets.back() + static_cast<int>(glen));
    }
    for (int k = 0; k < rom.m; ++k) rom.ladder_hat.push_back(in.mat());
    for (int k = 0; k < rom.m; ++k) rom.ladder.push_back(in.mat());
    if (rom.iface_offsets.back() != rom.ktilde) throw ConfigError("inconsistent ktilde in " + path.string());
    ar.roms.push_back(std::move(rom));
  }
  std::sort(ar.roms.begin(), ar.roms.end(),
            [](const SubdomainROM& a, const SubdomainROM& b) { return a.cell < b.cell; });
  return ar;
}

}  // namespace mswave

// ------------------------------------------------------------------ C ABI ---

// re-raise an ABI return code with its own class, so the caller sees the
// code msw_create / msw_set_* returned (2 config, 3 numerical, 4 device)
static void rethrow(int rc) {
  if (rc == MSW_OK) return;
  const std::string msg = msw_last_error();
  if (rc == MSW_NUMERICAL_ERROR) throw mswb::NumericalError(msg);
  if (rc == MSW_CUDA_ERROR) throw mswb::CudaError(msg);
  throw mswb::ConfigError(msg);
}

extern "C" int msw_create_from_archive(const char* dir, int device, msw_handle* out) {
  return mswb::guarded([&] {
    if (!dir || !out) throw mswb::ConfigError("null argument");
    mswave::RomArchive ar;
    try {
      ar = mswave::read_rom_archive(dir);
    } catch (const mswave::ConfigError& e) {
      throw mswb::ConfigError(e.what());
    }
    const int nc = static_cast<int>(ar.roms.size());
    const int nf = static_cast<int>(ar.basis.S.size());
    for (int c = 0; c < nc; ++c)
      if (ar.roms[c].cell != c) throw mswb::ConfigError("ROM archive cells are not numbered 0..n-1");
    // interface topology from the cells' ascending interface lists: ci < cj
    std::vector<int32_t> ci(nf, -1), cj(nf, -1), li(nf, -1), lj(nf, -1), sz(nf, 0);
    std::vector<int32_t> cm(nc), ckt(nc), cptr(1, 0), cids, coff;
    std::vector<int64_t> loff(nc);
    std::vector<double> lad;
    for (int c = 0; c < nc; ++c) {
      const mswave::SubdomainROM& r = ar.roms[c];
      cm[c] = r.m;
      ckt[c] = r.ktilde;
      for (size_t l = 0; l < r.iface_ids.size(); ++l) {
        const int f = r.iface_ids[l];
        cids.push_back(f);
        coff.push_back(r.iface_offsets[l]);
        if (ci[f] < 0) {
          ci[f] = c;
          li[f] = static_cast<int32_t>(l);
        } else if (cj[f] < 0) {
          cj[f] = c;
          lj[f] = static_cast<int32_t>(l);
        } else {
          throw mswb::ConfigError("interface " + std::to_string(f) + " listed by more than two cells");
        }
      }
      cptr.push_back(static_cast<int32_t>(cids.size()));
      loff[c] = static_cast<int64_t>(lad.size());
      for (const mswave::Mat& L : r.ladder) lad.insert(lad.end(), L.data(), L.data() + L.size());
      for (const mswave::Mat& L : r.ladder_hat) lad.insert(lad.end(), L.data(), L.data() + L.size());
    }
    std::vector<int64_t> ioff(nf + 1, 0);
    for (int f = 0; f < nf; ++f) {
      if (ci[f] < 0) throw mswb::ConfigError("interface " + std::to_string(f) + " belongs to no cell");
      sz[f] = static_cast<int32_t>(ar.basis.S[f].cols());
      ioff[f + 1] = ioff[f] + sz[f];
    }
    msw_system_desc d{};
    d.n_cells = nc;
    d.n_ifaces = nf;
    d.cell_m = cm.data();
    d.cell_ktilde = ckt.data();
    d.cell_iface_ptr = cptr.data();
    d.cell_iface_ids = cids.data();
    d.cell_iface_offsets = coff.data();
    d.cell_ladder_off = loff.data();
    d.ladders = lad.data();
    d.iface_ci = ci.data();
    d.iface_cj = cj.data();
    d.iface_li = li.data();
    d.iface_lj = lj.data();
    d.iface_size = sz.data();
    d.iface_mass = nullptr;  // assemble_system's Cholesky masses (msolver.cpp:66-74)
    msw_handle h = nullptr;
    rethrow(msw_create(&d, device, &h));
    // the archive's own source / receiver (both sides must agree bitwise,
    // msolver.cpp:58-64)
    std::vector<double> g(static_cast<size_t>(ioff[nf]), 0.0);
    std::vector<int32_t> rptr{0}, rif;
    std::vector<double> rq;
    for (int f = 0; f < nf; ++f) {
      const mswave::Vec& gi = ar.roms[ci[f]].g_proj[li[f]];
      const mswave::Vec& qi = ar.roms[ci[f]].q_proj[li[f]];
      if (cj[f] >= 0) {
        const mswave::Vec& gj = ar.roms[cj[f]].g_proj[lj[f]];
        const mswave::Vec& qj = ar.roms[cj[f]].q_proj[lj[f]];
        // value comparison as msolver.cpp:60-63 ((a - b).cwiseAbs().maxCoeff() != 0:
        // -0.0 equals +0.0, a NaN disagrees)
        auto differ = [](const mswave::Vec& a, const mswave::Vec& b) {
          if (a.size() != b.size()) return true;
          for (long i = 0; i < a.size(); ++i)
            if (!(std::abs(a[i] - b[i]) == 0.0)) return true;
          return false;
        };
        if (differ(gi, gj) || differ(qi, qj)) {
          msw_destroy(h);
          throw mswb::ConfigError("projected I/O disagrees between the two sides of interface " +
                                  std::to_string(f));
        }
      }
      bool nz = false;
      for (long i = 0; i < gi.size(); ++i) {
        g[ioff[f] + i] = gi[i];
        nz = nz || qi[i] != 0.0;
      }
      if (nz) {
        rif.push_back(f);
        rq.insert(rq.end(), qi.data(), qi.data() + qi.size());
      }
    }
    rptr.push_back(static_cast<int32_t>(rif.size()));
    int rc = msw_set_sources(h, 1, g.data());
    if (rc == 0) rc = msw_set_receivers(h, 1, rptr.data(), rif.data(), rq.data());
    if (rc != 0) {
      msw_destroy(h);
      rethrow(rc);
    }
    *out = h;
  });
}
