// io.cu — the reference's on-disk formats on the host side of the C ABI
// (SURVEY §8f-3), so CPU goldens and GPU outputs can be exchanged and diffed
// byte for byte:
//   * `unisparse.tn` tensor files (tensor_io.hpp:9-14, tensor_io.cpp:31-81):
//     12-byte magic "unisparse.tn", u32 version 1, u32 H, L, d_k (little
//     endian), then H*L*d_k f32 values, head major;
//   * RLE block-mask JSON (selection.cpp:90-144): {"H","N","P","heads","version"}
//     with heads[h][i] = [[start, len], ...] runs of selected key blocks, written
//     in nlohmann::json's dump(1, '\t') layout (keys sorted, one tab per level).
// Error texts follow the reference ("tensor file <path>: bad magic at offset 0").
// Pure host code: no CUDA call is made here.
#include <cstdint>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <fstream>
#include <sstream>
#include <string>
#include <vector>

#include "host_util.hpp"

namespace us {
namespace {

constexpr char kMagic[12] = {'u', 'n', 'i', 's', 'p', 'a', 'r', 's', 'e', '.', 't', 'n'};
constexpr uint32_t kVersion = 1;

us_status io_fail(const std::string& msg) {
  set_error(msg);
  return US_ERR_IO;
}

us_status tensor_fail(const char* path, const std::string& what) {
  return io_fail(std::string("tensor file ") + path + ": " + what);
}

// Reads and validates the header; leaves the stream at the payload.
us_status read_header(std::ifstream& is, const char* path, uint32_t* H, uint32_t* L, uint32_t* d) {
  if (!is) return tensor_fail(path, "cannot open for reading");
  char magic[12];
  is.read(magic, 12);
  if (!is || std::memcmp(magic, kMagic, 12) != 0) return tensor_fail(path, "bad magic at offset 0");
  uint32_t v = 0;
  is.read(reinterpret_cast<char*>(&v), 4);
  if (!is || v != kVersion) return tensor_fail(path, "unsupported version " + std::to_string(v) + " at offset 12");
  is.read(reinterpret_cast<char*>(H), 4);
  is.read(reinterpret_cast<char*>(L), 4);
  is.read(reinterpret_cast<char*>(d), 4);
  if (!is) return tensor_fail(path, "truncated header");
  if (*H == 0 || *L == 0 || *d == 0) return tensor_fail(path, "zero dimension in header at offset 16");
  return US_OK;
}

// Shortest decimal that round-trips (nlohmann::json prints doubles this way,
// with a trailing ".0" on integral values).
std::string json_double(double x) {
  char buf[64];
  for (int p = 1; p <= 17; ++p) {
    std::snprintf(buf, sizeof buf, "%.*g", p, x);
    if (std::strtod(buf, nullptr) == x) break;
  }
  std::string s(buf);
  if (s.find_first_of(".eEn") == std::string::npos) s += ".0";
  return s;
}

// ---- a minimal JSON reader (objects, arrays, numbers, strings)
struct JVal {
  enum Kind { NUM, ARR, OBJ, STR, OTHER } kind = OTHER;
  double num = 0.0;
  std::string str;
  std::vector<JVal> items;                  // array elements / object values
  std::vector<std::string> keys;            // object keys
  const JVal* get(const std::string& k) const {
    for (size_t i = 0; i < keys.size(); ++i)
      if (keys[i] == k) return &items[i];
    return nullptr;
  }
};

struct JParser {
  const std::string& s;
  size_t i = 0;
  bool ok = true;
  explicit JParser(const std::string& src) : s(src) {}
  void ws() {
    while (i < s.size() && (s[i] == ' ' || s[i] == '\t' || s[i] == '\n' || s[i] == '\r')) ++i;
  }
  JVal value() {
    JVal v;
    ws();
    if (i >= s.size()) {
      ok = false;
      return v;
    }
    const char c = s[i];
    if (c == '[' || c == '{') {
      const bool obj = c == '{';
      v.kind = obj ? JVal::OBJ : JVal::ARR;
      ++i;
      ws();
      if (i < s.size() && s[i] == (obj ? '}' : ']')) {
        ++i;
        return v;
      }
      while (ok) {
        if (obj) {
          JVal k = value();
          if (k.kind != JVal::STR) {
            ok = false;
            break;
          }
          ws();
          if (i >= s.size() || s[i] != ':') {
            ok = false;
            break;
          }
          ++i;
          v.keys.push_back(k.str);
        }
        v.items.push_back(value());
        ws();
        if (i < s.size() && s[i] == ',') {
          ++i;
          continue;
        }
        if (i < s.size() && s[i] == (obj ? '}' : ']')) {
          ++i;
          break;
        }
        ok = false;
      }
    } else if (c == '"') {
      v.kind = JVal::STR;
      ++i;
      while (i < s.size() && s[i] != '"') v.str += s[i++];
      if (i >= s.size()) ok = false;
      ++i;
    } else {
      char* end = nullptr;
      v.num = std::strtod(s.c_str() + i, &end);
      if (end == s.c_str() + i) {
        ok = false;
        return v;
      }
      v.kind = JVal::NUM;
      i = size_t(end - s.c_str());
    }
    return v;
  }
};

}  // namespace
}  // namespace us

using namespace us;

extern "C" {

us_status us_write_tensor(const char* path, const float* data, int32_t H, int32_t L, int32_t d_k) {
  if (!path || !data) return io_fail("write_tensor: null argument");
  if (H <= 0) return tensor_fail(path, "refusing to write empty head stack");
  if (L <= 0 || d_k <= 0) return tensor_fail(path, "heads disagree on shape");
  std::ofstream os(path, std::ios::binary);
  if (!os) return tensor_fail(path, "cannot open for writing");
  os.write(kMagic, 12);
  const uint32_t hdr[4] = {kVersion, uint32_t(H), uint32_t(L), uint32_t(d_k)};
  os.write(reinterpret_cast<const char*>(hdr), sizeof hdr);
  os.write(reinterpret_cast<const char*>(data), std::streamsize(sizeof(float)) * H * L * d_k);
  if (!os) return tensor_fail(path, "write failed");
  return US_OK;
}

us_status us_read_tensor_header(const char* path, int32_t* H, int32_t* L, int32_t* d_k) {
  if (!path || !H || !L || !d_k) return io_fail("read_tensor: null argument");
  std::ifstream is(path, std::ios::binary);
  uint32_t h = 0, l = 0, d = 0;
  us_status s = read_header(is, path, &h, &l, &d);
  if (s != US_OK) return s;
  *H = int32_t(h);
  *L = int32_t(l);
  *d_k = int32_t(d);
  return US_OK;
}

us_status us_read_tensor(const char* path, float* out, size_t capacity_floats) {
  if (!path || !out) return io_fail("read_tensor: null argument");
  std::ifstream is(path, std::ios::binary);
  uint32_t H = 0, L = 0, d = 0;
  us_status s = read_header(is, path, &H, &L, &d);
  if (s != US_OK) return s;
  const uint64_t per_head = uint64_t(L) * d;
  if (uint64_t(H) * per_head > capacity_floats) return tensor_fail(path, "destination smaller than H*L*d_k");
  for (uint32_t h = 0; h < H; ++h) {
    is.read(reinterpret_cast<char*>(out + h * per_head), std::streamsize(sizeof(float) * per_head));
    if (uint64_t(is.gcount()) != sizeof(float) * per_head)
      return tensor_fail(path, "payload shorter than header H*L*d_k at offset " +
                                   std::to_string(28 + uint64_t(sizeof(float)) * h * per_head));
  }
  is.peek();
  if (!is.eof()) return tensor_fail(path, "trailing bytes beyond header H*L*d_k");
  return US_OK;
}

us_status us_save_mask_json(const char* path, const uint32_t* mask_bits, int32_t H, int32_t N, int32_t c_h,
                            double P) {
  if (!path || !mask_bits || H <= 0 || N <= 0 || c_h <= 0 || H % c_h)
    return io_fail("save_mask_json: bad arguments");
  const int W = (N + 31) / 32;
  std::ostringstream o;
  const auto tabs = [&](int n) { o << std::string(size_t(n), '\t'); };
  o << "{\n";
  tabs(1);
  o << "\"H\": " << H << ",\n";
  tabs(1);
  o << "\"N\": " << N << ",\n";
  tabs(1);
  o << "\"P\": " << json_double(P) << ",\n";
  tabs(1);
  o << "\"heads\": [\n";
  for (int h = 0; h < H; ++h) {
    const uint32_t* plane = mask_bits + size_t(h / c_h) * N * W;  // selection.cpp:80-84 broadcast
    tabs(2);
    o << "[\n";
    for (int i = 0; i < N; ++i) {
      const uint32_t* row = plane + size_t(i) * W;
      std::vector<std::pair<int, int>> runs;
      int j0 = -1;
      for (int b = 0; b <= N; ++b) {
        const bool on = b < N && ((row[b >> 5] >> (b & 31)) & 1u);
        if (on && j0 < 0) j0 = b;
        if (!on && j0 >= 0) {
          runs.emplace_back(j0, b - j0);
          j0 = -1;
        }
      }
      tabs(3);
      if (runs.empty()) {
        o << "[]";
      } else {
        o << "[\n";
        for (size_t r = 0; r < runs.size(); ++r) {
          // nlohmann prints the two-element run compactly: [start,len]
          tabs(4);
          o << "[" << runs[r].first << "," << runs[r].second << "]" << (r + 1 < runs.size() ? ",\n" : "\n");
        }
        tabs(3);
        o << "]";
      }
      o << (i + 1 < N ? ",\n" : "\n");
    }
    tabs(2);
    o << "]" << (h + 1 < H ? ",\n" : "\n");
  }
  tabs(1);
  o << "],\n";
  tabs(1);
  o << "\"version\": 1\n}\n";
  std::ofstream os(path);
  if (!os) return io_fail(std::string("save_mask_json: cannot open ") + path);
  os << o.str();
  if (!os) return io_fail(std::string("save_mask_json: write failed ") + path);
  return US_OK;
}

// Reads H, N, P (out_bits == NULL) or the per-head masks [H][N][ceil(N/32)].
us_status us_load_mask_json(const char* path, int32_t* H, int32_t* N, double* P, uint32_t* out_bits,
                            size_t capacity_words) {
  if (!path || !H || !N || !P) return io_fail("load_mask_json: null argument");
  std::ifstream is(path);
  if (!is) return io_fail(std::string("load_mask_json: cannot open ") + path);
  std::stringstream ss;
  ss << is.rdbuf();
  const std::string text = ss.str();
  JParser jp(text);
  const JVal root = jp.value();
  const auto bad = [&](const std::string& what) { return io_fail(std::string("load_mask_json: ") + path + ": " + what); };
  if (!jp.ok || root.kind != JVal::OBJ) return bad("parse error");
  const JVal *jh = root.get("H"), *jn = root.get("N"), *jpv = root.get("P"), *heads = root.get("heads");
  if (!jh || !jn || !jpv || !heads || jh->kind != JVal::NUM || jn->kind != JVal::NUM || jpv->kind != JVal::NUM ||
      heads->kind != JVal::ARR)
    return bad("missing H / N / P / heads");
  *H = int32_t(jh->num);
  *N = int32_t(jn->num);
  *P = jpv->num;
  if (!out_bits) return US_OK;
  const int W = (*N + 31) / 32;
  if (size_t(*H) * (*N) * W > capacity_words) return bad("destination too small");
  std::memset(out_bits, 0, sizeof(uint32_t) * size_t(*H) * (*N) * W);
  if (int(heads->items.size()) != *H) return bad("heads length differs from H");
  for (int h = 0; h < *H; ++h) {
    const JVal& rows = heads->items[h];
    if (rows.kind != JVal::ARR || int(rows.items.size()) != *N) return bad("rows length differs from N");
    for (int i = 0; i < *N; ++i) {
      for (const JVal& run : rows.items[i].items) {
        if (run.kind != JVal::ARR || run.items.size() != 2) return bad("malformed run");
        const int start = int(run.items[0].num), len = int(run.items[1].num);
        if (start < 0 || len < 0 || start + len > *N) return bad("run outside [0, N)");
        for (int b = start; b < start + len; ++b)
          out_bits[(size_t(h) * (*N) + i) * W + (b >> 5)] |= 1u << (b & 31);
      }
    }
  }
  return US_OK;
}

}  // extern "C"
