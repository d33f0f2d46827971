// Artifact formats of the D2FT pipeline: score tables,
// schedule tables, batch metrics and training history as JSON / CSV, the
// wire formats of the reference's serialize.hpp (core/include/d2ft/
// serialize.hpp:21-53, core/src/serialize.cpp:66-222), so files written here
// are read by the reference's CLI pipeline and vice versa.
//
// Host code only (file I/O and text).  The reference writes JSON with
// nlohmann::json::dump(2): keys in sorted order, two-space indent, one array
// element per line, doubles as the shortest round-trip digits laid out by
// nlohmann's format (1.0, 0.001, 1e-05, 1.5e+20, non-finite -> null).  This
// writer reproduces that layout and nlohmann's Grisu2 digits (json_double);
// byte-compared with the compiled reference in tests/test_artifacts_vs_ref_cpu.py.
// CSV doubles use format_double = std::to_chars, as the reference does.
#include <array>
#include <charconv>
#include <cmath>
#include <cstdio>
#include <cstring>
#include <fstream>
#include <map>
#include <memory>
#include <sstream>
#include <string>
#include <vector>

#include "../../include/d2ft_b200.h"
#include "common.cuh"

namespace d2ft_b200 {
namespace {

// format_double (serialize.cpp:17-21): shortest round trip, "%g"-free
std::string format_double(double v) {
  char buf[64];
  auto r = std::to_chars(buf, buf + sizeof(buf), v);
  return std::string(buf, r.ptr);
}

// ---- JSON doubles: nlohmann::json 3.11 dump() digits (Grisu2) and layout.
// nlohmann prints a double with Grisu2 (Loitsch, "Printing Floating-Point
// Numbers Quickly and Accurately with Integers", PLDI 2010): digits of the
// upper boundary M+ of the value's rounding interval (conservatively shrunk
// by one unit at 64-bit precision) until the rest fits the interval, then
// one weeding step toward the value.  The result is usually but not always
// the shortest round-trip string, so std::to_chars cannot stand in for it.
// Restated here: 64-bit "diy" floats, the cached powers 10^k (k = -300 + 8i,
// significands rounded to nearest; tools/gen_pow10_table.py), exponent window
// [-60, -32].
struct DiyFp {
  uint64_t f;
  int e;
};

DiyFp diy_mul(DiyFp a, DiyFp b) {  // upper 64 bits of the product, rounded half up
  unsigned __int128 p = (unsigned __int128)a.f * b.f;
  p += (unsigned __int128)1 << 63;
  return DiyFp{(uint64_t)(p >> 64), a.e + b.e + 64};
}

DiyFp diy_normalize(DiyFp x) {
  while (!(x.f >> 63)) {
    x.f <<= 1;
    --x.e;
  }
  return x;
}

struct Pow10 {
  uint64_t f;
  int e, k;
};
constexpr Pow10 kPow10[79] = {
    {0xAB70FE17C79AC6CAull, -1060, -300},
    {0xFF77B1FCBEBCDC4Full, -1034, -292},
    {0xBE5691EF416BD60Cull, -1007, -284},
    {0x8DD01FAD907FFC3Cull, -980, -276},
    {0xD3515C2831559A83ull, -954, -268},
    {0x9D71AC8FADA6C9B5ull, -927, -260},
    {0xEA9C227723EE8BCBull, -901, -252},
    {0xAECC49914078536Dull, -874, -244},
    {0x823C12795DB6CE57ull, -847, -236},
    {0xC21094364DFB5637ull, -821, -228},
    {0x9096EA6F3848984Full, -794, -220},
    {0xD77485CB25823AC7ull, -768, -212},
    {0xA086CFCD97BF97F4ull, -741, -204},
    {0xEF340A98172AACE5ull, -715, -196},
    {0xB23867FB2A35B28Eull, -688, -188},
    {0x84C8D4DFD2C63F3Bull, -661, -180},
    {0xC5DD44271AD3CDBAull, -635, -172},
    {0x936B9FCEBB25C996ull, -608, -164},
    {0xDBAC6C247D62A584ull, -582, -156},
    {0xA3AB66580D5FDAF6ull, -555, -148},
    {0xF3E2F893DEC3F126ull, -529, -140},
    {0xB5B5ADA8AAFF80B8ull, -502, -132},
    {0x87625F056C7C4A8Bull, -475, -124},
    {0xC9BCFF6034C13053ull, -449, -116},
    {0x964E858C91BA2655ull, -422, -108},
    {0xDFF9772470297EBDull, -396, -100},
    {0xA6DFBD9FB8E5B88Full, -369, -92},
    {0xF8A95FCF88747D94ull, -343, -84},
    {0xB94470938FA89BCFull, -316, -76},
    {0x8A08F0F8BF0F156Bull, -289, -68},
    {0xCDB02555653131B6ull, -263, -60},
    {0x993FE2C6D07B7FACull, -236, -52},
    {0xE45C10C42A2B3B06ull, -210, -44},
    {0xAA242499697392D3ull, -183, -36},
    {0xFD87B5F28300CA0Eull, -157, -28},
    {0xBCE5086492111AEBull, -130, -20},
    {0x8CBCCC096F5088CCull, -103, -12},
    {0xD1B71758E219652Cull, -77, -4},
    {0x9C40000000000000ull, -50, 4},
    {0xE8D4A51000000000ull, -24, 12},
    {0xAD78EBC5AC620000ull, 3, 20},
    {0x813F3978F8940984ull, 30, 28},
    {0xC097CE7BC90715B3ull, 56, 36},
    {0x8F7E32CE7BEA5C70ull, 83, 44},
    {0xD5D238A4ABE98068ull, 109, 52},
    {0x9F4F2726179A2245ull, 136, 60},
    {0xED63A231D4C4FB27ull, 162, 68},
    {0xB0DE65388CC8ADA8ull, 189, 76},
    {0x83C7088E1AAB65DBull, 216, 84},
    {0xC45D1DF942711D9Aull, 242, 92},
    {0x924D692CA61BE758ull, 269, 100},
    {0xDA01EE641A708DEAull, 295, 108},
    {0xA26DA3999AEF774Aull, 322, 116},
    {0xF209787BB47D6B85ull, 348, 124},
    {0xB454E4A179DD1877ull, 375, 132},
    {0x865B86925B9BC5C2ull, 402, 140},
    {0xC83553C5C8965D3Dull, 428, 148},
    {0x952AB45CFA97A0B3ull, 455, 156},
    {0xDE469FBD99A05FE3ull, 481, 164},
    {0xA59BC234DB398C25ull, 508, 172},
    {0xF6C69A72A3989F5Cull, 534, 180},
    {0xB7DCBF5354E9BECEull, 561, 188},
    {0x88FCF317F22241E2ull, 588, 196},
    {0xCC20CE9BD35C78A5ull, 614, 204},
    {0x98165AF37B2153DFull, 641, 212},
    {0xE2A0B5DC971F303Aull, 667, 220},
    {0xA8D9D1535CE3B396ull, 694, 228},
    {0xFB9B7CD9A4A7443Cull, 720, 236},
    {0xBB764C4CA7A44410ull, 747, 244},
    {0x8BAB8EEFB6409C1Aull, 774, 252},
    {0xD01FEF10A657842Cull, 800, 260},
    {0x9B10A4E5E9913129ull, 827, 268},
    {0xE7109BFBA19C0C9Dull, 853, 276},
    {0xAC2820D9623BF429ull, 880, 284},
    {0x80444B5E7AA7CF85ull, 907, 292},
    {0xBF21E44003ACDD2Dull, 933, 300},
    {0x8E679C2F5E44FF8Full, 960, 308},
    {0xD433179D9C8CB841ull, 986, 316},
    {0x9E19DB92B4E31BA9ull, 1013, 324},
};

// Digits of the positive finite double v: v ~= digits * 10^dexp.
void grisu2_digits(double v, std::string& digits, int& dexp) {
  uint64_t bits;
  std::memcpy(&bits, &v, 8);
  const uint64_t E = bits >> 52, F = bits & ((1ull << 52) - 1);
  const DiyFp w0 = E == 0 ? DiyFp{F, -1074} : DiyFp{F + (1ull << 52), (int)E - 1075};
  // rounding interval [m-, m+] around v; the lower neighbour is closer when v
  // is a power of two above the smallest normal
  const DiyFp mp0{2 * w0.f + 1, w0.e - 1};
  const DiyFp mm0 = (F == 0 && E > 1) ? DiyFp{4 * w0.f - 1, w0.e - 2} : DiyFp{2 * w0.f - 1, w0.e - 1};
  const DiyFp mp = diy_normalize(mp0);
  const DiyFp mm{mm0.f << (mm0.e - mp.e), mp.e};
  const DiyFp w = diy_normalize(w0);
  // cached power c ~= 10^-k with -60 <= e(w * c) <= -32
  const int fe = -60 - mp.e - 1;
  const int kk = (fe * 78913) / (1 << 18) + (fe > 0 ? 1 : 0);
  const Pow10 c = kPow10[(300 + kk + 7) / 8];
  const DiyFp cw{c.f, c.e};
  const DiyFp W = diy_mul(w, cw), Wm = diy_mul(mm, cw), Wp = diy_mul(mp, cw);
  const DiyFp Mm{Wm.f + 1, Wm.e}, Mp{Wp.f - 1, Wp.e};
  dexp = -c.k;
  uint64_t delta = Mp.f - Mm.f, dist = Mp.f - W.f;
  const int sh = -Mp.e;
  const uint64_t one = 1ull << sh;
  uint32_t p1 = (uint32_t)(Mp.f >> sh);
  uint64_t p2 = Mp.f & (one - 1);
  digits.clear();
  // weed the last digit toward w while it stays inside the interval
  auto round_last = [&](uint64_t rest, uint64_t ten_k) {
    while (rest < dist && delta - rest >= ten_k && (rest + ten_k < dist || dist - rest > rest + ten_k - dist)) {
      digits.back()--;
      rest += ten_k;
    }
  };
  uint32_t pow10 = 1;
  int n = 1;
  while (n < 10 && p1 >= pow10 * 10u) {
    pow10 *= 10u;
    ++n;
  }
  // integral part
  while (n > 0) {
    digits.push_back((char)('0' + p1 / pow10));
    p1 %= pow10;
    --n;
    const uint64_t rest = ((uint64_t)p1 << sh) + p2;
    if (rest <= delta) {
      dexp += n;
      round_last(rest, (uint64_t)pow10 << sh);
      return;
    }
    pow10 /= 10u;
  }
  // fractional part
  int m = 0;
  for (;;) {
    p2 *= 10;
    digits.push_back((char)('0' + (p2 >> sh)));
    p2 &= one - 1;
    ++m;
    delta *= 10;
    dist *= 10;
    if (p2 <= delta) break;
  }
  dexp -= m;
  round_last(p2, one);
}

// nlohmann::detail::to_chars layout of a finite double: fixed notation for
// 10^-4 <= |v| < 10^15 (".0" on integral values), else d.ddde[+-]XX
std::string json_double(double v) {
  if (!std::isfinite(v)) return "null";
  std::string out;
  if (std::signbit(v)) {
    out += '-';
    v = -v;
  }
  if (v == 0.0) return out + "0.0";
  std::string digits;
  int dexp = 0;
  grisu2_digits(v, digits, dexp);
  const int k = (int)digits.size();
  const int n = k + dexp;  // value = 0.digits * 10^n
  constexpr int kMinExp = -4, kMaxExp = 15;
  if (k <= n && n <= kMaxExp) return out + digits + std::string(n - k, '0') + ".0";
  if (0 < n && n <= kMaxExp) return out + digits.substr(0, n) + "." + digits.substr(n);
  if (kMinExp < n && n <= 0) return out + "0." + std::string(-n, '0') + digits;
  out += digits.substr(0, 1);
  if (k > 1) out += "." + digits.substr(1);
  int e = n - 1;
  out += 'e';
  out += e < 0 ? '-' : '+';
  e = e < 0 ? -e : e;
  char eb[8];
  std::snprintf(eb, sizeof(eb), e < 10 ? "0%d" : "%d", e);
  return out + eb;
}

std::string json_string(const std::string& s) {
  std::string o = "\"";
  for (unsigned char c : s) {
    switch (c) {
      case '"': o += "\\\""; break;
      case '\\': o += "\\\\"; break;
      case '\b': o += "\\b"; break;
      case '\f': o += "\\f"; break;
      case '\n': o += "\\n"; break;
      case '\r': o += "\\r"; break;
      case '\t': o += "\\t"; break;
      default:
        if (c < 0x20) {
          char b[8];
          std::snprintf(b, sizeof(b), "\\u%04x", c);
          o += b;
        } else {
          o += (char)c;
        }
    }
  }
  return o + "\"";
}

// ---------------------------------------------------------------- JSON values
struct Json {
  enum Kind { Null, Bool, Int, Float, Str, Arr, Obj } kind = Null;
  bool b = false;
  long long i = 0;
  double f = 0.0;
  std::string s;
  std::vector<Json> a;
  std::map<std::string, Json> o;  // sorted keys, as nlohmann::json's default object

  static Json integer(long long v) {
    Json j;
    j.kind = Int;
    j.i = v;
    return j;
  }
  static Json number(double v) {
    Json j;
    j.kind = Float;
    j.f = v;
    return j;
  }
  static Json string(std::string v) {
    Json j;
    j.kind = Str;
    j.s = std::move(v);
    return j;
  }
  static Json array() {
    Json j;
    j.kind = Arr;
    return j;
  }
  static Json object() {
    Json j;
    j.kind = Obj;
    return j;
  }
};

// nlohmann::json::dump(2) layout
void dump(const Json& j, std::string& out, int indent) {
  switch (j.kind) {
    case Json::Null: out += "null"; return;
    case Json::Bool: out += j.b ? "true" : "false"; return;
    case Json::Int: out += std::to_string(j.i); return;
    case Json::Float: out += json_double(j.f); return;
    case Json::Str: out += json_string(j.s); return;
    case Json::Arr:
      if (j.a.empty()) {
        out += "[]";
        return;
      }
      out += "[\n";
      for (size_t x = 0; x < j.a.size(); ++x) {
        out.append(indent + 2, ' ');
        dump(j.a[x], out, indent + 2);
        out += x + 1 < j.a.size() ? ",\n" : "\n";
      }
      out.append(indent, ' ');
      out += ']';
      return;
    case Json::Obj: {
      if (j.o.empty()) {
        out += "{}";
        return;
      }
      out += "{\n";
      size_t x = 0;
      for (const auto& kv : j.o) {
        out.append(indent + 2, ' ');
        out += json_string(kv.first) + ": ";
        dump(kv.second, out, indent + 2);
        out += ++x < j.o.size() ? ",\n" : "\n";
      }
      out.append(indent, ' ');
      out += '}';
      return;
    }
  }
}

std::string dump2(const Json& j) {
  std::string out;
  dump(j, out, 0);
  return out + "\n";
}

// Minimal RFC 8259 parser (the subset nlohmann accepts for these files).
struct Parser {
  const char* p;
  const char* end;
  bool ok = true;
  void ws() {
    while (p < end && (*p == ' ' || *p == '\n' || *p == '\r' || *p == '\t')) ++p;
  }
  bool lit(const char* w) {
    const size_t n = std::strlen(w);
    if ((size_t)(end - p) >= n && std::memcmp(p, w, n) == 0) {
      p += n;
      return true;
    }
    return false;
  }
  Json fail() {
    ok = false;
    return Json{};
  }
  Json value(int depth) {
    if (depth > 64) return fail();
    ws();
    if (p >= end) return fail();
    if (*p == '{') {
      ++p;
      Json j = Json::object();
      ws();
      if (p < end && *p == '}') {
        ++p;
        return j;
      }
      while (ok) {
        ws();
        if (p >= end || *p != '"') return fail();
        Json key = str();
        if (!ok) return j;
        ws();
        if (p >= end || *p != ':') return fail();
        ++p;
        j.o[key.s] = value(depth + 1);
        ws();
        if (p < end && *p == ',') {
          ++p;
          continue;
        }
        if (p < end && *p == '}') {
          ++p;
          return j;
        }
        return fail();
      }
      return j;
    }
    if (*p == '[') {
      ++p;
      Json j = Json::array();
      ws();
      if (p < end && *p == ']') {
        ++p;
        return j;
      }
      while (ok) {
        j.a.push_back(value(depth + 1));
        ws();
        if (p < end && *p == ',') {
          ++p;
          continue;
        }
        if (p < end && *p == ']') {
          ++p;
          return j;
        }
        return fail();
      }
      return j;
    }
    if (*p == '"') return str();
    if (lit("true")) {
      Json j;
      j.kind = Json::Bool;
      j.b = true;
      return j;
    }
    if (lit("false")) {
      Json j;
      j.kind = Json::Bool;
      return j;
    }
    if (lit("null")) return Json{};
    return num();
  }
  Json str() {
    ++p;  // opening quote
    std::string s;
    while (p < end && *p != '"') {
      if ((unsigned char)*p < 0x20) return fail();
      if (*p == '\\') {
        ++p;
        if (p >= end) return fail();
        switch (*p) {
          case '"': s += '"'; break;
          case '\\': s += '\\'; break;
          case '/': s += '/'; break;
          case 'b': s += '\b'; break;
          case 'f': s += '\f'; break;
          case 'n': s += '\n'; break;
          case 'r': s += '\r'; break;
          case 't': s += '\t'; break;
          case 'u': {
            if (end - p < 5) return fail();
            unsigned cp = 0;
            for (int q = 1; q <= 4; ++q) {
              const char c = p[q];
              cp = cp * 16 + (c >= '0' && c <= '9' ? c - '0' : c >= 'a' && c <= 'f' ? c - 'a' + 10
                                                            : c >= 'A' && c <= 'F' ? c - 'A' + 10 : 99);
              if (cp > 0xffff) return fail();
            }
            p += 4;
            if (cp < 0x80) {
              s += (char)cp;
            } else if (cp < 0x800) {
              s += (char)(0xc0 | (cp >> 6));
              s += (char)(0x80 | (cp & 0x3f));
            } else {
              s += (char)(0xe0 | (cp >> 12));
              s += (char)(0x80 | ((cp >> 6) & 0x3f));
              s += (char)(0x80 | (cp & 0x3f));
            }
            break;
          }
          default: return fail();
        }
        ++p;
      } else {
        s += *p++;
      }
    }
    if (p >= end) return fail();
    ++p;
    return Json::string(std::move(s));
  }
  Json num() {
    const char* b = p;
    if (p < end && *p == '-') ++p;
    if (p >= end || !(*p >= '0' && *p <= '9')) return fail();
    if (*p == '0') ++p;
    else
      while (p < end && *p >= '0' && *p <= '9') ++p;
    bool is_float = false;
    if (p < end && *p == '.') {
      is_float = true;
      ++p;
      if (p >= end || !(*p >= '0' && *p <= '9')) return fail();
      while (p < end && *p >= '0' && *p <= '9') ++p;
    }
    if (p < end && (*p == 'e' || *p == 'E')) {
      is_float = true;
      ++p;
      if (p < end && (*p == '+' || *p == '-')) ++p;
      if (p >= end || !(*p >= '0' && *p <= '9')) return fail();
      while (p < end && *p >= '0' && *p <= '9') ++p;
    }
    if (!is_float) {
      long long v = 0;
      auto r = std::from_chars(b, p, v);
      if (r.ec == std::errc()) return Json::integer(v);
    }
    double d = 0.0;
    auto r = std::from_chars(b, p, d);
    if (r.ec != std::errc() && r.ec != std::errc::result_out_of_range) return fail();
    return Json::number(d);
  }
};

Json parse_json(const char* text, size_t n, const char* what) {
  Parser ps{text, text + n};
  Json j = ps.value(0);
  ps.ws();
  D2FT_REQUIRE(ps.ok && ps.p == ps.end, kInput, std::string(what) + ": malformed JSON");
  return j;
}

const Json& field(const Json& j, const char* name, const char* what) {
  D2FT_REQUIRE(j.kind == Json::Obj, kInput, std::string(what) + ": missing field '" + name + "'");
  auto it = j.o.find(name);
  D2FT_REQUIRE(it != j.o.end(), kInput, std::string(what) + ": missing field '" + name + "'");
  return it->second;
}

[[noreturn]] void wrong_type(const char* name, const char* what) {
  throw Fail{kInput, std::string(what) + ": field '" + name + "' has the wrong type"};
}

double as_double(const Json& v, const char* name, const char* what) {
  if (v.kind == Json::Int) return (double)v.i;
  if (v.kind == Json::Float) return v.f;
  wrong_type(name, what);
}

long long as_int(const Json& v, const char* name, const char* what) {
  if (v.kind == Json::Int) return v.i;
  if (v.kind == Json::Float) return (long long)v.f;  // nlohmann get<int>() on a float truncates
  wrong_type(name, what);
}

template <class F>
void rows_of(const Json& v, const char* name, const char* what, F&& per_row) {
  if (v.kind != Json::Arr) wrong_type(name, what);
  for (const Json& r : v.a) {
    if (r.kind != Json::Arr) wrong_type(name, what);
    per_row(r);
  }
}

const char* kMetricNames[4] = {"fisher_information", "weight_magnitude", "gradient_magnitude",
                               "taylor_importance"};  // scoring.cpp:12-20

int metric_from_name(const std::string& s) {  // scoring.cpp:22-28
  for (int m = 0; m < 4; ++m)
    if (s == kMetricNames[m]) return m;
  throw Fail{kConfig, "unknown metric: " + s};
}

const char* metric_name(int m) {
  D2FT_REQUIRE(m >= 0 && m < 4, kConfig, "unknown metric id " + std::to_string(m));
  return kMetricNames[m];
}

// copy a result string into a caller buffer: *len = bytes (without the NUL);
// kSize when cap is too small (len still set, so callers can size and retry)
void emit(const std::string& s, char* buf, size_t cap, size_t* len) {
  if (len) *len = s.size();
  D2FT_REQUIRE(buf && cap > s.size(), kSize, "output buffer too small: need " + std::to_string(s.size() + 1));
  std::memcpy(buf, s.data(), s.size());
  buf[s.size()] = '\0';
}

Json rows_json(const double* v, int K, int N) {
  Json rows = Json::array();
  for (int k = 0; k < K; ++k) {
    Json r = Json::array();
    for (int i = 0; i < N; ++i) r.a.push_back(Json::number(v[(size_t)k * N + i]));
    rows.a.push_back(std::move(r));
  }
  return rows;
}

}  // namespace
}  // namespace d2ft_b200

using namespace d2ft_b200;

extern "C" {

int d2ft_format_double(double v, char* buf, size_t cap, size_t* len) {
  return guarded([&] { emit(format_double(v), buf, cap, len); });
}

int d2ft_json_double(double v, char* buf, size_t cap, size_t* len) {
  return guarded([&] { emit(json_double(v), buf, cap, len); });
}

int d2ft_score_table_to_json(const double* fwd, const double* bwd, int K, int N, int fwd_metric, int bwd_metric,
                             char* buf, size_t cap, size_t* len) {
  return guarded([&] {
    D2FT_REQUIRE(K >= 0 && N >= 0, kInput, "score table: negative dimensions");
    Json j = Json::object();
    j.o["subnets"] = Json::integer(K);
    j.o["micro_batches"] = Json::integer(N);
    j.o["fwd_metric"] = Json::string(metric_name(fwd_metric));
    j.o["bwd_metric"] = Json::string(metric_name(bwd_metric));
    j.o["forward"] = rows_json(fwd, K, N);
    j.o["backward"] = rows_json(bwd, K, N);
    emit(dump2(j), buf, cap, len);
  });
}

int d2ft_score_table_from_json(const char* text, size_t n, int* K, int* N, int* fwd_metric, int* bwd_metric,
                               double* fwd, double* bwd, size_t cap_cells) {
  return guarded([&] {
    const char* what = "score table";
    Json j = parse_json(text, n, what);
    const int k = (int)as_int(field(j, "subnets", what), "subnets", what);
    const int nb = (int)as_int(field(j, "micro_batches", what), "micro_batches", what);
    const Json& fm = field(j, "fwd_metric", what);
    if (fm.kind != Json::Str) wrong_type("fwd_metric", what);
    const int fmi = metric_from_name(fm.s);
    const Json& bm = field(j, "bwd_metric", what);
    if (bm.kind != Json::Str) wrong_type("bwd_metric", what);
    const int bmi = metric_from_name(bm.s);
    std::vector<std::vector<double>> sides[2];
    const char* names[2] = {"forward", "backward"};
    for (int s = 0; s < 2; ++s)
      rows_of(field(j, names[s], what), names[s], what, [&](const Json& r) {
        std::vector<double> row;
        for (const Json& v : r.a) row.push_back(as_double(v, names[s], what));
        sides[s].push_back(std::move(row));
      });
    // ScoreTable::validate (scoring.cpp:30-47): forward side first
    for (int s = 0; s < 2; ++s) {
      D2FT_REQUIRE((int)sides[s].size() == k, kInput, std::string(names[s]) + " scores: row count mismatch");
      for (const auto& row : sides[s]) {
        D2FT_REQUIRE((int)row.size() == nb, kInput, std::string(names[s]) + " scores: column count mismatch");
        for (double v : row) {
          D2FT_REQUIRE(std::isfinite(v), kNumeric, "score table contains non-finite entries");
          D2FT_REQUIRE(v >= 0.0, kNumeric, "score table contains negative entries");
        }
      }
    }
    *K = k;
    *N = nb;
    *fwd_metric = fmi;
    *bwd_metric = bmi;
    D2FT_REQUIRE(fwd && bwd && cap_cells >= (size_t)k * nb, kSize, "score table: output buffers too small");
    for (int r = 0; r < k; ++r)
      for (int i = 0; i < nb; ++i) {
        fwd[(size_t)r * nb + i] = sides[0][r][i];
        bwd[(size_t)r * nb + i] = sides[1][r][i];
      }
  });
}

int d2ft_score_table_to_csv(const double* fwd, const double* bwd, int K, int N, char* buf, size_t cap, size_t* len) {
  return guarded([&] {
    std::string out = "subnet_id,micro_batch,fwd,bwd\n";
    for (int k = 0; k < K; ++k)
      for (int i = 0; i < N; ++i)
        out += std::to_string(k) + "," + std::to_string(i) + "," + format_double(fwd[(size_t)k * N + i]) + "," +
               format_double(bwd[(size_t)k * N + i]) + "\n";
    emit(out, buf, cap, len);
  });
}

int d2ft_schedule_table_to_json(const uint8_t* codes, int K, int N, char* buf, size_t cap, size_t* len) {
  return guarded([&] {
    D2FT_REQUIRE(K >= 0 && N >= 0, kInput, "schedule table: dimension mismatch");
    Json rows = Json::array();
    for (int k = 0; k < K; ++k) {
      Json r = Json::array();
      for (int i = 0; i < N; ++i) r.a.push_back(Json::integer(codes[(size_t)k * N + i]));
      rows.a.push_back(std::move(r));
    }
    Json j = Json::object();
    j.o["devices"] = Json::integer(K);
    j.o["micro_batches"] = Json::integer(N);
    j.o["codes"] = std::move(rows);
    emit(dump2(j), buf, cap, len);
  });
}

int d2ft_schedule_table_from_json(const char* text, size_t n, int* K, int* N, uint8_t* codes, size_t cap_cells) {
  return guarded([&] {
    const char* what = "schedule table";
    Json j = parse_json(text, n, what);
    const int k = (int)as_int(field(j, "devices", what), "devices", what);
    const int nb = (int)as_int(field(j, "micro_batches", what), "micro_batches", what);
    std::vector<std::vector<long long>> rows;
    rows_of(field(j, "codes", what), "codes", what, [&](const Json& r) {
      std::vector<long long> row;
      for (const Json& v : r.a) row.push_back(as_int(v, "codes", what));
      rows.push_back(std::move(row));
    });
    D2FT_REQUIRE((int)rows.size() == k, kInput, "schedule table: codes row count mismatch");
    D2FT_REQUIRE(k >= 0 && nb >= 0, kInput, "schedule table: dimension mismatch");
    for (const auto& row : rows) {
      D2FT_REQUIRE((int)row.size() == nb, kInput, "schedule table: codes column count mismatch");
      for (long long c : row) D2FT_REQUIRE(c >= 1 && c <= 3, kInput, "schedule table: code out of range");
    }
    *K = k;
    *N = nb;
    D2FT_REQUIRE(codes && cap_cells >= (size_t)k * nb, kSize, "schedule table: output buffer too small");
    for (int r = 0; r < k; ++r)
      for (int i = 0; i < nb; ++i) codes[(size_t)r * nb + i] = (uint8_t)rows[r][i];
  });
}

int d2ft_schedule_table_to_csv(const uint8_t* codes, int K, int N, char* buf, size_t cap, size_t* len) {
  return guarded([&] {
    std::string out = "subnet_id,micro_batch,code\n";
    for (int k = 0; k < K; ++k)
      for (int i = 0; i < N; ++i)
        out += std::to_string(k) + "," + std::to_string(i) + "," + std::to_string((int)codes[(size_t)k * N + i]) +
               "\n";
    emit(out, buf, cap, len);
  });
}

int d2ft_batch_metrics_to_json(const d2ft_batch_metrics* m, const double* per_device_busy_ms, int n_dev,
                               const char* run_id, const char* method, char* buf, size_t cap, size_t* len) {
  return guarded([&] {
    Json j = Json::object();
    j.o["run_id"] = Json::string(run_id ? run_id : "");
    j.o["method"] = Json::string(method ? method : "");
    j.o["compute_fraction"] = Json::number(m->compute_fraction);
    j.o["comm_fraction"] = Json::number(m->comm_fraction);
    j.o["workload_variance"] = Json::number(m->workload_variance);
    j.o["makespan_ms"] = Json::number(m->makespan_ms);
    Json busy = Json::array();
    for (int p = 0; p < n_dev; ++p) busy.a.push_back(Json::number(per_device_busy_ms[p]));
    j.o["per_device_busy_ms"] = std::move(busy);
    j.o["imbalance_residual"] = Json::number(m->imbalance_residual);
    emit(dump2(j), buf, cap, len);
  });
}

int d2ft_batch_metrics_csv_header(char* buf, size_t cap, size_t* len) {
  return guarded([&] {
    emit("run_id,method,compute_fraction,comm_fraction,workload_variance,makespan_ms,imbalance_residual\n", buf, cap,
         len);
  });
}

int d2ft_batch_metrics_to_csv_row(const d2ft_batch_metrics* m, const char* run_id, const char* method, char* buf,
                                  size_t cap, size_t* len) {
  return guarded([&] {
    emit(std::string(run_id ? run_id : "") + "," + (method ? method : "") + "," + format_double(m->compute_fraction) +
             "," + format_double(m->comm_fraction) + "," + format_double(m->workload_variance) + "," +
             format_double(m->makespan_ms) + "," + format_double(m->imbalance_residual) + "\n",
         buf, cap, len);
  });
}

int d2ft_history_to_csv(const int32_t* epoch, const double* loss, const double* top1, const double* compute_fraction,
                        const double* comm_fraction, int n, char* buf, size_t cap, size_t* len) {
  return guarded([&] {
    std::string out = "epoch,loss,top1,compute_fraction,comm_fraction\n";
    for (int r = 0; r < n; ++r)
      out += std::to_string(epoch[r]) + "," + format_double(loss[r]) + "," + format_double(top1[r]) + "," +
             format_double(compute_fraction[r]) + "," + format_double(comm_fraction[r]) + "\n";
    emit(out, buf, cap, len);
  });
}

int d2ft_history_to_json(const int32_t* epoch, const double* loss, const double* top1, const double* compute_fraction,
                         const double* comm_fraction, int n, char* buf, size_t cap, size_t* len) {
  return guarded([&] {
    Json epochs = Json::array();
    for (int r = 0; r < n; ++r) {
      Json e = Json::object();
      e.o["epoch"] = Json::integer(epoch[r]);
      e.o["loss"] = Json::number(loss[r]);
      e.o["top1"] = Json::number(top1[r]);
      e.o["compute_fraction"] = Json::number(compute_fraction[r]);
      e.o["comm_fraction"] = Json::number(comm_fraction[r]);
      epochs.a.push_back(std::move(e));
    }
    Json j = Json::object();
    j.o["epochs"] = std::move(epochs);
    emit(dump2(j), buf, cap, len);
  });
}

// history_from_csv (serialize.cpp:200-222): header skipped, empty lines
// skipped, five fields per row.  *n = rows parsed; kSize if cap < rows.
int d2ft_history_from_csv(const char* text, size_t n_text, int32_t* epoch, double* loss, double* top1,
                          double* compute_fraction, double* comm_fraction, int cap, int* n) {
  return guarded([&] {
    std::istringstream in(std::string(text, n_text));
    std::string line;
    D2FT_REQUIRE((bool)std::getline(in, line), kInput, "history csv: empty file");
    std::vector<std::array<double, 5>> rows;
    while (std::getline(in, line)) {
      if (line.empty()) continue;
      std::istringstream ls(line);
      std::string f;
      std::array<double, 5> r{};
      for (int c = 0; c < 5; ++c) {
        D2FT_REQUIRE((bool)std::getline(ls, f, ','), kInput, "history csv: short row");
        try {
          r[c] = c == 0 ? (double)std::stoi(f) : std::stod(f);
        } catch (const std::exception&) {
          throw Fail{kInput, "history csv: bad field '" + f + "'"};
        }
      }
      rows.push_back(r);
    }
    *n = (int)rows.size();
    D2FT_REQUIRE(cap >= *n, kSize, "history csv: output buffers too small");
    for (int r = 0; r < *n; ++r) {
      epoch[r] = (int32_t)rows[r][0];
      loss[r] = rows[r][1];
      top1[r] = rows[r][2];
      compute_fraction[r] = rows[r][3];
      comm_fraction[r] = rows[r][4];
    }
  });
}

// atomic_write_file / read_file (serialize.cpp:23-42): temp file + rename
int d2ft_atomic_write_file(const char* path, const char* data, size_t n) {
  return guarded([&] {
    const std::string tmp = std::string(path) + ".tmp";
    {
      std::ofstream out(tmp, std::ios::binary | std::ios::trunc);
      D2FT_REQUIRE((bool)out, kInput, "cannot open for writing: " + tmp);
      out.write(data, (std::streamsize)n);
      D2FT_REQUIRE((bool)out, kInput, "write failed: " + tmp);
    }
    D2FT_REQUIRE(std::rename(tmp.c_str(), path) == 0, kInput, std::string("cannot move into place: ") + path);
  });
}

int d2ft_read_file(const char* path, char* buf, size_t cap, size_t* len) {
  return guarded([&] {
    std::ifstream in(path, std::ios::binary);
    D2FT_REQUIRE((bool)in, kInput, std::string("cannot open: ") + path);
    std::ostringstream ss;
    ss << in.rdbuf();
    emit(ss.str(), buf, cap, len);
  });
}

}  // extern "C"
