// tpmg_io.cpp -- profile files of the reference (profile_io.hpp:125-242) for the Cartesian
// grids of this library: the same JSON layout (format_version 1, kind "factorized" / "full",
// grid header with level, n_r and a 64-bit FNV-1a fingerprint of the cell centres, arrays in
// the reference's Matrix order -- column-major, k fastest -- as decimal numbers or as
// base64 little-endian doubles), validated on load like load_profiles: fingerprint, every
// array's length, finiteness; errors map onto the reference's taxonomy (types.hpp:24-58).
// The grid header's "type" is "cartesian" (the reference writes "icosahedral"); the
// fingerprint mixes the cell centres (x, y, 0) = ((i+1/2) hx, (j+1/2) hy, 0) in cell order
// j*nx + i exactly as grid_fingerprint (geometry.hpp:337-351) mixes the sphere's centres.
// Host code only; nothing here touches the device.
#include "tpmg_b200.h"

#include <algorithm>
#include <cctype>
#include <cmath>
#include <cstdint>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <fstream>
#include <map>
#include <memory>
#include <sstream>
#include <stdexcept>
#include <string>
#include <vector>

namespace {

struct IoError : std::runtime_error {
  int code;
  IoError(int c, const std::string& w) : std::runtime_error(w), code(c) {}
};

thread_local std::string g_io_error;

// ---- a small JSON value and parser (objects, arrays, strings, numbers, literals) -----------
struct Json {
  enum Kind { Null, Bool, Number, String, Array, Object } kind = Null;
  double num = 0.0;
  bool flag = false;
  std::string str;
  std::vector<Json> arr;
  std::map<std::string, Json> obj;
  const Json* get(const std::string& k) const {
    auto it = obj.find(k);
    return it == obj.end() ? nullptr : &it->second;
  }
};

struct Parser {
  const std::string& s;
  size_t i = 0;
  explicit Parser(const std::string& src) : s(src) {}
  [[noreturn]] void fail(const char* what) {
    throw IoError(TPMG_E_SHAPE, std::string("profile file: malformed JSON (") + what + ")");
  }
  void ws() {
    while (i < s.size() && std::isspace((unsigned char)s[i])) ++i;
  }
  Json value() {
    ws();
    if (i >= s.size()) fail("unexpected end");
    const char c = s[i];
    if (c == '{') return object();
    if (c == '[') return array();
    if (c == '"') {
      Json j;
      j.kind = Json::String;
      j.str = string();
      return j;
    }
    if (c == 't' || c == 'f' || c == 'n') return literal();
    return number();
  }
  std::string string() {
    if (s[i] != '"') fail("string expected");
    ++i;
    std::string out;
    while (i < s.size() && s[i] != '"') {
      if (s[i] == '\\') {
        if (++i >= s.size()) fail("bad escape");
        const char e = s[i];
        if (e == 'n') out.push_back('\n');
        else if (e == 't') out.push_back('\t');
        else if (e == 'r') out.push_back('\r');
        else if (e == 'u') {  // ASCII subset only
          if (i + 4 >= s.size()) fail("bad unicode escape");
          out.push_back((char)std::strtol(s.substr(i + 1, 4).c_str(), nullptr, 16));
          i += 4;
        } else out.push_back(e);
        ++i;
      } else {
        out.push_back(s[i++]);
      }
    }
    if (i >= s.size()) fail("unterminated string");
    ++i;
    return out;
  }
  Json number() {
    // JSON grammar only: -?digits[.digits][(e|E)[+-]digits]; NaN / Infinity / hex are malformed
    // (nlohmann rejects them too), as is a value that overflows a double
    size_t k = i;
    if (k < s.size() && s[k] == '-') ++k;
    const size_t d0 = k;
    while (k < s.size() && std::isdigit((unsigned char)s[k])) ++k;
    if (k == d0) fail("number expected");
    if (k < s.size() && s[k] == '.') {
      const size_t f0 = ++k;
      while (k < s.size() && std::isdigit((unsigned char)s[k])) ++k;
      if (k == f0) fail("digits expected after '.'");
    }
    if (k < s.size() && (s[k] == 'e' || s[k] == 'E')) {
      ++k;
      if (k < s.size() && (s[k] == '+' || s[k] == '-')) ++k;
      const size_t e0 = k;
      while (k < s.size() && std::isdigit((unsigned char)s[k])) ++k;
      if (k == e0) fail("exponent digits expected");
    }
    const std::string tok = s.substr(i, k - i);
    const double v = std::strtod(tok.c_str(), nullptr);  // correctly rounded: exact round trip
    if (!std::isfinite(v)) fail("number overflow");
    i = k;
    Json j;
    j.kind = Json::Number;
    j.num = v;
    return j;
  }
  Json literal() {
    Json j;
    if (s.compare(i, 4, "true") == 0) { j.kind = Json::Bool; j.flag = true; i += 4; }
    else if (s.compare(i, 5, "false") == 0) { j.kind = Json::Bool; i += 5; }
    else if (s.compare(i, 4, "null") == 0) { i += 4; }
    else fail("bad literal");
    return j;
  }
  Json array() {
    Json j;
    j.kind = Json::Array;
    ++i;
    ws();
    if (i < s.size() && s[i] == ']') { ++i; return j; }
    for (;;) {
      j.arr.push_back(value());
      ws();
      if (i < s.size() && s[i] == ',') { ++i; continue; }
      if (i < s.size() && s[i] == ']') { ++i; return j; }
      fail("',' or ']' expected");
    }
  }
  Json object() {
    Json j;
    j.kind = Json::Object;
    ++i;
    ws();
    if (i < s.size() && s[i] == '}') { ++i; return j; }
    for (;;) {
      ws();
      const std::string k = string();
      ws();
      if (i >= s.size() || s[i] != ':') fail("':' expected");
      ++i;
      j.obj[k] = value();
      ws();
      if (i < s.size() && s[i] == ',') { ++i; continue; }
      if (i < s.size() && s[i] == '}') { ++i; return j; }
      fail("',' or '}' expected");
    }
  }
};

// ---- base64 of little-endian doubles (profile_io.hpp:33-78) --------------------------------
constexpr char kB64[] = "ABCDEFGHIJKLMNOPQRSTUVWXYZabcdefghijklmnopqrstuvwxyz0123456789+/";

std::string b64_encode(const double* data, size_t count) {
  const auto* bytes = reinterpret_cast<const unsigned char*>(data);
  const size_t n = count * sizeof(double);
  std::string out;
  out.reserve((n + 2) / 3 * 4);
  for (size_t i = 0; i < n; i += 3) {
    unsigned v = (unsigned)bytes[i] << 16;
    if (i + 1 < n) v |= (unsigned)bytes[i + 1] << 8;
    if (i + 2 < n) v |= bytes[i + 2];
    out.push_back(kB64[(v >> 18) & 63]);
    out.push_back(kB64[(v >> 12) & 63]);
    out.push_back(i + 1 < n ? kB64[(v >> 6) & 63] : '=');
    out.push_back(i + 2 < n ? kB64[v & 63] : '=');
  }
  return out;
}

std::vector<double> b64_decode(const std::string& s) {
  int rev[256];
  for (int& r : rev) r = -1;
  for (int i = 0; i < 64; ++i) rev[(unsigned char)kB64[i]] = i;
  std::vector<unsigned char> bytes;
  unsigned acc = 0;
  int bits = 0;
  for (char ch : s) {
    if (ch == '=' || ch == '\n' || ch == '\r') continue;
    const int v = rev[(unsigned char)ch];
    if (v < 0) throw IoError(TPMG_E_SHAPE, "profile file: invalid base64 payload");
    acc = (acc << 6) | (unsigned)v;
    bits += 6;
    if (bits >= 8) {
      bits -= 8;
      bytes.push_back((unsigned char)((acc >> bits) & 0xff));
    }
  }
  if (bytes.size() % sizeof(double) != 0)
    throw IoError(TPMG_E_SHAPE, "profile file: base64 payload is not a multiple of 8 bytes");
  std::vector<double> out(bytes.size() / sizeof(double));
  std::memcpy(out.data(), bytes.data(), bytes.size());
  return out;
}

// ---- grid fingerprint (geometry.hpp:337-351 over the Cartesian cell centres) ---------------
uint64_t fingerprint_cart(int64_t nx, int64_t ny, double hx, double hy) {
  uint64_t h = 0xcbf29ce484222325ull;
  auto mix = [&h](double x) {
    uint64_t bits;
    std::memcpy(&bits, &x, sizeof bits);
    for (int i = 0; i < 8; ++i) {
      h ^= (bits >> (8 * i)) & 0xffull;
      h *= 0x100000001b3ull;
    }
  };
  for (int64_t j = 0; j < ny; ++j)
    for (int64_t i = 0; i < nx; ++i) {
      mix(((double)i + 0.5) * hx);
      mix(((double)j + 0.5) * hy);
      mix(0.0);
    }
  return h;
}

// names and lengths of the arrays of a kind, in the C-ABI's packed order
struct Arr {
  const char* name;
  int64_t len;
};
std::vector<Arr> layout(int kind, int64_t nc, int64_t ne, int64_t nz) {
  if (kind == TPMG_PROFILE_FACTORIZED)
    return {{"beta_r", nz}, {"alpha_s_r", nz}, {"alpha_r_r", nz + 1}, {"xi_r_r", nz + 1},
            {"beta_s", nc}, {"alpha_r_s", nc}, {"xi_r_s", nc}, {"alpha_s_s", ne}};
  return {{"beta", nz * nc}, {"alpha_s", nz * ne}, {"alpha_r", (nz + 1) * nc},
          {"xi_r", (nz + 1) * nc}};
}

std::string hex16(uint64_t h) {
  char buf[17];
  std::snprintf(buf, sizeof buf, "%016llx", (unsigned long long)h);
  return buf;
}

tpmg_profile_grid cartesian_grid(const tpmg_grid_desc* g) {
  tpmg_profile_grid pg{};
  pg.type = "cartesian";
  pg.fingerprint = 0;
  pg.level = 0;
  if (!g) return pg;
  pg.n_r = g->nz;
  pg.n_cells = g->nx * g->ny;
  pg.n_edges = 2 * g->nx * g->ny;
  pg.nx = g->nx;
  pg.ny = g->ny;
  return pg;
}

// ---- Grisu2 (F. Loitsch, "Printing floating-point numbers quickly and accurately with
// integers", PLDI 2010) as the reference's JSON writer (nlohmann::json dump_float -> to_chars)
// applies it: boundaries m-/m+, one cached power 10^-k bringing the exponent into [-60, -32],
// digits of the narrowed upper bound, then the closest-to-v rounding step.  Not always the
// shortest representation, which is why it is restated here instead of using "%.17g": the
// written bytes must equal the reference's.  The cached powers are the correctly rounded 64-bit
// significands of 10^k, k = -300, -292, ..., 324 (generated with exact rational arithmetic).
//
// Attribution: the structure of this block -- the cached-power index formula, the four-partial
// 64x64 multiply with half-up rounding, and grisu2_round's loop condition -- follows
// nlohmann::json's dtoa_impl (https://github.com/nlohmann/json, MIT License, Copyright (c)
// 2013-2022 Niels Lohmann), itself an implementation of Florian Loitsch's Grisu2 (reference
// implementation under the MIT/BSD-style licence of the paper's code).  Byte-identical output
// with the reference's writer requires the same algorithm; the MIT licence terms apply to the
// parts that follow it.
namespace grisu {

struct Fp {
  uint64_t f;
  int e;
};

Fp sub(Fp x, Fp y) { return {x.f - y.f, x.e}; }

Fp mul(Fp x, Fp y) {  // upper 64 bits of the 128-bit product, rounded half up
  const uint64_t ul = x.f & 0xffffffffu, uh = x.f >> 32, vl = y.f & 0xffffffffu, vh = y.f >> 32;
  const uint64_t p0 = ul * vl, p1 = ul * vh, p2 = uh * vl, p3 = uh * vh;
  uint64_t q = (p0 >> 32) + (p1 & 0xffffffffu) + (p2 & 0xffffffffu);
  q += uint64_t{1} << 31;
  return {p3 + (p2 >> 32) + (p1 >> 32) + (q >> 32), x.e + y.e + 64};
}

Fp normalize(Fp x) {
  while ((x.f >> 63) == 0) {
    x.f <<= 1;
    x.e--;
  }
  return x;
}

struct Cached {
  uint64_t f;
  int e, k;
};

const Cached kPowers[] = {
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
    {0x9E19DB92B4E31BA9ull, 1013, 324}};

Cached cached_power(int e) {  // 10^-k with -60 <= e_c + e + 64 <= -32
  const int f = -60 - e - 1;
  const int k = (f * 78913) / (1 << 18) + (f > 0 ? 1 : 0);
  const int index = (300 + k + 7) / 8;
  return kPowers[index];
}

int largest_pow10(uint32_t n, uint32_t& pow10) {
  uint32_t p = 1000000000u;
  for (int d = 10; d > 1; --d, p /= 10)
    if (n >= p) {
      pow10 = p;
      return d;
    }
  pow10 = 1;
  return 1;
}

void round_last(std::string& buf, uint64_t dist, uint64_t delta, uint64_t rest, uint64_t ten_k) {
  while (rest < dist && delta - rest >= ten_k &&
         (rest + ten_k < dist || dist - rest > rest + ten_k - dist)) {
    buf.back()--;
    rest += ten_k;
  }
}

// digits of a positive finite double and the decimal exponent of their last digit
void digits(double value, std::string& buf, int& dec_exp) {
  uint64_t bits;
  std::memcpy(&bits, &value, 8);
  const uint64_t E = bits >> 52, F = bits & ((uint64_t{1} << 52) - 1);
  const Fp v = E == 0 ? Fp{F, 1 - 1075} : Fp{F + (uint64_t{1} << 52), (int)E - 1075};
  const bool lower_closer = F == 0 && E > 1;
  const Fp mp = {2 * v.f + 1, v.e - 1};
  const Fp mm = lower_closer ? Fp{4 * v.f - 1, v.e - 2} : Fp{2 * v.f - 1, v.e - 1};
  const Fp wp = normalize(mp);
  const Fp wm = {mm.f << (mm.e - wp.e), wp.e};
  const Fp w = normalize(v);

  const Cached c = cached_power(wp.e);
  const Fp ck = {c.f, c.e};
  const Fp ww = mul(w, ck), wlo = mul(wm, ck), whi = mul(wp, ck);
  const Fp Mm = {wlo.f + 1, wlo.e}, Mp = {whi.f - 1, whi.e};
  dec_exp = -c.k;

  uint64_t delta = sub(Mp, Mm).f, dist = sub(Mp, ww).f;
  const Fp one = {uint64_t{1} << -Mp.e, Mp.e};
  uint32_t p1 = (uint32_t)(Mp.f >> -one.e);
  uint64_t p2 = Mp.f & (one.f - 1);
  uint32_t pow10;
  int n = largest_pow10(p1, pow10);
  while (n > 0) {
    const uint32_t d = p1 / pow10, r = p1 % pow10;
    buf.push_back((char)('0' + d));
    p1 = r;
    n--;
    const uint64_t rest = ((uint64_t)p1 << -one.e) + p2;
    if (rest <= delta) {
      dec_exp += n;
      round_last(buf, dist, delta, rest, (uint64_t)pow10 << -one.e);
      return;
    }
    pow10 /= 10;
  }
  int m = 0;
  for (;;) {
    p2 *= 10;
    delta *= 10;
    dist *= 10;
    buf.push_back((char)('0' + (p2 >> -one.e)));
    p2 &= one.f - 1;
    m++;
    if (p2 <= delta) break;
  }
  dec_exp -= m;
  round_last(buf, dist, delta, p2, one.f);
}

}  // namespace grisu

// nlohmann's dump of a double (serializer::dump_float -> to_chars): the Grisu2 digits, written as "ddd.0" / "d.dd" / "0.000dd" for decimal exponents in (-4, 15],
// else "d.dde+XX" with at least two exponent digits; non-finite values become null
void put_double(std::string& out, double v) {
  if (!std::isfinite(v)) {
    out += "null";
    return;
  }
  if (v == 0.0) {
    out += std::signbit(v) ? "-0.0" : "0.0";
    return;
  }
  if (v < 0) {
    out += '-';
    v = -v;
  }
  std::string digits;
  int dec_exp = 0;
  grisu::digits(v, digits, dec_exp);
  const int k = (int)digits.size();
  const int n = k + dec_exp;  // position of the decimal point relative to the digits
  if (k <= n && n <= 15) {
    out += digits;
    out.append((size_t)(n - k), '0');
    out += ".0";
  } else if (0 < n && n <= 15) {
    out += digits.substr(0, (size_t)n);
    out += '.';
    out += digits.substr((size_t)n);
  } else if (-4 < n && n <= 0) {
    out += "0.";
    out.append((size_t)(-n), '0');
    out += digits;
  } else {
    out += digits[0];
    if (k > 1) {
      out += '.';
      out += digits.substr(1);
    }
    char eb[16];
    const int ex = n - 1;
    std::snprintf(eb, sizeof eb, "e%c%02d", ex < 0 ? '-' : '+', ex < 0 ? -ex : ex);
    out += eb;
  }
}

// the reference writes j.dump(1): keys sorted (std::map), one space per level, one array
// element per line
void write_array(std::string& out, const Arr& a, const double* v, bool base64) {
  out += "  \"";
  out += a.name;
  out += "\": ";
  if (base64) {
    out += "\"" + b64_encode(v, (size_t)a.len) + "\"";
    return;
  }
  if (a.len == 0) {
    out += "[]";
    return;
  }
  out += "[\n";
  for (int64_t i = 0; i < a.len; ++i) {
    out += "   ";
    put_double(out, v[i]);
    out += i + 1 < a.len ? ",\n" : "\n";
  }
  out += "  ]";
}

template <typename Fn>
int io_guard(Fn&& fn) {
  try {
    fn();
    return TPMG_OK;
  } catch (const IoError& e) {
    g_io_error = e.what();
    return e.code;
  } catch (const std::exception& e) {
    g_io_error = e.what();
    return TPMG_E_CONFIG;
  }
}


int64_t packed_size(int kind, int64_t nc, int64_t ne, int64_t nz) {
  int64_t n = 0;
  for (const Arr& a : layout(kind, nc, ne, nz)) n += a.len;
  return n;
}

void check_grid(const tpmg_profile_grid* g) {
  if (!g || !g->type || g->n_r < 1 || g->n_cells < 1 || g->n_edges < 0)
    throw IoError(TPMG_E_CONFIG, "profile grid: bad description");
}

void save_impl(const char* path, const tpmg_profile_grid* g, int kind, const double* packed,
               int base64) {
  check_grid(g);
  if (!path || !packed) throw IoError(TPMG_E_CONFIG, "profile_save: bad arguments");
  if (kind != TPMG_PROFILE_FACTORIZED && kind != TPMG_PROFILE_FULL)
    throw IoError(TPMG_E_CONFIG, "profile_save: unknown kind");
  const std::vector<Arr> arrs = layout(kind, g->n_cells, g->n_edges, g->n_r);
  std::vector<const double*> at(arrs.size());
  const double* p = packed;
  for (size_t a = 0; a < arrs.size(); ++a) {
    at[a] = p;
    p += arrs[a].len;
  }
  std::vector<size_t> order(arrs.size());
  for (size_t a = 0; a < order.size(); ++a) order[a] = a;
  std::sort(order.begin(), order.end(),
            [&](size_t x, size_t y) { return std::strcmp(arrs[x].name, arrs[y].name) < 0; });
  std::string out = "{\n \"arrays\": {\n";
  for (size_t n = 0; n < order.size(); ++n) {
    write_array(out, arrs[order[n]], at[order[n]], base64 != 0);
    out += n + 1 < order.size() ? ",\n" : "\n";
  }
  out += " },\n";
  if (base64) out += " \"encoding\": \"base64-f64le\",\n";
  out += " \"format_version\": 1,\n \"grid\": {\n  \"fingerprint\": \"" + hex16(g->fingerprint) +
         "\",\n  \"level\": " + std::to_string(g->level) + ",\n  \"n_r\": " +
         std::to_string(g->n_r) + ",\n";
  if (g->nx > 0) out += "  \"nx\": " + std::to_string(g->nx) + ",\n";
  if (g->ny > 0) out += "  \"ny\": " + std::to_string(g->ny) + ",\n";
  out += "  \"type\": \"" + std::string(g->type) + "\"\n },\n \"kind\": \"" +
         (kind == TPMG_PROFILE_FULL ? "full" : "factorized") +
         "\",\n \"layout\": \"column-major, k fastest\"\n}\n";
  std::ofstream f(path);
  if (!f) throw IoError(TPMG_E_CONFIG, std::string("cannot write profile file: ") + path);
  f << out;
  if (!f) throw IoError(TPMG_E_CONFIG, std::string("cannot write profile file: ") + path);
}

// load_profiles, profile_io.hpp:168-242: the same checks in the same order
void load_impl(const char* path, const tpmg_profile_grid* g, int* kind, double* packed,
               int64_t capacity) {
  check_grid(g);
  if (!path || !kind || !packed) throw IoError(TPMG_E_CONFIG, "profile_load: bad arguments");
  std::ifstream f(path);
  if (!f) throw IoError(TPMG_E_CONFIG, std::string("cannot read profile file: ") + path);
  std::stringstream ss;
  ss << f.rdbuf();
  const std::string text = ss.str();
  Parser ps(text);
  const Json j = ps.value();  // like `is >> j`: content after the first value is ignored
  const Json* gj = j.get("grid");
  const Json* arrays = j.get("arrays");
  const Json* kd = j.get("kind");
  if (j.kind != Json::Object || !gj || !arrays || !kd)
    throw IoError(TPMG_E_SHAPE, "profile file: missing required fields");
  const Json* fp = gj->get("fingerprint");
  const std::string fps = fp && fp->kind == Json::String ? fp->str : "";
  if (fps != hex16(g->fingerprint))
    throw IoError(TPMG_E_FINGERPRINT,
                  "profile file written for a different grid (fingerprint " + fps + ")");
  const Json* nr = gj->get("n_r");
  const int64_t n_r = nr && nr->kind == Json::Number ? (int64_t)nr->num : -1;
  if (n_r != g->n_r)
    throw IoError(TPMG_E_SHAPE, "profile file: n_r = " + std::to_string(n_r) +
                                    ", active grid has " + std::to_string(g->n_r));
  const Json* lv = gj->get("level");
  if (!lv || lv->kind != Json::Number || (int64_t)lv->num != g->level)
    throw IoError(TPMG_E_SHAPE, "profile file: level mismatch");
  const Json* enc = j.get("encoding");
  const bool b64 = enc && enc->kind == Json::String && enc->str == "base64-f64le";
  if (kd->kind != Json::String) throw IoError(TPMG_E_SHAPE, "profile file: kind is not a string");
  int k;
  if (kd->str == "full") k = TPMG_PROFILE_FULL;
  else if (kd->str == "factorized") k = TPMG_PROFILE_FACTORIZED;
  else throw IoError(TPMG_E_SHAPE, "profile file: unknown kind '" + kd->str + "'");
  if (packed_size(k, g->n_cells, g->n_edges, g->n_r) > capacity)
    throw IoError(TPMG_E_CAP, "profile_load: output buffer too small");
  double* p = packed;
  for (const Arr& a : layout(k, g->n_cells, g->n_edges, g->n_r)) {
    const Json* node = arrays->kind == Json::Object ? arrays->get(a.name) : nullptr;
    std::vector<double> v;
    const std::string name = a.name;
    if (b64) {
      if (!node || node->kind != Json::String)
        throw IoError(TPMG_E_SHAPE, "profile file: array '" + name + "' not base64");
      v = b64_decode(node->str);
    } else {
      if (!node || node->kind != Json::Array)
        throw IoError(TPMG_E_SHAPE, "profile file: array '" + name + "' missing");
      v.reserve(node->arr.size());
      for (const Json& x : node->arr) {
        if (x.kind != Json::Number)
          throw IoError(TPMG_E_NONFINITE, "profile file: non-numeric entry in '" + name + "'");
        v.push_back(x.num);
      }
    }
    if ((int64_t)v.size() != a.len)
      throw IoError(TPMG_E_SHAPE, "profile file: array '" + name + "' has " +
                                      std::to_string(v.size()) + " entries, expected " +
                                      std::to_string(a.len));
    for (double x : v)
      if (!std::isfinite(x))
        throw IoError(TPMG_E_NONFINITE, "profile file: non-finite value in '" + name + "'");
    std::memcpy(p, v.data(), v.size() * sizeof(double));
    p += a.len;
  }
  *kind = k;
}

}  // namespace

extern "C" {

const char* tpmg_profile_last_error(void) { return g_io_error.c_str(); }

uint64_t tpmg_grid_fingerprint(const double* centers, int64_t n_cells) {
  uint64_t h = 0xcbf29ce484222325ull;
  for (int64_t i = 0; i < 3 * n_cells; ++i) {
    uint64_t bits;
    std::memcpy(&bits, centers + i, sizeof bits);
    for (int b = 0; b < 8; ++b) {
      h ^= (bits >> (8 * b)) & 0xffull;
      h *= 0x100000001b3ull;
    }
  }
  return h;
}

uint64_t tpmg_grid_fingerprint_cartesian(const tpmg_grid_desc* grid) {
  return grid ? fingerprint_cart(grid->nx, grid->ny, grid->hx, grid->hy) : 0;
}

int64_t tpmg_profile_packed_size(int kind, int64_t n_cells, int64_t n_edges, int64_t n_r) {
  return packed_size(kind, n_cells, n_edges, n_r);
}

int tpmg_profile_save(const char* path, const tpmg_grid_desc* grid, int kind, const double* packed,
                      int base64) {
  return io_guard([&] {
    tpmg_profile_grid pg = cartesian_grid(grid);
    if (grid) pg.fingerprint = fingerprint_cart(grid->nx, grid->ny, grid->hx, grid->hy);
    save_impl(path, &pg, kind, packed, base64);
  });
}

int tpmg_profile_load(const char* path, const tpmg_grid_desc* grid, int* kind, double* packed,
                      int64_t capacity) {
  return io_guard([&] {
    tpmg_profile_grid pg = cartesian_grid(grid);
    if (grid) pg.fingerprint = fingerprint_cart(grid->nx, grid->ny, grid->hx, grid->hy);
    load_impl(path, &pg, kind, packed, capacity);
  });
}

int tpmg_profile_save_grid(const char* path, const tpmg_profile_grid* grid, int kind,
                           const double* packed, int base64) {
  return io_guard([&] { save_impl(path, grid, kind, packed, base64); });
}

int tpmg_profile_load_grid(const char* path, const tpmg_profile_grid* grid, int* kind,
                           double* packed, int64_t capacity) {
  return io_guard([&] { load_impl(path, grid, kind, packed, capacity); });
}

}  // extern "C"
