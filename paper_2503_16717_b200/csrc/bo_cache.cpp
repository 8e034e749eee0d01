// bo_cache.cpp — the raw FP64 panel cache for C2 inputs (SURVEY.md §8(f)2,
// §8(d) C2: "generate once and cache as raw FP64 + SHA-256").
//
// File layout (little endian):
//   bytes  0..7    magic "BOPC0001"
//   bytes  8..15   rows  (uint64)
//   bytes 16..23   cols  (uint64)
//   bytes 24..55   SHA-256 of the payload
//   bytes 56..311  generator description (NUL-padded text, e.g.
//                  "gen_glued(8000000, 6, 11, 100, 100, 7)")
//   bytes 312..    payload: rows x cols doubles, column-major, ld = rows
// Reading verifies the digest, so a bench or test that consumes a cache knows
// it holds exactly the bytes the reference generator produced.
#include <algorithm>
#include <cstdint>
#include <cstdio>
#include <cstring>
#include <string>
#include <vector>

#include "../../include/bo_cuda.h"

namespace {

constexpr char kMagic[8] = {'B', 'O', 'P', 'C', '0', '0', '0', '1'};
constexpr size_t kHeader = 312, kDescLen = 256;

int fail(bo_status* st, int code, const std::string& msg) {
  if (st) {
    st->code = code;
    st->index = 0;
    st->pivot = 0.0;
    std::snprintf(st->msg, sizeof st->msg, "%s", msg.c_str());
  }
  return code;
}
void ok(bo_status* st) {
  if (st) {
    st->code = 0;
    st->index = 0;
    st->pivot = 0.0;
    st->msg[0] = 0;
  }
}

// SHA-256 (FIPS 180-4), streaming
struct Sha256 {
  uint32_t h[8] = {0x6a09e667u, 0xbb67ae85u, 0x3c6ef372u, 0xa54ff53au,
                   0x510e527fu, 0x9b05688cu, 0x1f83d9abu, 0x5be0cd19u};
  unsigned char buf[64];
  size_t fill = 0;
  uint64_t bits = 0;
  static uint32_t rotr(uint32_t x, int n) { return (x >> n) | (x << (32 - n)); }
  void block(const unsigned char* p) {
    static const uint32_t k[64] = {
        0x428a2f98u, 0x71374491u, 0xb5c0fbcfu, 0xe9b5dba5u, 0x3956c25bu, 0x59f111f1u, 0x923f82a4u, 0xab1c5ed5u,
        0xd807aa98u, 0x12835b01u, 0x243185beu, 0x550c7dc3u, 0x72be5d74u, 0x80deb1feu, 0x9bdc06a7u, 0xc19bf174u,
        0xe49b69c1u, 0xefbe4786u, 0x0fc19dc6u, 0x240ca1ccu, 0x2de92c6fu, 0x4a7484aau, 0x5cb0a9dcu, 0x76f988dau,
        0x983e5152u, 0xa831c66du, 0xb00327c8u, 0xbf597fc7u, 0xc6e00bf3u, 0xd5a79147u, 0x06ca6351u, 0x14292967u,
        0x27b70a85u, 0x2e1b2138u, 0x4d2c6dfcu, 0x53380d13u, 0x650a7354u, 0x766a0abbu, 0x81c2c92eu, 0x92722c85u,
        0xa2bfe8a1u, 0xa81a664bu, 0xc24b8b70u, 0xc76c51a3u, 0xd192e819u, 0xd6990624u, 0xf40e3585u, 0x106aa070u,
        0x19a4c116u, 0x1e376c08u, 0x2748774cu, 0x34b0bcb5u, 0x391c0cb3u, 0x4ed8aa4au, 0x5b9cca4fu, 0x682e6ff3u,
        0x748f82eeu, 0x78a5636fu, 0x84c87814u, 0x8cc70208u, 0x90befffau, 0xa4506cebu, 0xbef9a3f7u, 0xc67178f2u};
    uint32_t w[64];
    for (int i = 0; i < 16; ++i)
      w[i] = (uint32_t)p[4 * i] << 24 | (uint32_t)p[4 * i + 1] << 16 | (uint32_t)p[4 * i + 2] << 8 | p[4 * i + 3];
    for (int i = 16; i < 64; ++i) {
      const uint32_t s0 = rotr(w[i - 15], 7) ^ rotr(w[i - 15], 18) ^ (w[i - 15] >> 3);
      const uint32_t s1 = rotr(w[i - 2], 17) ^ rotr(w[i - 2], 19) ^ (w[i - 2] >> 10);
      w[i] = w[i - 16] + s0 + w[i - 7] + s1;
    }
    uint32_t a = h[0], b = h[1], c = h[2], d = h[3], e = h[4], f = h[5], g = h[6], hh = h[7];
    for (int i = 0; i < 64; ++i) {
      const uint32_t t1 = hh + (rotr(e, 6) ^ rotr(e, 11) ^ rotr(e, 25)) + ((e & f) ^ (~e & g)) + k[i] + w[i];
      const uint32_t t2 = (rotr(a, 2) ^ rotr(a, 13) ^ rotr(a, 22)) + ((a & b) ^ (a & c) ^ (b & c));
      hh = g;
      g = f;
      f = e;
      e = d + t1;
      d = c;
      c = b;
      b = a;
      a = t1 + t2;
    }
    h[0] += a, h[1] += b, h[2] += c, h[3] += d, h[4] += e, h[5] += f, h[6] += g, h[7] += hh;
  }
  void update(const void* data, size_t len) {
    const unsigned char* p = static_cast<const unsigned char*>(data);
    bits += (uint64_t)len * 8;
    if (fill) {
      const size_t take = std::min<size_t>(64 - fill, len);
      std::memcpy(buf + fill, p, take);
      fill += take, p += take, len -= take;
      if (fill == 64) {
        block(buf);
        fill = 0;
      }
    }
    for (; len >= 64; p += 64, len -= 64) block(p);
    if (len) {
      std::memcpy(buf, p, len);
      fill = len;
    }
  }
  void final(unsigned char out[32]) {
    const uint64_t b = bits;
    const unsigned char one = 0x80, zero = 0;
    update(&one, 1);
    while (fill != 56) update(&zero, 1);
    unsigned char len[8];
    for (int i = 0; i < 8; ++i) len[i] = (unsigned char)(b >> (56 - 8 * i));
    update(len, 8);
    for (int i = 0; i < 8; ++i)
      for (int j = 0; j < 4; ++j) out[4 * i + j] = (unsigned char)(h[i] >> (24 - 8 * j));
  }
};

void hex(const unsigned char d[32], char out[65]) {
  static const char* x = "0123456789abcdef";
  for (int i = 0; i < 32; ++i) out[2 * i] = x[d[i] >> 4], out[2 * i + 1] = x[d[i] & 15];
  out[64] = 0;
}

// the payload of a column-major host block (ld >= rows) as it is stored
template <typename F>
void for_each_column(const double* a, uint64_t rows, uint64_t cols, uint64_t ld, F&& f) {
  for (uint64_t c = 0; c < cols; ++c) f(a + c * ld, rows * sizeof(double));
}

struct Header {
  uint64_t rows = 0, cols = 0;
  unsigned char sha[32] = {};
  char desc[kDescLen + 1] = {};
};

int read_header(std::FILE* f, Header& h, const char* path, bo_status* st) {
  unsigned char raw[kHeader];
  if (std::fread(raw, 1, kHeader, f) != kHeader)
    return fail(st, BO_INVALID, std::string("panel cache: truncated header in ") + path);
  if (std::memcmp(raw, kMagic, 8) != 0) return fail(st, BO_INVALID, std::string("panel cache: bad magic in ") + path);
  std::memcpy(&h.rows, raw + 8, 8);
  std::memcpy(&h.cols, raw + 16, 8);
  std::memcpy(h.sha, raw + 24, 32);
  std::memcpy(h.desc, raw + 56, kDescLen);
  h.desc[kDescLen] = 0;
  return BO_OK;
}

}  // namespace

extern "C" int bo_sha256(const void* data, uint64_t len, char hex_out[65]) {
  Sha256 s;
  s.update(data, (size_t)len);
  unsigned char d[32];
  s.final(d);
  hex(d, hex_out);
  return BO_OK;
}

extern "C" int bo_panel_cache_write(const char* path, const double* a, uint64_t rows, uint64_t cols, uint64_t ld,
                                    const char* desc, char sha_hex[65], bo_status* st) {
  ok(st);
  if (!a || ld < rows) return fail(st, BO_INVALID, "panel cache: bad block");
  Sha256 s;
  for_each_column(a, rows, cols, ld, [&](const double* c, size_t bytes) { s.update(c, bytes); });
  unsigned char d[32];
  s.final(d);
  unsigned char raw[kHeader] = {};
  std::memcpy(raw, kMagic, 8);
  std::memcpy(raw + 8, &rows, 8);
  std::memcpy(raw + 16, &cols, 8);
  std::memcpy(raw + 24, d, 32);
  if (desc) std::strncpy(reinterpret_cast<char*>(raw + 56), desc, kDescLen - 1);
  const std::string tmp = std::string(path) + ".tmp";
  std::FILE* f = std::fopen(tmp.c_str(), "wb");
  if (!f) return fail(st, BO_INVALID, std::string("panel cache: cannot open ") + tmp);
  bool good = std::fwrite(raw, 1, kHeader, f) == kHeader;
  for_each_column(a, rows, cols, ld, [&](const double* c, size_t bytes) {
    good = good && std::fwrite(c, 1, bytes, f) == bytes;
  });
  good = (std::fclose(f) == 0) && good;
  if (!good || std::rename(tmp.c_str(), path) != 0) {
    std::remove(tmp.c_str());
    return fail(st, BO_INVALID, std::string("panel cache: write failed for ") + path);
  }
  if (sha_hex) hex(d, sha_hex);
  return BO_OK;
}

// rows, cols, digest and generator text of a cache file (no payload read)
extern "C" int bo_panel_cache_info(const char* path, uint64_t* rows, uint64_t* cols, char sha_hex[65],
                                   char desc[256], bo_status* st) {
  ok(st);
  std::FILE* f = std::fopen(path, "rb");
  if (!f) return fail(st, BO_INVALID, std::string("panel cache: cannot open ") + path);
  Header h;
  const int rc = read_header(f, h, path, st);
  std::fclose(f);
  if (rc != BO_OK) return rc;
  if (rows) *rows = h.rows;
  if (cols) *cols = h.cols;
  if (sha_hex) hex(h.sha, sha_hex);
  if (desc) std::memcpy(desc, h.desc, kDescLen);
  return BO_OK;
}

// read the payload into a column-major host block (ld >= rows), verifying the digest
extern "C" int bo_panel_cache_read(const char* path, double* a, uint64_t rows, uint64_t cols, uint64_t ld,
                                   bo_status* st) {
  ok(st);
  std::FILE* f = std::fopen(path, "rb");
  if (!f) return fail(st, BO_INVALID, std::string("panel cache: cannot open ") + path);
  Header h;
  int rc = read_header(f, h, path, st);
  if (rc == BO_OK && (h.rows != rows || h.cols != cols || ld < rows))
    rc = fail(st, BO_INVALID, "panel cache: " + std::string(path) + " holds " + std::to_string(h.rows) + " x " +
                                  std::to_string(h.cols) + ", asked for " + std::to_string(rows) + " x " +
                                  std::to_string(cols));
  Sha256 s;
  bool good = rc == BO_OK;
  for (uint64_t c = 0; good && c < cols; ++c) {
    double* dst = a + c * ld;
    const size_t bytes = rows * sizeof(double);
    good = std::fread(dst, 1, bytes, f) == bytes;
    if (good) s.update(dst, bytes);
  }
  std::fclose(f);
  if (rc != BO_OK) return rc;
  if (!good) return fail(st, BO_INVALID, std::string("panel cache: truncated payload in ") + path);
  unsigned char d[32];
  s.final(d);
  if (std::memcmp(d, h.sha, 32) != 0)
    return fail(st, BO_INVALID, std::string("panel cache: SHA-256 mismatch in ") + path);
  return BO_OK;
}
