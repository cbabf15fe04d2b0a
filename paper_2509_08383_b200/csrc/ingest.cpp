// ingest.cpp — logit files for the batch API.
//
//   LGT1:  "LGT1" | u16 version (= 1) | u32 count | u32 n | count*n little-endian float32
//   JSONL: one vector per line, a JSON array of numbers, all of the same length
//
// Readers write straight into a caller buffer (e.g. pinned host memory, which
// then feeds pam_cutmax_batch_* with a single async copy).  Errors follow the
// reference's errors.hpp: FormatError carries the byte offset of the problem,
// NonFiniteError the index of the first vector holding NaN/Inf.
// Plain C++17 on the host; no GPU involvement.
#include <cerrno>
#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <string>
#include <vector>

#include "../../include/pam_c_api.h"

namespace {

constexpr char kMagic[4] = {'L', 'G', 'T', '1'};
constexpr int kHeader = 14;  // magic 4 + version 2 + count 4 + n 4
constexpr uint16_t kVersion = 1;

uint32_t rd_u32(const unsigned char* p) {
  return (uint32_t)p[0] | ((uint32_t)p[1] << 8) | ((uint32_t)p[2] << 16) | ((uint32_t)p[3] << 24);
}

void wr_u32(unsigned char* p, uint32_t v) {
  for (int i = 0; i < 4; ++i) p[i] = (unsigned char)(v >> (8 * i));
}

float rd_f32(const unsigned char* p) {
  const uint32_t b = rd_u32(p);
  float f;
  std::memcpy(&f, &b, 4);
  return f;
}

void reset(pam_ingest_info* info) {
  if (!info) return;
  info->count = info->n = 0;
  info->err_offset = -1;
  info->bad_vector = -1;
}

int fail_format(pam_ingest_info* info, int64_t off) {
  if (info) info->err_offset = off;
  return PAM_ERR_FORMAT;
}

bool slurp(const char* path, std::vector<unsigned char>& out) {
  FILE* f = std::fopen(path, "rb");
  if (!f) return false;
  unsigned char buf[1 << 16];
  size_t got;
  while ((got = std::fread(buf, 1, sizeof buf, f)) > 0) out.insert(out.end(), buf, buf + got);
  std::fclose(f);
  return true;
}

// LGT1 header checks; on success count/n are set and the payload size verified.
int lgt1_header(const std::vector<unsigned char>& d, pam_ingest_info* info) {
  if (d.size() < 4) return fail_format(info, (int64_t)d.size());
  for (int i = 0; i < 4; ++i)
    if (d[i] != (unsigned char)kMagic[i]) return fail_format(info, i);  // magic exact match
  if (d.size() < (size_t)kHeader) return fail_format(info, (int64_t)d.size());
  const uint16_t ver = (uint16_t)(d[4] | (d[5] << 8));
  if (ver != kVersion) return fail_format(info, 4);
  const uint32_t count = rd_u32(&d[6]), n = rd_u32(&d[10]);
  const uint64_t payload = (uint64_t)count * n * 4u;
  if (d.size() - kHeader < payload) return fail_format(info, (int64_t)d.size());  // truncated payload
  if (d.size() - kHeader > payload) return fail_format(info, (int64_t)(kHeader + payload));  // trailing bytes
  info->count = count;
  info->n = n;
  return PAM_OK;
}

// JSON lines: parse every line into `vals` (row-major), checking equal lengths.
int jsonl_parse(const std::vector<unsigned char>& d, std::vector<double>* vals, pam_ingest_info* info) {
  const char* s = reinterpret_cast<const char*>(d.data());
  const size_t len = d.size();
  size_t i = 0;
  int64_t count = 0, n = -1;
  auto skip_ws = [&](bool newline_ok) {
    while (i < len && (s[i] == ' ' || s[i] == '\t' || s[i] == '\r' || (newline_ok && s[i] == '\n'))) ++i;
  };
  std::string tok;
  while (true) {
    skip_ws(true);
    if (i >= len) break;
    if (s[i] != '[') return fail_format(info, (int64_t)i);
    ++i;
    int64_t k = 0;
    skip_ws(false);
    if (i < len && s[i] == ']') return fail_format(info, (int64_t)i);  // empty vector
    while (true) {
      skip_ws(false);
      // a JSON number: -?digits(.digits)?([eE][+-]?digits)?
      const size_t start = i;
      if (i < len && s[i] == '-') ++i;
      size_t digits = 0;
      while (i < len && s[i] >= '0' && s[i] <= '9') ++i, ++digits;
      if (i < len && s[i] == '.') {
        ++i;
        while (i < len && s[i] >= '0' && s[i] <= '9') ++i, ++digits;
      }
      if (digits == 0) return fail_format(info, (int64_t)start);
      if (i < len && (s[i] == 'e' || s[i] == 'E')) {
        ++i;
        if (i < len && (s[i] == '+' || s[i] == '-')) ++i;
        size_t ed = 0;
        while (i < len && s[i] >= '0' && s[i] <= '9') ++i, ++ed;
        if (ed == 0) return fail_format(info, (int64_t)i);
      }
      tok.assign(s + start, i - start);
      const double v = std::strtod(tok.c_str(), nullptr);  // out-of-range -> +-inf (checked by the caller)
      if (vals) vals->push_back(v);
      ++k;
      skip_ws(false);
      if (i < len && s[i] == ',') {
        ++i;
        continue;
      }
      if (i < len && s[i] == ']') {
        ++i;
        break;
      }
      return fail_format(info, (int64_t)i);
    }
    skip_ws(false);
    if (i < len && s[i] != '\n') return fail_format(info, (int64_t)i);  // one array per line
    if (n < 0) n = k;
    if (k != n) return fail_format(info, (int64_t)i);  // ragged lines
    ++count;
  }
  if (count == 0) return fail_format(info, 0);
  info->count = count;
  info->n = n;
  return PAM_OK;
}

}  // namespace

extern "C" {

int pam_lgt1_probe(const char* path, pam_ingest_info* info) {
  if (!path || !info) return PAM_ERR_BAD_ARGUMENT;
  reset(info);
  std::vector<unsigned char> d;
  if (!slurp(path, d)) return PAM_ERR_BAD_ARGUMENT;
  return lgt1_header(d, info);
}

int pam_lgt1_read(const char* path, float* dst, int64_t capacity, pam_ingest_info* info) {
  if (!path || !info) return PAM_ERR_BAD_ARGUMENT;
  reset(info);
  std::vector<unsigned char> d;
  if (!slurp(path, d)) return PAM_ERR_BAD_ARGUMENT;
  int st = lgt1_header(d, info);
  if (st) return st;
  const int64_t total = info->count * info->n;
  if (!dst || capacity < total) return PAM_ERR_BAD_ARGUMENT;
  const unsigned char* p = d.data() + kHeader;
  for (int64_t r = 0; r < info->count; ++r) {
    bool finite = true;
    for (int64_t j = 0; j < info->n; ++j) {
      const float v = rd_f32(p + 4 * (r * info->n + j));
      dst[r * info->n + j] = v;
      finite = finite && std::isfinite(v);
    }
    if (!finite && info->bad_vector < 0) info->bad_vector = r;
  }
  return info->bad_vector >= 0 ? PAM_ERR_NON_FINITE : PAM_OK;  // parsed vectors, validated finite
}

int pam_lgt1_write(const char* path, const float* src, int64_t count, int64_t n) {
  if (!path || (count > 0 && !src) || count < 0 || n < 0 || count > 0xffffffffLL || n > 0xffffffffLL)
    return PAM_ERR_BAD_ARGUMENT;
  FILE* f = std::fopen(path, "wb");
  if (!f) return PAM_ERR_BAD_ARGUMENT;
  unsigned char hdr[kHeader];
  std::memcpy(hdr, kMagic, 4);
  hdr[4] = (unsigned char)(kVersion & 0xff);
  hdr[5] = (unsigned char)(kVersion >> 8);
  wr_u32(hdr + 6, (uint32_t)count);
  wr_u32(hdr + 10, (uint32_t)n);
  bool ok = std::fwrite(hdr, 1, kHeader, f) == (size_t)kHeader;
  std::vector<unsigned char> row((size_t)n * 4);
  for (int64_t r = 0; ok && r < count; ++r) {
    for (int64_t j = 0; j < n; ++j) {
      uint32_t b;
      std::memcpy(&b, &src[r * n + j], 4);
      wr_u32(&row[(size_t)j * 4], b);  // little-endian on any host
    }
    ok = std::fwrite(row.data(), 1, row.size(), f) == row.size();
  }
  ok = (std::fclose(f) == 0) && ok;
  return ok ? PAM_OK : PAM_ERR_BAD_ARGUMENT;
}

int pam_jsonl_probe(const char* path, pam_ingest_info* info) {
  if (!path || !info) return PAM_ERR_BAD_ARGUMENT;
  reset(info);
  std::vector<unsigned char> d;
  if (!slurp(path, d)) return PAM_ERR_BAD_ARGUMENT;
  return jsonl_parse(d, nullptr, info);
}

int pam_jsonl_read(const char* path, double* dst, int64_t capacity, pam_ingest_info* info) {
  if (!path || !info) return PAM_ERR_BAD_ARGUMENT;
  reset(info);
  std::vector<unsigned char> d;
  if (!slurp(path, d)) return PAM_ERR_BAD_ARGUMENT;
  std::vector<double> vals;
  int st = jsonl_parse(d, &vals, info);
  if (st) return st;
  if (!dst || capacity < info->count * info->n) return PAM_ERR_BAD_ARGUMENT;
  for (int64_t r = 0; r < info->count; ++r) {
    bool finite = true;
    for (int64_t j = 0; j < info->n; ++j) {
      const double v = vals[(size_t)(r * info->n + j)];
      dst[r * info->n + j] = v;
      finite = finite && std::isfinite(v);
    }
    if (!finite && info->bad_vector < 0) info->bad_vector = r;
  }
  return info->bad_vector >= 0 ? PAM_ERR_NON_FINITE : PAM_OK;
}

}  // extern "C"
