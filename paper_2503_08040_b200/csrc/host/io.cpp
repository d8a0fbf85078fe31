// Wire formats: the reference's ".fmat" dense fp32 matrix
// (matrix.cpp:75-142, matrix.hpp:86-90) read and written byte-compatibly, with
// the reference's FormatError checks and byte offsets, plus a ".fqt" sidecar
// for block-quantized / fallback tensors (codes, scales, fallback bitmap,
// residual plane) so golden vectors and gemm-check inputs move between machines.
//
// .fmat : "FMAT" | u32 version=1 | u64 rows | u64 cols | rows*cols f32 (LE, row-major)
// .fqt  : "FQT1" | u32 version=1 | u64 rows | u64 cols | u32 block=128 | u32 bits=8 |
//         u32 flags (bit 0: fallback) | u32 reserved=0 |
//         codes int8 rows*cols | scales f32 grid (ceil(r/128) x ceil(c/128)) |
//         [fallback: mask u32 ceil(blocks/32) | residual codes int8 rows*cols |
//          residual scales f32 grid]
#include <cmath>
#include <cstdint>
#include <cstring>
#include <fstream>
#include <string>
#include <vector>

#include "../../../include/fbq_b200_host.h"

namespace {

thread_local std::string g_io_err;
thread_local uint64_t g_io_off = 0;

int fail(const std::string& what, uint64_t off) {
  g_io_err = what + " (byte offset " + std::to_string(off) + ")";
  g_io_off = off;
  return FBQ_ERR_FORMAT;
}
int64_t cdiv(int64_t a, int64_t b) { return (a + b - 1) / b; }

struct FmatHeader {
  uint64_t rows = 0, cols = 0;
};

// header checks of load_matrix (matrix.cpp:107-126)
int read_fmat_header(std::ifstream& in, const char* path, FmatHeader& h) {
  if (!in) return fail(std::string("cannot open '") + path + "'", 0);
  char header[24];
  in.read(header, sizeof(header));
  if (in.gcount() != (std::streamsize)sizeof(header)) return fail("truncated header", (uint64_t)in.gcount());
  if (std::memcmp(header, "FMAT", 4) != 0) return fail("bad magic", 0);
  uint32_t version;
  std::memcpy(&version, header + 4, 4);
  std::memcpy(&h.rows, header + 8, 8);
  std::memcpy(&h.cols, header + 16, 8);
  if (version != 1) return fail("unsupported version", 4);
  if (h.rows > (1ull << 31) || h.cols > (1ull << 31) || (h.rows != 0 && h.cols > (1ull << 40) / h.rows))
    return fail("implausible dimensions", 8);
  return FBQ_OK;
}

}  // namespace

extern "C" {

const char* fbq_io_last_error(void) { return g_io_err.c_str(); }
uint64_t fbq_io_last_offset(void) { return g_io_off; }

int fbq_fmat_save(const char* path, const float* data, int64_t rows, int64_t cols) {
  if (!path || rows < 0 || cols < 0 || (rows * cols > 0 && !data)) return FBQ_ERR_ARG;
  std::ofstream out(path, std::ios::binary | std::ios::trunc);
  if (!out) return fail(std::string("cannot open '") + path + "' for writing", 0);
  char header[24];
  const uint32_t version = 1;
  const uint64_t r = (uint64_t)rows, c = (uint64_t)cols;
  std::memcpy(header, "FMAT", 4);
  std::memcpy(header + 4, &version, 4);
  std::memcpy(header + 8, &r, 8);
  std::memcpy(header + 16, &c, 8);
  out.write(header, 24);
  out.write(reinterpret_cast<const char*>(data), (std::streamsize)(rows * cols * 4));
  if (!out) return fail(std::string("short write to '") + path + "'", 24);
  return FBQ_OK;
}

int fbq_fmat_info(const char* path, int64_t* rows, int64_t* cols) {
  if (!path || !rows || !cols) return FBQ_ERR_ARG;
  std::ifstream in(path, std::ios::binary);
  FmatHeader h;
  if (int st = read_fmat_header(in, path, h)) return st;
  *rows = (int64_t)h.rows;
  *cols = (int64_t)h.cols;
  return FBQ_OK;
}

int fbq_fmat_load(const char* path, float* data, int64_t capacity, int64_t* rows, int64_t* cols) {
  if (!path || !rows || !cols) return FBQ_ERR_ARG;
  std::ifstream in(path, std::ios::binary);
  FmatHeader h;
  if (int st = read_fmat_header(in, path, h)) return st;
  const uint64_t count = h.rows * h.cols;
  if ((int64_t)count > capacity || (count && !data)) return FBQ_ERR_ARG;
  in.read(reinterpret_cast<char*>(data), (std::streamsize)(count * 4));
  const uint64_t got = (uint64_t)in.gcount();
  if (got != count * 4) return fail("truncated payload", 24 + got);
  for (uint64_t i = 0; i < count; ++i)
    if (!std::isfinite(data[i])) return fail("non-finite value", 24 + i * 4);
  *rows = (int64_t)h.rows;
  *cols = (int64_t)h.cols;
  return FBQ_OK;
}

int fbq_fqt_save(const char* path, int64_t rows, int64_t cols, const int8_t* codes, int64_t ldq,
                 const float* scales, const uint32_t* mask_bits, const int8_t* res_codes,
                 const float* res_scales) {
  if (!path || rows < 0 || cols < 0 || ldq < cols) return FBQ_ERR_ARG;
  const int64_t blocks = cdiv(rows, 128) * cdiv(cols, 128);
  if (rows * cols > 0 && (!codes || !scales)) return FBQ_ERR_ARG;
  const bool fb = mask_bits != nullptr;
  if (fb && rows * cols > 0 && (!res_codes || !res_scales)) return FBQ_ERR_ARG;
  std::ofstream out(path, std::ios::binary | std::ios::trunc);
  if (!out) return fail(std::string("cannot open '") + path + "' for writing", 0);
  char header[40];
  const uint32_t version = 1, block = 128, bits = 8, flags = fb ? 1u : 0u, reserved = 0;
  const uint64_t r = (uint64_t)rows, c = (uint64_t)cols;
  std::memcpy(header, "FQT1", 4);
  std::memcpy(header + 4, &version, 4);
  std::memcpy(header + 8, &r, 8);
  std::memcpy(header + 16, &c, 8);
  std::memcpy(header + 24, &block, 4);
  std::memcpy(header + 28, &bits, 4);
  std::memcpy(header + 32, &flags, 4);
  std::memcpy(header + 36, &reserved, 4);
  out.write(header, 40);
  auto plane = [&](const int8_t* p) {
    for (int64_t i = 0; i < rows; ++i) out.write(reinterpret_cast<const char*>(p + i * ldq), cols);
  };
  plane(codes);
  out.write(reinterpret_cast<const char*>(scales), blocks * 4);
  if (fb) {
    out.write(reinterpret_cast<const char*>(mask_bits), cdiv(blocks, 32) * 4);
    plane(res_codes);
    out.write(reinterpret_cast<const char*>(res_scales), blocks * 4);
  }
  if (!out) return fail(std::string("short write to '") + path + "'", 40);
  return FBQ_OK;
}

int fbq_fqt_info(const char* path, int64_t* rows, int64_t* cols, int* has_fallback) {
  if (!path || !rows || !cols || !has_fallback) return FBQ_ERR_ARG;
  std::ifstream in(path, std::ios::binary);
  if (!in) return fail(std::string("cannot open '") + path + "'", 0);
  char header[40];
  in.read(header, 40);
  if (in.gcount() != 40) return fail("truncated header", (uint64_t)in.gcount());
  if (std::memcmp(header, "FQT1", 4) != 0) return fail("bad magic", 0);
  uint32_t version, block, bits, flags;
  uint64_t r, c;
  std::memcpy(&version, header + 4, 4);
  std::memcpy(&r, header + 8, 8);
  std::memcpy(&c, header + 16, 8);
  std::memcpy(&block, header + 24, 4);
  std::memcpy(&bits, header + 28, 4);
  std::memcpy(&flags, header + 32, 4);
  if (version != 1) return fail("unsupported version", 4);
  if (r > (1ull << 31) || c > (1ull << 31) || (r != 0 && c > (1ull << 40) / r))
    return fail("implausible dimensions", 8);
  if (block != 128 || bits != 8) return fail("unsupported geometry", 24);
  *rows = (int64_t)r;
  *cols = (int64_t)c;
  *has_fallback = (int)(flags & 1u);
  return FBQ_OK;
}

int fbq_fqt_load(const char* path, int8_t* codes, int64_t ldq, float* scales, uint32_t* mask_bits,
                 int8_t* res_codes, float* res_scales) {
  int64_t rows, cols;
  int fb;
  if (int st = fbq_fqt_info(path, &rows, &cols, &fb)) return st;
  if (ldq < cols || (rows * cols > 0 && (!codes || !scales))) return FBQ_ERR_ARG;
  if (fb && rows * cols > 0 && (!mask_bits || !res_codes || !res_scales)) return FBQ_ERR_ARG;
  std::ifstream in(path, std::ios::binary);
  in.seekg(40);
  uint64_t off = 40;
  const int64_t blocks = cdiv(rows, 128) * cdiv(cols, 128);
  auto get = [&](char* p, int64_t n) -> bool {
    in.read(p, n);
    off += (uint64_t)in.gcount();
    return in.gcount() == n;
  };
  auto plane = [&](int8_t* p) -> bool {
    for (int64_t i = 0; i < rows; ++i)
      if (!get(reinterpret_cast<char*>(p + i * ldq), cols)) return false;
    return true;
  };
  if (!plane(codes) || !get(reinterpret_cast<char*>(scales), blocks * 4))
    return fail("truncated payload", off);
  if (fb) {
    if (!get(reinterpret_cast<char*>(mask_bits), cdiv(blocks, 32) * 4) || !plane(res_codes) ||
        !get(reinterpret_cast<char*>(res_scales), blocks * 4))
      return fail("truncated payload", off);
  }
  return FBQ_OK;
}

}  // extern "C"
