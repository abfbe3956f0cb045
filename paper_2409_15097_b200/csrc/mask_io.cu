// mask_io.cu — the reference's BBMK mask file and BBLK occupancy sidecar (mask_io.hpp:14-207),
// with a device path: a BBMK payload (ceil(n/8)-byte rows, LSB = lowest column) is uploaded
// as-is and unpacked into the preprocessor's padded u64 layout by a kernel, so a mask file goes
// to block metadata without a host-side bit loop.
//
// Errors follow MaskIoError's kinds (mask_io.hpp:24-42), one bbm_status each; the header checks,
// the 4M-token cap and the exact payload size are the reference's (mask_io.hpp:95-131).
#include <cuda_runtime.h>

#include <cstdint>
#include <cstring>
#include <fstream>
#include <iterator>
#include <string>
#include <vector>

#include "../../include/bbm_capi.h"
#include "bbm_internal.h"

namespace bbm {
namespace {

struct IoError : std::runtime_error {
  bbm_status code;
  IoError(bbm_status c, const std::string& w) : std::runtime_error(w), code(c) {}
};

constexpr uint64_t kMaxMaskTokens = uint64_t{1} << 22;

std::string read_all(const char* path) {
  std::ifstream in(path, std::ios::binary);
  if (!in) throw IoError(BBM_ERR_IO_FAILURE, std::string("cannot open ") + path);
  std::string data((std::istreambuf_iterator<char>(in)), std::istreambuf_iterator<char>());
  if (in.bad()) throw IoError(BBM_ERR_IO_FAILURE, std::string("read failed: ") + path);
  return data;
}

void write_all(const char* path, const std::string& data) {
  std::ofstream out(path, std::ios::binary | std::ios::trunc);
  if (!out) throw IoError(BBM_ERR_IO_FAILURE, std::string("cannot open ") + path);
  out.write(data.data(), static_cast<std::streamsize>(data.size()));
  if (!out) throw IoError(BBM_ERR_IO_FAILURE, std::string("write failed: ") + path);
}

uint64_t le64(const unsigned char* p) {
  uint64_t v = 0;
  for (int b = 0; b < 8; ++b) v |= uint64_t{p[b]} << (8 * b);
  return v;
}
uint32_t le32(const unsigned char* p) {
  uint32_t v = 0;
  for (int b = 0; b < 4; ++b) v |= uint32_t{p[b]} << (8 * b);
  return v;
}
void put_le(std::string& out, uint64_t v, int bytes) {
  for (int b = 0; b < bytes; ++b) out.push_back(static_cast<char>((v >> (8 * b)) & 0xff));
}

// mask_io.hpp:100-131: magic, header length, version, dimension cap, exact payload size
uint64_t parse_header(const std::string& d, const char* magic, size_t extra) {
  if (d.size() < 4 || std::memcmp(d.data(), magic, 4) != 0)
    throw IoError(BBM_ERR_IO_BAD_MAGIC, std::string("bad magic, expected ") + magic);
  if (d.size() < 13 + extra) throw IoError(BBM_ERR_IO_TRUNCATED, "truncated header");
  if (d[4] != 1) throw IoError(BBM_ERR_IO_BAD_VERSION, "unsupported version " + std::to_string(int(d[4])));
  const uint64_t n = le64(reinterpret_cast<const unsigned char*>(d.data()) + 5);
  if (n > kMaxMaskTokens)
    throw IoError(BBM_ERR_IO_DIMENSION_OVERFLOW, "mask dimension " + std::to_string(n) + " exceeds limit");
  return n;
}

void check_payload(const std::string& d, uint64_t offset, uint64_t rows, uint64_t row_bytes) {
  const uint64_t expected = offset + rows * row_bytes;
  if (d.size() < expected)
    throw IoError(BBM_ERR_IO_TRUNCATED, "payload truncated: have " + std::to_string(d.size()) +
                                            " bytes, expected " + std::to_string(expected));
  if (d.size() > expected) throw IoError(BBM_ERR_IO_TRAILING_DATA, "unexpected trailing bytes after payload");
}

template <class F>
bbm_status io_guarded(F&& f) {
  try {
    f();
    return BBM_OK;
  } catch (const IoError& e) {
    g_last_error = e.what();
    return e.code;
  } catch (const ArgError& e) {
    g_last_error = e.what();
    return BBM_ERR_INVALID;
  } catch (const CudaError& e) {
    g_last_error = e.what();
    return BBM_ERR_CUDA;
  } catch (const std::exception& e) {
    g_last_error = e.what();
    return BBM_ERR_INTERNAL;
  }
}

// byte rows -> u64 words: word w of row i takes bytes [8w, 8w+8) of the row (little endian, so
// bit j&63 is column 64w + (j&63), the Mask layout, mask.hpp:20-28); bits past n are cleared.
__global__ void bytes_to_words_kernel(const uint8_t* __restrict__ payload, uint64_t n, uint64_t row_bytes,
                                      uint64_t out_wpr, uint64_t rows_out, uint64_t* __restrict__ out) {
  const uint64_t total = rows_out * out_wpr;
  for (uint64_t t = blockIdx.x * static_cast<uint64_t>(blockDim.x) + threadIdx.x; t < total;
       t += static_cast<uint64_t>(gridDim.x) * blockDim.x) {
    const uint64_t i = t / out_wpr, w = t % out_wpr;
    uint64_t word = 0;
    if (i < n) {
      const uint8_t* row = payload + i * row_bytes;
      for (uint32_t b = 0; b < 8; ++b) {
        const uint64_t byte = w * 8 + b;
        if (byte < row_bytes) word |= uint64_t{row[byte]} << (8 * b);
      }
      const uint64_t c0 = w * 64;
      if (c0 >= n) word = 0;
      else if (n - c0 < 64) word &= (uint64_t{1} << (n - c0)) - 1;
    }
    out[t] = word;
  }
}

}  // namespace

// Unpack a BBMK payload already on the device into `n x wpr` packed words (wpr >= ceil(n/64)).
void launch_bbmk_unpack(const uint8_t* d_payload, uint64_t n, uint64_t* d_words, uint64_t wpr,
                        uint64_t rows_out, cudaStream_t s) {
  const uint64_t total = rows_out * wpr;
  const unsigned grid = static_cast<unsigned>(std::max<uint64_t>(1, std::min<uint64_t>((total + 255) / 256, 148ull * 32)));
  bytes_to_words_kernel<<<grid, 256, 0, s>>>(d_payload, n, (n + 7) / 8, wpr, rows_out, d_words);
  BBM_CUDA(cudaGetLastError());
}

}  // namespace bbm

using namespace bbm;

extern "C" {

bbm_status bbm_write_mask_file(const char* path, const uint64_t* words, uint64_t n) {
  return io_guarded([&] {
    require(path && (words || n == 0), "null argument");
    const uint64_t wpr = (n + 63) / 64, rb = (n + 7) / 8;
    std::string out;
    out.reserve(13 + n * rb);
    out += "BBMK";
    out.push_back(1);
    put_le(out, n, 8);
    for (uint64_t i = 0; i < n; ++i)
      for (uint64_t b = 0; b < rb; ++b) out.push_back(static_cast<char>((words[i * wpr + b / 8] >> (8 * (b % 8))) & 0xff));
    write_all(path, out);
  });
}

bbm_status bbm_read_mask_file(const char* path, uint64_t* n_out, uint64_t* words) {
  return io_guarded([&] {
    require(path && n_out, "null argument");
    const std::string d = read_all(path);
    const uint64_t n = parse_header(d, "BBMK", 0), rb = (n + 7) / 8, wpr = (n + 63) / 64;
    check_payload(d, 13, n, rb);
    *n_out = n;
    if (!words) return;
    const auto* bytes = reinterpret_cast<const unsigned char*>(d.data()) + 13;
    for (uint64_t i = 0; i < n; ++i)
      for (uint64_t w = 0; w < wpr; ++w) {
        uint64_t word = 0;
        for (uint64_t b = 0; b < 8 && w * 8 + b < rb; ++b) word |= uint64_t{bytes[i * rb + w * 8 + b]} << (8 * b);
        if (n - w * 64 < 64) word &= (uint64_t{1} << (n - w * 64)) - 1;
        words[i * wpr + w] = word;
      }
  });
}

bbm_status bbm_write_occupancy_file(const char* path, const uint8_t* occ, uint64_t n_tokens,
                                    uint64_t block_i, uint64_t block_j) {
  return io_guarded([&] {
    require(path && occ, "null argument");
    require(block_i >= 1 && block_j >= 1, "block sizes must be >= 1");
    const uint64_t rows = (n_tokens + block_i - 1) / block_i, cols = (n_tokens + block_j - 1) / block_j;
    std::string out = "BBLK";
    out.push_back(1);
    put_le(out, n_tokens, 8);
    put_le(out, block_i, 4);
    put_le(out, block_j, 4);
    for (uint64_t p = 0; p < rows; ++p)
      for (uint64_t b = 0; b < (cols + 7) / 8; ++b) {
        unsigned byte = 0;
        for (uint64_t q = b * 8; q < std::min(cols, b * 8 + 8); ++q)
          if (occ[p * cols + q]) byte |= 1u << (q - b * 8);
        out.push_back(static_cast<char>(byte));
      }
    write_all(path, out);
  });
}

bbm_status bbm_read_occupancy_file(const char* path, uint64_t* n_tokens, uint64_t* block_i,
                                   uint64_t* block_j, uint8_t* occ) {
  return io_guarded([&] {
    require(path && n_tokens && block_i && block_j, "null argument");
    const std::string d = read_all(path);
    const uint64_t n = parse_header(d, "BBLK", 8);
    const auto* base = reinterpret_cast<const unsigned char*>(d.data());
    const uint64_t bi = le32(base + 13), bj = le32(base + 17);
    if (bi == 0 || bj == 0) throw IoError(BBM_ERR_IO_DIMENSION_OVERFLOW, "zero block size");
    const uint64_t rows = (n + bi - 1) / bi, cols = (n + bj - 1) / bj, rb = (cols + 7) / 8;
    check_payload(d, 21, rows, rb);
    *n_tokens = n;
    *block_i = bi;
    *block_j = bj;
    if (!occ) return;
    for (uint64_t p = 0; p < rows; ++p)
      for (uint64_t q = 0; q < cols; ++q) occ[p * cols + q] = (base[21 + p * rb + (q >> 3)] >> (q & 7)) & 1u;
  });
}

bbm_status bbm_preprocess_mask_file(const char* path, uint64_t block_i, uint64_t block_j, int device,
                                    bbm_prep* out) {
  return io_guarded([&] {
    require(path && out, "null argument");
    const std::string d = read_all(path);
    const uint64_t n = parse_header(d, "BBMK", 0), rb = (n + 7) / 8, wpr = (n + 63) / 64;
    check_payload(d, 13, n, rb);
    require(n >= 1, "mask must be non-empty");
    int prev = 0;
    BBM_CUDA(cudaGetDevice(&prev));
    BBM_CUDA(cudaSetDevice(device));
    uint8_t* d_payload = nullptr;
    uint64_t* d_words = nullptr;
    cudaStream_t s = nullptr;
    bbm_status st = BBM_OK;
    try {
      BBM_CUDA(cudaStreamCreateWithFlags(&s, cudaStreamNonBlocking));
      BBM_CUDA(cudaMalloc(&d_payload, std::max<uint64_t>(1, n * rb)));
      BBM_CUDA(cudaMalloc(&d_words, n * wpr * 8));
      BBM_CUDA(cudaMemcpyAsync(d_payload, d.data() + 13, n * rb, cudaMemcpyHostToDevice, s));
      launch_bbmk_unpack(d_payload, n, d_words, wpr, n, s);
      st = bbm_preprocess_packed_device(d_words, n, block_i, block_j, s, out);
      BBM_CUDA(cudaStreamSynchronize(s));
    } catch (...) {
      cudaFree(d_payload), cudaFree(d_words);
      if (s) cudaStreamDestroy(s);
      cudaSetDevice(prev);
      throw;
    }
    cudaFree(d_payload), cudaFree(d_words);
    cudaStreamDestroy(s);
    cudaSetDevice(prev);
    if (st != BBM_OK) throw IoError(st, g_last_error);
  });
}

}  // extern "C"
