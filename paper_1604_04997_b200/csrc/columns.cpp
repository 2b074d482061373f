// Columnar binary side format for bulk bindings, timings and predictions
// ("kcg-columns v1"). The reference's interchange formats
// stay as they are -- the measurement CSV (csvio.cpp:104-190, %.17g text) and
// the weights JSON (jsonio.cpp:96-143) -- but a 1e9-row grid is 24+ GB of
// int64 that CSV text cannot carry at PCIe speed. Layout (little endian):
//
//   0   "KCGCOL01"                     magic
//   8   u32 version = 1, u32 n_cols
//   16  u64 n_rows
//   24  u64 reserved[5]
//   64  n_cols x 64-byte entries: char name[40] (NUL padded), u32 dtype
//       (1 int64, 2 float64, 3 uint8, 4 int32), u32 reserved, u64 offset,
//       u64 nbytes
//   data: each column contiguous at a 4096-byte aligned offset
//
// Reading maps the file; kcg_columns_load streams rows of a column to the
// device -- through the page-locked mapping when the driver accepts it
// (cudaHostRegisterReadOnly), otherwise through a pinned staging ring.
#include <cuda_runtime.h>
#include <fcntl.h>
#include <sys/mman.h>
#include <sys/stat.h>
#include <unistd.h>

#include <algorithm>
#include <cstring>
#include <memory>
#include <string>
#include <vector>

#include "../../include/kcg.h"
#include "kcg_host.hpp"

kcg_columns::~kcg_columns() {
  if (pending) {  // DMA out of the mapping must finish before it goes away
    cudaEventSynchronize(static_cast<cudaEvent_t>(pending));
    cudaEventDestroy(static_cast<cudaEvent_t>(pending));
  }
  if (registered) cudaHostUnregister(map);
  if (map && map != MAP_FAILED) munmap(map, map_len);
  if (fd >= 0) close(fd);
}

namespace kcg {

namespace {

constexpr char kMagic[8] = {'K', 'C', 'G', 'C', 'O', 'L', '0', '1'};
constexpr uint64_t kAlign = 4096;

size_t dtype_size(int dt) {
  switch (dt) {
    case KCG_COL_INT64:
    case KCG_COL_FLOAT64: return 8;
    case KCG_COL_UINT8: return 1;
    case KCG_COL_INT32: return 4;
    default: throw KcgError(KCG_E_INVALID_ARGUMENT, "unknown column dtype " + std::to_string(dt));
  }
}

void write_all(int fd, const void* p, size_t n, const std::string& path) {
  const char* c = static_cast<const char*>(p);
  while (n) {
    const ssize_t w = ::write(fd, c, n);
    if (w <= 0) throw KcgError(KCG_E_IO, "write failed: " + path);
    c += w;
    n -= static_cast<size_t>(w);
  }
}

}  // namespace

void columns_write(const char* path, int n_cols, const char* const* names, const int* dtypes,
                   const void* const* data, uint64_t n_rows) {
  if (!path || n_cols < 0 || (n_cols > 0 && (!names || !dtypes || !data)))
    throw KcgError(KCG_E_INVALID_ARGUMENT, "bad kcg_columns_write arguments");
  std::vector<unsigned char> head(64 + 64 * static_cast<size_t>(n_cols), 0);
  std::memcpy(head.data(), kMagic, 8);
  const uint32_t ver = 1, nc = static_cast<uint32_t>(n_cols);
  std::memcpy(head.data() + 8, &ver, 4);
  std::memcpy(head.data() + 12, &nc, 4);
  std::memcpy(head.data() + 16, &n_rows, 8);
  uint64_t off = (head.size() + kAlign - 1) / kAlign * kAlign;
  std::vector<uint64_t> offs(n_cols), lens(n_cols);
  for (int j = 0; j < n_cols; ++j) {
    const size_t nl = std::strlen(names[j]);
    if (nl == 0 || nl >= 40) throw KcgError(KCG_E_INVALID_ARGUMENT, "column names need 1..39 bytes");
    unsigned char* e = head.data() + 64 + 64 * static_cast<size_t>(j);
    std::memcpy(e, names[j], nl);
    const uint32_t dt = static_cast<uint32_t>(dtypes[j]);
    lens[j] = n_rows * dtype_size(dtypes[j]);
    offs[j] = off;
    std::memcpy(e + 40, &dt, 4);
    std::memcpy(e + 48, &offs[j], 8);
    std::memcpy(e + 56, &lens[j], 8);
    off = (off + lens[j] + kAlign - 1) / kAlign * kAlign;
  }
  const int fd = ::open(path, O_WRONLY | O_CREAT | O_TRUNC, 0644);
  if (fd < 0) throw KcgError(KCG_E_IO, std::string("cannot create ") + path);
  try {
    write_all(fd, head.data(), head.size(), path);
    uint64_t pos = head.size();
    static const std::vector<char> zeros(kAlign, 0);
    for (int j = 0; j < n_cols; ++j) {
      write_all(fd, zeros.data(), offs[j] - pos, path);
      write_all(fd, data[j], lens[j], path);
      pos = offs[j] + lens[j];
    }
    write_all(fd, zeros.data(), (off - pos) % kAlign, path);
  } catch (...) {
    ::close(fd);
    throw;
  }
  if (::close(fd) != 0) throw KcgError(KCG_E_IO, std::string("close failed: ") + path);
}

kcg_columns* columns_open(const char* path) {
  if (!path) throw KcgError(KCG_E_INVALID_ARGUMENT, "null path");
  auto h = std::make_unique<kcg_columns>();
  h->fd = ::open(path, O_RDONLY);
  if (h->fd < 0) throw KcgError(KCG_E_IO, std::string("cannot open ") + path);
  struct stat st;
  if (fstat(h->fd, &st) != 0 || st.st_size < 64) throw KcgError(KCG_E_PARSE, std::string("not a kcg-columns file: ") + path);
  h->map_len = static_cast<size_t>(st.st_size);
  h->map = mmap(nullptr, h->map_len, PROT_READ, MAP_SHARED, h->fd, 0);
  if (h->map == MAP_FAILED) throw KcgError(KCG_E_IO, std::string("mmap failed: ") + path);
  const unsigned char* b = static_cast<const unsigned char*>(h->map);
  uint32_t ver, nc;
  std::memcpy(&ver, b + 8, 4);
  std::memcpy(&nc, b + 12, 4);
  std::memcpy(&h->n_rows, b + 16, 8);
  if (std::memcmp(b, kMagic, 8) != 0 || ver != 1) throw KcgError(KCG_E_PARSE, std::string("not a kcg-columns v1 file: ") + path);
  if (64 + 64 * static_cast<uint64_t>(nc) > h->map_len) throw KcgError(KCG_E_PARSE, "truncated column table");
  for (uint32_t j = 0; j < nc; ++j) {
    const unsigned char* e = b + 64 + 64 * static_cast<size_t>(j);
    kcg_columns::Col c;
    c.name.assign(reinterpret_cast<const char*>(e), strnlen(reinterpret_cast<const char*>(e), 40));
    uint32_t dt;
    std::memcpy(&dt, e + 40, 4);
    c.dtype = static_cast<int>(dt);
    std::memcpy(&c.offset, e + 48, 8);
    std::memcpy(&c.nbytes, e + 56, 8);
    if (c.nbytes != h->n_rows * dtype_size(c.dtype) || c.offset % kAlign || c.offset + c.nbytes > h->map_len)
      throw KcgError(KCG_E_PARSE, "column '" + c.name + "' is inconsistent with the file");
    h->cols.push_back(std::move(c));
  }
  return h.release();
}

void columns_load(kcg_columns* h, int j, uint64_t row0, size_t n, void* dev, void* stream_) {
  if (!h || j < 0 || j >= static_cast<int>(h->cols.size()) || !dev)
    throw KcgError(KCG_E_INVALID_ARGUMENT, "bad kcg_columns_load arguments");
  if (row0 + n > h->n_rows) throw KcgError(KCG_E_INVALID_ARGUMENT, "rows beyond the end of the column");
  const auto& c = h->cols[j];
  const size_t es = dtype_size(c.dtype);
  const char* src = static_cast<const char*>(h->map) + c.offset + row0 * es;
  const size_t bytes = n * es;
  const cudaStream_t stream = static_cast<cudaStream_t>(stream_);
  if (!h->registered) {
    // page-lock the read-only mapping once: DMA straight from the page cache
    h->registered = cudaHostRegister(h->map, h->map_len, cudaHostRegisterReadOnly) == cudaSuccess;
    if (!h->registered) cudaGetLastError();  // clear; fall back to staging
  }
  if (h->registered) {
    if (cudaMemcpyAsync(dev, src, bytes, cudaMemcpyHostToDevice, stream) != cudaSuccess)
      throw KcgError(KCG_E_CUDA, "kcg_columns_load copy failed");
    if (!h->pending) {
      cudaEvent_t ev;
      if (cudaEventCreateWithFlags(&ev, cudaEventDisableTiming) != cudaSuccess)
        throw KcgError(KCG_E_CUDA, "cudaEventCreate failed");
      h->pending = ev;
    }
    // close waits for the last copy (stream-ordered loads complete in order)
    cudaEventRecord(static_cast<cudaEvent_t>(h->pending), stream);
    return;
  }
  // pinned staging ring: memcpy chunk k+1 while chunk k is in flight
  constexpr size_t kChunk = 32u << 20;
  void* ring[2] = {nullptr, nullptr};
  cudaEvent_t ev[2];
  if (cudaMallocHost(&ring[0], kChunk) != cudaSuccess || cudaMallocHost(&ring[1], kChunk) != cudaSuccess)
    throw KcgError(KCG_E_CUDA, "cudaMallocHost failed");
  cudaEventCreateWithFlags(&ev[0], cudaEventDisableTiming);
  cudaEventCreateWithFlags(&ev[1], cudaEventDisableTiming);
  bool used[2] = {false, false};
  int k = 0;
  for (size_t done = 0; done < bytes; done += kChunk, k ^= 1) {
    const size_t len = std::min(kChunk, bytes - done);
    if (used[k]) cudaEventSynchronize(ev[k]);
    std::memcpy(ring[k], src + done, len);
    cudaMemcpyAsync(static_cast<char*>(dev) + done, ring[k], len, cudaMemcpyHostToDevice, stream);
    cudaEventRecord(ev[k], stream);
    used[k] = true;
  }
  const cudaError_t e = cudaStreamSynchronize(stream);
  cudaEventDestroy(ev[0]);
  cudaEventDestroy(ev[1]);
  cudaFreeHost(ring[0]);
  cudaFreeHost(ring[1]);
  if (e != cudaSuccess) throw KcgError(KCG_E_CUDA, std::string("kcg_columns_load: ") + cudaGetErrorString(e));
}

}  // namespace kcg
