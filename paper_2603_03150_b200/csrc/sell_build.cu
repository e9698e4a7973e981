// sell_build.cu -- device construction of the sliced-ELL layout of one operator.
//
// SELL-32: slices of 32 consecutive rows; inside a slice the k-th entry of
// every row is stored contiguously (slot = sptr[slice] + 32*k + lane), so the
// step kernel's warp loads 32 values (256 B) and 32 indices (128 B) per
// instruction and each lane sums its own row sequentially -- no lane
// reductions, no shuffles.  Slots beyond a row's length are never read
// (the kernel predicates on the row length), so padding costs memory, not
// bandwidth.  Heavy rows (longer than heavy_threshold) are left to the
// block-per-row CSR path and do not widen their slice.  Row order is the
// natural one: the epilogue of a slice is the coalesced epilogue of 32
// consecutive rows.  Measured on config 4's A' (rows of ~20 entries):
// 0.75 ms vs 0.90 ms for the CSR-vector SpMV (tools/spmv_lab.cu, v10).
#include "../../include/pdhg_b200.h"

#include <cuda_runtime.h>
#include <cub/cub.cuh>

#include <string>

namespace pdhg_internal {
int set_error(int code, const std::string& msg);
}

namespace {

using pdhg_internal::set_error;

#define SELL_TRY(expr)                                                                     \
  do {                                                                                     \
    cudaError_t e_ = (expr);                                                               \
    if (e_ != cudaSuccess)                                                                 \
      return set_error(PDHG_ERR_CUDA, std::string(#expr) + ": " + cudaGetErrorString(e_)); \
  } while (0)

// slice width = longest light row of the slice; w32 = 32 * width (scanned to sptr)
__global__ void k_sell_width(int rows, const int* __restrict__ ptr, int heavy, int* __restrict__ width,
                             long long* __restrict__ w32) {
  const int ns = (rows + 31) / 32;
  const int sl = blockIdx.x * blockDim.x + threadIdx.x;
  if (sl > ns) return;
  if (sl == ns) {
    w32[ns] = 0;
    return;
  }
  int w = 0;
  const int r1 = min(rows, sl * 32 + 32);
  for (int r = sl * 32; r < r1; ++r) {
    const int len = ptr[r + 1] - ptr[r];
    if (len <= heavy && len > w) w = len;
  }
  width[sl] = w;
  w32[sl] = 32LL * w;
}

// thread per slice: order the slice's rows by light length, descending
// (stable; heavy rows count as empty), so the lanes still active in round k
// are a prefix and every fetched sector is full.  perm[lane] = row offset,
// inv[row offset] = lane.
__global__ void k_sell_sort(int rows, const int* __restrict__ ptr, int heavy, unsigned char* __restrict__ perm,
                            unsigned char* __restrict__ inv) {
  const int sl = blockIdx.x * blockDim.x + threadIdx.x;
  if (sl >= (rows + 31) / 32) return;
  int len[32];
  unsigned char idx[32];
  for (int q = 0; q < 32; ++q) {
    const long long r = (long long)sl * 32 + q;
    int l = -1;  // rows past the end sort last
    if (r < rows) {
      l = ptr[r + 1] - ptr[r];
      if (l > heavy) l = 0;
    }
    len[q] = l;
    idx[q] = (unsigned char)q;
  }
  for (int a = 1; a < 32; ++a) {  // insertion sort, stable, descending
    const int lv = len[a];
    const unsigned char iv = idx[a];
    int b = a - 1;
    while (b >= 0 && len[b] < lv) {
      len[b + 1] = len[b];
      idx[b + 1] = idx[b];
      --b;
    }
    len[b + 1] = lv;
    idx[b + 1] = iv;
  }
  for (int q = 0; q < 32; ++q) {
    perm[(size_t)sl * 32 + q] = idx[q];
    inv[(size_t)sl * 32 + idx[q]] = (unsigned char)q;
  }
}

// warp per row: copies the row's entries to its slice column (lane inv[r] when sorted)
__global__ void k_sell_fill(int rows, const int* __restrict__ ptr, const int* __restrict__ col,
                            const double* __restrict__ val, int heavy, const long long* __restrict__ sptr,
                            const unsigned char* __restrict__ inv, int* __restrict__ scol,
                            double* __restrict__ sval) {
  const long long w = ((long long)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  const int lane = threadIdx.x & 31;
  if (w >= rows) return;
  const int r = (int)w;
  const int s = ptr[r], e = ptr[r + 1];
  if (e - s > heavy) return;
  const long long base = sptr[r >> 5] + (inv ? inv[r] : (r & 31));
  for (int k = lane; k < e - s; k += 32) {
    scol[base + 32LL * k] = col[s + k];
    sval[base + 32LL * k] = val[s + k];
  }
}

size_t cub_bytes(int len) {
  size_t b = 0;
  cub::DeviceScan::ExclusiveSum(nullptr, b, (long long*)nullptr, (long long*)nullptr, len);
  return b;
}

}  // namespace

extern "C" {

size_t pdhg_sell_tmp_bytes(int32_t rows) { return rows < 0 ? 0 : cub_bytes(rows / 32 + 2) + 256; }

int pdhg_sell_plan(int32_t rows, const int32_t* ptr, int32_t heavy_threshold, int32_t* width,
                   int64_t* sptr, void* tmp, size_t tmp_bytes, void* stream, int64_t* slots_out) {
  if (rows <= 0 || !ptr || !width || !sptr || !tmp || !slots_out)
    return set_error(PDHG_ERR_ARG, "sell_plan: bad argument");
  if (tmp_bytes < pdhg_sell_tmp_bytes(rows)) return set_error(PDHG_ERR_ARG, "sell_plan: tmp too small");
  cudaStream_t s = (cudaStream_t)stream;
  const int ns = (rows + 31) / 32;
  long long* w32 = reinterpret_cast<long long*>(sptr);
  k_sell_width<<<(ns + 256) / 256, 256, 0, s>>>(rows, ptr, heavy_threshold, width, w32);
  size_t b = tmp_bytes;
  SELL_TRY(cub::DeviceScan::ExclusiveSum(tmp, b, w32, w32, ns + 1, s));
  long long tot = 0;
  SELL_TRY(cudaMemcpyAsync(&tot, w32 + ns, 8, cudaMemcpyDeviceToHost, s));
  SELL_TRY(cudaStreamSynchronize(s));
  SELL_TRY(cudaGetLastError());
  *slots_out = tot;
  return 0;
}

int pdhg_sell_sort(int32_t rows, const int32_t* ptr, int32_t heavy_threshold, uint8_t* perm, uint8_t* inv,
                   void* stream) {
  if (rows <= 0 || !ptr || !perm || !inv) return set_error(PDHG_ERR_ARG, "sell_sort: bad argument");
  const int ns = (rows + 31) / 32;
  k_sell_sort<<<(ns + 127) / 128, 128, 0, (cudaStream_t)stream>>>(rows, ptr, heavy_threshold, perm, inv);
  SELL_TRY(cudaGetLastError());
  return 0;
}

int pdhg_sell_fill(int32_t rows, const int32_t* ptr, const int32_t* col, const double* val,
                   int32_t heavy_threshold, const int64_t* sptr, const uint8_t* inv, int32_t* scol,
                   double* sval, void* stream) {
  if (rows <= 0 || !ptr || !sptr || !scol || !sval) return set_error(PDHG_ERR_ARG, "sell_fill: bad argument");
  cudaStream_t s = (cudaStream_t)stream;
  k_sell_fill<<<(unsigned)(((long long)rows * 32 + 255) / 256), 256, 0, s>>>(
      rows, ptr, col, val, heavy_threshold, reinterpret_cast<const long long*>(sptr), inv, scol, sval);
  SELL_TRY(cudaGetLastError());
  return 0;
}

}  // extern "C"
