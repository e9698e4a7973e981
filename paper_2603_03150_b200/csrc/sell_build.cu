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

// warp per row: copies the row's entries to its slice column
__global__ void k_sell_fill(int rows, const int* __restrict__ ptr, const int* __restrict__ col,
                            const double* __restrict__ val, int heavy, const long long* __restrict__ sptr,
                            int* __restrict__ scol, double* __restrict__ sval) {
  const long long w = ((long long)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  const int lane = threadIdx.x & 31;
  if (w >= rows) return;
  const int r = (int)w;
  const int s = ptr[r], e = ptr[r + 1];
  if (e - s > heavy) return;
  const long long base = sptr[r >> 5] + (r & 31);
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

int pdhg_sell_fill(int32_t rows, const int32_t* ptr, const int32_t* col, const double* val,
                   int32_t heavy_threshold, const int64_t* sptr, int32_t* scol, double* sval,
                   void* stream) {
  if (rows <= 0 || !ptr || !sptr || !scol || !sval) return set_error(PDHG_ERR_ARG, "sell_fill: bad argument");
  cudaStream_t s = (cudaStream_t)stream;
  k_sell_fill<<<(unsigned)(((long long)rows * 32 + 255) / 256), 256, 0, s>>>(
      rows, ptr, col, val, heavy_threshold, reinterpret_cast<const long long*>(sptr), scol, sval);
  SELL_TRY(cudaGetLastError());
  return 0;
}

}  // extern "C"
