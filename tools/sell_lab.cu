// sell_lab.cu -- lab (not product): minimal y = A x kernels over the
// engine's own sliced-ELL layouts (DeviceLp._sell), to split the product step
// kernels' time into the gather/stream floor and everything else (epilogue,
// heavy rows, bookkeeping).  Driven by tools/sell_lab.py.
#include <cuda_runtime.h>

#include <cstdint>

namespace {

// kind 0: SpMV only (len per lane from the CSR ptr, as the product does)
// kind 1: SpMV + the dual epilogue's traffic (read b, y, ybar; write y, ybar)
template <int kU, int KIND>
__global__ void __launch_bounds__(256, 6) k_sell(int rows, int nslices, const long long* __restrict__ sptr,
                                                 const int* __restrict__ width, const int* __restrict__ col,
                                                 const double* __restrict__ val, const int* __restrict__ ptr,
                                                 int heavy, const double* __restrict__ x, double* __restrict__ y,
                                                 const double* __restrict__ b, double* __restrict__ v1,
                                                 double* __restrict__ v2) {
  const long long sl = ((long long)blockIdx.x * 256 + threadIdx.x) >> 5;
  const int lane = threadIdx.x & 31;
  if (sl >= nslices) return;
  const long long rl = sl * 32 + lane;
  int len = rl < rows ? ptr[rl + 1] - ptr[rl] : 0;
  if (len > heavy) len = 0;
  const int w = width[sl];
  const long long base = sptr[sl] + lane;
  double acc = 0.0;
  for (int k = 0; k < w; k += kU) {
    double av[kU], xv[kU];
    int jv[kU];
#pragma unroll
    for (int u = 0; u < kU; ++u) {
      const bool on = k + u < len;
      av[u] = on ? __ldcs(val + base + 32LL * (k + u)) : 0.0;
      jv[u] = on ? __ldcs(col + base + 32LL * (k + u)) : -1;
    }
#pragma unroll
    for (int u = 0; u < kU; ++u) xv[u] = jv[u] >= 0 ? __ldg(x + jv[u]) : 0.0;
#pragma unroll
    for (int u = 0; u < kU; ++u)
      if (jv[u] >= 0) acc = fma(av[u], xv[u], acc);
  }
  if (rl < rows) {
    if (KIND == 1) {
      const double bi = b[rl], yi = v1[rl], ai = v2[rl];
      const double yn = yi + 0.5 * (bi - acc);
      v1[rl] = yn;
      v2[rl] = ai + 0.25 * yn;
    } else {
      y[rl] = acc;
    }
  }
}

// kind 2 / 3: unpredicated main rounds of kU up to the warp's shortest row,
// then a tail of kT-entry rounds (predicated) up to the slice width -- fewer
// wasted slots than predicated kU rounds when row lengths are not multiples of kU
template <int kU, int kT>
__global__ void __launch_bounds__(256, 6) k_sell_tail(int rows, int nslices, const long long* __restrict__ sptr,
                                                      const int* __restrict__ width, const int* __restrict__ col,
                                                      const double* __restrict__ val, const int* __restrict__ ptr,
                                                      int heavy, const double* __restrict__ x,
                                                      double* __restrict__ y) {
  const long long sl = ((long long)blockIdx.x * 256 + threadIdx.x) >> 5;
  const int lane = threadIdx.x & 31;
  if (sl >= nslices) return;
  const long long rl = sl * 32 + lane;
  int len = rl < rows ? ptr[rl + 1] - ptr[rl] : 0;
  if (len > heavy) len = 0;
  const int w = width[sl];
  const int wmin = __reduce_min_sync(0xffffffffu, (unsigned)len);
  const long long base = sptr[sl] + lane;
  double acc = 0.0;
  int k = 0;
  for (; k + kU <= wmin; k += kU) {
    double av[kU], xv[kU];
    int jv[kU];
#pragma unroll
    for (int u = 0; u < kU; ++u) {
      av[u] = __ldcs(val + base + 32LL * (k + u));
      jv[u] = __ldcs(col + base + 32LL * (k + u));
    }
#pragma unroll
    for (int u = 0; u < kU; ++u) xv[u] = __ldg(x + jv[u]);
#pragma unroll
    for (int u = 0; u < kU; ++u) acc = fma(av[u], xv[u], acc);
  }
  for (; k < w; k += kT) {
    double av[kT], xv[kT];
    int jv[kT];
#pragma unroll
    for (int u = 0; u < kT; ++u) {
      const bool on = k + u < len;
      av[u] = on ? __ldcs(val + base + 32LL * (k + u)) : 0.0;
      jv[u] = on ? __ldcs(col + base + 32LL * (k + u)) : -1;
    }
#pragma unroll
    for (int u = 0; u < kT; ++u) xv[u] = jv[u] >= 0 ? __ldg(x + jv[u]) : 0.0;
#pragma unroll
    for (int u = 0; u < kT; ++u)
      if (jv[u] >= 0) acc = fma(av[u], xv[u], acc);
  }
  if (rl < rows) y[rl] = acc;
}

}  // namespace

extern "C" int sell_lab_time(int kind, int u, int rows, int nslices, const long long* sptr, const int* width,
                             const int* col, const double* val, const int* ptr, int heavy, const double* x,
                             double* y, const double* b, double* v1, double* v2, int reps, float* ms_out) {
  const unsigned grid = (unsigned)((nslices * 32LL + 255) / 256);
  auto launch = [&]() {
    if (kind == 0 && u == 10) k_sell<10, 0><<<grid, 256>>>(rows, nslices, sptr, width, col, val, ptr, heavy, x, y, b, v1, v2);
    else if (kind == 0 && u == 6) k_sell<6, 0><<<grid, 256>>>(rows, nslices, sptr, width, col, val, ptr, heavy, x, y, b, v1, v2);
    else if (kind == 2) k_sell_tail<10, 2><<<grid, 256>>>(rows, nslices, sptr, width, col, val, ptr, heavy, x, y);
    else if (kind == 3) k_sell_tail<10, 4><<<grid, 256>>>(rows, nslices, sptr, width, col, val, ptr, heavy, x, y);
    else if (kind == 4) k_sell_tail<8, 2><<<grid, 256>>>(rows, nslices, sptr, width, col, val, ptr, heavy, x, y);
    else if (kind == 5) k_sell_tail<6, 2><<<grid, 256>>>(rows, nslices, sptr, width, col, val, ptr, heavy, x, y);
    else if (kind == 1 && u == 10) k_sell<10, 1><<<grid, 256>>>(rows, nslices, sptr, width, col, val, ptr, heavy, x, y, b, v1, v2);
    else k_sell<6, 1><<<grid, 256>>>(rows, nslices, sptr, width, col, val, ptr, heavy, x, y, b, v1, v2);
  };
  launch();
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  cudaEventRecord(e0);
  for (int r = 0; r < reps; ++r) launch();
  cudaEventRecord(e1);
  cudaEventSynchronize(e1);
  float ms = 0.f;
  cudaEventElapsedTime(&ms, e0, e1);
  cudaEventDestroy(e0);
  cudaEventDestroy(e1);
  *ms_out = ms / reps;
  return (int)cudaGetLastError();
}
