// split_lab.cu -- lab (not product): a column-split dual step.  y = A x with
// x = 80 MB (config 4's xe) in one pass, against two passes over the column
// halves (pass 0: entries with column < n/2 -> per-row partial; pass 1: the
// rest, starting from the partial), each pass gathering from a 40 MB half
// that L2 keeps.  Sustained at the power cap, interleaved.
//
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 tools/split_lab.cu -o tools/split_lab
#include <cuda_runtime.h>

#include <algorithm>
#include <cmath>
#include <cstdint>
#include <cstdio>
#include <cstdlib>
#include <vector>

#define CK(x)                                                                            \
  do {                                                                                   \
    cudaError_t e_ = (x);                                                                \
    if (e_ != cudaSuccess) {                                                             \
      fprintf(stderr, "%s:%d %s: %s\n", __FILE__, __LINE__, #x, cudaGetErrorString(e_)); \
      exit(1);                                                                           \
    }                                                                                    \
  } while (0)

__device__ __forceinline__ uint64_t mix(uint64_t z) {
  z += 0x9e3779b97f4a7c15ULL;
  z = (z ^ (z >> 30)) * 0xbf58476d1ce4e5b9ULL;
  z = (z ^ (z >> 27)) * 0x94d049bb133111ebULL;
  return z ^ (z >> 31);
}

constexpr int W = 40;

__device__ void row_entries(long long i, int n, int* c, double* v) {
  for (int k = 0; k < W; ++k) {
    const uint64_t h = mix(((uint64_t)i << 8) + k);
    long long cc;
    if ((h & 1023) < 717) cc = 2 * i + (long long)((h >> 10) % 100001) - 50000;
    else cc = (long long)((h >> 10) % (uint64_t)n);
    cc %= n;
    if (cc < 0) cc += n;
    c[k] = (int)cc;
    v[k] = (double)((h >> 40) & 0xffffff) / 8388608.0 - 1.0;
  }
  for (int a = 1; a < W; ++a) {
    int cj = c[a];
    double vj = v[a];
    int b = a - 1;
    while (b >= 0 && c[b] > cj) {
      c[b + 1] = c[b];
      v[b + 1] = v[b];
      --b;
    }
    c[b + 1] = cj;
    v[b + 1] = vj;
  }
}

__global__ void k_count(int m, int n, int* len0) {
  const long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= m) return;
  int c[W];
  double v[W];
  row_entries(i, n, c, v);
  int h = 0;
  for (int k = 0; k < W; ++k) h += c[k] < n / 2;
  len0[i] = h;
}

__global__ void k_fill(int m, int n, int* col, double* val, const long long* sp0, const long long* sp1, int* col0,
                       double* val0, int* col1, double* val1) {
  const long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= m) return;
  int c[W];
  double v[W];
  row_entries(i, n, c, v);
  const long long s = i >> 5, l = i & 31;
  for (int k = 0; k < W; ++k) {
    col[s * 32 * W + 32LL * k + l] = c[k];
    val[s * 32 * W + 32LL * k + l] = v[k];
  }
  int k0 = 0, k1 = 0;
  for (int k = 0; k < W; ++k) {
    if (c[k] < n / 2) {
      col0[sp0[s] + 32LL * k0 + l] = c[k];
      val0[sp0[s] + 32LL * k0 + l] = v[k];
      ++k0;
    } else {
      col1[sp1[s] + 32LL * k1 + l] = c[k];
      val1[sp1[s] + 32LL * k1 + l] = v[k];
      ++k1;
    }
  }
}

// per-half renumbered layouts: slot s of part p holds row order_p[s]
__global__ void k_fill_part(int m, int n, int part, const int* __restrict__ order, const long long* __restrict__ sp,
                            int* colp, double* valp) {
  const long long s = (long long)blockIdx.x * blockDim.x + threadIdx.x;
  if (s >= m) return;
  const long long i = order[s];
  int c[W];
  double v[W];
  row_entries(i, n, c, v);
  const long long sl = s >> 5, l = s & 31;
  int k2 = 0;
  for (int k = 0; k < W; ++k) {
    if ((c[k] < n / 2) == (part == 0)) {
      colp[sp[sl] + 32LL * k2 + l] = c[k];
      valp[sp[sl] + 32LL * k2 + l] = v[k];
      ++k2;
    }
  }
}

template <int kU, bool FIRST>
__global__ void __launch_bounds__(256, 6) k_part_map(int m, const long long* __restrict__ sp,
                                                     const int* __restrict__ wid, const int* __restrict__ len,
                                                     const int* __restrict__ col, const double* __restrict__ val,
                                                     const double* __restrict__ x, const int* __restrict__ map0,
                                                     double* __restrict__ partial, double* __restrict__ y) {
  const long long sl = ((long long)blockIdx.x * 256 + threadIdx.x) >> 5;
  const int lane = threadIdx.x & 31;
  if (sl * 32 >= m) return;
  const long long r = sl * 32 + lane;
  const int L = len[r];
  const int w = wid[sl];
  const long long base = sp[sl] + lane;
  double acc = FIRST ? 0.0 : __ldcs(partial + r);
  for (int k = 0; k < w; k += kU) {
    double av[kU], xv[kU];
    int jv[kU];
#pragma unroll
    for (int u = 0; u < kU; ++u) {
      const bool on = k + u < L;
      av[u] = on ? __ldcs(val + base + 32LL * (k + u)) : 0.0;
      jv[u] = on ? __ldcs(col + base + 32LL * (k + u)) : -1;
    }
#pragma unroll
    for (int u = 0; u < kU; ++u) xv[u] = jv[u] >= 0 ? __ldg(x + jv[u]) : 0.0;
#pragma unroll
    for (int u = 0; u < kU; ++u)
      if (jv[u] >= 0) acc = fma(av[u], xv[u], acc);
  }
  if (FIRST) partial[map0[r]] = acc;   // scattered: the pass-1 slot of this row
  else y[r] = acc;
}

__global__ void k_fillx(long long n, double* x) {
  const long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x;
  if (i < n) x[i] = (double)(mix(i * 7 + 3) >> 11) / 9007199254740992.0 - 0.5;
}

template <int kU>
__global__ void __launch_bounds__(256, 6) k_one(int m, const int* __restrict__ col, const double* __restrict__ val,
                                                const double* __restrict__ x, double* __restrict__ y) {
  const long long sl = ((long long)blockIdx.x * 256 + threadIdx.x) >> 5;
  const int lane = threadIdx.x & 31;
  if (sl * 32 >= m) return;
  const long long base = sl * 32 * W + lane;
  double acc = 0.0;
  for (int k = 0; k < W; k += kU) {
    double av[kU], xv[kU];
    int jv[kU];
#pragma unroll
    for (int u = 0; u < kU; ++u) {
      const bool on = k + u < W;
      av[u] = on ? __ldcs(val + base + 32LL * (k + u)) : 0.0;
      jv[u] = on ? __ldcs(col + base + 32LL * (k + u)) : -1;
    }
#pragma unroll
    for (int u = 0; u < kU; ++u) xv[u] = jv[u] >= 0 ? __ldg(x + jv[u]) : 0.0;
#pragma unroll
    for (int u = 0; u < kU; ++u)
      if (jv[u] >= 0) acc = fma(av[u], xv[u], acc);
  }
  y[sl * 32 + lane] = acc;
}

// one pass over a part: slice widths wid[], lengths len[] (part lengths per row)
template <int kU, bool FIRST>
__global__ void __launch_bounds__(256, 6) k_part(int m, const long long* __restrict__ sp, const int* __restrict__ wid,
                                                 const int* __restrict__ len, const int* __restrict__ col,
                                                 const double* __restrict__ val, const double* __restrict__ x,
                                                 double* __restrict__ partial, double* __restrict__ y) {
  const long long sl = ((long long)blockIdx.x * 256 + threadIdx.x) >> 5;
  const int lane = threadIdx.x & 31;
  if (sl * 32 >= m) return;
  const long long r = sl * 32 + lane;
  const int L = len[r];
  const int w = wid[sl];
  const long long base = sp[sl] + lane;
  double acc = FIRST ? 0.0 : __ldcs(partial + r);
  for (int k = 0; k < w; k += kU) {
    double av[kU], xv[kU];
    int jv[kU];
#pragma unroll
    for (int u = 0; u < kU; ++u) {
      const bool on = k + u < L;
      av[u] = on ? __ldcs(val + base + 32LL * (k + u)) : 0.0;
      jv[u] = on ? __ldcs(col + base + 32LL * (k + u)) : -1;
    }
#pragma unroll
    for (int u = 0; u < kU; ++u) xv[u] = jv[u] >= 0 ? __ldg(x + jv[u]) : 0.0;
#pragma unroll
    for (int u = 0; u < kU; ++u)
      if (jv[u] >= 0) acc = fma(av[u], xv[u], acc);
  }
  if (FIRST) __stcs(partial + r, acc);
  else y[r] = acc;
}

int main(int argc, char** argv) {
  const int m = argc > 1 ? atoi(argv[1]) : 5000000;
  const long long n = 2LL * m;
  const long long nnz = (long long)m * W;
  const int ns = m / 32;
  int* len0;
  CK(cudaMalloc(&len0, m * 4));
  k_count<<<(m + 127) / 128, 128>>>(m, (int)n, len0);
  std::vector<int> L0(m), L1(m), w0(ns), w1(ns);
  CK(cudaMemcpy(L0.data(), len0, m * 4, cudaMemcpyDeviceToHost));
  for (int i = 0; i < m; ++i) L1[i] = W - L0[i];
  std::vector<long long> sp0(ns + 1, 0), sp1(ns + 1, 0);
  for (int s = 0; s < ns; ++s) {
    int a = 0, b = 0;
    for (int l = 0; l < 32; ++l) {
      a = std::max(a, L0[s * 32 + l]);
      b = std::max(b, L1[s * 32 + l]);
    }
    w0[s] = a;
    w1[s] = b;
    sp0[s + 1] = sp0[s] + 32LL * a;
    sp1[s + 1] = sp1[s] + 32LL * b;
  }
  int *col, *col0, *col1, *dlen1, *dw0, *dw1;
  double *val, *val0, *val1, *x, *y0, *y1, *partial;
  long long *dsp0, *dsp1;
  CK(cudaMalloc(&col, nnz * 4));
  CK(cudaMalloc(&val, nnz * 8));
  CK(cudaMalloc(&col0, sp0[ns] * 4));
  CK(cudaMalloc(&val0, sp0[ns] * 8));
  CK(cudaMalloc(&col1, sp1[ns] * 4));
  CK(cudaMalloc(&val1, sp1[ns] * 8));
  CK(cudaMalloc(&dlen1, m * 4));
  CK(cudaMalloc(&dw0, ns * 4));
  CK(cudaMalloc(&dw1, ns * 4));
  CK(cudaMalloc(&dsp0, (ns + 1) * 8));
  CK(cudaMalloc(&dsp1, (ns + 1) * 8));
  CK(cudaMalloc(&x, n * 8));
  CK(cudaMalloc(&y0, (size_t)m * 8));
  CK(cudaMalloc(&y1, (size_t)m * 8));
  CK(cudaMalloc(&partial, (size_t)m * 8));
  CK(cudaMemcpy(dlen1, L1.data(), m * 4, cudaMemcpyHostToDevice));
  CK(cudaMemcpy(dw0, w0.data(), ns * 4, cudaMemcpyHostToDevice));
  CK(cudaMemcpy(dw1, w1.data(), ns * 4, cudaMemcpyHostToDevice));
  CK(cudaMemcpy(dsp0, sp0.data(), (ns + 1) * 8, cudaMemcpyHostToDevice));
  CK(cudaMemcpy(dsp1, sp1.data(), (ns + 1) * 8, cudaMemcpyHostToDevice));
  k_fill<<<(m + 127) / 128, 128>>>(m, (int)n, col, val, dsp0, dsp1, col0, val0, col1, val1);
  k_fillx<<<(unsigned)((n + 255) / 256), 256>>>(n, x);
  CK(cudaDeviceSynchronize());
  const unsigned g = (unsigned)((ns * 32LL + 255) / 256);
  auto one = [&] { k_one<10><<<g, 256>>>(m, col, val, x, y0); };
  auto two = [&] {
    k_part<10, true><<<g, 256>>>(m, dsp0, dw0, len0, col0, val0, x, partial, y1);
    k_part<10, false><<<g, 256>>>(m, dsp1, dw1, dlen1, col1, val1, x, partial, y1);
  };
  auto blk = [&](auto f, int k) {
    cudaEvent_t a, b;
    cudaEventCreate(&a);
    cudaEventCreate(&b);
    cudaEventRecord(a);
    for (int i = 0; i < k; ++i) f();
    cudaEventRecord(b);
    cudaEventSynchronize(b);
    float ms = 0;
    cudaEventElapsedTime(&ms, a, b);
    return ms / k;
  };
  one();
  two();
  CK(cudaDeviceSynchronize());
  std::vector<double> h0(m), h1(m);
  CK(cudaMemcpy(h0.data(), y0, m * 8, cudaMemcpyDeviceToHost));
  CK(cudaMemcpy(h1.data(), y1, m * 8, cudaMemcpyDeviceToHost));
  double err = 0, mx = 0;
  for (int i = 0; i < m; ++i) {
    err = std::max(err, std::fabs(h0[i] - h1[i]));
    mx = std::max(mx, std::fabs(h0[i]));
  }
  // ---- per-half renumbered: order_p = rows by decreasing part length in 16k windows
  auto order_by = [&](const std::vector<int>& L) {
    std::vector<int> o(m);
    for (int i = 0; i < m; ++i) o[i] = i;
    for (int w0 = 0; w0 < m; w0 += 16384)
      std::stable_sort(o.begin() + w0, o.begin() + std::min(m, w0 + 16384), [&](int a, int b) { return L[a] > L[b]; });
    return o;
  };
  std::vector<int> o0 = order_by(L0), o1 = order_by(L1), inv1(m), map0(m), lo0(m), lo1(m);
  for (int s2 = 0; s2 < m; ++s2) inv1[o1[s2]] = s2;
  for (int s2 = 0; s2 < m; ++s2) {
    map0[s2] = inv1[o0[s2]];
    lo0[s2] = L0[o0[s2]];
    lo1[s2] = L1[o1[s2]];
  }
  std::vector<int> rw0(ns), rw1(ns);
  std::vector<long long> rsp0(ns + 1, 0), rsp1(ns + 1, 0);
  for (int s2 = 0; s2 < ns; ++s2) {
    int a = 0, b = 0;
    for (int l = 0; l < 32; ++l) {
      a = std::max(a, lo0[s2 * 32 + l]);
      b = std::max(b, lo1[s2 * 32 + l]);
    }
    rw0[s2] = a;
    rw1[s2] = b;
    rsp0[s2 + 1] = rsp0[s2] + 32LL * a;
    rsp1[s2 + 1] = rsp1[s2] + 32LL * b;
  }
  int *do0, *do1, *dmap0, *dlo0, *dlo1, *drw0, *drw1, *rcol0, *rcol1;
  long long *drsp0, *drsp1;
  double *rval0, *rval1, *y2;
  CK(cudaMalloc(&do0, m * 4));
  CK(cudaMalloc(&do1, m * 4));
  CK(cudaMalloc(&dmap0, m * 4));
  CK(cudaMalloc(&dlo0, m * 4));
  CK(cudaMalloc(&dlo1, m * 4));
  CK(cudaMalloc(&drw0, ns * 4));
  CK(cudaMalloc(&drw1, ns * 4));
  CK(cudaMalloc(&drsp0, (ns + 1) * 8));
  CK(cudaMalloc(&drsp1, (ns + 1) * 8));
  CK(cudaMalloc(&rcol0, rsp0[ns] * 4));
  CK(cudaMalloc(&rval0, rsp0[ns] * 8));
  CK(cudaMalloc(&rcol1, rsp1[ns] * 4));
  CK(cudaMalloc(&rval1, rsp1[ns] * 8));
  CK(cudaMalloc(&y2, (size_t)m * 8));
  CK(cudaMemcpy(do0, o0.data(), m * 4, cudaMemcpyHostToDevice));
  CK(cudaMemcpy(do1, o1.data(), m * 4, cudaMemcpyHostToDevice));
  CK(cudaMemcpy(dmap0, map0.data(), m * 4, cudaMemcpyHostToDevice));
  CK(cudaMemcpy(dlo0, lo0.data(), m * 4, cudaMemcpyHostToDevice));
  CK(cudaMemcpy(dlo1, lo1.data(), m * 4, cudaMemcpyHostToDevice));
  CK(cudaMemcpy(drw0, rw0.data(), ns * 4, cudaMemcpyHostToDevice));
  CK(cudaMemcpy(drw1, rw1.data(), ns * 4, cudaMemcpyHostToDevice));
  CK(cudaMemcpy(drsp0, rsp0.data(), (ns + 1) * 8, cudaMemcpyHostToDevice));
  CK(cudaMemcpy(drsp1, rsp1.data(), (ns + 1) * 8, cudaMemcpyHostToDevice));
  k_fill_part<<<(m + 127) / 128, 128>>>(m, (int)n, 0, do0, drsp0, rcol0, rval0);
  k_fill_part<<<(m + 127) / 128, 128>>>(m, (int)n, 1, do1, drsp1, rcol1, rval1);
  CK(cudaDeviceSynchronize());
  auto two_r = [&] {
    k_part_map<10, true><<<g, 256>>>(m, drsp0, drw0, dlo0, rcol0, rval0, x, dmap0, partial, y2);
    k_part_map<10, false><<<g, 256>>>(m, drsp1, drw1, dlo1, rcol1, rval1, x, dmap0, partial, y2);
  };
  two_r();
  CK(cudaDeviceSynchronize());
  {
    std::vector<double> h2(m);
    CK(cudaMemcpy(h2.data(), y2, m * 8, cudaMemcpyDeviceToHost));
    double e2 = 0;
    for (int s2 = 0; s2 < m; ++s2) e2 = std::max(e2, std::fabs(h2[s2] - h0[o1[s2]]));
    long long a0 = 0, a1 = 0;
    for (int i = 0; i < m; ++i) { a0 += L0[i]; a1 += L1[i]; }
    printf("{\"renumbered_parts\": true, \"pad_part0\": %.3f, \"pad_part1\": %.3f, \"max_rel_diff\": %.2e}\n",
           (double)rsp0[ns] / a0, (double)rsp1[ns] / a1, e2 / mx);
  }
  long long e0 = 0, e1 = 0;
  for (int i = 0; i < m; ++i) {
    e0 += L0[i];
    e1 += L1[i];
  }
  printf("{\"nnz\": %lld, \"part0_entries\": %lld, \"pad_part0\": %.3f, \"pad_part1\": %.3f, \"max_rel_diff\": %.2e}\n",
         nnz, e0, (double)sp0[ns] / e0, (double)sp1[ns] / e1, err / mx);
  printf("{\"cold\": true, \"one_pass_ms\": %.4f, \"two_pass_ms\": %.4f, \"two_pass_renumbered_ms\": %.4f}\n",
         blk(one, 20), blk(two, 20), blk(two_r, 20));
  blk(one, 2500);
  for (int r = 0; r < 8; ++r) {
    const float a1 = blk(one, 200), a2 = blk(two, 200), a3 = blk(two_r, 200);
    printf("{\"sustained_round\": %d, \"one_pass_ms\": %.4f, \"two_pass_ms\": %.4f, \"two_pass_renumbered_ms\": %.4f}\n",
           r, a1, a2, a3);
    fflush(stdout);
  }
  CK(cudaGetLastError());
  return 0;
}
