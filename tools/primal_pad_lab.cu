// primal_pad_lab.cu -- lab (not product): would renumbering the x-space
// (A's columns = A' rows) by length pay for the primal step?  Config 4's A'
// has Poisson-like rows (mean 20): its sliced ELL, slice-sorted in natural
// order (the product layout), pads to ~1.45x (each slice runs its longest
// row's rounds with the other lanes predicated off).  Renumbered rows (64k
// windows, longest first) pad to ~1.0x.  The loads a predicated lane skips
// cost no memory request, so the question is only issue slots / energy:
// timed sustained at the power cap, interleaved.
//
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 tools/primal_pad_lab.cu -o tools/primal_pad_lab
#include <cuda_runtime.h>

#include <algorithm>
#include <cstdint>
#include <cstdio>
#include <cstdlib>
#include <numeric>
#include <random>
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

constexpr int kMaxLen = 96;

// slot (slice r/32, lane pos[r] % 32) of row perm[r]
__global__ void k_gen(int m, int n, const int* __restrict__ perm, const int* __restrict__ len,
                      const int* __restrict__ lane_of, const long long* __restrict__ sptr, int* col, double* val) {
  const int r = blockIdx.x * blockDim.x + threadIdx.x;
  if (r >= m) return;
  const long long i = perm[r];
  const int L = len[r];
  int c[kMaxLen];
  double v[kMaxLen];
  for (int k = 0; k < L; ++k) {
    const uint64_t h = mix(((uint64_t)i << 8) + k);
    long long cc;
    if ((h & 1023) < 717) cc = i / 2 + (long long)((h >> 10) % 50001) - 25000;
    else cc = (long long)((h >> 10) % (uint64_t)n);
    cc %= n;
    if (cc < 0) cc += n;
    c[k] = (int)cc;
    v[k] = (double)((h >> 40) & 0xffffff) / 8388608.0 - 1.0;
  }
  for (int a = 1; a < L; ++a) {
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
  const long long base = sptr[r >> 5] + lane_of[r];
  for (int k = 0; k < L; ++k) {
    col[base + 32LL * k] = c[k];
    val[base + 32LL * k] = v[k];
  }
}

__global__ void k_fillx(long long n, double* x) {
  const long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x;
  if (i < n) x[i] = (double)(mix(i * 7 + 3) >> 11) / 9007199254740992.0 - 0.5;
}

// lane l of slice s: length lens[32 s + l] (layout order), the product's loop
template <int kU>
__global__ void __launch_bounds__(256, 8) k_sell(int m, int ns, const long long* __restrict__ sptr,
                                                 const int* __restrict__ width, const int* __restrict__ len,
                                                 const int* __restrict__ col, const double* __restrict__ val,
                                                 const double* __restrict__ x, double* __restrict__ y) {
  const long long sl = ((long long)blockIdx.x * 256 + threadIdx.x) >> 5;
  const int lane = threadIdx.x & 31;
  if (sl >= ns) return;
  const long long r = sl * 32 + lane;
  const int L = r < m ? len[r] : 0;
  const int w = width[sl];
  const long long base = sptr[sl] + lane;
  double acc = 0.0;
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
  if (r < m) y[r] = acc;
}

struct Dev {
  int ns;
  long long slots;
  int *len, *width, *col;
  long long* sptr;
  double* val;
};

// order: rows in layout order; slice-sorted: lanes of each slice by length desc
static Dev make(const std::vector<int>& lens, std::vector<int> order, int n) {
  const int m = (int)lens.size();
  Dev d;
  d.ns = (m + 31) / 32;
  std::vector<int> L(m), lane(m), width(d.ns, 0);
  for (int r = 0; r < m; ++r) L[r] = lens[order[r]];
  for (int r = 0; r < m; ++r) width[r / 32] = std::max(width[r / 32], L[r]);
  std::vector<long long> sptr(d.ns + 1, 0);
  for (int s = 0; s < d.ns; ++s) sptr[s + 1] = sptr[s] + 32LL * width[s];
  for (int r = 0; r < m; ++r) lane[r] = r & 31;
  d.slots = sptr[d.ns];
  int *dperm, *dlane;
  CK(cudaMalloc(&dperm, m * 4));
  CK(cudaMalloc(&dlane, m * 4));
  CK(cudaMalloc(&d.len, m * 4));
  CK(cudaMalloc(&d.width, d.ns * 4));
  CK(cudaMalloc(&d.sptr, (d.ns + 1) * 8));
  CK(cudaMalloc(&d.col, d.slots * 4));
  CK(cudaMalloc(&d.val, d.slots * 8));
  CK(cudaMemcpy(dperm, order.data(), m * 4, cudaMemcpyHostToDevice));
  CK(cudaMemcpy(dlane, lane.data(), m * 4, cudaMemcpyHostToDevice));
  CK(cudaMemcpy(d.len, L.data(), m * 4, cudaMemcpyHostToDevice));
  CK(cudaMemcpy(d.width, width.data(), d.ns * 4, cudaMemcpyHostToDevice));
  CK(cudaMemcpy(d.sptr, sptr.data(), (d.ns + 1) * 8, cudaMemcpyHostToDevice));
  CK(cudaMemset(d.col, 0xFF, d.slots * 4));
  k_gen<<<(m + 127) / 128, 128>>>(m, n, dperm, d.len, dlane, d.sptr, d.col, d.val);
  CK(cudaDeviceSynchronize());
  cudaFree(dperm);
  cudaFree(dlane);
  return d;
}

int main(int argc, char** argv) {
  const int m = argc > 1 ? atoi(argv[1]) : 10000000;
  const int n = m / 2;
  std::mt19937_64 rng(5);
  std::poisson_distribution<int> po(20.0);
  std::vector<int> lens(m);
  long long nnz = 0;
  for (int i = 0; i < m; ++i) {
    lens[i] = std::min(kMaxLen, std::max(1, po(rng)));
    nnz += lens[i];
  }
  // natural order, slice-sorted (the product's A' layout)
  std::vector<int> nat(m);
  std::iota(nat.begin(), nat.end(), 0);
  for (int s0 = 0; s0 < m; s0 += 32)
    std::stable_sort(nat.begin() + s0, nat.begin() + std::min(m, s0 + 32), [&](int a, int b) { return lens[a] > lens[b]; });
  // renumbered: windows of 64k, rows longer than 24 first
  std::vector<int> ren(m);
  std::iota(ren.begin(), ren.end(), 0);
  std::stable_sort(ren.begin(), ren.end(), [&](int a, int b) {
    const bool la = lens[a] > 24, lb = lens[b] > 24;
    if (la != lb) return la;
    if (a / 65536 != b / 65536) return a / 65536 < b / 65536;
    return lens[a] > lens[b];
  });
  double *x, *y;
  CK(cudaMalloc(&x, (size_t)n * 8));
  CK(cudaMalloc(&y, (size_t)m * 8));
  k_fillx<<<(n + 255) / 256, 256>>>(n, x);
  Dev A = make(lens, nat, n), B = make(lens, ren, n);
  printf("{\"m\": %d, \"n\": %d, \"nnz\": %lld, \"pad_natural_sorted\": %.3f, \"pad_renumbered\": %.3f}\n", m, n, nnz,
         (double)A.slots / nnz, (double)B.slots / nnz);
  auto run = [&](const Dev& d) {
    const unsigned g = (unsigned)((d.ns * 32LL + 255) / 256);
    k_sell<6><<<g, 256>>>(m, d.ns, d.sptr, d.width, d.len, d.col, d.val, x, y);
  };
  auto blk = [&](const Dev& d, int k) {
    cudaEvent_t a, b;
    cudaEventCreate(&a);
    cudaEventCreate(&b);
    cudaEventRecord(a);
    for (int i = 0; i < k; ++i) run(d);
    cudaEventRecord(b);
    cudaEventSynchronize(b);
    float ms = 0;
    cudaEventElapsedTime(&ms, a, b);
    return ms / k;
  };
  printf("{\"cold\": true, \"natural_sorted_ms\": %.4f, \"renumbered_ms\": %.4f}\n", blk(A, 20), blk(B, 20));
  blk(A, 1500);
  blk(B, 1500);
  for (int r = 0; r < 8; ++r) {
    const float a = blk(A, 200), b = blk(B, 200);
    printf("{\"sustained_round\": %d, \"natural_sorted_ms\": %.4f, \"renumbered_ms\": %.4f}\n", r, a, b);
    fflush(stdout);
  }
  CK(cudaGetLastError());
  return 0;
}
