// rowlen_lab.cu -- lab (not product): how much of the sliced-ELL dual step's
// time on config 4 comes from the lognormal row lengths?  Same column
// pattern as tools/gather4_lab.cu (70 % within +-50k of column 2i, 30 %
// uniform, sorted per row), m = 5M rows, n = 10M, y = A x only, the product's
// row loop (10 entries in flight per lane, predicated on the row length):
//
//   uniform   : every row 40 entries
//   lognormal : lengths lognormal (mean 40, sigma 0.8, clipped to [1, 512]),
//               rows renumbered by decreasing length inside 64k-row windows
//               (GpuOptions.row_order), slice width = its longest row
//   lognormal, global : renumbered by length over all rows (one window)
//   lognormal, natural: no renumbering (slices padded to their longest row)
//
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 tools/rowlen_lab.cu -o tools/rowlen_lab
//   tools/rowlen_lab [m] [reps] [multi-slice 0/1] [case mask] [flat 0/1]
#include <cuda_runtime.h>

#include <algorithm>
#include <cmath>
#include <cstdint>
#include <cstdio>
#include <cstdlib>
#include <cstring>
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

constexpr int kMaxLen = 512;

// new row r (original row perm[r], len[r] entries) -> slice r/32, lane r%32
__global__ void k_gen(int m, int n, const int* __restrict__ perm, const int* __restrict__ len,
                      const long long* __restrict__ sptr, int* col, double* val) {
  const int r = blockIdx.x * blockDim.x + threadIdx.x;
  if (r >= m) return;
  const long long i = perm[r];
  const int L = len[r];
  int c[kMaxLen];
  double v[kMaxLen];
  for (int k = 0; k < L; ++k) {
    const uint64_t h = mix(((uint64_t)i << 10) + k);
    long long cc;
    if ((h & 1023) < 717) cc = 2 * i + (long long)((h >> 10) % 100001) - 50000;
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
  const long long base = sptr[r >> 5] + (r & 31);
  for (int k = 0; k < L; ++k) {
    col[base + 32LL * k] = c[k];
    val[base + 32LL * k] = v[k];
  }
}

__global__ void k_fillx(long long n, double* x) {
  const long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x;
  if (i < n) x[i] = (double)(mix(i * 7 + 3) >> 11) / 9007199254740992.0 - 0.5;
}

template <int kU>
__global__ void __launch_bounds__(256, 6) k_sell(int m, int ns, const long long* __restrict__ sptr,
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

// NS consecutive slices per warp, rounds interleaved: lane l sums rows
// 32*s_j + l (j < NS) side by side, each in its own entry order (bitwise the
// one-slice loop), with NS*kU entries in flight per lane
template <int kU, int NS, int MINB>
__global__ void __launch_bounds__(256, MINB) k_sell_multi(int m, int ns, const long long* __restrict__ sptr,
                                                        const int* __restrict__ width, const int* __restrict__ len,
                                                        const int* __restrict__ col, const double* __restrict__ val,
                                                        const double* __restrict__ x, double* __restrict__ y) {
  const long long w0 = (((long long)blockIdx.x * 256 + threadIdx.x) >> 5) * NS;
  const int lane = threadIdx.x & 31;
  if (w0 >= ns) return;
  int L[NS];
  long long base[NS];
  int W = 0;
#pragma unroll
  for (int j = 0; j < NS; ++j) {
    const long long sl = w0 + j;
    const long long r = sl * 32 + lane;
    L[j] = (sl < ns && r < m) ? len[r] : 0;
    base[j] = sl < ns ? sptr[sl] + lane : 0;
    W = max(W, sl < ns ? width[sl] : 0);
  }
  double acc[NS];
#pragma unroll
  for (int j = 0; j < NS; ++j) acc[j] = 0.0;
  for (int k = 0; k < W; k += kU) {
    double av[NS][kU], xv[NS][kU];
    int jv[NS][kU];
#pragma unroll
    for (int j = 0; j < NS; ++j)
#pragma unroll
      for (int u = 0; u < kU; ++u) {
        const bool on = k + u < L[j];
        av[j][u] = on ? __ldcs(val + base[j] + 32LL * (k + u)) : 0.0;
        jv[j][u] = on ? __ldcs(col + base[j] + 32LL * (k + u)) : -1;
      }
#pragma unroll
    for (int j = 0; j < NS; ++j)
#pragma unroll
      for (int u = 0; u < kU; ++u) xv[j][u] = jv[j][u] >= 0 ? __ldg(x + jv[j][u]) : 0.0;
#pragma unroll
    for (int j = 0; j < NS; ++j)
#pragma unroll
      for (int u = 0; u < kU; ++u)
        if (jv[j][u] >= 0) acc[j] = fma(av[j][u], xv[j][u], acc[j]);
  }
#pragma unroll
  for (int j = 0; j < NS; ++j) {
    const long long r = (w0 + j) * 32 + lane;
    if (w0 + j < ns && r < m) y[r] = acc[j];
  }
}

// Rounds that span slices: a warp walks NSW consecutive slices as one
// contiguous run of 32-lane columns (the SELL layout stores them back to
// back), kU columns per round whatever slice they belong to; a padding slot
// has col = -1; when a slice ends inside a round the lane stores its row and
// starts the next (warp-uniform branch).  Each row is still summed
// sequentially in its own entry order (bitwise the one-slice loop).
template <int kU, int NSW, int MINB = 6>
__global__ void __launch_bounds__(256, MINB) k_flat(int m, int ns, const long long* __restrict__ sptr,
                                                 const int* __restrict__ width, const int* __restrict__ col,
                                                 const double* __restrict__ val, const double* __restrict__ x,
                                                 double* __restrict__ y) {
  const long long s0 = (((long long)blockIdx.x * 256 + threadIdx.x) >> 5) * NSW;
  const int lane = threadIdx.x & 31;
  if (s0 >= ns) return;
  const int nsl = (int)min((long long)NSW, ns - s0);
  // lane j holds the width of slice s0 + j
  const int wj = lane < nsl ? width[s0 + lane] : 0;
  const long long q0 = sptr[s0] + lane;  // lane's slot of column 0
  int Q = 0;
#pragma unroll
  for (int j = 0; j < NSW; ++j) Q += __shfl_sync(0xffffffffu, wj, j);
  int j = 0;                                     // current slice (warp-uniform)
  int end = __shfl_sync(0xffffffffu, wj, 0);     // column where it ends
  double acc = 0.0;
  for (int q = 0; q < Q; q += kU) {
    double av[kU], xv[kU];
    int jv[kU];
#pragma unroll
    for (int u = 0; u < kU; ++u) {
      const bool on = q + u < Q;
      av[u] = on ? __ldcs(val + q0 + 32LL * (q + u)) : 0.0;
      jv[u] = on ? __ldcs(col + q0 + 32LL * (q + u)) : -1;
    }
#pragma unroll
    for (int u = 0; u < kU; ++u) xv[u] = jv[u] >= 0 ? __ldg(x + jv[u]) : 0.0;
#pragma unroll
    for (int u = 0; u < kU; ++u) {
      if (jv[u] >= 0) acc = fma(av[u], xv[u], acc);
      if (q + u + 1 == end) {     // slice j ends after this column (widths >= 1)
        const long long r = (s0 + j) * 32 + lane;
        if (r < m) y[r] = acc;
        acc = 0.0;
        ++j;
        end += __shfl_sync(0xffffffffu, wj, j & 31);
      }
    }
  }
}

// rows longer than T run warp-per-row (a CSR list, first blocks of the
// launch: kU-entry rounds per lane, butterfly at the end) -- the product's
// "medium" tier of the CSR step kernel -- and the sliced ELL holds the rest
__global__ void k_gen_csr(int nmed, int n, const int* __restrict__ rows, const int* __restrict__ ptr, int* col,
                          double* val) {
  const int w = blockIdx.x * blockDim.x + threadIdx.x;
  if (w >= nmed) return;
  const long long i = rows[w];
  const int s0 = ptr[w], L = ptr[w + 1] - s0;
  int c[kMaxLen];
  double v[kMaxLen];
  for (int k = 0; k < L; ++k) {
    const uint64_t h = mix(((uint64_t)i << 10) + k);
    long long cc;
    if ((h & 1023) < 717) cc = 2 * i + (long long)((h >> 10) % 100001) - 50000;
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
  for (int k = 0; k < L; ++k) {
    col[s0 + k] = c[k];
    val[s0 + k] = v[k];
  }
}

template <int kU, int kUM>
__global__ void __launch_bounds__(256, 6) k_sell_med(int m, int ns, const long long* __restrict__ sptr,
                                                     const int* __restrict__ width, const int* __restrict__ len,
                                                     const int* __restrict__ col, const double* __restrict__ val,
                                                     int nmed, int nmb, const int* __restrict__ mrow,
                                                     const int* __restrict__ mptr, const int* __restrict__ mcol,
                                                     const double* __restrict__ mval, const double* __restrict__ x,
                                                     double* __restrict__ y, double* __restrict__ ymed) {
  const int lane = threadIdx.x & 31;
  if ((int)blockIdx.x < nmb) {
    const int w = blockIdx.x * 8 + (threadIdx.x >> 5);
    if (w >= nmed) return;
    const int s0 = mptr[w], e = mptr[w + 1];
    double acc = 0.0;
    for (int k = s0 + lane; k < e; k += 32 * kUM) {
      double av[kUM], xv[kUM];
      int jv[kUM];
#pragma unroll
      for (int u = 0; u < kUM; ++u) {
        const int kk = k + 32 * u;
        av[u] = kk < e ? __ldcs(mval + kk) : 0.0;
        jv[u] = kk < e ? __ldcs(mcol + kk) : -1;
      }
#pragma unroll
      for (int u = 0; u < kUM; ++u) xv[u] = jv[u] >= 0 ? __ldg(x + jv[u]) : 0.0;
#pragma unroll
      for (int u = 0; u < kUM; ++u)
        if (jv[u] >= 0) acc = fma(av[u], xv[u], acc);
    }
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) acc += __shfl_xor_sync(0xffffffffu, acc, o);
    if (lane == 0) ymed[w] = acc;
    return;
  }
  const long long sl = ((long long)(blockIdx.x - nmb) * 256 + threadIdx.x) >> 5;
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

struct Layout {
  int m, ns;
  std::vector<int> perm, len, width;
  std::vector<long long> sptr;
  long long slots;
};

static uint64_t hmix(uint64_t z) {
  z += 0x9e3779b97f4a7c15ULL;
  z = (z ^ (z >> 30)) * 0xbf58476d1ce4e5b9ULL;
  z = (z ^ (z >> 27)) * 0x94d049bb133111ebULL;
  return z ^ (z >> 31);
}

// window > 0: rows sorted by decreasing length inside windows of `window`
// rows; shuffle: ties broken by a hash (a random order among equal lengths)
static Layout make_layout(const std::vector<int>& lens, int window, bool shuffle = false, int longfirst = 0) {
  Layout L;
  L.m = (int)lens.size();
  L.ns = (L.m + 31) / 32;
  L.perm.resize(L.m);
  std::iota(L.perm.begin(), L.perm.end(), 0);
  if (longfirst > 0) {
    // rows longer than `longfirst` first (in their window order, longest first
    // inside each window), then the rest windowed as usual: the long slices
    // start at the head of the grid instead of every window's head
    const int W = window > 0 ? window : L.m;
    std::stable_sort(L.perm.begin(), L.perm.end(), [&](int a, int b) {
      const bool la = lens[a] > longfirst, lb = lens[b] > longfirst;
      if (la != lb) return la;
      if (a / W != b / W) return a / W < b / W;
      return lens[a] > lens[b];
    });
    window = 0;
  }
  if (window > 0)
    for (int w0 = 0; w0 < L.m; w0 += window) {
      const int w1 = std::min(L.m, w0 + window);
      std::stable_sort(L.perm.begin() + w0, L.perm.begin() + w1, [&](int a, int b) {
        if (lens[a] != lens[b]) return lens[a] > lens[b];
        return shuffle ? hmix(a) < hmix(b) : false;
      });
    }
  L.len.resize(L.m);
  for (int r = 0; r < L.m; ++r) L.len[r] = lens[L.perm[r]];
  L.width.assign(L.ns, 0);
  for (int r = 0; r < L.m; ++r) L.width[r / 32] = std::max(L.width[r / 32], L.len[r]);
  L.sptr.assign(L.ns + 1, 0);
  for (int s = 0; s < L.ns; ++s) L.sptr[s + 1] = L.sptr[s] + 32LL * L.width[s];
  L.slots = L.sptr[L.ns];
  return L;
}

int main(int argc, char** argv) {
  const int m = argc > 1 ? atoi(argv[1]) : 5000000;
  const int reps = argc > 2 ? atoi(argv[2]) : 20;
  const bool variants = argc > 3 && atoi(argv[3]) != 0;  // multi-slice kernels (measured: no gain)
  const long long n = 2LL * m;
  std::mt19937_64 rng(4);
  const double sigma = 0.8, mu = std::log(40.0) - 0.5 * sigma * sigma;
  std::lognormal_distribution<double> ln(mu, sigma);
  std::vector<int> logn(m), unif(m, 40), u20(m, 20), u80(m, 80), bim(m), lnc(m);
  for (int i = 0; i < m; ++i) bim[i] = (hmix(i) & 1) ? 20 : 60;
  long long nnz_l = 0;
  for (int i = 0; i < m; ++i) {
    logn[i] = (int)std::min<double>(kMaxLen, std::max(1.0, std::nearbyint(ln(rng))));
    lnc[i] = std::min(logn[i], 100);
    nnz_l += logn[i];
  }
  double* x;
  CK(cudaMalloc(&x, n * 8));
  k_fillx<<<(unsigned)((n + 255) / 256), 256>>>(n, x);
  double* y;
  CK(cudaMalloc(&y, (size_t)m * 8));
  struct Case {
    const char* name;
    const std::vector<int>* lens;
    int window;
    bool shuffle;
    int longfirst = 0;
  } cases[] = {{"uniform40", &unif, 0, false},
               {"uniform40_shuffled_win64k", &unif, 65536, true},
               {"lognormal_win64k", &logn, 65536, false},
               {"lognormal_win16k", &logn, 16384, false},
               {"lognormal_win4k", &logn, 4096, false},
               {"lognormal_win1k", &logn, 1024, false},
               {"lognormal_global", &logn, 1 << 30, false},
               {"lognormal_natural", &logn, 0, false},
               {"uniform20", &u20, 0, false},
               {"uniform80", &u80, 0, false},
               {"bimodal20_60_win64k", &bim, 65536, false},
               {"lognormal_clip100_win64k", &lnc, 65536, false},
               {"lognormal_win64k_long128first", &logn, 65536, false, 128},
               {"lognormal_win64k_long64first", &logn, 65536, false, 64},
               {"lognormal_win64k_long256first", &logn, 65536, false, 256},
               {"lognormal_win64k_long96first", &logn, 65536, false, 96},
               {"lognormal_win64k_long48first", &logn, 65536, false, 48},
               {"lognormal_win64k_long32first", &logn, 65536, false, 32},
               {"lognormal_win256k_long64first", &logn, 262144, false, 64},
               {"lognormal_win16k_long64first", &logn, 16384, false, 64}};
  const unsigned mask = argc > 4 ? (unsigned)strtoul(argv[4], nullptr, 0) : 0xFFu;
  const bool flat = argc > 5 && atoi(argv[5]) != 0;
  int ci = -1;
  for (const Case& cs : cases) {
    if (!((mask >> ++ci) & 1)) continue;
    Layout L = make_layout(*cs.lens, cs.window, cs.shuffle, cs.longfirst);
    int *dperm, *dlen, *dwidth, *col;
    long long* dsptr;
    double* val;
    CK(cudaMalloc(&dperm, m * 4));
    CK(cudaMalloc(&dlen, m * 4));
    CK(cudaMalloc(&dwidth, L.ns * 4));
    CK(cudaMalloc(&dsptr, (L.ns + 1) * 8));
    CK(cudaMalloc(&col, L.slots * 4));
    CK(cudaMalloc(&val, L.slots * 8));
    CK(cudaMemcpy(dperm, L.perm.data(), m * 4, cudaMemcpyHostToDevice));
    CK(cudaMemcpy(dlen, L.len.data(), m * 4, cudaMemcpyHostToDevice));
    CK(cudaMemcpy(dwidth, L.width.data(), L.ns * 4, cudaMemcpyHostToDevice));
    CK(cudaMemcpy(dsptr, L.sptr.data(), (L.ns + 1) * 8, cudaMemcpyHostToDevice));
    CK(cudaMemset(col, 0xFF, L.slots * 4));   // padding slots: col = -1
    CK(cudaMemset(val, 0, L.slots * 8));
    k_gen<<<(m + 127) / 128, 128>>>(m, (int)n, dperm, dlen, dsptr, col, val);
    CK(cudaDeviceSynchronize());
    long long nnz = 0;
    for (int v : L.len) nnz += v;
    const unsigned grid = (unsigned)((L.ns * 32LL + 255) / 256);
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0);
    cudaEventCreate(&e1);
    for (int rep = 0; rep < 2; ++rep) {
      for (int i = 0; i < 3; ++i) k_sell<10><<<grid, 256>>>(m, L.ns, dsptr, dwidth, dlen, col, val, x, y);
      cudaEventRecord(e0);
      for (int i = 0; i < reps; ++i) k_sell<10><<<grid, 256>>>(m, L.ns, dsptr, dwidth, dlen, col, val, x, y);
      cudaEventRecord(e1);
      CK(cudaEventSynchronize(e1));
      float ms = 0;
      cudaEventElapsedTime(&ms, e0, e1);
      ms /= reps;
      printf("{\"layout\": \"%s\", \"kernel\": \"1 slice/warp, 10 in flight\", \"nnz\": %lld, \"pad\": %.3f, \"ms\": %.4f, \"Gentries_s\": %.1f}\n", cs.name, nnz,
             (double)L.slots / nnz, ms, nnz / (ms * 1e6));
      fflush(stdout);
    }
    {
      std::vector<double> h0(m), h1(m);
      CK(cudaMemcpy(h0.data(), y, (size_t)m * 8, cudaMemcpyDeviceToHost));
      auto runf = [&](auto kern, int NSW, const char* nm) {
        const unsigned g = (unsigned)(((L.ns + NSW - 1) / NSW * 32LL + 255) / 256);
        CK(cudaMemset(y, 0, (size_t)m * 8));
        for (int i = 0; i < 3; ++i) kern<<<g, 256>>>(m, L.ns, dsptr, dwidth, col, val, x, y);
        cudaEventRecord(e0);
        for (int i = 0; i < reps; ++i) kern<<<g, 256>>>(m, L.ns, dsptr, dwidth, col, val, x, y);
        cudaEventRecord(e1);
        CK(cudaEventSynchronize(e1));
        float ms = 0;
        cudaEventElapsedTime(&ms, e0, e1);
        ms /= reps;
        CK(cudaMemcpy(h1.data(), y, (size_t)m * 8, cudaMemcpyDeviceToHost));
        const bool same = memcmp(h0.data(), h1.data(), (size_t)m * 8) == 0;
        printf("{\"layout\": \"%s\", \"kernel\": \"%s\", \"ms\": %.4f, \"Gentries_s\": %.1f, \"bitwise_equal\": %s}\n",
               cs.name, nm, ms, nnz / (ms * 1e6), same ? "true" : "false");
        fflush(stdout);
      };
      if (!flat) goto noflat;
      runf(k_flat<10, 1>, 1, "flat rounds, 1 slice/warp");
      runf(k_flat<10, 2>, 2, "flat rounds, 2 slices/warp");
      runf(k_flat<10, 4>, 4, "flat rounds, 4 slices/warp");
      runf(k_flat<10, 8>, 8, "flat rounds, 8 slices/warp");
      runf(k_flat<10, 16>, 16, "flat rounds, 16 slices/warp");
      runf(k_flat<8, 4>, 4, "flat rounds 8, 4 slices/warp");
      runf(k_flat<12, 4>, 4, "flat rounds 12, 4 slices/warp");
      runf(k_flat<10, 4, 5>, 4, "flat rounds, 4 slices/warp, 5 blocks/SM");
      runf(k_flat<10, 8, 5>, 8, "flat rounds, 8 slices/warp, 5 blocks/SM");
      runf(k_flat<8, 8, 5>, 8, "flat rounds 8, 8 slices/warp, 5 blocks/SM");
    }
  noflat:
    if (!variants) goto done;
    {
      std::vector<double> h0(m), h1(m);
      CK(cudaMemcpy(h0.data(), y, (size_t)m * 8, cudaMemcpyDeviceToHost));
      auto run = [&](auto kern, int NS, const char* nm) {
        const unsigned g = (unsigned)(((L.ns + NS - 1) / NS * 32LL + 255) / 256);
        for (int i = 0; i < 3; ++i) kern<<<g, 256>>>(m, L.ns, dsptr, dwidth, dlen, col, val, x, y);
        cudaEventRecord(e0);
        for (int i = 0; i < reps; ++i) kern<<<g, 256>>>(m, L.ns, dsptr, dwidth, dlen, col, val, x, y);
        cudaEventRecord(e1);
        CK(cudaEventSynchronize(e1));
        float ms = 0;
        cudaEventElapsedTime(&ms, e0, e1);
        ms /= reps;
        CK(cudaMemcpy(h1.data(), y, (size_t)m * 8, cudaMemcpyDeviceToHost));
        const bool same = memcmp(h0.data(), h1.data(), (size_t)m * 8) == 0;
        printf("{\"layout\": \"%s\", \"kernel\": \"%s\", \"ms\": %.4f, \"Gentries_s\": %.1f, \"bitwise_equal\": %s}\n",
               cs.name, nm, ms, nnz / (ms * 1e6), same ? "true" : "false");
        fflush(stdout);
      };
      run(k_sell_multi<5, 2, 6>, 2, "2 slices/warp x 5 in flight, 6 blocks/SM (spills)");
      run(k_sell_multi<5, 2, 4>, 2, "2 slices/warp x 5 in flight, 4 blocks/SM");
      run(k_sell_multi<6, 2, 4>, 2, "2 slices/warp x 6 in flight, 4 blocks/SM");
      run(k_sell_multi<8, 2, 4>, 2, "2 slices/warp x 8 in flight, 4 blocks/SM");
      run(k_sell_multi<4, 3, 4>, 3, "3 slices/warp x 4 in flight, 4 blocks/SM");
      run(k_sell_multi<3, 4, 4>, 4, "4 slices/warp x 3 in flight, 4 blocks/SM");
      run(k_sell_multi<5, 2, 3>, 2, "2 slices/warp x 5 in flight, 3 blocks/SM");
      run(k_sell_multi<10, 1, 6>, 1, "1 slice/warp x 10 (multi kernel)");
    }
  done:
    cudaFree(dperm);
    cudaFree(dlen);
    cudaFree(dwidth);
    cudaFree(dsptr);
    cudaFree(col);
    cudaFree(val);
  }
  // medium tier: lognormal rows > T on warp-per-row CSR, the rest in the windowed sliced ELL
  if (mask & 0x1000) {
    for (int T : {192, 256, 320}) {
      std::vector<int> lsell(m), mrows;
      std::vector<int> mptr(1, 0);
      for (int i = 0; i < m; ++i) {
        if (logn[i] > T) {
          lsell[i] = 0;
          mrows.push_back(i);
          mptr.push_back(mptr.back() + logn[i]);
        } else {
          lsell[i] = logn[i];
        }
      }
      Layout L = make_layout(lsell, 65536, false);
      const int nmed = (int)mrows.size();
      int *dperm, *dlen, *dwidth, *col, *dmrow, *dmptr, *mcol;
      long long* dsptr;
      double *val, *mval, *ymed;
      CK(cudaMalloc(&dperm, m * 4));
      CK(cudaMalloc(&dlen, m * 4));
      CK(cudaMalloc(&dwidth, L.ns * 4));
      CK(cudaMalloc(&dsptr, (L.ns + 1) * 8));
      CK(cudaMalloc(&col, std::max(1LL, L.slots) * 4));
      CK(cudaMalloc(&val, std::max(1LL, L.slots) * 8));
      CK(cudaMalloc(&dmrow, std::max(1, nmed) * 4));
      CK(cudaMalloc(&dmptr, (nmed + 1) * 4));
      CK(cudaMalloc(&mcol, std::max(1, mptr.back()) * 4));
      CK(cudaMalloc(&mval, std::max(1, mptr.back()) * 8));
      CK(cudaMalloc(&ymed, std::max(1, nmed) * 8));
      CK(cudaMemcpy(dperm, L.perm.data(), m * 4, cudaMemcpyHostToDevice));
      CK(cudaMemcpy(dlen, L.len.data(), m * 4, cudaMemcpyHostToDevice));
      CK(cudaMemcpy(dwidth, L.width.data(), L.ns * 4, cudaMemcpyHostToDevice));
      CK(cudaMemcpy(dsptr, L.sptr.data(), (L.ns + 1) * 8, cudaMemcpyHostToDevice));
      CK(cudaMemcpy(dmrow, mrows.data(), nmed * 4, cudaMemcpyHostToDevice));
      CK(cudaMemcpy(dmptr, mptr.data(), (nmed + 1) * 4, cudaMemcpyHostToDevice));
      k_gen<<<(m + 127) / 128, 128>>>(m, (int)n, dperm, dlen, dsptr, col, val);
      k_gen_csr<<<(nmed + 127) / 128, 128>>>(nmed, (int)n, dmrow, dmptr, mcol, mval);
      CK(cudaDeviceSynchronize());
      const int nmb = (nmed + 7) / 8;
      const unsigned grid = (unsigned)(nmb + (L.ns * 32LL + 255) / 256);
      long long nnz = mptr.back();
      for (int v : L.len) nnz += v;
      cudaEvent_t e0, e1;
      cudaEventCreate(&e0);
      cudaEventCreate(&e1);
      auto go = [&](auto kern, const char* nm) {
        for (int i = 0; i < 3; ++i)
          kern<<<grid, 256>>>(m, L.ns, dsptr, dwidth, dlen, col, val, nmed, nmb, dmrow, dmptr, mcol, mval, x, y, ymed);
        cudaEventRecord(e0);
        for (int i = 0; i < reps; ++i)
          kern<<<grid, 256>>>(m, L.ns, dsptr, dwidth, dlen, col, val, nmed, nmb, dmrow, dmptr, mcol, mval, x, y, ymed);
        cudaEventRecord(e1);
        CK(cudaEventSynchronize(e1));
        float ms = 0;
        cudaEventElapsedTime(&ms, e0, e1);
        ms /= reps;
        printf("{\"layout\": \"lognormal_win64k_medium%d\", \"kernel\": \"%s\", \"nnz\": %lld, \"medium_rows\": %d, "
               "\"medium_entries\": %d, \"ms\": %.4f, \"Gentries_s\": %.1f}\n",
               T, nm, nnz, nmed, mptr.back(), ms, nnz / (ms * 1e6));
        fflush(stdout);
      };
      go(k_sell_med<10, 4>, "SELL 10 + warp-per-row 4");
      go(k_sell_med<10, 6>, "SELL 10 + warp-per-row 6");
      cudaFree(dperm); cudaFree(dlen); cudaFree(dwidth); cudaFree(dsptr); cudaFree(col); cudaFree(val);
      cudaFree(dmrow); cudaFree(dmptr); cudaFree(mcol); cudaFree(mval); cudaFree(ymed);
    }
  }
  return 0;
}
