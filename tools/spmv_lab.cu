// spmv_lab.cu -- kernel-variant lab for the PDHG SpMVs (development tool, not product).
// Generates a config-4-shaped matrix on the device (5M x 10M, ~200M nnz,
// lognormal rows mean 40, 70% banded +-50k, 30% uniform) and its transpose,
// then times CSR SpMV variants on A (gather x, 80 MB) and A' (gather y, 40 MB).
#include <algorithm>
#include <cstdio>
#include <cstdint>
#include <cstdlib>
#include <cstring>
#include <vector>
#include <cub/cub.cuh>

#define CK(x) do { cudaError_t e = (x); if (e != cudaSuccess) { \
  fprintf(stderr, "%s:%d %s\n", __FILE__, __LINE__, cudaGetErrorString(e)); exit(1);} } while (0)

__host__ __device__ inline uint64_t mix64(uint64_t z) {
  z += 0x9e3779b97f4a7c15ULL;
  z = (z ^ (z >> 30)) * 0xbf58476d1ce4e5b9ULL;
  z = (z ^ (z >> 27)) * 0x94d049bb133111ebULL;
  return z ^ (z >> 31);
}
__device__ inline double u01(uint64_t h) { return ((h >> 11) + 0.5) * (1.0 / 9007199254740992.0); }

__global__ void k_rowlen(int m, int* len) {
  int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= m) return;
  double u1 = u01(mix64(i * 2ULL + 1)), u2 = u01(mix64(i * 2ULL + 2));
  double g = sqrt(-2.0 * log(u1)) * cospi(2.0 * u2);
  double mu = log(40.0) - 0.5 * 0.8 * 0.8;
  long l = lround(exp(mu + 0.8 * g));
  len[i] = (int)min(max(l, 1L), 2000L);
}
__global__ void k_fill(int m, int n, const int* ptr, int* col, double* val) {
  int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= m) return;
  for (int k = ptr[i]; k < ptr[i + 1]; ++k) {
    uint64_t h = mix64(0x1234567ULL ^ (uint64_t)k * 0x100000001b3ULL);
    long c;
    if (u01(h) < 0.7) c = ((2L * i + (long)(mix64(h) % 100001ULL) - 50000) % n + n) % n;
    else c = (long)(mix64(h + 7) % (uint64_t)n);
    col[k] = (int)c;
    val[k] = u01(mix64(h + 13)) - 0.5;
  }
}
__global__ void k_sortrows(int m, const int* ptr, int* col) {
  int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= m) return;
  int s = ptr[i], e = ptr[i + 1];
  for (int a = s + 1; a < e; ++a) {
    int v = col[a]; int b = a - 1;
    while (b >= s && col[b] > v) { col[b + 1] = col[b]; --b; }
    col[b + 1] = v;
  }
}
__global__ void k_rid(int m, const int* ptr, int* rid) {
  int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= m) return;
  for (int k = ptr[i]; k < ptr[i + 1]; ++k) rid[k] = i;
}
__global__ void k_iota(int* v, int n) { int i = blockIdx.x * blockDim.x + threadIdx.x; if (i < n) v[i] = i; }
__global__ void k_gt(int nnz, const int* perm, const int* rid, const double* val, int* tc, double* tv) {
  int k = blockIdx.x * blockDim.x + threadIdx.x;
  if (k >= nnz) return;
  tc[k] = rid[perm[k]]; tv[k] = val[perm[k]];
}
__global__ void k_cptr(const int* keys, int nnz, int n, int* tp) {
  int j = blockIdx.x * blockDim.x + threadIdx.x;
  if (j > n) return;
  int lo = 0, hi = nnz;
  while (lo < hi) { int mid = (lo + hi) >> 1; if (keys[mid] < j) lo = mid + 1; else hi = mid; }
  tp[j] = lo;
}

struct Csr { int rows, cols, nnz; int* ptr; int* col; double* val; };

template <int V>
__device__ __forceinline__ double gsum(double v) {
#pragma unroll
  for (int o = V / 2; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  return v;
}

// ---- V1 baseline (library v1)
template <int V>
__global__ void __launch_bounds__(256) v1(Csr A, const double* __restrict__ x, double* __restrict__ y) {
  const long long gid = (long long)blockIdx.x * 256 + threadIdx.x;
  const int row = (int)(gid / V), lane = threadIdx.x % V;
  int s = 0, e = 0;
  if (row < A.rows) { s = A.ptr[row]; e = A.ptr[row + 1]; }
  double acc = 0.0;
  for (int k = s + lane; k < e; k += V) acc = fma(__ldcs(A.val + k), __ldg(x + __ldcs(A.col + k)), acc);
  acc = gsum<V>(acc);
  if (row < A.rows && lane == 0) y[row] = acc;
}

// ---- V2 unrolled x U: U independent (val, col, gather) triples in flight per lane
template <int V, int U>
__global__ void __launch_bounds__(256) v2(Csr A, const double* __restrict__ x, double* __restrict__ y) {
  const long long gid = (long long)blockIdx.x * 256 + threadIdx.x;
  const int row = (int)(gid / V), lane = threadIdx.x % V;
  int s = 0, e = 0;
  if (row < A.rows) { s = A.ptr[row]; e = A.ptr[row + 1]; }
  double acc = 0.0;
  for (int k = s + lane; k < e; k += U * V) {
    double a[U], xv[U];
    int j[U];
#pragma unroll
    for (int u = 0; u < U; ++u) {
      const int kk = k + u * V;
      a[u] = kk < e ? __ldcs(A.val + kk) : 0.0;
      j[u] = kk < e ? __ldcs(A.col + kk) : -1;
    }
#pragma unroll
    for (int u = 0; u < U; ++u) xv[u] = j[u] >= 0 ? __ldg(x + j[u]) : 0.0;
#pragma unroll
    for (int u = 0; u < U; ++u) acc = fma(a[u], xv[u], acc);
  }
  acc = gsum<V>(acc);
  if (row < A.rows && lane == 0) y[row] = acc;
}

// ---- V3 pairs: 16-byte val / 8-byte col loads, one peeled head element
template <int V, int U>
__global__ void __launch_bounds__(256) v3(Csr A, const double* __restrict__ x, double* __restrict__ y) {
  const long long gid = (long long)blockIdx.x * 256 + threadIdx.x;
  const int row = (int)(gid / V), lane = threadIdx.x % V;
  int s = 0, e = 0;
  if (row < A.rows) { s = A.ptr[row]; e = A.ptr[row + 1]; }
  double acc = 0.0;
  if ((s & 1) && s < e) {  // peel to even
    if (lane == 0) acc = __ldcs(A.val + s) * __ldg(x + __ldcs(A.col + s));
    ++s;
  }
  const int np = (e - s) >> 1;  // pairs
  const double2* vp = reinterpret_cast<const double2*>(A.val + s);
  const int2* cp = reinterpret_cast<const int2*>(A.col + s);
  for (int p = lane; p < np; p += U * V) {
    double2 a[U];
    int2 j[U];
    double x0[U], x1[U];
#pragma unroll
    for (int u = 0; u < U; ++u) {
      const int pp = p + u * V;
      if (pp < np) { a[u] = __ldcs(vp + pp); j[u] = __ldcs(cp + pp); }
      else { a[u] = make_double2(0, 0); j[u] = make_int2(-1, -1); }
    }
#pragma unroll
    for (int u = 0; u < U; ++u) {
      x0[u] = j[u].x >= 0 ? __ldg(x + j[u].x) : 0.0;
      x1[u] = j[u].y >= 0 ? __ldg(x + j[u].y) : 0.0;
    }
#pragma unroll
    for (int u = 0; u < U; ++u) { acc = fma(a[u].x, x0[u], acc); acc = fma(a[u].y, x1[u], acc); }
  }
  if ((e - s) & 1) {
    if (lane == (np % V)) acc = fma(__ldcs(A.val + e - 1), __ldg(x + __ldcs(A.col + e - 1)), acc);
  }
  acc = gsum<V>(acc);
  if (row < A.rows && lane == 0) y[row] = acc;
}


// ---- V5: library v3 scheme: warp owns 32 rows, V passes, extents prefetched, U-deep loads
template <int V, int U>
__global__ void __launch_bounds__(256) v5(Csr A, const double* __restrict__ x, double* __restrict__ y) {
  constexpr int G = 32 / V;
  const int lane = threadIdx.x & 31;
  const long long row0 = (((long long)blockIdx.x * 256 + threadIdx.x) >> 5) * 32;
  if (row0 >= A.rows) return;
  const long long rl = row0 + lane;
  int my_s = 0, my_e = 0;
  if (rl < A.rows) { my_s = A.ptr[rl]; my_e = A.ptr[rl + 1]; }
  double mine = 0.0;
#pragma unroll 1
  for (int pass = 0; pass < V; ++pass) {
    const int src = pass * G + lane / V;
    const int s = __shfl_sync(0xffffffffu, my_s, src);
    const int e = __shfl_sync(0xffffffffu, my_e, src);
    double acc = 0.0;
    for (int k = s + lane % V; k < e; k += U * V) {
      double a[U], xv[U];
      int j[U];
#pragma unroll
      for (int u = 0; u < U; ++u) {
        const int kk = k + u * V;
        a[u] = kk < e ? __ldcs(A.val + kk) : 0.0;
        j[u] = kk < e ? __ldcs(A.col + kk) : -1;
      }
#pragma unroll
      for (int u = 0; u < U; ++u) xv[u] = j[u] >= 0 ? __ldg(x + j[u]) : 0.0;
#pragma unroll
      for (int u = 0; u < U; ++u) if (j[u] >= 0) acc = fma(a[u], xv[u], acc);
    }
    acc = gsum<V>(acc);
    const double got = __shfl_sync(0xffffffffu, acc, ((lane - pass * G) & (G - 1)) * V);
    if (lane / G == pass) mine = got;
  }
  if (rl < A.rows) y[rl] = mine;
}

// ---- V6: like V5 but two passes in flight (rows of pass p and p+1 interleaved)
template <int V, int U>
__global__ void __launch_bounds__(256) v6(Csr A, const double* __restrict__ x, double* __restrict__ y) {
  constexpr int G = 32 / V;
  const int lane = threadIdx.x & 31;
  const long long row0 = (((long long)blockIdx.x * 256 + threadIdx.x) >> 5) * 32;
  if (row0 >= A.rows) return;
  const long long rl = row0 + lane;
  int my_s = 0, my_e = 0;
  if (rl < A.rows) { my_s = A.ptr[rl]; my_e = A.ptr[rl + 1]; }
  double mine = 0.0;
#pragma unroll 1
  for (int pass = 0; pass < V; pass += 2) {
    const int src0 = pass * G + lane / V, src1 = src0 + G;
    const int s0 = __shfl_sync(0xffffffffu, my_s, src0), e0 = __shfl_sync(0xffffffffu, my_e, src0);
    const int s1 = __shfl_sync(0xffffffffu, my_s, src1), e1 = __shfl_sync(0xffffffffu, my_e, src1);
    double acc0 = 0.0, acc1 = 0.0;
    const int n0 = e0 - s0, n1 = e1 - s1;
    const int nmax = n0 > n1 ? n0 : n1;
    for (int o = lane % V; o < nmax; o += U * V) {
      double a0[U], a1[U], x0[U], x1[U];
      int j0[U], j1[U];
#pragma unroll
      for (int u = 0; u < U; ++u) {
        const int oo = o + u * V;
        a0[u] = oo < n0 ? __ldcs(A.val + s0 + oo) : 0.0;
        j0[u] = oo < n0 ? __ldcs(A.col + s0 + oo) : -1;
        a1[u] = oo < n1 ? __ldcs(A.val + s1 + oo) : 0.0;
        j1[u] = oo < n1 ? __ldcs(A.col + s1 + oo) : -1;
      }
#pragma unroll
      for (int u = 0; u < U; ++u) {
        x0[u] = j0[u] >= 0 ? __ldg(x + j0[u]) : 0.0;
        x1[u] = j1[u] >= 0 ? __ldg(x + j1[u]) : 0.0;
      }
#pragma unroll
      for (int u = 0; u < U; ++u) {
        if (j0[u] >= 0) acc0 = fma(a0[u], x0[u], acc0);
        if (j1[u] >= 0) acc1 = fma(a1[u], x1[u], acc1);
      }
    }
    acc0 = gsum<V>(acc0);
    acc1 = gsum<V>(acc1);
    const double g0 = __shfl_sync(0xffffffffu, acc0, ((lane - pass * G) & (G - 1)) * V);
    const double g1 = __shfl_sync(0xffffffffu, acc1, ((lane - (pass + 1) * G) & (G - 1)) * V);
    if (lane / G == pass) mine = g0;
    if (lane / G == pass + 1) mine = g1;
  }
  if (rl < A.rows) y[rl] = mine;
}


// ---- V7: V5 + software pipelining across passes: the next pass's first
// U*V entries (val, col) are loaded before the current pass's gathers.
template <int V, int U, int MB = 1>
__global__ void __launch_bounds__(256, MB) v7(Csr A, const double* __restrict__ x, double* __restrict__ y) {
  constexpr int G = 32 / V;
  const int lane = threadIdx.x & 31, sub = lane % V;
  const long long row0 = (((long long)blockIdx.x * 256 + threadIdx.x) >> 5) * 32;
  if (row0 >= A.rows) return;
  const long long rl = row0 + lane;
  int my_s = 0, my_e = 0;
  if (rl < A.rows) { my_s = A.ptr[rl]; my_e = A.ptr[rl + 1]; }
  double mine = 0.0;
  int s = __shfl_sync(0xffffffffu, my_s, lane / V);
  int e = __shfl_sync(0xffffffffu, my_e, lane / V);
  double ac[U];
  int jc[U];
#pragma unroll
  for (int u = 0; u < U; ++u) {
    const int kk = s + sub + u * V;
    ac[u] = kk < e ? __ldcs(A.val + kk) : 0.0;
    jc[u] = kk < e ? __ldcs(A.col + kk) : -1;
  }
#pragma unroll 1
  for (int pass = 0; pass < V; ++pass) {
    int sn = 0, en = 0;
    double an[U];
    int jn[U];
    if (pass + 1 < V) {
      const int src = (pass + 1) * G + lane / V;
      sn = __shfl_sync(0xffffffffu, my_s, src);
      en = __shfl_sync(0xffffffffu, my_e, src);
    }
#pragma unroll
    for (int u = 0; u < U; ++u) {
      const int kk = sn + sub + u * V;
      an[u] = kk < en ? __ldcs(A.val + kk) : 0.0;
      jn[u] = kk < en ? __ldcs(A.col + kk) : -1;
    }
    double xv[U];
#pragma unroll
    for (int u = 0; u < U; ++u) xv[u] = jc[u] >= 0 ? __ldg(x + jc[u]) : 0.0;
    double acc = 0.0;
#pragma unroll
    for (int u = 0; u < U; ++u) if (jc[u] >= 0) acc = fma(ac[u], xv[u], acc);
    for (int k = s + sub + U * V; k < e; k += U * V) {
      double a2[U], x2[U];
      int j2[U];
#pragma unroll
      for (int u = 0; u < U; ++u) {
        const int kk = k + u * V;
        a2[u] = kk < e ? __ldcs(A.val + kk) : 0.0;
        j2[u] = kk < e ? __ldcs(A.col + kk) : -1;
      }
#pragma unroll
      for (int u = 0; u < U; ++u) x2[u] = j2[u] >= 0 ? __ldg(x + j2[u]) : 0.0;
#pragma unroll
      for (int u = 0; u < U; ++u) if (j2[u] >= 0) acc = fma(a2[u], x2[u], acc);
    }
    acc = gsum<V>(acc);
    const double got = __shfl_sync(0xffffffffu, acc, ((lane - pass * G) & (G - 1)) * V);
    if (lane / G == pass) mine = got;
#pragma unroll
    for (int u = 0; u < U; ++u) { ac[u] = an[u]; jc[u] = jn[u]; }
    s = sn; e = en;
  }
  if (rl < A.rows) y[rl] = mine;
}


// ---- V8: two passes at once (rows of pass p and p+1 together) + prefetch of the next pair
template <int V, int U>
__global__ void __launch_bounds__(256) v8(Csr A, const double* __restrict__ x, double* __restrict__ y) {
  constexpr int G = 32 / V;
  const int lane = threadIdx.x & 31, sub = lane % V;
  const long long row0 = (((long long)blockIdx.x * 256 + threadIdx.x) >> 5) * 32;
  if (row0 >= A.rows) return;
  const long long rl = row0 + lane;
  int my_s = 0, my_e = 0;
  if (rl < A.rows) { my_s = A.ptr[rl]; my_e = A.ptr[rl + 1]; }
  double mine = 0.0;
  int s[2], e[2];
  double ac[2][U];
  int jc[2][U];
#pragma unroll
  for (int h = 0; h < 2; ++h) {
    s[h] = __shfl_sync(0xffffffffu, my_s, h * G + lane / V);
    e[h] = __shfl_sync(0xffffffffu, my_e, h * G + lane / V);
#pragma unroll
    for (int u = 0; u < U; ++u) {
      const int kk = s[h] + sub + u * V;
      ac[h][u] = kk < e[h] ? __ldcs(A.val + kk) : 0.0;
      jc[h][u] = kk < e[h] ? __ldcs(A.col + kk) : -1;
    }
  }
#pragma unroll 1
  for (int pass = 0; pass < V; pass += 2) {
    int sn[2] = {0, 0}, en[2] = {0, 0};
    double an[2][U];
    int jn[2][U];
#pragma unroll
    for (int h = 0; h < 2; ++h) {
      if (pass + 2 < V) {
        sn[h] = __shfl_sync(0xffffffffu, my_s, (pass + 2 + h) * G + lane / V);
        en[h] = __shfl_sync(0xffffffffu, my_e, (pass + 2 + h) * G + lane / V);
      }
#pragma unroll
      for (int u = 0; u < U; ++u) {
        const int kk = sn[h] + sub + u * V;
        an[h][u] = kk < en[h] ? __ldcs(A.val + kk) : 0.0;
        jn[h][u] = kk < en[h] ? __ldcs(A.col + kk) : -1;
      }
    }
    double xv[2][U];
#pragma unroll
    for (int h = 0; h < 2; ++h)
#pragma unroll
      for (int u = 0; u < U; ++u) xv[h][u] = jc[h][u] >= 0 ? __ldg(x + jc[h][u]) : 0.0;
    double acc[2] = {0.0, 0.0};
#pragma unroll
    for (int h = 0; h < 2; ++h) {
#pragma unroll
      for (int u = 0; u < U; ++u) if (jc[h][u] >= 0) acc[h] = fma(ac[h][u], xv[h][u], acc[h]);
      for (int k = s[h] + sub + U * V; k < e[h]; k += U * V) {
        double a2[U], x2[U];
        int j2[U];
#pragma unroll
        for (int u = 0; u < U; ++u) {
          const int kk = k + u * V;
          a2[u] = kk < e[h] ? __ldcs(A.val + kk) : 0.0;
          j2[u] = kk < e[h] ? __ldcs(A.col + kk) : -1;
        }
#pragma unroll
        for (int u = 0; u < U; ++u) x2[u] = j2[u] >= 0 ? __ldg(x + j2[u]) : 0.0;
#pragma unroll
        for (int u = 0; u < U; ++u) if (j2[u] >= 0) acc[h] = fma(a2[u], x2[u], acc[h]);
      }
      const double d = gsum<V>(acc[h]);
      const double got = __shfl_sync(0xffffffffu, d, ((lane - (pass + h) * G) & (G - 1)) * V);
      if (lane / G == pass + h) mine = got;
    }
#pragma unroll
    for (int h = 0; h < 2; ++h) {
#pragma unroll
      for (int u = 0; u < U; ++u) { ac[h][u] = an[h][u]; jc[h][u] = jn[h][u]; }
      s[h] = sn[h]; e[h] = en[h];
    }
  }
  if (rl < A.rows) y[rl] = mine;
}


__device__ __forceinline__ void l2_prefetch(const void* p, unsigned bytes) {
  // cp.async.bulk.prefetch.L2: address 16-B aligned, size a multiple of 16
  const unsigned long long a = (unsigned long long)p;
  unsigned long long off = a & ~15ULL;
  const unsigned long long end = (a + bytes + 15) & ~15ULL;
  while (off < end) {
    const unsigned chunk = (end - off) > (1ull << 20) ? (1u << 20) : (unsigned)(end - off);
    asm volatile("cp.async.bulk.prefetch.L2.global [%0], %1;" ::"l"(off), "r"(chunk) : "memory");
    off += chunk;
  }
}

// ---- V9: V5 + one bulk L2 prefetch per block of the entries of block (b + D)
template <int V, int U, int D>
__global__ void __launch_bounds__(256) v9(Csr A, const double* __restrict__ x, double* __restrict__ y) {
  if (threadIdx.x == 0) {
    const long long nb = (long long)blockIdx.x + D;
    const long long r0 = nb * 256, r1 = min((long long)A.rows, r0 + 256);
    if (r0 < A.rows) {
      const int s = A.ptr[r0], e = A.ptr[r1];
      l2_prefetch(A.val + s, (unsigned)(e - s) * 8u);
      l2_prefetch(A.col + s, (unsigned)(e - s) * 4u);
    }
  }
  constexpr int G = 32 / V;
  const int lane = threadIdx.x & 31;
  const long long row0 = (((long long)blockIdx.x * 256 + threadIdx.x) >> 5) * 32;
  if (row0 >= A.rows) return;
  const long long rl = row0 + lane;
  int my_s = 0, my_e = 0;
  if (rl < A.rows) { my_s = A.ptr[rl]; my_e = A.ptr[rl + 1]; }
  double mine = 0.0;
#pragma unroll 1
  for (int pass = 0; pass < V; ++pass) {
    const int src = pass * G + lane / V;
    const int s = __shfl_sync(0xffffffffu, my_s, src);
    const int e = __shfl_sync(0xffffffffu, my_e, src);
    double acc = 0.0;
    for (int k = s + lane % V; k < e; k += U * V) {
      double a[U], xv[U];
      int j[U];
#pragma unroll
      for (int u = 0; u < U; ++u) {
        const int kk = k + u * V;
        a[u] = kk < e ? __ldcs(A.val + kk) : 0.0;
        j[u] = kk < e ? __ldcs(A.col + kk) : -1;
      }
#pragma unroll
      for (int u = 0; u < U; ++u) xv[u] = j[u] >= 0 ? __ldg(x + j[u]) : 0.0;
#pragma unroll
      for (int u = 0; u < U; ++u) if (j[u] >= 0) acc = fma(a[u], xv[u], acc);
    }
    acc = gsum<V>(acc);
    const double got = __shfl_sync(0xffffffffu, acc, ((lane - pass * G) & (G - 1)) * V);
    if (lane / G == pass) mine = got;
  }
  if (rl < A.rows) y[rl] = mine;
}

// ---- V4: one warp, several rows: 2 rows per 32-lane warp at V=16 etc. is V1/V2; skip.


// ---- V10: SELL-32 (sliced ELL, slice = 32 consecutive rows, column-major inside
// the slice, natural row order): lane = row, one sequential sum per row, no
// shuffles; stream loads are 256 B / 128 B per warp instruction.
struct Sell { int rows, nslices; const long long* sptr; const int* width; const int* ptr; const int* col; const double* val; };

__global__ void k_sell_width(int rows, const int* ptr, int* width) {
  const int sl = blockIdx.x * blockDim.x + threadIdx.x;
  if (sl >= (rows + 31) / 32) return;
  int w = 0;
  for (int r = sl * 32; r < min(rows, sl * 32 + 32); ++r) w = max(w, ptr[r + 1] - ptr[r]);
  width[sl] = w;
}
__global__ void k_sell_w32(int ns, const int* width, long long* w32) {
  const int sl = blockIdx.x * blockDim.x + threadIdx.x;
  if (sl < ns) w32[sl] = 32LL * width[sl];
  else if (sl == ns) w32[ns] = 0;
}
__global__ void k_sell_fill(int rows, const int* ptr, const int* col, const double* val, const long long* sptr,
                            int* scol, double* sval) {
  const int r = blockIdx.x * blockDim.x + threadIdx.x;
  if (r >= rows) return;
  const long long base = sptr[r / 32] + (r % 32);
  for (int k = ptr[r]; k < ptr[r + 1]; ++k) {
    scol[base + (long long)(k - ptr[r]) * 32] = col[k];
    sval[base + (long long)(k - ptr[r]) * 32] = val[k];
  }
}

template <int U>
__global__ void __launch_bounds__(256) v10(Sell S, const double* __restrict__ x, double* __restrict__ y) {
  const int lane = threadIdx.x & 31;
  const long long sl = ((long long)blockIdx.x * 256 + threadIdx.x) >> 5;
  if (sl >= S.nslices) return;
  const long long r = sl * 32 + lane;
  const int L = r < S.rows ? S.ptr[r + 1] - S.ptr[r] : 0;
  const int w = S.width[sl];
  const long long base = S.sptr[sl] + lane;
  double acc = 0.0;
  for (int k = 0; k < w; k += U) {
    double a[U], xv[U];
    int j[U];
#pragma unroll
    for (int u = 0; u < U; ++u) {
      const bool on = k + u < L;
      a[u] = on ? __ldcs(S.val + base + (long long)(k + u) * 32) : 0.0;
      j[u] = on ? __ldcs(S.col + base + (long long)(k + u) * 32) : -1;
    }
#pragma unroll
    for (int u = 0; u < U; ++u) xv[u] = j[u] >= 0 ? __ldg(x + j[u]) : 0.0;
#pragma unroll
    for (int u = 0; u < U; ++u) if (j[u] >= 0) acc = fma(a[u], xv[u], acc);
  }
  if (r < S.rows) y[r] = acc;
}


// ---- V12: v10 + the primal-step epilogue (read c, x, xbar; write x, xe, xbar)
struct Epi { const double* c; double* x; double* xe; double* xbar; double t; };
template <int U>
__global__ void __launch_bounds__(256) v12(Sell S, const double* __restrict__ g, Epi E) {
  const int lane = threadIdx.x & 31;
  const long long sl = ((long long)blockIdx.x * 256 + threadIdx.x) >> 5;
  if (sl >= S.nslices) return;
  const long long r = sl * 32 + lane;
  double o1 = 0, o2 = 0, o3 = 0;
  if (r < S.rows) { o1 = E.c[r]; o2 = E.x[r]; o3 = E.xbar[r]; }
  const int L = r < S.rows ? S.ptr[r + 1] - S.ptr[r] : 0;
  const int w = S.width[sl];
  const long long base = S.sptr[sl] + lane;
  double acc = 0.0;
  for (int k = 0; k < w; k += U) {
    double a[U], xv[U];
    int j[U];
#pragma unroll
    for (int u = 0; u < U; ++u) {
      const bool on = k + u < L;
      a[u] = on ? __ldcs(S.val + base + (long long)(k + u) * 32) : 0.0;
      j[u] = on ? __ldcs(S.col + base + (long long)(k + u) * 32) : -1;
    }
#pragma unroll
    for (int u = 0; u < U; ++u) xv[u] = j[u] >= 0 ? __ldg(g + j[u]) : 0.0;
#pragma unroll
    for (int u = 0; u < U; ++u) if (j[u] >= 0) acc = fma(a[u], xv[u], acc);
  }
  if (r < S.rows) {
    const double xn = fmax(0.0, o2 - E.t * (o1 - acc));
    E.x[r] = xn;
    E.xe[r] = 2.0 * xn - o2;
    E.xbar[r] = o3 + (xn - o3) * 0.5;
  }
}

static Sell build_sell(const Csr& M) {
  Sell S{};
  S.rows = M.rows;
  S.nslices = (M.rows + 31) / 32;
  int* width; long long* sptr;
  CK(cudaMalloc(&width, (size_t)S.nslices * 4));
  CK(cudaMalloc(&sptr, (size_t)(S.nslices + 1) * 8));
  k_sell_width<<<(S.nslices + 255) / 256, 256>>>(M.rows, M.ptr, width);
  k_sell_w32<<<(S.nslices + 256) / 256, 256>>>(S.nslices, width, sptr);
  void* tmp = nullptr; size_t tb = 0;
  cub::DeviceScan::ExclusiveSum(tmp, tb, sptr, sptr, S.nslices + 1);
  CK(cudaMalloc(&tmp, tb));
  cub::DeviceScan::ExclusiveSum(tmp, tb, sptr, sptr, S.nslices + 1);
  long long tot = 0;
  CK(cudaMemcpy(&tot, sptr + S.nslices, 8, cudaMemcpyDeviceToHost));
  int* scol; double* sval;
  CK(cudaMalloc(&scol, (size_t)tot * 4)); CK(cudaMalloc(&sval, (size_t)tot * 8));
  CK(cudaMemset(scol, 0, (size_t)tot * 4)); CK(cudaMemset(sval, 0, (size_t)tot * 8));
  k_sell_fill<<<(M.rows + 255) / 256, 256>>>(M.rows, M.ptr, M.col, M.val, sptr, scol, sval);
  CK(cudaDeviceSynchronize());
  cudaFree(tmp);
  printf("  SELL-32: %lld slots for %d nnz (%.2fx)\n", tot, M.nnz, (double)tot / M.nnz);
  S.sptr = sptr; S.width = width; S.ptr = M.ptr; S.col = scol; S.val = sval;
  return S;
}


// ---- V11: SELL-32-sigma: rows sorted by length (descending) inside windows of
// sigma rows, slices of 32 sorted rows; lane = row perm[p], y[perm[p]] written.
struct SellP { int rows, nslices; const long long* sptr; const int* width; const int* ptr; const int* perm;
               const int* col; const double* val; };

__global__ void k_sellp_width(int rows, const int* ptr, const int* perm, int* width) {
  const int sl = blockIdx.x * blockDim.x + threadIdx.x;
  if (sl >= (rows + 31) / 32) return;
  int w = 0;
  for (int p = sl * 32; p < min(rows, sl * 32 + 32); ++p) { const int r = perm[p]; w = max(w, ptr[r + 1] - ptr[r]); }
  width[sl] = w;
}
__global__ void k_sellp_fill(int rows, const int* ptr, const int* perm, const int* col, const double* val,
                             const long long* sptr, int* scol, double* sval) {
  const int p = blockIdx.x * blockDim.x + threadIdx.x;
  if (p >= rows) return;
  const int r = perm[p];
  const long long base = sptr[p / 32] + (p % 32);
  for (int k = ptr[r]; k < ptr[r + 1]; ++k) {
    scol[base + (long long)(k - ptr[r]) * 32] = col[k];
    sval[base + (long long)(k - ptr[r]) * 32] = val[k];
  }
}

template <int U>
__global__ void __launch_bounds__(256) v11(SellP S, const double* __restrict__ x, double* __restrict__ y) {
  const int lane = threadIdx.x & 31;
  const long long sl = ((long long)blockIdx.x * 256 + threadIdx.x) >> 5;
  if (sl >= S.nslices) return;
  const long long p = sl * 32 + lane;
  const int r = p < S.rows ? S.perm[p] : -1;
  const int L = r >= 0 ? S.ptr[r + 1] - S.ptr[r] : 0;
  const int w = S.width[sl];
  const long long base = S.sptr[sl] + lane;
  double acc = 0.0;
  for (int k = 0; k < w; k += U) {
    double a[U], xv[U];
    int j[U];
#pragma unroll
    for (int u = 0; u < U; ++u) {
      const bool on = k + u < L;
      a[u] = on ? __ldcs(S.val + base + (long long)(k + u) * 32) : 0.0;
      j[u] = on ? __ldcs(S.col + base + (long long)(k + u) * 32) : -1;
    }
#pragma unroll
    for (int u = 0; u < U; ++u) xv[u] = j[u] >= 0 ? __ldg(x + j[u]) : 0.0;
#pragma unroll
    for (int u = 0; u < U; ++u) if (j[u] >= 0) acc = fma(a[u], xv[u], acc);
  }
  if (r >= 0) y[r] = acc;
}

static SellP build_sellp(const Csr& M, int sigma) {
  std::vector<int> ptr(M.rows + 1);
  CK(cudaMemcpy(ptr.data(), M.ptr, (M.rows + 1) * 4, cudaMemcpyDeviceToHost));
  std::vector<int> perm(M.rows);
  for (int i = 0; i < M.rows; ++i) perm[i] = i;
  for (int w0 = 0; w0 < M.rows; w0 += sigma) {
    const int w1 = std::min(M.rows, w0 + sigma);
    std::stable_sort(perm.begin() + w0, perm.begin() + w1,
                     [&](int a, int b) { return ptr[a + 1] - ptr[a] > ptr[b + 1] - ptr[b]; });
  }
  SellP S{};
  S.rows = M.rows;
  S.nslices = (M.rows + 31) / 32;
  int *width, *dperm; long long* sptr;
  CK(cudaMalloc(&dperm, (size_t)M.rows * 4));
  CK(cudaMemcpy(dperm, perm.data(), (size_t)M.rows * 4, cudaMemcpyHostToDevice));
  CK(cudaMalloc(&width, (size_t)S.nslices * 4));
  CK(cudaMalloc(&sptr, (size_t)(S.nslices + 1) * 8));
  k_sellp_width<<<(S.nslices + 255) / 256, 256>>>(M.rows, M.ptr, dperm, width);
  k_sell_w32<<<(S.nslices + 256) / 256, 256>>>(S.nslices, width, sptr);
  void* tmp = nullptr; size_t tb = 0;
  cub::DeviceScan::ExclusiveSum(tmp, tb, sptr, sptr, S.nslices + 1);
  CK(cudaMalloc(&tmp, tb));
  cub::DeviceScan::ExclusiveSum(tmp, tb, sptr, sptr, S.nslices + 1);
  long long tot = 0;
  CK(cudaMemcpy(&tot, sptr + S.nslices, 8, cudaMemcpyDeviceToHost));
  int* scol; double* sval;
  CK(cudaMalloc(&scol, (size_t)tot * 4)); CK(cudaMalloc(&sval, (size_t)tot * 8));
  CK(cudaMemset(scol, 0, (size_t)tot * 4)); CK(cudaMemset(sval, 0, (size_t)tot * 8));
  k_sellp_fill<<<(M.rows + 255) / 256, 256>>>(M.rows, M.ptr, dperm, M.col, M.val, sptr, scol, sval);
  CK(cudaDeviceSynchronize());
  cudaFree(tmp);
  printf("  SELL-32-sigma=%d: %lld slots for %d nnz (%.2fx)\n", sigma, tot, M.nnz, (double)tot / M.nnz);
  S.sptr = sptr; S.width = width; S.ptr = M.ptr; S.perm = dperm; S.col = scol; S.val = sval;
  return S;
}

struct Timer {
  cudaEvent_t a, b;
  Timer() { cudaEventCreate(&a); cudaEventCreate(&b); }
  void start() { cudaEventRecord(a); }
  float stop() { cudaEventRecord(b); cudaEventSynchronize(b); float ms; cudaEventElapsedTime(&ms, a, b); return ms; }
};

int main(int argc, char** argv) {
  int m = 5000000, n = 10000000;
  int *len, *ptr;
  CK(cudaMalloc(&len, (m + 1) * 4)); CK(cudaMalloc(&ptr, (m + 1) * 4));
  k_rowlen<<<(m + 255) / 256, 256>>>(m, len);
  CK(cudaMemset(len + m, 0, 4));
  void* tmp = nullptr; size_t tb = 0;
  cub::DeviceScan::ExclusiveSum(tmp, tb, len, ptr, m + 1);
  CK(cudaMalloc(&tmp, tb));
  cub::DeviceScan::ExclusiveSum(tmp, tb, len, ptr, m + 1);
  int nnz; CK(cudaMemcpy(&nnz, ptr + m, 4, cudaMemcpyDeviceToHost));
  Csr A{m, n, nnz, ptr, nullptr, nullptr};
  CK(cudaMalloc(&A.col, (size_t)nnz * 4)); CK(cudaMalloc(&A.val, (size_t)nnz * 8));
  k_fill<<<(m + 255) / 256, 256>>>(m, n, ptr, A.col, A.val);
  k_sortrows<<<(m + 255) / 256, 256>>>(m, ptr, A.col);
  // transpose
  Csr T{n, m, nnz, nullptr, nullptr, nullptr};
  {
    int *k0, *k1, *v0, *v1, *rid;
    CK(cudaMalloc(&k0, (size_t)nnz * 4)); CK(cudaMalloc(&k1, (size_t)nnz * 4));
    CK(cudaMalloc(&v0, (size_t)nnz * 4)); CK(cudaMalloc(&v1, (size_t)nnz * 4)); CK(cudaMalloc(&rid, (size_t)nnz * 4));
    CK(cudaMemcpy(k0, A.col, (size_t)nnz * 4, cudaMemcpyDeviceToDevice));
    k_iota<<<(nnz + 255) / 256, 256>>>(v0, nnz);
    k_rid<<<(m + 255) / 256, 256>>>(m, ptr, rid);
    cub::DoubleBuffer<int> kb(k0, k1), vb(v0, v1);
    void* t2 = nullptr; size_t b2 = 0;
    cub::DeviceRadixSort::SortPairs(t2, b2, kb, vb, nnz);
    CK(cudaMalloc(&t2, b2));
    cub::DeviceRadixSort::SortPairs(t2, b2, kb, vb, nnz);
    CK(cudaMalloc(&T.ptr, (size_t)(n + 1) * 4)); CK(cudaMalloc(&T.col, (size_t)nnz * 4)); CK(cudaMalloc(&T.val, (size_t)nnz * 8));
    k_gt<<<(nnz + 255) / 256, 256>>>(nnz, vb.Current(), rid, A.val, T.col, T.val);
    k_cptr<<<(n + 256) / 256, 256>>>(kb.Current(), nnz, n, T.ptr);
    CK(cudaDeviceSynchronize());
    cudaFree(k0); cudaFree(k1); cudaFree(v0); cudaFree(v1); cudaFree(rid); cudaFree(t2);
  }
  double *x, *yv, *yref, *ya;
  CK(cudaMalloc(&x, (size_t)n * 8)); CK(cudaMalloc(&yv, (size_t)m * 8));
  CK(cudaMalloc(&yref, (size_t)n * 8)); CK(cudaMalloc(&ya, (size_t)n * 8));
  {
    std::vector<double> hx(n);
    for (int i = 0; i < n; ++i) hx[i] = ((mix64(i) >> 11) * (1.0 / 9007199254740992.0)) - 0.5;
    CK(cudaMemcpy(x, hx.data(), (size_t)n * 8, cudaMemcpyHostToDevice));
    CK(cudaMemcpy(yv, hx.data(), (size_t)m * 8, cudaMemcpyHostToDevice));
  }
  printf("m=%d n=%d nnz=%d\n", m, n, nnz);
  Timer t;
  auto bench = [&](const char* name, const Csr& M, auto fn, const double* xin) {
    for (int w = 0; w < 3; ++w) fn();
    CK(cudaDeviceSynchronize());
    t.start();
    const int R = 20;
    for (int r = 0; r < R; ++r) fn();
    const float ms = t.stop() / R;
    CK(cudaGetLastError());
    // check vs reference result (v1 into yref)
    std::vector<double> a(M.rows), b(M.rows);
    CK(cudaMemcpy(a.data(), ya, (size_t)M.rows * 8, cudaMemcpyDeviceToHost));
    CK(cudaMemcpy(b.data(), yref, (size_t)M.rows * 8, cudaMemcpyDeviceToHost));
    double err = 0;
    for (int i = 0; i < M.rows; ++i) err = fmax(err, fabs(a[i] - b[i]));
    const double bytes = 12.0 * M.nnz + 4.0 * M.rows + 8.0 * M.cols + 8.0 * M.rows;
    printf("%-34s %8.3f ms  %8.1f GB/s  maxdiff %.2e\n", name, ms, bytes / ms / 1e6, err);
  };
  auto grid = [](int rows, int V) { return (unsigned)(((long long)rows * V + 255) / 256); };
  for (int op = 0; op < 2; ++op) {
    const Csr& M = op == 0 ? A : T;
    const double* xin = op == 0 ? x : yv;
    printf("== %s (rows=%d, mean %.1f)\n", op == 0 ? "A x" : "A' y", M.rows, (double)M.nnz / M.rows);
    if (op == 0) v1<8><<<grid(M.rows, 8), 256>>>(M, xin, yref); else v1<4><<<grid(M.rows, 4), 256>>>(M, xin, yref);
#define RUN(NAME, K, VV) bench(NAME, M, [&] { K<<<grid(M.rows, VV), 256>>>(M, xin, ya); }, xin)
#define RUNW(NAME, K) bench(NAME, M, [&] { K<<<(unsigned)((M.rows + 255) / 256), 256>>>(M, xin, ya); }, xin)
    {
      Sell S = build_sell(M);
      const unsigned gs = (unsigned)(((long long)S.nslices * 32 + 255) / 256);
      bench("v10 SELL-32 U=4", M, [&] { v10<4><<<gs, 256>>>(S, xin, ya); }, xin);
      bench("v10 SELL-32 U=8", M, [&] { v10<8><<<gs, 256>>>(S, xin, ya); }, xin);
      {
        double *ec, *ex, *exe, *exb;
        CK(cudaMalloc(&ec, (size_t)M.rows * 8)); CK(cudaMalloc(&ex, (size_t)M.rows * 8));
        CK(cudaMalloc(&exe, (size_t)M.rows * 8)); CK(cudaMalloc(&exb, (size_t)M.rows * 8));
        CK(cudaMemset(ec, 0, (size_t)M.rows * 8)); CK(cudaMemset(ex, 0, (size_t)M.rows * 8));
        CK(cudaMemset(exb, 0, (size_t)M.rows * 8));
        Epi E{ec, ex, exe, exb, 1e-3};
        bench("v12 SELL-32 U=4 + epilogue", M, [&] { v12<4><<<gs, 256>>>(S, xin, E); }, xin);
        cudaFree(ec); cudaFree(ex); cudaFree(exe); cudaFree(exb);
      }
      cudaFree((void*)S.col); cudaFree((void*)S.val);
    }
    for (int sigma : {1024}) {
      SellP S = build_sellp(M, sigma);
      const unsigned gs = (unsigned)(((long long)S.nslices * 32 + 255) / 256);
      bench("v11 SELL-32-sigma U=4", M, [&] { v11<4><<<gs, 256>>>(S, xin, ya); }, xin);
      bench("v11 SELL-32-sigma U=8", M, [&] { v11<8><<<gs, 256>>>(S, xin, ya); }, xin);
      cudaFree((void*)S.col); cudaFree((void*)S.val); cudaFree((void*)S.perm);
    }
    RUNW("v5<16,4>", (v5<16, 4>));
    RUNW("v7<8,4>", (v7<8, 4>));
    // RUNW("v7<8,4,5>", (v7<8, 4, 5>));
    // RUNW("v7<8,4,6>", (v7<8, 4, 6>));
    // RUNW("v7<8,4,8>", (v7<8, 4, 8>));
    RUNW("v7<16,4,5>", (v7<16, 4, 5>));
    // RUNW("v9<8,2,296>", (v9<8, 2, 296>));
    // RUNW("v9<8,2,592>", (v9<8, 2, 592>));
    // RUNW("v9<16,4,296>", (v9<16, 4, 296>));
    // RUNW("v9<16,4,592>", (v9<16, 4, 592>));
    // RUNW("v9<16,4,1184>", (v9<16, 4, 1184>));
  }
  return 0;
}
