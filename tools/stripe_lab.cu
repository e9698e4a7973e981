// stripe_lab.cu -- development lab (not product): column-stripe SpMV for the PDHG steps.
//
// Question: on config 4 the CSR-vector step kernels are bound by L2-slice
// (LTS) throughput -- every gather of the 80 MB / 40 MB vector costs a 32 B
// sector for 8 useful bytes.  The stripe layout serves the dense part of each
// row from shared memory instead: the columns are cut into stripes of W
// (stripe s = columns [sW, (s+1)W)); a (row, stripe) run of >= T entries is a
// *segment* and goes to the stripe part, the rest of the row stays in a
// remote CSR.  Kernel 1 (one 1024-thread CTA per SM) stages a stripe of the
// vector in shared memory once, then computes every segment of that stripe
// (groups of 32 segments, V lanes per segment) and writes one partial per
// segment, coalesced.  Kernel 2 (warp per 32 rows) sums each row's partials in
// stripe order, adds the remote dot (global gathers) and writes the row.
//
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -lineinfo -o tools/stripe_lab tools/stripe_lab.cu
//   tools/stripe_lab [W] [T]
#include <algorithm>
#include <cstdint>
#include <cstdio>
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

// ---------------------------------------------------------------- baseline (product k_step's SpMV)
template <int V, int U>
__device__ __forceinline__ double warp_rows(const int* __restrict__ ptr, const int* __restrict__ col,
                                            const double* __restrict__ val, int rows, long long row0,
                                            int lane, const double* __restrict__ x) {
  constexpr int G = 32 / V;
  const int sub = lane % V;
  const long long rl = row0 + lane;
  int my_s = 0, my_e = 0;
  if (rl < rows) { my_s = ptr[rl]; my_e = ptr[rl + 1]; }
  double mine = 0.0;
  int s = __shfl_sync(0xffffffffu, my_s, lane / V);
  int e = __shfl_sync(0xffffffffu, my_e, lane / V);
  double ac[U];
  int jc[U];
#pragma unroll
  for (int u = 0; u < U; ++u) {
    const int kk = s + sub + u * V;
    ac[u] = kk < e ? __ldcs(val + kk) : 0.0;
    jc[u] = kk < e ? __ldcs(col + kk) : -1;
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
      an[u] = kk < en ? __ldcs(val + kk) : 0.0;
      jn[u] = kk < en ? __ldcs(col + kk) : -1;
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
        a2[u] = kk < e ? __ldcs(val + kk) : 0.0;
        j2[u] = kk < e ? __ldcs(col + kk) : -1;
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
  return mine;
}

template <int V, int U>
__global__ void __launch_bounds__(256) k_csr(Csr A, const double* __restrict__ x, double* __restrict__ y) {
  const int lane = threadIdx.x & 31;
  const long long row0 = (((long long)blockIdx.x * 256 + threadIdx.x) >> 5) * 32;
  if (row0 >= A.rows) return;
  const double d = warp_rows<V, U>(A.ptr, A.col, A.val, A.rows, row0, lane, x);
  if (row0 + lane < A.rows) y[row0 + lane] = d;
}

// ---------------------------------------------------------------- stripe layout
struct Stripes {
  int rows, cols, W, nstripes, ngroups;
  const int* stripe_g;          // nstripes+1
  const int* cta_g;             // ncta+1
  const int* gbase;             // ngroups: first entry of the group
  const unsigned short* cnt;    // ngroups*32
  const double* val;            // stripe entries
  const unsigned short* col16;  // column inside the stripe
  const double* val2;           // same entries, slot-major compacted per group
  const unsigned short* col2;
  const int* seg_ptr;           // rows+1 (per row: its segments' slots, stripe order)
  const int* seg_slot;
  Csr rem;                      // remote entries (CSR, rows x cols)
  // v3: chunk records (TMA bulk-copied): [int4 header][cnt ng*32 u16][col16 ne u16, pad16][val ne f64, pad16]
  const unsigned char* rec;
  const long long* chunk_off;   // nchunks+1 byte offsets into rec
  const int* chunk_stripe;      // nchunks
  const int* cta_chunk;         // ncta+1
};

// One group of 32 segments: lane l's segment is slot g*32+l.  V lanes per
// segment, 32/V segments per pass, all passes' first entries loaded up front.
template <int V>
__device__ __forceinline__ double group_dot(const Stripes& L, int g, int lane, const double* win) {
  constexpr int G = 32 / V;
  const int sub = lane % V;
  const int c = L.cnt[(size_t)g * 32 + lane];
  int incl = c;
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    const int t = __shfl_up_sync(0xffffffffu, incl, o);
    if (lane >= o) incl += t;
  }
  const int my_s = L.gbase[g] + incl - c, my_e = my_s + c;
  double a[V];
  int j[V], kk[V], ee[V];
#pragma unroll
  for (int p = 0; p < V; ++p) {
    const int src = p * G + lane / V;
    const int s = __shfl_sync(0xffffffffu, my_s, src);
    ee[p] = __shfl_sync(0xffffffffu, my_e, src);
    kk[p] = s + sub;
    a[p] = kk[p] < ee[p] ? __ldcs(L.val + kk[p]) : 0.0;
    j[p] = kk[p] < ee[p] ? (int)__ldcs(L.col16 + kk[p]) : -1;
  }
  double mine = 0.0;
#pragma unroll
  for (int p = 0; p < V; ++p) {
    double acc = 0.0;
    if (j[p] >= 0) acc = a[p] * win[j[p]];
    for (int k = kk[p] + V; k < ee[p]; k += V) acc = fma(__ldcs(L.val + k), win[__ldcs(L.col16 + k)], acc);
    acc = gsum<V>(acc);
    const double got = __shfl_sync(0xffffffffu, acc, ((lane - p * G) & (G - 1)) * V);
    if (lane / G == p) mine = got;
  }
  return mine;
}

template <int V>
__global__ void __launch_bounds__(1024, 1) k_stripe(Stripes L, const double* __restrict__ x,
                                                    double* __restrict__ part) {
  extern __shared__ double win[];
  const int g0 = L.cta_g[blockIdx.x], g1 = L.cta_g[blockIdx.x + 1];
  if (g0 >= g1) return;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31, nw = blockDim.x >> 5;
  int lo = 0, hi = L.nstripes;  // last s with stripe_g[s] <= g0
  while (hi - lo > 1) { const int mid = (lo + hi) >> 1; if (L.stripe_g[mid] <= g0) lo = mid; else hi = mid; }
  int s = lo, g = g0;
  while (g < g1) {
    const int ge = min(g1, L.stripe_g[s + 1]);
    if (ge > g) {
      __syncthreads();
      const long long c0 = (long long)s * L.W;
      const int len = (int)min((long long)L.W, L.cols - c0);
      for (int k = threadIdx.x; k < len; k += blockDim.x) win[k] = __ldg(x + c0 + k);
      __syncthreads();
      for (int gg = g + warp; gg < ge; gg += nw) {
        const double d = group_dot<V>(L, gg, lane, win);
        part[(size_t)gg * 32 + lane] = d;
      }
    }
    g = ge;
    ++s;
  }
}

// v2: slot-major compacted groups, one warp per group at a time, the next
// group's entries issued before the current group is consumed (register
// double buffering), cnt/gbase prefetched two groups ahead.
template <int KMAX>
__device__ __forceinline__ int issue_group(const Stripes& L, int c, int base, int lane, double (&a)[KMAX],
                                           int (&j)[KMAX]) {
  const unsigned lt = (1u << lane) - 1u;
#pragma unroll
  for (int k = 0; k < KMAX; ++k) {
    const unsigned mask = __ballot_sync(0xffffffffu, c > k);
    const int idx = base + __popc(mask & lt);
    a[k] = c > k ? __ldcs(L.val2 + idx) : 0.0;
    j[k] = c > k ? (int)__ldcs(L.col2 + idx) : -1;
    base += __popc(mask);
  }
  return base;
}

template <int KMAX>
__device__ __forceinline__ double consume_group(const Stripes& L, int c, int tail, int lane,
                                                const double (&a)[KMAX], const int (&j)[KMAX],
                                                const double* win) {
  double acc = 0.0;
#pragma unroll
  for (int k = 0; k < KMAX; ++k)
    if (j[k] >= 0) acc = (k == 0) ? a[k] * win[j[k]] : fma(a[k], win[j[k]], acc);
  const unsigned lt = (1u << lane) - 1u;
  for (int k = KMAX; __any_sync(0xffffffffu, c > k); ++k) {  // rare: segments longer than KMAX
    const unsigned mask = __ballot_sync(0xffffffffu, c > k);
    if (c > k) {
      const int idx = tail + __popc(mask & lt);
      acc = fma(__ldcs(L.val2 + idx), win[__ldcs(L.col2 + idx)], acc);
    }
    tail += __popc(mask);
  }
  return acc;
}

template <int KMAX, int NT>
__global__ void __launch_bounds__(NT, 1) k_stripe2(Stripes L, const double* __restrict__ x,
                                                   double* __restrict__ part) {
  extern __shared__ double win[];
  const int g0 = L.cta_g[blockIdx.x], g1 = L.cta_g[blockIdx.x + 1];
  if (g0 >= g1) return;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  constexpr int nw = NT / 32;
  int lo = 0, hi = L.nstripes;
  while (hi - lo > 1) { const int mid = (lo + hi) >> 1; if (L.stripe_g[mid] <= g0) lo = mid; else hi = mid; }
  for (int s = lo, g = g0; g < g1; ++s) {
    const int ge = min(g1, L.stripe_g[s + 1]);
    if (ge <= g) continue;
    int gc = g + warp;
    int c_cur = 0, b_cur = 0, c_nx = 0, b_nx = 0;
    if (gc < ge) { c_cur = L.cnt[(size_t)gc * 32 + lane]; b_cur = L.gbase[gc]; }
    if (gc + nw < ge) { c_nx = L.cnt[(size_t)(gc + nw) * 32 + lane]; b_nx = L.gbase[gc + nw]; }
    __syncthreads();
    {
      const long long c0 = (long long)s * L.W;
      const int len = (int)min((long long)L.W, L.cols - c0);
      const double2* src = reinterpret_cast<const double2*>(x + c0);
      double2* dst = reinterpret_cast<double2*>(win);
      for (int k = threadIdx.x; k < len / 2; k += NT) dst[k] = __ldg(src + k);
      if ((len & 1) && threadIdx.x == 0) win[len - 1] = __ldg(x + c0 + len - 1);
    }
    double a[KMAX];
    int j[KMAX];
    int tail = 0;
    if (gc < ge) tail = issue_group<KMAX>(L, c_cur, b_cur, lane, a, j);
    __syncthreads();
    for (; gc < ge; gc += nw) {
      const int gn = gc + nw, gn2 = gc + 2 * nw;
      int c_n2 = 0, b_n2 = 0;
      if (gn2 < ge) { c_n2 = L.cnt[(size_t)gn2 * 32 + lane]; b_n2 = L.gbase[gn2]; }
      double an[KMAX];
      int jn[KMAX];
      int tailn = 0;
      if (gn < ge) tailn = issue_group<KMAX>(L, c_nx, b_nx, lane, an, jn);
      const double d = consume_group<KMAX>(L, c_cur, tail, lane, a, j, win);
      part[(size_t)gc * 32 + lane] = d;
#pragma unroll
      for (int k = 0; k < KMAX; ++k) { a[k] = an[k]; j[k] = jn[k]; }
      tail = tailn;
      c_cur = c_nx; c_nx = c_n2; b_nx = b_n2;
    }
    g = ge;
  }
}

template <int V, int U>
__global__ void __launch_bounds__(256) k_final2(Stripes L, const double* __restrict__ part,
                                                const double* __restrict__ x, double* __restrict__ y) {
  const int lane = threadIdx.x & 31;
  const long long row0 = (((long long)blockIdx.x * 256 + threadIdx.x) >> 5) * 32;
  if (row0 >= L.rows) return;
  const long long rl = row0 + lane;
  int a = 0, b = 0;
  if (rl < L.rows) { a = L.seg_ptr[rl]; b = L.seg_ptr[rl + 1]; }
  constexpr int KP = 8;
  int sl[KP];
#pragma unroll
  for (int u = 0; u < KP; ++u) sl[u] = a + u < b ? __ldcs(L.seg_slot + a + u) : -1;
  double pv[KP];
#pragma unroll
  for (int u = 0; u < KP; ++u) pv[u] = sl[u] >= 0 ? __ldcg(part + sl[u]) : 0.0;
  const double d = warp_rows<V, U>(L.rem.ptr, L.rem.col, L.rem.val, L.rem.rows, row0, lane, x);
  double ps = 0.0;
#pragma unroll
  for (int u = 0; u < KP; ++u) if (sl[u] >= 0) ps += pv[u];
  for (int k = a + KP; k < b; ++k) ps += __ldcg(part + __ldcs(L.seg_slot + k));
  if (rl < L.rows) y[rl] = ps + d;
}

template <int V, int U>
__global__ void __launch_bounds__(256) k_final(Stripes L, const double* __restrict__ part,
                                               const double* __restrict__ x, double* __restrict__ y) {
  const int lane = threadIdx.x & 31;
  const long long row0 = (((long long)blockIdx.x * 256 + threadIdx.x) >> 5) * 32;
  if (row0 >= L.rows) return;
  const long long rl = row0 + lane;
  double ps = 0.0;
  if (rl < L.rows) {
    const int a = L.seg_ptr[rl], b = L.seg_ptr[rl + 1];
    for (int k = a; k < b; k += 4) {
      double t[4];
#pragma unroll
      for (int u = 0; u < 4; ++u) t[u] = (k + u < b) ? __ldcg(part + __ldcs(L.seg_slot + k + u)) : 0.0;
#pragma unroll
      for (int u = 0; u < 4; ++u) if (k + u < b) ps += t[u];
    }
  }
  const double d = warp_rows<V, U>(L.rem.ptr, L.rem.col, L.rem.val, L.rem.rows, row0, lane, x);
  if (rl < L.rows) y[rl] = ps + d;
}

// ---------------------------------------------------------------- v3: TMA-fed chunks
__device__ __forceinline__ uint32_t saddr(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }
__device__ __forceinline__ void mbar_init(uint64_t* bar, uint32_t count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(saddr(bar)), "r"(count) : "memory");
}
__device__ __forceinline__ void fence_mbar_init() { asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory"); }
__device__ __forceinline__ void fence_proxy_async() { asm volatile("fence.proxy.async.shared::cta;" ::: "memory"); }
__device__ __forceinline__ void mbar_expect_tx(uint64_t* bar, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(saddr(bar)), "r"(bytes) : "memory");
}
__device__ __forceinline__ void bulk_g2s(void* dst, const void* src, uint32_t bytes, uint64_t* bar) {
  asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];"
               ::"r"(saddr(dst)), "l"(src), "r"(bytes), "r"(saddr(bar)) : "memory");
}
__device__ __forceinline__ void mbar_wait(uint64_t* bar, uint32_t parity) {
  uint32_t done = 0;
  while (!done) {
    asm volatile("{\n .reg .pred p;\n mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\n selp.u32 %0, 1, 0, p;\n}\n"
                 : "=r"(done) : "r"(saddr(bar)), "r"(parity) : "memory");
  }
}

constexpr int kStage3 = 5328;  // 16 + 8*64 + 480*2 + 480*8 (CE = 480 entries, CG = 8 groups)

template <int NW, int NS>
__global__ void __launch_bounds__(NW * 32, 1) k_stripe3(Stripes L, const double* __restrict__ x,
                                                        double* __restrict__ part) {
  extern __shared__ __align__(16) unsigned char smem3[];
  double* win = reinterpret_cast<double*>(smem3);
  unsigned char* ring = smem3 + (size_t)L.W * 8;
  uint64_t* bars = reinterpret_cast<uint64_t*>(ring + (size_t)NW * NS * kStage3);
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int c0 = L.cta_chunk[blockIdx.x], c1 = L.cta_chunk[blockIdx.x + 1];
  if (c0 >= c1) return;
  uint64_t* mybar = bars + warp * NS;
  unsigned char* mystage = ring + (size_t)warp * NS * kStage3;
  if (lane == 0) {
    for (int s = 0; s < NS; ++s) mbar_init(&mybar[s], 1);
    fence_mbar_init();
  }
  __syncthreads();
  auto issue = [&](int ord) {
    const int c = c0 + warp + ord * NW;
    if (c >= c1) return;
    const long long o0 = L.chunk_off[c], o1 = L.chunk_off[c + 1];
    const int s = ord % NS;
    mbar_expect_tx(&mybar[s], (uint32_t)(o1 - o0));
    bulk_g2s(mystage + (size_t)s * kStage3, L.rec + o0, (uint32_t)(o1 - o0), &mybar[s]);
  };
  if (lane == 0) {
    fence_proxy_async();
    for (int k = 0; k < NS; ++k) issue(k);
  }
  const unsigned lt = (1u << lane) - 1u;
  int ord = 0;
  int cs = c0;
  while (cs < c1) {
    const int stripe = L.chunk_stripe[cs];
    int ce = cs + 1;
    while (ce < c1 && L.chunk_stripe[ce] == stripe) ++ce;
    __syncthreads();
    {
      const long long col0 = (long long)stripe * L.W;
      const int len = (int)min((long long)L.W, L.cols - col0);
      const double2* src = reinterpret_cast<const double2*>(x + col0);
      double2* dst = reinterpret_cast<double2*>(win);
#pragma unroll 8
      for (int k = threadIdx.x; k < len / 2; k += NW * 32) dst[k] = __ldg(src + k);
      if ((len & 1) && threadIdx.x == 0) win[len - 1] = __ldg(x + col0 + len - 1);
    }
    __syncthreads();
    for (; c0 + warp + ord * NW < ce; ++ord) {
      const int s = ord % NS;
      mbar_wait(&mybar[s], (uint32_t)((ord / NS) & 1));
      const unsigned char* st = mystage + (size_t)s * kStage3;
      const int4 hdr = *reinterpret_cast<const int4*>(st);
      const unsigned short* cntp = reinterpret_cast<const unsigned short*>(st + 16);
      const unsigned short* colp = cntp + hdr.x * 32;
      const double* valp = reinterpret_cast<const double*>(st + 16 + hdr.x * 64 + ((hdr.y * 2 + 15) & ~15));
      int base = 0;
      for (int gi = 0; gi < hdr.x; ++gi) {
        const int c = cntp[gi * 32 + lane];
        const int maxc = __reduce_max_sync(0xffffffffu, c);
        double acc = 0.0;
        for (int k = 0; k < maxc; k += 4) {
          double a[4];
          int j[4];
#pragma unroll
          for (int u = 0; u < 4; ++u) {
            const unsigned mask = __ballot_sync(0xffffffffu, c > k + u);
            const int idx = base + __popc(mask & lt);
            a[u] = c > k + u ? valp[idx] : 0.0;
            j[u] = c > k + u ? (int)colp[idx] : -1;
            base += __popc(mask);
          }
#pragma unroll
          for (int u = 0; u < 4; ++u)
            if (j[u] >= 0) acc = (k + u == 0) ? a[u] * win[j[u]] : fma(a[u], win[j[u]], acc);
        }
        part[(size_t)(hdr.z + gi) * 32 + lane] = acc;
      }
      __syncwarp();
      if (lane == 0) {
        fence_proxy_async();
        issue(ord + NS);
      }
    }
    cs = ce;
  }
}

struct HostStripes {
  Stripes d;
  long long stripe_ent, remote_ent, nseg, nchunks, rec_bytes;
  int ncta;
};

static HostStripes build_stripes(const Csr& M, int W, int T, int ncta, int smax = 0, int CE = 512, int CG = 8) {
  std::vector<int> ptr(M.rows + 1), col(M.nnz);
  std::vector<double> val(M.nnz);
  CK(cudaMemcpy(ptr.data(), M.ptr, (M.rows + 1) * 4, cudaMemcpyDeviceToHost));
  CK(cudaMemcpy(col.data(), M.col, (size_t)M.nnz * 4, cudaMemcpyDeviceToHost));
  CK(cudaMemcpy(val.data(), M.val, (size_t)M.nnz * 8, cudaMemcpyDeviceToHost));
  const int ns = (M.cols + W - 1) / W;
  std::vector<long long> segc(ns, 0), entc(ns, 0);
  std::vector<int> remc(M.rows, 0);
  for (int i = 0; i < M.rows; ++i) {
    int k = ptr[i];
    const int e = ptr[i + 1];
    while (k < e) {
      const int s = col[k] / W;
      int r = k;
      while (r < e && col[r] / W == s) ++r;
      if (r - k >= T) { segc[s] += smax > 0 ? (r - k + smax - 1) / smax : 1; entc[s] += r - k; } else remc[i] += r - k;
      k = r;
    }
  }
  std::vector<int> stripe_g(ns + 1, 0);
  std::vector<long long> e0(ns + 1, 0);
  for (int s = 0; s < ns; ++s) {
    stripe_g[s + 1] = stripe_g[s] + (int)((segc[s] + 31) / 32);
    e0[s + 1] = e0[s] + entc[s];
  }
  const int G = stripe_g[ns];
  const long long NE = e0[ns];
  std::vector<unsigned short> cnt((size_t)G * 32, 0);
  std::vector<double> sval(NE);
  std::vector<unsigned short> scol(NE);
  std::vector<int> seg_ptr(M.rows + 1, 0), seg_slot;
  std::vector<int> rptr(M.rows + 1, 0);
  for (int i = 0; i < M.rows; ++i) rptr[i + 1] = rptr[i] + remc[i];
  std::vector<int> rcol(rptr[M.rows]);
  std::vector<double> rval(rptr[M.rows]);
  std::vector<long long> segfill(ns, 0), ecur(e0.begin(), e0.end() - 1);
  seg_slot.reserve(M.nnz / 4);
  for (int i = 0; i < M.rows; ++i) {
    int k = ptr[i], rc = rptr[i];
    const int e = ptr[i + 1];
    while (k < e) {
      const int s = col[k] / W;
      int r = k;
      while (r < e && col[r] / W == s) ++r;
      if (r - k >= T) {
        for (int k2 = k; k2 < r;) {
          const int r2 = smax > 0 ? std::min(r, k2 + smax) : r;
          const long long slot = (long long)stripe_g[s] * 32 + segfill[s]++;
          cnt[slot] = (unsigned short)(r2 - k2);
          seg_slot.push_back((int)slot);
          for (int q = k2; q < r2; ++q) { sval[ecur[s]] = val[q]; scol[ecur[s]] = (unsigned short)(col[q] - s * W); ++ecur[s]; }
          k2 = r2;
        }
      } else {
        for (int q = k; q < r; ++q) { rcol[rc] = col[q]; rval[rc] = val[q]; ++rc; }
      }
      k = r;
    }
    seg_ptr[i + 1] = (int)seg_slot.size();
  }
  std::vector<int> gbase(G);
  for (int s = 0; s < ns; ++s) {
    long long off = e0[s];
    for (int g = stripe_g[s]; g < stripe_g[s + 1]; ++g) {
      gbase[g] = (int)off;
      for (int l = 0; l < 32; ++l) off += cnt[(size_t)g * 32 + l];
    }
  }
  // slot-major compacted copy: slot k of group g holds the k-th entry of each
  // segment with more than k entries, in lane order
  std::vector<double> sval2(NE);
  std::vector<unsigned short> scol2(NE);
  for (int g = 0; g < G; ++g) {
    const unsigned short* cg = &cnt[(size_t)g * 32];
    int st[32], mx = 0;
    int o = gbase[g];
    for (int l = 0; l < 32; ++l) { st[l] = o; o += cg[l]; mx = std::max(mx, (int)cg[l]); }
    int w = gbase[g];
    for (int k = 0; k < mx; ++k)
      for (int l = 0; l < 32; ++l)
        if (cg[l] > k) { sval2[w] = sval[st[l] + k]; scol2[w] = scol[st[l] + k]; ++w; }
  }
  // CTA ranges: equal cost, cost(group) = entries + 32 * 6 (per-segment overhead)
  std::vector<long long> cum(G + 1, 0);
  for (int g = 0; g < G; ++g) {
    long long c = 32 * 6;
    for (int l = 0; l < 32; ++l) c += cnt[(size_t)g * 32 + l];
    cum[g + 1] = cum[g] + c;
  }
  std::vector<int> cta_g(ncta + 1, 0);
  for (int c = 0; c <= ncta; ++c) {
    const long long target = cum[G] * c / ncta;
    cta_g[c] = (int)(std::lower_bound(cum.begin(), cum.end(), target) - cum.begin());
  }
  cta_g[ncta] = G;
  // chunk records for v3: per CTA, consecutive groups of one stripe, <= CE entries, <= CG groups
  std::vector<unsigned char> rec;
  std::vector<long long> chunk_off;
  std::vector<int> chunk_stripe, cta_chunk(ncta + 1, 0);
  {
    std::vector<int> g_stripe(G);
    for (int s2 = 0; s2 < ns; ++s2) for (int g = stripe_g[s2]; g < stripe_g[s2 + 1]; ++g) g_stripe[g] = s2;
    auto gent = [&](int g) { int t = 0; for (int l = 0; l < 32; ++l) t += cnt[(size_t)g * 32 + l]; return t; };
    auto pad16 = [](size_t v) { return (v + 15) & ~(size_t)15; };
    auto emit = [&](int ga, int gb) {
      int ne = 0;
      for (int g = ga; g < gb; ++g) ne += gent(g);
      const size_t off = rec.size();
      const int ng = gb - ga;
      const size_t hb = 16, cb = (size_t)ng * 64, colb = pad16((size_t)ne * 2), vb = pad16((size_t)ne * 8);
      rec.resize(off + hb + cb + colb + vb, 0);
      int hdr[4] = {ng, ne, ga, g_stripe[ga]};
      memcpy(&rec[off], hdr, 16);
      memcpy(&rec[off + hb], &cnt[(size_t)ga * 32], cb);
      if (ne) {
        memcpy(&rec[off + hb + cb], &scol2[gbase[ga]], (size_t)ne * 2);
        memcpy(&rec[off + hb + cb + colb], &sval2[gbase[ga]], (size_t)ne * 8);
      }
      chunk_off.push_back((long long)off);
      chunk_stripe.push_back(g_stripe[ga]);
    };
    for (int c = 0; c < ncta; ++c) {
      cta_chunk[c] = (int)chunk_off.size();
      int ga = cta_g[c];
      while (ga < cta_g[c + 1]) {
        int gb = ga, ne = 0;
        while (gb < cta_g[c + 1] && gb - ga < CG && g_stripe[gb] == g_stripe[ga] && ne + gent(gb) <= CE) {
          ne += gent(gb);
          ++gb;
        }
        if (gb == ga) { fprintf(stderr, "group %d has %d entries > CE %d\n", ga, gent(ga), CE); exit(1); }
        emit(ga, gb);
        ga = gb;
      }
    }
    cta_chunk[ncta] = (int)chunk_off.size();
    chunk_off.push_back((long long)rec.size());
  }
  auto up = [](const void* h, size_t bytes) { void* d; CK(cudaMalloc(&d, bytes ? bytes : 8)); if (bytes) CK(cudaMemcpy(d, h, bytes, cudaMemcpyHostToDevice)); return d; };
  HostStripes H{};
  Stripes& L = H.d;
  L.rows = M.rows; L.cols = M.cols; L.W = W; L.nstripes = ns; L.ngroups = G;
  L.stripe_g = (int*)up(stripe_g.data(), stripe_g.size() * 4);
  L.cta_g = (int*)up(cta_g.data(), cta_g.size() * 4);
  L.gbase = (int*)up(gbase.data(), gbase.size() * 4);
  L.cnt = (unsigned short*)up(cnt.data(), cnt.size() * 2);
  L.val = (double*)up(sval.data(), sval.size() * 8);
  L.col16 = (unsigned short*)up(scol.data(), scol.size() * 2);
  L.val2 = (double*)up(sval2.data(), sval2.size() * 8);
  L.col2 = (unsigned short*)up(scol2.data(), scol2.size() * 2);
  L.seg_ptr = (int*)up(seg_ptr.data(), seg_ptr.size() * 4);
  L.seg_slot = (int*)up(seg_slot.data(), seg_slot.size() * 4);
  L.rem.rows = M.rows; L.rem.cols = M.cols; L.rem.nnz = rptr[M.rows];
  L.rem.ptr = (int*)up(rptr.data(), rptr.size() * 4);
  L.rem.col = (int*)up(rcol.data(), rcol.size() * 4);
  L.rem.val = (double*)up(rval.data(), rval.size() * 8);
  L.rec = (unsigned char*)up(rec.data(), rec.size());
  L.chunk_off = (long long*)up(chunk_off.data(), chunk_off.size() * 8);
  L.chunk_stripe = (int*)up(chunk_stripe.data(), chunk_stripe.size() * 4);
  L.cta_chunk = (int*)up(cta_chunk.data(), cta_chunk.size() * 4);
  H.nchunks = (long long)chunk_stripe.size();
  H.rec_bytes = (long long)rec.size();
  H.stripe_ent = NE; H.remote_ent = rptr[M.rows]; H.nseg = (long long)seg_slot.size(); H.ncta = ncta;
  return H;
}

struct Timer {
  cudaEvent_t a, b;
  Timer() { cudaEventCreate(&a); cudaEventCreate(&b); }
  void start() { cudaEventRecord(a); }
  float stop() { cudaEventRecord(b); cudaEventSynchronize(b); float ms; cudaEventElapsedTime(&ms, a, b); return ms; }
};

int main(int argc, char** argv) {
  const int W = argc > 1 ? atoi(argv[1]) : 16384;
  const int T = argc > 2 ? atoi(argv[2]) : 2;
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
  Csr T2{n, m, nnz, nullptr, nullptr, nullptr};
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
    CK(cudaMalloc(&T2.ptr, (size_t)(n + 1) * 4)); CK(cudaMalloc(&T2.col, (size_t)nnz * 4)); CK(cudaMalloc(&T2.val, (size_t)nnz * 8));
    k_gt<<<(nnz + 255) / 256, 256>>>(nnz, vb.Current(), rid, A.val, T2.col, T2.val);
    k_cptr<<<(n + 256) / 256, 256>>>(kb.Current(), nnz, n, T2.ptr);
    CK(cudaDeviceSynchronize());
    cudaFree(k0); cudaFree(k1); cudaFree(v0); cudaFree(v1); cudaFree(rid); cudaFree(t2);
  }
  double *x, *yv, *yref, *ya, *part;
  CK(cudaMalloc(&x, (size_t)n * 8)); CK(cudaMalloc(&yv, (size_t)m * 8));
  CK(cudaMalloc(&yref, (size_t)n * 8)); CK(cudaMalloc(&ya, (size_t)n * 8));
  {
    std::vector<double> hx(n);
    for (int i = 0; i < n; ++i) hx[i] = ((mix64(i) >> 11) * (1.0 / 9007199254740992.0)) - 0.5;
    CK(cudaMemcpy(x, hx.data(), (size_t)n * 8, cudaMemcpyHostToDevice));
    CK(cudaMemcpy(yv, hx.data(), (size_t)m * 8, cudaMemcpyHostToDevice));
  }
  int nsm = 0;
  CK(cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, 0));
  printf("m=%d n=%d nnz=%d W=%d T=%d sms=%d\n", m, n, nnz, W, T, nsm);
  Timer t;
  auto timeit = [&](auto fn) {
    for (int w = 0; w < 3; ++w) fn();
    CK(cudaDeviceSynchronize());
    t.start();
    const int R = 20;
    for (int r = 0; r < R; ++r) fn();
    const float ms = t.stop() / R;
    CK(cudaGetLastError());
    return ms;
  };
  auto maxrel = [&](int rows) {
    std::vector<double> a(rows), b(rows);
    CK(cudaMemcpy(a.data(), ya, (size_t)rows * 8, cudaMemcpyDeviceToHost));
    CK(cudaMemcpy(b.data(), yref, (size_t)rows * 8, cudaMemcpyDeviceToHost));
    double err = 0, sc = 0;
    for (int i = 0; i < rows; ++i) { err = fmax(err, fabs(a[i] - b[i])); sc = fmax(sc, fabs(b[i])); }
    return err / sc;
  };
  auto g256 = [](long long rows) { return (unsigned)((rows + 255) / 256); };
  const size_t smem = (size_t)W * 8;
  for (int op = 0; op < 2; ++op) {
    const Csr& M = op == 0 ? A : T2;
    const double* xin = op == 0 ? x : yv;
    printf("== %s (rows=%d, mean %.1f)\n", op == 0 ? "A x (dual)" : "A' y (primal)", M.rows, (double)M.nnz / M.rows);
    float tb0;
    if (op == 0) tb0 = timeit([&] { k_csr<16, 4><<<g256(M.rows), 256>>>(M, xin, yref); });
    else tb0 = timeit([&] { k_csr<8, 4><<<g256(M.rows), 256>>>(M, xin, yref); });
    printf("  baseline csr-vector          %8.3f ms\n", tb0);
    for (int WW : {W}) {
      HostStripes H = build_stripes(M, WW, T, nsm);
      CK(cudaMalloc(&part, (size_t)H.d.ngroups * 32 * 8));
      printf("  stripes W=%d: %lld stripe entries (%.1f%%), %lld segments (mean %.2f), %lld remote, groups %d (pad %.1f%%)\n",
             WW, H.stripe_ent, 100.0 * H.stripe_ent / M.nnz, H.nseg, (double)H.stripe_ent / H.nseg,
             H.remote_ent, H.d.ngroups, 100.0 * (H.d.ngroups * 32.0 - H.nseg) / H.nseg);
      auto runs = [&](auto ks, auto kf, const char* name) {
        CK(cudaFuncSetAttribute(ks, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
        const float t1 = timeit([&] { ks<<<H.ncta, 1024, smem>>>(H.d, xin, part); });
        const float t2 = timeit([&] { kf<<<g256(M.rows), 256>>>(H.d, part, xin, ya); });
        const float t3 = timeit([&] { ks<<<H.ncta, 1024, smem>>>(H.d, xin, part); kf<<<g256(M.rows), 256>>>(H.d, part, xin, ya); });
        printf("  %-28s stripe %7.3f  final %7.3f  both %7.3f ms  (%.2fx)  maxrel %.2e\n", name, t1, t2, t3, tb0 / t3, maxrel(M.rows));
      };
      {
        HostStripes H3 = build_stripes(M, WW, T, nsm, 15, 480, 8);
        double* part3;
        CK(cudaMalloc(&part3, (size_t)H3.d.ngroups * 32 * 8));
        constexpr int NW3 = 6, NS3 = 3;
        const size_t smem3 = (size_t)WW * 8 + (size_t)NW3 * NS3 * kStage3 + NW3 * NS3 * 8;
        auto ks = k_stripe3<NW3, NS3>;
        CK(cudaFuncSetAttribute(ks, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem3));
        printf("  v3: %lld stripe entries, %lld segments (mean %.2f), %lld chunks, %.1f MB records, smem %zu\n",
               H3.stripe_ent, H3.nseg, (double)H3.stripe_ent / H3.nseg, H3.nchunks, H3.rec_bytes / 1e6, smem3);
        const float t1 = timeit([&] { ks<<<H3.ncta, NW3 * 32, smem3>>>(H3.d, xin, part3); });
        float t2, t3;
        if (op == 0) {
          t2 = timeit([&] { k_final<8, 4><<<g256(M.rows), 256>>>(H3.d, part3, xin, ya); });
          t3 = timeit([&] { ks<<<H3.ncta, NW3 * 32, smem3>>>(H3.d, xin, part3); k_final<8, 4><<<g256(M.rows), 256>>>(H3.d, part3, xin, ya); });
        } else {
          t2 = timeit([&] { k_final<4, 4><<<g256(M.rows), 256>>>(H3.d, part3, xin, ya); });
          t3 = timeit([&] { ks<<<H3.ncta, NW3 * 32, smem3>>>(H3.d, xin, part3); k_final<4, 4><<<g256(M.rows), 256>>>(H3.d, part3, xin, ya); });
        }
        printf("  %-28s stripe %7.3f  final %7.3f  both %7.3f ms  (%.2fx)  maxrel %.2e\n", "v3 TMA chunks", t1, t2, t3,
               tb0 / t3, maxrel(M.rows));
        cudaFree(part3);
      }
      auto runs2 = [&](auto ks, int nt, auto kf, const char* name) {
        CK(cudaFuncSetAttribute(ks, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
        const float t1 = timeit([&] { ks<<<H.ncta, nt, smem>>>(H.d, xin, part); });
        const float t2 = timeit([&] { kf<<<g256(M.rows), 256>>>(H.d, part, xin, ya); });
        const float t3 = timeit([&] { ks<<<H.ncta, nt, smem>>>(H.d, xin, part); kf<<<g256(M.rows), 256>>>(H.d, part, xin, ya); });
        printf("  %-28s stripe %7.3f  final %7.3f  both %7.3f ms  (%.2fx)  maxrel %.2e\n", name, t1, t2, t3, tb0 / t3, maxrel(M.rows));
      };
      cudaFree(part);
    }
  }
  return 0;
}
