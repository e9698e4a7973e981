// Calibration probe (not product code): how fast can a B200 stream a
// config-4-shaped fp64 CSR matrix and gather the vector it multiplies?
// Builds a 5M x 10M, ~200M nnz lognormal-row / banded+uniform-column matrix
// on the device, then times several SpMV variants with CUDA events.
#include <cstdio>
#include <cstdint>
#include <cstdlib>
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
  if (l < 1) l = 1;
  if (l > 2000) l = 2000;
  len[i] = (int)l;
}

__global__ void k_fill(int m, int n, const int* ptr, int* col, double* val) {
  int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= m) return;
  for (int k = ptr[i]; k < ptr[i + 1]; ++k) {
    uint64_t h = mix64(0x1234567ULL ^ (uint64_t)k * 0x100000001b3ULL);
    long c;
    if (u01(h) < 0.7) {
      long center = 2L * i;
      long off = (long)(mix64(h) % 100001ULL) - 50000;
      c = ((center + off) % n + n) % n;
    } else {
      c = (long)(mix64(h + 7) % (uint64_t)n);
    }
    col[k] = (int)c;
    val[k] = u01(mix64(h + 13)) - 0.5;
  }
}

// sort columns inside each row (insertion sort, rows are short)
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

template <int V>
__global__ void __launch_bounds__(256) k_spmv_vec(int m, const int* __restrict__ ptr,
    const int* __restrict__ col, const double* __restrict__ val,
    const double* __restrict__ x, double* __restrict__ y) {
  int gid = blockIdx.x * blockDim.x + threadIdx.x;
  int row = gid / V, lane = gid % V;
  if (row >= m) return;
  int s = ptr[row], e = ptr[row + 1];
  double acc = 0.0;
  for (int k = s + lane; k < e; k += V) acc += __ldcs(val + k) * __ldg(x + __ldcs(col + k));
#pragma unroll
  for (int o = V / 2; o > 0; o >>= 1) acc += __shfl_down_sync(0xffffffff, acc, o, V);
  if (lane == 0) y[row] = acc;
}

// gather-only: isolates the random-read cost
template <int V>
__global__ void __launch_bounds__(256) k_gather_only(int m, const int* __restrict__ ptr,
    const int* __restrict__ col, const double* __restrict__ x, double* __restrict__ y) {
  int gid = blockIdx.x * blockDim.x + threadIdx.x;
  int row = gid / V, lane = gid % V;
  if (row >= m) return;
  int s = ptr[row], e = ptr[row + 1];
  double acc = 0.0;
  for (int k = s + lane; k < e; k += V) acc += __ldg(x + __ldcs(col + k));
#pragma unroll
  for (int o = V / 2; o > 0; o >>= 1) acc += __shfl_down_sync(0xffffffff, acc, o, V);
  if (lane == 0) y[row] = acc;
}

// stream-only: values and indices, no gather
template <int V>
__global__ void __launch_bounds__(256) k_stream_only(int m, const int* __restrict__ ptr,
    const int* __restrict__ col, const double* __restrict__ val, double* __restrict__ y) {
  int gid = blockIdx.x * blockDim.x + threadIdx.x;
  int row = gid / V, lane = gid % V;
  if (row >= m) return;
  int s = ptr[row], e = ptr[row + 1];
  double acc = 0.0;
  for (int k = s + lane; k < e; k += V) acc += __ldcs(val + k) * (double)__ldcs(col + k);
#pragma unroll
  for (int o = V / 2; o > 0; o >>= 1) acc += __shfl_down_sync(0xffffffff, acc, o, V);
  if (lane == 0) y[row] = acc;
}

__global__ void k_copy(const double2* __restrict__ a, double2* __restrict__ b, size_t n) {
  size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x;
  size_t st = (size_t)gridDim.x * blockDim.x;
  for (; i < n; i += st) b[i] = __ldcs(a + i);
}

__global__ void k_gather_rand(const double* __restrict__ x, int n, long cnt, double* out) {
  long i = blockIdx.x * (long)blockDim.x + threadIdx.x;
  long st = (long)gridDim.x * blockDim.x;
  double acc = 0;
  for (; i < cnt; i += st) acc += __ldg(x + (mix64(i) % n));
  if (acc == 12345.678) out[0] = acc;
}


__global__ void k_gather_win(const double* __restrict__ x, int win, long cnt, double* out) {
  long i = blockIdx.x * (long)blockDim.x + threadIdx.x;
  long st = (long)gridDim.x * blockDim.x;
  double acc = 0;
  for (; i < cnt; i += st) acc += __ldg(x + (mix64(i) % win));
  if (acc == 12345.678) out[0] = acc;
}
__global__ void k_gather_smem(int win, long cnt, double* out) {
  extern __shared__ double sm[];
  for (int k = threadIdx.x; k < win; k += blockDim.x) sm[k] = k * 0.5;
  __syncthreads();
  long i = blockIdx.x * (long)blockDim.x + threadIdx.x;
  long st = (long)gridDim.x * blockDim.x;
  double acc = 0;
  for (; i < cnt; i += st) acc += sm[mix64(i) % win];
  if (acc == 12345.678) out[0] = acc;
}
__global__ void k_hash_only(long cnt, double* out) {
  long i = blockIdx.x * (long)blockDim.x + threadIdx.x;
  long st = (long)gridDim.x * blockDim.x;
  double acc = 0;
  for (; i < cnt; i += st) acc += (double)(mix64(i) % 1000);
  if (acc == 12345.678) out[0] = acc;
}
// stream 12 B/nnz with 128-bit loads, flat
__global__ void k_stream_vec(const double2* __restrict__ v, const int4* __restrict__ c, long nq, double* out) {
  long i = blockIdx.x * (long)blockDim.x + threadIdx.x;
  long st = (long)gridDim.x * blockDim.x;
  double acc = 0;
  for (; i < nq; i += st) {
    int4 ci = __ldcs(c + i);
    double2 a = __ldcs(v + 2 * i), b = __ldcs(v + 2 * i + 1);
    acc += a.x * ci.x + a.y * ci.y + b.x * ci.z + b.y * ci.w;
  }
  if (acc == 12345.678) out[0] = acc;
}


template <int MODE>
__global__ void __launch_bounds__(512) k_gidx(const int4* __restrict__ c, long nq, const double* __restrict__ x, int mask, double* out) {
  extern __shared__ double sm[];
  if (MODE == 2) { for (int k = threadIdx.x; k <= mask; k += blockDim.x) sm[k] = k * 0.5; __syncthreads(); }
  long i = blockIdx.x * (long)blockDim.x + threadIdx.x;
  long st = (long)gridDim.x * blockDim.x;
  double acc = 0;
  for (; i < nq; i += st) {
    int4 ci = __ldcs(c + i);
    if (MODE == 0) acc += __ldg(x + ci.x) + __ldg(x + ci.y) + __ldg(x + ci.z) + __ldg(x + ci.w);
    if (MODE == 1) acc += __ldg(x + (ci.x & mask)) + __ldg(x + (ci.y & mask)) + __ldg(x + (ci.z & mask)) + __ldg(x + (ci.w & mask));
    if (MODE == 2) acc += sm[ci.x & mask] + sm[ci.y & mask] + sm[ci.z & mask] + sm[ci.w & mask];
    if (MODE == 3) { int b = (int)(i >> 3) ; acc += __ldg(x + b) + __ldg(x + b + 1) + __ldg(x + b + 2) + __ldg(x + b + 3); }
  }
  if (acc == 12345.678) out[0] = acc;
}

struct Timer {
  cudaEvent_t a, b;
  Timer() { cudaEventCreate(&a); cudaEventCreate(&b); }
  void start() { cudaEventRecord(a); }
  float stop() { cudaEventRecord(b); cudaEventSynchronize(b); float ms; cudaEventElapsedTime(&ms, a, b); return ms; }
};

int main(int argc, char** argv) {
  CK(cudaFuncSetAttribute(k_gather_smem, cudaFuncAttributeMaxDynamicSharedMemorySize, 200*1024));
  CK(cudaFuncSetAttribute(k_gidx<2>, cudaFuncAttributeMaxDynamicSharedMemorySize, 200*1024));
  int m = 5000000, n = 10000000;
  if (argc > 1) m = atoi(argv[1]);
  if (argc > 2) n = atoi(argv[2]);
  int* len; int* ptr;
  CK(cudaMalloc(&len, (m + 1) * sizeof(int)));
  CK(cudaMalloc(&ptr, (m + 1) * sizeof(int)));
  k_rowlen<<<(m + 255) / 256, 256>>>(m, len);
  CK(cudaMemset(len + m, 0, sizeof(int)));
  void* tmp = nullptr; size_t tb = 0;
  cub::DeviceScan::ExclusiveSum(tmp, tb, len, ptr, m + 1);
  CK(cudaMalloc(&tmp, tb));
  cub::DeviceScan::ExclusiveSum(tmp, tb, len, ptr, m + 1);
  int nnz; CK(cudaMemcpy(&nnz, ptr + m, sizeof(int), cudaMemcpyDeviceToHost));
  printf("m=%d n=%d nnz=%d\n", m, n, nnz);
  int* col; double* val; double *x, *y;
  CK(cudaMalloc(&col, (size_t)nnz * 4));
  CK(cudaMalloc(&val, (size_t)nnz * 8));
  CK(cudaMalloc(&x, (size_t)n * 8));
  CK(cudaMalloc(&y, (size_t)m * 8));
  k_fill<<<(m + 255) / 256, 256>>>(m, n, ptr, col, val);
  k_sortrows<<<(m + 255) / 256, 256>>>(m, ptr, col);
  CK(cudaMemset(x, 0, (size_t)n * 8));
  CK(cudaDeviceSynchronize());
  Timer t;
  double algo = 12.0 * nnz + 4.0 * m + 8.0 * n + 8.0 * m;  // matrix + ptr + x once + y write
  auto run = [&](const char* name, auto fn, double bytes) {
    for (int w = 0; w < 3; ++w) fn();
    CK(cudaDeviceSynchronize());
    t.start();
    const int R = 10;
    for (int r = 0; r < R; ++r) fn();
    float ms = t.stop() / R;
    CK(cudaGetLastError());
    printf("%-28s %8.3f ms  %8.1f GB/s\n", name, ms, bytes / ms / 1e6);
  };
  {
    size_t N = (size_t)1 << 28;  // 4 GiB each
    double2 *a, *b;
    CK(cudaMalloc(&a, N * 16)); CK(cudaMalloc(&b, N * 16));
    CK(cudaMemset(a, 0, N * 16));
    run("copy 4GiB", [&] { k_copy<<<148 * 8, 512>>>(a, b, N); }, 2.0 * N * 16);
    CK(cudaFree(a)); CK(cudaFree(b));
  }
  auto blocks = [&](int V) { return (int)(((long)m * V + 255) / 256); };
  run("stream-only V=8", [&] { k_stream_only<8><<<blocks(8), 256>>>(m, ptr, col, val, y); }, 12.0 * nnz + 12.0 * m);
  run("stream-only V=32", [&] { k_stream_only<32><<<blocks(32), 256>>>(m, ptr, col, val, y); }, 12.0 * nnz + 12.0 * m);
  run("gather-only V=8", [&] { k_gather_only<8><<<blocks(8), 256>>>(m, ptr, col, x, y); }, 4.0 * nnz + 12.0 * m);
  run("spmv V=4", [&] { k_spmv_vec<4><<<blocks(4), 256>>>(m, ptr, col, val, x, y); }, algo);
  run("spmv V=8", [&] { k_spmv_vec<8><<<blocks(8), 256>>>(m, ptr, col, val, x, y); }, algo);
  run("spmv V=16", [&] { k_spmv_vec<16><<<blocks(16), 256>>>(m, ptr, col, val, x, y); }, algo);
  run("spmv V=32", [&] { k_spmv_vec<32><<<blocks(32), 256>>>(m, ptr, col, val, x, y); }, algo);
  long cnt = nnz;
  run("random gather 80MB vec", [&] { k_gather_rand<<<148 * 16, 256>>>(x, n, cnt, y); }, 8.0 * cnt);
  run("random gather 8MB vec", [&] { k_gather_rand<<<148 * 16, 256>>>(x, 1000000, cnt, y); }, 8.0 * cnt);

  run("hash-only", [&] { k_hash_only<<<148 * 16, 256>>>(cnt, y); }, 8.0 * cnt);
  run("gather win 8K (64KB, L1)", [&] { k_gather_win<<<148 * 16, 256>>>(x, 8192, cnt, y); }, 8.0 * cnt);
  run("gather win 128K (1MB)", [&] { k_gather_win<<<148 * 16, 256>>>(x, 131072, cnt, y); }, 8.0 * cnt);
  run("gather smem 16K (128KB)", [&] { k_gather_smem<<<148, 1024, 16384 * 8>>>(16384, cnt, y); }, 8.0 * cnt);
  run("gather smem 4K (32KB) x4occ", [&] { k_gather_smem<<<148 * 4, 512, 4096 * 8>>>(4096, cnt, y); }, 8.0 * cnt);
  run("stream vec128 12B/nnz", [&] { k_stream_vec<<<148 * 8, 512>>>((const double2*)val, (const int4*)col, nnz / 4, y); }, 12.0 * (nnz / 4 * 4));

  long nq = nnz / 4;
  run("gidx real cols", [&] { k_gidx<0><<<148 * 4, 512>>>((const int4*)col, nq, x, 0, y); }, 12.0 * nq * 4);
  run("gidx mask 4K (32KB)", [&] { k_gidx<1><<<148 * 4, 512>>>((const int4*)col, nq, x, 4095, y); }, 12.0 * nq * 4);
  run("gidx mask 128K (1MB)", [&] { k_gidx<1><<<148 * 4, 512>>>((const int4*)col, nq, x, 131071, y); }, 12.0 * nq * 4);
  run("gidx mask 4M (32MB)", [&] { k_gidx<1><<<148 * 4, 512>>>((const int4*)col, nq, x, 4194303, y); }, 12.0 * nq * 4);
  run("gidx smem 16K", [&] { k_gidx<2><<<148, 512, 16384 * 8>>>((const int4*)col, nq, x, 16383, y); }, 12.0 * nq * 4);
  run("gidx smem 4K x4", [&] { k_gidx<2><<<148 * 4, 512, 4096 * 8>>>((const int4*)col, nq, x, 4095, y); }, 12.0 * nq * 4);
  run("gidx sequential", [&] { k_gidx<3><<<148 * 4, 512>>>((const int4*)col, nq, x, 0, y); }, 12.0 * nq * 4);
  printf("nnz/s needed for 60%%: %.1f G\n", 4800.0 / 24.0);
  return 0;
}
