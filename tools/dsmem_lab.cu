// dsmem_lab.cu -- random 8-byte gathers served from distributed shared memory
// (a cluster's pooled shared memory) vs the same gathers from global memory.
//
// Question: can a column window of the iterate held in a cluster's shared
// memory serve the band gathers of the step kernels faster than L2?
//
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -o tools/dsmem_lab tools/dsmem_lab.cu
//   tools/dsmem_lab
#include <cooperative_groups.h>
#include <cuda_runtime.h>

#include <cstdio>
#include <cstdlib>
#include <vector>

namespace cg = cooperative_groups;

#define CK(x)                                                                             \
  do {                                                                                    \
    cudaError_t e = (x);                                                                  \
    if (e != cudaSuccess) {                                                               \
      printf("%s:%d %s: %s\n", __FILE__, __LINE__, #x, cudaGetErrorString(e));            \
      exit(1);                                                                            \
    }                                                                                     \
  } while (0)

constexpr int kThreads = 1024;

// Each thread: R rounds of U independent gathers at indices idx[...] (streamed,
// coalesced), summing the values.  MODE 0: cluster DSMEM window (W doubles per
// CTA, CL CTAs), 1: local smem only (index mod W), 2: global vector.
template <int MODE, int U>
__global__ void __launch_bounds__(kThreads, 1) k_gather(const int* __restrict__ idx, long long n_idx,
                                                        const double* __restrict__ g, int W, int CL,
                                                        double* __restrict__ out) {
  extern __shared__ double win[];
  cg::cluster_group cluster = cg::this_cluster();
  if (MODE != 2) {
    const unsigned rank = cluster.block_rank();
    for (int i = threadIdx.x; i < W; i += blockDim.x) win[i] = g[(long long)rank * W + i];
    cluster.sync();
  }
  double acc = 0.0;
  const long long stride = (long long)gridDim.x * blockDim.x;
  for (long long base = (long long)blockIdx.x * blockDim.x + threadIdx.x; base < n_idx; base += stride * U) {
    int j[U];
    double v[U];
#pragma unroll
    for (int u = 0; u < U; ++u) {
      const long long p = base + u * stride;
      j[u] = p < n_idx ? __ldcs(idx + p) : -1;
    }
#pragma unroll
    for (int u = 0; u < U; ++u) {
      if (j[u] < 0) {
        v[u] = 0.0;
      } else if (MODE == 0) {
        const int r = j[u] / W, o = j[u] - r * W;
        const double* rp = cluster.map_shared_rank(win, r);
        v[u] = rp[o];
      } else if (MODE == 1) {
        v[u] = win[j[u] % W];
      } else {
        v[u] = __ldg(g + j[u]);
      }
    }
#pragma unroll
    for (int u = 0; u < U; ++u) acc += v[u];
  }
  if (MODE != 2) cluster.sync();  // keep every window alive until the cluster is done
  out[(long long)blockIdx.x * blockDim.x + threadIdx.x] = acc;
}

template <int MODE, int U>
float run(const int* idx, long long n, const double* g, int W, int CL, double* out, int grid) {
  const size_t smem = MODE == 2 ? 0 : (size_t)W * 8;
  CK(cudaFuncSetAttribute(k_gather<MODE, U>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
  if (MODE != 2) CK(cudaFuncSetAttribute(k_gather<MODE, U>, cudaFuncAttributeNonPortableClusterSizeAllowed, 1));
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3(grid);
  cfg.blockDim = dim3(kThreads);
  cfg.dynamicSmemBytes = smem;
  cudaLaunchAttribute at[1];
  at[0].id = cudaLaunchAttributeClusterDimension;
  at[0].val.clusterDim.x = MODE == 2 ? 1 : CL;
  at[0].val.clusterDim.y = 1;
  at[0].val.clusterDim.z = 1;
  cfg.attrs = at;
  cfg.numAttrs = 1;
  cudaEvent_t a, b;
  CK(cudaEventCreate(&a));
  CK(cudaEventCreate(&b));
  for (int w = 0; w < 2; ++w) CK(cudaLaunchKernelEx(&cfg, k_gather<MODE, U>, idx, n, g, W, CL, out));
  CK(cudaEventRecord(a));
  const int reps = 5;
  for (int r = 0; r < reps; ++r) CK(cudaLaunchKernelEx(&cfg, k_gather<MODE, U>, idx, n, g, W, CL, out));
  CK(cudaEventRecord(b));
  CK(cudaEventSynchronize(b));
  float ms;
  CK(cudaEventElapsedTime(&ms, a, b));
  return ms / reps;
}

int main() {
  const long long n = 140'000'000;  // ~ the band gathers of one config-4 step
  const int W = 28 * 1024;          // doubles per CTA (224 KB)
  int dev_sms;
  CK(cudaDeviceGetAttribute(&dev_sms, cudaDevAttrMultiProcessorCount, 0));
  double* out;
  CK(cudaMalloc(&out, (size_t)148 * 4 * kThreads * 8));
  for (int CL : {2, 4, 8}) {
    const long long span = (long long)W * CL;
    std::vector<int> h(n);
    unsigned long long s = 88172645463325252ULL;
    for (long long i = 0; i < n; ++i) {
      s ^= s << 13; s ^= s >> 7; s ^= s << 17;
      h[i] = (int)(s % span);
    }
    int* idx;
    double* g;
    CK(cudaMalloc(&idx, n * 4));
    CK(cudaMemcpy(idx, h.data(), n * 4, cudaMemcpyHostToDevice));
    CK(cudaMalloc(&g, span * 8));
    std::vector<double> hg(span, 1.0);
    CK(cudaMemcpy(g, hg.data(), span * 8, cudaMemcpyHostToDevice));
    // grid: as many whole clusters as fit (one CTA per SM)
    cudaLaunchConfig_t q = {};
    q.blockDim = dim3(kThreads);
    q.dynamicSmemBytes = (size_t)W * 8;
    cudaLaunchAttribute at[1];
    at[0].id = cudaLaunchAttributeClusterDimension;
    at[0].val.clusterDim.x = CL;
    at[0].val.clusterDim.y = 1;
    at[0].val.clusterDim.z = 1;
    q.attrs = at;
    q.numAttrs = 1;
    CK(cudaFuncSetAttribute(k_gather<0, 4>, cudaFuncAttributeMaxDynamicSharedMemorySize, W * 8));
    CK(cudaFuncSetAttribute(k_gather<0, 4>, cudaFuncAttributeNonPortableClusterSizeAllowed, 1));
    int nclusters = 0;
    q.gridDim = dim3(CL * 64);
    CK(cudaOccupancyMaxActiveClusters(&nclusters, k_gather<0, 4>, &q));
    const int grid = nclusters * CL;
    const float t0 = run<0, 4>(idx, n, g, W, CL, out, grid);
    const float t0b = run<0, 8>(idx, n, g, W, CL, out, grid);
    const float t1 = run<1, 4>(idx, n, g, W, CL, out, grid);
    const float t2 = run<2, 4>(idx, n, g, W, CL, out, dev_sms * 2);
    printf("cluster %d (%d clusters, %d CTAs), window %lld doubles: DSMEM %.3f ms (U=8 %.3f), local smem %.3f ms, "
           "global(L2/L1) %.3f ms  [%.0f / %.0f / %.0f G gathers/s]\n",
           CL, nclusters, grid, span, t0, t0b, t1, t2, n / t0 / 1e6, n / t1 / 1e6, n / t2 / 1e6);
    CK(cudaFree(idx));
    CK(cudaFree(g));
  }
  return 0;
}
