// panel_lab.cu -- lab kernel (not product): y = A x with the band of each row
// block staged in shared memory by TMA, measured against the product SpMV.
//
// Layout (built by tools/panel_lab.py on the GPU): rows in blocks of R = 4096
// rows, one 1024-thread CTA per block at a time (persistent grid); thread t
// owns rows t, t+1024, t+2048, t+3072 (tag q = 0..3) and keeps their sums in
// four registers.  Each block's entries are split into a remote list (column
// outside the block's band window: gathered from global memory) and panels of
// W columns of the window (gathered from shared memory).  Inside a (block,
// panel) every thread's entries (its four rows, row-major, column order) sit
// at slot k*32 + lane of its warp's region (width = the warp's longest list,
// padding slots carry tag 0xFFFFFFFF), so every load of the stream is one
// coalesced 256 B (values) / 128 B (col|tag) warp access and a gather from a
// staged panel is a shared-memory load: no L1 miss request per band entry.
// The panel of x arrives with one cp.async.bulk per panel (TMA, no L1 miss
// requests either), double-buffered behind mbarriers.
#include <cuda_runtime.h>

#include <cstdint>

namespace {

constexpr int kThreads = 1024;
constexpr int kWarps = 32;
constexpr int kTagShift = 27;           // col (27 bits) | q << 27
constexpr unsigned kPad = 0xFFFFFFFFu;

struct PL {
  int nblk, R, W;
  const int* __restrict__ blk_pan;      // nblk+1: panel list of block b (first = remote list)
  const int* __restrict__ pan_base;     // first column of the panel (-1: remote list)
  const int* __restrict__ pan_len;      // columns in the panel
  const long long* __restrict__ wslot;  // per (panel, warp): first slot
  const int* __restrict__ wwidth;       // per (panel, warp): slots per lane
  const double* __restrict__ val;
  const unsigned* __restrict__ cq;
};

__device__ __forceinline__ uint32_t saddr(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }

__device__ __forceinline__ void mbar_init(uint64_t* bar, uint32_t count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(saddr(bar)), "r"(count) : "memory");
}
__device__ __forceinline__ void mbar_expect_tx(uint64_t* bar, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(saddr(bar)), "r"(bytes) : "memory");
}
__device__ __forceinline__ void bulk_g2s(void* dst, const void* src, uint32_t bytes, uint64_t* bar) {
  asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
                   saddr(dst)), "l"(src), "r"(bytes), "r"(saddr(bar)) : "memory");
}
__device__ __forceinline__ void mbar_wait(uint64_t* bar, uint32_t parity) {
  uint32_t done = 0;
  while (!done) {
    asm volatile("{\n .reg .pred p;\n mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\n selp.u32 %0, 1, 0, p;\n}\n"
                 : "=r"(done) : "r"(saddr(bar)), "r"(parity) : "memory");
  }
}

template <int RPT>
__device__ __forceinline__ void add_tagged(double (&acc)[RPT], unsigned q, double p) {
#pragma unroll
  for (int i = 0; i < RPT; ++i) acc[i] += q == (unsigned)i ? p : 0.0;
}

template <int U, bool SMEM, int RPT>
__device__ __forceinline__ void run_list(const PL& L, int pi, int warp, int lane, const double* __restrict__ xs,
                                         const double* __restrict__ xg, double (&acc)[RPT]) {
  const long long base = L.wslot[(size_t)pi * kWarps + warp] + lane;
  const int width = L.wwidth[(size_t)pi * kWarps + warp];
  for (int k = 0; k < width; k += U) {
    double v[U];
    unsigned c[U];
#pragma unroll
    for (int u = 0; u < U; ++u) {
      const bool on = k + u < width;
      v[u] = on ? __ldcs(L.val + base + 32LL * (k + u)) : 0.0;
      c[u] = on ? __ldcs(L.cq + base + 32LL * (k + u)) : kPad;
    }
    double xv[U];
#pragma unroll
    for (int u = 0; u < U; ++u) {
      if (SMEM) xv[u] = c[u] != kPad ? xs[c[u] & 0x7FFFFFFu] : 0.0;
      else xv[u] = c[u] != kPad ? __ldg(xg + (c[u] & 0x7FFFFFFu)) : 0.0;
    }
#pragma unroll
    for (int u = 0; u < U; ++u)
      if (c[u] != kPad) add_tagged<RPT>(acc, c[u] >> kTagShift, v[u] * xv[u]);
  }
}

// mode (timing experiments): bit 0 skip the TMA panel loads, bit 1 skip the
// remote lists, bit 2 skip the panel lists
// Software-pipelined staged-panel list: the next U slots' values and
// col|tag are loaded before the current U are consumed, so a warp keeps
// 2U stream loads in flight across rounds (no dependent gather chain: the
// gathers hit shared memory).
template <int U, int RPT>
__device__ __forceinline__ void run_panel_pipe(const PL& L, int pi, int warp, int lane,
                                               const double* __restrict__ xs, double (&acc)[RPT]) {
  const long long base = L.wslot[(size_t)pi * kWarps + warp] + lane;
  const int width = L.wwidth[(size_t)pi * kWarps + warp];
  double v[U];
  unsigned c[U];
#pragma unroll
  for (int u = 0; u < U; ++u) {
    const bool on = u < width;
    v[u] = on ? __ldcs(L.val + base + 32LL * u) : 0.0;
    c[u] = on ? __ldcs(L.cq + base + 32LL * u) : kPad;
  }
  for (int k = 0; k < width; k += U) {
    double vn[U];
    unsigned cn[U];
#pragma unroll
    for (int u = 0; u < U; ++u) {
      const bool on = k + U + u < width;
      vn[u] = on ? __ldcs(L.val + base + 32LL * (k + U + u)) : 0.0;
      cn[u] = on ? __ldcs(L.cq + base + 32LL * (k + U + u)) : kPad;
    }
#pragma unroll
    for (int u = 0; u < U; ++u)
      if (c[u] != kPad) add_tagged<RPT>(acc, c[u] >> kTagShift, v[u] * xs[c[u] & 0x7FFFFFFu]);
#pragma unroll
    for (int u = 0; u < U; ++u) {
      v[u] = vn[u];
      c[u] = cn[u];
    }
  }
}

template <int RPT>
__global__ void __launch_bounds__(kThreads, 1) k_panel_spmv(PL L, const double* __restrict__ x, int rows,
                                                           double* __restrict__ y, int mode) {
  extern __shared__ __align__(128) double xs[];  // 2 buffers of W doubles
  __shared__ uint64_t bar[2];
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  if (threadIdx.x == 0) {
    mbar_init(&bar[0], 1);
    mbar_init(&bar[1], 1);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  __syncthreads();
  uint32_t phase[2] = {0, 0};
  for (int b = blockIdx.x; b < L.nblk; b += gridDim.x) {
    const int p0 = L.blk_pan[b], p1 = L.blk_pan[b + 1];
    // issue the first staged panel, then run the remote list while it lands
    const bool tma = !(mode & 1);
    if (tma && threadIdx.x == 0 && p0 + 1 < p1) {
      const uint32_t bytes = (uint32_t)L.pan_len[p0 + 1] * 8u;
      mbar_expect_tx(&bar[0], bytes);
      bulk_g2s(xs, x + L.pan_base[p0 + 1], bytes, &bar[0]);
    }
    double acc[RPT];
#pragma unroll
    for (int i = 0; i < RPT; ++i) acc[i] = 0.0;
    if (!(mode & 2)) run_list<6, false, RPT>(L, p0, warp, lane, nullptr, x, acc);
    for (int pi = p0 + 1, s = 0; pi < p1; ++pi, s ^= 1) {
      if (tma && threadIdx.x == 0 && pi + 1 < p1) {   // prefetch the next panel into the other buffer
        const uint32_t bytes = (uint32_t)L.pan_len[pi + 1] * 8u;
        mbar_expect_tx(&bar[s ^ 1], bytes);
        bulk_g2s(xs + (size_t)(s ^ 1) * L.W, x + L.pan_base[pi + 1], bytes, &bar[s ^ 1]);
      }
      if (tma) {
        mbar_wait(&bar[s], phase[s]);
        phase[s] ^= 1;
      }
      if (!(mode & 4)) {
        if (mode & 8) run_panel_pipe<8, RPT>(L, pi, warp, lane, xs + (size_t)s * L.W, acc);
        else run_list<6, true, RPT>(L, pi, warp, lane, xs + (size_t)s * L.W, nullptr, acc);
      }
      __syncthreads();   // buffer s is free before it is refilled two panels later
    }
    const long long r0 = (long long)b * L.R;
#pragma unroll
    for (int q = 0; q < RPT; ++q) {
      const long long r = r0 + threadIdx.x + q * kThreads;
      if (r < rows) y[r] = acc[q];
    }
    __syncthreads();
  }
}

}  // namespace

extern "C" {

int panel_spmv(int nblk, int R, int W, const int* blk_pan, const int* pan_base, const int* pan_len,
               const long long* wslot, const int* wwidth, const double* val, const unsigned* cq,
               const double* x, int rows, double* y, int grid, void* stream, int mode) {
  PL L{nblk, R, W, blk_pan, pan_base, pan_len, wslot, wwidth, val, cq};
  const size_t smem = 2ull * W * 8;
  if (R == 4096) {
    cudaFuncSetAttribute(k_panel_spmv<4>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    k_panel_spmv<4><<<grid, kThreads, smem, (cudaStream_t)stream>>>(L, x, rows, y, mode);
  } else if (R == 8192) {
    cudaFuncSetAttribute(k_panel_spmv<8>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    k_panel_spmv<8><<<grid, kThreads, smem, (cudaStream_t)stream>>>(L, x, rows, y, mode);
  } else {
    cudaFuncSetAttribute(k_panel_spmv<2>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    k_panel_spmv<2><<<grid, kThreads, smem, (cudaStream_t)stream>>>(L, x, rows, y, mode);
  }
  return (int)cudaGetLastError();
}

}  // extern "C"
