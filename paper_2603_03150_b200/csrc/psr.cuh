// psr.cuh -- panel-staged rows (PSR): the SpMV layout of the PDHG step kernels.
//
// Why: on config 4 the gathered vector (xe: 80 MB, y: 40 MB) does not stay
// in L2 against 2.4 GB of streamed matrix per launch, so CSR-vector gathers
// become 32-byte DRAM sectors (v1 profile: 1.5-2.1x the algorithmic bytes,
// profiles/r01_v1_summary.md); the SpMV is bound by random gathers, not by
// streaming (tools/spmv_lab.cu).  PSR cuts the matrix into row blocks of R
// rows; inside a block, entries whose column falls in a dense W-wide column
// bin ("panel") are grouped per panel, and that panel of the gathered vector
// is copied once into shared memory with a TMA bulk copy (cp.async.bulk into
// a 3-stage ring behind mbarriers), so those gathers become shared-memory
// loads with a 16-bit in-panel column index.  Entries in sparse bins form
// one "remote" tile per block, gathered from global memory.
//
// Execution: one persistent 1024-thread CTA per SM walks row blocks.  Rows
// are dealt to warps in groups of 32 (warp w owns groups w, w+32, ...), one
// row per lane, and each lane keeps its rows' partial sums in registers
// across all tiles of the block -- no shared-memory accumulators, no
// atomics, no cross-lane reductions.  A row's sum runs panels ascending,
// then the remote tile, entries in column order: fixed by the layout, so
// results are bitwise reproducible run to run.
//
// Layout (entries in tile order, inside a tile in CSR (row, column) order):
//   blk_tile_ptr[b]                 first tile of row block b       (nblk+1)
//   tile_bin[t]                     panel index of tile t, -1 = remote
//   gstart[t*(ngroups+1)+g]         first entry of row group g (32 rows) in tile t
//   rcnt[(t*ngroups+g)*32+l]        entries of row 32g+l in tile t (u16)
//   entries of a (tile, group) are stored slot-major (see group_tile)
//   val[e] (f64), col16[e] (column inside the panel, u16), col[e] (global column, i32)
#pragma once

#include <cuda_runtime.h>
#include <cstdint>

namespace psr {

constexpr int kThreads = 1024;
constexpr int kWarps = kThreads / 32;
constexpr int kMaxRows = 8192;                      // rows per block
constexpr int kLanes = 1;                           // lanes per row
constexpr int kGroupRows = 32 / kLanes;             // rows per group (one warp pass)
constexpr int kGroupsPerWarp = kMaxRows / kGroupRows / kWarps;
constexpr int kPanel = 8192;                        // W: 64 KB of fp64 per panel buffer
constexpr int kStages = 3;                          // panel ring depth

struct Layout {
  int rows, cols, R, W, nblk, ntiles, ngroups;
  const int* __restrict__ blk_tile_ptr;
  const int* __restrict__ tile_bin;
  const int* __restrict__ gstart;
  const unsigned short* __restrict__ rcnt;
  const double* __restrict__ val;
  const unsigned short* __restrict__ col16;
  const int* __restrict__ col;
  const unsigned char* __restrict__ heavy;  // per-row flag: rows handled by the CSR heavy path
};

__host__ __device__ inline size_t smem_bytes(int W) { return (size_t)kStages * W * 8; }

// ------------------------------------------------------------ PTX wrappers

__device__ __forceinline__ uint32_t saddr(const void* p) {
  return (uint32_t)__cvta_generic_to_shared(p);
}

__device__ __forceinline__ void mbar_init(uint64_t* bar, uint32_t count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(saddr(bar)), "r"(count) : "memory");
}

__device__ __forceinline__ void fence_mbar_init() {
  asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
}

__device__ __forceinline__ void fence_proxy_async() {
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
}

__device__ __forceinline__ void mbar_expect_tx(uint64_t* bar, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(saddr(bar)), "r"(bytes)
               : "memory");
}

__device__ __forceinline__ void bulk_g2s(void* dst, const void* src, uint32_t bytes, uint64_t* bar) {
  asm volatile(
      "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
          saddr(dst)),
      "l"(src), "r"(bytes), "r"(saddr(bar))
      : "memory");
}

__device__ __forceinline__ void mbar_wait(uint64_t* bar, uint32_t parity) {
  uint32_t done = 0;
  while (!done) {
    asm volatile(
        "{\n .reg .pred p;\n mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\n selp.u32 %0, 1, 0, p;\n}\n"
        : "=r"(done)
        : "r"(saddr(bar)), "r"(parity)
        : "memory");
  }
}

// ------------------------------------------------------------ compute

// acc += (row 32g+lane of tile t) . x, one row per lane.  A (tile, group)
// stores its entries slot-major: slot k holds the k-th entry of every row
// with more than k entries, in lane order, so the loads of a slot are
// contiguous across the active lanes (coalesced) and a lane finds its entry
// with one ballot + popc; slot k of a row is its k-th entry in column order,
// so the row sum runs in column order.  kU slots are loaded before use.
template <bool STAGED>
__device__ __forceinline__ double group_tile(const Layout& L, int t, int g, int lane,
                                             const double* __restrict__ px,
                                             const double* __restrict__ gx, double acc) {
  constexpr int kU = 4;
  const int* gs = L.gstart + (size_t)t * (L.ngroups + 1);
  int base = gs[g];
  const int end = gs[g + 1];
  if (base == end) return acc;  // warp-uniform: no entries of this group in the tile
  const int cnt = L.rcnt[((size_t)t * L.ngroups + g) * kGroupRows + lane];
  const int maxc = __reduce_max_sync(0xffffffffu, cnt);
  const unsigned lt = (1u << lane) - 1u;
  for (int k = 0; k < maxc; k += kU) {
    int idx[kU];
#pragma unroll
    for (int u = 0; u < kU; ++u) {
      const bool has = cnt > k + u;
      const unsigned mask = __ballot_sync(0xffffffffu, has);
      idx[u] = has ? base + __popc(mask & lt) : -1;
      base += __popc(mask);
    }
    double a[kU], xv[kU];
    int c[kU];
#pragma unroll
    for (int u = 0; u < kU; ++u) {
      a[u] = idx[u] >= 0 ? __ldcs(L.val + idx[u]) : 0.0;
      c[u] = idx[u] >= 0 ? (STAGED ? (int)__ldcs(L.col16 + idx[u]) : __ldcs(L.col + idx[u])) : 0;
    }
#pragma unroll
    for (int u = 0; u < kU; ++u) xv[u] = idx[u] >= 0 ? (STAGED ? px[c[u]] : __ldg(gx + c[u])) : 0.0;
#pragma unroll
    for (int u = 0; u < kU; ++u)
      if (idx[u] >= 0) acc = fma(a[u], xv[u], acc);
  }
  return acc;
}

__device__ __forceinline__ void issue_panel(const Layout& L, int t, int buf, double* panels,
                                            const double* gx, uint64_t* bars) {
  const int bin = L.tile_bin[t];
  const long long start = (long long)bin * L.W;
  long long len = (long long)L.cols - start;
  if (len > L.W) len = L.W;
  const uint32_t bytes = (uint32_t)(((len * 8) + 15) & ~15LL);
  mbar_expect_tx(&bars[buf], bytes);
  bulk_g2s(panels + (size_t)buf * L.W, gx + start, bytes, &bars[buf]);
}

// Row block b: dot products of all (non-heavy) rows with gx, then epi(row, dot).
// `bars` are kStages mbarriers, `ph` their phase bits (uniform across the CTA).
template <class Epi>
__device__ __forceinline__ void block_rows(const Layout& L, int b, const double* __restrict__ gx,
                                           double* panels, uint64_t* bars, uint32_t* ph, Epi&& epi) {
  const int tid = threadIdx.x, lane = tid & 31, w = tid >> 5;
  const int row0 = b * L.R;
  int rows_b = L.rows - row0;
  if (rows_b > L.R) rows_b = L.R;
  const int t0 = L.blk_tile_ptr[b], t1 = L.blk_tile_ptr[b + 1];
  const int nst = t1 - t0 - 1;
  double acc[kGroupsPerWarp];
#pragma unroll
  for (int gi = 0; gi < kGroupsPerWarp; ++gi) acc[gi] = 0.0;
  if (tid == 0) {
    fence_proxy_async();
    for (int k = 0; k < nst && k < kStages; ++k) issue_panel(L, t0 + k, k, panels, gx, bars);
  }
  for (int k = 0; k < nst; ++k) {
    const int buf = k % kStages;
    mbar_wait(&bars[buf], ph[buf]);
    ph[buf] ^= 1u;
    const double* px = panels + (size_t)buf * L.W;
#pragma unroll
    for (int gi = 0; gi < kGroupsPerWarp; ++gi) {
      const int g = w + gi * kWarps;
      if (g < L.ngroups) acc[gi] = group_tile<true>(L, t0 + k, g, lane, px, gx, acc[gi]);
    }
    __syncthreads();  // every warp is done with panel `buf`
    if (tid == 0 && k + kStages < nst) {
      fence_proxy_async();
      issue_panel(L, t0 + k + kStages, buf, panels, gx, bars);
    }
  }
#pragma unroll
  for (int gi = 0; gi < kGroupsPerWarp; ++gi) {
    const int g = w + gi * kWarps;
    if (g < L.ngroups) acc[gi] = group_tile<false>(L, t1 - 1, g, lane, nullptr, gx, acc[gi]);
  }
#pragma unroll
  for (int gi = 0; gi < kGroupsPerWarp; ++gi) {
    const int g = w + gi * kWarps;
    if (g < L.ngroups) {  // warp-uniform
      double d = acc[gi];
#pragma unroll
      for (int o = 1; o < kLanes; o <<= 1) d += __shfl_xor_sync(0xffffffffu, d, o);
      const int r = g * kGroupRows + lane / kLanes;
      if (lane % kLanes == 0 && r < rows_b) {
        const int row = row0 + r;
        if (!L.heavy[row]) epi(row, d);
      }
    }
  }
}

}  // namespace psr
