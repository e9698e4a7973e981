// psr.cuh -- panel-staged rows (PSR): the SpMV layout of the PDHG step kernels.
//
// Why: on config 4 the gathered vector (xe: 80 MB, y: 40 MB) does not stay
// in L2 against 2.4 GB of streamed matrix per launch, so CSR-vector gathers
// become 32-byte DRAM sectors (v1 profile: 1.5-2.1x the algorithmic bytes,
// profiles/r01_v1_summary.md).  PSR cuts the matrix into row blocks of R
// rows; inside a block, entries whose column falls in a dense W-wide column
// bin ("panel") are grouped per panel, and the panel of the gathered vector
// is copied once into shared memory with a TMA bulk copy (cp.async.bulk,
// double-buffered behind mbarriers), so those gathers become LDS.  Entries
// in sparse bins form one "remote" tile gathered from global memory.
//
// Layout (all in tile order; a block's tiles are its staged panels in
// ascending column order, then its remote tile):
//   blk_tile_ptr[b]            first tile of row block b          (nblk+1)
//   blk_warp_row[b*(NW+1)+w]   first block-local row of warp w    (nblk*(NW+1))
//   tile_bin[t]                panel index (column bin), -1 = remote
//   tile_ent[t*(NW+1)+w]       first entry of warp w in tile t    (ntiles*(NW+1))
//   val[e], meta[e] = row_local<<16 | col_in_panel, col[e] (global column)
// Entries of a tile are in row-major CSR order, so each warp owns a
// contiguous range of rows and a contiguous range of entries per tile.
//
// Determinism: a warp owns its rows exclusively; per 32-entry chunk,
// products are summed per row segment left to right by the segment's last
// lane, and chunk results are added to the row accumulator in order.  The
// summation order of a row is fixed by the layout: panels ascending, then
// remote, entries in CSR order -- bitwise reproducible run to run.
#pragma once

#include <cuda_runtime.h>
#include <cstdint>

namespace psr {

constexpr int kThreads = 1024;
constexpr int kWarps = kThreads / 32;
constexpr int kMaxRows = 8192;   // acc[] in smem: 64 KB
constexpr int kPanel = 8192;     // W: 64 KB of fp64 per panel buffer

struct Layout {
  int rows, cols, R, W, nblk, ntiles;
  const int* __restrict__ blk_tile_ptr;
  const int* __restrict__ blk_warp_row;
  const int* __restrict__ tile_bin;
  const int* __restrict__ tile_ent;
  const double* __restrict__ val;
  const unsigned* __restrict__ meta;
  const int* __restrict__ col;
  const unsigned char* __restrict__ heavy;  // per-row flag, rows handled elsewhere
};

__host__ __device__ inline size_t smem_bytes(int R, int W) {
  return (size_t)2 * W * 8 + (size_t)R * 8 + (size_t)kWarps * 32 * 8;
}

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

// Accumulate one warp's entries [e0, e1) of a tile into acc[row_local].
// STAGED: x from the shared-memory panel; otherwise gathered from global.
// kUnroll chunks of 32 entries are loaded before any is consumed, so each
// warp keeps kUnroll x (8+4[+4]) B per lane of streaming loads (and, for the
// remote tile, kUnroll gathers) in flight -- one CTA of 32 warps per SM
// needs that memory-level parallelism to cover DRAM latency.
constexpr int kUnroll = 4;

__device__ __forceinline__ void seg_commit(double p, unsigned mt, bool v, double* acc, double* prodw,
                                           int lane) {
  const int r = (int)(mt >> 16);
  const int rp = __shfl_up_sync(0xffffffffu, r, 1);
  const unsigned hm = __ballot_sync(0xffffffffu, lane == 0 || rp != r);
  prodw[lane] = p;
  __syncwarp();
  const bool tail = v && (lane == 31 || ((hm >> (lane + 1)) & 1u));
  if (tail) {
    const unsigned below = (lane == 31) ? hm : (hm & ((2u << lane) - 1u));
    const int h = 31 - __clz(below);
    double s = prodw[h];
    for (int k = h + 1; k <= lane; ++k) s += prodw[k];
    acc[r] += s;
  }
  __syncwarp();
}

template <bool STAGED, int NR>
__device__ __forceinline__ void seg_accumulate(const Layout& L, int e0, int e1,
                                               const double* const* px, const double* const* gx,
                                               double* acc, double* prodw, int lane) {
  static_assert(NR == 1, "PSR step kernels take one right-hand side");
  for (int base = e0; base < e1; base += 32 * kUnroll) {
    unsigned mt[kUnroll];
    double a[kUnroll], xv[kUnroll];
    int cc[kUnroll];
#pragma unroll
    for (int u = 0; u < kUnroll; ++u) {
      const int e = base + u * 32 + lane;
      const bool v = e < e1;
      mt[u] = v ? __ldcs(L.meta + e) : 0xFFFF0000u;
      a[u] = v ? __ldcs(L.val + e) : 0.0;
      if (!STAGED) cc[u] = v ? __ldcs(L.col + e) : -1;
    }
    if (!STAGED) {
#pragma unroll
      for (int u = 0; u < kUnroll; ++u) xv[u] = cc[u] >= 0 ? __ldg(gx[0] + cc[u]) : 0.0;
    }
#pragma unroll
    for (int u = 0; u < kUnroll; ++u) {
      if (base + u * 32 >= e1) break;  // warp-uniform
      const bool v = base + u * 32 + lane < e1;
      const double x = STAGED ? (v ? px[0][mt[u] & 0xFFFFu] : 0.0) : xv[u];
      seg_commit(a[u] * x, mt[u], v, acc, prodw, lane);
    }
  }
}

// Row-block driver: computes acc[r] = (A x)[row0 + r] for all rows of block b
// (heavy rows excluded) into shared memory, panel staging double-buffered.
// Caller zeroes nothing; this routine zeroes acc, runs all tiles and ends
// with a __syncthreads() so acc is complete for the epilogue.
struct Pipe {
  uint64_t* bars;   // 2 mbarriers
  uint32_t ph[2];
};

template <int NR>
__device__ __forceinline__ void issue_panel(const Layout& L, int t, int buf, double* panels,
                                            const double* const* gx, uint64_t* bars) {
  const int bin = L.tile_bin[t];
  const long long start = (long long)bin * L.W;
  long long len = (long long)L.cols - start;
  if (len > L.W) len = L.W;
  const uint32_t bytes = (uint32_t)(((len * 8) + 15) & ~15LL);
  mbar_expect_tx(&bars[buf], bytes * NR);
#pragma unroll
  for (int q = 0; q < NR; ++q)
    bulk_g2s(panels + (size_t)(buf * NR + q) * L.W, gx[q] + start, bytes, &bars[buf]);
}

template <int NR>
__device__ __forceinline__ void block_spmv(const Layout& L, int b, const double* const* gx,
                                           double* panels, double* acc, double* prodw, Pipe& pp) {
  const int tid = threadIdx.x, lane = tid & 31, w = tid >> 5;
  const int row0 = b * L.R;
  int rows_b = L.rows - row0;
  if (rows_b > L.R) rows_b = L.R;
  const int t0 = L.blk_tile_ptr[b], t1 = L.blk_tile_ptr[b + 1];
  const int nst = t1 - t0 - 1;
  for (int r = tid; r < rows_b; r += kThreads) {
#pragma unroll
    for (int q = 0; q < NR; ++q) acc[q * kMaxRows + r] = 0.0;
  }
  if (tid == 0) {
    fence_proxy_async();
    for (int k = 0; k < nst && k < 2; ++k) issue_panel<NR>(L, t0 + k, k, panels, gx, pp.bars);
  }
  __syncthreads();
  for (int k = 0; k < nst; ++k) {
    const int buf = k & 1;
    mbar_wait(&pp.bars[buf], pp.ph[buf]);
    pp.ph[buf] ^= 1u;
    const int t = t0 + k;
    const int e0 = L.tile_ent[(size_t)t * (kWarps + 1) + w];
    const int e1 = L.tile_ent[(size_t)t * (kWarps + 1) + w + 1];
    const double* px[NR];
#pragma unroll
    for (int q = 0; q < NR; ++q) px[q] = panels + (size_t)(buf * NR + q) * L.W;
    seg_accumulate<true, NR>(L, e0, e1, px, gx, acc, prodw, lane);
    __syncthreads();
    if (tid == 0 && k + 2 < nst) {
      fence_proxy_async();
      issue_panel<NR>(L, t + 2, buf, panels, gx, pp.bars);
    }
  }
  {
    const int t = t1 - 1;  // remote tile
    const int e0 = L.tile_ent[(size_t)t * (kWarps + 1) + w];
    const int e1 = L.tile_ent[(size_t)t * (kWarps + 1) + w + 1];
    seg_accumulate<false, NR>(L, e0, e1, gx, gx, acc, prodw, lane);
  }
  __syncthreads();
}

}  // namespace psr
