// psr_build.cu -- device construction of the panel-staged-rows layout (psr.cuh).
//
// Input: one operator in CSR (row pointers, int32 columns, fp64 values) --
// A for the dual step, A' (= scipy's CSC of A, built by pdhg_transpose_csr)
// for the primal step.  Everything runs on the caller's stream; the only
// host round trips are three small scalars per phase.  The build is
// deterministic: counts use integer atomics, ordering uses a stable radix
// sort keyed by tile, so entries keep CSR (row, column) order inside a tile.
#include "../../include/pdhg_b200.h"
#include "psr.cuh"

#include <cuda_runtime.h>
#include <cub/cub.cuh>

#include <algorithm>
#include <climits>
#include <string>
#include <vector>

namespace pdhg_internal {
int set_error(int code, const std::string& msg);
}

namespace {

using pdhg_internal::set_error;

#define PSR_TRY(expr)                                                                          \
  do {                                                                                         \
    cudaError_t e_ = (expr);                                                                   \
    if (e_ != cudaSuccess)                                                                     \
      return set_error(PDHG_ERR_CUDA, std::string(#expr) + ": " + cudaGetErrorString(e_));     \
  } while (0)


struct Geo {
  int R, W, nblk, nbins;
};

// R: rows per row block, chosen so the block count is a multiple of 148 (one
// persistent CTA per SM, no tail wave) with R <= kMaxRows.
Geo geometry(int rows, int cols) {
  Geo g;
  const long long per_wave = 148LL * psr::kMaxRows;
  const long long k = std::max(1LL, (rows + per_wave - 1) / per_wave);
  long long R = (rows + 148 * k - 1) / (148 * k);
  R = std::max(2LL, (R + 1) & ~1LL);
  g.R = (int)std::min<long long>(R, psr::kMaxRows);
  g.W = psr::kPanel;
  g.nblk = (int)((rows + g.R - 1) / g.R);
  g.nbins = (int)((cols + (long long)g.W - 1) / g.W);
  return g;
}

size_t a256(size_t v) { return (v + 255) & ~(size_t)255; }

struct Tmp {
  int* counts;    // nblk*nbins
  int* tile_of;   // nblk*nbins
  int* ntile_b;   // nblk+1
  int* bptr;      // nblk+1
  long long* staged_b;  // nblk
  int* scal;      // 4
  int* k0; int* k1; int* v0; int* v1; int* rid;  // nnz each
  double* rm_val; unsigned short* rm_c16; int* rm_col;  // row-major staging before slot-major
  int* tstart;    // nblk*(nbins+1)+1
  void* cub; size_t cub_bytes;
};

size_t cub_need(long long nnz, int nblk) {
  size_t a = 0, b = 0;
  cub::DoubleBuffer<int> kk(nullptr, nullptr), vv(nullptr, nullptr);
  cub::DeviceRadixSort::SortPairs(nullptr, a, kk, vv, (int)std::max(1LL, nnz));
  cub::DeviceScan::ExclusiveSum(nullptr, b, (int*)nullptr, (int*)nullptr, nblk + 1);
  return std::max(a, b);
}

size_t tmp_size(int rows, int cols, long long nnz) {
  const Geo g = geometry(rows, cols);
  const size_t grid = (size_t)g.nblk * g.nbins;
  size_t s = 0;
  s += 2 * a256(grid * 4);
  s += 2 * a256((size_t)(g.nblk + 1) * 4);
  s += a256((size_t)g.nblk * 8);
  s += a256(16);
  s += 5 * a256((size_t)std::max(1LL, nnz) * 4);
  s += a256((size_t)std::max(1LL, nnz) * 8) + a256((size_t)std::max(1LL, nnz) * 2) +
       a256((size_t)std::max(1LL, nnz) * 4);
  s += a256(((size_t)g.nblk * (g.nbins + 1) + 2) * 4);
  s += a256(cub_need(nnz, g.nblk));
  return s;
}

Tmp carve(void* base, int rows, int cols, long long nnz) {
  const Geo g = geometry(rows, cols);
  const size_t grid = (size_t)g.nblk * g.nbins;
  char* p = (char*)base;
  auto take = [&](size_t bytes) { char* r = p; p += a256(bytes); return (void*)r; };
  Tmp t;
  t.counts = (int*)take(grid * 4);
  t.tile_of = (int*)take(grid * 4);
  t.ntile_b = (int*)take((size_t)(g.nblk + 1) * 4);
  t.bptr = (int*)take((size_t)(g.nblk + 1) * 4);
  t.staged_b = (long long*)take((size_t)g.nblk * 8);
  t.scal = (int*)take(16);
  const size_t ne = (size_t)std::max(1LL, nnz) * 4;
  t.k0 = (int*)take(ne); t.k1 = (int*)take(ne); t.v0 = (int*)take(ne); t.v1 = (int*)take(ne);
  t.rid = (int*)take(ne);
  t.rm_val = (double*)take((size_t)std::max(1LL, nnz) * 8);
  t.rm_c16 = (unsigned short*)take((size_t)std::max(1LL, nnz) * 2);
  t.rm_col = (int*)take((size_t)std::max(1LL, nnz) * 4);
  t.tstart = (int*)take(((size_t)g.nblk * (g.nbins + 1) + 2) * 4);
  t.cub_bytes = cub_need(nnz, g.nblk);
  t.cub = take(t.cub_bytes);
  return t;
}

// ---------------------------------------------------------------- kernels

// One CTA per row block; shared-memory histogram when the bins fit.
__global__ void k_count(int rows, const int* __restrict__ ptr, const int* __restrict__ col, int H,
                        int R, int W, int nbins, int* __restrict__ counts, bool smem_hist) {
  extern __shared__ int hist[];
  const int b = blockIdx.x;
  int* out = counts + (size_t)b * nbins;
  if (smem_hist) {
    for (int i = threadIdx.x; i < nbins; i += blockDim.x) hist[i] = 0;
    __syncthreads();
  }
  const int r0 = b * R;
  const int r1 = min(rows, r0 + R);
  // warp per row
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5, nw = blockDim.x >> 5;
  for (int r = r0 + wid; r < r1; r += nw) {
    const int s = ptr[r], e = ptr[r + 1];
    if (e - s > H) continue;
    for (int k = s + lane; k < e; k += 32) {
      const int bin = col[k] / W;
      atomicAdd(smem_hist ? &hist[bin] : &out[bin], 1);
    }
  }
  if (smem_hist) {
    __syncthreads();
    for (int i = threadIdx.x; i < nbins; i += blockDim.x) out[i] = hist[i];
  }
}

__global__ void k_tiles(int nblk, int nbins, const int* __restrict__ counts, int min_staged,
                        int* __restrict__ tile_of, int* __restrict__ ntile_b,
                        long long* __restrict__ staged_b) {
  const int b = blockIdx.x * blockDim.x + threadIdx.x;
  if (b >= nblk) return;
  int nst = 0;
  long long st = 0;
  const int* c = counts + (size_t)b * nbins;
  int* to = tile_of + (size_t)b * nbins;
  for (int i = 0; i < nbins; ++i) {
    if (c[i] >= min_staged) {
      to[i] = nst++;
      st += c[i];
    } else {
      to[i] = -1;
    }
  }
  ntile_b[b] = nst + 1;
  staged_b[b] = st;
}

__global__ void k_tile_bin(int nblk, int nbins, const int* __restrict__ tile_of,
                           const int* __restrict__ bptr, int* __restrict__ tile_bin) {
  const int b = blockIdx.x * blockDim.x + threadIdx.x;
  if (b >= nblk) return;
  const int* to = tile_of + (size_t)b * nbins;
  for (int i = 0; i < nbins; ++i)
    if (to[i] >= 0) tile_bin[bptr[b] + to[i]] = i;
  tile_bin[bptr[b + 1] - 1] = -1;
}

__global__ void k_keys(int rows, const int* __restrict__ ptr, const int* __restrict__ col, int H,
                       int R, int W, int nbins, const int* __restrict__ tile_of,
                       const int* __restrict__ bptr, int ntiles, int* __restrict__ key,
                       int* __restrict__ idx, int* __restrict__ rid) {
  const int lane = threadIdx.x & 31;
  const long long wg = ((long long)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  if (wg >= rows) return;
  const int r = (int)wg;
  const int s = ptr[r], e = ptr[r + 1];
  const bool heavy = e - s > H;
  const int b = r / R;
  const int* to = tile_of + (size_t)b * nbins;
  const int remote = bptr[b + 1] - 1;
  for (int k = s + lane; k < e; k += 32) {
    int t;
    if (heavy) {
      t = ntiles;
    } else {
      const int tl = to[col[k] / W];
      t = tl >= 0 ? bptr[b] + tl : remote;
    }
    key[k] = t;
    idx[k] = k;
    rid[k] = r;
  }
}

__global__ void k_scatter(long long nnz, const int* __restrict__ skey, const int* __restrict__ sidx,
                          const int* __restrict__ rid, const int* __restrict__ col,
                          const double* __restrict__ val, const int* __restrict__ tile_bin, int ntiles,
                          int R, int W, double* __restrict__ val_out, unsigned short* __restrict__ col16_out,
                          int* __restrict__ col_out, int* __restrict__ rowl) {
  const long long s = (long long)blockIdx.x * blockDim.x + threadIdx.x;
  if (s >= nnz) return;
  const int t = skey[s];
  if (t >= ntiles) return;
  const int e = sidx[s];
  const int r = rid[e];
  const int c = col[e];
  const int bin = tile_bin[t];
  val_out[s] = val[e];
  col_out[s] = c;
  col16_out[s] = (unsigned short)(bin >= 0 ? c - bin * W : 0);
  rowl[s] = r - (r / R) * R;
}

__global__ void k_tile_start(const int* __restrict__ skey, long long nnz, int ntiles,
                             int* __restrict__ tstart) {
  const int t = blockIdx.x * blockDim.x + threadIdx.x;
  if (t > ntiles) return;
  long long lo = 0, hi = nnz;
  while (lo < hi) {
    const long long mid = (lo + hi) >> 1;
    if (skey[mid] < t) lo = mid + 1; else hi = mid;
  }
  tstart[t] = (int)lo;
}

// For tile t and block-local row r in [0, ngroups*G]: p(r) = first entry of
// the tile whose row is >= r.  gstart[t][g] = p(G g); rcnt[t][r] = p(r+1) - p(r).
__global__ void k_groups(int ntiles, int ngroups, const int* __restrict__ tstart,
                         const int* __restrict__ rowl, int* __restrict__ gstart,
                         unsigned short* __restrict__ rcnt) {
  constexpr int G = psr::kGroupRows;
  const long long gid = (long long)blockIdx.x * blockDim.x + threadIdx.x;
  const long long per = (long long)ngroups * G + 1;
  if (gid >= (long long)ntiles * per) return;
  const int t = (int)(gid / per), r = (int)(gid % per);
  const int s = tstart[t], e = tstart[t + 1];
  auto lb = [&](int target) {
    int a = s, z = e;
    while (a < z) {
      const int mid = (a + z) >> 1;
      if (rowl[mid] < target) a = mid + 1; else z = mid;
    }
    return a;
  };
  const int p = lb(r);
  if (r % G == 0) gstart[(size_t)t * (ngroups + 1) + r / G] = p;
  if (r < ngroups * G) rcnt[(size_t)t * ngroups * G + r] = (unsigned short)(lb(r + 1) - p);
}

// One warp per (tile, group): move the group's entries from row-major to
// slot-major order (slot k = k-th entry of each row with > k entries, lanes
// in row order), the order group_tile consumes.
__global__ void k_slot_major(int ntiles, int ngroups, const int* __restrict__ gstart,
                             const unsigned short* __restrict__ rcnt,
                             const double* __restrict__ val_in, const unsigned short* __restrict__ c16_in,
                             const int* __restrict__ col_in, double* __restrict__ val_out,
                             unsigned short* __restrict__ c16_out, int* __restrict__ col_out) {
  constexpr int G = psr::kGroupRows;
  const long long w = ((long long)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  const int lane = threadIdx.x & 31;
  if (w >= (long long)ntiles * ngroups) return;
  const int t = (int)(w / ngroups), g = (int)(w % ngroups);
  const int base = gstart[(size_t)t * (ngroups + 1) + g];
  const int cnt = rcnt[((size_t)t * ngroups + g) * G + lane];
  // row-major start of this lane's row: exclusive prefix of counts
  int pre = cnt;
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    const int v = __shfl_up_sync(0xffffffffu, pre, o);
    if (lane >= o) pre += v;
  }
  const int src0 = base + pre - cnt;
  const int maxc = __reduce_max_sync(0xffffffffu, cnt);
  const unsigned lt = (1u << lane) - 1u;
  int slot_base = base;
  for (int k = 0; k < maxc; ++k) {
    const bool has = cnt > k;
    const unsigned mask = __ballot_sync(0xffffffffu, has);
    if (has) {
      const int dst = slot_base + __popc(mask & lt);
      const int src = src0 + k;
      val_out[dst] = val_in[src];
      c16_out[dst] = c16_in[src];
      col_out[dst] = col_in[src];
    }
    slot_base += __popc(mask);
  }
}

__global__ void k_heavy_flags(int rows, const int* __restrict__ ptr, int H, unsigned char* out) {
  const int r = blockIdx.x * blockDim.x + threadIdx.x;
  if (r < rows) out[r] = (ptr[r + 1] - ptr[r]) > H ? 1 : 0;
}

unsigned blocks(long long n, int t) { return (unsigned)((n + t - 1) / t); }

}  // namespace

extern "C" {

size_t pdhg_psr_tmp_bytes(int32_t rows, int32_t cols, int64_t nnz) {
  if (rows <= 0 || cols <= 0 || nnz < 0) return 0;
  return tmp_size(rows, cols, nnz);
}

int pdhg_psr_plan(int32_t rows, int32_t cols, int64_t nnz, const int32_t* ptr, const int32_t* col,
                  int32_t heavy_threshold, int32_t min_staged, void* tmp, size_t tmp_bytes,
                  void* stream, int32_t* R_out, int32_t* W_out, int32_t* nblk_out,
                  int32_t* ngroups_out, int32_t* ntiles_out, int64_t* staged_out, int64_t* nent_out) {
  if (rows <= 0 || cols <= 0 || nnz < 0 || nnz >= INT_MAX || !ptr || !tmp)
    return set_error(PDHG_ERR_ARG, "psr_plan: bad argument");
  if (tmp_bytes < tmp_size(rows, cols, nnz)) return set_error(PDHG_ERR_ARG, "psr_plan: tmp too small");
  cudaStream_t s = (cudaStream_t)stream;
  const Geo g = geometry(rows, cols);
  Tmp t = carve(tmp, rows, cols, nnz);
  const size_t grid = (size_t)g.nblk * g.nbins;
  PSR_TRY(cudaMemsetAsync(t.counts, 0, grid * 4, s));
  const bool sh = (size_t)g.nbins * 4 <= 96 * 1024;
  if (sh) PSR_TRY(cudaFuncSetAttribute(k_count, cudaFuncAttributeMaxDynamicSharedMemorySize, 96 * 1024));
  k_count<<<g.nblk, 512, sh ? (size_t)g.nbins * 4 : 0, s>>>(rows, ptr, col, heavy_threshold, g.R, g.W,
                                                          g.nbins, t.counts, sh);
  k_tiles<<<blocks(g.nblk, 128), 128, 0, s>>>(g.nblk, g.nbins, t.counts, min_staged, t.tile_of,
                                              t.ntile_b, t.staged_b);
  PSR_TRY(cudaMemsetAsync(t.ntile_b + g.nblk, 0, 4, s));
  PSR_TRY(cub::DeviceScan::ExclusiveSum(t.cub, t.cub_bytes, t.ntile_b, t.bptr, g.nblk + 1, s));
  PSR_TRY(cudaGetLastError());
  int ntiles = 0;
  PSR_TRY(cudaMemcpyAsync(&ntiles, t.bptr + g.nblk, 4, cudaMemcpyDeviceToHost, s));
  std::vector<long long> st(g.nblk);
  PSR_TRY(cudaMemcpyAsync(st.data(), t.staged_b, (size_t)g.nblk * 8, cudaMemcpyDeviceToHost, s));
  std::vector<int> hptr(2);
  PSR_TRY(cudaStreamSynchronize(s));
  long long staged = 0;
  for (long long v : st) staged += v;
  // entries of non-heavy rows
  std::vector<int> rp(rows + 1);
  PSR_TRY(cudaMemcpy(rp.data(), ptr, (size_t)(rows + 1) * 4, cudaMemcpyDeviceToHost));
  long long nent = 0;
  for (int r = 0; r < rows; ++r) {
    const int len = rp[r + 1] - rp[r];
    if (len <= heavy_threshold) nent += len;
  }
  if (R_out) *R_out = g.R;
  if (W_out) *W_out = g.W;
  if (nblk_out) *nblk_out = g.nblk;
  if (ngroups_out) *ngroups_out = (g.R + psr::kGroupRows - 1) / psr::kGroupRows;
  if (ntiles_out) *ntiles_out = ntiles;
  if (staged_out) *staged_out = staged;
  if (nent_out) *nent_out = nent;
  return 0;
}

int pdhg_psr_build(int32_t rows, int32_t cols, int64_t nnz, const int32_t* ptr, const int32_t* col,
                   const double* val, int32_t heavy_threshold, void* tmp, size_t tmp_bytes,
                   void* stream, int32_t* blk_tile_ptr, int32_t* tile_bin, int32_t* gstart,
                   uint16_t* rcnt, double* val_out, uint16_t* col16_out, int32_t* col_out,
                   uint8_t* heavy_out) {
  if (rows <= 0 || cols <= 0 || nnz < 0 || nnz >= INT_MAX || !tmp)
    return set_error(PDHG_ERR_ARG, "psr_build: bad argument");
  if (tmp_bytes < tmp_size(rows, cols, nnz)) return set_error(PDHG_ERR_ARG, "psr_build: tmp too small");
  cudaStream_t s = (cudaStream_t)stream;
  const Geo g = geometry(rows, cols);
  if ((long long)g.R > psr::kMaxRows || g.W > 65536) return set_error(PDHG_ERR_ARG, "psr: geometry overflow");
  const int ngroups = (g.R + psr::kGroupRows - 1) / psr::kGroupRows;
  Tmp t = carve(tmp, rows, cols, nnz);
  int ntiles = 0;
  PSR_TRY(cudaMemcpyAsync(&ntiles, t.bptr + g.nblk, 4, cudaMemcpyDeviceToHost, s));
  PSR_TRY(cudaStreamSynchronize(s));
  PSR_TRY(cudaMemcpyAsync(blk_tile_ptr, t.bptr, (size_t)(g.nblk + 1) * 4, cudaMemcpyDeviceToDevice, s));
  k_tile_bin<<<blocks(g.nblk, 128), 128, 0, s>>>(g.nblk, g.nbins, t.tile_of, t.bptr, tile_bin);
  int* rowl = t.k1;
  if (nnz > 0) {
    k_keys<<<blocks((long long)rows * 32, 256), 256, 0, s>>>(rows, ptr, col, heavy_threshold, g.R, g.W,
                                                              g.nbins, t.tile_of, t.bptr, ntiles, t.k0,
                                                              t.v0, t.rid);
    int bits = 1;
    while (bits < 31 && (1LL << bits) <= ntiles) ++bits;
    cub::DoubleBuffer<int> kb(t.k0, t.k1), vb(t.v0, t.v1);
    size_t cb = t.cub_bytes;
    PSR_TRY(cub::DeviceRadixSort::SortPairs(t.cub, cb, kb, vb, (int)nnz, 0, bits, s));
    k_tile_start<<<blocks(ntiles + 1, 256), 256, 0, s>>>(kb.Current(), nnz, ntiles, t.tstart);
    rowl = kb.Alternate();  // free after the sort: reused for block-local row ids
    k_scatter<<<blocks(nnz, 256), 256, 0, s>>>(nnz, kb.Current(), vb.Current(), t.rid, col, val,
                                               tile_bin, ntiles, g.R, g.W, t.rm_val, t.rm_c16, t.rm_col,
                                               rowl);
  } else {
    PSR_TRY(cudaMemsetAsync(t.tstart, 0, (size_t)(ntiles + 1) * 4, s));
  }
  const long long ng = (long long)ntiles * ((long long)ngroups * psr::kGroupRows + 1);
  k_groups<<<blocks(ng, 256), 256, 0, s>>>(ntiles, ngroups, t.tstart, rowl, gstart, rcnt);
  if (nnz > 0)
    k_slot_major<<<blocks((long long)ntiles * ngroups * 32, 256), 256, 0, s>>>(
        ntiles, ngroups, gstart, rcnt, t.rm_val, t.rm_c16, t.rm_col, val_out, col16_out, col_out);
  k_heavy_flags<<<blocks(rows, 256), 256, 0, s>>>(rows, ptr, heavy_threshold, heavy_out);
  PSR_TRY(cudaGetLastError());
  PSR_TRY(cudaStreamSynchronize(s));
  return 0;
}

}  // extern "C"
