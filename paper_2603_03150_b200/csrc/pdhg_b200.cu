// pdhg_b200.cu -- sm_100a kernels and the C ABI of the B200 PDHG engine.
//
// Hot path replaced: hybridlp.pdhg.run_pdhg and what it calls
// (/root/reference/pkg/src/hybridlp/pdhg.py:80-258, lp_core.py:106-142,430-485).
// The arithmetic runs on fp64 CSR layouts of A and A' (dual layout); every
// elementwise epilogue uses explicitly rounded operations (__dmul_rn etc.,
// no FMA contraction) in the reference's operation order so that, given
// the same SpMV results, iterates are bit-identical to numpy's.  SpMV and
// reduction sums use fixed-order warp/block trees (no float atomics), so
// results are bitwise reproducible run to run.
//
// Kernels
//   k_primal_step   pdhg.py:142,146-147 (+194): A'y SpMV over rows of A' fused
//                   with x+ = max(0, x - tau/omega (c - A'y)), xe = 2x+ - x,
//                   avg_x += (x+ - avg_x)/w, non-finite flag.
//   k_dual_step     pdhg.py:143,148 (+194): A xe SpMV over rows of A fused with
//                   y+ = y + sigma*omega (b - A xe), avg_y += (y+ - avg_y)/w.
//   k_check_primal  lp_core.py:436,441-443,458,476 for 1-2 points: A x with
//                   r_p = b - Ax, sum r_p^2, max|r_p|, b'y (fixed-order partials).
//   k_check_dual    pdhg.py:114 + lp_core.py:437,459,477: A'y with
//                   z = max(0, c - A'y), r_d = c - A'y - z, sum r_d^2, max|r_d|,
//                   c'x, x'z.
//   k_reduce        fixed-order combine of the per-block partials.
//   k_spmv / k_div  power iteration (pdhg.py:80-109) and the 1e-12 SpMV gate.
#include "../../include/pdhg_b200.h"
#if PDHG_EXPERIMENTAL
#include "psr.cuh"
#endif

#include <cuda_runtime.h>
#include <nvtx3/nvToolsExt.h>
#include <cooperative_groups.h>
#include <cub/cub.cuh>

#include <algorithm>
#include <climits>
#include <cmath>
#include <cstdio>
#include <cstring>
#include <map>
#include <string>
#include <vector>

namespace cg = cooperative_groups;

namespace {

thread_local std::string g_err;

int fail(int code, const std::string& msg) {
  g_err = msg;
  return code;
}

}  // namespace

namespace pdhg_internal {
int set_error(int code, const std::string& msg) {
  g_err = msg;
  return code;
}
}  // namespace pdhg_internal

namespace {

#define CUDA_TRY(expr)                                                                \
  do {                                                                                \
    cudaError_t e_ = (expr);                                                          \
    if (e_ != cudaSuccess)                                                            \
      return fail(PDHG_ERR_CUDA, std::string(#expr) + ": " + cudaGetErrorString(e_)); \
  } while (0)

constexpr int kBlock = 256;
constexpr int kWarps = kBlock / 32;
// Layouts and period modes that were built, parity-tested and measured
// SLOWER than the default path (profiles/r01_pipeline.md, r01_psr_notes.md):
// panel-staged rows (PSR, csrc/psr.cuh + psr_build.cu), the cooperative and
// single-block period kernels, L2 persisting windows.  Compiled only into the
// experiment build (python -m paper_2603_03150_b200.build --experimental);
// the product library holds the reachable kernels only.
#ifndef PDHG_EXPERIMENTAL
#define PDHG_EXPERIMENTAL 0
#endif

// Bounds-checked build (python -m paper_2603_03150_b200.build --checked;
// compute-sanitizer is not available on the GPU pool): every gathered-vector
// index, matrix-stream index and sliced-ELL slot is checked against its bound
// before the load; a violation is counted (pdhg_debug_oob), the first one kept,
// and the load is redirected to index 0 so the run continues without a fault.
#ifndef PDHG_BOUNDS_CHECK
#define PDHG_BOUNDS_CHECK 0
#endif
#if PDHG_BOUNDS_CHECK
__device__ unsigned long long g_oob_count;
__device__ long long g_oob_first[2];
__device__ __noinline__ void oob_hit(long long i, long long n) {
  if (atomicAdd(&g_oob_count, 1ULL) == 0ULL) {
    g_oob_first[0] = i;
    g_oob_first[1] = n;
  }
}
#define CHK(i, n) (((unsigned long long)(long long)(i) < (unsigned long long)(long long)(n)) ? (i) : (oob_hit((i), (n)), 0))
#else
#define CHK(i, n) (i)
#endif

#ifndef PDHG_CHECK_BPS
#define PDHG_CHECK_BPS 4
#endif
constexpr int kCheckBlocks = 148 * PDHG_CHECK_BPS;  // fixed grid => fixed reduction order
constexpr int kMaxQ = 2 * PDHG_NQ;

// ---------------------------------------------------------------- device utils

__device__ __forceinline__ double np_max0(double d) {
  // np.maximum(0.0, d): returns d unless 0.0 > d (NaN propagates, -0.0 kept)
  return (0.0 > d) ? 0.0 : d;
}

__device__ __forceinline__ double nan_max(double a, double b) {
  // np.max semantics: any NaN wins
  return (a != a || a > b) ? a : b;
}

__device__ __forceinline__ bool finite(double v) { return isfinite(v); }

// Matrix-stream and gather loads of the step/SpMV kernels.  PDHG_L2_HINT
// (compile time, default 0) selects cache policies for an experiment
// (tools/kernel_matrix.py --lib; all measured slower, profiles/r01_pipeline.md):
// 1 = stream L2 evict_first + gathers L2 evict_last, 2 = stream evict_first
// only, 3 = gathers evict_last only, 4 = gathers L1::no_allocate, 5 = 3 + 4.
#ifndef PDHG_L2_HINT
#define PDHG_L2_HINT 0
#endif
// Two-point KKT checks gather both points' vectors from one interleaved copy
// (k_pair, row_dot_pair); 0 = two separate gathers per entry.
#ifndef PDHG_CHECK_PAIR
#define PDHG_CHECK_PAIR 1
#endif
// Two-point checks over an operator with a sliced-ELL layout use it too
// (k_check_dual_sell); 0 = the CSR-vector check kernel.
#ifndef PDHG_CHECK_SELL
#define PDHG_CHECK_SELL 1
#endif
#ifndef PDHG_CHECK_EARLY
#define PDHG_CHECK_EARLY 1
#endif
// Programmatic dependent launch between the step kernels of a period: each
// step kernel is launched with programmatic stream serialisation and waits
// (griddepcontrol.wait) for its predecessor's completion and memory before
// touching any data, so kernel k+1's launch is processed while kernel k
// drains.  2 (default): the successor may launch once every block of the
// predecessor has exited -- config 1 iteration 19.7 -> 19.2 us, config 3
// and 4 unchanged (tools/period_ab.py).  1: each block also triggers its
// successor on entry -- the early blocks then sit on the SMs waiting and
// config 1 slows to 24.9 us.  0: plain stream order.
#ifndef PDHG_PDL
#define PDHG_PDL 2
#endif
// Entries in flight per lane: row_dot with V >= 16 lanes per row (4 -> 5:
// config 4 dual step 0.956 -> 0.940 ms, config 2 110 -> 106 us; 6 spills)
// and the pipelined V <= 8 routine.
#ifndef PDHG_ROW_U16
#define PDHG_ROW_U16 5
#endif
#ifndef PDHG_PIPE_U
#define PDHG_PIPE_U 4
#endif
// V >= 16 step kernels load their epilogue operands after the row loop
#ifndef PDHG_LATE16
#define PDHG_LATE16 1
#endif
// Two-point A-side check in the warp-owns-32-rows shape (k_check_primal_rows)
#ifndef PDHG_CHECK_ROWS
#define PDHG_CHECK_ROWS 1
#endif
// row_dot_pair (two-point checks): entries in flight per lane for V >= 16
#ifndef PDHG_PAIR_U16
#define PDHG_PAIR_U16 4
#endif

__device__ __forceinline__ void pdl_enter() {
#if PDHG_PDL == 1
  asm volatile("griddepcontrol.launch_dependents;" ::: "memory");
#endif
#if PDHG_PDL
  asm volatile("griddepcontrol.wait;" ::: "memory");
#endif
}

// Row reductions of the warp-owns-32-rows routines: 1 = per-pass partials
// kept in registers and reduced once per warp by a reduce-scatter
// (reduce_scatter_rows), 0 = butterfly + parking shuffle per pass.  Measured
// on config 4 (profiles/r01_pipeline.md): the pipelined V <= 8 form gains 7 %
// (primal 0.931 -> 0.862 ms); the V >= 16 form loses (dual 0.974 -> 1.199 ms:
// 16 partials raise registers 40 -> 64 and cut occupancy).
#ifndef PDHG_RS_PIPE
#define PDHG_RS_PIPE 1
#endif
#ifndef PDHG_RS_SEG
#define PDHG_RS_SEG 0
#endif

__device__ __forceinline__ uint64_t l2_policy_first() {
  uint64_t p;
  asm("createpolicy.fractional.L2::evict_first.b64 %0, 1.0;" : "=l"(p));
  return p;
}
__device__ __forceinline__ uint64_t l2_policy_last() {
  uint64_t p;
  asm("createpolicy.fractional.L2::evict_last.b64 %0, 1.0;" : "=l"(p));
  return p;
}

__device__ __forceinline__ double ld_stream(const double* p) {
#if PDHG_L2_HINT == 1 || PDHG_L2_HINT == 2
  double v;
  asm("ld.global.L1::no_allocate.L2::cache_hint.f64 %0, [%1], %2;"
               : "=d"(v) : "l"(p), "l"(l2_policy_first()));
  return v;
#else
  return __ldcs(p);
#endif
}
__device__ __forceinline__ int ld_stream(const int* p) {
#if PDHG_L2_HINT == 1 || PDHG_L2_HINT == 2
  int v;
  asm("ld.global.L1::no_allocate.L2::cache_hint.s32 %0, [%1], %2;"
               : "=r"(v) : "l"(p), "l"(l2_policy_first()));
  return v;
#else
  return __ldcs(p);
#endif
}
__device__ __forceinline__ double ld_gather(const double* p) {
#if PDHG_L2_HINT == 1 || PDHG_L2_HINT == 3
  double v;
  asm("ld.global.nc.L2::cache_hint.f64 %0, [%1], %2;" : "=d"(v) : "l"(p), "l"(l2_policy_last()));
  return v;
#elif PDHG_L2_HINT == 4
  double v;
  asm("ld.global.nc.L1::no_allocate.f64 %0, [%1];" : "=d"(v) : "l"(p));
  return v;
#elif PDHG_L2_HINT == 5
  double v;
  asm("ld.global.nc.L1::no_allocate.L2::cache_hint.f64 %0, [%1], %2;" : "=d"(v) : "l"(p), "l"(l2_policy_last()));
  return v;
#else
  return __ldg(p);
#endif
}

template <int V>
__device__ __forceinline__ double group_sum(double v) {
#pragma unroll
  for (int o = V / 2; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  return v;
}

// Row totals of a warp that computed 32 rows in V passes of G = 32/V rows
// (V lanes per row): lane (q*V + s) holds, in accs[p], its partial for row
// p*G + q.  A reduce-scatter by recursive halving (V-1 64-bit shuffles
// instead of V butterflies of log2 V) leaves lane (q*V + s) with the total
// of row s*G + q; one more shuffle parks row r's total in lane r.  Each
// step adds own + partner exactly as group_sum's butterfly does, in the
// same tree, so the totals are bitwise identical to group_sum's.
template <int V>
__device__ __forceinline__ double reduce_scatter_rows(double (&accs)[V], int lane) {
  constexpr int G = 32 / V;
  const int sub = lane % V;
#pragma unroll
  for (int k = V / 2; k >= 1; k >>= 1) {
    const bool upper = (sub & k) != 0;
#pragma unroll
    for (int i = 0; i < k; ++i) {
      const double send = upper ? accs[i] : accs[i + k];
      const double keep = upper ? accs[i + k] : accs[i];
      accs[i] = keep + __shfl_xor_sync(0xffffffffu, send, k);
    }
  }
  return __shfl_sync(0xffffffffu, accs[0], (lane % G) * V + lane / G);
}

// Block-wide sum; result valid in every thread.  Fixed tree order.
__device__ __forceinline__ double block_sum(double v, double* red) {
  v = group_sum<32>(v);
  const int w = threadIdx.x >> 5, l = threadIdx.x & 31;
  __syncthreads();
  if (l == 0) red[w] = v;
  __syncthreads();
  double t = (l < kWarps) ? red[l] : 0.0;
  t = group_sum<32>(t);
  return t;
}

__device__ __forceinline__ double block_max(double v, double* red) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v = nan_max(v, __shfl_xor_sync(0xffffffffu, v, o));
  const int w = threadIdx.x >> 5, l = threadIdx.x & 31;
  __syncthreads();
  if (l == 0) red[w] = v;
  __syncthreads();
  double t = (l < kWarps) ? red[l] : -1.0;
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) t = nan_max(t, __shfl_xor_sync(0xffffffffu, t, o));
  return t;
}

struct RowSet {
  const int* __restrict__ ptr;
  const int* __restrict__ col;
  const double* __restrict__ val;
  int rows;
  int heavy_threshold;
  int n_heavy;
  const int* __restrict__ heavy;
  // k_step only: rows with light_max < len <= heavy_threshold run one warp
  // per row (medium list, kWarps rows per block) instead of V lanes in the
  // warp-owns-32-rows path, whose warps a long row would hold for many
  // dependent load rounds.  Other kernels treat them as light rows.
  int light_max = 0x7fffffff;
  int n_medium = 0;
  const int* __restrict__ medium = nullptr;
  int ncols = 0x7fffffff;                // gathered-vector length (bounds-checked build)
  long long nnz = 0x7fffffffffffffffLL;  // entries (bounds-checked build)
};

// Partial dot of one row over lanes [lane, lane+V, ...]; NR right-hand sides
// share one pass over the row's values and indices.
// COH: gathered vector loads through L2 only (ld.global.cg) -- required in the
// persistent period kernel, where the vector is rewritten between phases and
// the non-coherent read-only path (ld.global.nc) could serve stale lines.
// (COH 2: ld.global.ca -- L1-cached and coherent within one block, for the
// single-block period kernel, where __syncthreads orders the phases.)
template <int COH>
__device__ __forceinline__ double gather_ld(const double* p) {
  if constexpr (COH == 1) return __ldcg(p);
  else if constexpr (COH == 2) return __ldca(p);
  else return ld_gather(p);
}

template <int V, int NR, int COH = 0>
__device__ __forceinline__ void row_dot(const RowSet& A, int s, int e, int lane,
                                        const double* const* __restrict__ xin, double* acc) {
  // kU entries per lane are loaded before any is consumed (memory-level
  // parallelism for the dependent gathers); the fma chain still runs in
  // entry order k, k+V, k+2V, ...  (V, kU) from tools/spmv_lab.cu on config 4
  // (profiles/r01_spmv_lab2.log): (16, 4) for mean-40 rows, (8, 2) for mean 20.
  constexpr int kU = V >= 16 ? PDHG_ROW_U16 : 2;
#pragma unroll
  for (int r = 0; r < NR; ++r) acc[r] = 0.0;
  for (int k = s + lane; k < e; k += kU * V) {
    double a[kU];
    int j[kU];
#pragma unroll
    for (int u = 0; u < kU; ++u) {
      const int kk = k + u * V;
      a[u] = kk < e ? ld_stream(A.val + CHK(kk, A.nnz)) : 0.0;
      j[u] = kk < e ? ld_stream(A.col + CHK(kk, A.nnz)) : -1;
    }
#pragma unroll
    for (int r = 0; r < NR; ++r) {
      double xv[kU];
#pragma unroll
      for (int u = 0; u < kU; ++u) xv[u] = j[u] >= 0 ? gather_ld<COH>(xin[r] + CHK(j[u], A.ncols)) : 0.0;
#pragma unroll
      for (int u = 0; u < kU; ++u)
        if (j[u] >= 0) acc[r] = fma(a[u], xv[u], acc[r]);
    }
  }
}

// Light rows, one warp per 32 consecutive rows: lane l fetches row
// (row0+l)'s extent (coalesced), the rows are computed in V passes of 32/V
// rows with V lanes each (row_dot's fixed lane order + butterfly), and row
// row0+l's dot is parked in lane l, so the caller's epilogue runs on all 32
// lanes with coalesced traffic (v1 ran it on one lane in V: ~110
// instructions per 32 entries in ncu).  ok = row exists and is not heavy.
// Segment form: row r's entries [sp[r], ep[r]) (a column chunk of the row
// when the SpMV is split by columns); "heavy" is judged on the full row.
template <int V, int COH = 0>
__device__ __forceinline__ double warp_rows_dot_seg(const RowSet& rs, const int* __restrict__ sp,
                                                    const int* __restrict__ ep, long long row0,
                                                    int lane, const double* const* __restrict__ xin,
                                                    bool& ok) {
  constexpr int G = 32 / V;
  const long long rl = row0 + lane;
  int my_s = 0, my_e = 0;
  ok = rl < rs.rows;
  if (ok) {
    if (rs.ptr[rl + 1] - rs.ptr[rl] > rs.heavy_threshold) {
      ok = false;
    } else {
      my_s = sp[rl];
      my_e = ep[rl];
    }
  }
#if PDHG_RS_SEG
  double accs[V];
#pragma unroll
  for (int pass = 0; pass < V; ++pass) {
    const int src = pass * G + lane / V;  // lane holding this group's row
    const int s = __shfl_sync(0xffffffffu, my_s, src);
    const int e = __shfl_sync(0xffffffffu, my_e, src);
    double acc[1];
    row_dot<V, 1, COH>(rs, s, e, lane % V, xin, acc);
    accs[pass] = acc[0];
  }
  return reduce_scatter_rows<V>(accs, lane);
#else
  double mine = 0.0;
#pragma unroll 1
  for (int pass = 0; pass < V; ++pass) {
    const int src = pass * G + lane / V;  // lane holding this group's row
    const int s = __shfl_sync(0xffffffffu, my_s, src);
    const int e = __shfl_sync(0xffffffffu, my_e, src);
    double acc[1];
    row_dot<V, 1, COH>(rs, s, e, lane % V, xin, acc);
    const double d = group_sum<V>(acc[0]);
    const double got = __shfl_sync(0xffffffffu, d, ((lane - pass * G) & (G - 1)) * V);
    if (lane / G == pass) mine = got;
  }
  return mine;
#endif
}

// Software-pipelined form for short rows (V <= 8): the next pass's first
// kU*V entries (values, indices) are loaded before the current pass's
// gathers, so index-load latency overlaps gather latency
// (tools/spmv_lab.cu v7: A' 0.888 -> 0.839 ms on config 4).  Summation
// order is row_dot's: entries k, k+V, ... of the lane, then the butterfly.
template <int V, int COH = 0>
__device__ __forceinline__ double warp_rows_dot_pipe(const RowSet& rs, long long row0, int lane,
                                                     const double* const* __restrict__ xin,
                                                     bool& ok) {
  constexpr int G = 32 / V;
  constexpr int kU = PDHG_PIPE_U;
  const int sub = lane % V;
  const long long rl = row0 + lane;
  int my_s = 0, my_e = 0;
  ok = rl < rs.rows;
  if (ok) {
    my_s = rs.ptr[rl];
    my_e = rs.ptr[rl + 1];
    if (my_e - my_s > rs.heavy_threshold) { ok = false; my_e = my_s; }
  }
  const double* __restrict__ x = xin[0];
  int s = __shfl_sync(0xffffffffu, my_s, lane / V);
  int e = __shfl_sync(0xffffffffu, my_e, lane / V);
  double ac[kU];
  int jc[kU];
#pragma unroll
  for (int u = 0; u < kU; ++u) {
    const int kk = s + sub + u * V;
    ac[u] = kk < e ? ld_stream(rs.val + CHK(kk, rs.nnz)) : 0.0;
    jc[u] = kk < e ? ld_stream(rs.col + CHK(kk, rs.nnz)) : -1;
  }
#if PDHG_RS_PIPE
  double accs[V];
#pragma unroll
#else
  double mine = 0.0;
#pragma unroll 1
#endif
  for (int pass = 0; pass < V; ++pass) {
    int sn = 0, en = 0;
    if (pass + 1 < V) {
      const int src = (pass + 1) * G + lane / V;
      sn = __shfl_sync(0xffffffffu, my_s, src);
      en = __shfl_sync(0xffffffffu, my_e, src);
    }
    double an[kU];
    int jn[kU];
#pragma unroll
    for (int u = 0; u < kU; ++u) {
      const int kk = sn + sub + u * V;
      an[u] = kk < en ? ld_stream(rs.val + CHK(kk, rs.nnz)) : 0.0;
      jn[u] = kk < en ? ld_stream(rs.col + CHK(kk, rs.nnz)) : -1;
    }
    double xv[kU];
#pragma unroll
    for (int u = 0; u < kU; ++u) xv[u] = jc[u] >= 0 ? gather_ld<COH>(x + CHK(jc[u], rs.ncols)) : 0.0;
    double acc = 0.0;
#pragma unroll
    for (int u = 0; u < kU; ++u)
      if (jc[u] >= 0) acc = fma(ac[u], xv[u], acc);
    for (int k = s + sub + kU * V; k < e; k += kU * V) {  // rows longer than kU*V
      double a2[kU], x2[kU];
      int j2[kU];
#pragma unroll
      for (int u = 0; u < kU; ++u) {
        const int kk = k + u * V;
        a2[u] = kk < e ? ld_stream(rs.val + CHK(kk, rs.nnz)) : 0.0;
        j2[u] = kk < e ? ld_stream(rs.col + CHK(kk, rs.nnz)) : -1;
      }
#pragma unroll
      for (int u = 0; u < kU; ++u) x2[u] = j2[u] >= 0 ? gather_ld<COH>(x + CHK(j2[u], rs.ncols)) : 0.0;
#pragma unroll
      for (int u = 0; u < kU; ++u)
        if (j2[u] >= 0) acc = fma(a2[u], x2[u], acc);
    }
#if PDHG_RS_PIPE
    accs[pass] = acc;
#else
    const double d = group_sum<V>(acc);
    const double got = __shfl_sync(0xffffffffu, d, ((lane - pass * G) & (G - 1)) * V);
    if (lane / G == pass) mine = got;
#endif
#pragma unroll
    for (int u = 0; u < kU; ++u) {
      ac[u] = an[u];
      jc[u] = jn[u];
    }
    s = sn;
    e = en;
  }
#if PDHG_RS_PIPE
  return reduce_scatter_rows<V>(accs, lane);
#else
  return mine;
#endif
}

template <int V, int COH = 0>
__device__ __forceinline__ double warp_rows_dot(const RowSet& rs, long long row0, int lane,
                                                const double* const* __restrict__ xin, bool& ok) {
  if (V <= 8) return warp_rows_dot_pipe<V, COH>(rs, row0, lane, xin, ok);
  return warp_rows_dot_seg<V, COH>(rs, rs.ptr, rs.ptr + 1, row0, lane, xin, ok);
}

// Device-resident per-period parameters (updated by one H2D copy per period
// so the captured CUDA graph of a period can be replayed unchanged).
// Fused all-gather (multi-GPU): the step's epilogue also
// stores each new xe (primal) / y (dual) value into every peer's full
// vector at this shard's slot -- NVLink peer stores that overlap the
// kernel, replacing the all-gather after it.  ptr: device array of n peer
// vector bases (same padded layout everywhere); off: this shard's slice.
struct Peers {
  double* const* __restrict__ ptr;
  int n;
  int off;
};



struct StepParams {
  double tau_w;    // tau / omega      (pdhg.py:142)
  double sigma_w;  // sigma * omega    (pdhg.py:143)
  double w0;       // avg_weight at period start (integer valued)
  long long iter0; // state.iterations at period start
  long long fail_iter;  // first iteration with a non-finite iterate (LLONG_MAX = none)
  Peers peers[2];  // fused all-gather targets: [0] xe (primal step), [1] y (dual step)
  // other shards' fail words (their StepParams::fail_iter): a non-finite
  // iterate stops every shard at the same iteration, as on one GPU
  unsigned long long* const* fail_peers;
  int nfail;
};

// The peer list lives in device memory (StepParams) rather than in the kernel
// parameters: read only in the epilogue, it keeps no registers live across
// the row loop (as a StepArgs member it pushed the 40-register dual step into
// a 16-byte spill, +9 %).
__device__ __noinline__ void bcast_peers(const StepParams* P, int k, int row, double v) {
  const int n = P->peers[k].n;
  for (int q = 0; q < n; ++q) P->peers[k].ptr[q][P->peers[k].off + row] = v;
}

__device__ __forceinline__ void bcast(const StepParams* P, int k, int row, double v) {
  if (P->peers[k].n) bcast_peers(P, k, row, v);  // out of line: no registers held in the hot loop
}

// first non-finite iterate: record it here and in every peer shard's fail word
__device__ __forceinline__ void fail_at(StepParams* P, long long iter) {
  atomicMin(&P->fail_iter, iter);
  for (int q = 0; q < P->nfail; ++q) atomicMin(reinterpret_cast<long long*>(P->fail_peers[q]), iter);
}

// k_step's form: the peer stores are compiled in only for the fused-all-gather
// instantiation, so the single-GPU step kernels keep their exact code.
template <bool PEERS>
__device__ __forceinline__ void bcast_if(const StepParams* P, int k, int row, double v) {
  if constexpr (PEERS) bcast(P, k, row, v);
}

// ------------------------------------------------------------------- steps

// L2 policy of the vectors the next half step gathers (xe from the primal
// step, y from the dual step): 0 = plain stores; PDHG_XE_LAST: xe stored
// with an L2 evict_last policy; PDHG_Y_EF: y stored evict-first.
#ifndef PDHG_XE_LAST
#define PDHG_XE_LAST 0
#endif
#ifndef PDHG_Y_EF
#define PDHG_Y_EF 0
#endif
__device__ __forceinline__ void st_xe(double* p, double v) {
#if PDHG_XE_LAST
  uint64_t pol;
  asm("createpolicy.fractional.L2::evict_last.b64 %0, 1.0;" : "=l"(pol));
  asm volatile("st.global.L2::cache_hint.f64 [%0], %1, %2;" ::"l"(p), "d"(v), "l"(pol) : "memory");
#else
  *p = v;
#endif
}
__device__ __forceinline__ void st_y(double* p, double v) {
#if PDHG_Y_EF
  __stcs(p, v);
#else
  *p = v;
#endif
}

// Epilogue of the primal step for row j of A' (= column j of A).
__device__ __forceinline__ double primal_epi(int j, double aty, const double* __restrict__ c,
                                           double* __restrict__ x, double* __restrict__ xe,
                                           double* __restrict__ xbar, double tau_w, double w,
                                           long long iter, StepParams* P) {
  const double xj = x[j];
  const double g = __dsub_rn(c[j], aty);                       // c - A'y
  const double xn = np_max0(__dsub_rn(xj, __dmul_rn(tau_w, g)));  // max(0, x - t g)
  const double xb = xbar[j];
  x[j] = xn;
  const double xev = __dsub_rn(__dmul_rn(2.0, xn), xj);       // 2 x+ - x
  st_xe(xe + j, xev);
  xbar[j] = __dadd_rn(xb, __ddiv_rn(__dsub_rn(xn, xb), w));    // avg += (x+ - avg)/w
  if (!finite(xn)) fail_at(P, iter);
  return xev;
}

__device__ __forceinline__ double dual_epi(int i, double ax, const double* __restrict__ b,
                                         double* __restrict__ y, double* __restrict__ ybar,
                                         double sigma_w, double w, long long iter, StepParams* P) {
  const double yi = y[i];
  const double yn = __dadd_rn(yi, __dmul_rn(sigma_w, __dsub_rn(b[i], ax)));
  const double yb = ybar[i];
  st_y(y + i, yn);
  ybar[i] = __dadd_rn(yb, __ddiv_rn(__dsub_rn(yn, yb), w));
  if (!finite(yn)) fail_at(P, iter);
  return yn;
}

// Same epilogues with the row's operands already in registers.
// Epilogue cache policy: the operands a step reads once and the outputs the
// next half step does not gather (c, x, x-bar loads and x, x-bar stores of the
// primal step; y-bar stores of the dual step) are streamed evict-first, so L2
// keeps the vector the next half step gathers (xe written by the primal step,
// y by the dual step).  Sliced-ELL steps, config 4, power-capped: 1.7556 vs
// 1.7591 ms per iteration, 3 alternating processes each (tools/lib_ab.py,
// profiles/r02_epi_hint_ab.log).  0 = plain loads and stores.
#ifndef PDHG_EPI_HINT
#define PDHG_EPI_HINT 1
#endif
__device__ __forceinline__ double epi_ld(const double* p) {
#if PDHG_EPI_HINT
  return __ldcs(p);
#else
  return *p;
#endif
}
__device__ __forceinline__ void epi_st(double* p, double v) {
#if PDHG_EPI_HINT
  __stcs(p, v);
#else
  *p = v;
#endif
}

__device__ __forceinline__ double primal_epi_pre(int j, double aty, double cj, double xj, double xb,
                                               double* __restrict__ x, double* __restrict__ xe,
                                               double* __restrict__ xbar, double tau_w, double w,
                                               long long iter, StepParams* P) {
  const double g = __dsub_rn(cj, aty);
  const double xn = np_max0(__dsub_rn(xj, __dmul_rn(tau_w, g)));
  epi_st(x + j, xn);
  const double xev = __dsub_rn(__dmul_rn(2.0, xn), xj);
  st_xe(xe + j, xev);
  epi_st(xbar + j, __dadd_rn(xb, __ddiv_rn(__dsub_rn(xn, xb), w)));
  if (!finite(xn)) fail_at(P, iter);
  return xev;
}

__device__ __forceinline__ double dual_epi_pre(int i, double ax, double bi, double yi, double yb,
                                             double* __restrict__ y, double* __restrict__ ybar,
                                             double sigma_w, double w, long long iter, StepParams* P) {
  const double yn = __dadd_rn(yi, __dmul_rn(sigma_w, __dsub_rn(bi, ax)));
  st_y(y + i, yn);
  epi_st(ybar + i, __dadd_rn(yb, __ddiv_rn(__dsub_rn(yn, yb), w)));
  if (!finite(yn)) fail_at(P, iter);
  return yn;
}

struct StepArgs {
  RowSet rs;
  const int* __restrict__ split;      // column-chunk split points, (nsplit-1) arrays of rows
  int nsplit;                         // 1 = unsplit
  double* partial;                    // per-row partial sums between split passes
  const double* __restrict__ gather;  // y (primal) or xe (dual)
  const double* __restrict__ cb;      // c (primal) or b (dual)
  double* x;      // x (primal) or y (dual)
  double* xe;     // xe (primal only)
  double* xbar;   // avg_x or avg_y
  StepParams* P;
};

// Occupancy: the V >= 16 form (config 4's dual step) is latency-bound and
// fits 32 registers -- 8 blocks (64 warps) per SM -- once the epilogue
// operands are loaded after the row loop: 0.975 -> 0.936 ms.  The pipelined
// V = 4, 8 forms keep their registers (reduce-scatter partials): 4 blocks.
// (Left to ptxas, an explicit minBlocks of 1 gave 56 / 80 registers and a
// 23 % slower dual step; profiles/r01_pipeline.md.)
// V <= 2 (short rows: config 1) fits 40 registers at 6 blocks: one config-1
// iteration 24.6 -> 20.6 us; V = 4, 8 spill below 64 registers.
template <int V>
constexpr int step_min_blocks() { return V >= 16 ? 8 : (V <= 2 ? 6 : 4); }

template <int V, bool PRIMAL, bool PEERS = false>
__global__ void __launch_bounds__(kBlock, step_min_blocks<V>()) k_step(StepArgs a, int j_in_period) {
  constexpr bool kLateEpi = V >= 16 && PDHG_LATE16;
  __shared__ double red[kWarps];
  pdl_enter();
  StepParams* P = a.P;
  const long long iter = P->iter0 + j_in_period + 1;  // state.iterations after this step
  if (P->fail_iter < iter) return;                    // pdhg.py:194-196: stop after failure
  const double w = P->w0 + (double)(j_in_period + 1);  // avg_weight + 1 (exact, integer valued)
  const double step = PRIMAL ? P->tau_w : P->sigma_w;
  const double* xin[1] = {a.gather};

  if ((int)blockIdx.x < a.rs.n_heavy) {  // one block per heavy row
    const int row = a.rs.heavy[blockIdx.x];
    const int s = a.rs.ptr[row], e = a.rs.ptr[row + 1];
    double acc[1];
    row_dot<kBlock, 1>(a.rs, s, e, threadIdx.x, xin, acc);
    const double d = block_sum(acc[0], red);
    if (threadIdx.x == 0) {
      if (PRIMAL) bcast_if<PEERS>(P, 0, row, primal_epi(row, d, a.cb, a.x, a.xe, a.xbar, step, w, iter, P));
      else bcast_if<PEERS>(P, 1, row, dual_epi(row, d, a.cb, a.x, a.xbar, step, w, iter, P));
    }
    return;
  }
  const int medium_blocks = (a.rs.n_medium + kWarps - 1) / kWarps;
  if ((int)blockIdx.x < a.rs.n_heavy + medium_blocks) {  // one warp per medium row
    const int h = ((int)blockIdx.x - a.rs.n_heavy) * kWarps + (int)(threadIdx.x >> 5);
    if (h >= a.rs.n_medium) return;  // warp-uniform
    const int row = a.rs.medium[h];
    double acc[1];
    row_dot<32, 1>(a.rs, a.rs.ptr[row], a.rs.ptr[row + 1], threadIdx.x & 31, xin, acc);
    const double d = group_sum<32>(acc[0]);
    if ((threadIdx.x & 31) == 0) {
      if (PRIMAL) bcast_if<PEERS>(P, 0, row, primal_epi(row, d, a.cb, a.x, a.xe, a.xbar, step, w, iter, P));
      else bcast_if<PEERS>(P, 1, row, dual_epi(row, d, a.cb, a.x, a.xbar, step, w, iter, P));
    }
    return;
  }
  // Light rows: a warp owns 32 consecutive rows.  It computes them in V
  // passes of 32/V rows (V lanes per row, fixed lane order), parks row k's
  // dot in lane k with one shuffle per pass, then all 32 lanes run the
  // epilogue together -- full lane utilisation and coalesced x/c/avg
  // traffic (v1 ran the epilogue on one lane in V: ncu showed ~110
  // instructions per 32 entries, profiles/r01_csr_epilogue.md).
  const int lane = threadIdx.x & 31;
  const long long warp_id =
      ((long long)(blockIdx.x - a.rs.n_heavy - medium_blocks) * kBlock + threadIdx.x) >> 5;
  const long long row0 = warp_id * 32;
  if (row0 >= a.rs.rows) return;  // warp-uniform
  const long long rl = row0 + lane;
  const bool in_range = rl < a.rs.rows;
  RowSet lrs = a.rs;  // the light path skips heavy and medium rows
  lrs.heavy_threshold = min(a.rs.heavy_threshold, a.rs.light_max);
  // epilogue operands: coalesced, loaded before the SpMV (V <= 8) or after it
  // (V >= 16, so that fewer registers are live in the row loop)
  double o1 = 0.0, o2 = 0.0, o3 = 0.0;
  if (!kLateEpi && in_range) {
    o1 = a.cb[rl];
    o2 = a.x[rl];
    o3 = a.xbar[rl];
  }
  bool my_ok;
  const double mine = warp_rows_dot<V>(lrs, row0, lane, xin, my_ok);
  if (kLateEpi && in_range) {
    o1 = a.cb[rl];
    o2 = a.x[rl];
    o3 = a.xbar[rl];
  }
  if (my_ok) {
    const int row = (int)rl;
    if (PRIMAL) bcast_if<PEERS>(P, 0, row, primal_epi_pre(row, mine, o1, o2, o3, a.x, a.xe, a.xbar, step, w, iter, P));
    else bcast_if<PEERS>(P, 1, row, dual_epi_pre(row, mine, o1, o2, o3, a.x, a.xbar, step, w, iter, P));
  }
}

// Step over a sliced-ELL layout (csrc/sell_build.cu): a warp owns one slice
// of 32 consecutive rows, lane l row 32*slice + l; each lane sums its row
// sequentially in entry order (kU entries' loads in flight), so there are no
// lane reductions and every matrix load instruction is 256 B (values) /
// 128 B (indices) contiguous.  Heavy rows: one block each, as in k_step.
struct SellSet {
  int rows, nslices;
  const long long* __restrict__ sptr;
  const int* __restrict__ width;
  const int* __restrict__ col;
  const double* __restrict__ val;
  const unsigned char* __restrict__ perm;  // lane -> row offset in the slice (nullptr = identity)
  bool u_long = false;                     // mean row >= PDHG_SELL_U_MEAN: PDHG_SELL_U_LONG in flight
  int ncols = 0x7fffffff;                  // gathered-vector length (bounds-checked build)
  long long nslots = 0x7fffffffffffffffLL; // slots (bounds-checked build)
};

// Row of lane `lane` of slice sl (natural or slice-sorted layout).
__device__ __forceinline__ long long sell_row(const SellSet& S, long long sl, int lane) {
  return sl * 32 + (S.perm ? S.perm[sl * 32 + lane] : lane);
}

// Entries in flight per lane in the SELL row loop: PDHG_SELL_U for short
// rows, PDHG_SELL_U_LONG for operators averaging >= PDHG_SELL_U_MEAN entries
// per row (config 4's A', mean 20: 4 -> 6 takes the primal step 0.816 ->
// 0.781 ms; config 3's A', mean 3, stays at 4: profiles/r01_pipeline.md).
#ifndef PDHG_SELL_U
#define PDHG_SELL_U 4
#endif
#ifndef PDHG_SELL_U_LONG
#define PDHG_SELL_U_LONG 6
#endif
#ifndef PDHG_SELL_U_MEAN
#define PDHG_SELL_U_MEAN 12
#endif

// Lane's row of slice sl: sequential sum over its len entries (kU entries'
// loads in flight per round).
template <int kU>
__device__ __forceinline__ double sell_row_dot(const SellSet& S, long long sl, int lane, int len,
                                               const double* __restrict__ x) {
  const int width = S.width[sl];
  const long long base = S.sptr[sl] + lane;
  double acc = 0.0;
  for (int k = 0; k < width; k += kU) {
    double av[kU], xv[kU];
    int jv[kU];
#pragma unroll
    for (int u = 0; u < kU; ++u) {
      const bool on = k + u < len;
      av[u] = on ? ld_stream(S.val + CHK(base + 32LL * (k + u), S.nslots)) : 0.0;
      jv[u] = on ? ld_stream(S.col + CHK(base + 32LL * (k + u), S.nslots)) : -1;
    }
#pragma unroll
    for (int u = 0; u < kU; ++u) xv[u] = jv[u] >= 0 ? ld_gather(x + CHK(jv[u], S.ncols)) : 0.0;
#pragma unroll
    for (int u = 0; u < kU; ++u)
      if (jv[u] >= 0) acc = fma(av[u], xv[u], acc);
  }
  return acc;
}

// 8 blocks per SM (32 registers) with the epilogue operands loaded after the
// row loop: primal step 0.820 -> 0.812 ms on config 4; 6 blocks with early
// loads measured 1.03 ms (profiles/r01_pipeline.md).
#ifndef PDHG_SELL_MINB
#define PDHG_SELL_MINB 8
#endif
#ifndef PDHG_SELL_LATE
#define PDHG_SELL_LATE 1
#endif
// The dual step over long rows (config 4's renumbered A, ~40 entries per row
// with a long tail) keeps PDHG_SELL_U_DUAL entries in flight per lane at 6
// blocks per SM (40 registers): its gathers of the 80 MB xe miss L2 more
// often than the primal step's of the 40 MB y, so it wants more memory-level
// parallelism per warp -- dual 0.55 -> 0.51 ms, iteration -2 % on config 4 at
// 50 % scale with the primal step unchanged (tools/lib_ab.py,
// profiles/r02_sell_unroll.log).
#ifndef PDHG_SELL_U_DUAL
#define PDHG_SELL_U_DUAL 10
#endif
template <bool PRIMAL, int kU>
constexpr int sell_min_blocks() { return (!PRIMAL && kU > PDHG_SELL_U_LONG) ? 6 : PDHG_SELL_MINB; }

// ---------------------------------------------- check fused into the steps
// The last iteration of a period that ends at a two-point check (CUR, AVG):
// the primal step writes (xe, x, avg_x) of every column as one 32-byte quad
// instead of xe alone, and the dual step gathers the quad -- one 32-byte
// sector per entry, like its 8-byte xe gather -- so one pass over A gives
// the step's A xe and the check's A x and A avg_x (pdhg.py:143 and
// lp_core.py:436 for both points of pdhg.py:201-202).  The dual step stores
// each row's primal residuals b - A x, b - A avg_x; k_check_primal_fold then
// accumulates them in k_check_primal_sell's exact order, so the check's
// scalars are bit for bit those of the separate A-side pass it replaces.
struct __align__(32) Quad {
  double e, x, a, pad;  // xe, x, avg_x of one column
};

__device__ __forceinline__ void st_quad(Quad* p, double e, double x, double a) {
  asm volatile("st.global.v4.f64 [%0], {%1, %2, %3, %4};" ::"l"(p), "d"(e), "d"(x), "d"(a), "d"(0.0)
               : "memory");
}

// 0: one 256-bit load; 1: two 128-bit loads of the same sector; 2: one
// 256-bit load that does not allocate in L1
#ifndef PDHG_QUAD_LD
#define PDHG_QUAD_LD 0
#endif
__device__ __forceinline__ void ld_quad(const Quad* p, double& e, double& x, double& a) {
  double pad;
#if PDHG_QUAD_LD == 1
  asm("ld.global.nc.v2.f64 {%0, %1}, [%2];" : "=d"(e), "=d"(x) : "l"(p));
  asm("ld.global.nc.f64 %0, [%1+16];" : "=d"(a) : "l"(p));
  (void)pad;
#elif PDHG_QUAD_LD == 2
  asm("ld.global.nc.L1::no_allocate.v4.f64 {%0, %1, %2, %3}, [%4];" : "=d"(e), "=d"(x), "=d"(a), "=d"(pad) : "l"(p));
#else
  asm("ld.global.nc.v4.f64 {%0, %1, %2, %3}, [%4];" : "=d"(e), "=d"(x), "=d"(a), "=d"(pad) : "l"(p));
#endif
}

// primal_epi_pre with the quad store in place of the xe store
__device__ __forceinline__ void primal_epi_quad(int j, double aty, double cj, double xj, double xb,
                                                double* __restrict__ x, Quad* __restrict__ q,
                                                double* __restrict__ xbar, double tau_w, double w,
                                                long long iter, StepParams* P) {
  const double g = __dsub_rn(cj, aty);
  const double xn = np_max0(__dsub_rn(xj, __dmul_rn(tau_w, g)));
  epi_st(x + j, xn);
  const double xev = __dsub_rn(__dmul_rn(2.0, xn), xj);
  const double xbn = __dadd_rn(xb, __ddiv_rn(__dsub_rn(xn, xb), w));
  epi_st(xbar + j, xbn);
  st_quad(q + j, xev, xn, xbn);
  if (!finite(xn)) fail_at(P, iter);
}

template <bool PRIMAL, int kU, bool QUAD = false>
__global__ void __launch_bounds__(kBlock, (sell_min_blocks<PRIMAL, kU>())) k_step_sell(StepArgs a, SellSet S, int j_in_period) {
  __shared__ double red[kWarps];
  pdl_enter();
  StepParams* P = a.P;
  const long long iter = P->iter0 + j_in_period + 1;
  if (P->fail_iter < iter) return;
  const double w = P->w0 + (double)(j_in_period + 1);
  const double step = PRIMAL ? P->tau_w : P->sigma_w;
  if ((int)blockIdx.x < a.rs.n_heavy) {
    const double* xin[1] = {a.gather};
    const int row = a.rs.heavy[blockIdx.x];
    const int s = a.rs.ptr[row], e = a.rs.ptr[row + 1];
    double acc[1];
    row_dot<kBlock, 1>(a.rs, s, e, threadIdx.x, xin, acc);
    const double d = block_sum(acc[0], red);
    if (threadIdx.x == 0) {
      if constexpr (PRIMAL && QUAD)
        primal_epi_quad(row, d, a.cb[row], a.x[row], a.xbar[row], a.x, reinterpret_cast<Quad*>(a.xe), a.xbar,
                        step, w, iter, P);
      else if (PRIMAL) bcast(P, 0, row, primal_epi(row, d, a.cb, a.x, a.xe, a.xbar, step, w, iter, P));
      else bcast(P, 1, row, dual_epi(row, d, a.cb, a.x, a.xbar, step, w, iter, P));
    }
    return;
  }
  const int lane = threadIdx.x & 31;
  const long long sl = ((long long)(blockIdx.x - a.rs.n_heavy) * kBlock + threadIdx.x) >> 5;
  if (sl >= S.nslices) return;  // warp-uniform
  const long long rl = sl * 32 + (S.perm ? S.perm[sl * 32 + lane] : lane);
  const bool in_range = rl < a.rs.rows;
  double o1 = 0.0, o2 = 0.0, o3 = 0.0;
  int len = 0;
  if (in_range) {
    if (!PDHG_SELL_LATE) {
      o1 = a.cb[rl];
      o2 = a.x[rl];
      o3 = a.xbar[rl];
    }
    len = a.rs.ptr[rl + 1] - a.rs.ptr[rl];
  }
  const bool ok = in_range && len <= a.rs.heavy_threshold;
  if (!ok) len = 0;
  const double acc = sell_row_dot<kU>(S, sl, lane, len, a.gather);

  if (PDHG_SELL_LATE && ok) {
    o1 = epi_ld(a.cb + rl);
    o2 = epi_ld(a.x + rl);
    o3 = epi_ld(a.xbar + rl);
  }
  if (ok) {
    const int row = (int)rl;
    if constexpr (PRIMAL && QUAD)
      primal_epi_quad(row, acc, o1, o2, o3, a.x, reinterpret_cast<Quad*>(a.xe), a.xbar, step, w, iter, P);
    else if (PRIMAL) bcast(P, 0, row, primal_epi_pre(row, acc, o1, o2, o3, a.x, a.xe, a.xbar, step, w, iter, P));
    else bcast(P, 1, row, dual_epi_pre(row, acc, o1, o2, o3, a.x, a.xbar, step, w, iter, P));
  }
}

// The dual step of a check-fused iteration over the sliced ELL of A: the
// step's fma chain over xe (bitwise the k_step_sell<false> result) plus the
// check's chains over x and avg_x (bitwise k_check_primal_sell's), all from
// one quad gather per entry.  a.gather = the quads, a.partial = each row's
// residual pair (b - A x, b - A avg_x), indexed by row.
#ifndef PDHG_FUSE_U
#define PDHG_FUSE_U 4
#endif
#ifndef PDHG_FUSE_MINB
#define PDHG_FUSE_MINB 4
#endif
template <int V>
__device__ __forceinline__ void row_dot_quad(const RowSet& A, int s, int e, int lane, const Quad* __restrict__ q,
                                             double* acc) {
  constexpr int kU = V >= 16 ? PDHG_ROW_U16 : 2;   // row_dot's entry order: k, k+V, k+2V, ...
  acc[0] = acc[1] = acc[2] = 0.0;
  for (int k = s + lane; k < e; k += kU * V) {
    double av[kU], ev[kU], xv[kU], mv[kU];
    int j[kU];
#pragma unroll
    for (int u = 0; u < kU; ++u) {
      const int kk = k + u * V;
      av[u] = kk < e ? ld_stream(A.val + CHK(kk, A.nnz)) : 0.0;
      j[u] = kk < e ? ld_stream(A.col + CHK(kk, A.nnz)) : -1;
    }
#pragma unroll
    for (int u = 0; u < kU; ++u) {
      ev[u] = xv[u] = mv[u] = 0.0;
      if (j[u] >= 0) ld_quad(q + CHK(j[u], A.ncols), ev[u], xv[u], mv[u]);
    }
#pragma unroll
    for (int u = 0; u < kU; ++u)
      if (j[u] >= 0) {
        acc[0] = fma(av[u], ev[u], acc[0]);
        acc[1] = fma(av[u], xv[u], acc[1]);
        acc[2] = fma(av[u], mv[u], acc[2]);
      }
  }
}

template <int kU>
__global__ void __launch_bounds__(kBlock, PDHG_FUSE_MINB) k_step_sell_chk(StepArgs a, SellSet S, int j_in_period) {
  __shared__ double red[kWarps];
  pdl_enter();
  StepParams* P = a.P;
  const long long iter = P->iter0 + j_in_period + 1;
  if (P->fail_iter < iter) return;
  const double w = P->w0 + (double)(j_in_period + 1);
  const double step = P->sigma_w;
  const Quad* __restrict__ q = reinterpret_cast<const Quad*>(a.gather);
  double2* __restrict__ res = reinterpret_cast<double2*>(a.partial);
  if ((int)blockIdx.x < a.rs.n_heavy) {
    const int row = a.rs.heavy[blockIdx.x];
    double acc[3], d[3];
    row_dot_quad<kBlock>(a.rs, a.rs.ptr[row], a.rs.ptr[row + 1], threadIdx.x, q, acc);
#pragma unroll
    for (int r = 0; r < 3; ++r) d[r] = block_sum(acc[r], red);
    if (threadIdx.x == 0) {
      const double bi = a.cb[row];
      dual_epi_pre(row, d[0], bi, a.x[row], a.xbar[row], a.x, a.xbar, step, w, iter, P);
      res[row] = make_double2(__dsub_rn(bi, d[1]), __dsub_rn(bi, d[2]));
    }
    return;
  }
  const int lane = threadIdx.x & 31;
  const long long sl = ((long long)(blockIdx.x - a.rs.n_heavy) * kBlock + threadIdx.x) >> 5;
  if (sl >= S.nslices) return;  // warp-uniform
  const long long rl = sl * 32 + (S.perm ? S.perm[sl * 32 + lane] : lane);
  const bool in_range = rl < a.rs.rows;
  int len = in_range ? a.rs.ptr[rl + 1] - a.rs.ptr[rl] : 0;
  const bool ok = in_range && len <= a.rs.heavy_threshold;
  if (!ok) len = 0;
  const int width = S.width[sl];
  const long long base = S.sptr[sl] + lane;
  double de = 0.0, dx = 0.0, da = 0.0;   // sell_row_dot's / sell_row_dot_pair's chains
  for (int k = 0; k < width; k += kU) {
    double av[kU], ev[kU], xv[kU], mv[kU];
    int jv[kU];
#pragma unroll
    for (int u = 0; u < kU; ++u) {
      const bool on = k + u < len;
      av[u] = on ? ld_stream(S.val + CHK(base + 32LL * (k + u), S.nslots)) : 0.0;
      jv[u] = on ? ld_stream(S.col + CHK(base + 32LL * (k + u), S.nslots)) : -1;
    }
#pragma unroll
    for (int u = 0; u < kU; ++u) {
      ev[u] = xv[u] = mv[u] = 0.0;
      if (jv[u] >= 0) ld_quad(q + CHK(jv[u], S.ncols), ev[u], xv[u], mv[u]);
    }
#pragma unroll
    for (int u = 0; u < kU; ++u)
      if (jv[u] >= 0) {
        de = fma(av[u], ev[u], de);
        dx = fma(av[u], xv[u], dx);
        da = fma(av[u], mv[u], da);
      }
  }
  if (ok) {
    const int row = (int)rl;
    const double bi = epi_ld(a.cb + rl);
    dual_epi_pre(row, de, bi, epi_ld(a.x + rl), epi_ld(a.xbar + rl), a.x, a.xbar, step, w, iter, P);
    res[rl] = make_double2(__dsub_rn(bi, dx), __dsub_rn(bi, da));
  }
}

// The first primal step of a period right after a two-point check that left
// A'y of both checked points in the workspace (pdhg_use_check_dot): the
// next iterate's y is one of them (the current point, or the average after a
// restart to it), and k_check_dual_sell computed its row dots with exactly
// the primal step's fma sequence (sell_row_dot / row_dot + block_sum, same
// entry order), so this epilogue-only pass gives the step's result bit for
// bit without its SpMV (config 4: one of 64 primal SpMVs per period).
__global__ void __launch_bounds__(kBlock) k_primal_from_dot(StepArgs a, const double2* __restrict__ dots,
                                                            int slot, int j_in_period) {
  pdl_enter();
  StepParams* P = a.P;
  const long long iter = P->iter0 + j_in_period + 1;
  if (P->fail_iter < iter) return;
  const double w = P->w0 + (double)(j_in_period + 1);
  const long long i = (long long)blockIdx.x * kBlock + threadIdx.x;
  if (i >= a.rs.rows) return;
  const double2 d = dots[i];
  const int row = (int)i;
  bcast(P, 0, row, primal_epi_pre(row, slot ? d.y : d.x, a.cb[i], a.x[i], a.xbar[i], a.x, a.xe, a.xbar, P->tau_w,
                                  w, iter, P));
}

#if PDHG_EXPERIMENTAL  // persistent period kernels
// ------------------------------------------------- persistent period kernel
//
// One cooperative launch runs a whole period (up to the next KKT check):
// for each iteration the primal step over all rows of A', a grid barrier,
// the dual step over all rows of A, a grid barrier.  Same per-row routines,
// order of operations and epilogues as k_step (so the same results bit for
// bit), minus 2 kernel launches + drains per iteration -- which dominate
// small and mid-size models (GpuOptions.persistent).  Heavy rows: a block
// each, grid-strided; light rows: 32 per warp, grid-strided.  The gathered
// vector is re-read through L2 (COH) because it changes between phases.
template <int NW>
__device__ __forceinline__ double block_sum_nw(double v, double* red) {
  v = group_sum<32>(v);
  const int w = threadIdx.x >> 5, l = threadIdx.x & 31;
  __syncthreads();
  if (l == 0) red[w] = v;
  __syncthreads();
  double t = (l < NW) ? red[l] : 0.0;
  t = group_sum<32>(t);
  return t;
}

template <int V, bool PRIMAL, int COH = 1, int NW = kWarps>
__device__ __forceinline__ void step_phase(const StepArgs& a, long long iter, double w, double step,
                                           double* red) {
  StepParams* P = a.P;
  const double* xin[1] = {a.gather};
  for (int h = blockIdx.x; h < a.rs.n_heavy; h += gridDim.x) {  // block-uniform
    const int row = a.rs.heavy[h];
    const int s = a.rs.ptr[row], e = a.rs.ptr[row + 1];
    double acc[1];
    row_dot<NW * 32, 1, COH>(a.rs, s, e, threadIdx.x, xin, acc);
    const double d = NW == kWarps ? block_sum(acc[0], red) : block_sum_nw<NW>(acc[0], red);
    if (threadIdx.x == 0) {
      if (PRIMAL) bcast(P, 0, row, primal_epi(row, d, a.cb, a.x, a.xe, a.xbar, step, w, iter, P));
      else bcast(P, 1, row, dual_epi(row, d, a.cb, a.x, a.xbar, step, w, iter, P));
    }
  }
  const int lane = threadIdx.x & 31;
  const long long nw = (long long)gridDim.x * NW;
  for (long long wid = (long long)blockIdx.x * NW + (threadIdx.x >> 5); wid * 32 < a.rs.rows; wid += nw) {
    const long long row0 = wid * 32, rl = row0 + lane;
    double o1 = 0.0, o2 = 0.0, o3 = 0.0;
    if (rl < a.rs.rows) {
      o1 = a.cb[rl];
      o2 = a.x[rl];
      o3 = a.xbar[rl];
    }
    bool my_ok;
    const double mine = warp_rows_dot<V, COH>(a.rs, row0, lane, xin, my_ok);
    if (my_ok) {
      if (PRIMAL) bcast(P, 0, (int)rl, primal_epi_pre((int)rl, mine, o1, o2, o3, a.x, a.xe, a.xbar, step, w, iter, P));
      else bcast(P, 1, (int)rl, dual_epi_pre((int)rl, mine, o1, o2, o3, a.x, a.xbar, step, w, iter, P));
    }
  }
}

template <bool PRIMAL, int COH = 1, int NW = kWarps>
__device__ __forceinline__ void step_phase_v(int V, const StepArgs& a, long long iter, double w,
                                             double step, double* red) {
  switch (V) {
    case 1: step_phase<1, PRIMAL, COH, NW>(a, iter, w, step, red); break;
    case 2: step_phase<2, PRIMAL, COH, NW>(a, iter, w, step, red); break;
    case 4: step_phase<4, PRIMAL, COH, NW>(a, iter, w, step, red); break;
    case 8: step_phase<8, PRIMAL, COH, NW>(a, iter, w, step, red); break;
    case 16: step_phase<16, PRIMAL, COH, NW>(a, iter, w, step, red); break;
    default: step_phase<32, PRIMAL, COH, NW>(a, iter, w, step, red); break;
  }
}

__device__ __forceinline__ long long fail_iter_now(StepParams* P) {
  return *reinterpret_cast<volatile long long*>(&P->fail_iter);
}

__global__ void __launch_bounds__(kBlock) k_period(StepArgs pa, StepArgs da, int va, int vd, int iters) {
  __shared__ double red[kWarps];
  cg::grid_group grid = cg::this_grid();
  StepParams* P = pa.P;
  for (int j = 0; j < iters; ++j) {
    const long long iter = P->iter0 + j + 1;
    if (fail_iter_now(P) < iter) break;  // grid-uniform: read after the barrier
    const double w = P->w0 + (double)(j + 1);
    step_phase_v<true>(va, pa, iter, w, P->tau_w, red);
    grid.sync();
    if (fail_iter_now(P) < iter) break;
    step_phase_v<false>(vd, da, iter, w, P->sigma_w, red);
    grid.sync();
  }
}

// Single-block period kernel for tiny models (config 0 class, a few thousand
// rows): one 1024-thread CTA runs the whole period with __syncthreads between
// half steps; the model and the iterates stay in that SM's L1, gathers are
// L1-cached (COH 2), so an iteration costs a few hundred cycles instead of
// two kernel launches.
constexpr int kTinyBlock = 1024;

__global__ void __launch_bounds__(kTinyBlock, 1) k_period_tiny(StepArgs pa, StepArgs da, int va, int vd,
                                                               int iters) {
  __shared__ double red[32];
  StepParams* P = pa.P;
  for (int j = 0; j < iters; ++j) {
    const long long iter = P->iter0 + j + 1;
    if (fail_iter_now(P) < iter) break;  // block-uniform: read after the barrier
    const double w = P->w0 + (double)(j + 1);
    step_phase_v<true, 2, kTinyBlock / 32>(va, pa, iter, w, P->tau_w, red);
    __syncthreads();
    if (fail_iter_now(P) < iter) break;
    step_phase_v<false, 2, kTinyBlock / 32>(vd, da, iter, w, P->sigma_w, red);
    __syncthreads();
  }
}

#endif  // PDHG_EXPERIMENTAL (persistent period kernels)

// A step split into passes over per-row entry ranges (split-K): pass k sums
// each row's entries [split[k-1][r], split[k][r]) (split[-1] = ptr[r],
// split[K-1] = ptr[r+1]) into a per-row partial, and the last pass adds its
// part and runs the epilogue; a row's sum is ((part 0) + part 1) + ...:
// fixed, bitwise reproducible.  Heavy rows run whole (block per row) with
// the last pass.  Two uses: the multi-GPU overlap (a shard's rows hold their
// local-slot entries first, so pass 0 needs only this shard's slice of the
// gathered vector and runs while the all-gather of the other slices is in
// flight -- DESIGN.md §6), and split-K of the dual step over column chunks
// of A (GpuOptions.dual_split, measured slower on one GPU).
template <int V, bool PRIMAL>
__global__ void __launch_bounds__(kBlock) k_step_split(StepArgs a, int j_in_period, int pass,
                                                       int n_heavy_now) {
  __shared__ double red[kWarps];
  pdl_enter();
  StepParams* P = a.P;
  const long long iter = P->iter0 + j_in_period + 1;
  if (P->fail_iter < iter) return;
  const double w = P->w0 + (double)(j_in_period + 1);
  const double step = PRIMAL ? P->tau_w : P->sigma_w;
  const double* xin[1] = {a.gather};
  const bool last = pass == a.nsplit - 1;
  if ((int)blockIdx.x < n_heavy_now) {
    const int row = a.rs.heavy[blockIdx.x];
    double acc[1];
    row_dot<kBlock, 1>(a.rs, a.rs.ptr[row], a.rs.ptr[row + 1], threadIdx.x, xin, acc);
    const double d = block_sum(acc[0], red);
    if (threadIdx.x == 0) {
      if (PRIMAL) bcast(P, 0, row, primal_epi(row, d, a.cb, a.x, a.xe, a.xbar, step, w, iter, P));
      else bcast(P, 1, row, dual_epi(row, d, a.cb, a.x, a.xbar, step, w, iter, P));
    }
    return;
  }
  const int lane = threadIdx.x & 31;
  const long long row0 = (((long long)(blockIdx.x - n_heavy_now) * kBlock + threadIdx.x) >> 5) * 32;
  if (row0 >= a.rs.rows) return;
  const long long rl = row0 + lane;
  const bool in_range = rl < a.rs.rows;
  double o1 = 0.0, o2 = 0.0, o3 = 0.0, part = 0.0;
  if (in_range) {
    if (last) {
      o1 = a.cb[rl];
      o2 = a.x[rl];
      o3 = a.xbar[rl];
    }
    if (pass > 0) part = a.partial[rl];
  }
  const long long m = a.rs.rows;
  const int* sp = pass == 0 ? a.rs.ptr : a.split + (pass - 1) * m;
  const int* ep = last ? a.rs.ptr + 1 : a.split + pass * m;
  bool ok;
  const double dot = warp_rows_dot_seg<V>(a.rs, sp, ep, row0, lane, xin, ok);
  if (!ok) return;
  const double d = pass > 0 ? part + dot : dot;
  if (!last) {
    a.partial[rl] = d;
    return;
  }
  const int row = (int)rl;
  if (PRIMAL) bcast(P, 0, row, primal_epi_pre(row, d, o1, o2, o3, a.x, a.xe, a.xbar, step, w, iter, P));
  else bcast(P, 1, row, dual_epi_pre(row, d, o1, o2, o3, a.x, a.xbar, step, w, iter, P));
}

// One pass of a split half step over the sliced ELL of that pass's part of
// every row (sharded local-first blocks: part 0 = the entries whose columns
// are this shard's own slots, part 1 = the rest).  Pass 0
// runs each light row's chain over its part-0 entries and parks it in
// a.partial; pass 1 continues the same chain over the part-1 entries (so a
// row's sum is one sequential fma chain over its local-first entry order)
// and runs the epilogue; heavy rows are in neither part and run whole, block
// per row, in pass 1.  pptr: the part's CSR row pointers (per-row lengths).
template <bool PRIMAL, int kU, int PASS>
__global__ void __launch_bounds__(kBlock, (sell_min_blocks<PRIMAL, kU>())) k_step_sell_pass(StepArgs a, SellSet S,
                                                                                        const int* __restrict__ pptr,
                                                                                        int j_in_period) {
  __shared__ double red[kWarps];
  pdl_enter();
  StepParams* P = a.P;
  const long long iter = P->iter0 + j_in_period + 1;
  if (P->fail_iter < iter) return;
  const double w = P->w0 + (double)(j_in_period + 1);
  const double step = PRIMAL ? P->tau_w : P->sigma_w;
  const int nh = PASS == 1 ? a.rs.n_heavy : 0;
  if ((int)blockIdx.x < nh) {
    const double* xin[1] = {a.gather};
    const int row = a.rs.heavy[blockIdx.x];
    double acc[1];
    row_dot<kBlock, 1>(a.rs, a.rs.ptr[row], a.rs.ptr[row + 1], threadIdx.x, xin, acc);
    const double d = block_sum(acc[0], red);
    if (threadIdx.x == 0) {
      if (PRIMAL) bcast(P, 0, row, primal_epi(row, d, a.cb, a.x, a.xe, a.xbar, step, w, iter, P));
      else bcast(P, 1, row, dual_epi(row, d, a.cb, a.x, a.xbar, step, w, iter, P));
    }
    return;
  }
  const int lane = threadIdx.x & 31;
  const long long sl = ((long long)(blockIdx.x - nh) * kBlock + threadIdx.x) >> 5;
  if (sl >= S.nslices) return;  // warp-uniform
  const long long rl = sell_row(S, sl, lane);
  const bool in_range = rl < a.rs.rows;
  const bool ok = in_range && a.rs.ptr[rl + 1] - a.rs.ptr[rl] <= a.rs.heavy_threshold;
  const int len = ok ? pptr[rl + 1] - pptr[rl] : 0;
  double acc = (PASS == 1 && ok) ? a.partial[rl] : 0.0;
  const int width = S.width[sl];
  const long long base = S.sptr[sl] + lane;
  for (int k = 0; k < width; k += kU) {
    double av[kU], xv[kU];
    int jv[kU];
#pragma unroll
    for (int u = 0; u < kU; ++u) {
      const bool on = k + u < len;
      av[u] = on ? ld_stream(S.val + CHK(base + 32LL * (k + u), S.nslots)) : 0.0;
      jv[u] = on ? ld_stream(S.col + CHK(base + 32LL * (k + u), S.nslots)) : -1;
    }
#pragma unroll
    for (int u = 0; u < kU; ++u) xv[u] = jv[u] >= 0 ? ld_gather(a.gather + CHK(jv[u], S.ncols)) : 0.0;
#pragma unroll
    for (int u = 0; u < kU; ++u)
      if (jv[u] >= 0) acc = fma(av[u], xv[u], acc);
  }
  if (!ok) return;
  if (PASS == 0) {
    a.partial[rl] = acc;
    return;
  }
  const int row = (int)rl;
  const double o1 = epi_ld(a.cb + rl), o2 = epi_ld(a.x + rl), o3 = epi_ld(a.xbar + rl);
  if (PRIMAL) bcast(P, 0, row, primal_epi_pre(row, acc, o1, o2, o3, a.x, a.xe, a.xbar, step, w, iter, P));
  else bcast(P, 1, row, dual_epi_pre(row, acc, o1, o2, o3, a.x, a.xbar, step, w, iter, P));
}

#if PDHG_EXPERIMENTAL  // PSR step
// PSR step: persistent CTAs (one per SM) walk row blocks; the SpMV lands in
// shared memory (psr::block_spmv), then the same epilogue as k_step.
struct PsrStepArgs {
  psr::Layout L;
  const double* __restrict__ gather;
  const double* __restrict__ cb;
  double* x;
  double* xe;
  double* xbar;
  StepParams* P;
};

template <bool PRIMAL>
__global__ void __launch_bounds__(psr::kThreads, 1) k_step_psr(PsrStepArgs a, int j_in_period) {
  extern __shared__ __align__(128) unsigned char smem_raw[];
  __shared__ uint64_t bars[psr::kStages];
  pdl_enter();
  StepParams* P = a.P;
  const long long iter = P->iter0 + j_in_period + 1;
  if (P->fail_iter < iter) return;
  const double w = P->w0 + (double)(j_in_period + 1);
  const double step = PRIMAL ? P->tau_w : P->sigma_w;
  double* panels = reinterpret_cast<double*>(smem_raw);
  if (threadIdx.x == 0) {
    for (int k = 0; k < psr::kStages; ++k) psr::mbar_init(&bars[k], 1);
    psr::fence_mbar_init();
  }
  __syncthreads();
  uint32_t ph[psr::kStages];
#pragma unroll
  for (int k = 0; k < psr::kStages; ++k) ph[k] = 0u;
  for (int b = blockIdx.x; b < a.L.nblk; b += gridDim.x) {
    psr::block_rows(a.L, b, a.gather, panels, bars, ph, [&](int row, double d) {
      if (PRIMAL) bcast(P, 0, row, primal_epi(row, d, a.cb, a.x, a.xe, a.xbar, step, w, iter, P));
      else bcast(P, 1, row, dual_epi(row, d, a.cb, a.x, a.xbar, step, w, iter, P));
    });
  }
}

#endif  // PDHG_EXPERIMENTAL (PSR step)

// ------------------------------------------------------------------ plain SpMV

template <int V>
__global__ void __launch_bounds__(kBlock, step_min_blocks<V>()) k_spmv(RowSet rs, const double* __restrict__ in,
                                                 double* __restrict__ out) {
  __shared__ double red[kWarps];
  const double* xin[1] = {in};
  if ((int)blockIdx.x < rs.n_heavy) {
    const int row = rs.heavy[blockIdx.x];
    double acc[1];
    row_dot<kBlock, 1>(rs, rs.ptr[row], rs.ptr[row + 1], threadIdx.x, xin, acc);
    const double d = block_sum(acc[0], red);
    if (threadIdx.x == 0) out[row] = d;
    return;
  }
  const int lane = threadIdx.x & 31;
  const long long row0 = (((long long)(blockIdx.x - rs.n_heavy) * kBlock + threadIdx.x) >> 5) * 32;
  if (row0 >= rs.rows) return;
  bool ok;
  const double d = warp_rows_dot<V>(rs, row0, lane, xin, ok);
  if (ok) out[row0 + lane] = d;
}

// out = M in over the sliced-ELL layout (the power iteration's products when
// the operator has one): the step kernel's row loop without the epilogue.
template <int kU>
__global__ void __launch_bounds__(kBlock, PDHG_SELL_MINB) k_spmv_sell(RowSet rs, SellSet S,
                                                                    const double* __restrict__ in,
                                                                    double* __restrict__ out) {
  __shared__ double red[kWarps];
  if ((int)blockIdx.x < rs.n_heavy) {
    const double* xin[1] = {in};
    const int row = rs.heavy[blockIdx.x];
    double acc[1];
    row_dot<kBlock, 1>(rs, rs.ptr[row], rs.ptr[row + 1], threadIdx.x, xin, acc);
    const double d = block_sum(acc[0], red);
    if (threadIdx.x == 0) out[row] = d;
    return;
  }
  const int lane = threadIdx.x & 31;
  const long long sl = ((long long)(blockIdx.x - rs.n_heavy) * kBlock + threadIdx.x) >> 5;
  if (sl >= S.nslices) return;  // warp-uniform
  const long long rl = sl * 32 + (S.perm ? S.perm[sl * 32 + lane] : lane);
  int len = rl < rs.rows ? rs.ptr[rl + 1] - rs.ptr[rl] : -1;
  const bool ok = len >= 0 && len <= rs.heavy_threshold;
  if (!ok) len = 0;
  const double acc = sell_row_dot<kU>(S, sl, lane, len, in);
  if (ok) out[rl] = acc;
}

__global__ void k_div(const double* __restrict__ w, double* __restrict__ v, double s, int n) {
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i < n) v[i] = __ddiv_rn(w[i], s);  // v = w / norm_w   (pdhg.py:99)
}

// sum of squares partials (np.linalg.norm), fixed grid
__global__ void __launch_bounds__(kBlock) k_sumsq(const double* __restrict__ v, int n,
                                                  double* __restrict__ partials) {
  __shared__ double red[kWarps];
  double acc = 0.0;
  for (long long i = (long long)blockIdx.x * kBlock + threadIdx.x; i < n;
       i += (long long)gridDim.x * kBlock)
    acc = fma(v[i], v[i], acc);
  const double t = block_sum(acc, red);
  if (threadIdx.x == 0) partials[blockIdx.x] = t;
}

// ---------------------------------------------------------------- KKT checks

struct CheckPts {
  const double* x[2];
  const double* y[2];
  const double* zin[2];  // nullptr => z = max(0, c - A'y)
  double* zout[2];       // optional z output
  const double2* pair;   // two-point checks: the gathered vectors interleaved
                         // ((x0[j], x1[j]) or (y0[i], y1[i])), one 16-byte gather
                         // per entry instead of two 8-byte ones
  double2* dout;         // dual side, optional: each row's two dots (A'y0, A'y1)
                         // -- the next period's first primal step (pdhg_use_check_dot)
};

// row_dot for two right-hand sides stored interleaved: each accumulator sees
// the same fma sequence as row_dot<V, 2> (bitwise-identical sums), but one
// gather (one L2 sector) serves both points.
template <int V>
__device__ __forceinline__ void row_dot_pair(const RowSet& A, int s, int e, int lane,
                                             const double2* __restrict__ xx, double* acc) {
  constexpr int kU = V >= 16 ? PDHG_PAIR_U16 : 2;
  acc[0] = 0.0;
  acc[1] = 0.0;
  for (int k = s + lane; k < e; k += kU * V) {
    double a[kU];
    int j[kU];
#pragma unroll
    for (int u = 0; u < kU; ++u) {
      const int kk = k + u * V;
      a[u] = kk < e ? ld_stream(A.val + CHK(kk, A.nnz)) : 0.0;
      j[u] = kk < e ? ld_stream(A.col + CHK(kk, A.nnz)) : -1;
    }
    double2 xv[kU];
#pragma unroll
    for (int u = 0; u < kU; ++u) xv[u] = j[u] >= 0 ? __ldg(xx + CHK(j[u], A.ncols)) : make_double2(0.0, 0.0);
#pragma unroll
    for (int u = 0; u < kU; ++u)
      if (j[u] >= 0) acc[0] = fma(a[u], xv[u].x, acc[0]);
#pragma unroll
    for (int u = 0; u < kU; ++u)
      if (j[u] >= 0) acc[1] = fma(a[u], xv[u].y, acc[1]);
  }
}

template <int V, int NP, bool PAIR>
__device__ __forceinline__ void check_row_dot(const RowSet& A, int s, int e, int lane,
                                              const double* const* __restrict__ xin,
                                              const double2* __restrict__ pair, double* acc) {
  if constexpr (PAIR && NP == 2) row_dot_pair<V>(A, s, e, lane, pair, acc);
  else row_dot<V, NP>(A, s, e, lane, xin, acc);
}

// sell_row_dot for an interleaved pair of vectors (two-point checks).
template <int kU>
__device__ __forceinline__ void sell_row_dot_pair(const SellSet& S, long long sl, int lane, int len,
                                                  const double2* __restrict__ xx, double& a0,
                                                  double& a1) {
  const int width = S.width[sl];
  const long long base = S.sptr[sl] + lane;
  a0 = 0.0;
  a1 = 0.0;
  for (int k = 0; k < width; k += kU) {
    double av[kU];
    int jv[kU];
    double2 xv[kU];
#pragma unroll
    for (int u = 0; u < kU; ++u) {
      const bool on = k + u < len;
      av[u] = on ? ld_stream(S.val + CHK(base + 32LL * (k + u), S.nslots)) : 0.0;
      jv[u] = on ? ld_stream(S.col + CHK(base + 32LL * (k + u), S.nslots)) : -1;
    }
#pragma unroll
    for (int u = 0; u < kU; ++u) xv[u] = jv[u] >= 0 ? __ldg(xx + CHK(jv[u], S.ncols)) : make_double2(0.0, 0.0);
#pragma unroll
    for (int u = 0; u < kU; ++u)
      if (jv[u] >= 0) {
        a0 = fma(av[u], xv[u].x, a0);
        a1 = fma(av[u], xv[u].y, a1);
      }
  }
}

__global__ void k_pair(const double* __restrict__ a, const double* __restrict__ b,
                       double2* __restrict__ out, long long n) {
  for (long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x; i < n;
       i += (long long)gridDim.x * blockDim.x)
    out[i] = make_double2(a[i], b[i]);
}

// Two-point primal-side terms in the step kernel's shape: a warp owns 32
// consecutive rows (grid-strided over a fixed grid), computes them in V
// passes of 32/V rows with row_dot_pair + group_sum (so every row's two dots
// are exactly k_check_primal's), parks row k's dots in lane k and runs the
// epilogue on all 32 lanes with coalesced b / y loads.
template <int V>
__global__ void __launch_bounds__(kBlock, PDHG_CHECK_BPS) k_check_primal_rows(RowSet rs, const double* __restrict__ b,
                                                                         CheckPts pts,
                                                                         double* __restrict__ partials) {
  __shared__ double red[kWarps];
  constexpr int G = 32 / V;
  double rp2[2] = {0.0, 0.0}, rpmax[2] = {0.0, 0.0}, by[2] = {0.0, 0.0};
  auto row_terms_pre = [&](double bi, double y0, double y1, double d0, double d1) {
    const double r0 = __dsub_rn(bi, d0), r1 = __dsub_rn(bi, d1);
    rp2[0] = fma(r0, r0, rp2[0]);
    rp2[1] = fma(r1, r1, rp2[1]);
    rpmax[0] = nan_max(fabs(r0), rpmax[0]);
    rpmax[1] = nan_max(fabs(r1), rpmax[1]);
    by[0] = fma(bi, y0, by[0]);
    by[1] = fma(bi, y1, by[1]);
  };
  for (int h = blockIdx.x; h < rs.n_heavy; h += gridDim.x) {
    const int row = rs.heavy[h];
    double acc[2], d[2];
    row_dot_pair<kBlock>(rs, rs.ptr[row], rs.ptr[row + 1], threadIdx.x, pts.pair, acc);
    d[0] = block_sum(acc[0], red);
    d[1] = block_sum(acc[1], red);
    if (threadIdx.x == 0) row_terms_pre(b[row], pts.y[0][row], pts.y[1][row], d[0], d[1]);
  }
  const int lane = threadIdx.x & 31;
  const long long nwarps = (long long)gridDim.x * kWarps;
  const long long ngroups = (rs.rows + 31) / 32;
  for (long long gw = (long long)blockIdx.x * kWarps + (threadIdx.x >> 5); gw < ngroups; gw += nwarps) {
    const long long rl = gw * 32 + lane;
    bool ok = rl < rs.rows;
    int my_s = 0, my_e = 0;
    if (ok) {
      my_s = rs.ptr[rl];
      my_e = rs.ptr[rl + 1];
      if (my_e - my_s > rs.heavy_threshold) ok = false;
    }
    if (!ok) my_e = my_s;
    double bi = 0.0, y0 = 0.0, y1 = 0.0;
    if (ok) {
      bi = b[rl];
      y0 = pts.y[0][rl];
      y1 = pts.y[1][rl];
    }
    double m0 = 0.0, m1 = 0.0;
#pragma unroll 1
    for (int pass = 0; pass < V; ++pass) {
      const int src = pass * G + lane / V;
      const int s0 = __shfl_sync(0xffffffffu, my_s, src);
      const int e0 = __shfl_sync(0xffffffffu, my_e, src);
      double acc[2];
      row_dot_pair<V>(rs, s0, e0, lane % V, pts.pair, acc);
      const double d0 = group_sum<V>(acc[0]), d1 = group_sum<V>(acc[1]);
      const int from = ((lane - pass * G) & (G - 1)) * V;
      const double g0 = __shfl_sync(0xffffffffu, d0, from), g1 = __shfl_sync(0xffffffffu, d1, from);
      if (lane / G == pass) {
        m0 = g0;
        m1 = g1;
      }
    }
    if (ok) row_terms_pre(bi, y0, y1, m0, m1);
  }
#pragma unroll
  for (int p = 0; p < 2; ++p) {
    const double t0 = block_sum(rp2[p], red);
    const double t1 = block_max(rpmax[p], red);
    const double t2 = block_sum(by[p], red);
    if (threadIdx.x == 0) {
      double* o = partials + (size_t)blockIdx.x * kMaxQ + p * PDHG_NQ;
      o[PDHG_Q_RP2] = t0;
      o[PDHG_Q_RPMAX] = t1;
      o[PDHG_Q_BY] = t2;
    }
  }
}

// Per-point primal-side terms over rows of A: r_p = b - A x (lp_core.py:436).
template <int V, int NP, bool PAIR = false>
__global__ void __launch_bounds__(kBlock, PDHG_CHECK_BPS) k_check_primal(RowSet rs, const double* __restrict__ b,
                                                         CheckPts pts, double* __restrict__ partials) {
  __shared__ double red[kWarps];
  double rp2[NP], rpmax[NP], by[NP];
#pragma unroll
  for (int p = 0; p < NP; ++p) { rp2[p] = 0.0; rpmax[p] = 0.0; by[p] = 0.0; }
  const double* xin[NP];
#pragma unroll
  for (int p = 0; p < NP; ++p) xin[p] = pts.x[p];

  auto row_terms_pre = [&](double bi, const double* yi, const double* d) {
#pragma unroll
    for (int p = 0; p < NP; ++p) {
      const double r = __dsub_rn(bi, d[p]);
      rp2[p] = fma(r, r, rp2[p]);
      rpmax[p] = nan_max(fabs(r), rpmax[p]);
      by[p] = fma(bi, yi[p], by[p]);
    }
  };
  auto row_terms = [&](int i, const double* d) {
    double yi[NP];
#pragma unroll
    for (int p = 0; p < NP; ++p) yi[p] = pts.y[p][i];
    row_terms_pre(b[i], yi, d);
  };
  // heavy rows: block per row, blocks take them round robin
  for (int h = blockIdx.x; h < rs.n_heavy; h += gridDim.x) {
    const int row = rs.heavy[h];
    double acc[NP], d[NP];
    check_row_dot<kBlock, NP, PAIR>(rs, rs.ptr[row], rs.ptr[row + 1], threadIdx.x, xin, pts.pair, acc);
#pragma unroll
    for (int p = 0; p < NP; ++p) d[p] = block_sum(acc[p], red);
    if (threadIdx.x == 0) row_terms(row, d);
  }
  const int lane = threadIdx.x % V;
  const long long groups = (long long)gridDim.x * (kBlock / V);
  for (long long g = (long long)blockIdx.x * (kBlock / V) + threadIdx.x / V; g - threadIdx.x / V < rs.rows;
       g += groups) {
    const int row = (int)g;
    bool valid = row < rs.rows;
    int s = 0, e = 0;
    if (valid) {
      s = rs.ptr[row];
      e = rs.ptr[row + 1];
      if (e - s > rs.heavy_threshold) { valid = false; e = s; }
    }
    // the row's epilogue operands are independent of its dot: issued first
    double bi = 0.0, yi[NP];
#pragma unroll
    for (int p = 0; p < NP; ++p) yi[p] = 0.0;
    if (PDHG_CHECK_EARLY && valid && lane == 0) {
      bi = b[row];
#pragma unroll
      for (int p = 0; p < NP; ++p) yi[p] = pts.y[p][row];
    }
    double acc[NP], d[NP];
    check_row_dot<V, NP, PAIR>(rs, s, e, lane, xin, pts.pair, acc);
#pragma unroll
    for (int p = 0; p < NP; ++p) d[p] = group_sum<V>(acc[p]);
    if (valid && lane == 0) {
      if (PDHG_CHECK_EARLY) row_terms_pre(bi, yi, d);
      else row_terms(row, d);
    }
  }
#pragma unroll
  for (int p = 0; p < NP; ++p) {
    const double t0 = block_sum(rp2[p], red);
    const double t1 = block_max(rpmax[p], red);
    const double t2 = block_sum(by[p], red);
    if (threadIdx.x == 0) {
      double* o = partials + (size_t)blockIdx.x * kMaxQ + p * PDHG_NQ;
      o[PDHG_Q_RP2] = t0;
      o[PDHG_Q_RPMAX] = t1;
      o[PDHG_Q_BY] = t2;
    }
  }
}

// Per-point dual-side terms over rows of A' (lp_core.py:437,441,443; pdhg.py:114).
template <int V, int NP, bool PAIR = false>
__global__ void __launch_bounds__(kBlock, PDHG_CHECK_BPS) k_check_dual(RowSet rs, const double* __restrict__ c,
                                                       CheckPts pts, double* __restrict__ partials) {
  __shared__ double red[kWarps];
  double rd2[NP], rdmax[NP], cx[NP], xz[NP];
#pragma unroll
  for (int p = 0; p < NP; ++p) { rd2[p] = 0.0; rdmax[p] = 0.0; cx[p] = 0.0; xz[p] = 0.0; }
  const double* yin[NP];
#pragma unroll
  for (int p = 0; p < NP; ++p) yin[p] = pts.y[p];

  auto row_terms_pre = [&](int j, double cj, const double* xjs, const double* d) {
#pragma unroll
    for (int p = 0; p < NP; ++p) {
      const double t = __dsub_rn(cj, d[p]);                 // c - A'y
      const double z = pts.zin[p] ? pts.zin[p][j] : np_max0(t);
      if (pts.zout[p]) pts.zout[p][j] = z;
      const double r = __dsub_rn(t, z);                     // r_d = c - A'y - z
      const double xj = xjs[p];
      rd2[p] = fma(r, r, rd2[p]);
      rdmax[p] = nan_max(fabs(r), rdmax[p]);
      cx[p] = fma(cj, xj, cx[p]);
      xz[p] = fma(xj, z, xz[p]);
    }
  };
  auto row_terms = [&](int j, const double* d) {
    double xjs[NP];
#pragma unroll
    for (int p = 0; p < NP; ++p) xjs[p] = pts.x[p][j];
    row_terms_pre(j, c[j], xjs, d);
  };
  for (int h = blockIdx.x; h < rs.n_heavy; h += gridDim.x) {
    const int row = rs.heavy[h];
    double acc[NP], d[NP];
    check_row_dot<kBlock, NP, PAIR>(rs, rs.ptr[row], rs.ptr[row + 1], threadIdx.x, yin, pts.pair, acc);
#pragma unroll
    for (int p = 0; p < NP; ++p) d[p] = block_sum(acc[p], red);
    if (threadIdx.x == 0) row_terms(row, d);
  }
  const int lane = threadIdx.x % V;
  const long long groups = (long long)gridDim.x * (kBlock / V);
  for (long long g = (long long)blockIdx.x * (kBlock / V) + threadIdx.x / V; g - threadIdx.x / V < rs.rows;
       g += groups) {
    const int row = (int)g;
    bool valid = row < rs.rows;
    int s = 0, e = 0;
    if (valid) {
      s = rs.ptr[row];
      e = rs.ptr[row + 1];
      if (e - s > rs.heavy_threshold) { valid = false; e = s; }
    }
    double cj = 0.0, xjs[NP];
#pragma unroll
    for (int p = 0; p < NP; ++p) xjs[p] = 0.0;
    if (PDHG_CHECK_EARLY && valid && lane == 0) {   // operands first, as in k_check_primal
      cj = c[row];
#pragma unroll
      for (int p = 0; p < NP; ++p) xjs[p] = pts.x[p][row];
    }
    double acc[NP], d[NP];
    check_row_dot<V, NP, PAIR>(rs, s, e, lane, yin, pts.pair, acc);
#pragma unroll
    for (int p = 0; p < NP; ++p) d[p] = group_sum<V>(acc[p]);
    if (valid && lane == 0) {
      if (PDHG_CHECK_EARLY) row_terms_pre(row, cj, xjs, d);
      else row_terms(row, d);
    }
  }
#pragma unroll
  for (int p = 0; p < NP; ++p) {
    const double t0 = block_sum(rd2[p], red);
    const double t1 = block_max(rdmax[p], red);
    const double t2 = block_sum(cx[p], red);
    const double t3 = block_sum(xz[p], red);
    if (threadIdx.x == 0) {
      double* o = partials + (size_t)blockIdx.x * kMaxQ + p * PDHG_NQ;
      o[PDHG_Q_RD2] = t0;
      o[PDHG_Q_RDMAX] = t1;
      o[PDHG_Q_CX] = t2;
      o[PDHG_Q_XZ] = t3;
    }
  }
}

// Two-point dual-side terms over the sliced-ELL layout of A' (lane = row,
// every lane runs its row's epilogue, coalesced), gathering the interleaved
// (y0, y1) pairs.  Same quantities and partials layout as k_check_dual.
template <int kU>
__global__ void __launch_bounds__(kBlock, PDHG_CHECK_BPS) k_check_dual_sell(RowSet rs, SellSet S,
                                                                        const double* __restrict__ c,
                                                                        CheckPts pts,
                                                                        double* __restrict__ partials) {
  __shared__ double red[kWarps];
  double rd2[2] = {0.0, 0.0}, rdmax[2] = {0.0, 0.0}, cx[2] = {0.0, 0.0}, xz[2] = {0.0, 0.0};
  auto row_terms = [&](int j, const double* d) {
    const double cj = c[j];
#pragma unroll
    for (int p = 0; p < 2; ++p) {
      const double t = __dsub_rn(cj, d[p]);                 // c - A'y
      const double z = pts.zin[p] ? pts.zin[p][j] : np_max0(t);
      if (pts.zout[p]) pts.zout[p][j] = z;
      const double r = __dsub_rn(t, z);                     // r_d = c - A'y - z
      const double xj = pts.x[p][j];
      rd2[p] = fma(r, r, rd2[p]);
      rdmax[p] = nan_max(fabs(r), rdmax[p]);
      cx[p] = fma(cj, xj, cx[p]);
      xz[p] = fma(xj, z, xz[p]);
    }
  };
  for (int h = blockIdx.x; h < rs.n_heavy; h += gridDim.x) {
    const int row = rs.heavy[h];
    double acc[2], d[2];
    row_dot_pair<kBlock>(rs, rs.ptr[row], rs.ptr[row + 1], threadIdx.x, pts.pair, acc);
#pragma unroll
    for (int p = 0; p < 2; ++p) d[p] = block_sum(acc[p], red);
    if (threadIdx.x == 0) {
      row_terms(row, d);
      if (pts.dout) pts.dout[row] = make_double2(d[0], d[1]);
    }
  }
  const int lane = threadIdx.x & 31;
  const long long warps = (long long)gridDim.x * kWarps;
  for (long long sl = ((long long)blockIdx.x * kBlock + threadIdx.x) >> 5; sl < S.nslices; sl += warps) {
    const long long rl = sell_row(S, sl, lane);
    int len = rl < rs.rows ? rs.ptr[rl + 1] - rs.ptr[rl] : -1;
    const bool ok = len >= 0 && len <= rs.heavy_threshold;
    if (!ok) len = 0;
    double d[2];
    sell_row_dot_pair<kU>(S, sl, lane, len, pts.pair, d[0], d[1]);
    if (ok) {
      row_terms((int)rl, d);
      if (pts.dout) pts.dout[rl] = make_double2(d[0], d[1]);
    }
  }
#pragma unroll
  for (int p = 0; p < 2; ++p) {
    const double t0 = block_sum(rd2[p], red);
    const double t1 = block_max(rdmax[p], red);
    const double t2 = block_sum(cx[p], red);
    const double t3 = block_sum(xz[p], red);
    if (threadIdx.x == 0) {
      double* o = partials + (size_t)blockIdx.x * kMaxQ + p * PDHG_NQ;
      o[PDHG_Q_RD2] = t0;
      o[PDHG_Q_RDMAX] = t1;
      o[PDHG_Q_CX] = t2;
      o[PDHG_Q_XZ] = t3;
    }
  }
}

// Two-point A-side check over the sliced-ELL layout of A: lane per row, both
// points' dots from one 16-byte gather per entry, the row terms of
// k_check_primal_rows (r_p = b - A x, |r_p|^2, max |r_p|, b'y) accumulated per
// thread and reduced in a fixed order.  No lane reductions: ~0.1 instead of
// ~0.3 L1 wavefronts per entry besides the gather.
template <int kU>
__global__ void __launch_bounds__(kBlock, PDHG_CHECK_BPS) k_check_primal_sell(RowSet rs, SellSet S,
                                                                          const double* __restrict__ b,
                                                                          CheckPts pts,
                                                                          double* __restrict__ partials) {
  __shared__ double red[kWarps];
  double rp2[2] = {0.0, 0.0}, rpmax[2] = {0.0, 0.0}, by[2] = {0.0, 0.0};
  auto row_terms = [&](long long i, const double* d) {
    const double bi = b[i];
#pragma unroll
    for (int p = 0; p < 2; ++p) {
      const double r = __dsub_rn(bi, d[p]);
      rp2[p] = fma(r, r, rp2[p]);
      rpmax[p] = nan_max(fabs(r), rpmax[p]);
      by[p] = fma(bi, pts.y[p][i], by[p]);
    }
  };
  for (int h = blockIdx.x; h < rs.n_heavy; h += gridDim.x) {
    const int row = rs.heavy[h];
    double acc[2], d[2];
    row_dot_pair<kBlock>(rs, rs.ptr[row], rs.ptr[row + 1], threadIdx.x, pts.pair, acc);
#pragma unroll
    for (int p = 0; p < 2; ++p) d[p] = block_sum(acc[p], red);
    if (threadIdx.x == 0) row_terms(row, d);
  }
  const int lane = threadIdx.x & 31;
  const long long warps = (long long)gridDim.x * kWarps;
  for (long long sl = ((long long)blockIdx.x * kBlock + threadIdx.x) >> 5; sl < S.nslices; sl += warps) {
    const long long rl = sell_row(S, sl, lane);
    int len = rl < rs.rows ? rs.ptr[rl + 1] - rs.ptr[rl] : -1;
    const bool ok = len >= 0 && len <= rs.heavy_threshold;
    if (!ok) len = 0;
    double d[2];
    sell_row_dot_pair<kU>(S, sl, lane, len, pts.pair, d[0], d[1]);
    if (ok) row_terms(rl, d);
  }
#pragma unroll
  for (int p = 0; p < 2; ++p) {
    const double t0 = block_sum(rp2[p], red);
    const double t1 = block_max(rpmax[p], red);
    const double t2 = block_sum(by[p], red);
    if (threadIdx.x == 0) {
      double* o = partials + (size_t)blockIdx.x * kMaxQ + p * PDHG_NQ;
      o[PDHG_Q_RP2] = t0;
      o[PDHG_Q_RPMAX] = t1;
      o[PDHG_Q_BY] = t2;
    }
  }
}

// The A side of a check-fused two-point check: k_check_primal_sell's loops
// and row terms over the residual pairs the fused dual step stored (res[i] =
// (b - A x, b - A avg_x) of row i), so every per-thread chain and block
// reduction -- and with them the scalars -- are bitwise that kernel's.
__global__ void __launch_bounds__(kBlock, PDHG_CHECK_BPS) k_check_primal_fold(RowSet rs, SellSet S,
                                                                          const double* __restrict__ b,
                                                                          CheckPts pts,
                                                                          const double2* __restrict__ res,
                                                                          double* __restrict__ partials) {
  __shared__ double red[kWarps];
  double rp2[2] = {0.0, 0.0}, rpmax[2] = {0.0, 0.0}, by[2] = {0.0, 0.0};
  auto row_terms = [&](long long i) {
    const double bi = b[i];
    const double2 rr = res[i];
    const double r2[2] = {rr.x, rr.y};
#pragma unroll
    for (int p = 0; p < 2; ++p) {
      const double r = r2[p];
      rp2[p] = fma(r, r, rp2[p]);
      rpmax[p] = nan_max(fabs(r), rpmax[p]);
      by[p] = fma(bi, pts.y[p][i], by[p]);
    }
  };
  if (threadIdx.x == 0)
    for (int h = blockIdx.x; h < rs.n_heavy; h += gridDim.x) row_terms(rs.heavy[h]);
  const int lane = threadIdx.x & 31;
  const long long warps = (long long)gridDim.x * kWarps;
  for (long long sl = ((long long)blockIdx.x * kBlock + threadIdx.x) >> 5; sl < S.nslices; sl += warps) {
    const long long rl = sell_row(S, sl, lane);
    const int len = rl < rs.rows ? rs.ptr[rl + 1] - rs.ptr[rl] : -1;
    if (len >= 0 && len <= rs.heavy_threshold) row_terms(rl);
  }
#pragma unroll
  for (int p = 0; p < 2; ++p) {
    const double t0 = block_sum(rp2[p], red);
    const double t1 = block_max(rpmax[p], red);
    const double t2 = block_sum(by[p], red);
    if (threadIdx.x == 0) {
      double* o = partials + (size_t)blockIdx.x * kMaxQ + p * PDHG_NQ;
      o[PDHG_Q_RP2] = t0;
      o[PDHG_Q_RPMAX] = t1;
      o[PDHG_Q_BY] = t2;
    }
  }
}

// Row relabelling of a CSR matrix (warp per new row): new row r is old row
// perm[r]; new_ptr must already hold the scanned lengths.  Entries keep their
// order inside each row.
__global__ void k_permute_rows(int rows, const int* __restrict__ perm, const int* __restrict__ ptr,
                               const int* __restrict__ col, const double* __restrict__ val,
                               const int* __restrict__ new_ptr, int* __restrict__ new_col,
                               double* __restrict__ new_val) {
  const long long w = ((long long)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  const int lane = threadIdx.x & 31;
  if (w >= rows) return;
  const int o = perm[w];
  const int s = ptr[o], e = ptr[o + 1], d = new_ptr[w];
  for (int k = lane; k < e - s; k += 32) {
    new_col[d + k] = col[s + k];
    new_val[d + k] = val[s + k];
  }
}

// One block per quantity: combine per-block partials in a fixed order.
__global__ void __launch_bounds__(kBlock) k_reduce(const double* __restrict__ partials, int nblk,
                                                   int stride, int nq, double* __restrict__ out) {
  __shared__ double red[kWarps];
  const int q = blockIdx.x;
  const bool is_max = (q % PDHG_NQ) == PDHG_Q_RPMAX || (q % PDHG_NQ) == PDHG_Q_RDMAX;
  double acc = is_max ? -1.0 : 0.0;
  for (int bi = threadIdx.x; bi < nblk; bi += kBlock) {
    const double v = partials[(size_t)bi * stride + q];
    acc = is_max ? nan_max(v, acc) : acc + v;
  }
  const double t = is_max ? block_max(acc, red) : block_sum(acc, red);
  if (threadIdx.x == 0) out[q] = ((q % PDHG_NQ) == PDHG_Q_RSV) ? 0.0 : t;
}

// ------------------------------------------------------------- layout helpers

__global__ void k_row_ids(const int* __restrict__ ptr, int rows, int* __restrict__ rid) {
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= rows) return;
  for (int k = ptr[i]; k < ptr[i + 1]; ++k) rid[k] = i;
}

// split[k-1][i] = first entry of row i with column >= k*chunk (k = 1..K-1);
// flags rows whose columns are not sorted (the split needs sorted rows).
__global__ void k_split(int m, const int* __restrict__ ptr, const int* __restrict__ col, int K,
                        int chunk, int* __restrict__ split, int* __restrict__ unsorted) {
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= m) return;
  const int s = ptr[i], e = ptr[i + 1];
  for (int k = s + 1; k < e; ++k)
    if (col[k] < col[k - 1]) { atomicOr(unsorted, 1); break; }
  for (int k = 1; k < K; ++k) {
    const int target = k * chunk;
    int lo = s, hi = e;
    while (lo < hi) {
      const int mid = (lo + hi) >> 1;
      if (col[mid] < target) lo = mid + 1; else hi = mid;
    }
    split[(size_t)(k - 1) * m + i] = lo;
  }
}

__global__ void k_iota(int* __restrict__ v, long long n) {
  const long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x;
  if (i < n) v[i] = (int)i;
}

__global__ void k_gather_t(const int* __restrict__ perm, const int* __restrict__ rid,
                           const double* __restrict__ val, int* __restrict__ at_col,
                           double* __restrict__ at_val, long long nnz) {
  const long long k = (long long)blockIdx.x * blockDim.x + threadIdx.x;
  if (k >= nnz) return;
  const int p = perm[k];
  at_col[k] = rid[p];
  at_val[k] = val[p];
}

// at_ptr[j] = first position of key >= j in the sorted column keys
__global__ void k_col_ptr(const int* __restrict__ keys, long long nnz, int n, int* __restrict__ at_ptr) {
  const int j = blockIdx.x * blockDim.x + threadIdx.x;
  if (j > n) return;
  long long lo = 0, hi = nnz;
  while (lo < hi) {
    const long long mid = (lo + hi) >> 1;
    if (keys[mid] < j) lo = mid + 1; else hi = mid;
  }
  at_ptr[j] = (int)lo;
}

// ---------------------------------------------------------------- dispatch

template <template <int> class F, class... Args>
int dispatch_lanes(int lanes, Args&&... args) {
  switch (lanes) {
    case 1: return F<1>::run(args...);
    case 2: return F<2>::run(args...);
    case 4: return F<4>::run(args...);
    case 8: return F<8>::run(args...);
    case 16: return F<16>::run(args...);
    case 32: return F<32>::run(args...);
    default: return fail(PDHG_ERR_ARG, "lanes must be 1,2,4,8,16 or 32");
  }
}

int grid_rows(const RowSet& rs, int lanes) {
  (void)lanes;  // a warp owns 32 rows whatever the lane count
  return rs.n_heavy + (int)((rs.rows + (long long)kBlock - 1) / kBlock);
}

// k_step's grid: heavy rows (a block each), medium rows (a warp each), light rows
int grid_step(const RowSet& rs) {
  return rs.n_heavy + (rs.n_medium + kWarps - 1) / kWarps + (int)((rs.rows + (long long)kBlock - 1) / kBlock);
}

template <int V>
struct SpmvLaunch {
  static int run(const RowSet& rs, const double* in, double* out, cudaStream_t s) {
    const int g = grid_rows(rs, V);
    if (g > 0) k_spmv<V><<<g, kBlock, 0, s>>>(rs, in, out);
    return 0;
  }
};

template <int V>
struct CheckLaunch {
  static int run(bool primal, int np, const RowSet& rs, const double* bc, const CheckPts& pts,
                 double* partials, cudaStream_t s) {
    if (primal) {
      if (np == 1) k_check_primal<V, 1><<<kCheckBlocks, kBlock, 0, s>>>(rs, bc, pts, partials);
      else if (pts.pair && V >= 16 && PDHG_CHECK_ROWS)
        k_check_primal_rows<(V >= 16 ? V : 16)><<<kCheckBlocks, kBlock, 0, s>>>(rs, bc, pts, partials);
      else if (pts.pair) k_check_primal<V, 2, true><<<kCheckBlocks, kBlock, 0, s>>>(rs, bc, pts, partials);
      else k_check_primal<V, 2><<<kCheckBlocks, kBlock, 0, s>>>(rs, bc, pts, partials);
    } else {
      if (np == 1) k_check_dual<V, 1><<<kCheckBlocks, kBlock, 0, s>>>(rs, bc, pts, partials);
      else if (pts.pair) k_check_dual<V, 2, true><<<kCheckBlocks, kBlock, 0, s>>>(rs, bc, pts, partials);
      else k_check_dual<V, 2><<<kCheckBlocks, kBlock, 0, s>>>(rs, bc, pts, partials);
    }
    return 0;
  }
};

int auto_lanes(long long nnz, int rows) {
  if (rows <= 0) return 1;
  const double mean = (double)nnz / rows;
  // measured on config 4 (tools/spmv_lab.cu, profiles/r01_spmv_lab2.log):
  // 16 lanes for mean-40 rows (A), 8 for mean 20 (A')
  if (mean >= 80) return 32;
  if (mean >= 32) return 16;
  if (mean >= 12) return 8;
  if (mean >= 6) return 4;
  if (mean >= 3) return 2;
  return 1;
}

size_t align_up(size_t v) { return (v + 255) & ~(size_t)255; }

}  // namespace

// ------------------------------------------------------------------ context

struct pdhg_ctx {
  pdhg_problem prob;
  int device;          // the CUDA device of `stream`; every ABI entry runs on it (DevGuard)
  RowSet A, At;
  int a_lanes, at_lanes;
  cudaStream_t stream;
  // workspace carve
  double *x, *xe, *xbar, *xbest, *zbest, *tn1, *tn2;
  double *y, *ybar, *ybest, *tm1, *tm2;
  double2 *px, *py;  // interleaved gather vectors of a two-point check
  double* partials;
  double* scalars;
  StepParams* P;
  // pinned host staging
  StepParams* P_host;
  double* scal_host;
  std::map<int, cudaGraphExec_t> graphs;
  int mf, nf;          // full (padded) lengths of the y- and x-space vectors
  int yo, xo;          // this shard's slice offsets in them
  bool has_psr[2];     // [0] = A (dual), [1] = A' (primal)
  bool has_sell[2];    // same indexing
  SellSet sell[2];
  bool has_sellp[2];   // split steps over sliced-ELL parts (pdhg_problem a_sell_part / at_sell_part)
  SellSet sellp[2][2];
  const int* pptr[2][2];
#if PDHG_EXPERIMENTAL
  psr::Layout psr_l[2];
  size_t psr_smem[2];
#endif
  int l2_persist, l2_maxwin;
  int l2_mask;         // bit0: window on y for the primal step, bit1: on xe for the dual step
  int coop_grid;       // > 0: periods run as one cooperative k_period launch of this many blocks
  bool tiny;           // periods run as one single-block k_period_tiny launch
  bool period_direct;  // periods launched kernel by kernel instead of as a graph
  double* const* peers[2];  // fused all-gather targets: [0] xe (primal), [1] y (dual)
  int npeers[2];
  // check -> next primal step reuse (pdhg_check_dot_enable / pdhg_use_check_dot):
  // a two-point check leaves A'y of both points interleaved in px (free once the
  // check's A side has run; rebuilt by the next check's k_pair)
  bool check_dot = false;  // enabled for this context
  bool dots_ready = false; // px holds the last two-point check's A'y pairs
  int first_dot = -1;      // armed: the next period's first primal step uses px[.].{x,y}
  // check fused into the last iteration of a period (pdhg_check_fuse_enable):
  // pq = (xe, x, avg_x) quads written by that iteration's primal step, pr = the
  // residual pairs its dual step leaves for k_check_primal_fold
  void* pq = nullptr;
  double2* pr = nullptr;
  bool check_fuse = false;  // enabled for this context
  bool fuse_next = false;   // the next launch_period fuses its last iteration
  bool fuse_ready = false;  // pr holds the residuals of the current (x, y) and average
};

namespace {

struct Carve {
  char* base;
  size_t off = 0;
  template <class T>
  T* take(size_t count) {
    T* p = reinterpret_cast<T*>(base + off);
    off += align_up(count * sizeof(T) + 256);  // +256: bulk copies round up to 16 B
    return p;
  }
};

size_t carve_bytes(int32_t m, int32_t n) {
  size_t b = 0;
  b += 7 * align_up((size_t)n * 8 + 256);
  b += 5 * align_up((size_t)m * 8 + 256);
  b += align_up((size_t)kCheckBlocks * kMaxQ * 8 + 256);
  b += align_up(64 * 8 + 256);
  b += align_up(sizeof(StepParams) + 256);
  b += align_up((size_t)n * 16 + 256) + align_up((size_t)m * 16 + 256);  // px, py
  b += align_up((size_t)n * 32 + 256) + align_up((size_t)m * 16 + 256);  // pq, pr
  return b;
}

cudaAccessPolicyWindow l2_window(const pdhg_ctx* c, const void* base, size_t bytes) {
  cudaAccessPolicyWindow w{};
  if (c->l2_persist <= 0 || c->l2_maxwin <= 0) return w;
  w.base_ptr = const_cast<void*>(base);
  w.num_bytes = std::min(bytes, (size_t)c->l2_maxwin);
  w.hitRatio = (float)std::min(1.0, (double)c->l2_persist / (double)w.num_bytes);
  w.hitProp = cudaAccessPropertyPersisting;
  w.missProp = cudaAccessPropertyStreaming;
  return w;
}

template <class K, class... Args>
int launch_ex(const pdhg_ctx* c, K kernel, dim3 grid, dim3 block, size_t smem, const void* win_base,
              size_t win_bytes, Args... args) {
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = grid;
  cfg.blockDim = block;
  cfg.dynamicSmemBytes = smem;
  cfg.stream = c->stream;
  cudaLaunchAttribute attr[2];
  cfg.attrs = attr;
  cfg.numAttrs = 0;
  if (win_base && c->l2_persist > 0) {
    attr[cfg.numAttrs].id = cudaLaunchAttributeAccessPolicyWindow;
    attr[cfg.numAttrs].val.accessPolicyWindow = l2_window(c, win_base, win_bytes);
    ++cfg.numAttrs;
  }
  if (PDHG_PDL) {  // every kernel launched here starts with pdl_enter()
    attr[cfg.numAttrs].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    attr[cfg.numAttrs].val.programmaticStreamSerializationAllowed = 1;
    ++cfg.numAttrs;
  }
  CUDA_TRY(cudaLaunchKernelEx(&cfg, kernel, args...));
  return 0;
}

template <int V>
struct SplitLaunch {
  // passes [p0, p1) of a split step
  static int run(const pdhg_ctx* c, bool primal, const StepArgs& a, int j, int p0, int p1) {
    for (int pass = p0; pass < p1; ++pass) {
      const int nh = pass == a.nsplit - 1 ? a.rs.n_heavy : 0;
      const int g = nh + (int)((a.rs.rows + (long long)kBlock - 1) / kBlock);
      int rc = primal ? launch_ex(c, k_step_split<V, true>, dim3(g), dim3(kBlock), 0, nullptr, 0, a, j, pass, nh)
                      : launch_ex(c, k_step_split<V, false>, dim3(g), dim3(kBlock), 0, nullptr, 0, a, j, pass, nh);
      if (rc) return rc;
    }
    return 0;
  }
};

template <int V>
struct StepLaunchEx {
  static int run(const pdhg_ctx* c, bool primal, const StepArgs& a, int j, int grid,
                 const void* win_base, size_t win) {
    if (grid == 0) return 0;
    if (c->npeers[primal ? 0 : 1] > 0) {
      if (primal) return launch_ex(c, k_step<V, true, true>, dim3(grid), dim3(kBlock), 0, win_base, win, a, j);
      return launch_ex(c, k_step<V, false, true>, dim3(grid), dim3(kBlock), 0, win_base, win, a, j);
    }
    if (primal) return launch_ex(c, k_step<V, true>, dim3(grid), dim3(kBlock), 0, win_base, win, a, j);
    return launch_ex(c, k_step<V, false>, dim3(grid), dim3(kBlock), 0, win_base, win, a, j);
  }
};

StepArgs step_args(const pdhg_ctx* c, bool primal) {
  StepArgs a;
  if (primal) {
    a.rs = c->At; a.gather = c->y; a.cb = c->prob.c;
    a.x = c->x + c->xo; a.xe = c->xe + c->xo; a.xbar = c->xbar + c->xo;
  } else {
    a.rs = c->A; a.gather = c->xe; a.cb = c->prob.b;
    a.x = c->y + c->yo; a.xe = nullptr; a.xbar = c->ybar + c->yo;
  }
  a.P = c->P;
  a.split = nullptr;
  a.nsplit = 1;
  a.partial = nullptr;
  return a;
}

int launch_period_persistent(pdhg_ctx* c, int iters);
int launch_step(pdhg_ctx* c, bool primal, int j);

// The iterations of one period: a cooperative / single-block kernel, direct
// stream launches (period_direct), or a CUDA graph captured once per length.
// First primal step of a period from the last check's A'y (slot 0 / 1).
int launch_primal_from_dot(pdhg_ctx* c, int slot, int j) {
  const StepArgs a = step_args(c, true);
  const int grid = (int)(((long long)a.rs.rows + kBlock - 1) / kBlock);
  return launch_ex(c, k_primal_from_dot, dim3(grid), dim3(kBlock), 0, nullptr, 0, a,
                   (const double2*)(c->px + c->xo), slot, j);
}

// The half steps of the last iteration of a check-fused period (sliced ELL
// of A and A', one GPU): the primal step writes the (xe, x, avg_x) quads, the
// dual step gathers them and leaves the check's residual pairs in pr.
int launch_step_fused(pdhg_ctx* c, bool primal, int j) {
  StepArgs a = step_args(c, primal);
  const SellSet& S = c->sell[primal ? 1 : 0];
  const int grid = a.rs.n_heavy + (int)(((long long)S.nslices * 32 + kBlock - 1) / kBlock);
  if (grid == 0) return 0;
  if (primal) {
    a.xe = reinterpret_cast<double*>(c->pq);
    return S.u_long ? launch_ex(c, k_step_sell<true, PDHG_SELL_U_LONG, true>, dim3(grid), dim3(kBlock), 0, nullptr,
                                0, a, S, j)
                    : launch_ex(c, k_step_sell<true, PDHG_SELL_U, true>, dim3(grid), dim3(kBlock), 0, nullptr, 0,
                                a, S, j);
  }
  a.gather = reinterpret_cast<const double*>(c->pq);
  a.partial = reinterpret_cast<double*>(c->pr);
  return launch_ex(c, k_step_sell_chk<PDHG_FUSE_U>, dim3(grid), dim3(kBlock), 0, nullptr, 0, a, S, j);
}

int launch_period(pdhg_ctx* c, int iters) {
  // an armed check-dot slot is consumed by this period (or dropped)
  const int first = c->first_dot;
  c->first_dot = -1;
  c->dots_ready = false;
  // a check-fused period needs a last iteration other than the first
  const bool fuse = c->fuse_next && iters >= 2 && c->coop_grid == 0;
  c->fuse_next = false;
  c->fuse_ready = false;
  if (iters <= 0) return 0;
  if (c->coop_grid > 0) return launch_period_persistent(c, iters);
  int rc = 0;
  auto half = [&](bool primal, int j) {
    if (fuse && j == iters - 1) return launch_step_fused(c, primal, j);
    if (primal && j == 0 && first >= 0) return launch_primal_from_dot(c, first, 0);
    return launch_step(c, primal, j);
  };
  if (c->period_direct) {
    for (int j = 0; j < iters && !rc; ++j) {
      rc = half(true, j);
      if (!rc) rc = half(false, j);
    }
    if (!rc) c->fuse_ready = fuse;
    return rc;
  }
  // graphs per (length, first step, fused check)
  const int key = iters + (first + 1) * (1 << 28) + (fuse ? (1 << 30) : 0);
  auto it = c->graphs.find(key);
  if (it == c->graphs.end()) {
    cudaGraph_t g;
    CUDA_TRY(cudaStreamBeginCapture(c->stream, cudaStreamCaptureModeThreadLocal));
    for (int j = 0; j < iters && !rc; ++j) {
      rc = half(true, j);
      if (!rc) rc = half(false, j);
    }
    cudaError_t ce = cudaStreamEndCapture(c->stream, &g);
    if (rc) return rc;
    if (ce != cudaSuccess) return fail(PDHG_ERR_CUDA, std::string("capture: ") + cudaGetErrorString(ce));
    cudaGraphExec_t ex;
    CUDA_TRY(cudaGraphInstantiate(&ex, g, 0));
    cudaGraphDestroy(g);
    it = c->graphs.emplace(key, ex).first;
  }
  CUDA_TRY(cudaGraphLaunch(it->second, c->stream));
  c->fuse_ready = fuse;
  return 0;
}

int launch_period_persistent(pdhg_ctx* c, int iters) {
#if !PDHG_EXPERIMENTAL
  (void)iters;
  return fail(PDHG_ERR_STATE, "persistent period kernels need the experiment build (PDHG_EXPERIMENTAL)");
#else
  StepArgs pa = step_args(c, true), da = step_args(c, false);
  int va = c->at_lanes, vd = c->a_lanes;
  if (c->tiny) {
    k_period_tiny<<<1, kTinyBlock, 0, c->stream>>>(pa, da, va, vd, iters);
    CUDA_TRY(cudaGetLastError());
    return 0;
  }
  void* args[] = {&pa, &da, &va, &vd, &iters};
  CUDA_TRY(cudaLaunchCooperativeKernel((const void*)k_period, dim3(c->coop_grid), dim3(kBlock), args, 0,
                                       c->stream));
  return 0;
#endif
}

int launch_step_pass(pdhg_ctx* c, bool primal, int j, int pass);

int launch_step(pdhg_ctx* c, bool primal, int j) { return launch_step_pass(c, primal, j, -1); }

// One half step, or one pass of a split half step (pass < 0: all passes; an
// unsplit operator runs whole at pass 0 and nothing at later passes).
int launch_step_pass(pdhg_ctx* c, bool primal, int j, int pass) {
  // gathers read the full (padded) vectors; the rows a shard owns are
  // written through pointers offset to its slice
  StepArgs a = step_args(c, primal);
  const int nsplit = primal ? c->prob.at_nsplit : c->prob.a_nsplit;
  if (nsplit > 1 && c->has_sellp[primal ? 1 : 0]) {  // sliced-ELL parts, 2 passes
    const int k = primal ? 1 : 0;
    a.partial = primal ? c->tn2 : c->tm2;
    const int p0 = pass < 0 ? 0 : pass, p1 = pass < 0 ? 2 : std::min(pass + 1, 2);
    for (int h = p0; h < p1; ++h) {
      const SellSet& S = c->sellp[k][h];
      const int nh = h == 1 ? a.rs.n_heavy : 0;
      const int grid = nh + (int)(((long long)S.nslices * 32 + kBlock - 1) / kBlock);
      if (grid == 0) continue;
      // entries in flight as the unsplit sliced-ELL steps (long rows: 6 primal, 10 dual)
      const int* pp = c->pptr[k][h];
      int rc;
      if (S.u_long) {
        if (h == 0)
          rc = primal ? launch_ex(c, k_step_sell_pass<true, PDHG_SELL_U_LONG, 0>, dim3(grid), dim3(kBlock), 0,
                                  nullptr, 0, a, S, pp, j)
                      : launch_ex(c, k_step_sell_pass<false, PDHG_SELL_U_DUAL, 0>, dim3(grid), dim3(kBlock), 0,
                                  nullptr, 0, a, S, pp, j);
        else
          rc = primal ? launch_ex(c, k_step_sell_pass<true, PDHG_SELL_U_LONG, 1>, dim3(grid), dim3(kBlock), 0,
                                  nullptr, 0, a, S, pp, j)
                      : launch_ex(c, k_step_sell_pass<false, PDHG_SELL_U_DUAL, 1>, dim3(grid), dim3(kBlock), 0,
                                  nullptr, 0, a, S, pp, j);
      } else {
        if (h == 0)
          rc = primal ? launch_ex(c, k_step_sell_pass<true, PDHG_SELL_U, 0>, dim3(grid), dim3(kBlock), 0, nullptr,
                                  0, a, S, pp, j)
                      : launch_ex(c, k_step_sell_pass<false, PDHG_SELL_U, 0>, dim3(grid), dim3(kBlock), 0, nullptr,
                                  0, a, S, pp, j);
        else
          rc = primal ? launch_ex(c, k_step_sell_pass<true, PDHG_SELL_U, 1>, dim3(grid), dim3(kBlock), 0, nullptr,
                                  0, a, S, pp, j)
                      : launch_ex(c, k_step_sell_pass<false, PDHG_SELL_U, 1>, dim3(grid), dim3(kBlock), 0, nullptr,
                                  0, a, S, pp, j);
      }
      if (rc) return rc;
    }
    return 0;
  }
  if (nsplit > 1 && !c->has_psr[primal ? 1 : 0]) {
    a.split = primal ? c->prob.at_split : c->prob.a_split;
    a.nsplit = nsplit;
    a.partial = primal ? c->tn2 : c->tm2;
    const int p0 = pass < 0 ? 0 : pass, p1 = pass < 0 ? nsplit : std::min(pass + 1, nsplit);
    return dispatch_lanes<SplitLaunch>(primal ? c->at_lanes : c->a_lanes, c, primal, a, j, p0, p1);
  }
  if (pass > 0) return 0;
  const size_t win = (size_t)(primal ? c->mf : c->nf) * 8;
  const void* win_base = (c->l2_mask & (primal ? 1 : 2)) ? a.gather : nullptr;
  const int lanes = primal ? c->at_lanes : c->a_lanes;
  const int k = primal ? 1 : 0;
#if PDHG_EXPERIMENTAL
  if (c->has_psr[k]) {
    PsrStepArgs pa{c->psr_l[k], a.gather, a.cb, a.x, a.xe, a.xbar, a.P};
    const int grid = std::min(c->psr_l[k].nblk, 148);
    int rc = primal ? launch_ex(c, k_step_psr<true>, dim3(grid), dim3(psr::kThreads), c->psr_smem[k],
                                win_base, win, pa, j)
                    : launch_ex(c, k_step_psr<false>, dim3(grid), dim3(psr::kThreads), c->psr_smem[k],
                                win_base, win, pa, j);
    if (rc) return rc;
    // heavy rows: block per row through the CSR kernel (grid = n_heavy => no light rows)
    return dispatch_lanes<StepLaunchEx>(lanes, c, primal, a, j, a.rs.n_heavy, win_base, win);
  }
#endif
  if (c->has_sell[k]) {
    const SellSet& S = c->sell[k];
    const int grid = a.rs.n_heavy + (int)(((long long)S.nslices * 32 + kBlock - 1) / kBlock);
    if (S.u_long)
      return primal ? launch_ex(c, k_step_sell<true, PDHG_SELL_U_LONG>, dim3(grid), dim3(kBlock), 0, win_base, win, a, S, j)
                    : launch_ex(c, k_step_sell<false, PDHG_SELL_U_DUAL>, dim3(grid), dim3(kBlock), 0, win_base, win, a, S, j);
    return primal ? launch_ex(c, k_step_sell<true, PDHG_SELL_U>, dim3(grid), dim3(kBlock), 0, win_base, win, a, S, j)
                  : launch_ex(c, k_step_sell<false, PDHG_SELL_U>, dim3(grid), dim3(kBlock), 0, win_base, win, a, S, j);
  }
  return dispatch_lanes<StepLaunchEx>(lanes, c, primal, a, j, grid_step(a.rs), win_base, win);
}

int spmv(pdhg_ctx* c, bool transpose, const double* in, double* out) {
  const int k = transpose ? 1 : 0;
  if (c->has_sell[k]) {
    const RowSet& rs = transpose ? c->At : c->A;
    const SellSet& S = c->sell[k];
    const int grid = rs.n_heavy + (int)(((long long)S.nslices * 32 + kBlock - 1) / kBlock);
    if (grid > 0) {
      if (S.u_long) k_spmv_sell<PDHG_SELL_U_LONG><<<grid, kBlock, 0, c->stream>>>(rs, S, in, out);
      else k_spmv_sell<PDHG_SELL_U><<<grid, kBlock, 0, c->stream>>>(rs, S, in, out);
    }
    CUDA_TRY(cudaGetLastError());
    return 0;
  }
  return dispatch_lanes<SpmvLaunch>(transpose ? c->at_lanes : c->a_lanes, transpose ? c->At : c->A,
                                    in, out, c->stream);
}

void point_xy(pdhg_ctx* c, int which, const double** x, const double** y) {
  switch (which & 3) {
    case PDHG_PT_AVG: *x = c->xbar; *y = c->ybar; break;
    case PDHG_PT_BEST: *x = c->xbest; *y = c->ybest; break;
    default: *x = c->x; *y = c->y; break;
  }
}

// reduce sum of squares of v (length len) into host scalar (syncs)
int sumsq_host(pdhg_ctx* c, const double* v, int len, double* out) {
  k_sumsq<<<kCheckBlocks, kBlock, 0, c->stream>>>(v, len, c->partials);
  k_reduce<<<1, kBlock, 0, c->stream>>>(c->partials, kCheckBlocks, 1, 1, c->scalars);
  CUDA_TRY(cudaGetLastError());
  CUDA_TRY(cudaMemcpyAsync(c->scal_host, c->scalars, sizeof(double), cudaMemcpyDeviceToHost, c->stream));
  CUDA_TRY(cudaStreamSynchronize(c->stream));
  *out = c->scal_host[0];
  return 0;
}

}  // namespace

namespace {
// Every ABI entry that takes a context runs on the context's device, whatever
// device is current in the calling thread (restored on return).
struct DevGuard {
  int prev = -1;
  explicit DevGuard(int dev) {
    int cur = -1;
    if (dev >= 0 && cudaGetDevice(&cur) == cudaSuccess && cur != dev && cudaSetDevice(dev) == cudaSuccess)
      prev = cur;
  }
  ~DevGuard() {
    if (prev >= 0) cudaSetDevice(prev);
  }
};
}  // namespace
#define CTX_DEVICE_GUARD(c) DevGuard dev_guard_((c) ? (c)->device : -1)

namespace {
// NVTX range over one ABI call (period, check, power iteration): the host-side
// timeline of a run in Nsight Systems (header-only NVTX v3; no-op without a tool).
struct NvtxRange {
  explicit NvtxRange(const char* name) { nvtxRangePushA(name); }
  ~NvtxRange() { nvtxRangePop(); }
};
}  // namespace

extern "C" {

int pdhg_abi_version(void) { return PDHG_ABI_VERSION; }

const char* pdhg_last_error(void) { return g_err.c_str(); }

size_t pdhg_workspace_bytes(int32_t m, int32_t n) { return carve_bytes(m, n); }

int pdhg_ctx_create(const pdhg_problem* prob, void* workspace, size_t workspace_bytes, void* stream,
                    pdhg_ctx** out) {
  if (!prob || !out) return fail(PDHG_ERR_ARG, "null argument");
  if (prob->m <= 0 || prob->n <= 0) return fail(PDHG_ERR_ARG, "empty model");
  const int mf = prob->m_full > 0 ? prob->m_full : prob->m;
  const int nf = prob->n_full > 0 ? prob->n_full : prob->n;
  if (prob->y_off < 0 || prob->x_off < 0 || prob->y_off + prob->m > mf || prob->x_off + prob->n > nf)
    return fail(PDHG_ERR_ARG, "shard slice outside the full vectors");
  if (workspace_bytes < carve_bytes(mf, nf))
    return fail(PDHG_ERR_ARG, "workspace too small");
  int dev = 0;
  if (cudaGetDevice(&dev) != cudaSuccess) return fail(PDHG_ERR_CUDA, "cudaGetDevice failed");
  if (stream && cudaStreamGetDevice((cudaStream_t)stream, &dev) != cudaSuccess)
    return fail(PDHG_ERR_CUDA, "cudaStreamGetDevice failed");
  DevGuard guard(dev);  // ctx_create reads device attributes and sets kernel attributes on it
  pdhg_ctx* c = new pdhg_ctx();
  c->device = dev;
  c->prob = *prob;
  c->stream = (cudaStream_t)stream;
  c->A = RowSet{prob->a_ptr, prob->a_col, prob->a_val, prob->m, prob->heavy_threshold,
                prob->a_n_heavy, prob->a_heavy};
  c->At = RowSet{prob->at_ptr, prob->at_col, prob->at_val, prob->n,
                 prob->at_heavy_threshold > 0 ? prob->at_heavy_threshold : prob->heavy_threshold,
                 prob->at_n_heavy, prob->at_heavy};
  c->A.ncols = prob->n_full > 0 ? prob->n_full : prob->n;   // gathers xe (x-space)
  c->A.nnz = prob->nnz;
  c->At.ncols = prob->m_full > 0 ? prob->m_full : prob->m;  // gathers y (y-space)
  c->At.nnz = prob->at_nnz > 0 ? prob->at_nnz : prob->nnz;
  for (int k = 0; k < 2; ++k) {  // medium rows (k_step only; not with a PSR layout)
    RowSet& rs = k == 0 ? c->A : c->At;
    const int nmed = k == 0 ? prob->a_n_medium : prob->at_n_medium;
    const int* med = k == 0 ? prob->a_medium : prob->at_medium;
    const int lmax = k == 0 ? prob->a_light_max : prob->at_light_max;
    const bool psr = (k == 0 ? prob->a_psr : prob->at_psr) != nullptr;
    if (nmed < 0 || (nmed > 0 && (!med || lmax <= 0))) return fail(PDHG_ERR_ARG, "bad medium-row list");
    if (nmed > 0 && !psr) {
      rs.n_medium = nmed;
      rs.medium = med;
      rs.light_max = lmax;
    }
  }
  c->a_lanes = prob->a_lanes > 0 ? prob->a_lanes : auto_lanes(prob->nnz, prob->m);
  c->at_lanes = prob->at_lanes > 0 ? prob->at_lanes
                                    : auto_lanes(prob->at_nnz > 0 ? prob->at_nnz : prob->nnz, prob->n);
  Carve cv{(char*)workspace};
  c->mf = mf; c->nf = nf; c->yo = prob->y_off; c->xo = prob->x_off;
  const int n = nf, m = mf;
  c->x = cv.take<double>(n); c->xe = cv.take<double>(n); c->xbar = cv.take<double>(n);
  c->xbest = cv.take<double>(n); c->zbest = cv.take<double>(n);
  c->tn1 = cv.take<double>(n); c->tn2 = cv.take<double>(n);
  c->y = cv.take<double>(m); c->ybar = cv.take<double>(m); c->ybest = cv.take<double>(m);
  c->tm1 = cv.take<double>(m);
  c->tm2 = cv.take<double>(m);
  c->partials = cv.take<double>((size_t)kCheckBlocks * kMaxQ);
  c->scalars = cv.take<double>(64);
  c->P = cv.take<StepParams>(1);
  c->px = cv.take<double2>(n);
  c->py = cv.take<double2>(m);
  c->pq = cv.take<Quad>(n);
  c->pr = cv.take<double2>(m);
  if ((prob->a_nsplit > 1 && !prob->a_split) || (prob->at_nsplit > 1 && !prob->at_split)) {
    delete c;
    return fail(PDHG_ERR_ARG, "split step without split points");
  }
  c->coop_grid = 0;
  c->tiny = false;
  c->period_direct = prob->persistent == 3;
  c->has_psr[0] = c->has_psr[1] = false;
  c->l2_mask = c->l2_persist = c->l2_maxwin = 0;
#if !PDHG_EXPERIMENTAL
  if (prob->persistent == 1 || prob->persistent == 2 || prob->a_psr || prob->at_psr || (prob->l2_persist & 3)) {
    delete c;
    return fail(PDHG_ERR_ARG, "PSR layouts, persistent periods and L2 windows need the experiment build "
                              "(PDHG_EXPERIMENTAL)");
  }
#else
  if (prob->persistent == 2 && !prob->a_sell && !prob->at_sell && !prob->a_psr && !prob->at_psr &&
      prob->a_nsplit <= 1 && mf == prob->m && nf == prob->n) {
    c->tiny = true;
    c->coop_grid = 1;
  } else if (prob->persistent == 1 && !prob->a_sell && !prob->at_sell && !prob->a_psr && !prob->at_psr &&
      prob->a_nsplit <= 1 && mf == prob->m && nf == prob->n) {
    int dev = 0, nsm = 0, per_sm = 0, coop = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, dev);
    cudaDeviceGetAttribute(&coop, cudaDevAttrCooperativeLaunch, dev);
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, k_period, kBlock, 0);
    cudaGetLastError();
    if (coop && per_sm > 0) c->coop_grid = nsm * per_sm;
  }
#endif
  for (int k = 0; k < 2; ++k) {
    const pdhg_sell* q = k == 0 ? prob->a_sell : prob->at_sell;
    c->has_sell[k] = q != nullptr;
    if (q) {
      const int rows = k == 0 ? prob->m : prob->n;
      if (q->rows != rows || q->nslices != (rows + 31) / 32 || !q->sptr || !q->width) {
        delete c;
        return fail(PDHG_ERR_ARG, "sell layout does not match the operator");
      }
      c->sell[k] = SellSet{q->rows, q->nslices, reinterpret_cast<const long long*>(q->sptr), q->width,
                           q->col, q->val, q->perm};
      const long long ops_nnz = k == 0 ? prob->nnz : (prob->at_nnz > 0 ? prob->at_nnz : prob->nnz);
      c->sell[k].u_long = q->rows > 0 && ops_nnz >= (long long)PDHG_SELL_U_MEAN * q->rows;
      c->sell[k].ncols = k == 0 ? c->A.ncols : c->At.ncols;
      c->sell[k].nslots = q->nslots > 0 ? q->nslots : 0x7fffffffffffffffLL;
    }
  }
  for (int k = 0; k < 2; ++k) {  // split steps' sliced-ELL parts
    const pdhg_sell* const* qs = k == 0 ? prob->a_sell_part : prob->at_sell_part;
    const int32_t* const* pp = k == 0 ? prob->a_part_ptr : prob->at_part_ptr;
    const int nsplit = k == 0 ? prob->a_nsplit : prob->at_nsplit;
    c->has_sellp[k] = qs[0] != nullptr || qs[1] != nullptr;
    if (!c->has_sellp[k]) continue;
    const int rows = k == 0 ? prob->m : prob->n;
    for (int h = 0; h < 2; ++h) {
      const pdhg_sell* q = qs[h];
      if (nsplit != 2 || !q || !pp[h] || q->rows != rows || q->nslices != (rows + 31) / 32 || !q->sptr ||
          !q->width) {
        delete c;
        return fail(PDHG_ERR_ARG, "split-step sell parts need 2 passes and match the operator");
      }
      c->sellp[k][h] = SellSet{q->rows, q->nslices, reinterpret_cast<const long long*>(q->sptr), q->width,
                               q->col, q->val, q->perm};
      const long long ops_nnz = k == 0 ? prob->nnz : (prob->at_nnz > 0 ? prob->at_nnz : prob->nnz);
      c->sellp[k][h].u_long = rows > 0 && ops_nnz >= (long long)PDHG_SELL_U_MEAN * rows;  // as sell[k]
      c->sellp[k][h].ncols = k == 0 ? c->A.ncols : c->At.ncols;
      c->sellp[k][h].nslots = q->nslots > 0 ? q->nslots : 0x7fffffffffffffffLL;
      c->pptr[k][h] = pp[h];
    }
  }
#if PDHG_EXPERIMENTAL
  for (int k = 0; k < 2; ++k) {
    const pdhg_psr* q = k == 0 ? prob->a_psr : prob->at_psr;
    c->has_psr[k] = q != nullptr;
    if (q) {
      if (q->R > psr::kMaxRows || q->W != psr::kPanel || !q->heavy || q->ngroups != (q->R + psr::kGroupRows - 1) / psr::kGroupRows) {
        delete c;
        return fail(PDHG_ERR_ARG, "psr layout geometry not supported");
      }
      c->psr_l[k] = psr::Layout{q->rows, q->cols, q->R, q->W, q->nblk, q->ntiles, q->ngroups,
                                q->blk_tile_ptr, q->tile_bin, q->gstart, q->rcnt, q->val, q->col16,
                                q->col, q->heavy};
      c->psr_smem[k] = psr::smem_bytes(q->W);
    }
  }
  {
    int dev = 0;
    cudaGetDevice(&dev);
    int maxp = 0, maxw = 0;
    cudaDeviceGetAttribute(&maxp, cudaDevAttrMaxPersistingL2CacheSize, dev);
    cudaDeviceGetAttribute(&maxw, cudaDevAttrMaxAccessPolicyWindowSize, dev);
    c->l2_mask = prob->l2_persist & 3;
    c->l2_persist = c->l2_mask ? maxp : 0;
    c->l2_maxwin = maxw;
    if (c->l2_persist > 0) cudaDeviceSetLimit(cudaLimitPersistingL2CacheSize, (size_t)maxp);
    cudaGetLastError();
    const size_t sm = psr::smem_bytes(psr::kPanel);
    cudaFuncSetAttribute(k_step_psr<true>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm);
    cudaFuncSetAttribute(k_step_psr<false>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm);
    cudaGetLastError();
  }
#endif
  cudaError_t e1 = cudaMallocHost(&c->P_host, sizeof(StepParams));
  cudaError_t e2 = cudaMallocHost(&c->scal_host, 64 * sizeof(double));
  if (e1 != cudaSuccess || e2 != cudaSuccess) {
    delete c;
    return fail(PDHG_ERR_CUDA, "cudaMallocHost failed");
  }
  std::memset(c->P_host, 0, sizeof(StepParams));  // no peers until pdhg_set_peers
  c->P_host->fail_iter = LLONG_MAX;
  *out = c;
  return 0;
}

int pdhg_ctx_destroy(pdhg_ctx* c) {
  if (!c) return 0;
  CTX_DEVICE_GUARD(c);
  for (auto& kv : c->graphs) cudaGraphExecDestroy(kv.second);
  cudaFreeHost(c->P_host);
  cudaFreeHost(c->scal_host);
  delete c;
  return 0;
}

int pdhg_spmv(pdhg_ctx* c, int transpose, const double* in, double* out) {
  CTX_DEVICE_GUARD(c);
  if (!c || !in || !out) return fail(PDHG_ERR_ARG, "null argument");
  int rc = spmv(c, transpose != 0, in, out);
  if (rc) return rc;
  CUDA_TRY(cudaGetLastError());
  return 0;
}

int pdhg_opnorm(pdhg_ctx* c, const double* v0_host, double tol, int32_t max_iters, double* lam_out,
                int32_t* iters_out) {
  CTX_DEVICE_GUARD(c);
  if (c) { c->first_dot = -1; c->dots_ready = false; }  // state changes: no check dots
  NvtxRange nvtx_range_("pdhg_opnorm");
  // pdhg.py:80-109.  v (tn1) <- v0; loop: w (tn2) = A'(A v); ||w||; v = w/||w||.
  if (!c || !v0_host || !lam_out) return fail(PDHG_ERR_ARG, "null argument");
  if (c->mf != c->prob.m || c->nf != c->prob.n)
    return fail(PDHG_ERR_STATE, "pdhg_opnorm is single-shard; sharded hosts drive the power iteration");
  const int n = c->prob.n;
  // host or device pointer (UVA): the engine hands a device copy already in
  // the context's (renumbered) column order
  CUDA_TRY(cudaMemcpyAsync(c->tn1, v0_host, (size_t)n * 8, cudaMemcpyDefault, c->stream));
  double lam = 0.0;
  int it = 0;
  int rc;
  for (; it < max_iters; ++it) {
    if ((rc = spmv(c, false, c->tn1, c->tm1))) return rc;
    if ((rc = spmv(c, true, c->tm1, c->tn2))) return rc;
    double ss;
    if ((rc = sumsq_host(c, c->tn2, n, &ss))) return rc;
    const double norm_w = std::sqrt(ss);
    if (norm_w == 0.0) break;
    const double new_lam = std::sqrt(norm_w);
    k_div<<<(n + kBlock - 1) / kBlock, kBlock, 0, c->stream>>>(c->tn2, c->tn1, norm_w, n);
    if (lam > 0 && std::fabs(new_lam - lam) <= tol * new_lam) {
      lam = new_lam;
      ++it;
      break;
    }
    lam = new_lam;
  }
  // safeguard multiply (pdhg.py:104-108)
  if ((rc = spmv(c, false, c->tn1, c->tm1))) return rc;
  if ((rc = spmv(c, true, c->tm1, c->tn2))) return rc;
  double ss;
  if ((rc = sumsq_host(c, c->tn2, n, &ss))) return rc;
  const double norm_w = std::sqrt(ss);
  if (norm_w > 0) lam = std::max(lam, std::sqrt(norm_w));
  *lam_out = lam;
  if (iters_out) *iters_out = it;
  return 0;
}

int pdhg_reset(pdhg_ctx* c) {
  CTX_DEVICE_GUARD(c);
  if (!c) return fail(PDHG_ERR_ARG, "null ctx");
  const size_t nb = (size_t)c->nf * 8, mb = (size_t)c->mf * 8;
  c->first_dot = -1;
  c->dots_ready = false;
  c->fuse_ready = false;
  CUDA_TRY(cudaMemsetAsync(c->x, 0, nb, c->stream));
  CUDA_TRY(cudaMemsetAsync(c->xe, 0, nb, c->stream));
  CUDA_TRY(cudaMemsetAsync(c->xbar, 0, nb, c->stream));
  CUDA_TRY(cudaMemsetAsync(c->y, 0, mb, c->stream));
  CUDA_TRY(cudaMemsetAsync(c->ybar, 0, mb, c->stream));
  return 0;
}

int pdhg_run_period(pdhg_ctx* c, int32_t iters, int64_t iter0, double tau_over_omega,
                    double sigma_omega, double w0, int64_t* fail_iter_out) {
  CTX_DEVICE_GUARD(c);
  NvtxRange nvtx_range_("pdhg_period");
  if (!c || iters < 0) return fail(PDHG_ERR_ARG, "bad argument");
  StepParams& h = *c->P_host;
  h.tau_w = tau_over_omega;
  h.sigma_w = sigma_omega;
  h.w0 = w0;
  h.iter0 = iter0;
  h.fail_iter = LLONG_MAX;
  CUDA_TRY(cudaMemcpyAsync(c->P, c->P_host, sizeof(StepParams), cudaMemcpyHostToDevice, c->stream));
  {
    int rc = launch_period(c, iters);
    if (rc) return rc;
  }
  CUDA_TRY(cudaMemcpyAsync(&c->P_host->fail_iter, &c->P->fail_iter, sizeof(long long),
                           cudaMemcpyDeviceToHost, c->stream));
  CUDA_TRY(cudaStreamSynchronize(c->stream));
  if (fail_iter_out) *fail_iter_out = (c->P_host->fail_iter == LLONG_MAX) ? -1 : c->P_host->fail_iter;
  return 0;
}

int pdhg_check_device(pdhg_ctx* c, int32_t npts, const int32_t* specs);

int pdhg_run_period_check(pdhg_ctx* c, int32_t iters, int64_t iter0, double tau_over_omega,
                          double sigma_omega, double w0, int32_t npts, const int32_t* specs,
                          int64_t* fail_iter_out, double* out_host) {
  CTX_DEVICE_GUARD(c);
  NvtxRange nvtx_range_("pdhg_period_check");
  // run_period + check with one host synchronisation: the graph of the
  // period, the check kernels and both device-to-host copies are queued
  // back to back on the stream.
  if (!c || iters < 0 || npts < 0 || npts > 2 || (npts > 0 && (!specs || !out_host)))
    return fail(PDHG_ERR_ARG, "run_period_check: bad argument");
  StepParams& h = *c->P_host;
  h.tau_w = tau_over_omega;
  h.sigma_w = sigma_omega;
  h.w0 = w0;
  h.iter0 = iter0;
  h.fail_iter = LLONG_MAX;
  CUDA_TRY(cudaMemcpyAsync(c->P, c->P_host, sizeof(StepParams), cudaMemcpyHostToDevice, c->stream));
  c->fuse_next = c->check_fuse && npts == 2 && specs[0] == PDHG_PT_CUR && specs[1] == PDHG_PT_AVG;
  int rc = launch_period(c, iters);
  if (rc) return rc;
  if (npts > 0) {
    if ((rc = pdhg_check_device(c, npts, specs))) return rc;
    CUDA_TRY(cudaMemcpyAsync(c->scal_host, c->scalars, (size_t)npts * PDHG_NQ * sizeof(double),
                             cudaMemcpyDeviceToHost, c->stream));
  }
  CUDA_TRY(cudaMemcpyAsync(&c->P_host->fail_iter, &c->P->fail_iter, sizeof(long long),
                           cudaMemcpyDeviceToHost, c->stream));
  CUDA_TRY(cudaStreamSynchronize(c->stream));
  if (fail_iter_out) *fail_iter_out = (c->P_host->fail_iter == LLONG_MAX) ? -1 : c->P_host->fail_iter;
  if (npts > 0) std::memcpy(out_host, c->scal_host, (size_t)npts * PDHG_NQ * sizeof(double));
  return 0;
}

int pdhg_check_device(pdhg_ctx* c, int32_t npts, const int32_t* specs) {
  CTX_DEVICE_GUARD(c);
  NvtxRange nvtx_range_("pdhg_check");
  if (!c || !specs || npts < 1 || npts > 2) return fail(PDHG_ERR_ARG, "bad argument");
  // primal side (rows of A): gathers full x, row-indexed y slice;
  // dual side (rows of A'): gathers full y, row-indexed x / z slices.
  CheckPts pp{}, pd{};
  for (int p = 0; p < npts; ++p) {
    const double *x, *y;
    point_xy(c, specs[p], &x, &y);
    pp.x[p] = x; pp.y[p] = y + c->yo; pp.zin[p] = nullptr; pp.zout[p] = nullptr;
    pd.x[p] = x + c->xo; pd.y[p] = y;
    pd.zin[p] = (specs[p] & PDHG_SPEC_BEST_Z) ? c->zbest + c->xo : nullptr;
    pd.zout[p] = nullptr;
  }
  // the period just run fused this check's A side into its last dual step
  const bool fused = c->fuse_ready && npts == 2 && specs[0] == PDHG_PT_CUR && specs[1] == PDHG_PT_AVG;
  c->fuse_ready = false;
  if (npts == 2 && PDHG_CHECK_PAIR) {
    // interleave the two points' gathered vectors (full padded length: the
    // check gathers by global index): 0.5 GB of copies on config 4 buys one
    // 16-byte gather per entry instead of two 8-byte ones
    const double *x0, *y0, *x1, *y1;
    point_xy(c, specs[0], &x0, &y0);
    point_xy(c, specs[1], &x1, &y1);
    if (!fused) k_pair<<<kCheckBlocks, kBlock, 0, c->stream>>>(x0, x1, c->px, c->nf);
    k_pair<<<kCheckBlocks, kBlock, 0, c->stream>>>(y0, y1, c->py, c->mf);
    pp.pair = c->px;
    pd.pair = c->py;
  }
  // A'y of both points for the next period's first primal step: written into
  // px by the dual side, which runs after the A side has finished gathering px
  const bool dots = c->check_dot && pd.pair && c->has_sell[1] && PDHG_CHECK_SELL;
  pd.dout = dots ? c->px + c->xo : nullptr;
  c->first_dot = -1;
  c->dots_ready = false;
  CUDA_TRY(cudaMemsetAsync(c->partials, 0, (size_t)kCheckBlocks * kMaxQ * 8, c->stream));
  int rc = 0;
  if (fused) {
    k_check_primal_fold<<<kCheckBlocks, kBlock, 0, c->stream>>>(c->A, c->sell[0], c->prob.b, pp, c->pr,
                                                                c->partials);
    CUDA_TRY(cudaGetLastError());
  } else if (pp.pair && c->has_sell[0] && PDHG_CHECK_SELL) {
    if (c->sell[0].u_long)
      k_check_primal_sell<PDHG_SELL_U_LONG><<<kCheckBlocks, kBlock, 0, c->stream>>>(c->A, c->sell[0], c->prob.b,
                                                                                  pp, c->partials);
    else
      k_check_primal_sell<PDHG_SELL_U><<<kCheckBlocks, kBlock, 0, c->stream>>>(c->A, c->sell[0], c->prob.b, pp,
                                                                             c->partials);
    CUDA_TRY(cudaGetLastError());
  } else {
    rc = dispatch_lanes<CheckLaunch>(c->a_lanes, true, (int)npts, c->A, c->prob.b, pp, c->partials,
                                     c->stream);
    if (rc) return rc;
  }
  if (pd.pair && c->has_sell[1] && PDHG_CHECK_SELL) {
    if (c->sell[1].u_long)
      k_check_dual_sell<PDHG_SELL_U_LONG><<<kCheckBlocks, kBlock, 0, c->stream>>>(c->At, c->sell[1], c->prob.c, pd,
                                                                                c->partials);
    else
      k_check_dual_sell<PDHG_SELL_U><<<kCheckBlocks, kBlock, 0, c->stream>>>(c->At, c->sell[1], c->prob.c, pd,
                                                                           c->partials);
    CUDA_TRY(cudaGetLastError());
  } else {
    rc = dispatch_lanes<CheckLaunch>(c->at_lanes, false, (int)npts, c->At, c->prob.c, pd, c->partials,
                                     c->stream);
    if (rc) return rc;
  }
  const int nq = npts * PDHG_NQ;
  k_reduce<<<nq, kBlock, 0, c->stream>>>(c->partials, kCheckBlocks, kMaxQ, nq, c->scalars);
  CUDA_TRY(cudaGetLastError());
  c->dots_ready = dots;
  return 0;
}

int pdhg_check_dot_enable(pdhg_ctx* c, int32_t on) {
  CTX_DEVICE_GUARD(c);
  if (!c) return fail(PDHG_ERR_ARG, "null ctx");
  c->first_dot = -1;
  c->dots_ready = false;
  if (!on) {
    c->check_dot = false;
    return 0;
  }
  // the check's dual side must run the primal step's own row loop (sliced ELL
  // of A'), on one GPU (no peers: the from-dot step has no fused all-gather)
  if (!c->has_sell[1] || !PDHG_CHECK_SELL || c->npeers[0] > 0 || c->has_psr[1] || c->coop_grid > 0 ||
      c->prob.at_nsplit > 1)
    return fail(PDHG_ERR_STATE, "check_dot: needs the sliced-ELL layout of A' on one GPU");
  c->check_dot = true;
  return 0;
}

int pdhg_check_fuse_enable(pdhg_ctx* c, int32_t on) {
  CTX_DEVICE_GUARD(c);
  if (!c) return fail(PDHG_ERR_ARG, "null ctx");
  c->fuse_next = c->fuse_ready = false;
  if (!on) {
    c->check_fuse = false;
    return 0;
  }
  // both steps on sliced ELL, one unsharded GPU, graph or direct periods
  if (!c->has_sell[0] || !c->has_sell[1] || !PDHG_CHECK_SELL || !PDHG_CHECK_PAIR || c->npeers[0] > 0 ||
      c->npeers[1] > 0 || c->has_psr[0] || c->has_psr[1] || c->coop_grid > 0 || c->prob.a_nsplit > 1 ||
      c->prob.at_nsplit > 1 || c->xo != 0 || c->yo != 0 || c->mf != c->prob.m || c->nf != c->prob.n)
    return fail(PDHG_ERR_STATE, "check_fuse: needs the sliced-ELL layouts of A and A' on one GPU");
  c->check_fuse = true;
  return 0;
}

int pdhg_use_check_dot(pdhg_ctx* c, int32_t slot) {
  CTX_DEVICE_GUARD(c);
  if (!c || slot < 0 || slot > 1) return fail(PDHG_ERR_ARG, "use_check_dot: bad argument");
  if (!c->dots_ready) return fail(PDHG_ERR_STATE, "use_check_dot: the last call was not a two-point check "
                                                  "with check_dot enabled");
  c->first_dot = slot;
  return 0;
}

int pdhg_check(pdhg_ctx* c, int32_t npts, const int32_t* specs, double* out_host) {
  CTX_DEVICE_GUARD(c);
  if (!out_host) return fail(PDHG_ERR_ARG, "null out_host");
  int rc = pdhg_check_device(c, npts, specs);
  if (rc) return rc;
  const int nq = npts * PDHG_NQ;
  CUDA_TRY(cudaMemcpyAsync(c->scal_host, c->scalars, nq * sizeof(double), cudaMemcpyDeviceToHost,
                           c->stream));
  CUDA_TRY(cudaStreamSynchronize(c->stream));
  std::memcpy(out_host, c->scal_host, nq * sizeof(double));
  return 0;
}

int pdhg_restart(pdhg_ctx* c, int32_t which) {
  CTX_DEVICE_GUARD(c);
  if (!c) return fail(PDHG_ERR_ARG, "null ctx");
  const size_t nb = (size_t)c->nf * 8, mb = (size_t)c->mf * 8;
  c->fuse_ready = false;
  if (which == PDHG_PT_CUR) {
    CUDA_TRY(cudaMemcpyAsync(c->xbar, c->x, nb, cudaMemcpyDeviceToDevice, c->stream));
    CUDA_TRY(cudaMemcpyAsync(c->ybar, c->y, mb, cudaMemcpyDeviceToDevice, c->stream));
  } else if (which == PDHG_PT_AVG) {
    CUDA_TRY(cudaMemcpyAsync(c->x, c->xbar, nb, cudaMemcpyDeviceToDevice, c->stream));
    CUDA_TRY(cudaMemcpyAsync(c->y, c->ybar, mb, cudaMemcpyDeviceToDevice, c->stream));
  } else {
    return fail(PDHG_ERR_ARG, "restart point must be CUR or AVG");
  }
  return 0;
}

int reduced_costs(pdhg_ctx* c, int32_t spec, double* z_slice) {
  const double *x, *y;
  point_xy(c, spec, &x, &y);
  CheckPts pd{};
  pd.x[0] = x + c->xo; pd.y[0] = y; pd.zin[0] = nullptr; pd.zout[0] = z_slice;
  int rc = dispatch_lanes<CheckLaunch>(c->at_lanes, false, 1, c->At, c->prob.c, pd, c->partials,
                                       c->stream);
  if (rc) return rc;
  CUDA_TRY(cudaGetLastError());
  return 0;
}

int pdhg_save_best(pdhg_ctx* c, int32_t which, int32_t flags) {
  CTX_DEVICE_GUARD(c);
  if (!c) return fail(PDHG_ERR_ARG, "null ctx");
  const double *x, *y;
  point_xy(c, which, &x, &y);
  if (flags & PDHG_BEST_Z) {
    int rc = reduced_costs(c, which, c->zbest + c->xo);
    if (rc) return rc;
  }
  if ((flags & PDHG_BEST_XY) && (which & 3) != PDHG_PT_BEST) {
    CUDA_TRY(cudaMemcpyAsync(c->xbest, x, (size_t)c->nf * 8, cudaMemcpyDeviceToDevice, c->stream));
    CUDA_TRY(cudaMemcpyAsync(c->ybest, y, (size_t)c->mf * 8, cudaMemcpyDeviceToDevice, c->stream));
  }
  return 0;
}

int pdhg_fetch(pdhg_ctx* c, int32_t spec, double* x_host, double* y_host, double* z_host) {
  CTX_DEVICE_GUARD(c);
  if (!c) return fail(PDHG_ERR_ARG, "null ctx");
  const double *x, *y;
  point_xy(c, spec, &x, &y);
  const size_t nb = (size_t)c->nf * 8, mb = (size_t)c->mf * 8;
  if (x_host) CUDA_TRY(cudaMemcpyAsync(x_host, x, nb, cudaMemcpyDeviceToHost, c->stream));
  if (y_host) CUDA_TRY(cudaMemcpyAsync(y_host, y, mb, cudaMemcpyDeviceToHost, c->stream));
  if (z_host) {
    if (spec & PDHG_SPEC_BEST_Z) {
      CUDA_TRY(cudaMemcpyAsync(z_host, c->zbest, nb, cudaMemcpyDeviceToHost, c->stream));
    } else {
      int rc = reduced_costs(c, spec, c->tn1 + c->xo);
      if (rc) return rc;
      CUDA_TRY(cudaMemcpyAsync(z_host, c->tn1, nb, cudaMemcpyDeviceToHost, c->stream));
    }
  }
  CUDA_TRY(cudaStreamSynchronize(c->stream));
  return 0;
}

int pdhg_point_device(pdhg_ctx* c, int32_t spec, const double** x_dev, const double** y_dev,
                      const double** z_dev) {
  CTX_DEVICE_GUARD(c);
  if (!c || !x_dev || !y_dev || !z_dev) return fail(PDHG_ERR_ARG, "null argument");
  point_xy(c, spec, x_dev, y_dev);
  if (spec & PDHG_SPEC_BEST_Z) {
    *z_dev = c->zbest;
  } else {
    int rc = reduced_costs(c, spec, c->tn1 + c->xo);
    if (rc) return rc;
    *z_dev = c->tn1;
  }
  return 0;
}

void* pdhg_vector(pdhg_ctx* c, int32_t which) {
  if (!c) return nullptr;
  switch (which) {
    case PDHG_VEC_X: return c->x;
    case PDHG_VEC_XE: return c->xe;
    case PDHG_VEC_XBAR: return c->xbar;
    case PDHG_VEC_XBEST: return c->xbest;
    case PDHG_VEC_ZBEST: return c->zbest;
    case PDHG_VEC_TN1: return c->tn1;
    case PDHG_VEC_TN2: return c->tn2;
    case PDHG_VEC_Y: return c->y;
    case PDHG_VEC_YBAR: return c->ybar;
    case PDHG_VEC_YBEST: return c->ybest;
    case PDHG_VEC_TM1: return c->tm1;
    case PDHG_VEC_SCALARS: return c->scalars;
    case PDHG_VEC_FAILWORD: return &c->P->fail_iter;
    default: fail(PDHG_ERR_ARG, "unknown vector id"); return nullptr;
  }
}

int pdhg_reduced_costs(pdhg_ctx* c, int32_t spec, double* z_slice) {
  CTX_DEVICE_GUARD(c);
  if (!c || !z_slice) return fail(PDHG_ERR_ARG, "null argument");
  return reduced_costs(c, spec, z_slice);
}

int pdhg_set_step(pdhg_ctx* c, int64_t iter0, double tau_over_omega, double sigma_omega, double w0) {
  CTX_DEVICE_GUARD(c);
  if (!c) return fail(PDHG_ERR_ARG, "null ctx");
  CUDA_TRY(cudaStreamSynchronize(c->stream));  // the pinned staging struct is reused
  StepParams& h = *c->P_host;
  h.tau_w = tau_over_omega; h.sigma_w = sigma_omega; h.w0 = w0; h.iter0 = iter0;
  h.fail_iter = LLONG_MAX;
  CUDA_TRY(cudaMemcpyAsync(c->P, c->P_host, sizeof(StepParams), cudaMemcpyHostToDevice, c->stream));
  return 0;
}

int pdhg_half_step(pdhg_ctx* c, int32_t primal, int32_t j) {
  CTX_DEVICE_GUARD(c);
  if (c) { c->first_dot = -1; c->dots_ready = false; }  // state changes: no check dots
  if (!c) return fail(PDHG_ERR_ARG, "null ctx");
  int rc = launch_step(c, primal != 0, j);
  if (rc) return rc;
  CUDA_TRY(cudaGetLastError());
  return 0;
}

int pdhg_half_step_pass(pdhg_ctx* c, int32_t primal, int32_t j, int32_t pass) {
  CTX_DEVICE_GUARD(c);
  if (c) { c->first_dot = -1; c->dots_ready = false; }  // state changes: no check dots
  if (!c) return fail(PDHG_ERR_ARG, "null ctx");
  int rc = launch_step_pass(c, primal != 0, j, pass);
  if (rc) return rc;
  CUDA_TRY(cudaGetLastError());
  return 0;
}

int pdhg_set_peers(pdhg_ctx* c, int32_t which, const double* const* peers_dev, int32_t npeers) {
  CTX_DEVICE_GUARD(c);
  if (c && which == 0 && npeers > 0) { c->check_dot = false; c->first_dot = -1; c->dots_ready = false; }
  if (c && which <= 1 && npeers > 0) c->check_fuse = c->fuse_next = c->fuse_ready = false;
  if (!c || which < 0 || which > 2 || npeers < 0 || (npeers > 0 && !peers_dev))
    return fail(PDHG_ERR_ARG, "set_peers: bad argument");
  if (which == 2) {  // peers' fail words (pdhg_vector(peer, PDHG_VEC_FAILWORD))
    c->P_host->fail_peers = reinterpret_cast<unsigned long long* const*>(const_cast<double**>(peers_dev));
    c->P_host->nfail = npeers;
    CUDA_TRY(cudaStreamSynchronize(c->stream));
    CUDA_TRY(cudaMemcpyAsync(c->P, c->P_host, sizeof(StepParams), cudaMemcpyHostToDevice, c->stream));
    CUDA_TRY(cudaStreamSynchronize(c->stream));
    return 0;
  }
  c->peers[which] = const_cast<double* const*>(peers_dev);
  c->npeers[which] = npeers;
  c->P_host->peers[which] = Peers{c->peers[which], npeers, which == 0 ? c->xo : c->yo};
  CUDA_TRY(cudaStreamSynchronize(c->stream));
  CUDA_TRY(cudaMemcpyAsync(&c->P->peers[which], &c->P_host->peers[which], sizeof(Peers),
                           cudaMemcpyHostToDevice, c->stream));
  for (auto& kv : c->graphs) cudaGraphExecDestroy(kv.second);  // captured StepArgs are stale
  c->graphs.clear();
  return 0;
}

int pdhg_fail_iter(pdhg_ctx* c, int64_t* fail_iter_out) {
  CTX_DEVICE_GUARD(c);
  if (!c || !fail_iter_out) return fail(PDHG_ERR_ARG, "null argument");
  CUDA_TRY(cudaMemcpyAsync(&c->P_host->fail_iter, &c->P->fail_iter, sizeof(long long),
                           cudaMemcpyDeviceToHost, c->stream));
  CUDA_TRY(cudaStreamSynchronize(c->stream));
  *fail_iter_out = (c->P_host->fail_iter == LLONG_MAX) ? -1 : c->P_host->fail_iter;
  return 0;
}

int pdhg_sumsq(pdhg_ctx* c, const double* v, int64_t len, double* out_dev) {
  CTX_DEVICE_GUARD(c);
  if (!c || !v || !out_dev || len < 0 || len >= INT_MAX) return fail(PDHG_ERR_ARG, "bad argument");
  k_sumsq<<<kCheckBlocks, kBlock, 0, c->stream>>>(v, (int)len, c->partials);
  k_reduce<<<1, kBlock, 0, c->stream>>>(c->partials, kCheckBlocks, 1, 1, out_dev);
  CUDA_TRY(cudaGetLastError());
  return 0;
}

int pdhg_div(pdhg_ctx* c, const double* w, double* v, int64_t len, double s) {
  CTX_DEVICE_GUARD(c);
  if (!c || !w || !v || len < 0 || len >= INT_MAX) return fail(PDHG_ERR_ARG, "bad argument");
  if (len > 0) k_div<<<(unsigned)((len + kBlock - 1) / kBlock), kBlock, 0, c->stream>>>(w, v, s, (int)len);
  CUDA_TRY(cudaGetLastError());
  return 0;
}

int pdhg_time_kernel(pdhg_ctx* c, int32_t which, int32_t reps, double tau_over_omega,
                     double sigma_omega, double* avg_ms_out) {
  CTX_DEVICE_GUARD(c);
  if (c) { c->first_dot = -1; c->dots_ready = false; }  // state changes: no check dots
  if (!c || reps < 1 || !avg_ms_out) return fail(PDHG_ERR_ARG, "bad argument");
  StepParams& h = *c->P_host;
  h.tau_w = tau_over_omega; h.sigma_w = sigma_omega; h.w0 = 0.0; h.iter0 = 0; h.fail_iter = LLONG_MAX;
  CUDA_TRY(cudaMemcpyAsync(c->P, c->P_host, sizeof(StepParams), cudaMemcpyHostToDevice, c->stream));
  cudaEvent_t e0, e1;
  CUDA_TRY(cudaEventCreate(&e0));
  CUDA_TRY(cudaEventCreate(&e1));
  // which: 0 = primal step, 1 = dual step, 2 = one iteration (primal then dual)
  int rc = launch_step(c, which != 1, 0);  // warm
  if (!rc && which == 2) rc = launch_step(c, false, 0);
  if (rc) return rc;
  CUDA_TRY(cudaEventRecord(e0, c->stream));
  for (int r = 0; r < reps && !rc; ++r) {
    rc = launch_step(c, which != 1, 0);
    if (!rc && which == 2) rc = launch_step(c, false, 0);
  }
  CUDA_TRY(cudaEventRecord(e1, c->stream));
  CUDA_TRY(cudaEventSynchronize(e1));
  float ms = 0.f;
  CUDA_TRY(cudaEventElapsedTime(&ms, e0, e1));
  cudaEventDestroy(e0);
  cudaEventDestroy(e1);
  if (rc) return rc;
  *avg_ms_out = ms / reps;
  return 0;
}

int pdhg_split_build(int32_t m, const int32_t* ptr, const int32_t* col, int32_t K, int32_t chunk,
                     int32_t* split_out, int32_t* flag_dev, void* stream, int32_t* unsorted_out) {
  if (m <= 0 || K < 2 || chunk <= 0 || !ptr || !col || !split_out || !flag_dev)
    return fail(PDHG_ERR_ARG, "split_build: bad argument");
  cudaStream_t s = (cudaStream_t)stream;
  CUDA_TRY(cudaMemsetAsync(flag_dev, 0, 4, s));
  k_split<<<(m + 255) / 256, 256, 0, s>>>(m, ptr, col, K, chunk, split_out, flag_dev);
  int h = 0;
  CUDA_TRY(cudaMemcpyAsync(&h, flag_dev, 4, cudaMemcpyDeviceToHost, s));
  CUDA_TRY(cudaStreamSynchronize(s));
  if (unsorted_out) *unsorted_out = h;
  return 0;
}

size_t pdhg_transpose_tmp_bytes(int64_t nnz, int32_t m, int32_t n) {
  size_t cub_bytes = 0;
  cub::DoubleBuffer<int> k(nullptr, nullptr), v(nullptr, nullptr);
  cub::DeviceRadixSort::SortPairs(nullptr, cub_bytes, k, v, (int)nnz);
  (void)m; (void)n;
  return 5 * align_up((size_t)nnz * 4 + 256) + align_up(cub_bytes + 256);
}

int pdhg_transpose_csr(int32_t m, int32_t n, int64_t nnz, const int32_t* a_ptr, const int32_t* a_col,
                       const double* a_val, int32_t* at_ptr, int32_t* at_col, double* at_val,
                       void* tmp, size_t tmp_bytes, void* stream) {
  if (nnz < 0 || nnz >= INT_MAX) return fail(PDHG_ERR_ARG, "nnz out of int32 range");
  if (tmp_bytes < pdhg_transpose_tmp_bytes(nnz, m, n)) return fail(PDHG_ERR_ARG, "tmp too small");
  cudaStream_t s = (cudaStream_t)stream;
  Carve cv{(char*)tmp};
  int* k0 = cv.take<int>(nnz);
  int* k1 = cv.take<int>(nnz);
  int* v0 = cv.take<int>(nnz);
  int* v1 = cv.take<int>(nnz);
  int* rid = cv.take<int>(nnz);
  size_t cub_bytes = tmp_bytes - cv.off;
  void* cub_tmp = (char*)tmp + cv.off;
  if (nnz > 0) {
    CUDA_TRY(cudaMemcpyAsync(k0, a_col, (size_t)nnz * 4, cudaMemcpyDeviceToDevice, s));
    k_iota<<<(unsigned)((nnz + 255) / 256), 256, 0, s>>>(v0, nnz);
    k_row_ids<<<(m + 255) / 256, 256, 0, s>>>(a_ptr, m, rid);
    cub::DoubleBuffer<int> kb(k0, k1), vb(v0, v1);
    int bits = 1;
    while (bits < 31 && (1LL << bits) <= n) ++bits;
    CUDA_TRY(cub::DeviceRadixSort::SortPairs(cub_tmp, cub_bytes, kb, vb, (int)nnz, 0, bits, s));
    k_gather_t<<<(unsigned)((nnz + 255) / 256), 256, 0, s>>>(vb.Current(), rid, a_val, at_col, at_val, nnz);
    k_col_ptr<<<(n + 1 + 255) / 256, 256, 0, s>>>(kb.Current(), nnz, n, at_ptr);
  } else {
    CUDA_TRY(cudaMemsetAsync(at_ptr, 0, (size_t)(n + 1) * 4, s));
  }
  CUDA_TRY(cudaGetLastError());
  return 0;
}

// Row relabelling (GpuOptions.row_order): new row r = old row perm[r]; the
// caller scans the permuted lengths into new_ptr (rows+1) first.
int pdhg_permute_rows(int32_t rows, const int32_t* perm, const int32_t* ptr, const int32_t* col,
                      const double* val, const int32_t* new_ptr, int32_t* new_col, double* new_val,
                      void* stream) {
  if (rows <= 0 || !perm || !ptr || !col || !val || !new_ptr || !new_col || !new_val)
    return fail(PDHG_ERR_ARG, "permute_rows: bad argument");
  k_permute_rows<<<(unsigned)(((long long)rows * 32 + 255) / 256), 256, 0, (cudaStream_t)stream>>>(
      rows, perm, ptr, col, val, new_ptr, new_col, new_val);
  CUDA_TRY(cudaGetLastError());
  return 0;
}

// Feature bits of this build: 1 = the experiment layouts (PSR, persistent
// periods, L2 windows; PDHG_EXPERIMENTAL).
int pdhg_features(void) { return (PDHG_EXPERIMENTAL ? 1 : 0) | (PDHG_BOUNDS_CHECK ? 2 : 0); }

#if !PDHG_EXPERIMENTAL
// The PSR builders live in psr_build.cu, compiled into the experiment build
// only; the product library keeps the symbols and reports the missing layout.
size_t pdhg_psr_tmp_bytes(int32_t, int32_t, int64_t) { return 0; }
int pdhg_psr_plan(int32_t, int32_t, int64_t, const int32_t*, const int32_t*, int32_t, int32_t, void*, size_t,
                  void*, int32_t*, int32_t*, int32_t*, int32_t*, int32_t*, int64_t*, int64_t*) {
  return fail(PDHG_ERR_ARG, "PSR layouts need the experiment build (PDHG_EXPERIMENTAL)");
}
int pdhg_psr_build(int32_t, int32_t, int64_t, const int32_t*, const int32_t*, const double*, int32_t, void*,
                   size_t, void*, int32_t*, int32_t*, int32_t*, uint16_t*, double*, uint16_t*, int32_t*,
                   uint8_t*) {
  return fail(PDHG_ERR_ARG, "PSR layouts need the experiment build (PDHG_EXPERIMENTAL)");
}
#endif

// Bounds-checked build only (PDHG_BOUNDS_CHECK): out-of-bounds loads seen
// since the last call (count, first index, its bound); resets the counter.
// Returns PDHG_ERR_STATE in the product build.
int pdhg_debug_oob(int64_t* count, int64_t* first_index, int64_t* first_bound) {
#if PDHG_BOUNDS_CHECK
  unsigned long long n = 0;
  long long first[2] = {0, 0};
  CUDA_TRY(cudaDeviceSynchronize());
  CUDA_TRY(cudaMemcpyFromSymbol(&n, g_oob_count, sizeof(n)));
  CUDA_TRY(cudaMemcpyFromSymbol(first, g_oob_first, sizeof(first)));
  const unsigned long long zero = 0;
  CUDA_TRY(cudaMemcpyToSymbol(g_oob_count, &zero, sizeof(zero)));
  if (count) *count = (int64_t)n;
  if (first_index) *first_index = first[0];
  if (first_bound) *first_bound = first[1];
  return 0;
#else
  (void)count; (void)first_index; (void)first_bound;
  return fail(PDHG_ERR_STATE, "pdhg_debug_oob needs the bounds-checked build (PDHG_BOUNDS_CHECK)");
#endif
}

}  // extern "C"
