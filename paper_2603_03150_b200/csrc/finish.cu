// finish.cu -- device finishing of the PDHG point.
//
// Restates, on the device, the functions that turn the PDHG result into a
// point on the user's model and measure it:
//   unscale_point           transform.py:87-93   x = C x_s, y = R y_s, z = z_s / C
//   restrict_point          lp_core.py:371-385   x = x_std[pos] + shift | x_pos - x_neg; z = c - A'y
//   lift_point              lp_core.py:388-427   clamp, slack activities, bound-row duals, z
//   violation_summary       lp_core.py:468-485   (via residuals, lp_core.py:430-444)
// Sparse products use scipy's csr_matvec order (one sequential sum per row
// from 0.0, products rounded before the add, no FMA), so restrict / lift are
// bit-identical to the reference; the three dot products of residuals()
// (OpenBLAS ddot in the reference) are fixed-order block trees, equal to
// rounding.
#include "../../include/pdhg_b200.h"

#include <cuda_runtime.h>

#include <string>

namespace pdhg_internal {
int set_error(int code, const std::string& msg);
}

namespace {

using pdhg_internal::set_error;

#define FN_TRY(expr)                                                                       \
  do {                                                                                     \
    cudaError_t e_ = (expr);                                                               \
    if (e_ != cudaSuccess)                                                                 \
      return set_error(PDHG_ERR_CUDA, std::string(#expr) + ": " + cudaGetErrorString(e_)); \
  } while (0)

constexpr int kT = 256;
constexpr int kDotBlocks = 148 * 4;  // fixed grid => fixed reduction order
unsigned nb(long long n) { return (unsigned)((n + kT - 1) / kT); }
size_t a256(size_t v) { return (v + 255) & ~(size_t)255; }

// out[r] = sum_k val[k] * v[col[k]] over row r in stored order, starting from
// 0.0 (csr_matvec); with base: out[r] = base[r] - sum
__global__ void k_spmv_seq(int rows, const int* __restrict__ ptr, const int* __restrict__ col,
                           const double* __restrict__ val, const double* __restrict__ v,
                           const double* __restrict__ base, double* __restrict__ out) {
  const int r = blockIdx.x * blockDim.x + threadIdx.x;
  if (r >= rows) return;
  double s = 0.0;
  for (int k = ptr[r], e = ptr[r + 1]; k < e; ++k) s = __dadd_rn(s, __dmul_rn(val[k], v[col[k]]));
  out[r] = base ? __dsub_rn(base[r], s) : s;
}

__global__ void k_unscale(int n, int m, const double* __restrict__ rs, const double* __restrict__ cs,
                          const double* __restrict__ xs, const double* __restrict__ ys,
                          const double* __restrict__ zs, double* __restrict__ x,
                          double* __restrict__ y, double* __restrict__ z) {
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i < n) {
    x[i] = __dmul_rn(cs[i], xs[i]);
    z[i] = __ddiv_rn(zs[i], cs[i]);
  }
  if (i < m) y[i] = __dmul_rn(rs[i], ys[i]);
}

// restrict_point x part (lp_core.py:377-380)
__global__ void k_restrict_x(int n, const int* __restrict__ pos, const int* __restrict__ neg,
                             const double* __restrict__ shifts, const double* __restrict__ xs,
                             double* __restrict__ x) {
  const int j = blockIdx.x * blockDim.x + threadIdx.x;
  if (j >= n) return;
  const double xp = xs[pos[j]];
  x[j] = neg[j] >= 0 ? __dsub_rn(xp, xs[neg[j]]) : __dadd_rn(xp, shifts[j]);
}

// np.maximum(a, b) == (a > b || isnan(a)) ? a : b  (ties return b: np.maximum(0.0, -0.0) is -0.0)
__device__ __forceinline__ double np_maximum(double a, double b) { return (a > b || a != a) ? a : b; }

// lift_point structural part (lp_core.py:404-409): np.maximum(shifted, 0.0)
__global__ void k_lift_x(int n, const double* __restrict__ x, const double* __restrict__ shifts,
                         const int* __restrict__ pos, const int* __restrict__ neg,
                         double* __restrict__ xs) {
  const int j = blockIdx.x * blockDim.x + threadIdx.x;
  if (j >= n) return;
  const double sh = __dsub_rn(x[j], shifts[j]);
  xs[pos[j]] = np_maximum(sh, 0.0);
  if (neg[j] >= 0) xs[neg[j]] = np_maximum(-sh, 0.0);
}

// slack values: builtin max(0.0, r/coef) keeps 0.0 unless r/coef > 0.0 (lp_core.py:411-417)
__global__ void k_lift_slacks(int m, const int* __restrict__ slack, const double* __restrict__ coef,
                              const double* __restrict__ r, double* __restrict__ xs) {
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= m || slack[i] < 0) return;
  const double v = __ddiv_rn(r[i], coef[i]);
  xs[slack[i]] = v > 0.0 ? v : 0.0;
}

// bound-row duals: builtin min(0.0, z) keeps 0.0 unless z < 0.0 (lp_core.py:419-424)
__global__ void k_lift_bound(int m, const int* __restrict__ bvar, const double* __restrict__ zgen,
                             double* __restrict__ ys) {
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= m || bvar[i] < 0) return;
  const double z = zgen[bvar[i]];
  ys[i] = z < 0.0 ? z : 0.0;
}

// out = np.maximum(0.0, v)
__global__ void k_max0(long long len, const double* __restrict__ v, double* __restrict__ out) {
  const long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= len) return;
  out[i] = np_maximum(0.0, v[i]);
}

// r_d = (c - A'y) - z   (lp_core.py:437; t = c - A'y already computed)
__global__ void k_sub(int n, const double* __restrict__ t, const double* __restrict__ z,
                      double* __restrict__ out) {
  const int j = blockIdx.x * blockDim.x + threadIdx.x;
  if (j < n) out[j] = __dsub_rn(t[j], z[j]);
}

__device__ __forceinline__ double nan_max(double a, double b) { return (a != a || a > b) ? a : b; }

// per-block partials over a contiguous chunk: [0] = sum a*b (or max |a| when b == nullptr)
__global__ void __launch_bounds__(kT) k_partial(long long len, const double* __restrict__ a,
                                                const double* __restrict__ b, double* __restrict__ part) {
  __shared__ double red[kT / 32];
  const long long chunk = (len + gridDim.x - 1) / gridDim.x;
  const long long s = blockIdx.x * chunk, e = s + chunk < len ? s + chunk : len;
  double acc = b ? 0.0 : 0.0;
  for (long long i = s + threadIdx.x; i < e; i += kT)
    acc = b ? __dadd_rn(acc, __dmul_rn(a[i], b[i])) : nan_max(acc, fabs(a[i]));
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) {
    const double t = __shfl_xor_sync(0xffffffffu, acc, o);
    acc = b ? acc + t : nan_max(acc, t);
  }
  const int w = threadIdx.x >> 5, l = threadIdx.x & 31;
  if (l == 0) red[w] = acc;
  __syncthreads();
  if (threadIdx.x == 0) {
    double t = red[0];
    for (int k = 1; k < kT / 32; ++k) t = b ? t + red[k] : nan_max(t, red[k]);
    part[blockIdx.x] = t;
  }
}

__global__ void k_final(const double* __restrict__ part, int nparts, int is_max, double* __restrict__ out) {
  if (threadIdx.x || blockIdx.x) return;
  double t = is_max ? 0.0 : 0.0;
  for (int k = 0; k < nparts; ++k) t = is_max ? nan_max(t, part[k]) : t + part[k];
  *out = t;
}

// numpy's clip for floats: MIN(MAX(v, lo), hi) with MAX(a,b) = isnan(a) ? a :
// (a > b ? a : b) and MIN(a,b) = isnan(a) ? a : (a < b ? a : b)
__device__ __forceinline__ double np_clip(double v, double lo, double hi) {
  const double t = (v != v) ? v : (v > lo ? v : lo);
  return (t != t) ? t : (t < hi ? t : hi);
}

// center_toward_target (warmstart.py:71-96), elementwise, the reference's ops in order
__global__ void k_center(long long n, const double* __restrict__ x, const double* __restrict__ z, double mu,
                         double a, double d, double* __restrict__ xo, double* __restrict__ zo) {
  const long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n) return;
  const double xp = np_maximum(x[i], a);
  const double zp = np_maximum(z[i], a);
  const bool x_first = xp < zp;
  double xn, zn;
  if (x_first) {
    const double x1 = np_clip(__ddiv_rn(mu, zp), __dsub_rn(xp, d), __dadd_rn(xp, d));
    xn = x1;
    zn = np_clip(__ddiv_rn(mu, x1), __dsub_rn(zp, d), __dadd_rn(zp, d));
  } else {
    const double z2 = np_clip(__ddiv_rn(mu, xp), __dsub_rn(zp, d), __dadd_rn(zp, d));
    zn = z2;
    xn = np_clip(__ddiv_rn(mu, z2), __dsub_rn(xp, d), __dadd_rn(xp, d));
  }
  xo[i] = np_maximum(xn, a);
  zo[i] = np_maximum(zn, a);
}

}  // namespace

extern "C" {

int pdhg_center_toward_target(int64_t n, const double* x, const double* z, double mu, double alpha_min,
                              double delta_max, double* x_out, double* z_out, void* stream) {
  if (n < 0 || (n > 0 && (!x || !z || !x_out || !z_out))) return set_error(PDHG_ERR_ARG, "center: bad argument");
  if (n == 0) return 0;
  k_center<<<nb(n), kT, 0, (cudaStream_t)stream>>>(n, x, z, mu, alpha_min, delta_max, x_out, z_out);
  FN_TRY(cudaGetLastError());
  return 0;
}

size_t pdhg_dot_tmp_bytes(void) { return a256((size_t)kDotBlocks * 8) + a256(8); }

int pdhg_dot(int64_t n, const double* a, const double* b, void* tmp, size_t tmp_bytes, void* stream,
             double* out_host) {
  if (n < 0 || !tmp || !out_host || (n > 0 && (!a || !b))) return set_error(PDHG_ERR_ARG, "dot: bad argument");
  if (tmp_bytes < pdhg_dot_tmp_bytes()) return set_error(PDHG_ERR_ARG, "dot: tmp too small");
  cudaStream_t s = (cudaStream_t)stream;
  double* part = (double*)tmp;
  double* res = (double*)((char*)tmp + a256((size_t)kDotBlocks * 8));
  FN_TRY(cudaMemsetAsync(res, 0, 8, s));
  if (n > 0) {
    k_partial<<<kDotBlocks, kT, 0, s>>>(n, a, b, part);
    k_final<<<1, 32, 0, s>>>(part, kDotBlocks, 0, res);
  }
  FN_TRY(cudaMemcpyAsync(out_host, res, 8, cudaMemcpyDeviceToHost, s));
  FN_TRY(cudaStreamSynchronize(s));
  FN_TRY(cudaGetLastError());
  return 0;
}

int pdhg_spmv_seq(int32_t rows, const int32_t* ptr, const int32_t* col, const double* val,
                  const double* v, const double* base, double* out, void* stream) {
  if (rows < 0 || (rows > 0 && (!ptr || !out))) return set_error(PDHG_ERR_ARG, "spmv_seq: bad argument");
  if (rows == 0) return 0;
  k_spmv_seq<<<nb(rows), kT, 0, (cudaStream_t)stream>>>(rows, ptr, col, val, v, base, out);
  FN_TRY(cudaGetLastError());
  return 0;
}

int pdhg_unscale_point(int32_t n, int32_t m, const double* row_scale, const double* col_scale,
                       const double* xs, const double* ys, const double* zs, double* x, double* y,
                       double* z, void* stream) {
  if (n < 0 || m < 0) return set_error(PDHG_ERR_ARG, "unscale_point: bad argument");
  const int len = n > m ? n : m;
  if (len == 0) return 0;
  k_unscale<<<nb(len), kT, 0, (cudaStream_t)stream>>>(n, m, row_scale, col_scale, xs, ys, zs, x, y, z);
  FN_TRY(cudaGetLastError());
  return 0;
}

int pdhg_restrict_x(int32_t n_general, const int32_t* pos_col, const int32_t* neg_col,
                    const double* shifts, const double* x_std, double* x, void* stream) {
  if (n_general < 0) return set_error(PDHG_ERR_ARG, "restrict_x: bad argument");
  if (n_general == 0) return 0;
  k_restrict_x<<<nb(n_general), kT, 0, (cudaStream_t)stream>>>(n_general, pos_col, neg_col, shifts, x_std, x);
  FN_TRY(cudaGetLastError());
  return 0;
}

int pdhg_lift_x(int32_t n_general, const double* x, const double* shifts, const int32_t* pos_col,
                const int32_t* neg_col, double* x_std, void* stream) {
  if (n_general < 0) return set_error(PDHG_ERR_ARG, "lift_x: bad argument");
  if (n_general == 0) return 0;
  k_lift_x<<<nb(n_general), kT, 0, (cudaStream_t)stream>>>(n_general, x, shifts, pos_col, neg_col, x_std);
  FN_TRY(cudaGetLastError());
  return 0;
}

int pdhg_lift_slacks(int32_t m_std, const int32_t* slack_of_row, const double* slack_coef,
                     const double* r, double* x_std, void* stream) {
  if (m_std < 0) return set_error(PDHG_ERR_ARG, "lift_slacks: bad argument");
  if (m_std == 0) return 0;
  k_lift_slacks<<<nb(m_std), kT, 0, (cudaStream_t)stream>>>(m_std, slack_of_row, slack_coef, r, x_std);
  FN_TRY(cudaGetLastError());
  return 0;
}

int pdhg_lift_bound_duals(int32_t m_std, const int32_t* bound_var, const double* z_gen,
                          double* y_std, void* stream) {
  if (m_std < 0) return set_error(PDHG_ERR_ARG, "lift_bound_duals: bad argument");
  if (m_std == 0) return 0;
  k_lift_bound<<<nb(m_std), kT, 0, (cudaStream_t)stream>>>(m_std, bound_var, z_gen, y_std);
  FN_TRY(cudaGetLastError());
  return 0;
}

int pdhg_max0(int64_t len, const double* v, double* out, void* stream) {
  if (len < 0) return set_error(PDHG_ERR_ARG, "max0: bad argument");
  if (len == 0) return 0;
  k_max0<<<nb(len), kT, 0, (cudaStream_t)stream>>>(len, v, out);
  FN_TRY(cudaGetLastError());
  return 0;
}

size_t pdhg_violation_tmp_bytes(int32_t m, int32_t n) {
  return a256((size_t)(m > 0 ? m : 1) * 8) + a256((size_t)(n > 0 ? n : 1) * 8) * 2 +
         a256((size_t)kDotBlocks * 8) + a256(8 * 8);
}

int pdhg_violation(int32_t m, int32_t n, const int32_t* a_ptr, const int32_t* a_col,
                   const double* a_val, const int32_t* at_ptr, const int32_t* at_col,
                   const double* at_val, const double* b, const double* c, const double* x,
                   const double* y, const double* z, void* tmp, size_t tmp_bytes, void* stream,
                   double* out_host) {
  if (m < 0 || n < 0 || !tmp || !out_host) return set_error(PDHG_ERR_ARG, "violation: bad argument");
  if (tmp_bytes < pdhg_violation_tmp_bytes(m, n)) return set_error(PDHG_ERR_ARG, "violation: tmp too small");
  cudaStream_t s = (cudaStream_t)stream;
  char* p = (char*)tmp;
  double* rp = (double*)p; p += a256((size_t)(m > 0 ? m : 1) * 8);
  double* t = (double*)p; p += a256((size_t)(n > 0 ? n : 1) * 8);
  double* rd = (double*)p; p += a256((size_t)(n > 0 ? n : 1) * 8);
  double* part = (double*)p; p += a256((size_t)kDotBlocks * 8);
  double* res = (double*)p;
  FN_TRY(cudaMemsetAsync(res, 0, 8 * 8, s));
  if (m > 0) k_spmv_seq<<<nb(m), kT, 0, s>>>(m, a_ptr, a_col, a_val, x, b, rp);           // r_p = b - A x
  if (n > 0) {
    k_spmv_seq<<<nb(n), kT, 0, s>>>(n, at_ptr, at_col, at_val, y, c, t);               // c - A'y
    k_sub<<<nb(n), kT, 0, s>>>(n, t, z, rd);                                           // - z
  }
  struct Q { long long len; const double* a; const double* b; int is_max; };
  const Q qs[5] = {{m, rp, nullptr, 1}, {n, rd, nullptr, 1}, {n, c, x, 0}, {m, b, y, 0}, {n, x, z, 0}};
  for (int q = 0; q < 5; ++q) {
    if (qs[q].len == 0) continue;
    k_partial<<<kDotBlocks, kT, 0, s>>>(qs[q].len, qs[q].a, qs[q].b, part);
    k_final<<<1, 32, 0, s>>>(part, kDotBlocks, qs[q].is_max, res + q);
  }
  FN_TRY(cudaMemcpyAsync(out_host, res, 5 * 8, cudaMemcpyDeviceToHost, s));
  FN_TRY(cudaStreamSynchronize(s));
  FN_TRY(cudaGetLastError());
  return 0;
}

}  // extern "C"
