// stdform.cu -- device standard-form builder.
//
// Restates hybridlp.lp_core.to_standard_form (lp_core.py:250-368) on the
// device.  The reference walks the columns in Python (one list extend per
// column, then a COO -> CSR conversion); here every output row is produced
// directly in CSR order:
//   column j with a finite lower bound   -> one column pos_col[j]   (shift lo)
//   column j with lower = -inf / NaN     -> columns pos_col[j], pos_col[j]+1
//                                            (+a, -a; cost c, -c)         (lp_core.py:270-301)
//   row i with sense <= / >=             -> slack column, coef +1 / -1    (lp_core.py:303-314)
//   column j with a finite upper bound   -> row m+t: x_pos (- x_neg) + slack = up - shift
//                                                                         (lp_core.py:316-338)
// pos_col is increasing in j and pos_col+1 < pos_col of the next column, and
// slack columns come after all structural ones, so a row emitted in its
// input column order is already sorted -- the same arrays scipy's
// csr_matrix((vals, (rows, cols))) builds (canonical input: sorted, no
// duplicates; the host wrapper canonicalises).
// b_work[i] -= a_ij * lo_j is applied for j ascending with finite, nonzero
// lo (lp_core.py:281-283): one sequential, explicitly rounded pass per row,
// bit-identical to numpy's fancy-indexed update.
#include "../../include/pdhg_b200.h"

#include <cuda_runtime.h>
#include <cub/cub.cuh>

#include <string>

namespace pdhg_internal {
int set_error(int code, const std::string& msg);
}

namespace {

using pdhg_internal::set_error;

#define SF_TRY(expr)                                                                       \
  do {                                                                                     \
    cudaError_t e_ = (expr);                                                               \
    if (e_ != cudaSuccess)                                                                 \
      return set_error(PDHG_ERR_CUDA, std::string(#expr) + ": " + cudaGetErrorString(e_)); \
  } while (0)

size_t a256(size_t v) { return (v + 255) & ~(size_t)255; }
unsigned nb(long long n, int t) { return (unsigned)((n + t - 1) / t); }

struct Tmp {
  int* ncol;    // n+1: 1 or 2 output columns per input column, then exclusive scan -> pos_col
  int* fub;     // n+1: 1 if the upper bound is finite, then scan -> bound-row index
  int* ineq;    // m+1: 1 for <= / >= rows, then scan -> slack index
  int* rowlen;  // m+n+1: output row lengths, then scan -> output row pointer
  int* flag;    // non-finite matrix entry seen
  void* cub;
  size_t cub_bytes;
};

size_t cub_bytes_for(int len) {
  size_t b = 0;
  cub::DeviceScan::ExclusiveSum(nullptr, b, (int*)nullptr, (int*)nullptr, len);
  return b;
}

Tmp carve(void* tmp, int m, int n) {
  Tmp t;
  char* p = (char*)tmp;
  t.ncol = (int*)p; p += a256((size_t)(n + 1) * 4);
  t.fub = (int*)p; p += a256((size_t)(n + 1) * 4);
  t.ineq = (int*)p; p += a256((size_t)(m + 1) * 4);
  t.rowlen = (int*)p; p += a256((size_t)(m + n + 1) * 4);
  t.flag = (int*)p; p += 256;
  t.cub = p;
  t.cub_bytes = cub_bytes_for(m + n + 1);
  return t;
}

// in-place exclusive scan of len ints (len-1 values + a trailing 0 -> total)
int scan(Tmp& t, int* v, int len, cudaStream_t s) {
  size_t b = t.cub_bytes;
  SF_TRY(cub::DeviceScan::ExclusiveSum(t.cub, b, v, v, len, s));
  return 0;
}

__global__ void k_colflags(int n, const double* __restrict__ lower, const double* __restrict__ upper,
                           int* __restrict__ ncol, int* __restrict__ fub) {
  const int j = blockIdx.x * blockDim.x + threadIdx.x;
  if (j < n) {
    ncol[j] = isfinite(lower[j]) ? 1 : 2;
    fub[j] = isfinite(upper[j]) ? 1 : 0;
  } else if (j == n) {
    ncol[n] = 0;
    fub[n] = 0;
  }
}

__global__ void k_rowflags(int m, const int8_t* __restrict__ sense, int* __restrict__ ineq) {
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i < m) ineq[i] = sense[i] != PDHG_SENSE_EQ ? 1 : 0;
  else if (i == m) ineq[m] = 0;
}

// warp per general row: output length = sum of ncol over its entries + slack;
// also flags non-finite matrix entries (GeneralLp.validate, lp_core.py:80-81)
__global__ void k_rowlen(int m, const int* __restrict__ ptr, const int* __restrict__ col,
                         const double* __restrict__ val, const int* __restrict__ ncol_scan,
                         const int8_t* __restrict__ sense, int* __restrict__ rowlen,
                         int* __restrict__ flag) {
  const long long w = ((long long)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  const int lane = threadIdx.x & 31;
  if (w >= m) return;
  const int s = ptr[w], e = ptr[w + 1];
  int cnt = 0;
  bool bad = false;
  for (int k = s + lane; k < e; k += 32) {
    const int j = col[k];
    cnt += ncol_scan[j + 1] - ncol_scan[j];
    bad |= !isfinite(val[k]);
  }
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) cnt += __shfl_xor_sync(0xffffffffu, cnt, o);
  if (__any_sync(0xffffffffu, bad) && lane == 0) atomicOr(flag, 1);
  if (lane == 0) rowlen[w] = cnt + (sense[w] != PDHG_SENSE_EQ ? 1 : 0);
}

// thread per general column with a finite upper bound: its bound-row length
__global__ void k_boundlen(int m, int n, const int* __restrict__ ncol_scan, const int* __restrict__ fub_scan,
                           int* __restrict__ rowlen) {
  const int j = blockIdx.x * blockDim.x + threadIdx.x;
  if (j >= n) return;
  if (fub_scan[j + 1] - fub_scan[j]) rowlen[m + fub_scan[j]] = 2 + (ncol_scan[j + 1] - ncol_scan[j] == 2);
}

// warp per general row: emit (pos_col, a) [and (pos_col+1, -a)] in input
// order via a warp prefix sum of the per-entry widths, then the slack entry.
// Lane 0 then applies the bound shifts to b sequentially (lp_core.py:281-283).
__global__ void k_fill_rows(int m, const int* __restrict__ ptr, const int* __restrict__ col,
                            const double* __restrict__ val, const int* __restrict__ pos,
                            const int8_t* __restrict__ sense, const int* __restrict__ ineq_scan,
                            int n_struct, const double* __restrict__ rhs,
                            const double* __restrict__ lower, const int* __restrict__ s_ptr,
                            int* __restrict__ s_col, double* __restrict__ s_val,
                            double* __restrict__ b_std, int* __restrict__ slack_of_row,
                            double* __restrict__ slack_coef, int* __restrict__ bound_var) {
  const long long w = ((long long)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  const int lane = threadIdx.x & 31;
  if (w >= m) return;
  const int s = ptr[w], e = ptr[w + 1];
  int out = s_ptr[w];
  for (int k0 = s; k0 < e; k0 += 32) {
    const int k = k0 + lane;
    int j = 0, width = 0;
    double a = 0.0;
    if (k < e) {
      j = col[k];
      a = val[k];
      width = pos[j + 1] - pos[j];
    }
    int incl = width;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const int t = __shfl_up_sync(0xffffffffu, incl, o);
      if (lane >= o) incl += t;
    }
    if (k < e) {
      const int p = out + incl - width;
      s_col[p] = pos[j];
      s_val[p] = a;
      if (width == 2) {
        s_col[p + 1] = pos[j] + 1;
        s_val[p + 1] = -a;
      }
    }
    out += __shfl_sync(0xffffffffu, incl, 31);
  }
  if (lane == 0) {
    const int8_t sn = sense[w];
    if (sn != PDHG_SENSE_EQ) {
      const double coef = sn == PDHG_SENSE_LE ? 1.0 : -1.0;
      s_col[out] = n_struct + ineq_scan[w];
      s_val[out] = coef;
      slack_of_row[w] = n_struct + ineq_scan[w];
      slack_coef[w] = coef;
    } else {
      slack_of_row[w] = -1;
      slack_coef[w] = 0.0;
    }
    bound_var[w] = -1;
    double bw = rhs[w];
    for (int k = s; k < e; ++k) {
      const double lo = lower[col[k]];
      if (isfinite(lo) && lo != 0.0) bw = __dsub_rn(bw, __dmul_rn(val[k], lo));
    }
    b_std[w] = bw;
  }
}

// thread per general column: column maps, c_std, and its bound row if any
__global__ void k_fill_cols(int m, int n, const double* __restrict__ c, const double* __restrict__ lower,
                            const double* __restrict__ upper, const int* __restrict__ pos,
                            const int* __restrict__ fub_scan, int slack0, const int* __restrict__ s_ptr,
                            int* __restrict__ s_col, double* __restrict__ s_val,
                            double* __restrict__ b_std, double* __restrict__ c_std,
                            double* __restrict__ shifts, int* __restrict__ pos_col,
                            int* __restrict__ neg_col, int* __restrict__ slack_of_row,
                            double* __restrict__ slack_coef, int* __restrict__ bound_var) {
  const int j = blockIdx.x * blockDim.x + threadIdx.x;
  if (j >= n) return;
  const double lo = lower[j];
  const bool fin = isfinite(lo);
  const int p = pos[j];
  const double shift = fin ? lo : 0.0;
  pos_col[j] = p;
  neg_col[j] = fin ? -1 : p + 1;
  shifts[j] = shift;
  c_std[p] = c[j];
  if (!fin) c_std[p + 1] = -c[j];
  if (fub_scan[j + 1] - fub_scan[j]) {
    const int t = fub_scan[j];
    const int r = m + t;
    int q = s_ptr[r];
    s_col[q] = p;
    s_val[q] = 1.0;
    ++q;
    if (!fin) {
      s_col[q] = p + 1;
      s_val[q] = -1.0;
      ++q;
    }
    s_col[q] = slack0 + t;
    s_val[q] = 1.0;
    b_std[r] = __dsub_rn(upper[j], shift);
    slack_of_row[r] = slack0 + t;
    slack_coef[r] = 1.0;
    bound_var[r] = j;
  }
}

}  // namespace

extern "C" {

size_t pdhg_stdform_tmp_bytes(int32_t m, int32_t n) {
  if (m < 0 || n < 0) return 0;
  return a256((size_t)(n + 1) * 4) * 2 + a256((size_t)(m + 1) * 4) + a256((size_t)(m + n + 1) * 4) +
         256 + a256(cub_bytes_for(m + n + 1));
}

int pdhg_stdform_plan(int32_t m, int32_t n, int64_t nnz, const int32_t* ptr, const int32_t* col,
                      const double* val, const int8_t* sense, const double* lower,
                      const double* upper, void* tmp, size_t tmp_bytes, void* stream,
                      pdhg_stdform_dims* out) {
  if (m < 0 || n < 0 || nnz < 0 || !out || !tmp || (m > 0 && (!ptr || !sense)) ||
      (n > 0 && (!lower || !upper)) || (nnz > 0 && (!col || !val)))
    return set_error(PDHG_ERR_ARG, "stdform_plan: bad argument");
  if (tmp_bytes < pdhg_stdform_tmp_bytes(m, n)) return set_error(PDHG_ERR_ARG, "stdform_plan: tmp too small");
  if ((long long)m + n >= INT32_MAX) return set_error(PDHG_ERR_ARG, "stdform_plan: model too large");
  cudaStream_t s = (cudaStream_t)stream;
  Tmp t = carve(tmp, m, n);
  SF_TRY(cudaMemsetAsync(t.flag, 0, 4, s));
  k_colflags<<<nb((long long)n + 1, 256), 256, 0, s>>>(n, lower, upper, t.ncol, t.fub);
  k_rowflags<<<nb((long long)m + 1, 256), 256, 0, s>>>(m, sense, t.ineq);
  int rc = scan(t, t.ncol, n + 1, s);
  if (!rc) rc = scan(t, t.fub, n + 1, s);
  if (!rc) rc = scan(t, t.ineq, m + 1, s);
  if (rc) return rc;
  int h[4] = {0, 0, 0, 0};  // n_struct, n_bound, n_ineq, bad
  SF_TRY(cudaMemcpyAsync(&h[0], t.ncol + n, 4, cudaMemcpyDeviceToHost, s));
  SF_TRY(cudaMemcpyAsync(&h[1], t.fub + n, 4, cudaMemcpyDeviceToHost, s));
  SF_TRY(cudaMemcpyAsync(&h[2], t.ineq + m, 4, cudaMemcpyDeviceToHost, s));
  SF_TRY(cudaStreamSynchronize(s));
  const long long m_std = (long long)m + h[1];
  const long long n_std = (long long)h[0] + h[2] + h[1];
  if (n_std >= INT32_MAX) return set_error(PDHG_ERR_ARG, "stdform_plan: standard form too large");
  if (m > 0)
    k_rowlen<<<nb((long long)m * 32, 256), 256, 0, s>>>(m, ptr, col, val, t.ncol, sense, t.rowlen, t.flag);
  if (n > 0) k_boundlen<<<nb(n, 256), 256, 0, s>>>(m, n, t.ncol, t.fub, t.rowlen);
  SF_TRY(cudaMemsetAsync(t.rowlen + m_std, 0, 4, s));
  rc = scan(t, t.rowlen, (int)m_std + 1, s);
  if (rc) return rc;
  // the last scanned value is the output nnz (int32: CSR of the standard form)
  int nz = 0;
  SF_TRY(cudaMemcpyAsync(&nz, t.rowlen + m_std, 4, cudaMemcpyDeviceToHost, s));
  SF_TRY(cudaMemcpyAsync(&h[3], t.flag, 4, cudaMemcpyDeviceToHost, s));
  SF_TRY(cudaStreamSynchronize(s));
  SF_TRY(cudaGetLastError());
  out->m_std = (int32_t)m_std;
  out->n_std = (int32_t)n_std;
  out->nnz_std = nz;
  out->n_struct = h[0];
  out->n_ineq = h[2];
  out->n_bound = h[1];
  out->nonfinite_entries = h[3];
  return 0;
}

int pdhg_stdform_build(int32_t m, int32_t n, int64_t nnz, const int32_t* ptr, const int32_t* col,
                       const double* val, const int8_t* sense, const double* rhs,
                       const double* lower, const double* upper, const double* c,
                       const pdhg_stdform_dims* dims, void* tmp, size_t tmp_bytes, void* stream,
                       int32_t* s_ptr, int32_t* s_col, double* s_val, double* b_std, double* c_std,
                       double* shifts, int32_t* pos_col, int32_t* neg_col, int32_t* slack_of_row,
                       double* slack_coef, int32_t* bound_var) {
  if (!dims || !tmp || !s_ptr || (dims->nnz_std > 0 && (!s_col || !s_val)) ||
      (dims->m_std > 0 && (!b_std || !slack_of_row || !slack_coef || !bound_var)) ||
      (n > 0 && (!c || !shifts || !pos_col || !neg_col || !c_std)) || (m > 0 && !rhs))
    return set_error(PDHG_ERR_ARG, "stdform_build: bad argument");
  if (tmp_bytes < pdhg_stdform_tmp_bytes(m, n)) return set_error(PDHG_ERR_ARG, "stdform_build: tmp too small");
  cudaStream_t s = (cudaStream_t)stream;
  Tmp t = carve(tmp, m, n);
  SF_TRY(cudaMemcpyAsync(s_ptr, t.rowlen, (size_t)(dims->m_std + 1) * 4, cudaMemcpyDeviceToDevice, s));
  if (dims->n_std > 0) SF_TRY(cudaMemsetAsync(c_std, 0, (size_t)dims->n_std * 8, s));
  if (m > 0)
    k_fill_rows<<<nb((long long)m * 32, 256), 256, 0, s>>>(
        m, ptr, col, val, t.ncol, sense, t.ineq, dims->n_struct, rhs, lower, t.rowlen, s_col, s_val,
        b_std, slack_of_row, slack_coef, bound_var);
  if (n > 0)
    k_fill_cols<<<nb(n, 256), 256, 0, s>>>(m, n, c, lower, upper, t.ncol, t.fub,
                                            dims->n_struct + dims->n_ineq, t.rowlen, s_col, s_val,
                                            b_std, c_std, shifts, pos_col, neg_col, slack_of_row,
                                            slack_coef, bound_var);
  SF_TRY(cudaGetLastError());
  SF_TRY(cudaStreamSynchronize(s));
  return 0;
}

}  // extern "C"
