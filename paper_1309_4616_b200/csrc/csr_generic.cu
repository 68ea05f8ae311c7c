// CSR row applies for every dtype combination of the reference's kernel
// module (_core.pyx:281-315 csr_fused_rows): int32 or int64 column indices x
// {f64 vals / f64 x, f32 / f32, f64 / c128, c128 / c128}.
//
// The int32 f64 and complex forms route to the tuned kernels of csr.cu; the
// int64 and float32 forms are the protocol's rare cases (matrices with more
// than 2^31-1 columns, float fields) and run one thread per row here,
// accumulating strictly in storage order with the reference's expression
// tree (acc = acc + vals[k] * x[col[k]]; y = alpha acc [+ beta x[r]]) in the
// reference's precision -- float arithmetic for float data, like the
// compiled core's fused `_csr_same[.., float]` instantiation.
#include "es_common.cuh"
#include "es_host.h"

namespace es {
namespace {

ES_DEV float fadd(float a, float b) { return __fadd_rn(a, b); }
ES_DEV float fmul(float a, float b) { return __fmul_rn(a, b); }

constexpr int GEN_T = 256;

template <typename I>
__global__ void __launch_bounds__(GEN_T) k_csr_rows_f64(int64_t row_lo, int64_t row_hi, const int64_t *__restrict__ rp,
                                                        const I *__restrict__ col, const double *__restrict__ vals,
                                                        const double *__restrict__ x, double *__restrict__ y,
                                                        double alpha, double beta, int use_beta) {
    const int64_t r = row_lo + (int64_t)blockIdx.x * GEN_T + threadIdx.x;
    if (r >= row_hi) return;
    double acc = 0.0;
    for (int64_t k = __ldg(rp + r), e = __ldg(rp + r + 1); k < e; ++k)
        acc = add(acc, mul(__ldg(vals + k), __ldg(x + (int64_t)__ldg(col + k))));
    y[r] = use_beta ? add(mul(alpha, acc), mul(beta, __ldg(x + r))) : mul(alpha, acc);
}

template <typename I>
__global__ void __launch_bounds__(GEN_T) k_csr_rows_f32(int64_t row_lo, int64_t row_hi, const int64_t *__restrict__ rp,
                                                        const I *__restrict__ col, const float *__restrict__ vals,
                                                        const float *__restrict__ x, float *__restrict__ y,
                                                        float alpha, float beta, int use_beta) {
    const int64_t r = row_lo + (int64_t)blockIdx.x * GEN_T + threadIdx.x;
    if (r >= row_hi) return;
    float acc = 0.0f;
    for (int64_t k = __ldg(rp + r), e = __ldg(rp + r + 1); k < e; ++k)
        acc = fadd(acc, fmul(__ldg(vals + k), __ldg(x + (int64_t)__ldg(col + k))));
    y[r] = use_beta ? fadd(fmul(alpha, acc), fmul(beta, __ldg(x + r))) : fmul(alpha, acc);
}

// complex: the compiled core's C99 complex product (cmul_c, csr.cu), real
// values promoted to (v, 0) as Cython does
template <typename I, bool VC>
__global__ void __launch_bounds__(GEN_T) k_csr_rows_z64(int64_t row_lo, int64_t row_hi, const int64_t *__restrict__ rp,
                                                        const I *__restrict__ col, const double *__restrict__ vals,
                                                        const double2 *__restrict__ x, double2 *__restrict__ y,
                                                        double ar, double ai, double br, double bi, int use_beta) {
    const int64_t r = row_lo + (int64_t)blockIdx.x * GEN_T + threadIdx.x;
    if (r >= row_hi) return;
    double2 acc = make_double2(0.0, 0.0);
    for (int64_t k = __ldg(rp + r), e = __ldg(rp + r + 1); k < e; ++k) {
        const double2 v = VC ? __ldg(reinterpret_cast<const double2 *>(vals) + k) : make_double2(__ldg(vals + k), 0.0);
        const double2 xv = __ldg(x + (int64_t)__ldg(col + k));
        const double2 t = cmul_c(v.x, v.y, xv.x, xv.y);
        acc = make_double2(add(acc.x, t.x), add(acc.y, t.y));
    }
    double2 out = cmul_c(ar, ai, acc.x, acc.y);
    if (use_beta) {
        const double2 xr = __ldg(x + r);
        const double2 t = cmul_c(br, bi, xr.x, xr.y);
        out = make_double2(add(out.x, t.x), add(out.y, t.y));
    }
    y[r] = out;
}

template <typename I>
int launch_generic(int64_t lo, int64_t hi, const int64_t *rp, const void *col, const void *vals, int vk,
                   const void *x, void *y, int xk, double ar, double ai, double br, double bi, int use_beta,
                   cudaStream_t s) {
    const unsigned grid = (unsigned)((hi - lo + GEN_T - 1) / GEN_T);
    const I *c = static_cast<const I *>(col);
    if (vk == ES_KIND_F64 && xk == ES_KIND_F64) {
        k_csr_rows_f64<I><<<grid, GEN_T, 0, s>>>(lo, hi, rp, c, static_cast<const double *>(vals),
                                                 static_cast<const double *>(x), static_cast<double *>(y), ar, br,
                                                 use_beta);
    } else if (vk == ES_KIND_F32 && xk == ES_KIND_F32) {
        k_csr_rows_f32<I><<<grid, GEN_T, 0, s>>>(lo, hi, rp, c, static_cast<const float *>(vals),
                                                 static_cast<const float *>(x), static_cast<float *>(y), (float)ar,
                                                 (float)br, use_beta);
    } else if (xk == ES_KIND_C128 && (vk == ES_KIND_F64 || vk == ES_KIND_C128)) {
        const double2 *xz = static_cast<const double2 *>(x);
        double2 *yz = static_cast<double2 *>(y);
        if (vk == ES_KIND_C128)
            k_csr_rows_z64<I, true><<<grid, GEN_T, 0, s>>>(lo, hi, rp, c, static_cast<const double *>(vals), xz, yz,
                                                            ar, ai, br, bi, use_beta);
        else
            k_csr_rows_z64<I, false><<<grid, GEN_T, 0, s>>>(lo, hi, rp, c, static_cast<const double *>(vals), xz,
                                                             yz, ar, ai, br, bi, use_beta);
    } else {
        return set_error(ES_ERR_TYPE, "CSR kernel does not support vals kind %d with x kind %d", vk, xk);
    }
    return check_launch("csr rows (generic)");
}

}  // namespace
}  // namespace es

using namespace es;

extern "C" int es_csr_fused_rows_ex(int64_t row_lo, int64_t row_hi, const int64_t *row_ptr, const void *col_idx,
                                    int32_t col_bytes, const void *vals, int32_t vals_kind, const void *x, void *y,
                                    int32_t x_kind, double alpha_re, double alpha_im, double beta_re, double beta_im,
                                    int32_t use_beta, void *stream) {
    if (row_lo < 0 || row_hi < row_lo) return set_error(ES_ERR_ARG, "bad row range");
    if (col_bytes != 4 && col_bytes != 8) return set_error(ES_ERR_TYPE, "column indices must be int32 or int64");
    const bool ok_kinds = (vals_kind == ES_KIND_F64 && x_kind == ES_KIND_F64) ||
                          (vals_kind == ES_KIND_F32 && x_kind == ES_KIND_F32) ||
                          (x_kind == ES_KIND_C128 && (vals_kind == ES_KIND_F64 || vals_kind == ES_KIND_C128));
    if (!ok_kinds)
        return set_error(ES_ERR_TYPE, "CSR kernel does not support vals kind %d with x kind %d", vals_kind, x_kind);
    if (row_hi == row_lo) return ES_OK;
    if (!row_ptr || !col_idx || !vals || !x || !y) return set_error(ES_ERR_ARG, "null pointer");
    cudaStream_t s = (cudaStream_t)stream;
    if (col_bytes == 4) {
        const int32_t *c = static_cast<const int32_t *>(col_idx);
        if (vals_kind == ES_KIND_F64 && x_kind == ES_KIND_F64)
            return launch_csr_rows(row_lo, row_hi, row_ptr, c, static_cast<const double *>(vals),
                                   static_cast<const double *>(x), static_cast<double *>(y), alpha_re, beta_re,
                                   use_beta, s);
        if (x_kind == ES_KIND_C128)
            return launch_csr_rows_z(row_lo, row_hi, row_ptr, c, static_cast<const double *>(vals),
                                     vals_kind == ES_KIND_C128, static_cast<const double *>(x), static_cast<double *>(y),
                                     alpha_re, alpha_im, beta_re, beta_im, use_beta, s);
        return launch_generic<int32_t>(row_lo, row_hi, row_ptr, col_idx, vals, vals_kind, x, y, x_kind, alpha_re,
                                       alpha_im, beta_re, beta_im, use_beta, s);
    }
    return launch_generic<int64_t>(row_lo, row_hi, row_ptr, col_idx, vals, vals_kind, x, y, x_kind, alpha_re,
                                   alpha_im, beta_re, beta_im, use_beta, s);
}
