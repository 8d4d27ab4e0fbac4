// ees_solve.cpp -- the steps either side of the hot path (SURVEY.md §8(f)
// NEXT-4; SPEC.md newton_step): the caller's linear pre-pass
// (ees_stamp_linear) and the sparse solve of A x = b (ees_solver_*), the role
// KLU plays in the paper's NR loop ("Matrix Solve ... KLU";
// P:176 names a GPU sparse solver as the next step).
//
// The solver follows the SPICE pattern of one symbolic analysis per topology
// and one numeric factorisation per NR iteration: at ees_solver_create the
// frozen CSR pattern of the context is ordered (symmetric approximate
// minimum degree of A + A^T), factorised once on the host with partial
// pivoting (threshold 1.0) at the caller's values, and the ordering, pivots
// and the L/U patterns are handed to cusolverRf; every ees_solver_factor
// then refactorises on the GPU with those pivots (values only), and
// ees_solver_solve runs the two triangular solves on the GPU.  A library
// solve (cuSOLVER) -- the hot path itself is in ees_kernels.cu.
// cuSOLVER marks its host LU and refactorisation "deprecated: use cuDSS";
// cuDSS is not in this image, so these are the library path.
#pragma GCC diagnostic ignored "-Wdeprecated-declarations"
#include <cuda_runtime.h>
#include <cusolverRf.h>
#include <cusolverSp.h>
#include <cusolverSp_LOWLEVEL_PREVIEW.h>
#include <cusparse.h>

#include <algorithm>
#include <cstring>
#include <new>
#include <vector>

#include "ees_internal.h"

struct ees_solver {
    int32_t n = 0, nnz = 0;
    int *d_rp = nullptr, *d_ci = nullptr, *d_P = nullptr, *d_Q = nullptr;
    double *d_T = nullptr;           // cusolverRf workspace [n]
    cusolverRfHandle_t rf = nullptr;
    cudaEvent_t ev_in = nullptr, ev_out = nullptr;
    int64_t nnz_L = 0, nnz_U = 0;
};

namespace {

void solver_free(ees_solver *s)
{
    if (!s) return;
    if (s->rf) cusolverRfDestroy(s->rf);
    cudaFree(s->d_rp);
    cudaFree(s->d_ci);
    cudaFree(s->d_P);
    cudaFree(s->d_Q);
    cudaFree(s->d_T);
    if (s->ev_in) cudaEventDestroy(s->ev_in);
    if (s->ev_out) cudaEventDestroy(s->ev_out);
    delete s;
}

// cusolverRf runs on the legacy default stream: order it after the caller's
// stream (ev_in) and the caller's stream after it (ev_out), no host sync.
cudaError_t enter_legacy(ees_solver *s, cudaStream_t st)
{
    cudaError_t e = cudaEventRecord(s->ev_in, st);
    return e == cudaSuccess ? cudaStreamWaitEvent(cudaStreamLegacy, s->ev_in, 0) : e;
}

cudaError_t leave_legacy(ees_solver *s, cudaStream_t st)
{
    cudaError_t e = cudaEventRecord(s->ev_out, cudaStreamLegacy);
    return e == cudaSuccess ? cudaStreamWaitEvent(st, s->ev_out, 0) : e;
}

__global__ void k_stamp_linear(double *A, const int64_t *slot, const double *val, int64_t n_a, double *b,
                               const int32_t *row, const double *bval, int64_t n_b)
{
    const int64_t T = (int64_t)gridDim.x * blockDim.x;
    for (int64_t k = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; k < n_a + n_b; k += T) {
        if (k < n_a) atomicAdd(A + slot[k], val[k]);
        else atomicAdd(b + row[k - n_a], bval[k - n_a]);
    }
}

}  // namespace

extern "C" {

ees_status ees_stamp_linear(const ees_ctx *ctx, int64_t n_a, const int64_t *slot, const double *val, int64_t n_b,
                            const int32_t *row, const double *bval, double *A_vals, double *b, ees_stream stream)
{
    if (!ctx || n_a < 0 || n_b < 0) return EES_EINVAL;
    if ((n_a && (!slot || !val || !A_vals)) || (n_b && (!row || !bval || !b))) return EES_EINVAL;
    if (n_a + n_b == 0) return EES_OK;
    const int64_t blocks = std::min<int64_t>((n_a + n_b + 255) / 256, 148 * 8);
    k_stamp_linear<<<(unsigned)blocks, 256, 0, (cudaStream_t)stream>>>(A_vals, slot, val, n_a, b, row, bval, n_b);
    return cudaPeekAtLastError() == cudaSuccess ? EES_OK : EES_ECUDA;
}

ees_status ees_solver_create(const ees_ctx *ctx, const double *A_vals_host, ees_solver **out)
{
    if (!ctx || !A_vals_host || !out) return EES_EINVAL;
    *out = nullptr;
    int32_t n = 0;
    int64_t nnz64 = 0;
    const int32_t *rp = nullptr, *ci = nullptr;
    ees_status st = ees_pattern(ctx, &n, &nnz64, &rp, &ci);
    if (st != EES_OK) return st;
    if (n <= 0 || nnz64 <= 0 || nnz64 > INT32_MAX) return EES_EINVAL;
    const int nnz = (int)nnz64;
    ees_solver *s = new (std::nothrow) ees_solver();
    if (!s) return EES_ENOMEM;
    s->n = n;
    s->nnz = nnz;
    cusolverSpHandle_t sp = nullptr;
    cusparseMatDescr_t dA = nullptr, dL = nullptr, dU = nullptr;
    csrluInfoHost_t info = nullptr;
    ees_status rc = EES_OK;
    try {
        std::vector<int> h_rp(rp, rp + n + 1), h_ci(ci, ci + nnz);
        std::vector<double> h_val(A_vals_host, A_vals_host + nnz);
        if (cusolverSpCreate(&sp) != CUSOLVER_STATUS_SUCCESS || cusparseCreateMatDescr(&dA) != CUSPARSE_STATUS_SUCCESS ||
            cusparseCreateMatDescr(&dL) != CUSPARSE_STATUS_SUCCESS || cusparseCreateMatDescr(&dU) != CUSPARSE_STATUS_SUCCESS)
            throw EES_ECUDA;
        cusparseSetMatType(dA, CUSPARSE_MATRIX_TYPE_GENERAL);
        cusparseSetMatIndexBase(dA, CUSPARSE_INDEX_BASE_ZERO);
        cusparseSetMatType(dL, CUSPARSE_MATRIX_TYPE_GENERAL);
        cusparseSetMatIndexBase(dL, CUSPARSE_INDEX_BASE_ZERO);
        cusparseSetMatFillMode(dL, CUSPARSE_FILL_MODE_LOWER);
        cusparseSetMatDiagType(dL, CUSPARSE_DIAG_TYPE_UNIT);
        cusparseSetMatType(dU, CUSPARSE_MATRIX_TYPE_GENERAL);
        cusparseSetMatIndexBase(dU, CUSPARSE_INDEX_BASE_ZERO);
        cusparseSetMatFillMode(dU, CUSPARSE_FILL_MODE_UPPER);
        cusparseSetMatDiagType(dU, CUSPARSE_DIAG_TYPE_NON_UNIT);
        // fill-reducing symmetric ordering q, then B = A(q, q)
        std::vector<int> q(n), map(nnz);
        if (cusolverSpXcsrsymamdHost(sp, n, nnz, dA, h_rp.data(), h_ci.data(), q.data()) != CUSOLVER_STATUS_SUCCESS)
            throw EES_ECUDA;
        std::vector<int> b_rp(h_rp), b_ci(h_ci);
        for (int k = 0; k < nnz; k++) map[k] = k;
        size_t pbytes = 0;
        if (cusolverSpXcsrperm_bufferSizeHost(sp, n, n, nnz, dA, b_rp.data(), b_ci.data(), q.data(), q.data(),
                                              &pbytes) != CUSOLVER_STATUS_SUCCESS)
            throw EES_ECUDA;
        std::vector<char> pbuf(pbytes + 1);
        if (cusolverSpXcsrpermHost(sp, n, n, nnz, dA, b_rp.data(), b_ci.data(), q.data(), q.data(), map.data(),
                                   pbuf.data()) != CUSOLVER_STATUS_SUCCESS)
            throw EES_ECUDA;
        std::vector<double> b_val(nnz);
        for (int k = 0; k < nnz; k++) b_val[k] = h_val[map[k]];
        // host LU of B with partial pivoting
        if (cusolverSpCreateCsrluInfoHost(&info) != CUSOLVER_STATUS_SUCCESS) throw EES_ECUDA;
        if (cusolverSpXcsrluAnalysisHost(sp, n, nnz, dA, b_rp.data(), b_ci.data(), info) != CUSOLVER_STATUS_SUCCESS)
            throw EES_ECUDA;
        size_t internal = 0, work = 0;
        if (cusolverSpDcsrluBufferInfoHost(sp, n, nnz, dA, b_val.data(), b_rp.data(), b_ci.data(), info, &internal,
                                           &work) != CUSOLVER_STATUS_SUCCESS)
            throw EES_ECUDA;
        std::vector<char> wbuf(work + 1);
        if (cusolverSpDcsrluFactorHost(sp, n, nnz, dA, b_val.data(), b_rp.data(), b_ci.data(), info, 1.0,
                                       wbuf.data()) != CUSOLVER_STATUS_SUCCESS)
            throw EES_ECUDA;
        int singular = -1;
        if (cusolverSpDcsrluZeroPivotHost(sp, info, 1e-300, &singular) != CUSOLVER_STATUS_SUCCESS) throw EES_ECUDA;
        if (singular >= 0) throw EES_EINVAL;                   // structurally or numerically singular
        int nL = 0, nU = 0;
        if (cusolverSpXcsrluNnzHost(sp, &nL, &nU, info) != CUSOLVER_STATUS_SUCCESS) throw EES_ECUDA;
        std::vector<int> Plu(n), Qlu(n), L_rp(n + 1), L_ci(std::max(1, nL)), U_rp(n + 1), U_ci(std::max(1, nU));
        std::vector<double> L_val(std::max(1, nL)), U_val(std::max(1, nU));
        if (cusolverSpDcsrluExtractHost(sp, Plu.data(), Qlu.data(), dL, L_val.data(), L_rp.data(), L_ci.data(), dU,
                                        U_val.data(), U_rp.data(), U_ci.data(), info, wbuf.data()) !=
            CUSOLVER_STATUS_SUCCESS)
            throw EES_ECUDA;
        s->nnz_L = nL;
        s->nnz_U = nU;
        // P A Q^T = L U with P = Plu o q, Q = Qlu o q
        std::vector<int> P(n), Q(n);
        for (int j = 0; j < n; j++) {
            P[j] = q[Plu[j]];
            Q[j] = q[Qlu[j]];
        }
        if (cusolverRfCreate(&s->rf) != CUSOLVER_STATUS_SUCCESS) throw EES_ECUDA;
        if (cusolverRfSetMatrixFormat(s->rf, CUSOLVERRF_MATRIX_FORMAT_CSR, CUSOLVERRF_UNIT_DIAGONAL_ASSUMED_L) !=
                CUSOLVER_STATUS_SUCCESS ||
            cusolverRfSetResetValuesFastMode(s->rf, CUSOLVERRF_RESET_VALUES_FAST_MODE_ON) != CUSOLVER_STATUS_SUCCESS ||
            cusolverRfSetNumericProperties(s->rf, 0.0, 0.0) != CUSOLVER_STATUS_SUCCESS)
            throw EES_ECUDA;
        if (cusolverRfSetupHost(n, nnz, h_rp.data(), h_ci.data(), h_val.data(), nL, L_rp.data(), L_ci.data(),
                                L_val.data(), nU, U_rp.data(), U_ci.data(), U_val.data(), P.data(), Q.data(),
                                s->rf) != CUSOLVER_STATUS_SUCCESS)
            throw EES_ECUDA;
        if (cudaDeviceSynchronize() != cudaSuccess) throw EES_ECUDA;
        if (cusolverRfAnalyze(s->rf) != CUSOLVER_STATUS_SUCCESS) throw EES_ECUDA;
        auto up = [&](int **d, const std::vector<int> &v) {
            if (cudaMalloc(d, sizeof(int) * v.size()) != cudaSuccess) throw EES_ENOMEM;
            if (cudaMemcpy(*d, v.data(), sizeof(int) * v.size(), cudaMemcpyHostToDevice) != cudaSuccess)
                throw EES_ECUDA;
        };
        up(&s->d_rp, h_rp);
        up(&s->d_ci, h_ci);
        up(&s->d_P, P);
        up(&s->d_Q, Q);
        if (cudaMalloc(&s->d_T, sizeof(double) * (size_t)n) != cudaSuccess) throw EES_ENOMEM;
        if (cudaEventCreateWithFlags(&s->ev_in, cudaEventDisableTiming) != cudaSuccess ||
            cudaEventCreateWithFlags(&s->ev_out, cudaEventDisableTiming) != cudaSuccess)
            throw EES_ECUDA;
    } catch (ees_status e) {
        rc = e;
    } catch (const std::bad_alloc &) {
        rc = EES_ENOMEM;
    }
    if (info) cusolverSpDestroyCsrluInfoHost(info);
    if (dA) cusparseDestroyMatDescr(dA);
    if (dL) cusparseDestroyMatDescr(dL);
    if (dU) cusparseDestroyMatDescr(dU);
    if (sp) cusolverSpDestroy(sp);
    if (rc != EES_OK) {
        cudaGetLastError();
        solver_free(s);
        return rc;
    }
    *out = s;
    return EES_OK;
}

ees_status ees_solver_factor(ees_solver *s, const double *A_vals, ees_stream stream)
{
    if (!s || !A_vals) return EES_EINVAL;
    cudaStream_t st = (cudaStream_t)stream;
    if (enter_legacy(s, st) != cudaSuccess) return EES_ECUDA;
    if (cusolverRfResetValues(s->n, s->nnz, s->d_rp, s->d_ci, const_cast<double *>(A_vals), s->d_P, s->d_Q, s->rf) !=
        CUSOLVER_STATUS_SUCCESS)
        return EES_ECUDA;
    const cusolverStatus_t r = cusolverRfRefactor(s->rf);
    if (r == CUSOLVER_STATUS_ZERO_PIVOT) return EES_EINVAL;
    if (r != CUSOLVER_STATUS_SUCCESS) return EES_ECUDA;
    return leave_legacy(s, st) == cudaSuccess ? EES_OK : EES_ECUDA;
}

ees_status ees_solver_solve(ees_solver *s, const double *b, double *x, ees_stream stream)
{
    if (!s || !b || !x) return EES_EINVAL;
    cudaStream_t st = (cudaStream_t)stream;
    if (b != x && cudaMemcpyAsync(x, b, sizeof(double) * (size_t)s->n, cudaMemcpyDeviceToDevice, st) != cudaSuccess)
        return EES_ECUDA;
    if (enter_legacy(s, st) != cudaSuccess) return EES_ECUDA;
    if (cusolverRfSolve(s->rf, s->d_P, s->d_Q, 1, s->d_T, s->n, x, s->n) != CUSOLVER_STATUS_SUCCESS) return EES_ECUDA;
    return leave_legacy(s, st) == cudaSuccess ? EES_OK : EES_ECUDA;
}

ees_status ees_solver_info(const ees_solver *s, int64_t *nnz_L, int64_t *nnz_U)
{
    if (!s) return EES_EINVAL;
    if (nnz_L) *nnz_L = s->nnz_L;
    if (nnz_U) *nnz_U = s->nnz_U;
    return EES_OK;
}

ees_status ees_solver_destroy(ees_solver *s)
{
    if (!s) return EES_EINVAL;
    cudaDeviceSynchronize();
    solver_free(s);
    return EES_OK;
}

}  // extern "C"
