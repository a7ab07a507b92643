// baseline/cusparse_spsv.cu -- cuSPARSE SpSV / SpSM (the library's sparse
// triangular solves, one and many right-hand sides) as CONTEXT for bench.py ("cuSPARSE SpSV on the same box
// as context").  Not on the product path: the product is libsptrsv.so.
// The caller passes the CSR of the triangle to solve (opposite-triangle
// entries already removed), device pointers.
#include <cuda_runtime.h>
#include <cusparse.h>
#include <cstdint>

struct SpsvCtx {
    cusparseHandle_t h = nullptr;
    cusparseSpMatDescr_t A = nullptr;
    cusparseDnVecDescr_t X = nullptr, Y = nullptr;
    cusparseSpSVDescr_t d = nullptr;
    void *buf = nullptr;
    cudaDataType t = CUDA_R_64F;
};

extern "C" int spsv_create(int n, int64_t nnz, const int32_t *rowptr, const int32_t *colidx, const void *vals,
                           int upper, int unit, int f32, void *b, void *x, void **out, float *analysis_ms) {
    SpsvCtx *c = new SpsvCtx;
    c->t = f32 ? CUDA_R_32F : CUDA_R_64F;
    if (cusparseCreate(&c->h) != CUSPARSE_STATUS_SUCCESS) return 1;
    if (cusparseCreateCsr(&c->A, n, n, nnz, (void *)rowptr, (void *)colidx, (void *)vals, CUSPARSE_INDEX_32I,
                          CUSPARSE_INDEX_32I, CUSPARSE_INDEX_BASE_ZERO, c->t) != CUSPARSE_STATUS_SUCCESS)
        return 2;
    cusparseFillMode_t fm = upper ? CUSPARSE_FILL_MODE_UPPER : CUSPARSE_FILL_MODE_LOWER;
    cusparseDiagType_t dt = unit ? CUSPARSE_DIAG_TYPE_UNIT : CUSPARSE_DIAG_TYPE_NON_UNIT;
    cusparseSpMatSetAttribute(c->A, CUSPARSE_SPMAT_FILL_MODE, &fm, sizeof(fm));
    cusparseSpMatSetAttribute(c->A, CUSPARSE_SPMAT_DIAG_TYPE, &dt, sizeof(dt));
    cusparseCreateDnVec(&c->X, n, b, c->t);
    cusparseCreateDnVec(&c->Y, n, x, c->t);
    if (cusparseSpSV_createDescr(&c->d) != CUSPARSE_STATUS_SUCCESS) return 3;
    double one = 1.0;
    float onef = 1.0f;
    const void *alpha = f32 ? (const void *)&onef : (const void *)&one;
    size_t bytes = 0;
    if (cusparseSpSV_bufferSize(c->h, CUSPARSE_OPERATION_NON_TRANSPOSE, alpha, c->A, c->X, c->Y, c->t,
                                CUSPARSE_SPSV_ALG_DEFAULT, c->d, &bytes) != CUSPARSE_STATUS_SUCCESS)
        return 4;
    if (cudaMalloc(&c->buf, bytes > 0 ? bytes : 16) != cudaSuccess) return 5;
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0);
    cudaEventCreate(&e1);
    cudaEventRecord(e0, 0);
    if (cusparseSpSV_analysis(c->h, CUSPARSE_OPERATION_NON_TRANSPOSE, alpha, c->A, c->X, c->Y, c->t,
                              CUSPARSE_SPSV_ALG_DEFAULT, c->d, c->buf) != CUSPARSE_STATUS_SUCCESS)
        return 6;
    cudaEventRecord(e1, 0);
    cudaEventSynchronize(e1);
    float ms = 0.f;
    cudaEventElapsedTime(&ms, e0, e1);
    if (analysis_ms) *analysis_ms = ms;
    cudaEventDestroy(e0);
    cudaEventDestroy(e1);
    *out = c;
    return 0;
}

// one solve x = T^{-1} b on `stream` (the b / x given at creation)
extern "C" int spsv_solve(void *ctx, void *stream) {
    SpsvCtx *c = (SpsvCtx *)ctx;
    cusparseSetStream(c->h, (cudaStream_t)stream);
    double one = 1.0;
    float onef = 1.0f;
    const void *alpha = c->t == CUDA_R_32F ? (const void *)&onef : (const void *)&one;
    return cusparseSpSV_solve(c->h, CUSPARSE_OPERATION_NON_TRANSPOSE, alpha, c->A, c->X, c->Y, c->t,
                              CUSPARSE_SPSV_ALG_DEFAULT, c->d) == CUSPARSE_STATUS_SUCCESS ? 0 : 7;
}

extern "C" void spsv_destroy(void *ctx) {
    SpsvCtx *c = (SpsvCtx *)ctx;
    if (!c) return;
    cusparseSpSV_destroyDescr(c->d);
    cusparseDestroyDnVec(c->X);
    cusparseDestroyDnVec(c->Y);
    cusparseDestroySpMat(c->A);
    cusparseDestroy(c->h);
    cudaFree(c->buf);
    delete c;
}

// SpSM: X = T^{-1} B for nrhs right-hand sides, B and X row-major n x nrhs
// (the layout of sptrsv_solve), device pointers
struct SpsmCtx {
    cusparseHandle_t h = nullptr;
    cusparseSpMatDescr_t A = nullptr;
    cusparseDnMatDescr_t B = nullptr, C = nullptr;
    cusparseSpSMDescr_t d = nullptr;
    void *buf = nullptr;
    cudaDataType t = CUDA_R_64F;
};

extern "C" int spsm_create(int n, int64_t nnz, const int32_t *rowptr, const int32_t *colidx, const void *vals,
                           int upper, int unit, int f32, int nrhs, void *b, void *x, void **out, float *analysis_ms) {
    SpsmCtx *c = new SpsmCtx;
    c->t = f32 ? CUDA_R_32F : CUDA_R_64F;
    if (cusparseCreate(&c->h) != CUSPARSE_STATUS_SUCCESS) return 1;
    if (cusparseCreateCsr(&c->A, n, n, nnz, (void *)rowptr, (void *)colidx, (void *)vals, CUSPARSE_INDEX_32I,
                          CUSPARSE_INDEX_32I, CUSPARSE_INDEX_BASE_ZERO, c->t) != CUSPARSE_STATUS_SUCCESS)
        return 2;
    cusparseFillMode_t fm = upper ? CUSPARSE_FILL_MODE_UPPER : CUSPARSE_FILL_MODE_LOWER;
    cusparseDiagType_t dt = unit ? CUSPARSE_DIAG_TYPE_UNIT : CUSPARSE_DIAG_TYPE_NON_UNIT;
    cusparseSpMatSetAttribute(c->A, CUSPARSE_SPMAT_FILL_MODE, &fm, sizeof(fm));
    cusparseSpMatSetAttribute(c->A, CUSPARSE_SPMAT_DIAG_TYPE, &dt, sizeof(dt));
    if (cusparseCreateDnMat(&c->B, n, nrhs, nrhs, b, c->t, CUSPARSE_ORDER_ROW) != CUSPARSE_STATUS_SUCCESS) return 3;
    if (cusparseCreateDnMat(&c->C, n, nrhs, nrhs, x, c->t, CUSPARSE_ORDER_ROW) != CUSPARSE_STATUS_SUCCESS) return 3;
    if (cusparseSpSM_createDescr(&c->d) != CUSPARSE_STATUS_SUCCESS) return 3;
    double one = 1.0;
    float onef = 1.0f;
    const void *alpha = f32 ? (const void *)&onef : (const void *)&one;
    size_t bytes = 0;
    if (cusparseSpSM_bufferSize(c->h, CUSPARSE_OPERATION_NON_TRANSPOSE, CUSPARSE_OPERATION_NON_TRANSPOSE, alpha, c->A,
                                c->B, c->C, c->t, CUSPARSE_SPSM_ALG_DEFAULT, c->d, &bytes) != CUSPARSE_STATUS_SUCCESS)
        return 4;
    if (cudaMalloc(&c->buf, bytes > 0 ? bytes : 16) != cudaSuccess) return 5;
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0);
    cudaEventCreate(&e1);
    cudaEventRecord(e0, 0);
    if (cusparseSpSM_analysis(c->h, CUSPARSE_OPERATION_NON_TRANSPOSE, CUSPARSE_OPERATION_NON_TRANSPOSE, alpha, c->A,
                              c->B, c->C, c->t, CUSPARSE_SPSM_ALG_DEFAULT, c->d, c->buf) != CUSPARSE_STATUS_SUCCESS)
        return 6;
    cudaEventRecord(e1, 0);
    cudaEventSynchronize(e1);
    float ms = 0.f;
    cudaEventElapsedTime(&ms, e0, e1);
    if (analysis_ms) *analysis_ms = ms;
    cudaEventDestroy(e0);
    cudaEventDestroy(e1);
    *out = c;
    return 0;
}

extern "C" int spsm_solve(void *ctx, void *stream) {
    SpsmCtx *c = (SpsmCtx *)ctx;
    cusparseSetStream(c->h, (cudaStream_t)stream);
    double one = 1.0;
    float onef = 1.0f;
    const void *alpha = c->t == CUDA_R_32F ? (const void *)&onef : (const void *)&one;
    return cusparseSpSM_solve(c->h, CUSPARSE_OPERATION_NON_TRANSPOSE, CUSPARSE_OPERATION_NON_TRANSPOSE, alpha, c->A,
                              c->B, c->C, c->t, CUSPARSE_SPSM_ALG_DEFAULT, c->d) == CUSPARSE_STATUS_SUCCESS ? 0 : 7;
}

extern "C" void spsm_destroy(void *ctx) {
    SpsmCtx *c = (SpsmCtx *)ctx;
    if (!c) return;
    cusparseSpSM_destroyDescr(c->d);
    cusparseDestroyDnMat(c->B);
    cusparseDestroyDnMat(c->C);
    cusparseDestroySpMat(c->A);
    cusparseDestroy(c->h);
    cudaFree(c->buf);
    delete c;
}
