// Exact posit-quire GEMM entry points: matmul_quire (proj/src/tensor_ops.cpp:
// 166-185, via matmul :461-487), C[i,j] = round(sum_k A[i,k] * B[k,j]), A and
// B row-major packed codes.  The pipeline itself is in quire_gemm_core.cuh.
#include "quire_gemm_core.cuh"

namespace pnn_b200 {

int quire_gemm_plan(int nbits, int es, int64_t M, int64_t N, int64_t K, int64_t max_kb_per_split,
                    QuireGemmPlan* plan) {
    return plan_quire_gemm(make_fmt(nbits, es), M, N, K, max_kb_per_split, false, plan);
}

int quire_gemm_launch(int nbits, int es, const void* A, const void* B, void* C, int64_t M,
                      int64_t N, int64_t K, int64_t lda, int64_t ldb, int64_t ldc, void* workspace,
                      size_t workspace_bytes, int64_t max_kb_per_split, cudaStream_t st,
                      QuireGemmStats* stats, bool pack_b) {
    GemmArgs g;
    g.pack_b = pack_b;
    g.f = make_fmt(nbits, es);
    g.M = M;
    g.N = N;
    g.K = K;
    g.max_kb_per_split = max_kb_per_split;
    g.row_nar = true;  // every product is in the term set: row/column NaR flags are exact
    g.col_nar = true;
    if (nbits <= 8)
        return run_quire_gemm<uint8_t>(g, FetchRowMajor<uint8_t>{static_cast<const uint8_t*>(A), lda},
                                       FetchColMajor<uint8_t>{static_cast<const uint8_t*>(B), ldb},
                                       out_rowmajor<uint8_t>(C, ldc), workspace, workspace_bytes, st,
                                       stats);
    return run_quire_gemm<uint16_t>(g, FetchRowMajor<uint16_t>{static_cast<const uint16_t*>(A), lda},
                                    FetchColMajor<uint16_t>{static_cast<const uint16_t*>(B), ldb},
                                    out_rowmajor<uint16_t>(C, ldc), workspace, workspace_bytes, st,
                                    stats);
}

}  // namespace pnn_b200
