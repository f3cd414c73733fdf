// Internal host interface of the tcgen05 quire GEMM (see quire_gemm.cu).
#pragma once

#include <cuda_runtime.h>

#include <cstddef>
#include <cstdint>

namespace pnn_b200 {

struct QuireGemmPlan {
    int D, NT, KB;
    int64_t mtiles, ntiles, kbt, kb_per_split, splits;
    size_t a_img_bytes, b_img_bytes, row_nar_bytes, col_nar_bytes, partial_bytes;
    size_t off_a, off_b, off_row_nar, off_col_nar, off_flags, off_glut, off_partial, workspace_bytes;
    int smem_bytes;
    int pair;               // 1: CTA-pair (cta_group::2) kernel
    int64_t mtiles_alloc;   // A image m-tiles (even in pair mode)
};

// Optional per-phase CUDA events (pack start, pack end / GEMM start, GEMM end,
// finalize end) recorded on the launch stream.
struct QuireGemmStats {
    cudaEvent_t ev[4];
};

// 0 ok, 2 unsupported format.  max_kb_per_split <= 0: only the exactness limit.
int quire_gemm_plan(int nbits, int es, int64_t M, int64_t N, int64_t K, int64_t max_kb_per_split,
                    QuireGemmPlan* plan);

// A (M x K, lda), B (K x N, ldb), C (M x N, ldc): device pointers to packed
// codes (uint8 for nbits <= 8, else uint16).  0 ok, 2 unsupported format,
// 3 workspace too small, 4 CUDA launch error.  pack_b = false reuses B's
// digit image and NaR flags left in the workspace by an earlier launch of the
// same B whose plan had the same workspace layout (row panels of one GEMM).
int quire_gemm_launch(int nbits, int es, const void* A, const void* B, void* C, int64_t M,
                      int64_t N, int64_t K, int64_t lda, int64_t ldb, int64_t ldc, void* workspace,
                      size_t workspace_bytes, int64_t max_kb_per_split, cudaStream_t st,
                      QuireGemmStats* stats, bool pack_b = true);

}  // namespace pnn_b200
