/* hetermoe.h — C ABI of libhetermoe_kernels.so, the B200 (sm_100a) expert-layer hot path.
 *
 * The reference (zpsim, /root/reference/pkg) has no native layer: every hot-path operator is an
 * opaque duration inside a Task. These entry points are the kernels that the
 * reference's task kinds stand for; each comment names the reference interface it replaces:
 *
 *   ATTN_F  (taskgraph.py:220-246, costmodel.py:19-25)   -> hm_router_topk, hm_dispatch_permute, hm_combine
 *   EXP_F / OFF_EXP_F (costmodel.py:28-37 expert_duration) -> hm_grouped_ffn_fwd
 *   EXP_B / OFF_EXP_B (same, x gamma, taskgraph.py:441-451) -> hm_grouped_ffn_bwd
 *   ATTN_B  (taskgraph.py:476)                            -> hm_combine_bwd, hm_router_bwd / hm_unpermute_sum
 *
 * Conventions:
 *   - every pointer is a DEVICE pointer owned by the caller; the library never allocates;
 *   - bf16 tensors are passed as `const void*` / `void*` (IEEE bfloat16, row-major, contiguous);
 *   - `stream` is a cudaStream_t (NULL = legacy default stream); every call is asynchronous and
 *     stream-ordered, no host synchronisation happens inside;
 *   - return 0 on success, a cudaError_t value on a CUDA error, or an HM_E_* code on a shape /
 *     alignment error; hm_last_error() returns a thread-local message for the last failure;
 *   - calls are reentrant across threads when streams and buffers are distinct.
 */
#ifndef HETERMOE_H_
#define HETERMOE_H_

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define HM_ABI_VERSION 3

#define HM_E_SHAPE 1001     /* unsupported or inconsistent shape */
#define HM_E_ALIGN 1002     /* pointer / stride alignment violated (16 bytes) */
#define HM_E_DRIVER 1003    /* driver entry point (cuTensorMapEncodeTiled) unavailable */
#define HM_E_ARG 1004       /* bad enum / null argument */

/* grouped GEMM modes (see paper_2504_03871_b200/csrc/grouped_gemm.cuh) */
#define HM_GEMM_FWD_UPGATE 0 /* act,h = SwiGLU(A[rows,K] . B[e][N][K]^T)           (N = 2f) */
#define HM_GEMM_FWD_DOWN 1   /* out = A[rows,K] . B[e][N][K]^T                                 */
#define HM_GEMM_BWD_DACT 2   /* dH = SwiGLU'(A[rows,K] . B[e][K][N], h)              (N = f)  */
#define HM_GEMM_BWD_DX 3     /* out = A[rows,K] . B[e][K][N]                                   */
#define HM_GEMM_WGRAD 4      /* out[e][M][N] = A[seg_e, M]^T . B[seg_e, N]   (bf16 out)          */
#define HM_GEMM_WGRAD_ACC 5  /* out[e][M][N] += A[seg_e, M]^T . B[seg_e, N]  (fp32 out, accumulate) */

int hm_abi_version(void);
const char* hm_last_error(void);
/* number of SMs of the current device (grid sizing for max_ctas) */
int hm_num_sms(void);
/* diagnostics: grouped-GEMM cycle accounting gathered when HM_GEMM_STATS=1 (8 counters, see
 * csrc/grouped_gemm.cuh g_gemm_stats); reads and resets them, synchronising the device */
int hm_gemm_stats(unsigned long long* out);

/* ---- K1 router: logits (fixed-order fp32), top-k, softmax over the k, histogram, offsets ----
 * x[T,d] bf16, wg[d,E] bf16, bias[E] fp32 or NULL (logits = x . wg + bias). Outputs: idx[T,k] int32, w[T,k] fp32,
 * logits[T,E] fp32 (required scratch, also a result), counts[E], offsets[E+1] int32,
 * chunk_base[hm_router_chunk_elems(T,E)] int32 (per-chunk row bases, consumed by
 * hm_dispatch_permute; its last element is the fused kernel's completion counter).
 * Requires d % 256 == 0, d <= 16384, 1 <= k <= 8, k <= E <= 256.
 * Replaces: the router/gate folded into ATTN_F (taskgraph.py:220-246). */
int hm_router_topk(const void* x, const void* wg, const float* bias, int T, int d, int E, int k,
                   int32_t* idx, float* w, float* logits, int32_t* counts, int32_t* offsets,
                   int32_t* chunk_base, void* stream);
size_t hm_router_chunk_elems(int T, int E);
/* kernel launches hm_router_topk issues for this shape (1 when logits, top-k, histogram and
 * scan run fused: E <= 8 for d <= 4096), 0 for an unsupported shape or T = 0 */
int hm_router_launches(int T, int d, int E);

/* ---- K2 dispatch permute: x[T,d] -> x_perm[T*k,d] grouped by expert, stable in token order --
 * row_src[T*k] = source token of each permuted row, row_of[T,k] = permuted row of (t, slot).
 * Replaces: the dispatch side of DISP_F (taskgraph.py:244). */
int hm_dispatch_permute(const void* x, const int32_t* idx, const int32_t* chunk_base, int T, int d,
                        int E, int k, void* x_perm, int32_t* row_src, int32_t* row_of,
                        void* stream);
/* dx[t] = sum_s dx_perm[row_of[t,s]] (backward of the permute) */
int hm_unpermute_sum(const void* dx_perm, const int32_t* row_of, int T, int d, int k, void* dx,
                     void* stream);

/* ---- K4 combine: y[t] = sum_s w[t,s] * y_perm[row_of[t,s]] ----
 * Replaces: the combine folded into ATTN_F(l+1) after COMB_F (taskgraph.py:266-283). */
int hm_combine(const void* y_perm, const int32_t* row_of, const float* w, int T, int d, int k,
               void* y, void* stream);
/* dy_perm[row_of[t,s]] = w[t,s] * dy[t];  dw[t,s] = <dy[t], y_perm[row_of[t,s]]> */
int hm_combine_bwd(const void* dy, const void* y_perm, const int32_t* row_of, const float* w,
                   int T, int d, int k, void* dy_perm, float* dw, void* stream);

/* ---- router backward fused with the unpermute-sum ----
 * dlogit = softmax-backward of the k selected weights; dx = unpermute_sum(dx_perm) + dlogit . wg^T;
 * dwg[d,E] (bf16) = sum over tokens of x[t] (x) dlogit_dense[t] (x_perm/offsets from the forward;
 * for E <= 8 each token's row is read once: from x[T,d] (the router input, may be NULL) streamed
 * through shared memory when d % 512 == 0, else from its first routed copy). wg_t = wg
 * transposed ([E,d], see hm_transpose_bf16); part = fp32 workspace of
 * hm_router_bwd_part_elems(T,d,E,k) elements. dwg may be NULL (then x/x_perm/offsets/part unused). */
int hm_router_bwd(const void* dx_perm, const int32_t* row_of, const int32_t* idx, const float* w,
                  const float* dw, const void* x, const void* x_perm, const int32_t* offsets, const void* wg_t,
                  int T, int d, int E, int k, void* dx, float* dlogit, void* dwg, float* part,
                  void* stream);
size_t hm_router_bwd_part_elems(int T, int d, int E, int k);
int hm_transpose_bf16(const void* in, int R, int C, void* out, void* stream);

/* ---- NVLink peer-memory transport (fused compute + dispatch/combine; the DISP and COMB lanes,
 * taskgraph.py:56-59) ----
 * dest_base[E]: device pointers (possibly peer-mapped) of each expert owner's receive buffer;
 * dest_start[E]: first row of THIS sender's rows of expert e in that buffer. Row (t,s) of expert e
 * is written to dest_base[e] + (dest_start[e] + row_of[t,s] - offsets[e]) * d. */
int hm_dispatch_permute_p2p(const void* x, const int32_t* idx, const int32_t* chunk_base,
                            const int32_t* offsets, int T, int d, int E, int k, void* x_perm,
                            int32_t* row_src, int32_t* row_of, const unsigned long long* dest_base,
                            const int32_t* dest_start, void* stream);
/* combine backward whose dy_perm rows go straight to the owners (same addressing); dw local */
int hm_combine_bwd_p2p(const void* dy, const void* y_perm, const int32_t* row_of, const int32_t* idx,
                       const float* w, const int32_t* offsets, int T, int d, int k,
                       const unsigned long long* dest_base, const int32_t* dest_start, float* dw,
                       void* stream);
/* grouped GEMM (HM_GEMM_FWD_DOWN / HM_GEMM_BWD_DX) whose epilogue stores output row r at the
 * device pointer out_rows[r] (local or peer): the expert FFN's last GEMM fused with the return */
int hm_grouped_gemm_rows(int mode, const void* a, const void* b, const int32_t* seg_offsets,
                         int E, int rows, int M, int N, int K, void* out, int ldo, void* out2,
                         int ldo2, const void* aux, int ld_aux, void* workspace,
                         const unsigned long long* out_rows, int max_ctas, void* stream);
/* hm_grouped_gemm_rows whose operands may sit in a pool at a device-computed base (no host sync
 * on the routed row counts): the A tensor map spans a_rows rows (0: rows), and row_shift (device,
 * 8-byte aligned int[2], or NULL) holds {a, o}: rows added to the segment rows of A and of the
 * out / out2 / aux buffers (o must be 0 when out_rows is given). rows bounds the grid (the
 * receive capacity); the tile count comes from seg_offsets on the device. GROUP_M modes only. */
int hm_grouped_gemm_shifted(int mode, const void* a, const void* b, const int32_t* seg_offsets,
                            int E, int rows, int a_rows, int M, int N, int K, void* out, int ldo,
                            void* out2, int ldo2, const void* aux, int ld_aux, void* workspace,
                            const unsigned long long* out_rows, const int32_t* row_shift,
                            int max_ctas, void* stream);
/* ---- device-side receive layout (ZP peer-memory transport, one call per (layer, micro-batch)) ----
 * From the all-gathered expert counts counts_all[M][E] (attention ranks) and the layer's
 * owners[E], on the device, with no host synchronisation:
 *   sender (me < M):   dest_start[E]  first row of my rows of expert e in its owner's expert-major
 *                                     receive slot (experts in id order, senders in rank order)
 *   owner (n_own > 0): seg[n_own+1]   segment offsets of my experts in my receive slot
 *                      out_rows_y/dx[cap]  per received row, the device address of its row in the
 *                                     sender's y slot (y_base[a] + row * row_bytes) / + dx_delta
 *                      shifts[8]      {a, o} row shifts for hm_grouped_gemm_shifted: up+gate
 *                                     {0, f}, down {f, 0}, SwiGLU bwd {0, f}, dX {f, 0}, where
 *                                     f = pool_base + *top is bump-allocated in the layer's pool
 *                                     region of pool_rows rows (*top: device counter, zeroed by the
 *                                     caller before the layer's first micro-batch)
 * A pool or slot overflow ORs 1 / 4 (pool / receive slot) into *err and empties the segments (the
 * GEMMs then skip this micro-batch), an owner id outside [0, 16) ORs 8; the caller checks *err
 * after the step.
 * Replaces the host-side receive layout of the count exchange. */
int hm_zp_layout(const int32_t* counts_all, int M, int E, const int32_t* owners, int me, int n_own,
                 int cap, const unsigned long long* y_base, long long dx_delta, int row_bytes,
                 int32_t* dest_start, int32_t* seg, unsigned long long* out_rows_y,
                 unsigned long long* out_rows_dx, int32_t* shifts, int32_t* top, int pool_base,
                 int pool_rows, int32_t* err, void* stream);
/* after this stream's prior work: atomically add 1 (release, system scope) to n <= 8 counters
 * (host array of device pointers, typically peer-mapped) */
int hm_signal_peers(const unsigned long long* flag_ptrs, int n, void* stream);
/* stall this stream until the local counters flags[i*stride] >= targets[i] (acquire, system) */
int hm_wait_flags(const unsigned int* flags, int stride, const unsigned int* targets, int n,
                  void* stream);

/* ---- K3 grouped expert GEMM (tcgen05 / TMEM / TMA) ----
 * seg_offsets[E+1] (device) delimit each expert's rows of the activation buffers.
 * GROUP_M modes: a = activations [rows, K]; b = per-expert weights ([E][N][K] or [E][K][N]).
 * WGRAD(_ACC): a = [rows, M], b = [rows, N], out = [E][M][N]; needs a 128-byte aligned device
 * workspace of hm_grouped_gemm_workspace_bytes(mode, E) bytes (per-expert TMA views).
 * max_ctas caps the persistent grid (capacity-weight emulation; <= 0 means all SMs). */
int hm_grouped_gemm(int mode, const void* a, const void* b, const int32_t* seg_offsets, int E,
                    int rows, int M, int N, int K, void* out, int ldo, void* out2, int ldo2,
                    const void* aux, int ld_aux, void* workspace, int max_ctas, void* stream);
size_t hm_grouped_gemm_workspace_bytes(int mode, int E);

/* Weight gradient over R segments (micro-batches) at once: out[e] (+)= sum_j A_j[seg_j(e)]^T . B_j[seg_j(e)]
 * a_list/b_list: R host arrays of device pointers ([rows_j, M] and [rows_j, N] bf16); rows_list: R
 * host ints; seg_offsets: device [R][E+1]; out bf16 (accumulate=0) or fp32 (accumulate=1,
 * out += ...). One GEMM whose K loop runs over each expert's rows in every segment, so
 * micro-batched weight gradients are formed once per layer instead of read-modify-written per
 * micro-batch. workspace: hm_grouped_wgrad_multi_workspace_bytes(E, R), 128-byte aligned.
 * R <= 16. Replaces the per-micro-batch part of EXP_B / OFF_EXP_B. */
int hm_grouped_wgrad_multi(int accumulate, const void* const* a_list, const void* const* b_list,
                           const int* rows_list, const int32_t* seg_offsets, int R, int E, int M,
                           int N, void* out, int ldo, void* workspace, int max_ctas,
                           void* stream);
size_t hm_grouped_wgrad_multi_workspace_bytes(int E, int R);
/* hm_grouped_wgrad_multi with per-segment pool bases: rows of A_j / B_j are offset by
 * shift_a[j * shift_stride] / shift_b[j * shift_stride] (device ints, either may be NULL) */
int hm_grouped_wgrad_multi_shifted(int accumulate, const void* const* a_list, const void* const* b_list,
                                   const int* rows_list, const int32_t* seg_offsets, int R, int E, int M,
                                   int N, void* out, int ldo, const int32_t* shift_a,
                                   const int32_t* shift_b, int shift_stride, void* workspace,
                                   int max_ctas, void* stream);

/* SwiGLU expert FFN forward over permuted rows:
 *   h[rows,2f]  = x_perm . w_ug[e]^T   (gate|up interleaved in 128-column blocks, saved for bwd)
 *   act[rows,f] = silu(gate) * up
 *   y_perm[rows,d] = act . w_d[e]^T
 * w_ug: [E][2f][d] (rows 256*j .. +127 = gate f-cols 128*j.., rows +128 .. +255 = up), w_d: [E][d][f].
 * Replaces: expert_duration (costmodel.py:28-37), i.e. the EXP_F / OFF_EXP_F tasks. */
int hm_grouped_ffn_fwd(const void* x_perm, int rows, const int32_t* seg_offsets, int E,
                       const void* w_ug, const void* w_d, int d, int f, void* h, void* act,
                       void* y_perm, int max_ctas, void* stream);
/* backward: dh = SwiGLU'(dy_perm . w_d[e]) (workspace [rows,2f]); dx_perm = dh . w_ug[e];
 * dw_ug[e] = dh_e^T . x_e; dw_d[e] = dy_e^T . act_e. workspace: 2 * hm_grouped_gemm_workspace_bytes(
 * HM_GEMM_WGRAD, E) bytes, 128-byte aligned. Replaces EXP_B / OFF_EXP_B. */
int hm_grouped_ffn_bwd(const void* dy_perm, const void* x_perm, const void* h, const void* act,
                       int rows, const int32_t* seg_offsets, int E, const void* w_ug,
                       const void* w_d, int d, int f, void* dh, void* dx_perm, void* dw_ug,
                       void* dw_d, void* workspace, int max_ctas, void* stream);

#ifdef __cplusplus
}
#endif

#endif /* HETERMOE_H_ */
