/*
 * b200moe -- C ABI of the B200-native E8T2 MoE layer.
 *
 * The reference (`moefold`, a numpy package) has no FFI: its "plugin
 * interface" is the Python module API of moefold/moe.py, moefold/upcycle.py and
 * moefold/tensor.py:503 (importance_penalty).  Each entry point below replaces
 * the numpy work behind one of those functions; the host package
 * `paper_2412_09952_b200` binds them with ctypes and keeps
 * the reference's Python signatures on top.
 *
 * Conventions
 *  - Every pointer is a DEVICE pointer unless named *_host.  No function
 *    allocates: outputs and workspaces are caller-owned (PyTorch's allocator).
 *  - All work is enqueued on `stream`; nothing synchronises the host.  The
 *    state a call leaves for the next one lives on the device (the dispatch
 *    scan's epoch word, the router-wgrad tickets, segment counts read by the
 *    GEMMs), so a sequence of calls can be recorded into a CUDA graph and
 *    replayed (paper_2412_09952_b200/graphs.py does this for a layer step).
 *  - bf16 tensors are passed as `void*` (row-major, contiguous).
 *  - Return 0 on success or a negative B200MOE_ERR_* code; the message is in
 *    b200moe_last_error() (thread-local).  Codes map to the reference's
 *    exception classes (moefold/errors.py:12-25): SHAPE -> ShapeError,
 *    CONFIG -> ConfigError, GATE -> GateError, CUDA -> RuntimeError.
 *  - Device-side gate errors (a token row with no finite kept logit,
 *    moefold/tensor.py:283-284) are reported through `err_flag` (int32, set to
 *    1), checked by the host when routing statistics are materialised.
 *
 * Layouts
 *  - x, dx:              [T, H] bf16
 *  - W_g, W_noise:       [H, E] fp32 (reference [in, out] layout, moe.py:133,143)
 *  - logits, gates, probs, noise_act, z, dg, dh, dn: [T, E] fp32
 *  - slot_rank:          [T, E] int32: rank of token t among the kept tokens of
 *                        expert e in token order, -1 if (t, e) is not kept
 *  - expert segments:    permuted activations are grouped by expert; segment s
 *                        starts at row seg_base[s], holds seg_count[s] rows and
 *                        is zero-padded to a multiple of 128 rows.
 *  - expert weights:     W1, W3 [E_local, F, H], W2 [E_local, H, F] bf16
 *                        (= the reference's w1 [H,F], w2 [F,H], w3 [H,F] of each
 *                        expert, transposed; upcycle_copy produces them).
 */
#ifndef B200MOE_H
#define B200MOE_H

#include <stdint.h>
#include <cuda_runtime.h>

#ifdef __cplusplus
extern "C" {
#endif

#define B200MOE_OK 0
#define B200MOE_ERR_SHAPE (-1)
#define B200MOE_ERR_CONFIG (-2)
#define B200MOE_ERR_GATE (-3)
#define B200MOE_ERR_CUDA (-4)

#define B200MOE_ROUTER_MIXTRAL 0 /* moe.py:171 gate_mixtral */
#define B200MOE_ROUTER_ST 1      /* moe.py:176 gate_st */
#define B200MOE_POLICY_POSITION 0
#define B200MOE_POLICY_SCORE 1
#define B200MOE_LAYOUT_COMPACT 0 /* seg_base = prefix of round_up(count,128) */
#define B200MOE_LAYOUT_FIXED 1   /* seg_base[e] = e * seg_stride (EP send buffers) */

const char* b200moe_last_error(void);
int b200moe_version(void);

/* Router forward (K1).  Replaces moe.py:136-149 router_logits + moe.py:152-186
 * top_k_mask / gate_mixtral / gate_st + tensor.py:267-297 softmax.
 * h = x.W_g (+ z * softplus(x.W_noise) when z != NULL).  gates are bit-exact
 * with numpy float32 given the same logits.  probs (router_type st): full
 * softmax s; may be NULL for mixtral.  noise_act = x.W_noise (needed by the
 * backward; NULL when z == NULL).  err_flag (nullable): set to 1 on a GateError
 * row (callers of the layer read it from the dispatch stats instead).
 * E <= 16 and H % 64 == 0 run on the tensor cores (x . W with W split into
 * three bf16 parts, fp32 accumulation); otherwise on the CUDA cores.
 * workspace: b200moe_router_workspace_floats(H, E) floats; on return
 * it holds the swizzled W_g (and W_noise) tables b200moe_router_bwd can reuse. */
int b200moe_router_fwd(const void* x, const float* w_g, const float* w_noise, const float* z, int T, int H, int E,
                       int k, int router_type, float* logits, float* gates, float* probs, float* noise_act,
                       float* workspace, int32_t* err_flag, cudaStream_t stream);

size_t b200moe_router_workspace_floats(int H, int E);
int b200moe_router_set_fma(int on);   /* diagnostics (thread-local): 1 = CUDA-core K1 even where tcgen05 applies */

/* Gating only, from given fp32 logits (moe.py:152-186).  Used to check the
 * device gate arithmetic against the reference's own gates bit-for-bit.
 * topk_mask (uint8 [T,E], nullable) = top_k_mask(logits, k) (moe.py:152). */
int b200moe_gate_from_logits(const float* logits, int T, int E, int k, int router_type, float* gates, float* probs,
                             uint8_t* topk_mask, int32_t* err_flag, cudaStream_t stream);

/* Backward of the standalone gate functions (moe.py:171-186 through the
 * softmax closure tensor.py:292-295, and the st mask product moe.py:186):
 * dh = softmax'(dgates) over the kept k (mixtral) or over all E with the
 * top-k mask (st, probs = full softmax).  gates/probs from
 * b200moe_gate_from_logits. */
int b200moe_gate_bwd(const float* dgates, const float* gates, const float* probs, int T, int E, int router_type,
                     float* dh, cudaStream_t stream);

/* Backward of the standalone router_logits (moe.py:136-149 through the
 * matmul/softplus closures tensor.py:192-207, 220-227): given dh = dL/dlogits,
 * dn = dh*z*sigmoid(noise_act) (noise only), dx = dh.W_g^T + dn.W_noise^T
 * (bf16, NULL to skip), dW_g = x^T dh, dW_noise = x^T dn (fp32, NULL to skip).
 * workspace: >= 2*H*32 + ceil(T/64)*H*E floats. */
int b200moe_router_logits_bwd(const void* x, const float* dh, const float* w_g, const float* w_noise, const float* z,
                              const float* noise_act, int T, int H, int E, void* dx, float* dw_g, float* dw_noise,
                              float* dn, float* workspace, cudaStream_t stream);

/* Capacity + dispatch (K1b).  Replaces moe.py:189-240 (expert_capacity is
 * evaluated by the host; capacity < 0 means dropless).  A slot exists iff
 * gate > 0; `position` keeps the earliest tokens, `score` the largest gates
 * (stable, position breaks ties).  Outputs slot_rank [T,E], counts [E]
 * (= RoutingStats.assigned), seg_base [E], gate_mass [E] (sum of kept gates),
 * importance [E] (sum of all gates, the aux-loss input), stats[3] =
 * {dropped, total_slots, gate_error} (int64; gate_error = 1 if some token row
 * has no positive gate, i.e. the router hit an all-masked softmax row).  importance_loss (nullable, [1] fp32): the
 * importance penalty var/mean^2 of `importance` (tensor.py:503-521), with
 * importance_err (nullable int32) set when mean <= 0.  workspace:
 * b200moe_dispatch_workspace_words(T) int32 words, zeroed once before first
 * use (the kernel leaves it reusable; one workspace per stream).
 * Position policy and dropless run a multi-CTA decoupled look-back scan over
 * 256-token tiles; score with a capacity selects per expert. */
int b200moe_dispatch(const float* gates, int T, int E, int capacity, int policy, int layout, int seg_stride,
                     int32_t* slot_rank, int32_t* counts, int32_t* seg_base, float* gate_mass, float* importance,
                     int64_t* stats, float* importance_loss, int32_t* importance_err, int32_t* workspace,
                     cudaStream_t stream);
size_t b200moe_dispatch_workspace_words(int T);

/* Token permute (K2): xp[seg_base[e] + slot_rank[t,e]] = x[t] for every kept
 * (t,e); pad rows of each segment up to a multiple of 128 are zeroed.
 * Replaces tensor.py:371-380 take_rows (moe.py:276). */
int b200moe_permute(const void* x, const int32_t* slot_rank, const int32_t* seg_base, const int32_t* counts, int T,
                    int H, int E, void* xp, cudaStream_t stream);

/* Weighted combine (K5): y[t] = sum_{e kept, ascending} gates[t,e] * o[row(t,e)]
 * (fp32 accumulation, bf16 out); fully dropped tokens get exactly 0.
 * Replaces moe.py:278-282 (mul + put_rows + add). */
int b200moe_combine(const void* o, const float* gates, const int32_t* slot_rank, const int32_t* seg_base, int T,
                    int H, int E, void* y, cudaStream_t stream);

/* Combine backward (K6): dout[row] = gates[t,e]*dy[t]; dg[t,e] = <dy[t], o[row]>
 * (0 where not kept); pad rows of dout zeroed. */
int b200moe_combine_bwd(const void* dy, const void* o, const float* gates, const int32_t* slot_rank,
                        const int32_t* seg_base, const int32_t* counts, int T, int H, int E, void* dout, float* dg,
                        cudaStream_t stream);

/* Router backward (K10+K11): dg_total = dg + dgates_ext (strided, may be NULL);
 * dh = softmax' (mixtral over the kept k, st over all E with the top-k mask);
 * dx[t] = sum_{kept e ascending} dxp[row] + dh.W_g^T (+ dn.W_noise^T with
 * dn = dh*z*sigmoid(noise_act)).  Writes dx (bf16), dh, dn (fp32, dn only with
 * noise).  Replaces tensor.py:292-295, 224, 375-378 and moe.py's router matmuls.
 * wg_swz / wn_swz (nullable): the swizzled W_g / W_noise tables that
 * b200moe_router_fwd left in the first 2*H*E_pad floats of its workspace
 * (E_pad = E rounded up to 4/8/16/32); passing them skips re-swizzling.
 * workspace: >= 2*H*32 + T*32 floats. */
int b200moe_router_bwd(const void* dxp, const int32_t* slot_rank, const int32_t* seg_base, const float* dg,
                       const float* dgates_ext, int64_t dgates_stride_t, int64_t dgates_stride_e, const float* gates,
                       const float* probs, const float* w_g, const float* w_noise, const float* z,
                       const float* noise_act, const float* wg_swz, const float* wn_swz, int T, int H, int E, int k,
                       int router_type, void* dx, float* dh, float* dn, float* workspace, cudaStream_t stream);

/* ---- Expert parallelism fused with the exchange (NVLink peer memory) ----
 * The *_peer variants address expert e's rows in the buffer of its owner rank
 * d = e / e_per_rank: `*_bufs` is a DEVICE array of the per-rank base pointers
 * (symmetric memory mapped into this process), and seg_base[e] is the row of
 * this rank's segment inside the owner's receive buffer.  permute_peer writes
 * every kept token straight into its owner's buffer (+ zero pads) and publishes
 * counts[e] into the owner's receive table count_bufs[d][rank*e_per_rank + e%e_per_rank];
 * combine_peer / combine_bwd_peer / router_bwd_peer read expert outputs (and
 * write combine gradients) in the owners' buffers.  The caller orders ranks
 * with a device barrier between producer and consumer kernels.  These replace
 * the NCCL all-to-alls of the dispatch / combine exchange. */
int b200moe_permute_peer(const void* x, const int32_t* slot_rank, const int32_t* seg_base, const int32_t* counts,
                         int T, int H, int E, int e_per_rank, int rank, const uint64_t* xp_bufs,
                         const uint64_t* count_bufs, cudaStream_t stream);
/* og (optional, [T, og_k, H] bf16): combine_peer also writes every token's
 * gathered expert rows there (row j = its j-th kept expert, ascending), and
 * combine_bwd_peer then reads them locally instead of from the owners' buffers,
 * so the backward's NVLink traffic is only the dO stores.  NULL: read remote. */
int b200moe_combine_peer(const uint64_t* o_bufs, int e_per_rank, const float* gates, const int32_t* slot_rank,
                         const int32_t* seg_base, int T, int H, int E, void* y, void* og, int og_k,
                         cudaStream_t stream);
int b200moe_combine_bwd_peer(const void* dy, const uint64_t* o_bufs, const float* gates, const int32_t* slot_rank,
                             const int32_t* seg_base, const int32_t* counts, int T, int H, int E, int e_per_rank,
                             const uint64_t* dout_bufs, float* dg, const void* og, int og_k, cudaStream_t stream);
/* FWD2 / BWD1 fused with the return exchange: every output row tile goes
 * straight from the epilogue (TMA bulk store) into its source rank's receive
 * plane over NVLink, overlapped with the next tiles' MMAs.  Segment s of this
 * owner is (src, el) = (s / E_local, s % E_local) (nseg = world * E_local, the
 * receive layout of permute_peer); its rows land at row
 * (rank * E_local + el) * cap_pad + r of rank src's plane -- the source's own
 * expert-major dispatch layout (LAYOUT_FIXED, seg_stride = cap_pad) -- so the
 * source's combine / router backward then read them locally.  dst_host: HOST
 * array of the world planes' device base pointers (dst_rows x H bf16 each).
 * The caller orders ranks with a device barrier before the consumers run. */
int b200moe_expert_fwd2_peer(const void* h, const void* w2, const int* seg_base, const int* seg_count,
                             const int* seg_expert, int nseg, int rows, int H, int F, int E_local,
                             const uint64_t* dst_host, int world, int rank, int cap_pad, int dst_rows,
                             cudaStream_t stream);
int b200moe_expert_bwd1_peer(const void* da, const void* db, const void* w1, const void* w3, const int* seg_base,
                             const int* seg_count, const int* seg_expert, int nseg, int rows, int H, int F,
                             int E_local, const uint64_t* dst_host, int world, int rank, int cap_pad, int dst_rows,
                             cudaStream_t stream);
int b200moe_router_bwd_peer(const uint64_t* dxp_bufs, int e_per_rank, const int32_t* slot_rank,
                            const int32_t* seg_base, const float* dg, const float* dgates_ext,
                            int64_t dgates_stride_t, int64_t dgates_stride_e, const float* gates, const float* probs,
                            const float* w_g, const float* w_noise, const float* z, const float* noise_act,
                            const float* wg_swz, const float* wn_swz, int T,
                            int H, int E, int k, int router_type, void* dx, float* dh, float* dn, float* workspace,
                            cudaStream_t stream);

/* Router weight gradients: dW_g = x^T.dh, dW_noise = x^T.dn (fp32, [H,E]),
 * deterministic (fixed-order partial sums).  workspace: >= ceil(T/64)*H*E
 * floats.  tickets (nullable): ceil(H/128) int32, zeroed once and left zeroed
 * -- with it (E <= 8) the last block of each hidden block finishes the
 * reduction in the same launch (on tcgen05 when H % 128 == 0: x read once
 * for both matrices); without it a second kernel does. */
int b200moe_router_wgrad(const void* x, const float* dh, const float* dn, int T, int H, int E, float* dw_g,
                         float* dw_noise, float* workspace, int32_t* tickets, cudaStream_t stream);

/* Importance (CV^2) penalty, tensor.py:503-521: loss = var(imp)/mean(imp)^2
 * with imp = sum_t gates[t,:].  Forward writes imp [E] and loss [1] (fp32);
 * backward writes dimp[e] = gscale[0] * dloss/dimp_e (the per-token gradient
 * is dimp broadcast over tokens). */
int b200moe_importance_fwd(const float* gates, int T, int E, float* imp, float* loss, int32_t* err_flag,
                           cudaStream_t stream);
int b200moe_importance_bwd(const float* imp, const float* gscale, int E, float* dimp, cudaStream_t stream);
/* Loss only, from an importance vector already reduced by b200moe_dispatch
 * (`importance` output) for the same gates. */
int b200moe_importance_loss(const float* imp, int E, float* loss, int32_t* err_flag, cudaStream_t stream);

/* Grouped expert GEMMs on tcgen05/TMEM/TMA (see gemm.cu).  `rows` = rows of
 * the permuted activation buffers.  H and F must be multiples of 256. */
int b200moe_expert_fwd1(const void* xp, const void* w1, const void* w3, const int* seg_base, const int* seg_count,
                        const int* seg_expert, int nseg, int rows, int H, int F, int E_local, void* a_out,
                        void* b_out, void* h_out, cudaStream_t stream);
int b200moe_expert_fwd2(const void* h, const void* w2, const int* seg_base, const int* seg_count,
                        const int* seg_expert, int nseg, int rows, int H, int F, int E_local, void* o_out,
                        cudaStream_t stream);
int b200moe_expert_bwd2(const void* dout, const void* w2, const void* a_pre, const void* b_pre, const int* seg_base,
                        const int* seg_count, const int* seg_expert, int nseg, int rows, int H, int F, int E_local,
                        void* da_out, void* db_out, cudaStream_t stream);
int b200moe_expert_bwd1(const void* da, const void* db, const void* w1, const void* w3, const int* seg_base,
                        const int* seg_count, const int* seg_expert, int nseg, int rows, int H, int F, int E_local,
                        void* dxp_out, cudaStream_t stream);
int b200moe_expert_wgrad(const void* xp, const void* h, const void* dout, const void* da, const void* db,
                         const int* seg_base, const int* seg_count, const int* seg_expert, int nseg, int rows, int H,
                         int F, int E_local, void* dw1, void* dw2, void* dw3, cudaStream_t stream);
/* Same, adding into dw1/dw2/dw3 (bf16, fp32 add, one rounding) when accumulate != 0:
 * gradient accumulation over micro-batches without a separate add pass. */
int b200moe_expert_wgrad_acc(const void* xp, const void* h, const void* dout, const void* da, const void* db,
                             const int* seg_base, const int* seg_count, const int* seg_expert, int nseg, int rows,
                             int H, int F, int E_local, void* dw1, void* dw2, void* dw3, int accumulate,
                             cudaStream_t stream);
/* Per-call variants.  grid_ctas > 0 caps the persistent grid at that many
 * CTAs (rounded down to the CTA-pair size) so that two GEMMs of the backward
 * can run concurrently on disjoint parts of the chip; 0 = one CTA per SM.
 * subs (WGRAD): bit 0 dW1, bit 1 dW3, bit 2 dW2 -- the sub-problems to compute
 * (dW2 needs only dout and h, so it can start before BWD2 has produced da/db). */
int b200moe_expert_bwd2_ex(const void* dout, const void* w2, const void* a_pre, const void* b_pre,
                           const int* seg_base, const int* seg_count, const int* seg_expert, int nseg, int rows,
                           int H, int F, int E_local, void* da_out, void* db_out, int grid_ctas, cudaStream_t stream);
/* BWD2 that also writes h = silu(a) * b (bf16, [rows, F]) rebuilt from the
 * stored a, b, for a caller that did not keep the forward's h (memory): WGRAD's
 * dW2 operand.  h_out NULL = b200moe_expert_bwd2_ex.  The rebuilt h rounds
 * silu(bf16 a) * bf16 b, where the forward's h rounds the fp32 accumulators. */
int b200moe_expert_bwd2_h(const void* dout, const void* w2, const void* a_pre, const void* b_pre,
                          const int* seg_base, const int* seg_count, const int* seg_expert, int nseg, int rows,
                          int H, int F, int E_local, void* da_out, void* db_out, void* h_out, int grid_ctas,
                          cudaStream_t stream);
int b200moe_expert_bwd1_ex(const void* da, const void* db, const void* w1, const void* w3, const int* seg_base,
                           const int* seg_count, const int* seg_expert, int nseg, int rows, int H, int F, int E_local,
                           void* dxp_out, int grid_ctas, cudaStream_t stream);
int b200moe_expert_wgrad_ex(const void* xp, const void* h, const void* dout, const void* da, const void* db,
                            const int* seg_base, const int* seg_count, const int* seg_expert, int nseg, int rows,
                            int H, int F, int E_local, void* dw1, void* dw2, void* dw3, int accumulate, int subs,
                            int grid_ctas, cudaStream_t stream);

/* Dense GEMMs of the transformer step around the layer (qkv / wo / lm-head,
 * reference model.py:135-169 via tensor.py:192-207 matmul) on the same
 * tcgen05 kernel, weights in the reference [in, out] layout w [K, N]:
 *   fwd   y[M,N]  = x[M,K] . w        (ld* = row pitches in elements)
 *   dgrad dx[M,K] = dy[M,N] . w^T
 *   wgrad dw[K,N] = x^T . dy          (lddw must equal N)
 * bf16 in / out, fp32 accumulation; K and N multiples of 256, any M >= 1.
 * seg_base / seg_count / seg_expert: a device segment table of one segment
 * {0, M, 0} (int32).  grid_ctas: persistent grid cap (0 = one CTA per SM);
 * the model step leaves a few SMs to the overlapped NCCL reductions and
 * optimizer updates running on other streams. */
int b200moe_dense_fwd(const void* x, const void* w, const int* seg_base, const int* seg_count, const int* seg_expert,
                      int M, int K, int N, int ldx, int ldw, int ldy, void* y, int grid_ctas, cudaStream_t stream);
int b200moe_dense_dgrad(const void* dy, const void* w, const int* seg_base, const int* seg_count,
                        const int* seg_expert, int M, int K, int N, int lddy, int ldw, int lddx, void* dx,
                        int grid_ctas, cudaStream_t stream);
int b200moe_dense_wgrad(const void* x, const void* dy, const int* seg_base, const int* seg_count,
                        const int* seg_expert, int M, int K, int N, int ldx, int lddy, int lddw, void* dw,
                        int grid_ctas, cudaStream_t stream);

/* Diagnostics knobs for tests and A/B tools, NOT part of the product path:
 * thread-local (they affect only GEMM launches issued by the calling thread;
 * other threads always run the defaults), so the entry points above stay
 * re-entrant.  Reset them before returning (tests use try/finally). */
int b200moe_gemm_set_cta_group(int cta_group); /* 2 (CTA pairs, default) or 1 */
int b200moe_gemm_set_max_ctas(int n);          /* persistent grid size (default 148) */
int b200moe_gemm_set_debug(int flags);         /* experiment bits (0 = product kernels) */

/* Online upcycling copy (K12), upcycle.py:104-112 / 216-224: replicate one
 * dense FFN ([in,out] layout: w1,w3 [H,F], w2 [F,H]; fp32 or bf16 source,
 * src_is_fp32) into E_local experts of the kernel layout (W1,W3 [E,F,H],
 * W2 [E,H,F], bf16, round-to-nearest-even).  Bitwise equal to the reference
 * copy after the dtype cast. */
int b200moe_upcycle_copy(const void* w1, const void* w2, const void* w3, int src_is_fp32, int H, int F, int E_local,
                         void* W1, void* W2, void* W3, cudaStream_t stream);

/* ---------------------------------------------------------------------------
 * The transformer step around the MoE layer (model.cu).
 * Residual stream fp32 [T, H]; normalised activations bf16 [T, H].
 * ------------------------------------------------------------------------- */

/* x_out = x + delta (delta bf16, optional: NULL = no add, x_out unused);
 * y = rmsnorm(x_out) * gain (bf16); rstd[T] = (mean(x_out^2) + eps)^-1/2.
 * Replaces moefold/tensor.py:307-313 (rmsnorm forward) fused with the block's
 * residual add (moefold/model.py:151,156). */
int b200moe_rmsnorm_fwd(const float* x, const void* delta, const float* gain, int T, int H, float eps, float* x_out,
                        void* y, float* rstd, cudaStream_t stream);
/* dx = rmsnorm'(dy) + dres (dres optional), written as fp32 (dx) and/or bf16
 * (dx_bf16); dgain[H] = sum_t dy*x*rstd.  workspace >= ceil(T/8) * H floats.
 * Replaces moefold/tensor.py:314-319. */
int b200moe_rmsnorm_bwd(const void* dy, const float* x, const float* rstd, const float* gain, const float* dres, int T,
                        int H, float* dx, void* dx_bf16, float* dgain, float* workspace, cudaStream_t stream);
/* out[t] = table[ids[t]] (fp32); ids outside [0, V) set *err_flag = 1.
 * Replaces moefold/tensor.py:324-331. */
int b200moe_embedding_fwd(const float* table, const int64_t* ids, int T, int H, int V, float* out, int* err_flag,
                          cudaStream_t stream);
/* grad[seg_id[s]] = sum over i in [seg_start[s], seg_start[s+1]) of g[order[i]]
 * in order (order = stable argsort of the ids); other rows untouched.
 * Replaces the np.add.at of moefold/tensor.py:333-336. */
int b200moe_embedding_bwd(const float* g, const int* order, const int* seg_start, const int* seg_id, int n_seg, int H,
                          float* grad, cudaStream_t stream);
/* Same sums from a device-side stable sort: sorted_ids[i] = ids[order[i]]
 * (n entries); rows of grad for absent ids untouched.  Used for the
 * data-parallel embedding gradient over all ranks' gathered tokens. */
int b200moe_embedding_bwd_sorted(const float* g, const int64_t* order, const int64_t* sorted_ids, int n, int H,
                                 float* grad, cudaStream_t stream);
/* nll[t] = logsumexp(logits[t]) - logits[t, targets[t]], lse[t], loss[0] =
 * mean(nll); logits bf16 [T, V].  Replaces moefold/tensor.py:340-359. */
int b200moe_cross_entropy_fwd(const void* logits, const int64_t* targets, int T, int V, float* nll, float* lse,
                              float* loss, int* err_flag, cudaStream_t stream);
/* dlogits = (softmax(logits) - onehot(targets)) * dloss[0] / T (bf16).
 * Replaces moefold/tensor.py:361-364. */
int b200moe_cross_entropy_bwd(const void* logits, const int64_t* targets, const float* lse, const float* dloss, int T,
                              int V, void* dlogits, cudaStream_t stream);

#define B200MOE_OPT_ADAM 0 /* moefold/train.py:161-171 */
#define B200MOE_OPT_SGD 1  /* moefold/train.py:172-176 */

/* One optimizer tensor: fp32 master `param`, moments m (and v for Adam),
 * gradient (fp32 or bf16), optional bf16 compute copy refreshed in place. */
typedef struct {
    float* param;
    float* m;
    float* v;
    const void* grad;
    void* shadow;
    long long n;
    int grad_bf16;
    int reserved;
} b200moe_opt_tensor;

/* Elements per chunk of the optimizer's work list. */
int b200moe_optimizer_chunk(void);
/* One step over every tensor of `tensors` (device array); the work list is
 * n_chunks (tensor index, element offset) pairs of b200moe_optimizer_chunk()
 * elements.  Scalars are the float32-rounded constants of the reference's
 * expressions (1-beta, 1-beta^t).  Replaces moefold/train.py:_Optimizer.step. */
int b200moe_optimizer_step(const b200moe_opt_tensor* tensors, const int* chunk_tensor, const long long* chunk_off,
                           int n_chunks, int kind, float lr, float beta1, float one_minus_beta1, float beta2,
                           float one_minus_beta2, float eps, float bias_corr1, float bias_corr2, float momentum,
                           cudaStream_t stream);

/* ---------------------------------------------------------------------------
 * Checkpoint payload checksums (crc32c.cu).
 * ------------------------------------------------------------------------- */

/* Bytes of device workspace b200moe_crc32c needs (accumulator + tables). */
long long b200moe_crc32c_workspace_bytes(void);
/* Build the fixed lookup tables into a workspace (once per workspace). */
int b200moe_crc32c_init(void* workspace, cudaStream_t stream);
/* *out (device uint32) = CRC32C (Castagnoli, init/xorout 0xFFFFFFFF) of the
 * nbytes at `data` (device, 16-byte aligned), using a workspace prepared by
 * b200moe_crc32c_init; calls sharing a workspace must be stream-ordered.  Replaces the pure-Python
 * slicing-by-8 crc32c of moefold/checkpoint.py:60-78 used on every tensor
 * payload by save/load (checkpoint.py:108-118, 215-216). */
int b200moe_crc32c(const void* data, long long nbytes, unsigned int* out, void* workspace, cudaStream_t stream);

#ifdef __cplusplus
}
#endif
#endif /* B200MOE_H */
