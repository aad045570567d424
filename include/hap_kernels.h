/*
 * hap_kernels.h — C-ABI of the B200 (sm_100a) HAP MoE-block executor.
 *
 * The reference (moeplan, /root/reference/pkg/src/moeplan) has NO forward
 * implementation: it only *models* these ops through its FLOP and
 * collective-volume formulas.  Each entry point below is the executable
 * counterpart of one modelled term, cited per function:
 *   - attention_flops  arch.py:145-162  -> hap_gemm_bf16 (QKV/O projections),
 *                                          hap_attn_prefill / hap_attn_decode
 *   - expert_flops     arch.py:165-178  -> hap_router_topk (router term),
 *                                          hap_grouped_gemm_bf16 (gate/up/down)
 *   - comm_volume EP rows strategies.py:334-340 -> hap_moe_permute /
 *                                          hap_moe_combine (dispatch/combine
 *                                          token re-layout around the a2a)
 *
 * Conventions (all functions):
 *   - every pointer is a DEVICE pointer owned by the caller; the library never
 *     allocates, frees, or synchronises; calls are stream-ordered on `stream`
 *     (a cudaStream_t passed as void*) and CUDA-graph capturable;
 *   - bf16 tensors are row-major with the given leading dimension (elements);
 *   - return 0 (HAP_OK) or a negative hap_status.  Argument errors are
 *     detected before any launch.
 */
#ifndef HAP_KERNELS_H_
#define HAP_KERNELS_H_

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef enum {
  HAP_OK = 0,
  HAP_ERR_INVALID_ARG = -1, /* bad shape / null pointer / out-of-range value */
  HAP_ERR_UNSUPPORTED = -2, /* shape legal but not supported by this build   */
  HAP_ERR_MISALIGNED = -3,  /* pointer / leading dimension alignment          */
  HAP_ERR_LAUNCH = -4,      /* CUDA launch failure                            */
  HAP_ERR_WORKSPACE = -5,   /* workspace too small                            */
  HAP_ERR_DRIVER = -6       /* driver entry point (cuTensorMapEncodeTiled)    */
} hap_status;

/* GEMM epilogues */
#define HAP_EPI_STORE 0  /* C = acc (+bias) (+residual)                        */
#define HAP_EPI_SWIGLU 1 /* C = silu(acc[:, gate]) * acc[:, up] per tile        */
#define HAP_EPI_F32 2    /* C (float, ldc == N) = acc: the raw fp32 accumulator */

const char* hap_status_string(int status);

/* Enable peer access from the current device to peer_device (NVLink P2P) so
 * kernels can store through CUDA-IPC mappings of that device's buffers.
 * Idempotent; HAP_ERR_UNSUPPORTED when the pair has no P2P path. */
int hap_enable_peer_access(int peer_device);
int hap_abi_version(void);

/* Largest SwiGLU tile half-width (multiple of 8, <= 128) dividing `inter_dim`;
 * the gate/up weight interleave (see hap_grouped_gemm_bf16) must use it. */
int64_t hap_swiglu_half_width(int64_t inter_dim);

/*
 * Grouped GEMM on 5th-gen tensor cores (tcgen05 + TMEM + TMA), bf16 in,
 * fp32 accumulate, bf16 out.
 *
 *   for s in [0, n_segs): g = seg_group ? seg_group[s] : s;
 *       rows r in [seg[s], seg[s+1]) of A:
 *       C[r, :] = epilogue( A[r, :K] . B[g*N:(g+1)*N, :K]^T )
 *
 * A: [a_rows, K] (lda), B: [n_groups*N, K] contiguous (nn.Linear weight
 * layout, one block of N rows per group), C: [a_rows, out_cols] (ldc).
 * seg: device int32[n_segs+1] row offsets (NULL => one segment spanning all
 * a_rows); seg_group: device int32[n_segs] weight group per segment (NULL =>
 * identity, n_segs == n_groups).  Several segments may share a group (EP:
 * rows received from different source ranks for the same local expert).
 * Segments need not be aligned; rows outside every segment are untouched.
 *
 * HAP_EPI_SWIGLU: B rows are interleaved in blocks of 2*swiglu_half:
 * block j = [gate rows j*hw..j*hw+hw-1 ; up rows j*hw..j*hw+hw-1] with
 * hw = swiglu_half; out_cols = N/2 and C[r, j*hw+i] = silu(g)*u.
 * HAP_EPI_STORE: optional bias (bf16[N]) and residual (bf16, ldr) are added in
 * fp32 before the single bf16 rounding.
 * HAP_EPI_F32: C is float [a_rows, N] (ldc == N) and receives the fp32 TMEM
 * accumulator unrounded (no bias/residual) — the fp32-accumulate parity
 * check of the expert and projection GEMMs.
 *
 * Replaces: the per-expert gated-MLP FLOP term of expert_flops (arch.py:174-176)
 * and the projection term of attention_flops (arch.py:157-160).
 */
int hap_grouped_gemm_bf16(const void* A, int64_t a_rows, int64_t lda, int64_t K, const void* B,
                          int64_t n_groups, int64_t N, const int32_t* seg, int64_t n_segs,
                          const int32_t* seg_group, void* C, int64_t ldc, int32_t epilogue,
                          int64_t swiglu_half, const void* bias, const void* residual, int64_t ldr,
                          void* stream);

/*
 * Fused QKV projection + rotary embedding (same tcgen05 kernel, RoPE in the
 * epilogue): C = A . W^T (+bias), then for the first n_rope_heads heads of
 * each row (the q and k heads of a [q | k | v] row) the rotate-half RoPE with
 * angle positions[r] * theta^(-2i/head_dim) (fp32), one bf16 rounding.
 * head_dim in {64, 128}; N % head_dim == 0.
 * Replaces: the Q/K/V projection term of attention_flops (arch.py:157-160)
 * plus the (unmodelled) rotary embedding.
 */
int hap_gemm_qkv_rope(const void* A, int64_t M, int64_t lda, int64_t K, const void* W, int64_t N,
                      const void* bias, void* C, int64_t ldc, const int32_t* positions, int64_t n_rope_heads,
                      int64_t head_dim, float theta, void* stream);

/*
 * Attention-module prologue in one call: hn = RMSNorm(x; norm_w, eps) exactly
 * as hap_rmsnorm, then C = hap_gemm_qkv_rope(hn, ...).  Decode-size launches
 * (1-2 rows on the GEMV path) normalise the rows while staging them and never
 * write hn (one launch instead of two); otherwise hn (caller scratch, M x K
 * bf16, leading dimension ldhn) receives the normalised rows.  The contents
 * of hn after the call are unspecified; C is bit-identical to the two calls.
 * Replaces: the attention module's norm + QKV projection whose weights the
 * reference streams per decode step (arch.py:145-161, costmodel decode rows).
 */
int hap_rmsnorm_gemm_qkv_rope(const void* x, int64_t M, int64_t ldx, int64_t K, const void* norm_w, float eps,
                              void* hn, int64_t ldhn, const void* W, int64_t N, const void* bias, void* C,
                              int64_t ldc, const int32_t* positions, int64_t n_rope_heads, int64_t head_dim,
                              float theta, void* workspace, size_t ws_bytes, void* stream);

/*
 * Split-K variants of the two GEMM entry points (same semantics).  With a
 * workspace, shapes whose tiles cannot cover the 148 SMs (small-M weight
 * streaming: decode projections, TP-sharded layers) cut K into slices run by
 * different CTAs, each writing fp32 partials to the workspace; a second kernel
 * sums the slices in slice order (deterministic, no atomics) and applies the
 * epilogue.  workspace: device scratch of ws_bytes (hap_gemm_splitk_workspace_bytes()
 * is the size the library plans for; smaller => fewer slices); it must not be
 * shared by GEMMs running concurrently.  NULL workspace == the plain entry points.
 */
size_t hap_gemm_splitk_workspace_bytes(void);
int hap_grouped_gemm_bf16_ex(const void* A, int64_t a_rows, int64_t lda, int64_t K, const void* B,
                             int64_t n_groups, int64_t N, const int32_t* seg, int64_t n_segs,
                             const int32_t* seg_group, void* C, int64_t ldc, int32_t epilogue,
                             int64_t swiglu_half, const void* bias, const void* residual, int64_t ldr,
                             void* workspace, size_t ws_bytes, void* stream);
int hap_gemm_qkv_rope_ex(const void* A, int64_t M, int64_t lda, int64_t K, const void* W, int64_t N,
                         const void* bias, void* C, int64_t ldc, const int32_t* positions, int64_t n_rope_heads,
                         int64_t head_dim, float theta, void* workspace, size_t ws_bytes, void* stream);
/* hap_grouped_gemm_bf16_ex on at most sm_budget SMs (0 = all): the persistent
 * grid and the split-K plan are sized for that many SMs, leaving the rest to
 * kernels on other streams — the executor runs the shared expert's decode
 * GEMMs this way on a side stream beside the routed path (half the SMs). */
int hap_grouped_gemm_bf16_sms(const void* A, int64_t a_rows, int64_t lda, int64_t K, const void* B,
                              int64_t n_groups, int64_t N, const int32_t* seg, int64_t n_segs,
                              const int32_t* seg_group, void* C, int64_t ldc, int32_t epilogue,
                              int64_t swiglu_half, const void* bias, const void* residual, int64_t ldr,
                              void* workspace, size_t ws_bytes, int32_t sm_budget, void* stream);

/*
 * EP combine over peer memory: hap_grouped_gemm_bf16 with HAP_EPI_STORE whose
 * output rows are scattered per segment: row r of segment s (rows
 * [seg[s], seg[s+1]) of A) is stored at
 *     (bf16*)seg_dst[s] + (r - seg[s] + seg_dst_row0[s]) * ldc
 * seg_dst (device int64[n_segs]) holds device addresses — in the executor the
 * peer-mapped (CUDA IPC) output buffers of the ranks the rows came from, so the
 * down-projection epilogue writes each expert output straight back to its
 * source rank over NVLink (the combine all-to-all of strategies.py:334-338,
 * fused into the GEMM).  No bias / residual / split-K.
 */
int hap_grouped_gemm_bf16_scatter(const void* A, int64_t a_rows, int64_t lda, int64_t K, const void* B,
                                  int64_t n_groups, int64_t N, const int32_t* seg, int64_t n_segs,
                                  const int32_t* seg_group, const int64_t* seg_dst, const int32_t* seg_dst_row0,
                                  int64_t ldc, void* stream);

/*
 * EP dispatch over peer memory: rows [seg[s], seg[s+1]) of src (bf16 [*, h],
 * contiguous) are copied to (bf16*)dst_base[s] + (dst_row0[s] + i) * ldd,
 * dst_base holding (peer-mapped) device addresses (the dispatch all-to-all of
 * strategies.py:334-338 as direct NVLink stores).  rows_max bounds seg[n_segs]
 * (grid sizing only); seg, dst_base, dst_row0 are device arrays.
 */
int hap_peer_copy_rows(const void* src, int64_t rows_max, int64_t h, const int32_t* seg, int64_t n_segs,
                       const int64_t* dst_base, const int64_t* dst_row0, int64_t ldd, void* stream);

/*
 * One-shot all-reduce (sum) of n bf16 elements over peer-mapped memory for
 * decode-size messages.  Each rank owns a symmetric region data (2 * n_max
 * bf16, double-buffered by call parity) and sig (hap_peer_allreduce_sig_bytes
 * int32 flags, zeroed once on every rank before the first call), and a local
 * epoch array (n_ctas int32, zeroed once).  All arrays of addresses are device
 * int64[n_ranks]: in_ptrs / out_ptrs / epoch_ptrs are read at the entries of
 * the ranks this launch plays (rank0 .. rank0 + ranks_in_launch - 1; a
 * multi-GPU rank plays itself, ranks_in_launch = 1), data_ptrs / sig_ptrs hold
 * every rank's (peer-mapped) region.  Sum in rank order in fp32, one bf16
 * rounding: every rank gets identical bytes.  in == out is allowed.  No host
 * synchronisation (CUDA-graph capturable); every rank must use the same n_ctas.
 * Replaces: the AllReduce rows of comm_volume (strategies.py:314-322, 341-342)
 * on the decode path.
 */
/*
 * One-shot all-reduce through NVLink SHARP (NVSwitch multicast memory): the
 * caller binds one physical allocation per device to a multicast object and
 * passes this rank's unicast (uc_base) and multicast (mc_base) views of it,
 * hap_nvls_allreduce_bytes(n_max, n_ctas) bytes, zero-filled before the first
 * call, and an int32 epoch[n_ctas] (zero).  Each CTA copies its slice into
 * its own buffer, arrives with one multimem.red on a per-CTA counter, waits
 * for all ranks and reads its slice with multimem.ld_reduce (in-switch sum,
 * fp32 accumulation, one bf16 rounding).  No host work: graph capturable.
 * Replaces: the decode-size AllReduce rows of comm_volume (strategies.py:314-322,
 * 341-342).
 */
size_t hap_nvls_allreduce_bytes(int64_t n_max, int32_t n_ctas);
int hap_nvls_allreduce_bf16(const void* in, void* out, void* uc_base, void* mc_base, int32_t* epoch, int64_t n,
                            int64_t n_max, int32_t n_ranks, int32_t n_ctas, void* stream);

size_t hap_peer_allreduce_sig_bytes(int32_t n_ranks, int32_t n_ctas);
int hap_peer_allreduce_bf16(const int64_t* in_ptrs, const int64_t* out_ptrs, const int64_t* epoch_ptrs,
                            const int64_t* data_ptrs, const int64_t* sig_ptrs, int64_t n, int64_t n_max,
                            int32_t n_ranks, int32_t rank0, int32_t ranks_in_launch, int32_t n_ctas, void* stream);

/*
 * Router: logits[t,e] = x[t,:] . w[e,:] in fp32 with a FIXED reduction
 * order — h is cut into 8 equal contiguous ranges; in range p the partial is
 * the sequential chain acc = fma(x[t,j], w[e,j], acc) (bf16*bf16 products are
 * exact in fp32, so this is the sequential fp32 sum of products), and the
 * partials are added in order ((p0 + p1) + p2) + ... — the order the oracle
 * computes.  Softmax in fp32, top-k selected on logits with ties to the
 * lower expert index, weights = softmax probabilities of the selected
 * experts, renormalised to sum 1 when `renormalize`.
 * If has_shared_gate, w has n_experts+1 rows and row n_experts is the
 * shared-expert gate: shared_gate[t] = sigmoid(x[t] . w[E]) (fp32).
 * logits_out (fp32 [T, n_experts]) is optional.
 * Requires h % 64 == 0, n_experts + has_shared_gate <= 72, top_k <= 32.
 * Workspace (caller-owned, zero-filled once before first use; the kernel
 * leaves it zeroed): hap_router_workspace_bytes(T, n_experts, has_shared_gate)
 * bytes, non-zero only for T <= 1024 with more than 8 router rows, where the
 * work is spread over CTAs per (token, 8 rows) that meet in the workspace.
 * With a NULL / smaller workspace such calls use one CTA per token instead
 * (same logits bit for bit, slower for wide routers).  Concurrent calls need
 * distinct workspaces.
 * Replaces: the router term 2*T*h*E of expert_flops (arch.py:177).
 */
size_t hap_router_workspace_bytes(int64_t T, int64_t n_experts, int32_t has_shared_gate);
int hap_router_topk(const void* x, int64_t T, int64_t h, const void* w, int64_t n_experts, int64_t top_k,
                    int32_t renormalize, int32_t has_shared_gate, int32_t* topk_idx, float* topk_w,
                    float* shared_gate, float* logits_out, void* workspace, size_t ws_bytes, void* stream);

/*
 * Stable counting-sort permute (scan + scatter).  Row r of the logical input
 * (r in [0, R)) carries expert id e_r = expert_of_row[r] and payload
 * x[r / src_row_div, :h].  Rows are placed at
 *     dst_of_row[r] = seg[e_r] + #{r' < r : e_r' == e_r}
 * i.e. sorted by (expert, r) — with R = T*k and src_row_div = k this is the
 * canonical (expert, token, slot) order.  seg (int32[n_experts+1]) receives
 * the exclusive prefix of per-expert counts.  Rows with e_r outside
 * [0, n_experts) are dropped (dst_of_row = -1).  x_out may be NULL (index
 * only).  Bit-exact by construction (no atomics on the ordering path).
 * Workspace: hap_moe_permute_workspace_bytes(R, n_experts).
 */
size_t hap_moe_permute_workspace_bytes(int64_t R, int64_t n_experts);
int hap_moe_permute(const int32_t* expert_of_row, int64_t R, int64_t n_experts, const void* x,
                    int64_t src_row_div, int64_t h, void* x_out, int32_t* dst_of_row, int32_t* seg,
                    void* workspace, size_t ws_bytes, void* stream);

/*
 * Weighted combine (unpermute):
 *   out[t] = sum_j w[t,j] * y[dst[t*k+j]]  (+ sg[t] * shared_y[t])
 *            (+ residual[t - res_row0]  if res_row0 <= t < res_row0 + res_rows)
 * fp32 accumulation in slot order, one bf16 rounding.  dst < 0 => slot skipped.
 * residual / shared_y / shared_gate may be NULL.  The residual row window lets
 * a rank add the residual only to the rows a following reduce-scatter hands
 * back to it (so the sum over ranks counts it once).
 */
int hap_moe_combine(const void* y, const int32_t* dst_of_row, const float* topk_w, int64_t T, int64_t k,
                    int64_t h, const void* residual, int64_t res_row0, int64_t res_rows, const void* shared_y,
                    const float* shared_gate, void* out, void* stream);

/*
 * Combine whose output rows leave as a reduce-scatter push: token t's row goes
 * to row (slot*chunk_rows + t % chunk_rows) of the buffer dst_tab[t / chunk_rows]
 * (device int64 table of peer-mapped bases, one per chunk owner; T a multiple
 * of chunk_rows).  With slot = this rank's index in the group every owner
 * receives the partial sums of its chunk from every rank, in slot order, for
 * hap_reduce_slots_bf16.  Same arithmetic as hap_moe_combine.
 * Replaces: the expert-TP ReduceScatter / DP<-TP boundary of comm_volume
 * (strategies.py:324-332, 341-342) as a separate NCCL call.
 */
int hap_moe_combine_chunked(const void* y, const int32_t* dst_of_row, const float* topk_w, int64_t T, int64_t k,
                            int64_t h, const void* residual, int64_t res_row0, int64_t res_rows,
                            const void* shared_y, const float* shared_gate, const int64_t* dst_tab,
                            int64_t chunk_rows, int64_t slot, void* stream);

/* RMSNorm (fp32 statistics): out = w * (x * rsqrt(mean(x^2) + eps)). */
int hap_rmsnorm(const void* x, int64_t T, int64_t h, int64_t ldx, const void* w, float eps, void* out,
                int64_t ldo, void* stream);

/*
 * RMSNorm whose rows are stored to every base in dst_tab (device int64 table
 * of n_dst <= 64 bases, typically this replica's row block in every rank's
 * peer-mapped gather buffer): the DP->TP boundary AllGather pushed by the
 * kernel that produces the rows (strategies.py:324-332).
 */
int hap_rmsnorm_multi(const void* x, int64_t T, int64_t h, int64_t ldx, const void* w, float eps,
                      const int64_t* dst_tab, int32_t n_dst, int64_t ldo, void* stream);

/*
 * Device-side group barrier over peer memory: sig_tab holds n_ranks device
 * addresses of each rank's int32[n_ranks] flag row (peer-mapped), epoch is
 * this rank's int32 counter (device).  Waits for every earlier kernel of the
 * stream, publishes epoch+1 to every rank (system-scope release) and spins
 * until all ranks published it.  Flags and counters start at 0 on every
 * rank.  No host work: CUDA-graph capturable.
 */
int hap_peer_barrier(const int64_t* sig_tab, int32_t* epoch, int32_t n_ranks, int32_t rank, void* stream);

/*
 * out[r, :] = sum_{s < n_slots} slots[s*rows + r, :]  (fp32 in slot order,
 * one bf16 rounding): the owner side of a pushed reduce-scatter.
 */
int hap_reduce_slots_bf16(const void* slots, int64_t n_slots, int64_t rows, int64_t h, void* out, void* stream);

/* Copy n int32 from src to (dst_tab[p] + dst_offset_bytes) for each of the n_dst device bases. */
int hap_peer_broadcast_i32(const int32_t* src, int64_t n, const int64_t* dst_tab, int32_t n_dst,
                           int64_t dst_offset_bytes, void* stream);

/*
 * EP dispatch/combine plan on the device from the gathered segment offsets
 * segs[s][0..E] (int32 [ep][E+1], E = ep*experts_local) of every EP rank s:
 * dst_row0[e] (int64) = row of this rank's expert-e segment in rank
 * e/experts_local's receive buffer (blocks (source, local expert) in
 * lexicographic order); seg_r (int32 [E+1]) = this rank's receive-block
 * offsets; seg_dst_row0 (int32 [E]) = for receive block (s, j) the row of
 * source s's permuted segment of expert me*experts_local + j.  Replaces the
 * host-side count exchange of the EP all-to-alls (strategies.py:334-338).
 */
int hap_ep_exchange_plan(const int32_t* segs, int32_t ep, int32_t experts_local, int32_t me, int64_t* dst_row0,
                         int32_t* seg_r, int32_t* seg_dst_row0, void* stream);

/*
 * In-place rotary embedding (rotate-half convention) on the q and k heads of
 * a fused qkv row buffer: row t = [q (n_q*d) | k (n_kv*d) | v (n_kv*d)],
 * leading dimension ld.  positions: int32[T].  inv_freq[i] = theta^(-2i/d).
 */
int hap_rope_qk(void* qkv, int64_t T, int64_t ld, int64_t n_q_heads, int64_t n_kv_heads, int64_t head_dim,
                const int32_t* positions, float theta, void* stream);

/*
 * Causal (or full) GQA prefill attention on tcgen05/TMEM, bf16 in/out, fp32
 * softmax.  Token (s, i) = row s*seq_len + i.  q/k/v/out addressed by leading
 * dims (multiples of 8, 16-byte aligned bases); head h of a row starts at
 * column h*head_dim.  head_dim in {64, 128}.  The persistent kernel hands out
 * work items through two int32 tickets in the caller's workspace
 * (hap_attn_prefill_workspace_bytes(), 4-byte aligned, zero-filled once before
 * first use; the kernel re-zeroes them on exit, so a workspace is reusable by
 * the next call on its stream).  Concurrent calls need distinct workspaces.
 * Replaces: score+value term 4*n*kv_len*h of attention_flops (arch.py:161).
 */
size_t hap_attn_prefill_workspace_bytes(void);
int hap_attn_prefill(const void* q, int64_t ldq, const void* k, int64_t ldk, const void* v, int64_t ldv,
                     void* out, int64_t ldo, int64_t n_seqs, int64_t seq_len, int64_t n_q_heads,
                     int64_t n_kv_heads, int64_t head_dim, float scale, int32_t causal, void* workspace,
                     size_t ws_bytes, void* stream);

/*
 * Prefill: copy the (post-RoPE) k and v of every token of n_seqs sequences of
 * seq_len tokens (fused qkv rows, token (s,i) = row s*seq_len+i) into
 * positions [0, seq_len) of a [n_seqs, n_kv, max_len, d] cache.
 */
int hap_kv_cache_fill(const void* qkv, int64_t ldqkv, int64_t n_seqs, int64_t seq_len, int64_t n_q_heads,
                      int64_t n_kv_heads, int64_t head_dim, void* k_cache, void* v_cache, int64_t max_len,
                      void* stream);

/*
 * Append one token's k/v (from a fused qkv row buffer) into a [B, max_len,
 * n_kv, d] cache at position pos[b], then split-KV GQA decode attention of
 * q over cache rows [0, pos[b]] for each sequence b.
 * Workspace: hap_attn_decode_workspace_bytes(B, n_q_heads, head_dim, max_len).
 */
size_t hap_attn_decode_workspace_bytes(int64_t B, int64_t n_q_heads, int64_t head_dim, int64_t max_len);
int hap_attn_decode(const void* qkv, int64_t ldqkv, void* k_cache, void* v_cache, int64_t max_len,
                    const int32_t* pos, int64_t B, int64_t n_q_heads, int64_t n_kv_heads, int64_t head_dim,
                    float scale, void* out, int64_t ldo, void* workspace, size_t ws_bytes, void* stream);

/*
 * Paged KV cache: k_pool / v_pool hold n_pages pages [n_kv, page_size, d]
 * (page_size a multiple of 16); int32 block_table[b * max_pages + j] is the
 * page of sequence b's keys [j*page_size, (j+1)*page_size) (< 0: none; the
 * caller allocates the pages covering [0, pos[b]] before the call).  Same
 * arithmetic as the contiguous entry points with max_len = max_pages *
 * page_size (identical split plan, bit-identical outputs); workspace:
 * hap_attn_decode_workspace_bytes(B, n_q, d, max_pages * page_size).
 * Replaces: the KV bytes the reference grows per decode step
 * (arch.py:193-201, simulate.py:78-114) with a non-contiguous cache.
 */
int hap_kv_cache_fill_paged(const void* qkv, int64_t ldqkv, int64_t n_seqs, int64_t seq_len, int64_t n_q_heads,
                            int64_t n_kv_heads, int64_t head_dim, void* k_pool, void* v_pool,
                            const int32_t* block_table, int64_t max_pages, int64_t page_size, void* stream);
int hap_attn_decode_paged(const void* qkv, int64_t ldqkv, void* k_pool, void* v_pool, int64_t n_pages,
                          int64_t page_size, const int32_t* block_table, int64_t max_pages, const int32_t* pos,
                          int64_t B, int64_t n_q_heads, int64_t n_kv_heads, int64_t head_dim, float scale, void* out,
                          int64_t ldo, void* workspace, size_t ws_bytes, void* stream);

/*
 * INT4 per-group dequantization of a GQI4 tensor (reference quant.py:19-22,
 * 61-116): codes packed low-nibble-first (4-byte aligned), float64 scale and
 * zero point per group of group_size elements, n original elements.
 * out_bf16 == 0: out is float64 and equals quant.py:dequantize bit for bit
 * (code*scale rounded, then + zero rounded; no FMA).  out_bf16 == 1: out is
 * bf16, the same value rounded to fp32 then bf16.
 * Replaces: the v_dequant / DequantTimeTable term of the stage-switch cost
 * (transition.py:46-97, 180-199).
 */
int hap_int4_dequant(const uint8_t* codes, const double* scales, const double* zero_points, int64_t group_size,
                     int64_t n, void* out, int32_t out_bf16, void* stream);

/*
 * Batched 2-D strided copy, one launch for up to any number of pieces.
 * descs (HOST memory, read before return): n_descs records of 6 int64 —
 * {src address, dst address, rows, row_bytes, src_pitch, dst_pitch} (bytes);
 * row i of a record copies row_bytes from src + i*src_pitch to dst +
 * i*dst_pitch.  Addresses, row_bytes and (rows > 1) pitches must be 16-byte
 * aligned (HAP_ERR_MISALIGNED otherwise); source and destination bytes must
 * not overlap; all records are validated before the first launch.
 * Replaces: the local pack / unpack phases of the expert reshard whose
 * volume the reference charges in reshard_volume (transition.py:153-177,
 * Eq.6 T_reshard transition.py:241-267).
 */
int hap_copy2d_batched(const int64_t* descs, int64_t n_descs, void* stream);

#ifdef __cplusplus
}
#endif
#endif /* HAP_KERNELS_H_ */
