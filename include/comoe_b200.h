/* comoe_b200.h — C ABI of the B200-native CoMoE MoE-layer hot path.
 *
 * Every entry point takes raw device pointers, sizes and a cudaStream_t
 * (passed as void*), enqueues asynchronous work on that stream, never
 * allocates, never synchronises the device, and returns 0 on success or a
 * negative status (see COMOE_E*) with a message in comoe_last_error().
 * Buffers are owned by the caller (the Python host layer allocates them with
 * PyTorch). Kernels are sm_100a only.
 *
 * The reference (pkg/src/comoe, pure Python/NumPy) has no FFI; each function
 * below cites the reference function whose behaviour it implements or the
 * analytic charge it replaces. Ties always go to the lowest index (reference
 * convention, pkg/src/comoe/aggregation.py:165,193).
 */
#ifndef COMOE_B200_H_
#define COMOE_B200_H_

#ifdef __cplusplus
extern "C" {
#endif

#define COMOE_B200_ABI_VERSION 2

/* status codes */
#define COMOE_OK 0
#define COMOE_EBADARG (-1)
#define COMOE_EUNSUPPORTED (-2)
#define COMOE_ECUDA (-3)
#define COMOE_ENODRIVER (-4)

/* activations of the expert FFN */
#define COMOE_ACT_RELU 0   /* Switch: relu(x Wi^T) Wo^T                       */
#define COMOE_ACT_SWIGLU 1 /* Mixtral: (silu(x W1^T) * (x W3^T)) W2^T          */

/* grouped-GEMM epilogues */
#define COMOE_EPI_RELU 0
#define COMOE_EPI_SWIGLU 1
#define COMOE_EPI_SCALE_SCATTER 2
#define COMOE_EPI_STORE 3

/* element types for merge / similarity */
#define COMOE_DTYPE_BF16 0
#define COMOE_DTYPE_F64 1

/* ---------------------------------------------------------------- misc */
int comoe_version(void);
const char* comoe_last_error(void);
int comoe_num_sms(int device);

/* ---------------------------------------------------------------- K1 gate
 * Replaces the synthetic routing source generate_routing
 * (pkg/src/comoe/moe.py:186-230) with a real fp32 router, and applies
 * ModelVariant.resolve (pkg/src/comoe/aggregation.py:101-103) as `slot_map`.
 *
 * comoe_gate_prepare: split the fp32 router Wg[d,E] (row-major, x @ Wg) into
 *   three bf16 terms wg_split[3][EP][d] (EP = comoe_gate_padded_experts(E));
 *   hi + mid + lo == Wg exactly. comoe_gate_topk uses hi + mid by default
 *   (logit error ~3e-7 at d = 768) or all three (env COMOE_GATE_TERMS=3).
 * comoe_gate_topk: for each token t of x[T,d] (bf16): logits = x_t . Wg (fp32,
 *   tensor cores), top-k on the logits (k in {1,2}), probabilities
 *   (norm_topk=0: softmax over all E; 1: renormalised over the k picks),
 *   group = slot_map[expert] (identity if NULL; when both picks map to one
 *   group the second is folded into the first), token-order rank inside its
 *   128-token tile, and the per-tile group histogram tile_hist[k][ntiles][G].
 *   logits_out[T,E] is optional (NULL to skip).
 */
int comoe_gate_padded_experts(int E);
int comoe_gate_num_tiles(int T);
int comoe_gate_prepare(const float* wg, int d, int E, void* wg_split, void* stream);
int comoe_gate_topk(const void* x, int T, int d, const void* wg_split, int E, int top_k,
                    int norm_topk, const int* slot_map, int n_groups, float* logits_out,
                    int* expert_idx, int* group_idx, float* gate_prob, int* local_rank,
                    int* tile_hist, void* stream);

/* comoe_gate_route: comoe_gate_topk and comoe_route_scan in ONE launch
 * (the router with capacity masking as one kernel). The gate epilogue
 * stores each 128-token tile's group histogram; after the last tile the
 * persistent (co-resident) grid meets at a device-side barrier, each CTA
 * scans whole histogram columns in stream order, and the last CTA to finish
 * writes group_count /
 * group_kept / group_base. Outputs are identical to comoe_gate_topk followed
 * by comoe_route_scan (tile_offset[k][ntiles][G] included; tile_hist is not
 * written). `workspace` (comoe_gate_route_workspace_bytes, 16-byte aligned)
 * must be zero-filled once before its first use and is then
 * self-maintaining (a device-side epoch advances per launch, so CUDA-graph
 * replays need no reset); one workspace per concurrently running launch.
 * Replaces the routing source generate_routing (pkg/src/comoe/moe.py:186-230)
 * and the per-expert counts of collect_stats (moe.py:250-262).
 */
long comoe_gate_route_workspace_bytes(int T, int top_k, int n_groups);
int comoe_gate_route(const void* x, int T, int d, const void* wg_split, int E, int top_k,
                     int norm_topk, const int* slot_map, int n_groups, int capacity,
                     float* logits_out, int* expert_idx, int* group_idx, float* gate_prob,
                     int* local_rank, int* tile_offset, int* group_count, int* group_kept,
                     int* group_base, void* workspace, void* stream);

/* Replayed routing: the tables comoe_gate_topk produces after top-k, from
 * given expert choices expert_idx[T,k] (a reference RoutingTrace,
 * pkg/src/comoe/moe.py:146-162, or any external router) and optional
 * probabilities probs[T,k] (NULL -> 1/k). Same slot remap, fold, tile
 * ranks and histograms; G <= 1024.
 */
int comoe_route_from_indices(const int* expert_idx, const float* probs, int T, int E, int top_k,
                             const int* slot_map, int n_groups, int* group_idx, float* gate_prob,
                             int* local_rank, int* tile_hist, void* stream);

/* ---------------------------------------------------------------- routing scan
 * Capacity in stream order (first choices in token order, then second
 * choices): tile_offset = exclusive scan of tile_hist per group,
 * group_count = assignments per group (pre-capacity; the per-group analogue
 * of collect_stats, pkg/src/comoe/moe.py:250-262), group_kept =
 * min(count, capacity), group_base = exclusive scan of group_kept.
 */
int comoe_route_scan(const int* tile_hist, int top_k, int ntiles, int G, int capacity,
                     int* tile_offset, int* group_count, int* group_kept, int* group_base,
                     void* stream);
/* counts[E] = histogram of original expert indices (collect_stats, moe.py:250-262) */
int comoe_expert_histogram(const int* expert_idx, long n, int E, int* counts, void* stream);

/* ---------------------------------------------------------------- K2 permute
 * Kept assignments are copied to x_perm[group_base[g] + rank] (expert-sorted,
 * compact); row_token/row_prob describe each row; token_pos[T,k] = row or -1.
 * If y_zero != NULL, rows of tokens with no kept assignment are zeroed there
 * (the top-1 fused-combine output). x_perm == NULL computes the routing
 * tables only (the GEMM then gathers token rows itself, see a_gather).
 */
int comoe_permute(const void* x, int T, int d, int top_k, const int* group_idx,
                  const float* gate_prob, const int* local_rank, const int* tile_offset,
                  const int* group_base, int n_groups, int capacity, void* x_perm,
                  int* row_token, float* row_prob, int* token_pos, void* y_zero, void* stream);

/* ---------------------------------------------------------------- K3 expert FFN
 * Replaces the analytic expert charge (pkg/src/comoe/simulator.py:705,
 * scenario.py:471 expert_flops) with tcgen05 grouped GEMMs over the HBM
 * expert slot pool: slot s holds [W_in (N1 x d) | W_out (d x d_ff)] bf16,
 * N1 = d_ff (ReLU) or 2*d_ff (SwiGLU, gate/up interleaved in 128-row blocks).
 * Group g covers rows [group_row_base[g], +group_rows[g]) of x_perm and uses
 * slot group_slot[g]. h_work[total_rows, d_ff] is scratch. If row_token is
 * given, the second GEMM scales by row_prob and scatters rows to
 * out[row_token[r]] (fused top-1 combine); otherwise it stores rows in place.
 * Requires d, d_ff multiples of 256 and of 64.
 * comoe_grouped_gemm: one GEMM of the pair; if a_gather != NULL, row r of
 * group g of the token operand is row a_gather[group_row_base[g] + r] of `a`
 * (TMA gather4 straight from the unpermuted tokens — no permuted copy; ReLU
 * epilogue only). Outputs stay in the compact row order.
 */
int comoe_grouped_gemm(const void* a, long a_rows, const void* pool, int n_slots, long slot_stride,
                       long b_offset, int N, int K, const int* group_rows,
                       const int* group_row_base, const int* group_slot, int G, int epi_mode,
                       void* out, int ldo, const int* row_token, const float* row_prob,
                       const int* a_gather, void* stream);
int comoe_grouped_ffn(const void* x_perm, long total_rows, int d, int d_ff, int act,
                      const void* pool, int n_slots, long slot_stride, const int* group_rows,
                      const int* group_row_base, const int* group_slot, int G, void* h_work,
                      void* out, int ldo, const int* row_token, const float* row_prob,
                      void* stream);
/* comoe_fused_ffn: the whole expert FFN in one launch with H kept on chip
 * (GEMM1 -> ReLU -> bf16 H in TMEM/shared memory -> GEMM2; no h_work, no
 * H round trip through HBM). Same group table and output semantics as
 * comoe_grouped_ffn. If gather_rows != NULL, token row r of the permuted
 * order is row gather_rows[r] of x (TMA gather4 from the unpermuted tokens,
 * so no permuted copy is needed; pass the permute kernel's row_token).
 * ReLU experts with d % 256 == 0, d <= 768, d_ff % 256 == 0, G <= 256
 * (comoe_fused_ffn_supported says whether a shape qualifies). Opt-in: with
 * env COMOE_FUSED_FFN=1 (comoe_fused_ffn_enabled() == 1) comoe_grouped_ffn
 * takes this path by itself for qualifying shapes (h_work may then be NULL);
 * by default the two-launch FFN runs, which measured faster (K3F).
 */
int comoe_fused_ffn(const void* x, long x_rows, const int* gather_rows, int d, int d_ff,
                    const void* pool, int n_slots, long slot_stride, const int* group_rows,
                    const int* group_row_base, const int* group_slot, int G, void* out, int ldo,
                    const int* row_token, const float* row_prob, void* stream);
int comoe_fused_ffn_supported(int d, int d_ff, int act, int G);
int comoe_fused_ffn_enabled(void);
/* dev: per-CTA-pair wait-cycle counters of the last fused FFN launched with
 * env COMOE_FUSED_DEBUG bit 256 (128 x 16 unsigned long long; synchronises) */
int comoe_debug_fused_prof(unsigned long long* out);

/* ---------------------------------------------------------------- K4 combine
 * y[t] = sum_j gate_prob[t,j] * y_perm[token_pos[t,j]] (token_pos -1 -> 0).
 */
int comoe_combine(const void* y_perm, const int* token_pos, const float* gate_prob, int T, int d,
                  int top_k, void* y, void* stream);

/* ------------------------------------------------ EP over NVLink peer memory
 * Replaces the two ncclAllToAll of the EP layer (ep.py ep_forward; the
 * reference has no EP at all — SURVEY §8e/§8f rank 1). Every rank maps its
 * peers' receive / output / count / pad buffers through CUDA IPC; the send
 * layout row r = (dst * El + le) * C + slot lives at row
 * src * block_rows + r % block_rows of rank dst's buffer
 * (block_rows = El * C). All calls are stream-ordered and never allocate. */
int comoe_permute_peers(const void* x, int T, int d, int top_k, const int* group_idx,
                        const float* gate_prob, const int* local_rank, const int* tile_offset,
                        const int* group_base, int n_groups, int capacity,
                        void* const* peer_rows, int n_peers, long block_rows, int src_rank,
                        int* row_token, float* row_prob, int* token_pos, void* stream);
int comoe_combine_peers(const void* const* peer_rows, int n_peers, long block_rows, int src_rank,
                        const int* token_pos, const float* gate_prob, int T, int d, int top_k,
                        void* y, void* stream);
/* counts[E] (rows of global expert e from src_rank) -> peer_counts[e / El][src_rank * El + e % El] */
int comoe_peer_scatter_counts(const int* counts, int E, int world, int src_rank,
                              int* const* peer_counts, void* stream);
/* flag barrier: publish epoch (> 0, increasing) into every peer's pad slot
 * [rank], wait for every peer's epoch in mine; on timeout *err = 1 + peer
 * (the kernel returns instead of hanging). pads: device array of world
 * pointers to int[world] pads. */
int comoe_peer_barrier(int* const* pads, int world, int rank, int epoch, long long timeout_ns,
                       int* err, void* stream);
int comoe_ipc_handle_size(void);
/* handle of the allocation holding ptr, and ptr's offset inside it */
int comoe_ipc_get_handle(const void* ptr, void* handle_out, long* offset_out);
int comoe_ipc_open(const void* handle, long offset, void** ptr_out);
int comoe_ipc_close(void* ptr, long offset);

/* ---------------------------------------------------------------- K5 merge
 * merge_group (pkg/src/comoe/aggregation.py:200-215) for n_groups groups in
 * one launch: out[g] = (sum_{j in g} weights[j] * member[j]) / divisor[g].
 * Host passes weights = f_j, divisor = sum f (or 1 and n for the
 * zero-frequency plain mean). F64 reproduces numpy's order bit-exactly.
 * All pointer tables live in device memory.
 */
int comoe_merge(int dtype, const void* const* member_ptrs, const int* group_offsets,
                const double* weights, const double* divisor, void* const* out_ptrs, int n_groups,
                int max_members, long D, void* stream);

/* ---------------------------------------------------------------- K6 similarity
 * similarity_matrix (pkg/src/comoe/moe.py:339-365) in two device stages:
 * comoe_sim_contract: gram[E,E] = P P^T and logits[E,n,B] =
 *   sum_d probes[n,d] P[e,d] proj[b,d] (the einsum at moe.py:351), split-K
 *   over D with a deterministic reduction; rows are expert vectors (bf16 or
 *   f64, by dtype); probes/proj are f64 [n,D] / [B,D]; work is scratch of
 *   comoe_sim_workspace_bytes(E, n, B, D) bytes.
 * comoe_sim_finalize: S = alpha*cos + (1-alpha)*clip(1 - meanKL, 0, 1) with
 *   log-softmax surrogate distributions (finite where the reference NaNs).
 * n_probes = 0 selects the cosine term only (probes/proj/logits may be NULL;
 * the functional term is then the constant 1): real-scale experts (D ~ 1e8)
 * where materialising the reference's n x D fp64 calibration is infeasible.
 */
long comoe_sim_workspace_bytes(int E, int n_probes, int buckets, long D);
/* Cosine Gram of 9..128 bf16 experts stored as consecutive rows of one
 * stride (a layer's pool slots): expert e at base + e * row_stride
 * (elements). tcgen05 split-K, fp64 result in gram[E,E]; work:
 * comoe_sim_workspace_bytes(E, 0, 0, D) bytes. */
int comoe_sim_tc_supported(int E, long D);
int comoe_sim_gram_strided(const void* base, long row_stride, int E, long D, double* gram,
                           void* work, void* stream);
int comoe_sim_contract(int dtype, const void* const* rows, int E, long D, const double* probes,
                       int n_probes, const double* proj, int buckets, double* gram,
                       double* logits, void* work, void* stream);
int comoe_sim_finalize(const double* gram, const double* logits, int E, int n_probes, int buckets,
                       double alpha, double* sim, void* stream);

/* ---------------------------------------------------------------- K8 predictor
 * PredictorMLP.forward_batch (pkg/src/comoe/offload.py:147-154) with the
 * input built as in predict_next_layer (offload.py:157-172): x = [K-hot of
 * slots[t] over E | emb[t] | ctx[t]]; probs = softmax(W2 relu(W1 x + b1) + b2).
 * f64 throughout. demand[E] (optional), reduced in token order within fixed
 * 256-token chunks, then chunk order (deterministic): demand_mode 0 =
 * sum_t probs[t] (expected picks), 1 = 1 - prod_t (1 - probs[t]) (the
 * probability that some token of the batch picks the expert). It needs
 * `work` of comoe_predictor_workspace_bytes(B, E) bytes (unused when demand
 * is NULL).
 * The weights are staged in shared memory: (E+emb+ctx)*hidden + hidden*E
 * doubles (+ small terms) must fit 227 KB, else kUnsupportedShape.
 */
long comoe_predictor_workspace_bytes(int B, int E);
int comoe_predictor_mlp(const int* slots, int B, int K, const double* emb, int emb_dim,
                        const double* ctx, int ctx_dim, const double* w1, const double* b1,
                        int hidden, const double* w2, const double* b2, int E, double* probs,
                        double* demand, int demand_mode, void* work, void* stream);

/* dev: {clock64, ns} at the start and end of CTA 0 of the last 2-SM grouped
 * GEMM launched with COMOE_GEMM_DEBUG bit 256 — the SM clock under load */
int comoe_debug_gemm_clock(unsigned long long* out4);
/* dev: gate timeline of CTAs 0 and 1 ([2][1024] = [cta][code * 32 + unit
 * iteration] of 1 + cycles since entry, 0 = not reached; COMOE_GATE_DEBUG bit
 * 256), counts [2] = entries per CTA; resets them */
int comoe_debug_gate_timeline(unsigned long long* out, unsigned int* counts);
/* dev: router-in-TMEM gate variant for later launches (1 on, 0 off, -1: COMOE_GATE_TM) */
int comoe_debug_set_gate_tm(int on);
/* dev: override COMOE_GEMM_DEBUG for later grouped-GEMM launches (-1: env value) */
int comoe_debug_set_gemm(int debug);

#ifdef __cplusplus
}
#endif

#endif /* COMOE_B200_H_ */
