/*
 * dkv.h — C ABI of the B200-native DiffKV KV memory manager (arXiv 2412.03131).
 *
 * The library implements the data-parallel hot path of DiffKV's on-GPU memory manager ("parallel KV
 * compaction", §5 of the paper) as hand-written sm_100a CUDA kernels:
 *
 *   planning      dkv_classify      per-(request, layer, KV-head) significance classification and page
 *                                   demand — "each attention head independently determines its memory
 *                                   allocation requirements"; Algorithm 1 in the
 *                                   generation phase, §4's thresholds in the prompt phase.
 *   coordination  dkv_compact_alloc recycle finished requests' pages into the circular free list and grant
 *                                   every head its pages from one exclusive scan — "a parallel prefix sum
 *                                   operation computes a unique offset for each head relative to the start
 *                                   or end pointer"; bidirectional table writes.
 *   compressor    dkv_quant_write   quantize K/V into unified pages at K8V4 / K4V2 (P:173-177, P:347-349,
 *                                   P:466-471).
 *   release       dkv_free          "once a request is finished, all pages allocated for that request are
 *                                   recycled".
 *
 * Citation convention: "P:n" = line n of the paper's LaTeX source; "Qn" = reading n of the
 * ambiguity ledger in DESIGN.md §3.  No torch types cross this boundary: device buffers are plain
 * pointers, host buffers are plain pointers, streams are CUDA runtime streams (cudaStream_t).
 *
 * Ownership.  The caller owns the device arena (>= dkv_arena_bytes(), 256-byte aligned, e.g. a torch
 * uint8 CUDA tensor), every per-call device buffer and the streams.  The library owns only the host
 * handle (created by dkv_pool_init, released by dkv_pool_destroy) and a host mirror of request states.
 * It never allocates device memory after dkv_pool_init and keeps no reference to per-call buffers beyond
 * stream-ordered execution; the arena must outlive the handle.  One handle = one host thread, calls
 * ordered on one stream (or event-synchronised).
 *
 * Errors.  Host-detectable errors (bad arguments, request state, call order) return a negative status
 * immediately, enqueue nothing and change nothing.  Device-detected errors (OOM, non-finite input,
 * table overflow) are recorded in a sticky device status word — first error wins; while it is set
 * dkv_classify / dkv_quant_write kernels are no-ops and dkv_compact_alloc only recycles.  dkv_pool_query
 * returns and clears it and re-synchronises the host mirror.  The product path has no CPU fallback:
 * every call fails with DKV_ERR_CUDA when no CUDA device is usable.
 *
 * Determinism.  Every output (decisions, ring, pointers, tables, counts, page bytes, window) is a pure
 * function of the inputs and the pool state, identical for any launch configuration (tile size).
 */
#ifndef DKV_H
#define DKV_H
#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef struct CUstream_st* dkv_stream_t;       /* a cudaStream_t; NULL = legacy default stream */
typedef struct dkv_pool* dkv_pool_t;            /* opaque host handle */
typedef int32_t dkv_status_t;

enum {
  DKV_OK = 0,
  DKV_ERR_INVALID_ARG = -1,   /* bad config / pointer / size / request id */
  DKV_ERR_STATE = -2,         /* request state or call order violated (host-detected) */
  DKV_ERR_OOM = -3,           /* device: demand > free pages; allocation not applied (Q15) */
  DKV_ERR_NONFINITE = -4,     /* device: NaN/Inf K/V, or significance NaN/Inf/negative */
  DKV_ERR_OVERFLOW = -5,      /* device: table slot collision (unreachable by construction, Q12) */
  DKV_ERR_CUDA = -6           /* CUDA runtime error (no device, launch failure, ...) */
};
enum { DKV_PHASE_DECODE = 0, DKV_PHASE_PREFILL = 1 };
enum { DKV_CLS_NONE = 0, DKV_CLS_HIGH = 1, DKV_CLS_LOW = 2, DKV_CLS_PRUNED = 3 };
enum { DKV_V_NONE = 0, DKV_V_KEEP = 1, DKV_V_DOWN = 2, DKV_V_PRUNE = 3 };
enum { DKV_GROW_NONE = 0, DKV_GROW_HIGH = 1, DKV_GROW_LOW = 2 };
enum { DKV_REQ_IDLE = 0, DKV_REQ_ADMITTING = 1, DKV_REQ_ACTIVE = 2, DKV_REQ_PENDING_FREE = 3 };

/* Pool configuration.  Units u = (r*num_layers + l)*num_kv_heads + h (Q13).
 * Constraints: head_dim in {64, 128}; bits in {2, 4, 8} with key bits >= 2; page_tokens_* multiples of 4,
 * page_tokens_low >= page_tokens_high ("low-precision pages always contain more tokens");
 * 1 <= num_pages < 2^31; window >= 0; alpha finite >= 0; units * table_len < 2^28. */
typedef struct {
  int32_t max_requests;        /* R: request slots */
  int32_t num_layers;          /* Ly */
  int32_t num_kv_heads;        /* H: KV heads held by THIS pool (one GPU's shard) */
  int32_t head_dim;            /* d */
  int32_t max_seq_len;         /* M: tokens per request incl. window */
  int32_t window;              /* W: recent FP16 window, "typically set to 64" (Q10) */
  int32_t page_tokens_high;    /* C_h (Q11) */
  int32_t page_tokens_low;     /* C_l (Q11) */
  int32_t kbits_high, vbits_high, kbits_low, vbits_low;   /* 8,4 / 4,2 = K8V4 / K4V2 */
  int32_t num_pages;           /* P */
  float   alpha_h, alpha_l;    /* thresholds (calibrated values P:702-703) */
  int32_t prompt_denominator;  /* Q4: 0 = 1-indexed position i; 1 = prompt length n */
  int32_t tile_units;          /* scan tile (units per CTA): 0 = default 1024; 256, 512 or 1024 */
  int32_t prefill_workflow;    /* prompt-phase allocation: 0 = exact (plan, then allocate ceil(n_h/C_h) +
                                  ceil(n_l/C_l) pages per head); 1 = the paper's workflow (Fig. 5):
                                  allocate ceil(kept/C_h) pages per head "assuming all tokens are stored at
                                  high precision", plan, keep high pages from the left and low pages from
                                  the right of each head's block, reclaim the middle at the end pointer
                                  (one extra page when the plan needs it, reading Q29).  Same final
                                  classes, counts and page bytes; different page IDs and ring order. */
  int32_t q_per_kv;            /* NEXT-2 (dkv_attend): query heads per KV head, the GQA group;
                                  0 = no attention; supported: 1, 2, 4, 5, 7, 8 */
  /* NEXT-4 three-level tier FP16-K8V4-K4V2 (readings Q38-Q44 of DESIGN.md): top_tier = 1 adds
     the FP16 class TOP above High — tokens with significance >= alpha_t / den (prompt) or alpha_t / N (decode)
     are kept unquantized, page_tokens_top (multiple of 4) per page, in a unidirectional table filled left to
     right next to the bidirectional one.  Requires alpha_t >= alpha_h, prefill_workflow = 0; dkv_attend and
     dkv_attend_tc return DKV_ERR_INVALID_ARG with the tier. */
  int32_t top_tier;
  float   alpha_t;
  int32_t page_tokens_top;
} dkv_config_t;
enum { DKV_CLS_TOP = 4, DKV_GROW_TOP = 3 };          /* NEXT-4: decision codes of the FP16 tier */

/* 16-byte per-unit decision written by dkv_classify(DECODE); padding-free, compared byte for byte.
 * tc_class: class of t_c, the token leaving the window, or NONE when the request is not
 *   ACTIVE or has no token outside the window.  v_action: fate of the victim t_v = lexicographic argmin
 *   of (score, position) over the section t_c joins (Q6/Q7).  grow: section gaining a token.
 *   demand: 1 iff the growing section's tail page is full.  Slots are section slot indices
 *   (-1 if none): v_slot = victim's slot, tc_slot = where t_c is written (t_c takes the victim's slot when
 *   the victim leaves, Q8), v_dst_slot = KV_l slot of a downgraded victim. */
typedef struct {
  uint8_t tc_class, v_action, grow, demand;
  int32_t v_slot, tc_slot, v_dst_slot;
} dkv_decision_t;

typedef struct {
  int64_t free_pages, used_pages, start, last_demand, last_freed;
  int32_t status, oom_count;
} dkv_stats_t;

/* Byte offsets of every buffer inside the arena plus the page segment geometry (Q18: segments in
 * the paper's order — K codes, K meta {s16,z16}, V codes, V meta, fp32 scores, int32 positions — each on
 * a 16-byte boundary, token-major rows, codes packed LSB-first (Q17)).  Index 1 = high, 2 = low. */
typedef struct {
  int64_t arena_bytes;
  int64_t off_ctrl, off_tile_status, off_ring, off_table, off_n_h, off_n_l, off_req_state, off_seq_len,
          off_prompt_len, off_admit, off_pf_nh, off_pf_nl, off_pf_seg, off_win_k, off_win_v, off_pages,
          off_stats;
  int32_t units, table_len, page_bytes, num_tiles, tile_units, seg_tokens, num_segs;
  int32_t C[3], k_row[3], v_row[3], off_k[3], off_kmeta[3], off_v[3], off_vmeta[3], off_score[3], off_pos[3];
  int64_t off_tile_sums;       /* int64[num_tiles][3] scratch of the prompt workflow's scans */
  int64_t off_rec;             /* int32[units][3] scratch of the deferred recycle copy */
  int64_t off_win_sig;         /* fp32[units][window]: significance of the window tokens (NEXT-2) */
  int64_t off_secmin;          /* int32[units][8]: per-section (significance, position, slot) minima written by
                                  dkv_attend, consumed by the next dkv_classify(DECODE) (NEXT-2) */
  int64_t off_head_alpha;      /* fp32[layers * kv_heads][2]: per-head (alpha_h, alpha_l) (NEXT-4) */
  int64_t off_att_scratch;     /* NEXT-2 long contexts: 296 slots of (ceil4(q_per_kv) + 2) * max_seq_len fp32 when
                                  those do not fit in shared memory (0 bytes otherwise) */
  int64_t off_ttable;          /* NEXT-4: int32[units][table_len_top] TOP page table (left to right) */
  int64_t off_n_t;             /* NEXT-4: int32[units] stored TOP tokens */
  int32_t table_len_top;       /* NEXT-4: ceil(max_seq_len / page_tokens_top), 1 without the tier */
  int32_t C_top, row_top, off_k_top, off_v_top, off_score_top, off_pos_top;   /* TOP page geometry (fp16 rows) */
  int64_t off_qpid;            /* int32[units][4] {page of t_c's slot (= the victim's KV_h page when it is
                                  downgraded), page of a downgraded victim's KV_l slot, the request length N
                                  when it is ACTIVE else 0, 0}: written by dkv_classify(DECODE) (existing pages,
                                  N) and by dkv_compact_alloc (granted pages), read by dkv_quant_write(DECODE)
                                  instead of the tables and the request state */
  int64_t off_tsum;            /* uint32[2][num_tiles][2] decode tile sums {demand, freed pages} that
                                  dkv_classify(DECODE) accumulates for the following dkv_compact_alloc (by the
                                  parity of the call counter) */
  int64_t off_tc_scratch;      /* dkv_attend_tc: 2 x 592 buffers of (max_seq_len rounded to 32, + 64) * (4 if
                                  q_per_kv <= 4 else 8) fp32 logit rows, two per persistent CTA (0 bytes when
                                  q_per_kv = 0 or with the FP16 tier) */
} dkv_layout_t;

/* Arena size for `cfg`, or 0 if the configuration is invalid. */
size_t dkv_arena_bytes(const dkv_config_t* cfg);

/* Fill *out with the arena layout of `cfg` (host only, no CUDA call).  DKV_ERR_INVALID_ARG if invalid. */
dkv_status_t dkv_pool_layout(const dkv_config_t* cfg, dkv_layout_t* out);

/* Carve `d_arena` (device, >= dkv_arena_bytes, 256-B aligned) and initialise it on `s`: ring = iota,
 * start = 0, free = P, tables = -1, counts = 0, pages and window zeroed.  *out receives the
 * handle.  Asynchronous on `s`. */
dkv_status_t dkv_pool_init(const dkv_config_t* cfg, void* d_arena, size_t arena_bytes, dkv_stream_t s,
                           dkv_pool_t* out);
dkv_status_t dkv_pool_destroy(dkv_pool_t p);

/* Planning.
 * DECODE : every ACTIVE request appends one token this step.  d_sig = device fp32[U]: significance of
 *          each unit's t_c (values for non-ACTIVE units are ignored), or NULL: t_c's significance is the one
 *          kept for its window slot (NEXT-2, maintained by dkv_attend).  Writes d_dec[U] (device).
 *          h_req/h_len/n/sig_stride/d_token_class unused (NULL/0).  DKV_ERR_STATE if an ACTIVE request
 *          already holds max_seq_len tokens.
 * PREFILL: admits host arrays h_req[0..n) (IDLE -> ADMITTING) with prompt lengths h_len[0..n) <= M.
 *          d_sig = device fp32[n][Ly*H][sig_stride] (request-major in h_req order, then l, then h; token
 *          t at index t; sig_stride >= max prompt length).  Per-unit class counts and per-segment ranks go
 *          to pool scratch; if d_token_class != NULL it receives u8[n][Ly*H][sig_stride] classes
 *          (DKV_CLS_*, NONE for window tokens).  d_dec unused. */
dkv_status_t dkv_classify(dkv_pool_t p, int32_t phase, const int32_t* h_req, const int32_t* h_len, int32_t n,
                          const float* d_sig, int64_t sig_stride, dkv_decision_t* d_dec, uint8_t* d_token_class,
                          dkv_stream_t s);

/* Coordination.  Recycles every PENDING_FREE request (its pages go to the ring at end = start + free in
 * canonical order, Q13; the request becomes IDLE), then grants the demand of the most recent dkv_classify
 * all-or-nothing (Q15): decode demand from d_dec (device, as written by dkv_classify(DECODE)); prefill
 * demand ceil(n_h/C_h) + ceil(n_l/C_l) from pool scratch (d_dec may be NULL), or with prefill_workflow = 1
 * the conservative block ceil(kept/C_h) (+1, Q29) whose unused middle is reclaimed in the same call.  Writes the bidirectional
 * tables (high left-to-right, low right-to-left) and counts, advances start/free.  On OOM: sticky
 * DKV_ERR_OOM, allocation state unchanged, recycling applied.  May be re-issued with the same d_dec
 * after an OOM (only ACTIVE / ADMITTING requests take part). */
dkv_status_t dkv_compact_alloc(dkv_pool_t p, const dkv_decision_t* d_dec, dkv_stream_t s);

/* KV compressor.
 * DECODE : d_dec as above; d_k/d_v = device fp16 bits [U][d], the new token of each unit (pushed into the
 *          window); d_sig = the same cand_sig as dkv_classify; kv_stride/sig_stride unused (0).  For each
 *          ACTIVE unit: downgrade t_v (re-quantize its stored K8V4 values at K4V2, Q9), quantize t_c out of
 *          the window into tc_slot, then write the new token into window slot (N-1) mod W.
 * PREFILL: d_k/d_v = device fp16 bits [n][Ly*H][kv_stride][d], d_sig = [n][Ly*H][sig_stride] as given to
 *          dkv_classify(PREFILL); writes every kept token into its pages (slot = rank within its class in
 *          position order) and the newest min(W, n) tokens into the window; ADMITTING -> ACTIVE. */
dkv_status_t dkv_quant_write(dkv_pool_t p, int32_t phase, const dkv_decision_t* d_dec, const uint16_t* d_k,
                             const uint16_t* d_v, int64_t kv_stride, const float* d_sig, int64_t sig_stride,
                             dkv_stream_t s);

/* NEXT-2 — decode attention over the compressed cache with the significance update (P:360-361, P:573-608,
 * readings Q31-Q34 of DESIGN.md).  For every ACTIVE unit: the q_per_kv query heads d_q (device fp16 bits
 * [U][q_per_kv][d], the newest token's queries) attend over the unit's stored tokens (keys and values
 * dequantized from their pages, X^ = s*Q + z) and its FP16 window (which holds the newest token after
 * dkv_quant_write(DECODE)); softmax(q.k / sqrt(d)); every token's significance becomes the running mean of
 * the (max over the group) scores it received from later queries — in place, in the page score segments
 * and the window's significance array — and each section's (significance, position) minimum is recorded so
 * the next dkv_classify(DECODE) needs no scan.  d_out (device fp32 [U][q_per_kv][d]) receives the attention
 * output, d_probs (device fp32 [U][max_seq_len]) the per-token scores (max over the group) in token order
 * (high slots, low slots, window oldest first); either may be NULL.  Deterministic: every floating-point
 * result is fixed by Q31-Q34 (bit-identical to the oracle).  Allowed between sequences; DKV_ERR_INVALID_ARG
 * if q_per_kv is 0 / unsupported.  Long contexts (logits beyond shared memory) run a persistent form whose
 * logits live in the arena's scratch slots (off_att_scratch).
 * With NEXT-2 the decode step passes d_sig = NULL to dkv_classify / dkv_quant_write: t_c's significance is
 * then read from the window. */
dkv_status_t dkv_attend(dkv_pool_t p, const uint16_t* d_q, float* d_out, float* d_probs, dkv_stream_t s);

/* NEXT-2 on tensor cores — the same operation as dkv_attend (Eq. 1 with GQA max, the running-mean significance
 * written back, the section minima for the next dkv_classify), computed with mma.sync tensor-core contractions on
 * the integer codes: logit = (s * q.codes + z * sum(q)) / sqrt(d), out = sum_t (a s) codes + sum_t a z, fp32
 * accumulation, the FP16 window on the same tensor-core path (online softmax, one pass over the pages).  Not bit-identical to dkv_attend / the oracle: results agree with
 * Eq. 1 evaluated in float64 to the tolerances of tests/test_gpu_attention_tc.py (outputs rtol 2e-4 / atol 2e-5,
 * scores rtol 2e-5 / atol 1e-7); the section minima are exact for the significance values it writes.  Same
 * arguments and errors as dkv_attend.  Falls back to dkv_attend when a class's pages are not the paper's K8V4 x16 /
 * K4V2 x32 tiles.  Persistent CTAs; each keeps its units' logits in its own two buffers of the arena's
 * off_tc_scratch (a unit's significance pass runs during the CTA's next unit).  With fewer ACTIVE units than SMs
 * and a longest request of >= 2048 tokens, the split-sequence form runs instead: each unit's pages split
 * over up to 32 CTAs whose partial softmax states are merged; same results to the same tolerances. */
dkv_status_t dkv_attend_tc(dkv_pool_t p, const uint16_t* d_q, float* d_out, float* d_probs, dkv_stream_t s);

/* Debug audit of the pool's invariants on the device (SURVEY §8 audit row): the memory layout of P:466-500
 * — every page of the unified pool is in the circular free list's free region [start, start + free) or in exactly
 * one occupied page-table slot; a unit's high pages fill its table row left to right and its low pages right to
 * left, so its occupied slots are exactly [0, ceil(n_h/C_h)) and [L - ceil(n_l/C_l), L) (and
 * [0, ceil(n_t/C_t)) of the NEXT-4 TOP table) and every other slot is -1 — and, for ACTIVE requests, every
 * stored position is unique within its unit and below N - W (a stored token has left the recent window).
 * d_scratch: caller-owned device buffer of at least num_pages uint32 (overwritten, a per-page histogram).
 * d_result: caller-owned device int64[8], overwritten with {pages owned more than once, pages owned by nobody,
 *   bad slots (an occupied slot or free-region entry outside [0, P), or an unoccupied slot != -1), used pages
 *   (occupied slots), free pages, duplicate stored positions, stored positions out of range, units whose page
 *   counts exceed their table}; a sound pool has zeros except used + free = num_pages.
 * Asynchronous on `s`; between sequences only (DKV_ERR_STATE otherwise); modifies nothing of the pool. */
dkv_status_t dkv_audit(dkv_pool_t p, uint32_t* d_scratch, int64_t* d_result, dkv_stream_t s);

/* NEXT-4 — per-head thresholds ("a shared set of thresholds for all attention heads" is the
 * paper's choice; per-head thresholds its stated extension; reading Q35).  h_alpha_h / h_alpha_l: host
 * arrays of num_layers * num_kv_heads finite values >= 0 in (layer, this pool's head) order; unit u uses
 * entry u mod (num_layers * num_kv_heads) in every classification (prompt thresholds alpha / i, Algorithm 1
 * thresholds alpha / N).  NULL restores the pool-wide alpha_h / alpha_l.  Between sequences only; the
 * values are copied on `s` (the host arrays may be reused once the call returns). */
dkv_status_t dkv_set_head_thresholds(dkv_pool_t p, const float* h_alpha_h, const float* h_alpha_l, dkv_stream_t s);

/* The whole decode step from HOST buffers — the e2e path (P:457-459 planning, P:485-488 coordination,
 * P:557 compressor; the three calls above in order).  h_sig: host fp32 [U] cand_sig as for
 * dkv_classify(DECODE), or NULL (NEXT-2: significance from the window); h_kv: host fp16 bits [2][U][d],
 * the new tokens' keys then values; h_dec: host dkv_decision_t[U] receiving the decisions, or NULL.
 * Host buffers should be pinned (page-locked) for the copies to be asynchronous.  d_stage: caller-owned
 * device staging of at least dkv_decode_stage_bytes(p) bytes (decisions, significance, K/V; it must
 * outlive the step's work on s).  The K/V copy runs on a library-owned copy stream (created on first use,
 * destroyed with the handle), ordered after the work already on s and overlapping classify +
 * compact_alloc; quant_write waits for it.  Every host-detectable error (call order, an ACTIVE request at
 * max_seq_len) is reported before anything is queued.  Results are identical to the three separate calls.  Asynchronous like the other calls: h_dec is valid once s has
 * completed.  Errors: DKV_ERR_INVALID_ARG (NULL handle / h_kv / d_stage, staging too small), otherwise
 * those of dkv_classify / dkv_compact_alloc / dkv_quant_write (the step stops at the first failing one). */
size_t dkv_decode_stage_bytes(dkv_pool_t p);
dkv_status_t dkv_decode_step_host(dkv_pool_t p, const float* h_sig, const uint16_t* h_kv, dkv_decision_t* h_dec,
                                  void* d_stage, size_t stage_bytes, dkv_stream_t s);

/* The decode step as a CUDA graph (launch-bound inner loop).  Captures `steps` consecutive
 * decode steps — each dkv_classify(DECODE) -> dkv_compact_alloc -> dkv_quant_write(DECODE), the same kernels and
 * results as the eager calls — into one CUDA graph replayed by dkv_decode_graph_launch.  Step t reads the
 * caller's device buffers d_sig + t*sig_step (fp32 [U], or d_sig NULL: significance from the window, NEXT-2),
 * d_k + t*kv_step and d_v + t*kv_step (fp16 bits [U][d]); a step of 0 reuses one buffer (update it between
 * launches).  Decisions go to d_dec (device [U]).  The buffers must outlive the graph.  Nothing in the step
 * depends on host state: a freed request's pages are recycled by the first step after dkv_free (its copies
 * done by that step's quant_write kernel), and the classify kernel form follows max_seq_len.
 * flags: DKV_GRAPH_PDL — programmatic dependent launch between the kernels (each kernel's launch and
 * prologue overlap its predecessor; every kernel waits (griddepcontrol.wait) before reading its predecessor's
 * output); DKV_GRAPH_EVENTS — an event node around each kernel for per-kernel times
 * (dkv_decode_graph_kernel_ms: h_ms[steps][3] = classify, compact_alloc, quant_write in ms; disables PDL).
 * Create: between sequences (DKV_ERR_STATE otherwise); DKV_ERR_CUDA if capture fails.  Launch: between
 * sequences, with every ACTIVE request at most max_seq_len - steps long (DKV_ERR_STATE otherwise, nothing
 * enqueued); asynchronous on `s`; the host mirror advances by `steps` steps.  Device errors follow the sticky
 * status rules above (dkv_pool_query after the launch reports them). */
typedef struct dkv_graph* dkv_graph_t;
enum { DKV_GRAPH_PDL = 1, DKV_GRAPH_EVENTS = 2 };
dkv_status_t dkv_decode_graph_create(dkv_pool_t p, int32_t steps, const float* d_sig, int64_t sig_step,
                                     const uint16_t* d_k, const uint16_t* d_v, int64_t kv_step, dkv_decision_t* d_dec,
                                     int32_t flags, dkv_graph_t* out);
dkv_status_t dkv_decode_graph_launch(dkv_graph_t g, dkv_stream_t s);
dkv_status_t dkv_decode_graph_kernel_ms(dkv_graph_t g, float* h_ms);
dkv_status_t dkv_decode_graph_destroy(dkv_graph_t g);

/* Release: host array h_req[0..n) of ACTIVE requests -> PENDING_FREE (double free / not active ->
 * DKV_ERR_STATE).  Allowed between sequences only (after dkv_quant_write, before dkv_classify).  Pages are
 * recycled by the next dkv_compact_alloc; the slot is IDLE (re-admissible) after that call. */
dkv_status_t dkv_free(dkv_pool_t p, const int32_t* h_req, int32_t n, dkv_stream_t s);

/* Synchronises `s`; fills *out; returns the sticky device status (DKV_OK if none) and clears it; re-syncs
 * the host mirror of request states and lengths from the device. */
dkv_status_t dkv_pool_query(dkv_pool_t p, dkv_stats_t* out, dkv_stream_t s);

/* Device address of the pool's int64[4] admission counters {free_pages, -last_demand, -used_pages,
 * status} (status <= 0, so the MIN shows an error on any GPU), rewritten by every dkv_compact_alloc — the payload of the per-step count all-reduce (MIN). */
int64_t* dkv_pool_stats_device_ptr(dkv_pool_t p);

const char* dkv_status_string(dkv_status_t st);

#ifdef __cplusplus
}
#endif
#endif /* DKV_H */
