/*
 * dkv_oracle.h — serial CPU oracle for DiffKV's on-GPU KV memory manager (arXiv 2412.03131).
 *
 * TEST INFRASTRUCTURE ONLY.  Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline /
 * --impl reference legs may load this library.  The product path (paper_2412_03131_b200/) never
 * includes, links or calls anything under oracle/, and this file includes nothing from the product.
 *
 * Citation convention: "P:n" = /root/reference/PAPER.md line n (LaTeX source of the paper).
 * Readings Q1..Q25 are the ambiguity ledger in DESIGN.md §3.
 *
 * Everything here is a plain, slow, obviously-correct transcription: one request, one unit, one
 * token, one slot at a time, in canonical order, no blocking, no fusion.
 */
#ifndef DKV_ORACLE_H
#define DKV_ORACLE_H
#include <stdint.h>
#include <stddef.h>

#ifdef __cplusplus
extern "C" {
#endif

enum { ORC_OK = 0, ORC_ERR_INVALID = -1, ORC_ERR_STATE = -2, ORC_ERR_OOM = -3,
       ORC_ERR_NONFINITE = -4, ORC_ERR_OVERFLOW = -5 };
enum { ORC_DECODE = 0, ORC_PREFILL = 1 };
enum { ORC_CLS_NONE = 0, ORC_CLS_HIGH = 1, ORC_CLS_LOW = 2, ORC_CLS_PRUNED = 3, ORC_CLS_TOP = 4 };   /* TOP: NEXT-4 FP16 tier */
enum { ORC_V_NONE = 0, ORC_V_KEEP = 1, ORC_V_DOWN = 2, ORC_V_PRUNE = 3 };
enum { ORC_GROW_NONE = 0, ORC_GROW_HIGH = 1, ORC_GROW_LOW = 2, ORC_GROW_TOP = 3 };
enum { ORC_REQ_IDLE = 0, ORC_REQ_ADMITTING = 1, ORC_REQ_ACTIVE = 2, ORC_REQ_PENDING_FREE = 3 };

typedef struct {
  int32_t R, Ly, H, d;          /* request slots, layers, KV heads (this shard), head_dim */
  int32_t M, W;                 /* max sequence length, recent window */
  int32_t Ch, Cl;               /* tokens per high / low page (Q11) */
  int32_t kbh, vbh, kbl, vbl;   /* K8V4 high, K4V2 low */
  int32_t P;                    /* pages in the pool */
  float alpha_h, alpha_l;       /* thresholds */
  int32_t prompt_denominator;   /* Q4: 0 = 1-indexed position i, 1 = prompt length n */
  int32_t prefill_workflow;     /* 0 = exact allocation after planning; 1 = the paper's prompt workflow
                                   (Fig. 5): conservative allocation, planning, reclaim (Q29) */
  int32_t q_per_kv;             /* NEXT-2: query heads per KV head (GQA group); 0 = no attention */
  /* NEXT-4 three-level tier FP16-K8V4-K4V2 (readings Q38-Q44): 1 adds the FP16 class TOP
     above High, threshold alpha_t >= alpha_h, pages of Ct FP16 tokens in a unidirectional table */
  int32_t top_tier;
  float alpha_t;
  int32_t Ct;
} orc_config;

/* 16-byte decision record per unit (same byte layout the product's ABI documents). */
typedef struct {
  uint8_t tc_class, v_action, grow, demand;
  int32_t v_slot, tc_slot, v_dst_slot;
} orc_decision;

/* Page segment geometry of one precision class (Q18). */
typedef struct {
  int32_t C, kbits, vbits;
  int32_t k_row, v_row;                     /* bytes of one token's packed K / V codes */
  int32_t off_k, off_kmeta, off_v, off_vmeta, off_score, off_pos, end;
} orc_class_geom;

typedef struct orc_pool {
  orc_config c;
  int32_t U, L, page_bytes;
  orc_class_geom g[5];                      /* index ORC_CLS_HIGH / ORC_CLS_LOW / ORC_CLS_TOP */
  int32_t *ring; int64_t start, free;       /* circular free page list */
  int32_t *table;                           /* [U][L] bidirectional page table */
  int32_t *n_h, *n_l;                       /* [U] stored tokens per section */
  int8_t  *req_state;                       /* [R] */
  int32_t *seq_len, *prompt_len;            /* [R] */
  uint8_t *pages;                           /* [P][page_bytes] unified pages */
  uint16_t *win_k, *win_v;                  /* [U][W][d] fp16 bits, FP16 recent window (Q10) */
  int32_t *pf_nh, *pf_nl;                   /* [U] prefill class counts (c.6) */
  int32_t *admit_list; int32_t n_admit;     /* prefill: admitted request ids in call order */
  int32_t status;                           /* sticky device-style status, first error wins */
  int32_t last_phase;                       /* phase of the most recent classify */
  int64_t last_demand, last_freed; int32_t oom_count;
  int64_t last_reclaimed;                   /* prefill_workflow 1: middle pages reclaimed by the last call */
  float   *win_sig;                         /* [U][W] significance of the window tokens (running averages) */
  float   *head_ah, *head_al;               /* NEXT-4: [Ly*H] per-(layer, head) thresholds (Q35) */
  int32_t use_head;                         /* 1: the per-head thresholds replace alpha_h / alpha_l */
  int32_t Lt;                               /* NEXT-4: slots of the unidirectional FP16 (TOP) table */
  int32_t *ttable;                          /* [U][Lt] TOP page table, filled left to right (Q41) */
  int32_t *n_t, *pf_nt;                     /* [U] stored TOP tokens; prefill TOP counts */
} orc_pool;

/* --- scalar primitives (exported for the pins) --- */
uint16_t orc_f16_from_f32(float x);         /* IEEE binary16, round-to-nearest-even */
float    orc_f32_from_f16(uint16_t h);
void     orc_f16_from_f32_array(const float* x, uint16_t* out, int64_t n);
/* Quantize x[0..d) at `bits` (Q16): packed codes (d*bits/8 bytes, LSB-first, Q17) and fp16 s, z.
   Returns ORC_OK or ORC_ERR_NONFINITE / ORC_ERR_INVALID. */
int32_t  orc_quantize(const float* x, int32_t d, int32_t bits, uint8_t* codes, uint16_t* s16, uint16_t* z16);
void     orc_dequantize(const uint8_t* codes, int32_t d, int32_t bits, uint16_t s16, uint16_t z16, float* out);

/* --- geometry --- */
int32_t  orc_geometry(const orc_config* c, int32_t* U, int32_t* L, int32_t* page_bytes, orc_class_geom* high, orc_class_geom* low);
int64_t  orc_table_bytes(int64_t batch, int64_t layers, int64_t kv_heads, int64_t L);

/* --- pool --- */
orc_pool* orc_pool_new(const orc_config* c);
void      orc_pool_delete(orc_pool* p);
int32_t   orc_classify_decode(orc_pool* p, const float* cand_sig, orc_decision* dec);
int32_t   orc_classify_prefill(orc_pool* p, const int32_t* req, const int32_t* len, int32_t n,
                               const float* sig, int64_t sig_stride, uint8_t* token_class);
int32_t   orc_compact_alloc(orc_pool* p, const orc_decision* dec);
int32_t   orc_quant_write_decode(orc_pool* p, const orc_decision* dec, const uint16_t* k_new,
                                 const uint16_t* v_new, const float* cand_sig);
int32_t   orc_quant_write_prefill(orc_pool* p, const uint16_t* k, const uint16_t* v, int64_t kv_stride,
                                  const float* sig, int64_t sig_stride);
int32_t   orc_free(orc_pool* p, const int32_t* req, int32_t n);
int32_t   orc_take_status(orc_pool* p);     /* returns and clears the sticky status */
/* NEXT-2: decode attention of every ACTIVE unit's G query heads over its stored
   (dequantized) tokens and its FP16 window, then the running-average significance update (Q31-Q34).
   q = fp16 bits [U][G][d]; out = fp32 [U][G][d] (may be NULL); probs (may be NULL) = fp32 [U][M] per-token
   attention (max over the G heads) in token order (high slots, low slots, window oldest first). */
int32_t   orc_attend(orc_pool* p, const uint16_t* q, float* out, float* probs);
float     orc_exp(float x);                 /* the normative exp of Q32 (x <= 0) */
/* NEXT-4: per-(layer, KV head) thresholds, arrays of Ly*H finite values >= 0 in (l, h) order;
   NULL restores the pool-wide alpha_h / alpha_l.  Allowed between sequences. */
int32_t   orc_set_head_thresholds(orc_pool* p, const float* alpha_h, const float* alpha_l);

/* NEXT-1 (Fig. 5): admit + plan + compact with prefill_workflow = 1 for this call (the
   pool's own setting is restored); reclaimed_out receives the reclaimed page IDs in ring order. */
int32_t   orc_prefill_conservative(orc_pool* p, const int32_t* req, const int32_t* len, int32_t n,
                                   const float* sig, int64_t sig_stride, int32_t* reclaimed_out, int64_t* n_reclaimed);

#ifdef __cplusplus
}
#endif
#endif
