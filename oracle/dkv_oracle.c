/*
 * dkv_oracle.c — serial CPU oracle for DiffKV's on-GPU KV memory manager (arXiv 2412.03131).
 *
 * TEST INFRASTRUCTURE ONLY (see dkv_oracle.h).  Built with -O2 -ffp-contract=off, no fast-math:
 * every float expression below is one IEEE binary32 operation rounded to nearest-even, in the order
 * written.  Shares no code with the CUDA path.
 *
 * Structure follows the paper:
 *   §2.2   asymmetric per-vector quantization            -> orc_quantize / orc_dequantize
 *   §4   prompt-phase classification                   -> orc_classify_prefill
 *   Alg.1  generation-phase policy                       -> orc_classify_decode
 *   §5.2   unified pages, circular free list, bidir table-> orc_geometry, orc_compact_alloc
 *   §5.3   compaction workflow (prompt / generation)     -> orc_compact_alloc, orc_quant_write_*,
 *                                                                       orc_prefill_conservative (Fig. 5)
 */
#include "dkv_oracle.h"
#include <math.h>
#include <stdlib.h>
#include <string.h>

/* ------------------------------------------------------------------------------------------------
 * IEEE binary16 conversion, round-to-nearest-even (Q16: "FP16 RNE").  value = m * 2^E exactly;
 * pick the binary16 quantum 2^k for its magnitude, round m*2^(E-k) to an integer with RNE.
 * ----------------------------------------------------------------------------------------------*/
uint16_t orc_f16_from_f32(float x) {
  uint32_t b;
  memcpy(&b, &x, 4);
  uint16_t sign = (uint16_t)((b >> 16) & 0x8000u);
  uint32_t exp = (b >> 23) & 0xFFu, man = b & 0x7FFFFFu;
  if (exp == 0xFFu) return (uint16_t)(sign | (man ? 0x7E00u : 0x7C00u));
  if (exp == 0 && man == 0) return sign;
  int64_t m = exp ? (int64_t)(man | 0x800000u) : (int64_t)man;
  int32_t E = exp ? (int32_t)exp - 150 : -149;
  int32_t msb = 63 - __builtin_clzll((unsigned long long)m);
  int32_t k = msb + E - 10;            /* quantum exponent for an 11-bit significand */
  if (k < -24) k = -24;                /* binary16 subnormal quantum */
  int32_t sh = k - E;
  int64_t q;
  if (sh <= 0) {
    q = m << (-sh);
  } else if (sh >= 40) {
    q = 0;
  } else {
    q = m >> sh;
    int64_t rem = m & ((((int64_t)1) << sh) - 1), half = ((int64_t)1) << (sh - 1);
    if (rem > half || (rem == half && (q & 1))) q++;
  }
  if (k == -24 && q < 1024) return (uint16_t)(sign | (uint16_t)q);   /* subnormal or zero */
  if (q == 2048) { q = 1024; k++; }
  int32_t e16 = k + 25;
  if (e16 >= 31) return (uint16_t)(sign | 0x7C00u);                 /* overflow -> inf */
  return (uint16_t)(sign | (uint16_t)(e16 << 10) | (uint16_t)(q - 1024));
}

float orc_f32_from_f16(uint16_t h) {
  uint32_t sign = ((uint32_t)h & 0x8000u) << 16, e = (h >> 10) & 0x1Fu, m = h & 0x3FFu, b;
  if (e == 0) {
    if (m == 0) { b = sign; }
    else {                                       /* subnormal: m * 2^-24, normalise */
      int32_t sh = 0;
      while (!(m & 0x400u)) { m <<= 1; sh++; }
      m &= 0x3FFu;
      b = sign | ((uint32_t)(127 - 15 + 1 - sh) << 23) | (m << 13);
    }
  } else if (e == 31) {
    b = sign | 0x7F800000u | (m << 13);
  } else {
    b = sign | ((e - 15 + 127) << 23) | (m << 13);
  }
  float f;
  memcpy(&f, &b, 4);
  return f;
}

void orc_f16_from_f32_array(const float* x, uint16_t* out, int64_t n) {
  for (int64_t i = 0; i < n; i++) out[i] = orc_f16_from_f32(x[i]);
}

/* Total order on finite floats with -0 < +0 (Q16 "min/max under the total order"). */
static uint32_t total_key(float f) {
  uint32_t b;
  memcpy(&b, &f, 4);
  return (b & 0x80000000u) ? ~b : (b | 0x80000000u);
}

/* ------------------------------------------------------------------------------------------------
 * §2.2: "compute the scale s and zero point z based on X_min and X_max, then apply
 * quantization element-wise as Q = round((X - z)/s) ... X^ = s*Q + z ... metadata s and z are kept in
 * higher precision (e.g., FP16)"; applied "to each key and value vector independently".
 * Arithmetic fixed by reading Q16; packing by Q17.
 * ----------------------------------------------------------------------------------------------*/
int32_t orc_quantize(const float* x, int32_t d, int32_t bits, uint8_t* codes, uint16_t* s16, uint16_t* z16) {
  if (!(bits == 2 || bits == 4 || bits == 8) || d <= 0 || (d * bits) % 8) return ORC_ERR_INVALID;
  for (int32_t i = 0; i < d; i++)
    if (!isfinite(x[i])) return ORC_ERR_NONFINITE;
  float mn = x[0], mx = x[0];
  for (int32_t i = 1; i < d; i++) {
    if (total_key(x[i]) < total_key(mn)) mn = x[i];
    if (total_key(x[i]) > total_key(mx)) mx = x[i];
  }
  int32_t Q = (1 << bits) - 1;
  float s32 = mx - mn;                 /* fsub_rn */
  s32 = s32 / (float)Q;                /* fdiv_rn */
  *s16 = orc_f16_from_f32(s32);
  *z16 = orc_f16_from_f32(mn);
  float sf = orc_f32_from_f16(*s16), zf = orc_f32_from_f16(*z16);
  memset(codes, 0, (size_t)(d * bits / 8));
  for (int32_t i = 0; i < d; i++) {
    int32_t q = 0;
    if (sf != 0.0f) {
      float inv = 1.0f / sf;           /* fdiv_rn: reciprocal form is normative (Q16) */
      float t = x[i] - zf;             /* fsub_rn */
      t = t * inv;                     /* fmul_rn */
      float r = roundf(t);             /* round half away from zero */
      if (r < 0.0f) r = 0.0f;
      if (r > (float)Q) r = (float)Q;
      q = (int32_t)r;
    }
    int32_t bit = i * bits;            /* Q17: little-endian in the byte, lowest index in the LSBs */
    codes[bit >> 3] |= (uint8_t)(q << (bit & 7));
  }
  return ORC_OK;
}

void orc_dequantize(const uint8_t* codes, int32_t d, int32_t bits, uint16_t s16, uint16_t z16, float* out) {
  float sf = orc_f32_from_f16(s16), zf = orc_f32_from_f16(z16);
  int32_t Q = (1 << bits) - 1;
  for (int32_t i = 0; i < d; i++) {
    int32_t bit = i * bits;
    int32_t q = (codes[bit >> 3] >> (bit & 7)) & Q;
    float y = sf * (float)q;           /* exact: s16 has 11 significant bits, q <= 8 bits */
    out[i] = y + zf;                   /* fadd_rn */
  }
}

/* ------------------------------------------------------------------------------------------------
 * Geometry.  P:466-471: six segments in order (quantized keys, key metadata, quantized values, value
 * metadata, token scores, positions); tokens per page depend on the precision (Q11: C_h, C_l given).
 * Every segment starts on a 16-byte boundary; page size = max over classes, rounded to 128 B (Q18).
 * P:499 table length, corrected by Q12: L = ceil(M / C_h) + (W < C_h ? 1 : 0).
 * ----------------------------------------------------------------------------------------------*/
static int32_t align_up(int32_t x, int32_t a) { return (x + a - 1) / a * a; }

static void class_geom(int32_t d, int32_t C, int32_t kb, int32_t vb, orc_class_geom* g) {
  g->C = C; g->kbits = kb; g->vbits = vb;
  g->k_row = d * kb / 8;
  g->v_row = d * vb / 8;
  g->off_k = 0;
  g->off_kmeta = align_up(g->off_k + C * g->k_row, 16);
  g->off_v = align_up(g->off_kmeta + 4 * C, 16);
  g->off_vmeta = align_up(g->off_v + C * g->v_row, 16);
  g->off_score = align_up(g->off_vmeta + 4 * C, 16);
  g->off_pos = align_up(g->off_score + 4 * C, 16);
  g->end = g->off_pos + 4 * C;
}

/* NEXT-4 (Q40): an FP16 (TOP) page holds Ct tokens as plain fp16 K and V rows (2d bytes each), no quantization
   metadata, then the fp32 scores and int32 positions; segments 16-byte aligned in the same order. */
static void class_geom_fp16(int32_t d, int32_t C, orc_class_geom* g) {
  g->C = C; g->kbits = 16; g->vbits = 16;
  g->k_row = 2 * d;
  g->v_row = 2 * d;
  g->off_k = 0;
  g->off_kmeta = g->off_k + C * g->k_row;              /* empty */
  g->off_v = align_up(g->off_kmeta, 16);
  g->off_vmeta = g->off_v + C * g->v_row;              /* empty */
  g->off_score = align_up(g->off_vmeta, 16);
  g->off_pos = align_up(g->off_score + 4 * C, 16);
  g->end = g->off_pos + 4 * C;
}

static int bits_ok(int32_t b) { return b == 2 || b == 4 || b == 8; }

int32_t orc_geometry(const orc_config* c, int32_t* U, int32_t* L, int32_t* page_bytes,
                     orc_class_geom* high, orc_class_geom* low) {
  if (c->R < 1 || c->Ly < 1 || c->H < 1 || c->d < 8 || c->d % 8 || c->M < 1 || c->W < 0 ||
      c->Ch < 1 || c->Cl < c->Ch || c->P < 1 || !bits_ok(c->kbh) || !bits_ok(c->vbh) ||
      !bits_ok(c->kbl) || !bits_ok(c->vbl) || !isfinite(c->alpha_h) || !isfinite(c->alpha_l) ||
      c->alpha_h < 0 || c->alpha_l < 0 || (c->prompt_denominator != 0 && c->prompt_denominator != 1) ||
      (c->prefill_workflow != 0 && c->prefill_workflow != 1) || c->q_per_kv < 0 || c->q_per_kv > 16)
    return ORC_ERR_INVALID;
  /* NEXT-4 (Q38, Q43): alpha_t >= alpha_h, the exact prompt workflow only */
  if (c->top_tier != 0 && (c->top_tier != 1 || c->Ct < 1 || !isfinite(c->alpha_t) || c->alpha_t < c->alpha_h ||
                           c->prefill_workflow != 0))
    return ORC_ERR_INVALID;
  orc_class_geom gh, gl, gt;
  class_geom(c->d, c->Ch, c->kbh, c->vbh, &gh);
  class_geom(c->d, c->Cl, c->kbl, c->vbl, &gl);
  int32_t end = gh.end > gl.end ? gh.end : gl.end;
  if (c->top_tier) {
    class_geom_fp16(c->d, c->Ct, &gt);
    if (gt.end > end) end = gt.end;
  }
  if (U) *U = c->R * c->Ly * c->H;
  if (L) *L = (c->M + c->Ch - 1) / c->Ch + (c->W < c->Ch ? 1 : 0);
  if (page_bytes) *page_bytes = align_up(end, 128);
  if (high) *high = gh;
  if (low) *low = gl;
  return ORC_OK;
}

/* "with a batch size of 128 on Llama3-8B, which has 32 layers and 8 KV heads per layer, the total
   size of all bidirectional page tables is only 32 MB" — one 4-byte page ID per slot (Q19). */
int64_t orc_table_bytes(int64_t batch, int64_t layers, int64_t kv_heads, int64_t L) {
  return batch * layers * kv_heads * L * 4;
}

/* ------------------------------------------------------------------------------------------------
 * Pool state (c.1).  ring = iota, start = 0, free = P; tables = -1; counts = 0.
 * ----------------------------------------------------------------------------------------------*/
orc_pool* orc_pool_new(const orc_config* c) {
  orc_pool* p = (orc_pool*)calloc(1, sizeof(orc_pool));
  if (!p) return NULL;
  p->c = *c;
  if (orc_geometry(c, &p->U, &p->L, &p->page_bytes, &p->g[ORC_CLS_HIGH], &p->g[ORC_CLS_LOW]) != ORC_OK) {
    free(p);
    return NULL;
  }
  size_t U = (size_t)p->U, L = (size_t)p->L, P = (size_t)c->P, R = (size_t)c->R;
  if (c->top_tier) class_geom_fp16(c->d, c->Ct, &p->g[ORC_CLS_TOP]);
  p->Lt = c->top_tier ? (c->M + c->Ct - 1) / c->Ct : 1;         /* Q41: at most M tokens in the TOP section */
  p->ttable = (int32_t*)malloc(U * (size_t)p->Lt * 4);
  p->n_t = (int32_t*)calloc(U, 4);
  p->pf_nt = (int32_t*)calloc(U, 4);
  p->ring = (int32_t*)malloc(P * 4);
  p->table = (int32_t*)malloc(U * L * 4);
  p->n_h = (int32_t*)calloc(U, 4);
  p->n_l = (int32_t*)calloc(U, 4);
  p->req_state = (int8_t*)calloc(R, 1);
  p->seq_len = (int32_t*)calloc(R, 4);
  p->prompt_len = (int32_t*)calloc(R, 4);
  p->pages = (uint8_t*)calloc(P, (size_t)p->page_bytes);
  size_t wn = U * (size_t)c->W * (size_t)c->d;
  p->win_k = (uint16_t*)calloc(wn ? wn : 1, 2);
  p->win_v = (uint16_t*)calloc(wn ? wn : 1, 2);
  const size_t wsn = U * (size_t)c->W;
  p->win_sig = (float*)calloc(wsn ? wsn : 1, 4);
  p->pf_nh = (int32_t*)calloc(U, 4);
  p->pf_nl = (int32_t*)calloc(U, 4);
  p->admit_list = (int32_t*)calloc(R, 4);
  if (!p->ring || !p->table || !p->n_h || !p->n_l || !p->req_state || !p->seq_len || !p->prompt_len ||
      !p->pages || !p->win_k || !p->win_v || !p->win_sig || !p->pf_nh || !p->pf_nl || !p->admit_list ||
      !p->ttable || !p->n_t || !p->pf_nt) {
    orc_pool_delete(p);
    return NULL;
  }
  for (size_t i = 0; i < P; i++) p->ring[i] = (int32_t)i;
  for (size_t i = 0; i < U * L; i++) p->table[i] = -1;
  for (size_t i = 0; i < U * (size_t)p->Lt; i++) p->ttable[i] = -1;
  p->start = 0;
  p->free = c->P;
  p->last_phase = -1;
  return p;
}

void orc_pool_delete(orc_pool* p) {
  if (!p) return;
  free(p->ring); free(p->table); free(p->n_h); free(p->n_l); free(p->req_state); free(p->seq_len);
  free(p->prompt_len); free(p->pages); free(p->win_k); free(p->win_v); free(p->pf_nh); free(p->pf_nl);
  free(p->admit_list); free(p->win_sig); free(p->head_ah); free(p->head_al);
  free(p->ttable); free(p->n_t); free(p->pf_nt);
  free(p);
}

static void set_status(orc_pool* p, int32_t st) { if (p->status == ORC_OK) p->status = st; }

int32_t orc_take_status(orc_pool* p) { int32_t s = p->status; p->status = ORC_OK; return s; }

/* Section slot s of class c lives at page table[u][s/C_h] (High, left) or table[u][L-1-s/C_l] (Low,
   right), index s mod C (c.1). */
static uint8_t* slot_page(orc_pool* p, int cls, int32_t u, int32_t s, int32_t* idx) {
  const orc_class_geom* g = &p->g[cls];
  int32_t pid;
  if (cls == ORC_CLS_TOP) {                              /* Q41: TOP slot s at ttable[u][s / Ct] */
    pid = p->ttable[(size_t)u * p->Lt + s / g->C];
  } else {
    int32_t k = (cls == ORC_CLS_HIGH) ? s / g->C : p->L - 1 - s / g->C;
    pid = p->table[(size_t)u * p->L + k];
  }
  *idx = s % g->C;
  return p->pages + (size_t)pid * (size_t)p->page_bytes;
}

static float slot_sig(orc_pool* p, int cls, int32_t u, int32_t s) {
  int32_t idx; uint8_t* pg = slot_page(p, cls, u, s, &idx);
  float f; memcpy(&f, pg + p->g[cls].off_score + 4 * idx, 4); return f;
}

static int32_t slot_pos(orc_pool* p, int cls, int32_t u, int32_t s) {
  int32_t idx; uint8_t* pg = slot_page(p, cls, u, s, &idx);
  int32_t v; memcpy(&v, pg + p->g[cls].off_pos + 4 * idx, 4); return v;
}

/* Quantize one token's K and V (fp32 inputs) at class `cls` bits and store all six segments. */
static int32_t write_token(orc_pool* p, int cls, int32_t u, int32_t s, const float* k, const float* v,
                           float sig, int32_t pos) {
  const orc_class_geom* g = &p->g[cls];
  /* Q30: a token with a non-finite K or V element is rejected whole — nothing of it is written */
  for (int32_t i = 0; i < p->c.d; i++)
    if (!isfinite(k[i]) || !isfinite(v[i])) return ORC_ERR_NONFINITE;
  int32_t idx; uint8_t* pg = slot_page(p, cls, u, s, &idx);
  uint16_t ks, kz, vs, vz;
  int32_t st = orc_quantize(k, p->c.d, g->kbits, pg + g->off_k + idx * g->k_row, &ks, &kz);
  if (st != ORC_OK) return st;
  st = orc_quantize(v, p->c.d, g->vbits, pg + g->off_v + idx * g->v_row, &vs, &vz);
  if (st != ORC_OK) return st;
  uint8_t* km = pg + g->off_kmeta + 4 * idx; uint8_t* vm = pg + g->off_vmeta + 4 * idx;
  memcpy(km, &ks, 2); memcpy(km + 2, &kz, 2);          /* meta = {s16, z16}, s at the lower address */
  memcpy(vm, &vs, 2); memcpy(vm + 2, &vz, 2);
  memcpy(pg + g->off_score + 4 * idx, &sig, 4);
  memcpy(pg + g->off_pos + 4 * idx, &pos, 4);
  return ORC_OK;
}

/* NEXT-4 (Q40): a TOP token is stored as its fp16 K and V rows as given (no quantization); Q30 applies. */
static int32_t write_token_top(orc_pool* p, int32_t u, int32_t s, const uint16_t* k, const uint16_t* v, float sig,
                               int32_t pos) {
  const orc_class_geom* g = &p->g[ORC_CLS_TOP];
  for (int32_t i = 0; i < p->c.d; i++)
    if (!isfinite(orc_f32_from_f16(k[i])) || !isfinite(orc_f32_from_f16(v[i]))) return ORC_ERR_NONFINITE;
  int32_t idx; uint8_t* pg = slot_page(p, ORC_CLS_TOP, u, s, &idx);
  memcpy(pg + g->off_k + idx * g->k_row, k, (size_t)g->k_row);
  memcpy(pg + g->off_v + idx * g->v_row, v, (size_t)g->v_row);
  memcpy(pg + g->off_score + 4 * idx, &sig, 4);
  memcpy(pg + g->off_pos + 4 * idx, &pos, 4);
  return ORC_OK;
}

static void read_token(orc_pool* p, int cls, int32_t u, int32_t s, float* k, float* v, float* sig, int32_t* pos) {
  if (cls == ORC_CLS_TOP) {                              /* fp16 values, exactly */
    const orc_class_geom* g = &p->g[ORC_CLS_TOP];
    int32_t idx; uint8_t* pg = slot_page(p, cls, u, s, &idx);
    for (int32_t i = 0; i < p->c.d; i++) {
      uint16_t hk, hv;
      memcpy(&hk, pg + g->off_k + idx * g->k_row + 2 * i, 2);
      memcpy(&hv, pg + g->off_v + idx * g->v_row + 2 * i, 2);
      k[i] = orc_f32_from_f16(hk); v[i] = orc_f32_from_f16(hv);
    }
    memcpy(sig, pg + g->off_score + 4 * idx, 4);
    memcpy(pos, pg + g->off_pos + 4 * idx, 4);
    return;
  }
  const orc_class_geom* g = &p->g[cls];
  int32_t idx; uint8_t* pg = slot_page(p, cls, u, s, &idx);
  uint16_t ks, kz, vs, vz;
  memcpy(&ks, pg + g->off_kmeta + 4 * idx, 2); memcpy(&kz, pg + g->off_kmeta + 4 * idx + 2, 2);
  memcpy(&vs, pg + g->off_vmeta + 4 * idx, 2); memcpy(&vz, pg + g->off_vmeta + 4 * idx + 2, 2);
  orc_dequantize(pg + g->off_k + idx * g->k_row, p->c.d, g->kbits, ks, kz, k);
  orc_dequantize(pg + g->off_v + idx * g->v_row, p->c.d, g->vbits, vs, vz, v);
  memcpy(sig, pg + g->off_score + 4 * idx, 4);
  memcpy(pos, pg + g->off_pos + 4 * idx, 4);
}

static int32_t ceil_div(int32_t a, int32_t b) { return (a + b - 1) / b; }

/* ------------------------------------------------------------------------------------------------
 * Algorithm 1, generation phase, one unit at a time (c.2).
 *   N  = tokens of the request including the one appended this step (Q3)
 *   t_c = earliest window token, position N-1-W
 *   thresholds alpha/N in fp32 round-to-nearest (Q3); half-open classes (Q2)
 *   victim = lexicographic argmin of (score, position) over the section t_c joins, t_c included (Q6, Q7)
 *   t_c takes the victim's slot when the victim leaves; a downgraded victim goes to the KV_l tail (Q8)
 * ----------------------------------------------------------------------------------------------*/
/* Q35 (NEXT-4): the thresholds of unit u's (layer, head) — per head when set, else the pool-wide pair */
static float unit_ah(const orc_pool* p, int32_t u) {
  return p->use_head ? p->head_ah[u % (p->c.Ly * p->c.H)] : p->c.alpha_h;
}
static float unit_al(const orc_pool* p, int32_t u) {
  return p->use_head ? p->head_al[u % (p->c.Ly * p->c.H)] : p->c.alpha_l;
}

static void empty_decision(orc_decision* d) {
  memset(d, 0, sizeof(*d));
  d->v_slot = d->tc_slot = d->v_dst_slot = -1;
}

int32_t orc_classify_decode(orc_pool* p, const float* cand_sig, orc_decision* dec) {
  const orc_config* c = &p->c;
  for (int32_t r = 0; r < c->R; r++)
    if (p->req_state[r] == ORC_REQ_ACTIVE && p->seq_len[r] >= c->M) return ORC_ERR_STATE;
  p->last_phase = ORC_DECODE;
  int32_t LyH = c->Ly * c->H;
  const int32_t st0 = p->status;                             /* Q36: the status is taken once, at entry */
  for (int32_t u = 0; u < p->U; u++) {
    orc_decision* D = &dec[u];
    empty_decision(D);
    if (st0 != ORC_OK) continue;                             /* sticky error: no-op */
    int32_t r = u / LyH;
    if (p->req_state[r] != ORC_REQ_ACTIVE) continue;
    int32_t N = p->seq_len[r] + 1;
    int32_t pc = N - 1 - c->W;
    if (pc < 0) continue;                                     /* no token leaves the window yet */
    /* NULL cand_sig (NEXT-2): t_c's significance is the running average kept for its window slot */
    float sc = cand_sig ? cand_sig[u] : (c->W ? p->win_sig[(size_t)u * c->W + (size_t)(pc % c->W)] : 0.0f);
    if (!isfinite(sc) || sc < 0.0f) { set_status(p, ORC_ERR_NONFINITE); continue; }
    if (sc == 0.0f) sc = 0.0f;                                /* canonicalise -0 -> +0 (Q6) */
    float th = unit_ah(p, u) / (float)N;                      /* alpha_h / N */
    float tl = unit_al(p, u) / (float)N;                      /* alpha_l / N */
    /* NEXT-4 (Q38, Q39): with the FP16 tier, t_c at or above alpha_t / N is TOP */
    const int top = c->top_tier != 0;
    float tt = top ? c->alpha_t / (float)N : 0.0f;
    int cls;
    if (top && sc >= tt) cls = ORC_CLS_TOP;
    else if (sc >= th) cls = ORC_CLS_HIGH;                    /* line q_high */
    else if (sc >= tl) cls = ORC_CLS_LOW;                     /* line q_low  */
    else { D->tc_class = ORC_CLS_PRUNED; continue; }          /* t_c pruned */
    int32_t n = cls == ORC_CLS_TOP ? p->n_t[u] : ((cls == ORC_CLS_HIGH) ? p->n_h[u] : p->n_l[u]);
    /* t_v = argmin over the section with t_c added (lines v_high / v_low). */
    int32_t vslot = -1; float vs = sc; int32_t vp = pc;       /* start from t_c itself */
    for (int32_t s = 0; s < n; s++) {
      float sg = slot_sig(p, cls, u, s);
      int32_t ps = slot_pos(p, cls, u, s);
      if (sg < vs || (sg == vs && ps < vp)) { vs = sg; vp = ps; vslot = s; }
    }
    D->tc_class = (uint8_t)cls;
    if (cls == ORC_CLS_TOP) {                                 /* Q39: Algorithm 1 one level up */
      if (vslot < 0 || vs >= tt) {                            /* t_v stays in KV_t */
        D->v_action = ORC_V_KEEP; D->grow = ORC_GROW_TOP;
        D->demand = (p->n_t[u] % c->Ct == 0); D->tc_slot = p->n_t[u];
      } else if (vs >= th) {                                  /* t_v moves to KV_h (re-quantized at P_h) */
        D->v_action = ORC_V_DOWN; D->grow = ORC_GROW_HIGH;
        D->demand = (p->n_h[u] % c->Ch == 0);
        D->v_slot = vslot; D->tc_slot = vslot; D->v_dst_slot = p->n_h[u];
      } else if (vs >= tl) {                                  /* t_v moves to KV_l (re-quantized at P_l) */
        D->v_action = ORC_V_DOWN; D->grow = ORC_GROW_LOW;
        D->demand = (p->n_l[u] % c->Cl == 0);
        D->v_slot = vslot; D->tc_slot = vslot; D->v_dst_slot = p->n_l[u];
      } else {                                                /* prune t_v */
        D->v_action = ORC_V_PRUNE; D->grow = ORC_GROW_NONE; D->demand = 0;
        D->v_slot = vslot; D->tc_slot = vslot;
      }
    } else if (cls == ORC_CLS_HIGH) {
      if (vslot < 0 || vs >= th) {                            /* t_v stays in KV_h */
        D->v_action = ORC_V_KEEP; D->grow = ORC_GROW_HIGH;
        D->demand = (p->n_h[u] % c->Ch == 0); D->tc_slot = p->n_h[u];
      } else if (vs >= tl) {                                  /* line requant_high: downgrade t_v */
        D->v_action = ORC_V_DOWN; D->grow = ORC_GROW_LOW;
        D->demand = (p->n_l[u] % c->Cl == 0);
        D->v_slot = vslot; D->tc_slot = vslot; D->v_dst_slot = p->n_l[u];
      } else {                                                /* prune t_v */
        D->v_action = ORC_V_PRUNE; D->grow = ORC_GROW_NONE; D->demand = 0;
        D->v_slot = vslot; D->tc_slot = vslot;
      }
    } else {
      if (vslot < 0 || vs >= tl) {
        D->v_action = ORC_V_KEEP; D->grow = ORC_GROW_LOW;
        D->demand = (p->n_l[u] % c->Cl == 0); D->tc_slot = p->n_l[u];
      } else {                                                /* line prune_low */
        D->v_action = ORC_V_PRUNE; D->grow = ORC_GROW_NONE; D->demand = 0;
        D->v_slot = vslot; D->tc_slot = vslot;
      }
    }
  }
  return ORC_OK;
}

/* ------------------------------------------------------------------------------------------------
 * §4 prompt phase, c.6: token i (1-indexed) of a prompt of length n is High if its
 * significance >= alpha_h/den, Low if >= alpha_l/den, else pruned (Q2 half-open), den = i (Q4 default)
 * or n; the newest W tokens stay in the FP16 window (Q10).
 * ----------------------------------------------------------------------------------------------*/
static int32_t admit(orc_pool* p, const int32_t* req, const int32_t* len, int32_t n) {
  const orc_config* c = &p->c;
  if (n < 0 || n > c->R) return ORC_ERR_INVALID;
  for (int32_t i = 0; i < n; i++) {
    if (req[i] < 0 || req[i] >= c->R || len[i] < 0 || len[i] > c->M) return ORC_ERR_INVALID;
    if (p->req_state[req[i]] != ORC_REQ_IDLE) return ORC_ERR_STATE;
    for (int32_t j = 0; j < i; j++) if (req[j] == req[i]) return ORC_ERR_INVALID;
  }
  for (int32_t i = 0; i < n; i++) {
    p->req_state[req[i]] = ORC_REQ_ADMITTING;
    p->prompt_len[req[i]] = len[i];
    p->admit_list[i] = req[i];
  }
  p->n_admit = n;
  return ORC_OK;
}

int32_t orc_set_head_thresholds(orc_pool* p, const float* alpha_h, const float* alpha_l) {
  int32_t LyH = p->c.Ly * p->c.H;
  if (!alpha_h || !alpha_l) { p->use_head = 0; return ORC_OK; }
  for (int32_t i = 0; i < LyH; i++)
    if (!isfinite(alpha_h[i]) || !isfinite(alpha_l[i]) || alpha_h[i] < 0 || alpha_l[i] < 0 ||
        (p->c.top_tier && alpha_h[i] > p->c.alpha_t))                 /* Q38: alpha_t >= alpha_h */
      return ORC_ERR_INVALID;
  if (!p->head_ah) { p->head_ah = (float*)malloc(4 * (size_t)LyH); p->head_al = (float*)malloc(4 * (size_t)LyH); }
  if (!p->head_ah || !p->head_al) return ORC_ERR_INVALID;
  memcpy(p->head_ah, alpha_h, 4 * (size_t)LyH);
  memcpy(p->head_al, alpha_l, 4 * (size_t)LyH);
  p->use_head = 1;
  return ORC_OK;
}

static int prompt_class(const orc_pool* p, int32_t u, float s, int32_t t, int32_t n) {
  const orc_config* c = &p->c;
  float den = (c->prompt_denominator == 0) ? (float)(t + 1) : (float)n;
  float th = unit_ah(p, u) / den, tl = unit_al(p, u) / den;
  if (c->top_tier && s >= c->alpha_t / den) return ORC_CLS_TOP;     /* NEXT-4 (Q38) */
  if (s >= th) return ORC_CLS_HIGH;
  if (s >= tl) return ORC_CLS_LOW;
  return ORC_CLS_PRUNED;
}

int32_t orc_classify_prefill(orc_pool* p, const int32_t* req, const int32_t* len, int32_t n,
                             const float* sig, int64_t sig_stride, uint8_t* token_class) {
  const orc_config* c = &p->c;
  for (int32_t i = 0; i < n; i++) if (len[i] > sig_stride) return ORC_ERR_INVALID;
  int32_t st = admit(p, req, len, n);
  if (st != ORC_OK) return st;
  p->last_phase = ORC_PREFILL;
  int32_t LyH = c->Ly * c->H;
  const int32_t st0 = p->status;                             /* Q36: the status is taken once, at entry */
  for (int32_t i = 0; i < n; i++) {
    int32_t r = req[i], T = len[i];
    for (int32_t j = 0; j < LyH; j++) {
      int32_t u = r * LyH + j;
      const float* row = sig + ((int64_t)i * LyH + j) * sig_stride;
      uint8_t* crow = token_class ? token_class + ((int64_t)i * LyH + j) * sig_stride : NULL;
      int32_t nh = 0, nl = 0, nt = 0;
      for (int32_t t = 0; t < T; t++) {
        int cls = ORC_CLS_NONE;                               /* window token */
        if (t < T - c->W && st0 == ORC_OK) {
          float s = row[t];
          if (!isfinite(s) || s < 0.0f) { set_status(p, ORC_ERR_NONFINITE); s = 0.0f; }
          cls = prompt_class(p, u, s, t, T);
          if (cls == ORC_CLS_HIGH) nh++;
          if (cls == ORC_CLS_LOW) nl++;
          if (cls == ORC_CLS_TOP) nt++;
        }
        if (crow) crow[t] = (uint8_t)cls;
      }
      p->pf_nh[u] = nh;
      p->pf_nl[u] = nl;
      p->pf_nt[u] = nt;
    }
  }
  return ORC_OK;
}

/* ------------------------------------------------------------------------------------------------
 * The paper's prompt workflow (NEXT-1, fig:memory_management_flow), selected by
 * prefill_workflow = 1.  "Memory pages are conservatively allocated for each head, assuming all tokens
 * are stored at high precision": c_u = ceil(kept/C_h) pages, kept = prompt tokens outside the
 * window; "the end pointer advances", i.e. the allocation pointer (Q1).  Then "the planning phase
 * determines ... high-precision and low-precision pages", and each head keeps its high pages
 * from the left and its low pages from the right of its block while the pages in between are reclaimed
 * "via a parallel prefix-sum operation" and appended at the end pointer.
 * Q29 (the paper is silent): with C_l >= C_h, ceil(n_h/C_h) + ceil(n_l/C_l) can exceed c_u by one page
 * (e.g. one high and one low token in a 16-token block); such a head keeps its whole block and takes one
 * more page, granted from the start pointer after every conservative block (a second exclusive scan in
 * canonical order).  Blocks and top-ups are one all-or-nothing allocation (Q15).
 * ----------------------------------------------------------------------------------------------*/
static int32_t conservative_pages(const orc_pool* p, int32_t u) {
  const orc_config* c = &p->c;
  int32_t r = u / (c->Ly * c->H);
  int32_t kept = p->prompt_len[r] - c->W > 0 ? p->prompt_len[r] - c->W : 0;
  return ceil_div(kept, c->Ch);
}
static int32_t topup_pages(const orc_pool* p, int32_t u) {
  const orc_config* c = &p->c;
  int32_t need = ceil_div(p->pf_nh[u], c->Ch) + ceil_div(p->pf_nl[u], c->Cl);
  return need > conservative_pages(p, u) ? 1 : 0;
}
/* grants D = sum(c_u) + sum(e_u) pages from ring[start..), writes the final tables and appends the
 * reclaimed middles at end = start + free (before this allocation); sets p->last_reclaimed */
static void prefill_conservative_grant(orc_pool* p, int64_t D) {
  const orc_config* c = &p->c;
  int32_t LyH = c->Ly * c->H, L = p->L, P = c->P;
  int64_t end = (p->start + p->free) % P;
  int64_t sum_c = 0;
  for (int32_t u = 0; u < p->U; u++)
    if (p->req_state[u / LyH] == ORC_REQ_ADMITTING) sum_c += conservative_pages(p, u);
  int64_t off_c = 0, off_e = 0, off_m = 0;
  for (int32_t u = 0; u < p->U; u++) {
    if (p->req_state[u / LyH] != ORC_REQ_ADMITTING) continue;
    int32_t* row = &p->table[(size_t)u * L];
    int32_t cu = conservative_pages(p, u), eu = topup_pages(p, u);
    int32_t ph = ceil_div(p->pf_nh[u], c->Ch), pl = ceil_div(p->pf_nl[u], c->Cl);
    if (ph + pl > L) { set_status(p, ORC_ERR_OVERFLOW); off_c += cu; off_e += eu; continue; }
    /* block'[k]: the conservative block (scan 1), then the top-up page (scan 2) */
    int64_t base_c = p->start + off_c, pos_e = p->start + sum_c + off_e;
    int32_t nb = cu + eu;
#define BLOCK(k) p->ring[((k) < cu ? base_c + (k) : pos_e) % P]
    for (int32_t k = 0; k < ph; k++) row[k] = BLOCK(k);                  /* high: left to right */
    for (int32_t k = 0; k < pl; k++) row[L - 1 - k] = BLOCK(nb - 1 - k);  /* low: right to left */
    for (int32_t k = ph; k < nb - pl; k++) {                             /* reclaim the middle (scan 3) */
      p->ring[(end + off_m) % P] = BLOCK(k);
      off_m += 1;
    }
#undef BLOCK
    off_c += cu; off_e += eu;
  }
  (void)D;
  p->last_reclaimed = off_m;
}

/* ------------------------------------------------------------------------------------------------
 * Coordination (c.3).  P:485-488: "after each head determines the number of pages to be allocated or
 * freed, a parallel prefix sum ... computes a unique offset for each head relative to the start or end
 * pointer ... For memory allocation, each head concurrently retrieves its new page IDs from its
 * designated region ... with the start pointer incremented by the cumulative number of pages ...
 * for memory recycling, each head writes freed page IDs to its designated region, with the end pointer
 * incremented by the total number of pages released."  Serial here: the running offset IS the prefix
 * sum.  Order: recycle first (Q14), canonical order u = (r*Ly + l)*H + h (Q13), all-or-nothing (Q15).
 * ----------------------------------------------------------------------------------------------*/
int32_t orc_compact_alloc(orc_pool* p, const orc_decision* dec) {
  const orc_config* c = &p->c;
  int32_t LyH = c->Ly * c->H, L = p->L, P = c->P;
  if (p->last_phase == ORC_DECODE && !dec) return ORC_ERR_INVALID;
  if (p->last_phase < 0) return ORC_ERR_STATE;
  /* 1. recycle finished requests into the ring at end = start + free */
  int64_t freed = 0;
  for (int32_t r = 0; r < c->R; r++) {
    if (p->req_state[r] != ORC_REQ_PENDING_FREE) continue;
    for (int32_t j = 0; j < LyH; j++) {
      int32_t u = r * LyH + j;
      for (int32_t k = 0; k < p->Lt; k++) {                     /* NEXT-4 (Q41): the TOP table's slots first */
        int32_t* slot = &p->ttable[(size_t)u * p->Lt + k];
        if (*slot != -1) {
          p->ring[(p->start + p->free) % P] = *slot;
          p->free += 1; freed += 1;
          *slot = -1;
        }
      }
      p->n_t[u] = 0;
      for (int32_t k = 0; k < L; k++) {
        int32_t* slot = &p->table[(size_t)u * L + k];
        if (*slot != -1) {
          p->ring[(p->start + p->free) % P] = *slot;
          p->free += 1; freed += 1;
          *slot = -1;
        }
      }
      p->n_h[u] = 0; p->n_l[u] = 0;
    }
    p->req_state[r] = ORC_REQ_IDLE;
    p->seq_len[r] = 0;
    p->prompt_len[r] = 0;
  }
  p->last_freed = freed;
  if (p->status != ORC_OK) { p->last_demand = 0; return ORC_OK; }   /* allocation is a no-op */
  /* 2. per-head demand and the all-or-nothing check */
  int64_t D = 0;
  for (int32_t u = 0; u < p->U; u++) {
    int32_t r = u / LyH;
    if (p->last_phase == ORC_DECODE) {
      if (p->req_state[r] == ORC_REQ_ACTIVE) D += dec[u].demand;
    } else if (p->req_state[r] == ORC_REQ_ADMITTING) {
      if (c->prefill_workflow == 1) D += conservative_pages(p, u) + topup_pages(p, u);
      else D += ceil_div(p->pf_nh[u], c->Ch) + ceil_div(p->pf_nl[u], c->Cl) +
                (c->top_tier ? ceil_div(p->pf_nt[u], c->Ct) : 0);
    }
  }
  p->last_demand = D;
  p->last_reclaimed = 0;
  if (D > p->free) { set_status(p, ORC_ERR_OOM); p->oom_count++; return ORC_OK; }
  /* 3. grant in canonical order; high IDs left-to-right, low IDs right-to-left */
  int64_t off = 0;
  for (int32_t u = 0; u < p->U; u++) {
    int32_t r = u / LyH;
    int32_t* row = &p->table[(size_t)u * L];
    if (p->last_phase == ORC_DECODE) {
      if (p->req_state[r] != ORC_REQ_ACTIVE || !dec[u].demand) continue;
      if (dec[u].grow == ORC_GROW_TOP) {                        /* NEXT-4: the TOP table, left to right */
        if (p->n_t[u] / c->Ct >= p->Lt) { set_status(p, ORC_ERR_OVERFLOW); continue; }
        p->ttable[(size_t)u * p->Lt + p->n_t[u] / c->Ct] = p->ring[(p->start + off) % P];
        off += 1;
        continue;
      }
      int32_t ph = ceil_div(p->n_h[u], c->Ch), pl = ceil_div(p->n_l[u], c->Cl);
      if (ph + pl + 1 > L) { set_status(p, ORC_ERR_OVERFLOW); continue; }
      int32_t k = (dec[u].grow == ORC_GROW_HIGH) ? p->n_h[u] / c->Ch : L - 1 - p->n_l[u] / c->Cl;
      row[k] = p->ring[(p->start + off) % P];
      off += 1;
    } else if (c->prefill_workflow == 0) {
      if (p->req_state[r] != ORC_REQ_ADMITTING) continue;
      if (c->top_tier) {                                         /* Q41/Q43: a unit's TOP pages come first */
        int32_t pt = ceil_div(p->pf_nt[u], c->Ct);
        for (int32_t k = 0; k < pt; k++) { p->ttable[(size_t)u * p->Lt + k] = p->ring[(p->start + off) % P]; off += 1; }
      }
      int32_t ph = ceil_div(p->pf_nh[u], c->Ch), pl = ceil_div(p->pf_nl[u], c->Cl);
      if (ph + pl > L) { set_status(p, ORC_ERR_OVERFLOW); off += ph + pl; continue; }
      for (int32_t k = 0; k < ph; k++) { row[k] = p->ring[(p->start + off) % P]; off += 1; }
      for (int32_t k = 0; k < pl; k++) { row[L - 1 - k] = p->ring[(p->start + off) % P]; off += 1; }
    }
  }
  if (p->last_phase == ORC_PREFILL && c->prefill_workflow == 1) prefill_conservative_grant(p, D);
  p->start = (p->start + D) % P;
  p->free -= D;
  if (p->last_phase == ORC_PREFILL && c->prefill_workflow == 1) p->free += p->last_reclaimed;
  /* 4. counts (a5) and the request length */
  for (int32_t u = 0; u < p->U; u++) {
    int32_t r = u / LyH;
    if (p->last_phase == ORC_DECODE) {
      if (p->req_state[r] != ORC_REQ_ACTIVE) continue;
      if (dec[u].grow == ORC_GROW_HIGH) p->n_h[u] += 1;
      if (dec[u].grow == ORC_GROW_LOW) p->n_l[u] += 1;       /* DOWN: n_h unchanged, n_l + 1 */
      if (dec[u].grow == ORC_GROW_TOP) p->n_t[u] += 1;
    } else if (p->req_state[r] == ORC_REQ_ADMITTING) {
      p->n_h[u] = p->pf_nh[u];
      p->n_l[u] = p->pf_nl[u];
      p->n_t[u] = c->top_tier ? p->pf_nt[u] : 0;
    }
  }
  for (int32_t r = 0; r < c->R; r++) {
    if (p->last_phase == ORC_DECODE && p->req_state[r] == ORC_REQ_ACTIVE) p->seq_len[r] += 1;
    if (p->last_phase == ORC_PREFILL && p->req_state[r] == ORC_REQ_ADMITTING) p->seq_len[r] = p->prompt_len[r];
  }
  return ORC_OK;
}

/* ------------------------------------------------------------------------------------------------
 * KV compressor, generation step (c.4): downgrade t_v (Q9: re-quantize the stored P_h
 * values), quantize t_c out of the FP16 window into its slot, push the new token into the window.
 * ----------------------------------------------------------------------------------------------*/
int32_t orc_quant_write_decode(orc_pool* p, const orc_decision* dec, const uint16_t* k_new,
                               const uint16_t* v_new, const float* cand_sig) {
  if (p->status != ORC_OK) return ORC_OK;
  const orc_config* c = &p->c;
  int32_t LyH = c->Ly * c->H, d = c->d, W = c->W;
  float* kx = (float*)malloc((size_t)d * 4); float* vx = (float*)malloc((size_t)d * 4);
  for (int32_t u = 0; u < p->U; u++) {
    int32_t r = u / LyH;
    if (p->req_state[r] != ORC_REQ_ACTIVE) continue;
    const orc_decision* D = &dec[u];
    int32_t N = p->seq_len[r];                      /* already includes the new token */
    int32_t pc = N - 1 - W;
    if (D->v_action == ORC_V_DOWN) {
      /* the victim leaves the section t_c joins for the class `grow` (Q9; NEXT-4 Q42: a TOP victim's fp16
         values are quantized as they are) */
      float sg; int32_t ps;
      read_token(p, D->tc_class, u, D->v_slot, kx, vx, &sg, &ps);
      int32_t st = write_token(p, D->grow, u, D->v_dst_slot, kx, vx, sg, ps);
      if (st != ORC_OK) { set_status(p, st); continue; }
    }
    const uint16_t* kn = k_new + (size_t)u * d; const uint16_t* vn = v_new + (size_t)u * d;
    uint16_t* wk = W ? p->win_k + ((size_t)u * W + (size_t)((N - 1) % W)) * d : NULL;
    uint16_t* wv = W ? p->win_v + ((size_t)u * W + (size_t)((N - 1) % W)) * d : NULL;
    if (D->tc_class == ORC_CLS_TOP) {                         /* NEXT-4: t_c kept in FP16 */
      const uint16_t* sk = W ? wk : kn; const uint16_t* sv = W ? wv : vn;
      float sc = cand_sig ? cand_sig[u] : (W ? p->win_sig[(size_t)u * W + (size_t)((N - 1) % W)] : 0.0f);
      if (sc == 0.0f) sc = 0.0f;
      int32_t st = write_token_top(p, u, D->tc_slot, sk, sv, sc, pc);
      if (st != ORC_OK) { set_status(p, st); continue; }
    } else if (D->tc_class == ORC_CLS_HIGH || D->tc_class == ORC_CLS_LOW) {
      /* t_c sits in window slot p_c mod W == (N-1) mod W; read it before the push overwrites it */
      const uint16_t* sk = W ? wk : kn; const uint16_t* sv = W ? wv : vn;
      for (int32_t i = 0; i < d; i++) { kx[i] = orc_f32_from_f16(sk[i]); vx[i] = orc_f32_from_f16(sv[i]); }
      float sc = cand_sig ? cand_sig[u] : (W ? p->win_sig[(size_t)u * W + (size_t)((N - 1) % W)] : 0.0f);
      if (sc == 0.0f) sc = 0.0f;
      int32_t st = write_token(p, D->tc_class, u, D->tc_slot, kx, vx, sc, pc);
      if (st != ORC_OK) { set_status(p, st); continue; }
    }
    if (W) {
      memcpy(wk, kn, (size_t)d * 2); memcpy(wv, vn, (size_t)d * 2);
      p->win_sig[(size_t)u * W + (size_t)((N - 1) % W)] = 0.0f;   /* the new token: no later query yet (Q33) */
    }
  }
  free(kx); free(vx);
  return ORC_OK;
}

/* Prompt phase bulk write (a8): each kept token goes to the next slot of its class in position order;
   the newest min(W, n) tokens go to the window at slot pos mod W; then ADMITTING -> ACTIVE. */
int32_t orc_quant_write_prefill(orc_pool* p, const uint16_t* k, const uint16_t* v, int64_t kv_stride,
                                const float* sig, int64_t sig_stride) {
  if (p->status != ORC_OK) {
    /* Q36/Q37: an error at entry means this admission's planning or allocation did not happen (no pages
       were granted): the admission is rolled back, ADMITTING -> IDLE */
    for (int32_t i = 0; i < p->n_admit; i++) {
      int32_t r = p->admit_list[i];
      if (p->req_state[r] != ORC_REQ_ADMITTING) continue;
      p->req_state[r] = ORC_REQ_IDLE; p->seq_len[r] = 0; p->prompt_len[r] = 0;
    }
    p->n_admit = 0;
    return ORC_OK;
  }
  const orc_config* c = &p->c;
  int32_t LyH = c->Ly * c->H, d = c->d, W = c->W;
  float* kx = (float*)malloc((size_t)d * 4); float* vx = (float*)malloc((size_t)d * 4);
  for (int32_t i = 0; i < p->n_admit; i++) {
    int32_t r = p->admit_list[i], T = p->prompt_len[r];
    if (p->req_state[r] != ORC_REQ_ADMITTING) continue;
    for (int32_t j = 0; j < LyH; j++) {
      int32_t u = r * LyH + j;
      int32_t h = 0, l = 0, tp = 0;
      for (int32_t t = 0; t < T; t++) {
        const uint16_t* kr = k + (((int64_t)i * LyH + j) * kv_stride + t) * d;
        const uint16_t* vr = v + (((int64_t)i * LyH + j) * kv_stride + t) * d;
        if (t < T - W) {
          float s = sig[((int64_t)i * LyH + j) * sig_stride + t];
          if (s == 0.0f) s = 0.0f;
          int cls = prompt_class(p, u, s, t, T);
          if (cls == ORC_CLS_PRUNED) continue;
          if (cls == ORC_CLS_TOP) {                             /* NEXT-4: FP16 rows as given */
            int32_t st = write_token_top(p, u, tp++, kr, vr, s, t);
            if (st != ORC_OK) set_status(p, st);
            continue;
          }
          for (int32_t e = 0; e < d; e++) { kx[e] = orc_f32_from_f16(kr[e]); vx[e] = orc_f32_from_f16(vr[e]); }
          int32_t slot = (cls == ORC_CLS_HIGH) ? h++ : l++;
          int32_t st = write_token(p, cls, u, slot, kx, vx, s, t);
          if (st != ORC_OK) set_status(p, st);
        } else {
          memcpy(p->win_k + ((size_t)u * W + (size_t)(t % W)) * d, kr, (size_t)d * 2);
          memcpy(p->win_v + ((size_t)u * W + (size_t)(t % W)) * d, vr, (size_t)d * 2);
          float ws = sig[((int64_t)i * LyH + j) * sig_stride + t];
          if (ws == 0.0f) ws = 0.0f;
          p->win_sig[(size_t)u * W + (size_t)(t % W)] = ws;     /* the prompt phase's significance */
        }
      }
    }
  }
  free(kx); free(vx);
  /* Q30/Q37: a token rejected by this call does not stop the others; the request becomes ACTIVE (and can be
     freed) with the sticky status reporting the error */
  for (int32_t i = 0; i < p->n_admit; i++)
    if (p->req_state[p->admit_list[i]] == ORC_REQ_ADMITTING) p->req_state[p->admit_list[i]] = ORC_REQ_ACTIVE;
  p->n_admit = 0;
  return ORC_OK;
}

/* "Once a request is finished, all pages allocated for that request are recycled" — the request
   becomes PENDING_FREE; its pages return to the ring in the next orc_compact_alloc (a7). */
int32_t orc_free(orc_pool* p, const int32_t* req, int32_t n) {
  for (int32_t i = 0; i < n; i++) {
    if (req[i] < 0 || req[i] >= p->c.R) return ORC_ERR_INVALID;
    if (p->req_state[req[i]] != ORC_REQ_ACTIVE) return ORC_ERR_STATE;
    for (int32_t j = 0; j < i; j++) if (req[j] == req[i]) return ORC_ERR_STATE;
  }
  for (int32_t i = 0; i < n; i++) p->req_state[req[i]] = ORC_REQ_PENDING_FREE;
  return ORC_OK;
}

/* ------------------------------------------------------------------------------------------------
 * NEXT-2: decode attention over the compressed cache and the significance update.
 * Eq. 1 for the query of the newest token (position N-1) of every ACTIVE unit, G = q_per_kv
 * query heads sharing the KV head (GQA), over the unit's stored tokens (keys dequantized,
 * X^ = s*Q + z) and its FP16 window; every floating-point result is fixed by readings Q31-Q34:
 *   Q31 logit = fmul(dot, 1/sqrt(d)) with dot = serial fused multiply-add chain over elements e = 0..d-1,
 *       dot = fma(q_e, k_e, dot) from 0 (one rounding per element);
 *       tokens in the order: high slots 0..n_h-1, low slots 0..n_l-1, window oldest -> newest;
 *   Q32 p = exp(logit - max) with orc_exp (round-to-nearest range reduction + degree-6 polynomial, fixed
 *       operation order); Z = sum over pages in that order of the serial in-page sums (the window counts as
 *       pages of C_h tokens, oldest first, the last one possibly partial); a = fdiv(p, Z); the output row =
 *       the serial sum over pages (same order) of each page's fma chain over its tokens,
 *       o_page = fma(a, v_e, o_page) from 0;
 *   Q33 a token's significance is the mean of the scores it received from later tokens; a decode
 *       step adds the score of query N-1 (max over the G heads) to every token p < N-1:
 *       sig' = fdiv(fadd(fmul(sig, c), a), c + 1), c = N-2-p scores so far; a new token starts at 0;
 *   Q34 pages keep the updated significance in their score segment, the window in win_sig.
 * ----------------------------------------------------------------------------------------------*/
float orc_exp(float x) {
  const float log2e = 1.44269504088896341f;
  float t = x * log2e;                                   /* fmul_rn */
  if (t < -125.0f) return 0.0f;
  float n = rintf(t);                                    /* round to nearest even */
  float f = t - n;                                       /* exact, |f| <= 1/2 */
  /* 2^f = sum (ln2)^k f^k / k!, Horner, k = 0..6 */
  float r = 1.54035304e-4f;
  r = r * f + 1.33335581e-3f;
  r = r * f + 9.61812911e-3f;
  r = r * f + 5.55041087e-2f;
  r = r * f + 2.40226507e-1f;
  r = r * f + 6.93147181e-1f;
  r = r * f + 1.0f;
  uint32_t eb = (uint32_t)((int32_t)n + 127) << 23;      /* 2^n, n in [-125, 0] */
  float two_n;
  memcpy(&two_n, &eb, 4);
  return r * two_n;
}

typedef struct { const uint8_t* pg; int cls; int32_t idx; float* sig; int32_t pos; const uint16_t* wk;
                 const uint16_t* wv; } att_tok;

static void att_key(const orc_pool* p, const att_tok* t, float* k) {
  int32_t d = p->c.d;
  if (t->wk) { for (int32_t e = 0; e < d; e++) k[e] = orc_f32_from_f16(t->wk[e]); return; }
  const orc_class_geom* g = &p->g[t->cls];
  uint16_t s16, z16;
  memcpy(&s16, t->pg + g->off_kmeta + 4 * t->idx, 2); memcpy(&z16, t->pg + g->off_kmeta + 4 * t->idx + 2, 2);
  orc_dequantize(t->pg + g->off_k + t->idx * g->k_row, d, g->kbits, s16, z16, k);
}
static void att_val(const orc_pool* p, const att_tok* t, float* v) {
  int32_t d = p->c.d;
  if (t->wv) { for (int32_t e = 0; e < d; e++) v[e] = orc_f32_from_f16(t->wv[e]); return; }
  const orc_class_geom* g = &p->g[t->cls];
  uint16_t s16, z16;
  memcpy(&s16, t->pg + g->off_vmeta + 4 * t->idx, 2); memcpy(&z16, t->pg + g->off_vmeta + 4 * t->idx + 2, 2);
  orc_dequantize(t->pg + g->off_v + t->idx * g->v_row, d, g->vbits, s16, z16, v);
}

int32_t orc_attend(orc_pool* p, const uint16_t* q, float* out, float* probs) {
  const orc_config* c = &p->c;
  if (c->q_per_kv < 1 || c->top_tier) return ORC_ERR_INVALID;     /* NEXT-4 tier: no attention (Q44) */
  if (p->status != ORC_OK) return ORC_OK;
  const int32_t LyH = c->Ly * c->H, d = c->d, W = c->W, G = c->q_per_kv, M = c->M;
  att_tok* tok = (att_tok*)malloc(sizeof(att_tok) * (size_t)M);
  int32_t* tpage = (int32_t*)malloc(4 * (size_t)M);       /* page index of each token (window pages last) */
  float* lg = (float*)malloc(4 * (size_t)M * (size_t)G);
  float* a = (float*)malloc(4 * (size_t)M);
  float* kx = (float*)malloc(4 * (size_t)d);
  float* vx = (float*)malloc(4 * (size_t)d);
  float* pv = (float*)malloc(4 * (size_t)d);                  /* the current page's partial output row */
  const float scale = 1.0f / sqrtf((float)d);
  for (int32_t u = 0; u < p->U; u++) {
    int32_t r = u / LyH;
    if (p->req_state[r] != ORC_REQ_ACTIVE) continue;
    int32_t N = p->seq_len[r];
    /* token list (Q31 order) */
    int32_t n = 0, npage = 0;
    for (int cls = ORC_CLS_HIGH; cls <= ORC_CLS_LOW; cls++) {
      int32_t cnt = cls == ORC_CLS_HIGH ? p->n_h[u] : p->n_l[u], C = p->g[cls].C;
      for (int32_t s = 0; s < cnt; s++) {
        att_tok* t = &tok[n];
        int32_t idx;
        t->pg = slot_page(p, cls, u, s, &idx);
        t->cls = cls; t->idx = idx; t->wk = NULL; t->wv = NULL;
        t->sig = (float*)(t->pg + p->g[cls].off_score + 4 * idx);
        memcpy(&t->pos, t->pg + p->g[cls].off_pos + 4 * idx, 4);
        tpage[n] = npage + s / C;
        n++;
      }
      npage += (cnt + C - 1) / C;
    }
    const int32_t first = N - W > 0 ? N - W : 0, Cw = p->g[ORC_CLS_HIGH].C;
    for (int32_t ps = first; ps < N; ps++) {
      att_tok* t = &tok[n];
      size_t ws = (size_t)u * W + (size_t)(ps % W);
      t->pg = NULL; t->cls = 0; t->idx = 0; t->pos = ps;
      t->wk = p->win_k + ws * d; t->wv = p->win_v + ws * d; t->sig = &p->win_sig[ws];
      tpage[n] = npage + (ps - first) / Cw;                  /* Q32: window pages of C_h tokens, oldest first */
      n++;
    }
    for (int32_t i = 0; i < n; i++) a[i] = 0.0f;
    for (int32_t g = 0; g < G; g++) {
      const uint16_t* qg = q + ((size_t)u * G + g) * d;
      float m = -INFINITY;
      for (int32_t i = 0; i < n; i++) {
        att_key(p, &tok[i], kx);
        float dot = 0.0f;
        for (int32_t e = 0; e < d; e++) dot = fmaf(orc_f32_from_f16(qg[e]), kx[e], dot);   /* Q31 */
        float l = dot * scale;
        lg[(size_t)g * M + i] = l;
        if (l > m) m = l;
      }
      float Z = 0.0f, part = 0.0f;
      for (int32_t i = 0; i < n; i++) {
        float e = orc_exp(lg[(size_t)g * M + i] - m);
        lg[(size_t)g * M + i] = e;
        part = part + e;
        if (i == n - 1 || tpage[i + 1] != tpage[i]) { Z = Z + part; part = 0.0f; }
      }
      float* og = out ? out + ((size_t)u * G + g) * d : NULL;
      if (og) for (int32_t e = 0; e < d; e++) { og[e] = 0.0f; pv[e] = 0.0f; }
      for (int32_t i = 0; i < n; i++) {
        float ai = lg[(size_t)g * M + i] / Z;                /* fdiv_rn */
        if (ai > a[i]) a[i] = ai;                            /* GQA: max over the group */
        if (og) {                                            /* Q32: pages in order of in-page fma chains */
          att_val(p, &tok[i], vx);
          for (int32_t e = 0; e < d; e++) pv[e] = fmaf(ai, vx[e], pv[e]);
          if (i == n - 1 || tpage[i + 1] != tpage[i])
            for (int32_t e = 0; e < d; e++) { og[e] = og[e] + pv[e]; pv[e] = 0.0f; }
        }
      }
    }
    if (probs) for (int32_t i = 0; i < M; i++) probs[(size_t)u * M + i] = i < n ? a[i] : 0.0f;
    for (int32_t i = 0; i < n; i++) {                        /* Q33: running mean over later queries */
      int32_t cnt = N - 2 - tok[i].pos;
      if (cnt < 0) continue;                                 /* the query's own token */
      float sg;
      memcpy(&sg, tok[i].sig, 4);
      sg = (sg * (float)cnt + a[i]) / (float)(cnt + 1);
      memcpy(tok[i].sig, &sg, 4);
    }
  }
  free(tok); free(tpage); free(lg); free(a); free(kx); free(vx); free(pv);
  return ORC_OK;
}

/* ------------------------------------------------------------------------------------------------
 * NEXT-1 convenience entry point (used by the Fig. 5 replay): admit + plan + compact with
 * prefill_workflow = 1 for this call only; reclaimed_out receives the reclaimed IDs in ring order.
 * ----------------------------------------------------------------------------------------------*/
int32_t orc_prefill_conservative(orc_pool* p, const int32_t* req, const int32_t* len, int32_t n,
                                 const float* sig, int64_t sig_stride, int32_t* reclaimed_out, int64_t* n_reclaimed) {
  int32_t saved = p->c.prefill_workflow;
  int64_t end = (p->start + p->free) % p->c.P;
  int32_t st = orc_classify_prefill(p, req, len, n, sig, sig_stride, NULL);
  if (st == ORC_OK) {
    p->c.prefill_workflow = 1;
    st = orc_compact_alloc(p, NULL);
    p->c.prefill_workflow = saved;
  }
  if (st != ORC_OK) return st;
  for (int64_t k = 0; k < p->last_reclaimed; k++)
    if (reclaimed_out) reclaimed_out[k] = p->ring[(end + k) % p->c.P];
  if (n_reclaimed) *n_reclaimed = p->last_reclaimed;
  return ORC_OK;
}
