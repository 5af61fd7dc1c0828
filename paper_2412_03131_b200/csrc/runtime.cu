// runtime.cu — host side of the C ABI (include/dkv.h): validation, arena layout, the request-state
// mirror and call sequencing, kernel launches.  No device memory is allocated after dkv_pool_init; every
// call is asynchronous on the caller's stream except dkv_pool_query.
#include <stdlib.h>
#include <string.h>

#include <vector>

#include "dkv_internal.cuh"

using namespace dkv;

namespace {

constexpr int64_t kAlign = 256;
int64_t align_up(int64_t x, int64_t a) { return (x + a - 1) / a * a; }

bool bits_ok(int32_t b) { return b == 2 || b == 4 || b == 8; }

void class_geom(int d, int C, int kb, int vb, ClassGeom& g) {
  auto a16 = [](int x) { return (x + 15) / 16 * 16; };
  g.C = C; g.kbits = kb; g.vbits = vb;
  g.k_row = d * kb / 8;
  g.v_row = d * vb / 8;
  g.off_k = 0;
  g.off_kmeta = a16(g.off_k + C * g.k_row);
  g.off_v = a16(g.off_kmeta + 4 * C);
  g.off_vmeta = a16(g.off_v + C * g.v_row);
  g.off_score = a16(g.off_vmeta + 4 * C);
  g.off_pos = a16(g.off_score + 4 * C);
}
int class_end(const ClassGeom& g) { return g.off_pos + 4 * g.C; }

constexpr int kAttSlots = 296;                               // 2 x 148 SMs
constexpr int64_t kAttSmemLongThreshold = 160 * 1024;         // logits + (s, z) bytes beyond which HBM slots exist
constexpr int kTcSlots = 4 * 148;                              // dkv_attend_tc: persistent CTAs (<= 4 per SM)
// dkv_attend_tc's logit rows per CTA slot (GP of them): the longest context plus the padding of the unit's last
// high and last low page (rows are page-aligned: <= 15 + 31)
static int64_t tc_slot_rows(const dkv_config_t* c) { return (c->max_seq_len + 31) / 32 * 32 + 64; }
static int64_t tc_gp(const dkv_config_t* c) { return c->q_per_kv <= 4 ? 4 : 8; }
static bool tc_scratch_needed(const dkv_config_t* c) { return c->q_per_kv > 0 && !c->top_tier; }

struct Geometry {
  int32_t U, L, page_bytes, num_tiles, tile_units, nseg, Lt;
  ClassGeom g[3];
  ClassGeom gt;                                              // NEXT-4 TOP class (fp16 rows)
  int64_t off_pf_nt, off_pf_seg_t;                           // NEXT-4 prompt scratch (not in dkv_layout_t)
};

// NEXT-4 (Q40): a TOP page = C fp16 K rows, C fp16 V rows (no metadata), scores, positions; 16-B aligned
void top_geom(int d, int C, ClassGeom& g) {
  auto a16 = [](int x) { return (x + 15) / 16 * 16; };
  g.C = C; g.kbits = 16; g.vbits = 16;
  g.k_row = 2 * d;
  g.v_row = 2 * d;
  g.off_k = 0;
  g.off_kmeta = g.off_k + C * g.k_row;                       // empty
  g.off_v = a16(g.off_kmeta);
  g.off_vmeta = g.off_v + C * g.v_row;                       // empty
  g.off_score = a16(g.off_vmeta);
  g.off_pos = a16(g.off_score + 4 * C);
}

bool validate(const dkv_config_t* c, Geometry& G) {
  if (!c) return false;
  if (c->max_requests < 1 || c->num_layers < 1 || c->num_kv_heads < 1) return false;
  if (c->head_dim != 64 && c->head_dim != 128) return false;
  if (c->max_seq_len < 1 || c->window < 0 || c->window > c->max_seq_len) return false;
  if (c->page_tokens_high < 4 || c->page_tokens_high % 4 || c->page_tokens_low < c->page_tokens_high ||
      c->page_tokens_low % 4)
    return false;
  if (!bits_ok(c->kbits_high) || !bits_ok(c->vbits_high) || !bits_ok(c->kbits_low) || !bits_ok(c->vbits_low))
    return false;
  if (c->num_pages < 1) return false;
  if (!(c->alpha_h >= 0.0f && c->alpha_h <= 3.0e38f) || !(c->alpha_l >= 0.0f && c->alpha_l <= 3.0e38f)) return false;
  if (c->prompt_denominator != 0 && c->prompt_denominator != 1) return false;
  if (c->tile_units != 0 && c->tile_units != 256 && c->tile_units != 512 && c->tile_units != 1024) return false;
  if (c->prefill_workflow != 0 && c->prefill_workflow != 1) return false;
  if (c->q_per_kv < 0 || c->q_per_kv > 16) return false;
  // NEXT-4 (Q38, Q43): alpha_t >= alpha_h, TOP pages of whole 4-token groups, the exact prompt workflow
  if (c->top_tier != 0 && (c->top_tier != 1 || !(c->alpha_t >= c->alpha_h && c->alpha_t <= 3.0e38f) ||
                           c->page_tokens_top < 4 || c->page_tokens_top % 4 || c->prefill_workflow != 0))
    return false;
  const int64_t U = (int64_t)c->max_requests * c->num_layers * c->num_kv_heads;
  if (U >= (1 << 24)) return false;
  G.U = (int32_t)U;
  // P:499 table length, corrected by Q12
  G.L = (c->max_seq_len + c->page_tokens_high - 1) / c->page_tokens_high + (c->window < c->page_tokens_high ? 1 : 0);
  if ((int64_t)G.U * G.L >= (1 << 28)) return false;
  class_geom(c->head_dim, c->page_tokens_high, c->kbits_high, c->vbits_high, G.g[DKV_CLS_HIGH]);
  class_geom(c->head_dim, c->page_tokens_low, c->kbits_low, c->vbits_low, G.g[DKV_CLS_LOW]);
  G.g[0] = G.g[DKV_CLS_HIGH];
  int e = class_end(G.g[1]) > class_end(G.g[2]) ? class_end(G.g[1]) : class_end(G.g[2]);
  G.Lt = 1;
  memset(&G.gt, 0, sizeof(G.gt));
  if (c->top_tier) {
    top_geom(c->head_dim, c->page_tokens_top, G.gt);
    if (class_end(G.gt) > e) e = class_end(G.gt);
    G.Lt = (c->max_seq_len + c->page_tokens_top - 1) / c->page_tokens_top;   // Q41
    if ((int64_t)G.U * G.Lt >= (1 << 28)) return false;
  }
  G.page_bytes = (e + 127) / 128 * 128;
  G.tile_units = c->tile_units ? c->tile_units : 1024;
  G.num_tiles = (G.U + G.tile_units - 1) / G.tile_units;
  G.nseg = (c->max_seq_len + kSegTokens - 1) / kSegTokens;
  return true;
}

bool make_layout(const dkv_config_t* c, Geometry& G, dkv_layout_t& Lo) {
  if (!validate(c, G)) return false;
  memset(&Lo, 0, sizeof(Lo));
  const int64_t U = G.U, R = c->max_requests, P = c->num_pages;
  int64_t o = 0;
  auto take = [&](int64_t bytes) { int64_t at = o; o = align_up(o + bytes, kAlign); return at; };
  Lo.off_ctrl = take(256);
  Lo.off_stats = take(32);
  Lo.off_tile_status = take(8 * (int64_t)G.num_tiles);
  Lo.off_tile_sums = take(24 * (int64_t)G.num_tiles);
  Lo.off_tsum = take(16 * (int64_t)G.num_tiles);
  Lo.off_rec = take(16 * (int64_t)G.U);
  Lo.off_win_sig = take(4 * (int64_t)G.U * c->window);
  Lo.off_secmin = take(32 * (int64_t)G.U);
  Lo.off_head_alpha = take(8 * (int64_t)c->num_layers * c->num_kv_heads);
  // NEXT-2 long contexts: when q_per_kv * max_seq_len logits + (s, z) pairs cannot stay in shared memory
  // (227 KB per CTA on sm_100), kAttSlots persistent CTAs keep them in HBM slots
  {
    const int64_t GP = (c->q_per_kv + 3) / 4 * 4, Mp = (c->max_seq_len + 31) / 32 * 32;
    const bool need = c->q_per_kv > 0 && (GP + 2) * Mp * 4 > kAttSmemLongThreshold;
    Lo.off_att_scratch = take(need ? (int64_t)kAttSlots * (GP + 2) * Mp * 4 : 0);
  }
  Lo.off_tc_scratch = take(tc_scratch_needed(c) ? (int64_t)kTcSlots * 2 * tc_slot_rows(c) * tc_gp(c) * 4 : 0);
  Lo.off_qpid = take(16 * U);
  Lo.off_ring = take(4 * P);
  Lo.off_table = take(4 * U * G.L);
  Lo.off_ttable = take(4 * U * G.Lt);
  Lo.off_n_h = take(4 * U);
  Lo.off_n_l = take(4 * U);
  Lo.off_req_state = take(R);
  Lo.off_seq_len = take(4 * R);
  Lo.off_prompt_len = take(4 * R);
  Lo.off_admit = take(4 * R);
  Lo.off_pf_nh = take(4 * U);
  Lo.off_pf_nl = take(4 * U);
  Lo.off_pf_seg = take(8 * U * G.nseg);
  Lo.off_n_t = take(4 * U);                                  // NEXT-4 (zeroed with the prefill scratch)
  G.off_pf_nt = take(4 * U);
  G.off_pf_seg_t = take(4 * U * G.nseg);
  const int64_t wbytes = 2 * U * (int64_t)c->window * c->head_dim;
  Lo.off_win_k = take(wbytes);
  Lo.off_win_v = take(wbytes);
  o = align_up(o, 4096);
  Lo.off_pages = take(P * (int64_t)G.page_bytes);
  Lo.arena_bytes = o;
  Lo.units = G.U; Lo.table_len = G.L; Lo.page_bytes = G.page_bytes; Lo.num_tiles = G.num_tiles;
  Lo.tile_units = G.tile_units; Lo.seg_tokens = kSegTokens; Lo.num_segs = G.nseg;
  Lo.table_len_top = G.Lt;
  Lo.C_top = G.gt.C; Lo.row_top = G.gt.k_row; Lo.off_k_top = G.gt.off_k; Lo.off_v_top = G.gt.off_v;
  Lo.off_score_top = G.gt.off_score; Lo.off_pos_top = G.gt.off_pos;
  for (int k = 1; k <= 2; k++) {
    const ClassGeom& g = G.g[k];
    Lo.C[k] = g.C; Lo.k_row[k] = g.k_row; Lo.v_row[k] = g.v_row; Lo.off_k[k] = g.off_k;
    Lo.off_kmeta[k] = g.off_kmeta; Lo.off_v[k] = g.off_v; Lo.off_vmeta[k] = g.off_vmeta;
    Lo.off_score[k] = g.off_score; Lo.off_pos[k] = g.off_pos;
  }
  return true;
}

enum Seq { SEQ_IDLE = 0, SEQ_CLASSIFIED = 1, SEQ_COMPACTED = 2 };

}  // namespace

struct dkv_pool {
  dkv_config_t cfg;
  Geometry G;
  dkv_layout_t lay;
  PoolDev dev;
  uint8_t* base;
  std::vector<int8_t> req_state;     // host mirror
  std::vector<int32_t> seq_len;      // host mirror
  std::vector<int32_t> admitted;     // current admission batch
  std::vector<int32_t> admitted_len;
  int seq;                           // SEQ_*
  int phase;                         // phase of the last classify
  Ctrl* h_ctrl;                      // pinned host staging for query
  int8_t* h_req;
  int32_t* h_seq;
  bool recovering;                   // last query reported an error: frees allowed out of sequence
  cudaStream_t copy_stream;          // dkv_decode_step_host: the new tokens' K/V H2D copy (created on first use)
  cudaEvent_t ev_ready;              // ... ordered after prior work on the caller's stream
  cudaEvent_t ev_kv;                 // ... the K/V copy done
};

extern "C" {

const char* dkv_status_string(dkv_status_t st) {
  switch (st) {
    case DKV_OK: return "ok";
    case DKV_ERR_INVALID_ARG: return "invalid argument";
    case DKV_ERR_STATE: return "request state or call order violated";
    case DKV_ERR_OOM: return "out of pages (allocation not applied)";
    case DKV_ERR_NONFINITE: return "non-finite input";
    case DKV_ERR_OVERFLOW: return "page table overflow";
    case DKV_ERR_CUDA: return "CUDA error";
    default: return "unknown status";
  }
}

size_t dkv_arena_bytes(const dkv_config_t* cfg) {
  Geometry G;
  dkv_layout_t Lo;
  if (!make_layout(cfg, G, Lo)) return 0;
  return (size_t)Lo.arena_bytes;
}

dkv_status_t dkv_pool_layout(const dkv_config_t* cfg, dkv_layout_t* out) {
  Geometry G;
  if (!out || !make_layout(cfg, G, *out)) return DKV_ERR_INVALID_ARG;
  return DKV_OK;
}

dkv_status_t dkv_pool_init(const dkv_config_t* cfg, void* d_arena, size_t arena_bytes, dkv_stream_t s,
                           dkv_pool_t* out) {
  if (!out) return DKV_ERR_INVALID_ARG;
  *out = nullptr;
  Geometry G;
  dkv_layout_t Lo;
  if (!make_layout(cfg, G, Lo)) return DKV_ERR_INVALID_ARG;
  if (!d_arena || ((uintptr_t)d_arena % kAlign) || arena_bytes < (size_t)Lo.arena_bytes) return DKV_ERR_INVALID_ARG;
  int ndev = 0;
  if (cudaGetDeviceCount(&ndev) != cudaSuccess || ndev == 0) return DKV_ERR_CUDA;
  cudaPointerAttributes attr;
  if (cudaPointerGetAttributes(&attr, d_arena) != cudaSuccess || attr.type != cudaMemoryTypeDevice) {
    cudaGetLastError();
    return DKV_ERR_INVALID_ARG;
  }
  const int cores = compact_max_coresident(G.tile_units);
  if (cores <= 0) return DKV_ERR_CUDA;
  if (G.num_tiles > cores) return DKV_ERR_INVALID_ARG;   // the scan's grid barrier needs co-residency
  {
    // multiply-high division constants, checked over every dividend a kernel can pass (unreachable failure)
    const int32_t LyH = cfg->num_layers * cfg->num_kv_heads;
    if (!fastdiv_check(make_fastdiv(LyH), G.U) ||
        !fastdiv_check(make_fastdiv(cfg->window > 0 ? cfg->window : 1), (int64_t)cfg->max_seq_len + 1) ||
        !fastdiv_check(make_fastdiv(cfg->page_tokens_high), (int64_t)G.L * cfg->page_tokens_high) ||
        !fastdiv_check(make_fastdiv(cfg->page_tokens_low), (int64_t)G.L * cfg->page_tokens_low))
      return DKV_ERR_INVALID_ARG;
  }
  dkv_pool* p = new dkv_pool();
  p->cfg = *cfg;
  p->G = G;
  p->lay = Lo;
  p->base = (uint8_t*)d_arena;
  p->req_state.assign(cfg->max_requests, DKV_REQ_IDLE);
  p->seq_len.assign(cfg->max_requests, 0);
  p->seq = SEQ_IDLE;
  p->phase = -1;
  p->recovering = false;
  if (cudaMallocHost(&p->h_ctrl, sizeof(Ctrl)) != cudaSuccess ||
      cudaMallocHost(&p->h_req, cfg->max_requests) != cudaSuccess ||
      cudaMallocHost(&p->h_seq, 4 * (size_t)cfg->max_requests) != cudaSuccess) {
    delete p;
    return DKV_ERR_CUDA;
  }
  PoolDev& d = p->dev;
  memset(&d, 0, sizeof(d));
  d.R = cfg->max_requests; d.Ly = cfg->num_layers; d.H = cfg->num_kv_heads; d.LyH = d.Ly * d.H; d.U = G.U;
  d.d = cfg->head_dim; d.M = cfg->max_seq_len; d.W = cfg->window; d.L = G.L; d.P = cfg->num_pages;
  d.page_bytes = G.page_bytes; d.Ch = cfg->page_tokens_high; d.Cl = cfg->page_tokens_low;
  d.prompt_den = cfg->prompt_denominator; d.num_tiles = G.num_tiles; d.tile_units = G.tile_units; d.nseg = G.nseg;
  d.alpha_h = cfg->alpha_h; d.alpha_l = cfg->alpha_l;
  for (int k = 0; k < 3; k++) d.g[k] = G.g[k];
  d.div_LyH = make_fastdiv(d.LyH);
  d.div_W = make_fastdiv(d.W > 0 ? d.W : 1);
  d.div_Ch = make_fastdiv(d.Ch);
  d.div_Cl = make_fastdiv(d.Cl);
  uint8_t* b = p->base;
  d.ctrl = (Ctrl*)(b + Lo.off_ctrl);
  d.stats = (int64_t*)(b + Lo.off_stats);
  d.tile_status = (unsigned long long*)(b + Lo.off_tile_status);
  d.tile_sums = (int64_t*)(b + Lo.off_tile_sums);
  d.tsum = (uint32_t*)(b + Lo.off_tsum);
  d.rec = (int32_t*)(b + Lo.off_rec);
  d.win_sig = (float*)(b + Lo.off_win_sig);
  d.secmin = (int32_t*)(b + Lo.off_secmin);
  d.qpid = (int4*)(b + Lo.off_qpid);
  d.top = cfg->top_tier;
  d.alpha_t = cfg->alpha_t;
  d.Lt = G.Lt;
  d.Ct = cfg->top_tier ? cfg->page_tokens_top : 4;
  d.gt = G.gt;
  d.ttable = (int32_t*)(b + Lo.off_ttable);
  d.n_t = (int32_t*)(b + Lo.off_n_t);
  d.pf_nt = (int32_t*)(b + G.off_pf_nt);
  d.pf_seg_t = (int32_t*)(b + G.off_pf_seg_t);
  d.div_Ct = make_fastdiv(d.Ct);
  d.head_alpha = (float*)(b + Lo.off_head_alpha);
  {
    const int64_t GP = (cfg->q_per_kv + 3) / 4 * 4, Mp = (cfg->max_seq_len + 31) / 32 * 32;
    const bool need = cfg->q_per_kv > 0 && (GP + 2) * Mp * 4 > kAttSmemLongThreshold;
    d.att_scratch = need ? (float*)(b + Lo.off_att_scratch) : nullptr;
    d.att_slots = need ? kAttSlots : 0;
  }
  d.tc_scratch = tc_scratch_needed(cfg) ? (float*)(b + Lo.off_tc_scratch) : nullptr;
  d.tc_slots = tc_scratch_needed(cfg) ? kTcSlots : 0;
  d.tc_slot_rows = (int32_t)tc_slot_rows(cfg);
  d.use_head_alpha = 0;
  d.G = cfg->q_per_kv;
  d.prefill_wf = cfg->prefill_workflow;
  d.ring = (int32_t*)(b + Lo.off_ring);
  d.table = (int32_t*)(b + Lo.off_table);
  d.n_h = (int32_t*)(b + Lo.off_n_h);
  d.n_l = (int32_t*)(b + Lo.off_n_l);
  d.req_state = (int8_t*)(b + Lo.off_req_state);
  d.seq_len = (int32_t*)(b + Lo.off_seq_len);
  d.prompt_len = (int32_t*)(b + Lo.off_prompt_len);
  d.admit = (int32_t*)(b + Lo.off_admit);
  d.pf_nh = (int32_t*)(b + Lo.off_pf_nh);
  d.pf_nl = (int32_t*)(b + Lo.off_pf_nl);
  d.pf_seg = (int32_t*)(b + Lo.off_pf_seg);
  d.win_k = (__half*)(b + Lo.off_win_k);
  d.win_v = (__half*)(b + Lo.off_win_v);
  d.pages = b + Lo.off_pages;
  cudaError_t e = cudaMemsetAsync(b + Lo.off_pages, 0, (size_t)(Lo.arena_bytes - Lo.off_pages), s);
  if (e == cudaSuccess) e = cudaMemsetAsync(b + Lo.off_win_k, 0, (size_t)(Lo.off_pages - Lo.off_win_k), s);
  if (e == cudaSuccess) e = cudaMemsetAsync(b + Lo.off_pf_seg, 0, (size_t)(Lo.off_win_k - Lo.off_pf_seg), s);
  // control block, counters, scan / workflow / recycle scratch, window significance and section minima
  // (everything laid out before the ring) start zeroed: every byte initialised
  if (e == cudaSuccess) e = cudaMemsetAsync(b, 0, (size_t)Lo.off_ring, s);
  if (e == cudaSuccess) e = launch_init(d, s);
  if (e != cudaSuccess) {
    dkv_pool_destroy(p);
    return DKV_ERR_CUDA;
  }
  *out = p;
  return DKV_OK;
}

dkv_status_t dkv_pool_destroy(dkv_pool_t p) {
  if (!p) return DKV_ERR_INVALID_ARG;
  if (p->h_ctrl) cudaFreeHost(p->h_ctrl);
  if (p->h_req) cudaFreeHost(p->h_req);
  if (p->h_seq) cudaFreeHost(p->h_seq);
  if (p->copy_stream) cudaStreamDestroy(p->copy_stream);
  if (p->ev_ready) cudaEventDestroy(p->ev_ready);
  if (p->ev_kv) cudaEventDestroy(p->ev_kv);
  delete p;
  return DKV_OK;
}

// The host-detectable conditions of a decode dkv_classify: call order (a decode step interrupted by a device
// error may be abandoned: its compact_alloc applied nothing) and no ACTIVE request at max_seq_len.  *max_len
// receives the longest ACTIVE request.
static dkv_status_t decode_precheck(const dkv_pool* p, int* max_len) {
  if (p->seq != SEQ_IDLE && !(p->recovering && p->phase == DKV_PHASE_DECODE)) return DKV_ERR_STATE;
  int m = 0;
  for (int r = 0; r < p->cfg.max_requests; r++) {
    if (p->req_state[r] != DKV_REQ_ACTIVE) continue;
    if (p->seq_len[r] >= p->cfg.max_seq_len) return DKV_ERR_STATE;
    m = p->seq_len[r] > m ? p->seq_len[r] : m;
  }
  *max_len = m;
  return DKV_OK;
}

dkv_status_t dkv_classify(dkv_pool_t p, int32_t phase, const int32_t* h_req, const int32_t* h_len, int32_t n,
                          const float* d_sig, int64_t sig_stride, dkv_decision_t* d_dec, uint8_t* d_token_class,
                          dkv_stream_t s) {
  if (!p) return DKV_ERR_INVALID_ARG;
  const int R = p->cfg.max_requests;
  if (phase == DKV_PHASE_DECODE) {
    if (!d_dec) return DKV_ERR_INVALID_ARG;              // d_sig NULL: t_c's significance from the window
    int max_len = 0;
    const dkv_status_t pre = decode_precheck(p, &max_len);
    if (pre != DKV_OK) return pre;
    cudaError_t e = launch_classify_decode(p->dev, d_sig, d_dec, max_len, (cudaStream_t)s);
    if (e != cudaSuccess) return DKV_ERR_CUDA;
  } else if (phase == DKV_PHASE_PREFILL) {
    if (p->seq != SEQ_IDLE && !(p->recovering && p->phase == DKV_PHASE_DECODE)) return DKV_ERR_STATE;
    if (n < 0 || n > R || (n > 0 && (!h_req || !h_len || !d_sig))) return DKV_ERR_INVALID_ARG;
    int max_len = 0;
    std::vector<char> seen(R, 0);
    for (int i = 0; i < n; i++) {
      const int r = h_req[i];
      if (r < 0 || r >= R || h_len[i] < 0 || h_len[i] > p->cfg.max_seq_len || h_len[i] > sig_stride || seen[r])
        return DKV_ERR_INVALID_ARG;
      if (p->req_state[r] != DKV_REQ_IDLE) return DKV_ERR_STATE;
      seen[r] = 1;
      if (h_len[i] > max_len) max_len = h_len[i];
    }
    cudaError_t e = launch_set_requests(p->dev, h_req, h_len, n, 0, (cudaStream_t)s);
    if (e == cudaSuccess) e = launch_classify_prefill(p->dev, n, d_sig, sig_stride, d_token_class, max_len, (cudaStream_t)s);
    if (e != cudaSuccess) return DKV_ERR_CUDA;
    p->admitted.assign(h_req, h_req + n);
    p->admitted_len.assign(h_len, h_len + n);
    for (int i = 0; i < n; i++) p->req_state[h_req[i]] = DKV_REQ_ADMITTING;
  } else {
    return DKV_ERR_INVALID_ARG;
  }
  p->phase = phase;
  p->seq = SEQ_CLASSIFIED;
  return DKV_OK;
}

dkv_status_t dkv_compact_alloc(dkv_pool_t p, const dkv_decision_t* d_dec, dkv_stream_t s) {
  if (!p) return DKV_ERR_INVALID_ARG;
  if (p->seq == SEQ_IDLE && !p->recovering) return DKV_ERR_STATE;
  if (p->phase == DKV_PHASE_DECODE && !d_dec) return DKV_ERR_INVALID_ARG;
  cudaError_t e;
  if (p->phase == DKV_PHASE_PREFILL && p->cfg.prefill_workflow == 1) {
    // the paper's prompt workflow: recycle (no allocation), then conservative blocks + reclaim
    e = launch_compact_alloc(p->dev, d_dec, p->phase, (cudaStream_t)s, /*alloc=*/false);
    if (e == cudaSuccess) e = launch_prefill_conservative(p->dev, (cudaStream_t)s);
  } else {
    // decode steps that recycle finished requests: in the fast path the scan kernel only records each freed
    // unit's ring offset and a second, wide kernel copies the page IDs (one warp per freed unit, all SMs) —
    // inside the scan kernel the copy would run on the one or two CTAs whose tile holds the request.  (In a
    // decode-step CUDA graph, which has no host list, the quant_write kernel does these copies.)
    std::vector<int32_t> freed;
    if (p->phase == DKV_PHASE_DECODE)
      for (int r = 0; r < p->cfg.max_requests; r++)
        if (p->req_state[r] == DKV_REQ_PENDING_FREE) freed.push_back(r);
    e = launch_compact_alloc(p->dev, d_dec, p->phase, (cudaStream_t)s, /*alloc=*/true,
                             /*defer_recycle=*/p->phase == DKV_PHASE_DECODE);
    if (e == cudaSuccess && !freed.empty())
      e = launch_recycle(p->dev, freed.data(), (int)freed.size(), (cudaStream_t)s);
  }
  if (e != cudaSuccess) return DKV_ERR_CUDA;
  const int R = p->cfg.max_requests;
  for (int r = 0; r < R; r++) {
    if (p->req_state[r] == DKV_REQ_PENDING_FREE) { p->req_state[r] = DKV_REQ_IDLE; p->seq_len[r] = 0; }
    else if (p->phase == DKV_PHASE_DECODE && p->req_state[r] == DKV_REQ_ACTIVE) p->seq_len[r] += 1;
  }
  if (p->phase == DKV_PHASE_PREFILL)
    for (size_t i = 0; i < p->admitted.size(); i++) p->seq_len[p->admitted[i]] = p->admitted_len[i];
  p->seq = SEQ_COMPACTED;
  return DKV_OK;
}

dkv_status_t dkv_quant_write(dkv_pool_t p, int32_t phase, const dkv_decision_t* d_dec, const uint16_t* d_k,
                             const uint16_t* d_v, int64_t kv_stride, const float* d_sig, int64_t sig_stride,
                             dkv_stream_t s) {
  if (!p) return DKV_ERR_INVALID_ARG;
  if (p->seq != SEQ_COMPACTED || phase != p->phase) return DKV_ERR_STATE;
  cudaError_t e;
  if (phase == DKV_PHASE_DECODE) {
    if (!d_dec || !d_k || !d_v) return DKV_ERR_INVALID_ARG;
    e = launch_quant_decode(p->dev, d_dec, d_k, d_v, d_sig, (cudaStream_t)s);
  } else {
    const int n = (int)p->admitted.size();
    int max_len = 0;
    for (int i = 0; i < n; i++) max_len = p->admitted_len[i] > max_len ? p->admitted_len[i] : max_len;
    if (n > 0 && (!d_k || !d_v || !d_sig || kv_stride < max_len || sig_stride < max_len)) return DKV_ERR_INVALID_ARG;
    e = launch_quant_prefill(p->dev, n, d_k, d_v, kv_stride, d_sig, sig_stride, max_len, (cudaStream_t)s);
    for (int i = 0; i < n; i++) p->req_state[p->admitted[i]] = DKV_REQ_ACTIVE;
    p->admitted.clear();
    p->admitted_len.clear();
  }
  if (e != cudaSuccess) return DKV_ERR_CUDA;
  p->seq = SEQ_IDLE;
  p->recovering = false;
  return DKV_OK;
}

dkv_status_t dkv_attend(dkv_pool_t p, const uint16_t* d_q, float* d_out, float* d_probs, dkv_stream_t s) {
  if (!p || !d_q || p->cfg.top_tier) return DKV_ERR_INVALID_ARG;   // NEXT-4 tier: no attention (Q44)
  if (p->seq != SEQ_IDLE) return DKV_ERR_STATE;                // between sequences only
  const int G = p->cfg.q_per_kv;
  if (!(G == 1 || G == 2 || G == 4 || G == 5 || G == 7 || G == 8)) return DKV_ERR_INVALID_ARG;
  int dev = 0, optin = 0;
  if (cudaGetDevice(&dev) != cudaSuccess ||
      cudaDeviceGetAttribute(&optin, cudaDevAttrMaxSharedMemoryPerBlockOptin, dev) != cudaSuccess)
    return DKV_ERR_CUDA;
  int TS = 1;                                                    // tokens a unit can hold: <= its length
  for (int r = 0; r < p->cfg.max_requests; r++)
    if (p->req_state[r] == DKV_REQ_ACTIVE && p->seq_len[r] > TS) TS = p->seq_len[r];
  TS = (TS + 31) & ~31;
  if (attend_smem_bytes(p->dev, TS) > (size_t)optin) {
    // long context: logits in the HBM scratch slots (persistent kernel), token capacity = max_seq_len
    if (!p->dev.att_scratch || attend_long_smem_bytes(p->dev) > (size_t)optin) return DKV_ERR_INVALID_ARG;
    TS = -((p->cfg.max_seq_len + 31) & ~31);
  }
  cudaError_t e = launch_attend(p->dev, d_q, d_out, d_probs, TS, (cudaStream_t)s);
  return e == cudaSuccess ? DKV_OK : DKV_ERR_CUDA;
}

dkv_status_t dkv_attend_tc(dkv_pool_t p, const uint16_t* d_q, float* d_out, float* d_probs, dkv_stream_t s) {
  if (!p || !d_q || p->cfg.top_tier) return DKV_ERR_INVALID_ARG;
  if (p->seq != SEQ_IDLE) return DKV_ERR_STATE;
  const int G = p->cfg.q_per_kv;
  if (!(G == 1 || G == 2 || G == 4 || G == 5 || G == 7 || G == 8)) return DKV_ERR_INVALID_ARG;
  int dev = 0, optin = 0;
  if (cudaGetDevice(&dev) != cudaSuccess ||
      cudaDeviceGetAttribute(&optin, cudaDevAttrMaxSharedMemoryPerBlockOptin, dev) != cudaSuccess)
    return DKV_ERR_CUDA;
  // page geometries the kernel does not tile take the exact path (documented in dkv.h); logits live in the
  // arena's per-CTA scratch slots, so any context up to max_seq_len runs here
  if (!attend_tc_supported(p->dev) || attend_tc_smem_bytes(p->dev) > (size_t)optin)
    return dkv_attend(p, d_q, d_out, d_probs, s);
  int active = 0, max_len = 0;                                   // host mirror: chooses the split-sequence form
  for (int r = 0; r < p->cfg.max_requests; r++)
    if (p->req_state[r] == DKV_REQ_ACTIVE) { active++; max_len = p->seq_len[r] > max_len ? p->seq_len[r] : max_len; }
  const int units = active * p->cfg.num_layers * p->cfg.num_kv_heads;
  return launch_attend_tc(p->dev, d_q, d_out, d_probs, units, max_len, (cudaStream_t)s) == cudaSuccess ? DKV_OK
                                                                                                       : DKV_ERR_CUDA;
}

dkv_status_t dkv_audit(dkv_pool_t p, uint32_t* d_scratch, int64_t* d_result, dkv_stream_t s) {
  if (!p || !d_scratch || !d_result) return DKV_ERR_INVALID_ARG;
  if (p->seq != SEQ_IDLE) return DKV_ERR_STATE;                // between sequences only
  return launch_audit(p->dev, d_scratch, d_result, (cudaStream_t)s) == cudaSuccess ? DKV_OK : DKV_ERR_CUDA;
}

dkv_status_t dkv_set_head_thresholds(dkv_pool_t p, const float* h_alpha_h, const float* h_alpha_l, dkv_stream_t s) {
  if (!p) return DKV_ERR_INVALID_ARG;
  if (p->seq != SEQ_IDLE) return DKV_ERR_STATE;
  if (!h_alpha_h || !h_alpha_l) {
    p->dev.use_head_alpha = 0;
    return DKV_OK;
  }
  const int LyH = p->dev.LyH;
  std::vector<float> v(2 * (size_t)LyH);
  for (int i = 0; i < LyH; i++) {
    const float a = h_alpha_h[i], b = h_alpha_l[i];
    if (!(a >= 0.0f && a <= 3.0e38f) || !(b >= 0.0f && b <= 3.0e38f)) return DKV_ERR_INVALID_ARG;
    if (p->cfg.top_tier && a > p->cfg.alpha_t) return DKV_ERR_INVALID_ARG;   // Q38: alpha_h <= alpha_t
    v[2 * i] = a;
    v[2 * i + 1] = b;
  }
  // pageable source: cudaMemcpyAsync stages it before returning, so the host arrays may be reused
  cudaError_t e = cudaMemcpyAsync(p->dev.head_alpha, v.data(), 8 * (size_t)LyH, cudaMemcpyHostToDevice,
                                  (cudaStream_t)s);
  if (e != cudaSuccess) return DKV_ERR_CUDA;
  p->dev.use_head_alpha = 1;
  return DKV_OK;
}

dkv_status_t dkv_free(dkv_pool_t p, const int32_t* h_req, int32_t n, dkv_stream_t s) {
  if (!p) return DKV_ERR_INVALID_ARG;
  if (p->seq != SEQ_IDLE && !p->recovering) return DKV_ERR_STATE;
  const int R = p->cfg.max_requests;
  if (n < 0 || n > R || (n > 0 && !h_req)) return DKV_ERR_INVALID_ARG;
  std::vector<char> seen(R, 0);
  for (int i = 0; i < n; i++) {
    const int r = h_req[i];
    if (r < 0 || r >= R) return DKV_ERR_INVALID_ARG;
    if (p->req_state[r] != DKV_REQ_ACTIVE || seen[r]) return DKV_ERR_STATE;
    seen[r] = 1;
  }
  cudaError_t e = launch_set_requests(p->dev, h_req, nullptr, n, 1, (cudaStream_t)s);
  if (e != cudaSuccess) return DKV_ERR_CUDA;
  for (int i = 0; i < n; i++) p->req_state[h_req[i]] = DKV_REQ_PENDING_FREE;
  return DKV_OK;
}

dkv_status_t dkv_pool_query(dkv_pool_t p, dkv_stats_t* out, dkv_stream_t s) {
  if (!p) return DKV_ERR_INVALID_ARG;
  cudaStream_t st = (cudaStream_t)s;
  const int R = p->cfg.max_requests;
  cudaError_t e = cudaMemcpyAsync(p->h_ctrl, p->dev.ctrl, sizeof(Ctrl), cudaMemcpyDeviceToHost, st);
  if (e == cudaSuccess) e = cudaMemcpyAsync(p->h_req, p->dev.req_state, R, cudaMemcpyDeviceToHost, st);
  if (e == cudaSuccess) e = cudaMemcpyAsync(p->h_seq, p->dev.seq_len, 4 * (size_t)R, cudaMemcpyDeviceToHost, st);
  if (e == cudaSuccess) e = launch_clear_status(p->dev, st);
  if (e == cudaSuccess) e = cudaStreamSynchronize(st);
  if (e != cudaSuccess) return DKV_ERR_CUDA;
  Ctrl& c = *p->h_ctrl;
  if (c.status == DKV_OK) c.status = c.pending;         // an error classify found, not yet merged (Q36)
  if (out) {
    out->free_pages = c.free;
    out->used_pages = (int64_t)p->cfg.num_pages - c.free;
    out->start = c.start;
    out->last_demand = c.last_demand;
    out->last_freed = c.last_freed;
    out->status = c.status;
    out->oom_count = c.oom_count;
  }
  for (int r = 0; r < R; r++) { p->req_state[r] = p->h_req[r]; p->seq_len[r] = p->h_seq[r]; }
  if (c.status != DKV_OK) {
    p->recovering = true;
    // an interrupted sequence may be resumed (re-issue dkv_compact_alloc) or abandoned
    if (p->seq == SEQ_COMPACTED) p->seq = SEQ_CLASSIFIED;
  }
  return c.status;
}

int64_t* dkv_pool_stats_device_ptr(dkv_pool_t p) { return p ? p->dev.stats : nullptr; }

// ---- the whole decode step from host buffers (the e2e path; include/dkv.h)
static size_t stage_align(size_t x) { return (x + 255) & ~(size_t)255; }

size_t dkv_decode_stage_bytes(dkv_pool_t p) {
  if (!p) return 0;
  const size_t U = (size_t)p->G.U;
  return stage_align(U * sizeof(dkv_decision_t)) + stage_align(U * 4) + 2 * U * (size_t)p->cfg.head_dim * 2;
}

dkv_status_t dkv_decode_step_host(dkv_pool_t p, const float* h_sig, const uint16_t* h_kv, dkv_decision_t* h_dec,
                                  void* d_stage, size_t stage_bytes, dkv_stream_t st) {
  if (!p || !h_kv || !d_stage || stage_bytes < dkv_decode_stage_bytes(p)) return DKV_ERR_INVALID_ARG;
  // every host-detectable error before anything is queued (dkv.h: such errors enqueue nothing)
  int max_len = 0;
  const dkv_status_t pre = decode_precheck(p, &max_len);
  if (pre != DKV_OK) return pre;
  cudaStream_t s = (cudaStream_t)st;
  if (!p->copy_stream) {                                 // created all-or-nothing on first use
    cudaStream_t cs = nullptr;
    cudaEvent_t e0 = nullptr, e1 = nullptr;
    if (cudaStreamCreateWithFlags(&cs, cudaStreamNonBlocking) != cudaSuccess ||
        cudaEventCreateWithFlags(&e0, cudaEventDisableTiming) != cudaSuccess ||
        cudaEventCreateWithFlags(&e1, cudaEventDisableTiming) != cudaSuccess) {
      if (cs) cudaStreamDestroy(cs);
      if (e0) cudaEventDestroy(e0);
      if (e1) cudaEventDestroy(e1);
      return DKV_ERR_CUDA;
    }
    p->copy_stream = cs; p->ev_ready = e0; p->ev_kv = e1;
  }
  const size_t U = (size_t)p->G.U, d = (size_t)p->cfg.head_dim;
  uint8_t* b = (uint8_t*)d_stage;
  dkv_decision_t* d_dec = (dkv_decision_t*)b;
  float* d_sig = h_sig ? (float*)(b + stage_align(U * sizeof(dkv_decision_t))) : nullptr;
  uint16_t* d_kv = (uint16_t*)(b + stage_align(U * sizeof(dkv_decision_t)) + stage_align(U * 4));
  // the significance (U floats) first on s; the K/V copy (2·U·d halves, one transfer) on the copy stream,
  // ordered after everything already on s (the previous step's quant_write still reads the staging) and
  // overlapping classify + compact_alloc, which do not read it.  Measured (profiles/r1l_e2e_chunks.log):
  // splitting it into unit chunks that overlap quant_write is slower (2 / 4 / 8 chunks: 221 / 244 / 278 us
  // vs 220 us at the Llama-3-8B config), so it is one copy.
  if (h_sig && cudaMemcpyAsync(d_sig, h_sig, U * 4, cudaMemcpyHostToDevice, s) != cudaSuccess) return DKV_ERR_CUDA;
  if (cudaEventRecord(p->ev_ready, s) != cudaSuccess || cudaStreamWaitEvent(p->copy_stream, p->ev_ready, 0) != cudaSuccess)
    return DKV_ERR_CUDA;
  const cudaError_t ce = cudaMemcpyAsync(d_kv, h_kv, 2 * U * d * 2, cudaMemcpyHostToDevice, p->copy_stream);
  if (cudaEventRecord(p->ev_kv, p->copy_stream) != cudaSuccess) return DKV_ERR_CUDA;
  if (ce != cudaSuccess) {
    cudaStreamWaitEvent(s, p->ev_kv, 0);
    return DKV_ERR_CUDA;
  }
  dkv_status_t r = dkv_classify(p, DKV_PHASE_DECODE, nullptr, nullptr, 0, d_sig, 0, d_dec, nullptr, st);
  if (r == DKV_OK) r = dkv_compact_alloc(p, d_dec, st);
  // s waits for the copy on every path from here, so later writes to the staging stay ordered after it
  if (cudaStreamWaitEvent(s, p->ev_kv, 0) != cudaSuccess) return DKV_ERR_CUDA;
  if (r == DKV_OK) r = dkv_quant_write(p, DKV_PHASE_DECODE, d_dec, d_kv, d_kv + U * d, 0, d_sig, 0, st);
  if (r != DKV_OK) return r;
  if (h_dec && cudaMemcpyAsync(h_dec, d_dec, U * sizeof(dkv_decision_t), cudaMemcpyDeviceToHost, s) != cudaSuccess)
    return DKV_ERR_CUDA;
  return DKV_OK;
}

// ---- the decode step as a CUDA graph (dkv.h: dkv_decode_graph_*)
struct dkv_graph {
  dkv_pool* pool;
  int32_t steps, flags;
  cudaStream_t cap;                  // capture stream (library-owned)
  cudaGraph_t graph;
  cudaGraphExec_t exec;
  std::vector<cudaEvent_t> ev;       // DKV_GRAPH_EVENTS: [steps][4] boundaries of classify / compact / quant
};

dkv_status_t dkv_decode_graph_destroy(dkv_graph_t g) {
  if (!g) return DKV_ERR_INVALID_ARG;
  if (g->exec) cudaGraphExecDestroy(g->exec);
  if (g->graph) cudaGraphDestroy(g->graph);
  if (g->cap) cudaStreamDestroy(g->cap);
  for (cudaEvent_t e : g->ev)
    if (e) cudaEventDestroy(e);
  delete g;
  return DKV_OK;
}

dkv_status_t dkv_decode_graph_create(dkv_pool_t p, int32_t steps, const float* d_sig, int64_t sig_step,
                                     const uint16_t* d_k, const uint16_t* d_v, int64_t kv_step, dkv_decision_t* d_dec,
                                     int32_t flags, dkv_graph_t* out) {
  if (!out) return DKV_ERR_INVALID_ARG;
  *out = nullptr;
  if (!p || steps < 1 || !d_k || !d_v || !d_dec || sig_step < 0 || kv_step < 0 || (flags & ~3)) return DKV_ERR_INVALID_ARG;
  if (p->seq != SEQ_IDLE) return DKV_ERR_STATE;
  dkv_graph* g = new dkv_graph();
  g->pool = p; g->steps = steps; g->flags = flags;
  g->cap = nullptr; g->graph = nullptr; g->exec = nullptr;
  const bool events = (flags & DKV_GRAPH_EVENTS) != 0;
  PoolDev d = p->dev;
  d.pdl = ((flags & DKV_GRAPH_PDL) && !events) ? 1 : 0;    // event nodes between kernels would break the PDL edges
  if (cudaStreamCreateWithFlags(&g->cap, cudaStreamNonBlocking) != cudaSuccess) {
    dkv_decode_graph_destroy(g);
    return DKV_ERR_CUDA;
  }
  if (events) {
    g->ev.assign((size_t)steps * 4, nullptr);
    for (cudaEvent_t& e : g->ev)
      if (cudaEventCreate(&e) != cudaSuccess) { dkv_decode_graph_destroy(g); return DKV_ERR_CUDA; }
  }
  const size_t U = (size_t)p->G.U, D = (size_t)p->cfg.head_dim;
  // the classify instantiation cannot follow the longest active request inside a graph: it follows max_seq_len
  const int max_len = p->cfg.max_seq_len;
  cudaError_t e = cudaStreamBeginCapture(g->cap, cudaStreamCaptureModeThreadLocal);
  for (int32_t t = 0; t < steps && e == cudaSuccess; t++) {
    const float* sig = d_sig ? d_sig + (size_t)t * (size_t)sig_step : nullptr;
    const uint16_t* k = d_k + (size_t)t * (size_t)kv_step;
    const uint16_t* v = d_v + (size_t)t * (size_t)kv_step;
    cudaEvent_t* ev = events ? &g->ev[4 * (size_t)t] : nullptr;
    if (ev) e = cudaEventRecordWithFlags(ev[0], g->cap, cudaEventRecordExternal);
    if (e == cudaSuccess) e = launch_classify_decode(d, sig, d_dec, max_len, g->cap);
    if (e == cudaSuccess && ev) e = cudaEventRecordWithFlags(ev[1], g->cap, cudaEventRecordExternal);
    if (e == cudaSuccess) e = launch_compact_alloc(d, d_dec, DKV_PHASE_DECODE, g->cap, true, true);
    if (e == cudaSuccess && ev) e = cudaEventRecordWithFlags(ev[2], g->cap, cudaEventRecordExternal);
    if (e == cudaSuccess) e = launch_quant_decode(d, d_dec, k, v, sig, g->cap);
    if (e == cudaSuccess && ev) e = cudaEventRecordWithFlags(ev[3], g->cap, cudaEventRecordExternal);
  }
  const cudaError_t e2 = cudaStreamEndCapture(g->cap, &g->graph);
  if (e == cudaSuccess) e = e2;
  if (e == cudaSuccess) e = cudaGraphInstantiate(&g->exec, g->graph, 0);
  (void)U; (void)D;
  if (e != cudaSuccess) {
    cudaGetLastError();
    dkv_decode_graph_destroy(g);
    return DKV_ERR_CUDA;
  }
  *out = g;
  return DKV_OK;
}

dkv_status_t dkv_decode_graph_launch(dkv_graph_t g, dkv_stream_t s) {
  if (!g) return DKV_ERR_INVALID_ARG;
  dkv_pool* p = g->pool;
  if (p->seq != SEQ_IDLE) return DKV_ERR_STATE;
  // every step's dkv_classify needs the ACTIVE requests below max_seq_len
  for (int r = 0; r < p->cfg.max_requests; r++)
    if (p->req_state[r] == DKV_REQ_ACTIVE && p->seq_len[r] + g->steps > p->cfg.max_seq_len) return DKV_ERR_STATE;
  if (cudaGraphLaunch(g->exec, (cudaStream_t)s) != cudaSuccess) return DKV_ERR_CUDA;
  // the host mirror after `steps` decode steps: the first step recycles the freed requests
  for (int r = 0; r < p->cfg.max_requests; r++) {
    if (p->req_state[r] == DKV_REQ_PENDING_FREE) { p->req_state[r] = DKV_REQ_IDLE; p->seq_len[r] = 0; }
    else if (p->req_state[r] == DKV_REQ_ACTIVE) p->seq_len[r] += g->steps;
  }
  p->phase = DKV_PHASE_DECODE;
  p->recovering = false;
  return DKV_OK;
}

dkv_status_t dkv_decode_graph_kernel_ms(dkv_graph_t g, float* h_ms) {
  if (!g || !h_ms || !(g->flags & DKV_GRAPH_EVENTS)) return DKV_ERR_INVALID_ARG;
  for (int32_t t = 0; t < g->steps; t++)
    for (int k = 0; k < 3; k++)
      if (cudaEventElapsedTime(&h_ms[3 * (size_t)t + k], g->ev[4 * (size_t)t + k], g->ev[4 * (size_t)t + k + 1]) !=
          cudaSuccess)
        return DKV_ERR_CUDA;
  return DKV_OK;
}

}  // extern "C"
