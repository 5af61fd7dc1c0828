// k_bulk.cu — the KV compressor's prompt path (a8): the HBM-bound bulk writer behind
// dkv_quant_write(PREFILL).
//
// One warp per (admitted unit, 256-token segment); the segment's exclusive (high, low) ranks come from
// classify_prefill's checkpoints, so segments are independent and the grid load-balances.
//  phase A  re-classifies 32 tokens per step (§4 thresholds) and ranks them with ballot/popc into
//           two per-warp shared-memory lists (high from the front, low from the back);
//  phase B  walks each list with the class's bit widths as template parameters (K8V4 / K4V2 specialised,
//           others through the runtime-width quantizer): only the kept K/V rows are read (pruned rows never
//           are), 4 lanes per token, 8 tokens per warp step, lane q holding 16-B chunks q, q+4, ... so each
//           warp-wide load covers 64 contiguous bytes per token; the next step's rows are loaded while the
//           current step is quantized, then stored as token-major code rows + metadata + score + position;
//  phase C  copies the newest W tokens into the FP16 window.
#include <stdlib.h>

#include "dkv_internal.cuh"

namespace dkv {

#ifndef DKV_BULK_WARPS
#define DKV_BULK_WARPS 4
#endif
constexpr int kBulkWarps = DKV_BULK_WARPS;               // warps (segments) per CTA
constexpr int kBulkG = 4;                                // lanes per token
constexpr int kBulkTPS = 32 / kBulkG;                    // tokens per warp step

__device__ __forceinline__ int prompt_class_q(float ah, float al, int prompt_den, float s, int t, int T, int top = 0,
                                              float at = 0.0f) {
  const float den = (prompt_den == 0) ? (float)(t + 1) : (float)T;
  const float th = __fdiv_rn(ah, den), tl = __fdiv_rn(al, den);
  if (top && s >= __fdiv_rn(at, den)) return DKV_CLS_TOP;       // NEXT-4 (Q38): written by quant_prefill_top_kernel
  return s >= th ? DKV_CLS_HIGH : (s >= tl ? DKV_CLS_LOW : DKV_CLS_PRUNED);
}

template <int NCH>
__device__ __forceinline__ void load_rows(const uint16_t* kbase, const uint16_t* vbase, int t, int q, bool valid,
                                          uint32_t (&xk)[NCH][4], uint32_t (&xv)[NCH][4]) {
  constexpr int D = NCH * 32;
  const uint4* ks = reinterpret_cast<const uint4*>(kbase + (size_t)t * D);
  const uint4* vs = reinterpret_cast<const uint4*>(vbase + (size_t)t * D);
#pragma unroll
  for (int c = 0; c < NCH; c++) {
    uint4 a = make_uint4(0, 0, 0, 0), b = a;
    if (valid) { a = ld_stream_v4(ks + q + kBulkG * c); b = ld_stream_v4(vs + q + kBulkG * c); }
    xk[c][0] = a.x; xk[c][1] = a.y; xk[c][2] = a.z; xk[c][3] = a.w;
    xv[c][0] = b.x; xv[c][1] = b.y; xv[c][2] = b.z; xv[c][3] = b.w;
  }
}

struct ListCtx {
  const uint16_t* kbase;
  const uint16_t* vbase;
  const uint32_t* ent;       // this warp's list entries: (t - t0) | slot << 8
  const uint32_t* sig;       // matching canonical score bits
  const int32_t* row;        // this unit's table row
  int t0, cnt, front;        // front: list grows from index 0 upward (high) or from the back downward (low)
  int cls, L, page_bytes;
  uint8_t* pages;
  uint4* ring;               // PF == 2: this warp's TMA staging ring [kBulkStages][TPS][2][D/8] x 16 B
  uint64_t* bar;             // PF == 2: one mbarrier per stage
  uint32_t* phase;           // PF == 2: parity bit per stage (warp-uniform)
};

#ifndef DKV_BULK_STAGES
#define DKV_BULK_STAGES 2
#endif
#ifndef DKV_BULK_MINB
#define DKV_BULK_MINB 2   // the register cap ptxas schedules against (128 registers used either way): 2 measured
                          // best, 6.30-6.35 ms vs 6.54-6.57 at 4 (profiles/r2z_bulk_minb_sweep.log)
#endif
constexpr int kBulkStages = DKV_BULK_STAGES;               // staging depth (tuning: tools/sweep_bulk.sh)

// Walk one class list.  KB/VB > 0: compile-time widths; KB == 0: runtime widths from g.
// PF: 0 = rows loaded into registers right before use; 1 = register ping-pong; 2 = 1-D TMA
// (cp.async.bulk) ring of kBulkStages steps in shared memory, completion tracked by mbarrier transactions.
template <int D, int KB, int VB, int PF>
__device__ __forceinline__ void bulk_list(const ListCtx& c, const ClassGeom& g, int lane, bool& bad) {
  constexpr int NCH = D / 32;
  const int grp = lane / kBulkG, q = lane % kBulkG;
  const unsigned gmask = 0xFu << (grp * kBulkG);
  const int C = g.C;
  const bool pow2 = (C & (C - 1)) == 0;
  const int csh = __popc(C - 1);
  const int nsteps = (c.cnt + kBulkTPS - 1) / kBulkTPS;
  auto ix_of = [&](int e) { return c.front ? e : kSegTokens - 1 - e; };
  // one step: quantize the rows in (xk, xv) for list entry e, store codes / metadata / score / position
  auto step = [&](int e, uint32_t (&xk)[NCH][4], uint32_t (&xv)[NCH][4]) {
    const bool valid = e < c.cnt;
    const int ix = ix_of(e);
    const uint32_t ent = valid ? c.ent[ix] : 0u;
    const int slot = (int)(ent >> 8);
    const int k = pow2 ? (slot >> csh) : slot / C;
    const int idx = pow2 ? (slot & (C - 1)) : slot % C;
    const int pid = valid ? __ldg(c.row + (c.cls == DKV_CLS_HIGH ? k : c.L - 1 - k)) : 0;
    uint8_t* pg = c.pages + (size_t)pid * (size_t)c.page_bytes;
    uint32_t mk, mv;
    bool tok_ok;
    uint8_t* krow = pg + g.off_k + idx * g.k_row;
    uint8_t* vrow = pg + g.off_v + idx * g.v_row;
    if constexpr (KB > 0) {
      // statistics of both vectors first, so a token is validated whole before any store (Q30)
      const QStats sk = qstats_h16_ct<kBulkG, NCH, KB>(xk, gmask);
      const QStats sv = qstats_h16_ct<kBulkG, NCH, VB>(xv, gmask);
      mk = sk.meta; mv = sv.meta;
      tok_ok = sk.ok && sv.ok;
      uint2 pk[NCH];
      qencode_h16_ct<NCH, KB>(xk, sk, pk);
      if (valid && tok_ok) {
#pragma unroll
        for (int a = 0; a < NCH; a++) store_chunk_codes_ct<KB>(krow, q + kBulkG * a, pk[a]);
      }
      qencode_h16_ct<NCH, VB>(xv, sv, pk);
      if (valid && tok_ok) {
#pragma unroll
        for (int a = 0; a < NCH; a++) store_chunk_codes_ct<VB>(vrow, q + kBulkG * a, pk[a]);
      }
    } else {
      uint2 pkk[NCH], pkv[NCH];
      bool fk, fv;
      quant_chunks_h16<kBulkG, NCH>(xk, g.kbits, gmask, pkk, mk, fk);
      quant_chunks_h16<kBulkG, NCH>(xv, g.vbits, gmask, pkv, mv, fv);
      tok_ok = fk && fv;
      if (valid && tok_ok) {
#pragma unroll
        for (int a = 0; a < NCH; a++) {
          store_chunk_codes(krow, q + kBulkG * a, g.kbits, pkk[a]);
          store_chunk_codes(vrow, q + kBulkG * a, g.vbits, pkv[a]);
        }
      }
    }
    if (valid) bad |= !tok_ok;
    if (valid && tok_ok) {                               // Q30: a non-finite token is rejected whole
      uint32_t* w32 = nullptr;
      uint32_t val = 0;
      if (q == 0) { w32 = reinterpret_cast<uint32_t*>(pg + g.off_kmeta) + idx; val = mk; }
      if (q == 1) { w32 = reinterpret_cast<uint32_t*>(pg + g.off_vmeta) + idx; val = mv; }
      if (q == 2) { w32 = reinterpret_cast<uint32_t*>(pg + g.off_score) + idx; val = c.sig[ix]; }
      if (q == 3) { w32 = reinterpret_cast<uint32_t*>(pg + g.off_pos) + idx; val = (uint32_t)(c.t0 + (int)(ent & 255u)); }
      *w32 = val;
    }
  };
  auto load = [&](int e, uint32_t (&xk)[NCH][4], uint32_t (&xv)[NCH][4]) {
    const bool v = e < c.cnt;
    load_rows<NCH>(c.kbase, c.vbase, c.t0 + (int)((v ? c.ent[ix_of(e)] : 0u) & 255u), q, v, xk, xv);
  };
  if constexpr (PF == 0) {
#pragma unroll 1
    for (int st = 0; st < nsteps; st++) {
      uint32_t xk[NCH][4], xv[NCH][4];
      load(st * kBulkTPS + grp, xk, xv);
      step(st * kBulkTPS + grp, xk, xv);
    }
  } else if constexpr (PF == 3) {
    // per-lane cp.async staging ring in shared memory: each lane copies and later reads back only its own
    // chunks (q + 4a of token grp's K and V rows), so per-thread cp.async.wait_group is the only sync
    // needed; in-flight rows cost no registers.
    // slot (stage, a, lane) at ring[(stage * 2NCH + a) * 32 + lane]: lane-consecutive 16-B words, so the
    // read-back LDS.128 is bank-conflict free
    uint4* myring = c.ring + lane;
    auto issue = [&](int st) {
      const int e = st * kBulkTPS + grp;
      const bool v = e < c.cnt;
      const int t = c.t0 + (int)((v ? c.ent[ix_of(e)] : 0u) & 255u);
      const uint4* ks = reinterpret_cast<const uint4*>(c.kbase + (size_t)t * D);
      const uint4* vs = reinterpret_cast<const uint4*>(c.vbase + (size_t)t * D);
      uint4* dst = myring + (size_t)(st % kBulkStages) * 2 * NCH * 32;
#pragma unroll
      for (int a = 0; a < NCH; a++) {
        cp_async16(dst + a * 32, ks + q + kBulkG * a, v);
        cp_async16(dst + (NCH + a) * 32, vs + q + kBulkG * a, v);
      }
    };
#pragma unroll
    for (int st = 0; st < kBulkStages - 1; st++) {
      if (st < nsteps) issue(st);
      cp_async_commit();
    }
#pragma unroll 1
    for (int st = 0; st < nsteps; st++) {
      if (st + kBulkStages - 1 < nsteps) issue(st + kBulkStages - 1);
      cp_async_commit();
      cp_async_wait<kBulkStages - 1>();
      const uint4* src = myring + (size_t)(st % kBulkStages) * 2 * NCH * 32;
      uint32_t xk[NCH][4], xv[NCH][4];
#pragma unroll
      for (int a = 0; a < NCH; a++) {
        const uint4 x = src[a * 32], y = src[(NCH + a) * 32];
        xk[a][0] = x.x; xk[a][1] = x.y; xk[a][2] = x.z; xk[a][3] = x.w;
        xv[a][0] = y.x; xv[a][1] = y.y; xv[a][2] = y.z; xv[a][3] = y.w;
      }
      step(st * kBulkTPS + grp, xk, xv);
    }
    cp_async_wait<0>();
  } else if constexpr (PF == 2) {
    // lanes 0 .. 2*TPS-1 each move one 2*D-byte row (token lane/2, K if lane even else V) per step
    constexpr int ROWB = D * 2;
    auto issue = [&](int st, int s) {
      const int nv = min(kBulkTPS, c.cnt - st * kBulkTPS);
      fence_proxy_async_smem();                          // earlier generic reads of this stage come first
      if (lane == 0) mbar_arrive_expect_tx(&c.bar[s], (uint32_t)(nv * 2 * ROWB));
      __syncwarp();
      const int tok = lane >> 1;
      if (lane < 2 * kBulkTPS && tok < nv) {
        const int t = c.t0 + (int)(c.ent[ix_of(st * kBulkTPS + tok)] & 255u);
        const uint16_t* src = ((lane & 1) ? c.vbase : c.kbase) + (size_t)t * D;
        bulk_g2s(c.ring + ((size_t)(s * kBulkTPS + tok) * 2 + (lane & 1)) * (D / 8), src, ROWB, &c.bar[s]);
      }
    };
#pragma unroll 1
    for (int st = 0; st < min(nsteps, kBulkStages); st++) issue(st, st);
#pragma unroll 1
    for (int st = 0; st < nsteps; st++) {
      const int s = st % kBulkStages;
      mbar_wait(&c.bar[s], (*c.phase >> s) & 1u);
      *c.phase ^= 1u << s;
      uint32_t xk[NCH][4], xv[NCH][4];
      const uint4* rk = c.ring + ((size_t)(s * kBulkTPS + grp) * 2) * (D / 8);
      const uint4* rv = rk + D / 8;
#pragma unroll
      for (int a = 0; a < NCH; a++) {
        const uint4 x = rk[q + kBulkG * a], y = rv[q + kBulkG * a];
        xk[a][0] = x.x; xk[a][1] = x.y; xk[a][2] = x.z; xk[a][3] = x.w;
        xv[a][0] = y.x; xv[a][1] = y.y; xv[a][2] = y.z; xv[a][3] = y.w;
      }
      __syncwarp();
      if (st + kBulkStages < nsteps) issue(st + kBulkStages, s);
      step(st * kBulkTPS + grp, xk, xv);
    }
  } else {                                               // ping-pong buffers: load step s+1 while quantizing s
    uint32_t ak[NCH][4], av[NCH][4], bk[NCH][4], bv[NCH][4];
    load(grp, ak, av);
#pragma unroll 1
    for (int st = 0; st < nsteps; st += 2) {
      if (st + 1 < nsteps) load((st + 1) * kBulkTPS + grp, bk, bv);
      step(st * kBulkTPS + grp, ak, av);
      if (st + 1 >= nsteps) break;
      if (st + 2 < nsteps) load((st + 2) * kBulkTPS + grp, ak, av);
      step((st + 1) * kBulkTPS + grp, bk, bv);
    }
  }
}

template <int D, int PF>
__device__ __forceinline__ void bulk_dispatch(const ListCtx& c, const ClassGeom& g, int lane, bool& bad) {
  if (g.kbits == 8 && g.vbits == 4) bulk_list<D, 8, 4, PF>(c, g, lane, bad);
  else if (g.kbits == 4 && g.vbits == 2) bulk_list<D, 4, 2, PF>(c, g, lane, bad);
  else bulk_list<D, 0, 0, PF>(c, g, lane, bad);
}

template <int D>
constexpr size_t bulk_ring_bytes() { return (size_t)kBulkWarps * kBulkStages * kBulkTPS * 2 * D * 2; }

template <int D, int PF>
__global__ void __launch_bounds__(kBulkWarps * 32, PF == 1 ? 4 : (PF >= 2 ? DKV_BULK_MINB : 6))
quant_prefill_kernel(PoolDev p, int n, const uint16_t* __restrict__ kin, const uint16_t* __restrict__ vin,
                     int64_t kv_stride, const float* __restrict__ sig, int64_t sig_stride, int nseg_max) {
  __shared__ uint32_t s_ent[kBulkWarps][kSegTokens];   // (t - t0) | slot << 8; high from the front, low from the back
  __shared__ uint32_t s_sig[kBulkWarps][kSegTokens];
  __shared__ __align__(8) uint64_t s_bar[kBulkWarps][kBulkStages];
  __shared__ uint32_t s_phase[kBulkWarps];
  extern __shared__ __align__(128) uint4 s_ring[];      // PF == 2 only
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  if constexpr (PF == 2) {
    if (lane == 0) {
      for (int s = 0; s < kBulkStages; s++) mbar_init(&s_bar[warp][s], 1);
      s_phase[warp] = 0;
      fence_mbar_init();
    }
    __syncwarp();
  }
  const long item = (long)blockIdx.x * kBulkWarps + warp;
  const int seg = (int)(item % nseg_max);
  const long wi = item / nseg_max;                     // admitted unit index (i * LyH + j)
  if (wi >= (long)n * p.LyH) return;
  // the segment's 256 scores, all in flight at once before anything else (phase A used to wait for them one
  // 32-token step at a time: eight dependent round trips before the first K/V row was requested); indices up
  // to sig_stride are inside the caller's array (sig_stride >= the longest prompt), those >= T go unused
  const float* srow = sig + wi * sig_stride;
  constexpr int kSigPerLane = kSegTokens / 32;
  float sv[kSigPerLane];
#pragma unroll
  for (int k = 0; k < kSigPerLane; k++) {
    const long t = (long)seg * kSegTokens + 32 * k + lane;
    sv[k] = t < sig_stride ? __ldcs(srow + t) : 0.0f;
  }
  // the entry status, the admitted request and everything indexed by it in two round trips: the status is
  // checked only once they are in flight (a request index from an errored call is clamped, never used)
  const int entry_status = ld_volatile(&p.ctrl->qw_status);   // Q36, left by dkv_compact_alloc
  const int i = (int)(wi / p.LyH), j = (int)(wi % p.LyH);
  const int r = min(max(p.admit[i], 0), p.R - 1);
  const int u = r * p.LyH + j;
  const float ah = unit_alpha_h(p, u), al = unit_alpha_l(p, u);  // Q35
  const int T = p.prompt_len[r];
  int hr = p.pf_seg[((size_t)u * p.nseg + seg) * 2];    // seg < nseg_max <= nseg
  int lr = p.pf_seg[((size_t)u * p.nseg + seg) * 2 + 1];
  if (entry_status != 0) return;
  const int t0 = seg * kSegTokens;
  if (t0 >= T) return;
  const int t1 = min(t0 + kSegTokens, T);
  const int kept = max(T - p.W, 0);
  const int ke = min(t1, kept);
  const uint16_t* kbase = kin + wi * kv_stride * D;
  const uint16_t* vbase = vin + wi * kv_stride * D;

  // phase A: classes + per-class ranks (warp ballot/popc + running offsets) -> two kept lists
  int nh = 0, nl = 0;
  const unsigned lt = (1u << lane) - 1u;
#pragma unroll
  for (int k = 0; k < kSigPerLane; k++) {
    const int c = t0 + 32 * k;
    if (c >= ke) break;                                  // warp-uniform
    const int t = c + lane;
    int cl = DKV_CLS_NONE;
    float s = 0.0f;
    if (t < ke) {
      s = canon_zero(sv[k]);
      cl = prompt_class_q(ah, al, p.prompt_den, s, t, T, p.top, p.alpha_t);
    }
    const unsigned hm = __ballot_sync(kFull, cl == DKV_CLS_HIGH);
    const unsigned lm = __ballot_sync(kFull, cl == DKV_CLS_LOW);
    if (cl == DKV_CLS_HIGH) {
      const int e = nh + __popc(hm & lt);
      s_ent[warp][e] = (uint32_t)(t - t0) | ((uint32_t)(hr + __popc(hm & lt)) << 8);
      s_sig[warp][e] = __float_as_uint(s);
    } else if (cl == DKV_CLS_LOW) {
      const int e = kSegTokens - 1 - (nl + __popc(lm & lt));
      s_ent[warp][e] = (uint32_t)(t - t0) | ((uint32_t)(lr + __popc(lm & lt)) << 8);
      s_sig[warp][e] = __float_as_uint(s);
    }
    hr += __popc(hm); nh += __popc(hm);
    lr += __popc(lm); nl += __popc(lm);
  }
  __syncwarp();

  // phase B
  bool bad = false;
  ListCtx c;
  c.kbase = kbase; c.vbase = vbase; c.ent = s_ent[warp]; c.sig = s_sig[warp];
  c.row = p.table + (size_t)u * p.L; c.t0 = t0; c.L = p.L; c.page_bytes = p.page_bytes; c.pages = p.pages;
  c.ring = s_ring + (size_t)warp * kBulkStages * kBulkTPS * 2 * (D / 8);
  c.bar = s_bar[warp];
  c.phase = &s_phase[warp];
  c.cnt = nh; c.front = 1; c.cls = DKV_CLS_HIGH;
  if (nh > 0) bulk_dispatch<D, PF>(c, geom_of(p, DKV_CLS_HIGH), lane, bad);
  c.cnt = nl; c.front = 0; c.cls = DKV_CLS_LOW;
  if (nl > 0) bulk_dispatch<D, PF>(c, geom_of(p, DKV_CLS_LOW), lane, bad);

  // phase C: the newest min(W, T) tokens -> FP16 window slot t mod W (Q10)
  {
    constexpr int LPT = D / 8;                         // lanes per row (16-B chunks)
    constexpr int RPS = 32 / LPT;                      // rows per step
    const int rr = lane / LPT, cc = lane % LPT;
    for (int t = max(t0, kept) + rr; t < t1; t += RPS) {
      const uint4 a = ld_stream_v4(kbase + (size_t)t * D + cc * 8);
      const uint4 b = ld_stream_v4(vbase + (size_t)t * D + cc * 8);
      const size_t w = ((size_t)u * p.W + (t % p.W)) * D + cc * 8;
      *reinterpret_cast<uint4*>(p.win_k + w) = a;
      *reinterpret_cast<uint4*>(p.win_v + w) = b;
      if (cc == 0) p.win_sig[(size_t)u * p.W + (t % p.W)] = canon_zero(__ldg(srow + t));   // P:360, Q33
    }
  }
  if (seg == 0 && lane == 0) p.secmin[8 * (size_t)u + 6] = 0;   // no dkv_attend minima for a new prompt
  if (__any_sync(kFull, bad) && lane == 0) set_status(p.ctrl, DKV_ERR_NONFINITE);
}

// ADMITTING -> ACTIVE once every prompt token is written.  With an error at entry (Q36/Q37: the admission's
// planning or allocation failed, so it holds no pages) the admission is rolled back: ADMITTING -> IDLE.  A
// token rejected by this call (Q30) does not stop the others; the request becomes ACTIVE and can be freed.
__global__ void finish_prefill_kernel(PoolDev p, int n) {
  const bool rollback = ld_volatile(&p.ctrl->qw_status) != 0;
  for (int i = threadIdx.x; i < n; i += blockDim.x) {
    const int r = p.admit[i];
    if (p.req_state[r] != DKV_REQ_ADMITTING) continue;
    if (rollback) { p.req_state[r] = DKV_REQ_IDLE; p.seq_len[r] = 0; p.prompt_len[r] = 0; }
    else p.req_state[r] = DKV_REQ_ACTIVE;
  }
}

#ifndef DKV_BULK_PF
#define DKV_BULK_PF 3
#endif

// NEXT-4 (Q40): the prompt's TOP tokens, kept as their fp16 K and V rows.  A warp per (admitted unit, 256-token
// segment) as in quant_prefill_kernel: ranks from classify_prefill's TOP checkpoints plus a ballot per 32 tokens,
// then one token at a time the whole warp copies its rows (K: lanes 0..15, V: 16..31 at d = 128) into TOP slot
// `rank` (page ttable[u][rank / Ct]) with its significance and position.  A token with a non-finite element is
// rejected whole (Q30).
template <int D>
__global__ void __launch_bounds__(kBulkWarps * 32)
quant_prefill_top_kernel(PoolDev p, int n, const uint16_t* __restrict__ kin, const uint16_t* __restrict__ vin,
                         int64_t kv_stride, const float* __restrict__ sig, int64_t sig_stride, int nseg_max) {
  constexpr int LPR = D / 8;                                     // lanes per row (16-B chunks)
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const long item = (long)blockIdx.x * kBulkWarps + warp;
  const int seg = (int)(item % nseg_max);
  const long wi = item / nseg_max;
  if (wi >= (long)n * p.LyH) return;
  if (ld_volatile(&p.ctrl->qw_status) != 0) return;             // entry status (Q36)
  const int i = (int)(wi / p.LyH), j = (int)(wi % p.LyH);
  const int r = p.admit[i];
  const int u = r * p.LyH + j;
  const float ah = unit_alpha_h(p, u), al = unit_alpha_l(p, u);
  const int T = p.prompt_len[r];
  const int t0 = seg * kSegTokens;
  const int kept = max(T - p.W, 0);
  const int ke = min(t0 + kSegTokens, kept);
  if (t0 >= ke) return;
  const float* srow = sig + wi * sig_stride;
  const uint16_t* kbase = kin + wi * kv_stride * D;
  const uint16_t* vbase = vin + wi * kv_stride * D;
  int rank = p.pf_seg_t[(size_t)u * p.nseg + seg];
  const ClassGeom gt = p.gt;
  bool bad = false;
  for (int c = t0; c < ke; c += 32) {
    const int t = c + lane;
    float s = 0.0f;
    int cl = DKV_CLS_NONE;
    if (t < ke) {
      s = canon_zero(__ldg(srow + t));
      cl = prompt_class_q(ah, al, p.prompt_den, s, t, T, 1, p.alpha_t);
    }
    unsigned m = __ballot_sync(kFull, cl == DKV_CLS_TOP);
    while (m) {
      const int src = __ffs(m) - 1;
      m &= m - 1;
      const int tt = c + src;
      const float st = __shfl_sync(kFull, s, src);
      const int slot = rank++;
      const int pg = fdiv(p.div_Ct, slot), idx = slot - pg * p.Ct;
      uint8_t* page = p.pages + (size_t)p.ttable[(size_t)u * p.Lt + pg] * (size_t)p.page_bytes;
      uint4 x = make_uint4(0u, 0u, 0u, 0u);
      const bool isk = lane < LPR;
      if (lane < 2 * LPR) x = ld_stream_v4((isk ? kbase : vbase) + (size_t)tt * D + 8 * (isk ? lane : lane - LPR));
      const uint32_t w4[4] = {x.x, x.y, x.z, x.w};
      bool fin = true;
#pragma unroll
      for (int e = 0; e < 4; e++)
        fin &= ((w4[e] & 0x7C00u) != 0x7C00u) && ((w4[e] & 0x7C000000u) != 0x7C000000u);
      if (__any_sync(kFull, !fin)) { bad = true; continue; }       // Q30: nothing of the token is stored
      if (lane < 2 * LPR)
        *reinterpret_cast<uint4*>(page + (isk ? gt.off_k + idx * gt.k_row + 16 * lane
                                              : gt.off_v + idx * gt.v_row + 16 * (lane - LPR))) = x;
      if (lane == 0) {
        *reinterpret_cast<float*>(page + gt.off_score + 4 * idx) = st;
        *reinterpret_cast<int32_t*>(page + gt.off_pos + 4 * idx) = tt;
      }
    }
  }
  if (bad && lane == 0) set_status(p.ctrl, DKV_ERR_NONFINITE);
}

cudaError_t launch_quant_prefill(const PoolDev& p, int n, const uint16_t* k, const uint16_t* v, int64_t kv_stride,
                                 const float* sig, int64_t sig_stride, int max_len, cudaStream_t s) {
  const int nseg_max = (max_len + kSegTokens - 1) / kSegTokens;
  const long items = (long)n * p.LyH * nseg_max;
  if (items > 0) {
    const long grid = (items + kBulkWarps - 1) / kBulkWarps;
    constexpr int pf = DKV_BULK_PF;                   // staging form (build-time choice; 3 measured best)
    if (p.d == 128) {
      if (pf == 2 || pf == 3) {
        constexpr size_t sm = bulk_ring_bytes<128>();
        static bool attr = false;
        if (!attr) {
          cudaError_t e = cudaFuncSetAttribute(quant_prefill_kernel<128, 2>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm);
          if (e == cudaSuccess)
            e = cudaFuncSetAttribute(quant_prefill_kernel<128, 3>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm);
          if (e != cudaSuccess) return e;
          attr = true;
        }
        if (pf == 2) quant_prefill_kernel<128, 2><<<(unsigned)grid, kBulkWarps * 32, sm, s>>>(p, n, k, v, kv_stride, sig, sig_stride, nseg_max);
        else quant_prefill_kernel<128, 3><<<(unsigned)grid, kBulkWarps * 32, sm, s>>>(p, n, k, v, kv_stride, sig, sig_stride, nseg_max);
      } else if (pf == 1) {
        quant_prefill_kernel<128, 1><<<(unsigned)grid, kBulkWarps * 32, 0, s>>>(p, n, k, v, kv_stride, sig, sig_stride, nseg_max);
      } else {
        quant_prefill_kernel<128, 0><<<(unsigned)grid, kBulkWarps * 32, 0, s>>>(p, n, k, v, kv_stride, sig, sig_stride, nseg_max);
      }
    } else {
      quant_prefill_kernel<64, 0><<<(unsigned)grid, kBulkWarps * 32, 0, s>>>(p, n, k, v, kv_stride, sig, sig_stride, nseg_max);
    }
    cudaError_t e = cudaGetLastError();
    if (e != cudaSuccess) return e;
  }
  if (p.top && items > 0) {
    const long grid = (items + kBulkWarps - 1) / kBulkWarps;
    if (p.d == 128) quant_prefill_top_kernel<128><<<(unsigned)grid, kBulkWarps * 32, 0, s>>>(p, n, k, v, kv_stride, sig, sig_stride, nseg_max);
    else quant_prefill_top_kernel<64><<<(unsigned)grid, kBulkWarps * 32, 0, s>>>(p, n, k, v, kv_stride, sig, sig_stride, nseg_max);
    cudaError_t e = cudaGetLastError();
    if (e != cudaSuccess) return e;
  }
  finish_prefill_kernel<<<1, 256, 0, s>>>(p, n);
  return cudaGetLastError();
}

}  // namespace dkv
