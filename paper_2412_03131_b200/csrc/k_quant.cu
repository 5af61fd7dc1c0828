// k_quant.cu — the KV compressor: quantize K/V into unified pages at K8V4 / K4V2.
//
//  quant_decode  : one warp per unit; lanes [0, G) own the key vector, [G, 2G) the value vector, 8 fp16
//                  elements (one 16-B vector) per lane, G = d/8.  Order per unit (Q8, Q9): downgrade the
//                  victim (read its K8V4 codes before t_c overwrites the slot, re-quantize at K4V2 into the
//                  KV_l tail), quantize t_c out of window slot (N-1) mod W, then push the new token into
//                  that same window slot.
//  quant_prefill : the HBM-bound bulk writer.  One warp per (admitted unit, 256-token segment); the
//                  segment's (high, low) ranks come from classify_prefill's checkpoints, so segments are
//                  independent.  Phase A classifies 32 tokens per step (ballot/popc ranks) into a per-warp
//                  shared-memory list of kept tokens; phase B streams only the kept rows (pruned rows are
//                  never read) with 128-bit evict-first loads, 32/G tokens per warp step, 4 steps in
//                  flight, quantizes in registers and stores token-major code rows, metadata, score and
//                  position; phase C copies the newest W tokens into the FP16 window.
#include "dkv_internal.cuh"

namespace dkv {

constexpr int kQWarps = 8;

template <int G>
__global__ void __launch_bounds__(kQWarps * 32)
quant_decode_kernel(PoolDev p, const dkv_decision_t* __restrict__ dec, const uint16_t* __restrict__ knew,
                    const uint16_t* __restrict__ vnew, const float* __restrict__ cand_sig) {
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int u = blockIdx.x * kQWarps + warp;
  if (u >= p.U) return;
  if (ld_volatile(&p.ctrl->status) != 0) return;
  const int r = u / p.LyH;
  if (p.req_state[r] != DKV_REQ_ACTIVE) return;
  const int N = p.seq_len[r];                       // already includes this step's token (compact_alloc)
  const int pc = N - 1 - p.W;
  const int4 dw = reinterpret_cast<const int4*>(dec)[u];
  const int tc_class = dw.x & 0xFF, v_action = (dw.x >> 8) & 0xFF;
  const int v_slot = dw.y, tc_slot = dw.z, v_dst = dw.w;
  const int grp = lane / G, gl = lane % G;          // grp 0 = key, 1 = value, >= 2 idle (d = 64)
  const bool kv = grp < 2;
  const int d = p.d;

  // 1. downgrade t_v: K8V4 -> K4V2 (Q9: re-quantize the dequantized stored values)
  if (v_action == DKV_V_DOWN) {
    const ClassGeom& gh = p.g[DKV_CLS_HIGH];
    const ClassGeom& go = p.g[DKV_CLS_LOW];
    int is, id;
    const uint8_t* src = slot_page(p, DKV_CLS_HIGH, u, v_slot, is);
    uint8_t* dst = slot_page(p, DKV_CLS_LOW, u, v_dst, id);
    const int sb = grp == 0 ? gh.kbits : gh.vbits;
    uint64_t packed = 0;
    uint32_t meta = 0;
    if (kv) {
      packed = load_codes(src + (grp == 0 ? gh.off_k + is * gh.k_row : gh.off_v + is * gh.v_row) + gl * sb, sb);
      meta = *reinterpret_cast<const uint32_t*>(src + (grp == 0 ? gh.off_kmeta : gh.off_vmeta) + 4 * is);
    }
    float x[8];
    dequant8(packed, kv ? sb : 8, meta, x);
    const int db = grp == 0 ? go.kbits : go.vbits;
    uint32_t m2;
    bool fin;
    const uint64_t q = quantize8<G>(x, kv ? db : 8, m2, fin);
    if (kv) {
      store_codes(dst + (grp == 0 ? go.off_k + id * go.k_row : go.off_v + id * go.v_row) + gl * db, q, db);
      if (gl == 0) *reinterpret_cast<uint32_t*>(dst + (grp == 0 ? go.off_kmeta : go.off_vmeta) + 4 * id) = m2;
    }
    if (lane == 0) {
      const uint32_t sg = *reinterpret_cast<const uint32_t*>(src + gh.off_score + 4 * is);
      const int32_t ps = *reinterpret_cast<const int32_t*>(src + gh.off_pos + 4 * is);
      *reinterpret_cast<uint32_t*>(dst + go.off_score + 4 * id) = sg;
      *reinterpret_cast<int32_t*>(dst + go.off_pos + 4 * id) = ps;
    }
  }

  // 2. t_c: quantize window slot (N-1) mod W == p_c mod W at its class bits
  const int ws = p.W > 0 ? (N - 1) % p.W : 0;
  uint4 nv = make_uint4(0, 0, 0, 0), wv = make_uint4(0, 0, 0, 0);
  __half* wrow = nullptr;
  if (kv) {
    nv = *reinterpret_cast<const uint4*>((grp == 0 ? knew : vnew) + (size_t)u * d + gl * 8);
    if (p.W > 0) {
      wrow = (grp == 0 ? p.win_k : p.win_v) + ((size_t)u * p.W + ws) * d + gl * 8;
      wv = *reinterpret_cast<const uint4*>(wrow);
    }
  }
  if (tc_class == DKV_CLS_HIGH || tc_class == DKV_CLS_LOW) {
    const ClassGeom g = geom_of(p, tc_class);
    float x[8];
    unpack_h8(p.W > 0 ? wv : nv, x);
    const int b = grp == 0 ? g.kbits : g.vbits;
    uint32_t meta;
    bool fin;
    const uint64_t q = quantize8<G>(x, kv ? b : 8, meta, fin);
    if (!__all_sync(kFull, fin || !kv)) {
      if (lane == 0) set_status(p.ctrl, DKV_ERR_NONFINITE);
    } else {
      int idx;
      uint8_t* pg = slot_page(p, tc_class, u, tc_slot, idx);
      if (kv) {
        store_codes(pg + (grp == 0 ? g.off_k + idx * g.k_row : g.off_v + idx * g.v_row) + gl * b, q, b);
        if (gl == 0) *reinterpret_cast<uint32_t*>(pg + (grp == 0 ? g.off_kmeta : g.off_vmeta) + 4 * idx) = meta;
      }
      if (lane == 0) {
        *reinterpret_cast<float*>(pg + g.off_score + 4 * idx) = canon_zero(cand_sig[u]);
        *reinterpret_cast<int32_t*>(pg + g.off_pos + 4 * idx) = pc;
      }
    }
  }
  // 3. window push (read-before-write of the same slot by the same lane)
  if (kv && p.W > 0) *reinterpret_cast<uint4*>(wrow) = nv;
}

cudaError_t launch_quant_decode(const PoolDev& p, const dkv_decision_t* dec, const uint16_t* k, const uint16_t* v,
                                const float* sig, cudaStream_t s) {
  const int grid = (p.U + kQWarps - 1) / kQWarps;
  if (p.d == 128) quant_decode_kernel<16><<<grid, kQWarps * 32, 0, s>>>(p, dec, k, v, sig);
  else quant_decode_kernel<8><<<grid, kQWarps * 32, 0, s>>>(p, dec, k, v, sig);
  return cudaGetLastError();
}

// ------------------------------------------------------------------------------------------- bulk
// One warp per (admitted unit, 256-token segment).  Groups of 4 lanes own one token: lane quarter q of
// the group holds elements [q*d/4, (q+1)*d/4) of the K row and of the V row (d/4 halves = d/8 bytes*4).
constexpr int kBulkWarps = 4;
constexpr int kBulkG = 4;

__device__ __forceinline__ int prompt_class_q(const PoolDev& p, float s, int t, int T) {
  const float den = (p.prompt_den == 0) ? (float)(t + 1) : (float)T;
  const float th = __fdiv_rn(p.alpha_h, den), tl = __fdiv_rn(p.alpha_l, den);
  return s >= th ? DKV_CLS_HIGH : (s >= tl ? DKV_CLS_LOW : DKV_CLS_PRUNED);
}

template <int NW>
__device__ __forceinline__ void quant_store_vec(const uint32_t (&x)[NW], int bits, uint8_t* dst, uint32_t& meta,
                                                bool& ok) {
  // dst = this lane's part of the token's code row
  if (bits == 8) {
    uint32_t cw[NW / 2];
    quant_h16<kBulkG, NW, 8>(x, cw, meta, ok);
    store_words(dst, cw);
  } else if (bits == 4) {
    uint32_t cw[NW / 4];
    quant_h16<kBulkG, NW, 4>(x, cw, meta, ok);
    store_words(dst, cw);
  } else {
    uint32_t cw[(NW / 8) > 0 ? NW / 8 : 1];
    if constexpr (NW >= 8) {
      quant_h16<kBulkG, NW, 2>(x, cw, meta, ok);
      store_words(dst, cw);
    }
  }
}

template <int D>
__global__ void __launch_bounds__(kBulkWarps * 32)
quant_prefill_kernel(PoolDev p, int n, const uint16_t* __restrict__ kin, const uint16_t* __restrict__ vin,
                     int64_t kv_stride, const float* __restrict__ sig, int64_t sig_stride, int nseg_max) {
  constexpr int NW = D / 8;                            // half2 words per lane per vector (d/4 halves)
  constexpr int TPS = 32 / kBulkG;                     // tokens per warp step
  __shared__ uint32_t s_ent[kBulkWarps][kSegTokens];   // high list from the front, low list from the back
  __shared__ uint32_t s_sig[kBulkWarps][kSegTokens];
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const long item = (long)blockIdx.x * kBulkWarps + warp;
  const int seg = (int)(item % nseg_max);
  const long wi = item / nseg_max;                     // admitted unit index (i * LyH + j)
  if (wi >= (long)n * p.LyH) return;
  if (ld_volatile(&p.ctrl->status) != 0) return;
  const int i = (int)(wi / p.LyH), j = (int)(wi % p.LyH);
  const int r = p.admit[i];
  const int u = r * p.LyH + j;
  const int T = p.prompt_len[r];
  const int t0 = seg * kSegTokens;
  if (t0 >= T) return;
  const int t1 = min(t0 + kSegTokens, T);
  const int kept = max(T - p.W, 0);
  const int ke = min(t1, kept);
  const float* srow = sig + wi * sig_stride;
  const uint16_t* kbase = kin + wi * kv_stride * D;
  const uint16_t* vbase = vin + wi * kv_stride * D;

  // phase A: classes + per-class ranks (warp ballot/popc + running offsets) -> two kept lists
  int hr = p.pf_seg[((size_t)u * p.nseg + seg) * 2];
  int lr = p.pf_seg[((size_t)u * p.nseg + seg) * 2 + 1];
  int nh = 0, nl = 0;
  const unsigned lt = (1u << lane) - 1u;
  for (int c = t0; c < ke; c += 32) {
    const int t = c + lane;
    int cl = DKV_CLS_NONE;
    float s = 0.0f;
    if (t < ke) {
      s = canon_zero(__ldcs(srow + t));
      cl = prompt_class_q(p, s, t, T);
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

  // phase B: per class (warp-uniform bit widths), 8 tokens per step, only kept rows are read
  const int grp = lane / kBulkG, q = lane % kBulkG;
  bool bad = false;
#pragma unroll 1
  for (int cls = DKV_CLS_HIGH; cls <= DKV_CLS_LOW; cls++) {
    const ClassGeom g = geom_of(p, cls);
    const int cnt = cls == DKV_CLS_HIGH ? nh : nl;
    const int kbytes = (D / 4) * g.kbits / 8, vbytes = (D / 4) * g.vbits / 8;
#pragma unroll 1
    for (int e0 = 0; e0 < cnt; e0 += TPS) {
      const int e = e0 + grp;
      const bool valid = e < cnt;
      const int ix = cls == DKV_CLS_HIGH ? e : kSegTokens - 1 - e;
      const uint32_t ent = valid ? s_ent[warp][ix] : 0u;
      const int t = t0 + (int)(ent & 255u);
      const int slot = (int)(ent >> 8);
      uint32_t xk[NW], xv[NW];
      if (valid) {
        const uint4* ks = reinterpret_cast<const uint4*>(kbase + (size_t)t * D + q * (D / 4));
        const uint4* vs = reinterpret_cast<const uint4*>(vbase + (size_t)t * D + q * (D / 4));
#pragma unroll
        for (int w = 0; w < NW / 4; w++) {
          const uint4 a = ld_stream_v4(ks + w);
          xk[4 * w] = a.x; xk[4 * w + 1] = a.y; xk[4 * w + 2] = a.z; xk[4 * w + 3] = a.w;
        }
#pragma unroll
        for (int w = 0; w < NW / 4; w++) {
          const uint4 a = ld_stream_v4(vs + w);
          xv[4 * w] = a.x; xv[4 * w + 1] = a.y; xv[4 * w + 2] = a.z; xv[4 * w + 3] = a.w;
        }
      } else {
#pragma unroll
        for (int w = 0; w < NW; w++) { xk[w] = 0u; xv[w] = 0u; }
      }
      int idx;
      uint8_t* pg = valid ? slot_page(p, cls, u, slot, idx) : nullptr;
      if (!valid) idx = 0;
      uint32_t mk, mv;
      bool fk, fv;
      uint8_t* kd = pg + g.off_k + idx * g.k_row + q * kbytes;
      uint8_t* vd = pg + g.off_v + idx * g.v_row + q * vbytes;
      // quantize (all lanes; invalid groups compute on zeros and store nothing)
      uint32_t ck[NW / 2], cv[NW / 2];
      if (g.kbits == 8) quant_h16<kBulkG, NW, 8>(xk, *reinterpret_cast<uint32_t(*)[NW / 2]>(ck), mk, fk);
      else if (g.kbits == 4) quant_h16<kBulkG, NW, 4>(xk, *reinterpret_cast<uint32_t(*)[NW / 4]>(ck), mk, fk);
      else quant_h16<kBulkG, NW, 2>(xk, *reinterpret_cast<uint32_t(*)[NW / 8]>(ck), mk, fk);
      if (g.vbits == 8) quant_h16<kBulkG, NW, 8>(xv, *reinterpret_cast<uint32_t(*)[NW / 2]>(cv), mv, fv);
      else if (g.vbits == 4) quant_h16<kBulkG, NW, 4>(xv, *reinterpret_cast<uint32_t(*)[NW / 4]>(cv), mv, fv);
      else quant_h16<kBulkG, NW, 2>(xv, *reinterpret_cast<uint32_t(*)[NW / 8]>(cv), mv, fv);
      if (valid) {
        bad |= !(fk && fv);
        if (g.kbits == 8) store_words(kd, *reinterpret_cast<uint32_t(*)[NW / 2]>(ck));
        else if (g.kbits == 4) store_words(kd, *reinterpret_cast<uint32_t(*)[NW / 4]>(ck));
        else store_words(kd, *reinterpret_cast<uint32_t(*)[NW / 8]>(ck));
        if (g.vbits == 8) store_words(vd, *reinterpret_cast<uint32_t(*)[NW / 2]>(cv));
        else if (g.vbits == 4) store_words(vd, *reinterpret_cast<uint32_t(*)[NW / 4]>(cv));
        else store_words(vd, *reinterpret_cast<uint32_t(*)[NW / 8]>(cv));
        if (q == 0) *reinterpret_cast<uint32_t*>(pg + g.off_kmeta + 4 * idx) = mk;
        if (q == 1) *reinterpret_cast<uint32_t*>(pg + g.off_vmeta + 4 * idx) = mv;
        if (q == 2) *reinterpret_cast<uint32_t*>(pg + g.off_score + 4 * idx) = s_sig[warp][ix];
        if (q == 3) *reinterpret_cast<int32_t*>(pg + g.off_pos + 4 * idx) = t;
      }
    }
  }
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
    }
  }
  if (__any_sync(kFull, bad) && lane == 0) set_status(p.ctrl, DKV_ERR_NONFINITE);
}

// ADMITTING -> ACTIVE once every prompt token is written (skipped while an error is pending)
__global__ void finish_prefill_kernel(PoolDev p, int n) {
  if (ld_volatile(&p.ctrl->status) != 0) return;
  for (int i = threadIdx.x; i < n; i += blockDim.x) {
    const int r = p.admit[i];
    if (p.req_state[r] == DKV_REQ_ADMITTING) p.req_state[r] = DKV_REQ_ACTIVE;
  }
}

cudaError_t launch_quant_prefill(const PoolDev& p, int n, const uint16_t* k, const uint16_t* v, int64_t kv_stride,
                                 const float* sig, int64_t sig_stride, int max_len, cudaStream_t s) {
  const int nseg_max = (max_len + kSegTokens - 1) / kSegTokens;
  const long items = (long)n * p.LyH * nseg_max;
  if (items > 0) {
    const long grid = (items + kBulkWarps - 1) / kBulkWarps;
    if (p.d == 128)
      quant_prefill_kernel<128><<<(unsigned)grid, kBulkWarps * 32, 0, s>>>(p, n, k, v, kv_stride, sig, sig_stride, nseg_max);
    else
      quant_prefill_kernel<64><<<(unsigned)grid, kBulkWarps * 32, 0, s>>>(p, n, k, v, kv_stride, sig, sig_stride, nseg_max);
    cudaError_t e = cudaGetLastError();
    if (e != cudaSuccess) return e;
  }
  finish_prefill_kernel<<<1, 256, 0, s>>>(p, n);
  return cudaGetLastError();
}

}  // namespace dkv
