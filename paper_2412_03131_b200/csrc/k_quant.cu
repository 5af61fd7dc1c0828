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
constexpr int kBulkUnroll = 4;

__device__ __forceinline__ int prompt_class_q(const PoolDev& p, float s, int t, int T) {
  const float den = (p.prompt_den == 0) ? (float)(t + 1) : (float)T;
  const float th = __fdiv_rn(p.alpha_h, den), tl = __fdiv_rn(p.alpha_l, den);
  return s >= th ? DKV_CLS_HIGH : (s >= tl ? DKV_CLS_LOW : DKV_CLS_PRUNED);
}

template <int G>
__global__ void __launch_bounds__(kQWarps * 32)
quant_prefill_kernel(PoolDev p, int n, const uint16_t* __restrict__ kin, const uint16_t* __restrict__ vin,
                     int64_t kv_stride, const float* __restrict__ sig, int64_t sig_stride, int nseg_max) {
  constexpr int TPS = 32 / G;                        // tokens per warp step
  __shared__ uint32_t s_ent[kQWarps][kSegTokens];    // (t - t0) | cls << 9 | slot << 11
  __shared__ uint32_t s_sig[kQWarps][kSegTokens];
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const long item = (long)blockIdx.x * kQWarps + warp;
  const int seg = (int)(item % nseg_max);
  const long wi = item / nseg_max;                   // admitted unit index (i * LyH + j)
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
  const int d = p.d;
  const float* srow = sig + wi * sig_stride;
  const uint16_t* kbase = kin + wi * kv_stride * d;
  const uint16_t* vbase = vin + wi * kv_stride * d;

  // phase A: classes + ranks (ballot/popc) -> kept-token list
  int hr = p.pf_seg[((size_t)u * p.nseg + seg) * 2];
  int lr = p.pf_seg[((size_t)u * p.nseg + seg) * 2 + 1];
  int cnt = 0;
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
    const unsigned km = hm | lm;
    if (cl == DKV_CLS_HIGH || cl == DKV_CLS_LOW) {
      const int slot = cl == DKV_CLS_HIGH ? hr + __popc(hm & lt) : lr + __popc(lm & lt);
      const int e = cnt + __popc(km & lt);
      s_ent[warp][e] = (uint32_t)(t - t0) | ((uint32_t)cl << 9) | ((uint32_t)slot << 11);
      s_sig[warp][e] = __float_as_uint(s);
    }
    hr += __popc(hm);
    lr += __popc(lm);
    cnt += __popc(km);
  }
  __syncwarp();

  // phase B: stream kept rows, quantize, store
  const int grp = lane / G, gl = lane % G;
  bool bad = false;
  for (int e0 = 0; e0 < cnt; e0 += TPS * kBulkUnroll) {
    uint4 xk[kBulkUnroll], xv[kBulkUnroll];
    uint32_t ent[kBulkUnroll];
#pragma unroll
    for (int q = 0; q < kBulkUnroll; q++) {
      const int e = e0 + q * TPS + grp;
      ent[q] = e < cnt ? s_ent[warp][e] : 0xFFFFFFFFu;
      xk[q] = make_uint4(0, 0, 0, 0);
      xv[q] = make_uint4(0, 0, 0, 0);
      if (e < cnt) {
        const size_t t = (size_t)(t0 + (ent[q] & 511u));
        xk[q] = ld_stream_v4(kbase + t * d + gl * 8);
        xv[q] = ld_stream_v4(vbase + t * d + gl * 8);
      }
    }
#pragma unroll
    for (int q = 0; q < kBulkUnroll; q++) {
      if (e0 + q * TPS >= cnt) break;                // warp-uniform
      const bool valid = ent[q] != 0xFFFFFFFFu;
      const int cl = valid ? (int)((ent[q] >> 9) & 3u) : DKV_CLS_HIGH;
      const int slot = (int)(ent[q] >> 11);
      const ClassGeom g = geom_of(p, cl);
      float x[8];
      uint32_t mk, mv;
      bool fk, fv;
      unpack_h8(xk[q], x);
      const uint64_t qk = quantize8<G>(x, g.kbits, mk, fk);
      unpack_h8(xv[q], x);
      const uint64_t qv = quantize8<G>(x, g.vbits, mv, fv);
      if (valid) {
        bad |= !(fk && fv);
        int idx;
        uint8_t* pg = slot_page(p, cl, u, slot, idx);
        store_codes(pg + g.off_k + idx * g.k_row + gl * g.kbits, qk, g.kbits);
        store_codes(pg + g.off_v + idx * g.v_row + gl * g.vbits, qv, g.vbits);
        if (gl == 0) *reinterpret_cast<uint32_t*>(pg + g.off_kmeta + 4 * idx) = mk;
        if (gl == 1) *reinterpret_cast<uint32_t*>(pg + g.off_vmeta + 4 * idx) = mv;
        if (gl == 2) *reinterpret_cast<uint32_t*>(pg + g.off_score + 4 * idx) = s_sig[warp][e0 + q * TPS + grp];
        if (gl == 3) *reinterpret_cast<int32_t*>(pg + g.off_pos + 4 * idx) = t0 + (int)(ent[q] & 511u);
      }
    }
  }
  // phase C: the newest min(W, T) tokens -> FP16 window slot t mod W (Q10)
  for (int t = max(t0, kept) + grp; t < t1; t += TPS) {
    const uint4 a = ld_stream_v4(kbase + (size_t)t * d + gl * 8);
    const uint4 b = ld_stream_v4(vbase + (size_t)t * d + gl * 8);
    const size_t w = ((size_t)u * p.W + (t % p.W)) * d + gl * 8;
    *reinterpret_cast<uint4*>(p.win_k + w) = a;
    *reinterpret_cast<uint4*>(p.win_v + w) = b;
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
    const long grid = (items + kQWarps - 1) / kQWarps;
    if (p.d == 128)
      quant_prefill_kernel<16><<<(unsigned)grid, kQWarps * 32, 0, s>>>(p, n, k, v, kv_stride, sig, sig_stride, nseg_max);
    else
      quant_prefill_kernel<8><<<(unsigned)grid, kQWarps * 32, 0, s>>>(p, n, k, v, kv_stride, sig, sig_stride, nseg_max);
    cudaError_t e = cudaGetLastError();
    if (e != cudaSuccess) return e;
  }
  finish_prefill_kernel<<<1, 256, 0, s>>>(p, n);
  return cudaGetLastError();
}

}  // namespace dkv
