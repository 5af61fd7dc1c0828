// k_classify.cu — planning kernels ("each attention head independently determines its memory
// allocation requirements ... perfectly parallelizable").
//
//  classify_decode  : one warp per unit.  Algorithm 1 with the victim found by a warp-wide
//                     lexicographic (score, position) argmin over the score segments of the section t_c
//                     joins.  The scan is HBM-bound (4 B per stored token); scores are fetched as 16-B
//                     vectors (4 slots per lane, 128 slots per warp load), page IDs are preloaded 32 at
//                     a time and broadcast with shuffles, positions are read only on score ties.
//  classify_prefill : one warp per admitted unit; §4 thresholds per token, warp ballot/popc
//                     class counts, exclusive (high, low) rank checkpoints every 256 tokens so the bulk
//                     writer can start any segment independently.
#include "dkv_internal.cuh"

namespace dkv {

constexpr int kDecodeWarps = 8;
constexpr int kScanUnroll = 4;

// position of section slot s (rare path: ties only)
__device__ __forceinline__ uint32_t slot_pos(const PoolDev& p, int cls, int u, int s) {
  int idx;
  const uint8_t* pg = slot_page(p, cls, u, s, idx);
  const int off_pos = cls == DKV_CLS_HIGH ? p.g[1].off_pos : p.g[2].off_pos;
  return (uint32_t)__ldg(reinterpret_cast<const int32_t*>(pg + off_pos) + idx);
}

// Warp-wide argmin of (score, position) over slots [0, n) of section `cls` of unit u.
// Returns the winning slot (or -1 if n == 0) and its score bits (canonical, non-negative float bits).
__device__ __forceinline__ int section_argmin(const PoolDev& p, int cls, int u, int n, int lane, uint32_t& vbits) {
  const ClassGeom g = geom_of(p, cls);
  const int C = g.C;
  const int32_t* row = p.table + (size_t)u * p.L;
  const int npages = (n + C - 1) / C;
  uint32_t best = 0xFFFFFFFFu;
  int bslot = -1;
  int32_t bpos = -1;     // -1 = not loaded yet
  for (int kb = 0; kb < npages; kb += 32) {
    const int kk = kb + lane;
    int pidr = 0;
    if (kk < npages) pidr = __ldg(row + (cls == DKV_CLS_HIGH ? kk : p.L - 1 - kk));
    const int tok_lo = kb * C;
    const int tok_hi = min(n, (kb + 32) * C);
    for (int base = tok_lo; base < tok_hi; base += 128 * kScanUnroll) {
      uint4 v[kScanUnroll];
      int s0[kScanUnroll];
#pragma unroll
      for (int j = 0; j < kScanUnroll; j++) {
        s0[j] = base + j * 128 + lane * 4;
        int rel = s0[j] / C - kb;
        rel = rel < 0 ? 0 : (rel > 31 ? 31 : rel);
        const int pid = __shfl_sync(kFull, pidr, rel);
        v[j] = make_uint4(0xFFFFFFFFu, 0xFFFFFFFFu, 0xFFFFFFFFu, 0xFFFFFFFFu);
        if (s0[j] < tok_hi) {
          const uint8_t* src = p.pages + (size_t)pid * (size_t)p.page_bytes + g.off_score + 4 * (s0[j] % C);
          v[j] = ld_nc_v4(src);
        }
      }
#pragma unroll
      for (int j = 0; j < kScanUnroll; j++) {
        const uint32_t e4[4] = {v[j].x, v[j].y, v[j].z, v[j].w};
#pragma unroll
        for (int e = 0; e < 4; e++) {
          const int s = s0[j] + e;
          if (s >= tok_hi) continue;
          uint32_t b = e4[e];
          b = (b == 0x80000000u) ? 0u : b;              // -0 == +0 (Q6)
          if (b < best) {
            best = b; bslot = s; bpos = -1;
          } else if (b == best) {                        // score tie: older position wins (Q6)
            if (bpos < 0) bpos = (int32_t)slot_pos(p, cls, u, bslot);
            const int32_t ps = (int32_t)slot_pos(p, cls, u, s);
            if (ps < bpos) { bslot = s; bpos = ps; }
          }
        }
      }
    }
  }
  const uint32_t m = __reduce_min_sync(kFull, best);
  if (m == 0xFFFFFFFFu) { vbits = m; return -1; }
  const bool cand = (best == m) && (bslot >= 0);
  const unsigned tie = __ballot_sync(kFull, cand);
  int wl;
  if (__popc(tie) == 1) {
    wl = __ffs(tie) - 1;
  } else {
    if (cand && bpos < 0) bpos = (int32_t)slot_pos(p, cls, u, bslot);
    const uint32_t pk = cand ? (uint32_t)bpos : 0xFFFFFFFFu;
    const uint32_t mp = __reduce_min_sync(kFull, pk);
    wl = __ffs(__ballot_sync(kFull, cand && pk == mp)) - 1;
  }
  vbits = m;
  return __shfl_sync(kFull, bslot, wl);
}

__global__ void __launch_bounds__(kDecodeWarps * 32)
classify_decode_kernel(PoolDev p, const float* __restrict__ cand_sig, dkv_decision_t* __restrict__ dec) {
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int u = blockIdx.x * kDecodeWarps + warp;
  if (u >= p.U) return;
  if (ld_volatile(&p.ctrl->status) != 0) return;                 // sticky error: no-op
  const int r = u / p.LyH;
  uint8_t tc_class = DKV_CLS_NONE, v_action = DKV_V_NONE, grow = DKV_GROW_NONE, demand = 0;
  int v_slot = -1, tc_slot = -1, v_dst_slot = -1;
  if (p.req_state[r] == DKV_REQ_ACTIVE) {
    const int N = p.seq_len[r] + 1;                              // Q3: includes this step's token
    const int pc = N - 1 - p.W;                                  // t_c = earliest window token
    if (pc >= 0) {
      float sc = cand_sig[u];
      if (!finite_f(sc) || sc < 0.0f) {
        if (lane == 0) set_status(p.ctrl, DKV_ERR_NONFINITE);
      } else {
        sc = canon_zero(sc);
        const float th = __fdiv_rn(p.alpha_h, (float)N);         // alpha_h / N
        const float tl = __fdiv_rn(p.alpha_l, (float)N);         // alpha_l / N
        int cls = sc >= th ? DKV_CLS_HIGH : (sc >= tl ? DKV_CLS_LOW : DKV_CLS_PRUNED);
        if (cls == DKV_CLS_PRUNED) {
          tc_class = DKV_CLS_PRUNED;
        } else {
          const int nh = p.n_h[u], nl = p.n_l[u];
          const int n = (cls == DKV_CLS_HIGH) ? nh : nl;
          uint32_t vb;
          int vs = section_argmin(p, cls, u, n, lane, vb);
          // t_c has the largest position, so a stored token wins every score tie with it
          if (vs >= 0 && !(vb <= __float_as_uint(sc))) vs = -1;
          const float sv = __uint_as_float(vb);
          tc_class = (uint8_t)cls;
          if (cls == DKV_CLS_HIGH) {
            if (vs < 0 || sv >= th) {                            // t_v stays in KV_h
              v_action = DKV_V_KEEP; grow = DKV_GROW_HIGH; demand = (nh % p.Ch == 0); tc_slot = nh;
            } else if (sv >= tl) {                               // line requant_high
              v_action = DKV_V_DOWN; grow = DKV_GROW_LOW; demand = (nl % p.Cl == 0);
              v_slot = vs; tc_slot = vs; v_dst_slot = nl;
            } else {                                             // prune t_v
              v_action = DKV_V_PRUNE; v_slot = vs; tc_slot = vs;
            }
          } else {
            if (vs < 0 || sv >= tl) {
              v_action = DKV_V_KEEP; grow = DKV_GROW_LOW; demand = (nl % p.Cl == 0); tc_slot = nl;
            } else {                                             // line prune_low
              v_action = DKV_V_PRUNE; v_slot = vs; tc_slot = vs;
            }
          }
        }
      }
    }
  }
  if (lane == 0) {
    int4 w;
    w.x = (int)((uint32_t)tc_class | ((uint32_t)v_action << 8) | ((uint32_t)grow << 16) | ((uint32_t)demand << 24));
    w.y = v_slot; w.z = tc_slot; w.w = v_dst_slot;
    reinterpret_cast<int4*>(dec)[u] = w;
  }
}

cudaError_t launch_classify_decode(const PoolDev& p, const float* sig, dkv_decision_t* dec, cudaStream_t s) {
  const int grid = (p.U + kDecodeWarps - 1) / kDecodeWarps;
  classify_decode_kernel<<<grid, kDecodeWarps * 32, 0, s>>>(p, sig, dec);
  return cudaGetLastError();
}

// ------------------------------------------------------------------------------------------- prefill
constexpr int kPrefillWarps = 8;

__device__ __forceinline__ int prompt_class(const PoolDev& p, float s, int t, int T) {
  const float den = (p.prompt_den == 0) ? (float)(t + 1) : (float)T;
  const float th = __fdiv_rn(p.alpha_h, den), tl = __fdiv_rn(p.alpha_l, den);
  return s >= th ? DKV_CLS_HIGH : (s >= tl ? DKV_CLS_LOW : DKV_CLS_PRUNED);
}

__global__ void __launch_bounds__(kPrefillWarps * 32)
classify_prefill_kernel(PoolDev p, int n, const float* __restrict__ sig, int64_t sig_stride, uint8_t* __restrict__ cls_out) {
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int w = blockIdx.x * kPrefillWarps + warp;                 // (admitted index, unit-in-request)
  if (w >= n * p.LyH) return;
  if (ld_volatile(&p.ctrl->status) != 0) return;
  const int i = w / p.LyH, j = w % p.LyH;
  const int r = p.admit[i];
  const int u = r * p.LyH + j;
  const int T = p.prompt_len[r];
  const int kept = max(T - p.W, 0);
  const float* row = sig + (int64_t)w * sig_stride;
  uint8_t* crow = cls_out ? cls_out + (int64_t)w * sig_stride : nullptr;
  int32_t* seg = p.pf_seg + (size_t)u * p.nseg * 2;
  int nh = 0, nl = 0;
  bool bad = false;
  for (int t0 = 0; t0 < T; t0 += 32 * 4) {
    float sv[4];
#pragma unroll
    for (int c = 0; c < 4; c++) {
      const int t = t0 + c * 32 + lane;
      sv[c] = (t < kept) ? __ldcs(row + t) : 0.0f;
    }
#pragma unroll
    for (int c = 0; c < 4; c++) {
      const int tc = t0 + c * 32;
      if (tc >= T) break;
      const int t = tc + lane;
      if ((tc % kSegTokens) == 0 && lane == 0) {                   // rank checkpoint at segment start
        seg[2 * (tc / kSegTokens)] = nh;
        seg[2 * (tc / kSegTokens) + 1] = nl;
      }
      int cl = DKV_CLS_NONE;
      if (t < kept) {
        float s = sv[c];
        if (!finite_f(s) || s < 0.0f) { bad = true; s = 0.0f; }
        cl = prompt_class(p, canon_zero(s), t, T);
      }
      const unsigned hm = __ballot_sync(kFull, cl == DKV_CLS_HIGH);
      const unsigned lm = __ballot_sync(kFull, cl == DKV_CLS_LOW);
      nh += __popc(hm);
      nl += __popc(lm);
      if (crow && t < T) crow[t] = (uint8_t)cl;
    }
  }
  if (__any_sync(kFull, bad) && lane == 0) set_status(p.ctrl, DKV_ERR_NONFINITE);
  if (lane == 0) { p.pf_nh[u] = nh; p.pf_nl[u] = nl; }
}

cudaError_t launch_classify_prefill(const PoolDev& p, int n, const float* sig, int64_t sig_stride, uint8_t* cls,
                                    int max_len, cudaStream_t s) {
  (void)max_len;
  const int warps = n * p.LyH;
  if (warps == 0) return cudaSuccess;
  classify_prefill_kernel<<<(warps + kPrefillWarps - 1) / kPrefillWarps, kPrefillWarps * 32, 0, s>>>(p, n, sig,
                                                                                                    sig_stride, cls);
  return cudaGetLastError();
}

}  // namespace dkv
