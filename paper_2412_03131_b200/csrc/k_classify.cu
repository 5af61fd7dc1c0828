// k_classify.cu — planning kernels ("each attention head independently determines its memory
// allocation requirements ... perfectly parallelizable").
//
//  classify_decode  : one 128-thread CTA per unit.  Algorithm 1: the class of t_c from the
//                     thresholds alpha/N, then the victim = lexicographic (score, position) argmin over the
//                     score segments of the section t_c joins.  The section's page IDs are staged in shared
//                     memory with one coalesced pass over its table row, then every thread issues all its
//                     16-B score loads (4 slots each) at once, so a unit costs two dependent memory round
//                     trips; positions are read only on score ties.  HBM-bound: 4 B per stored token.
//  classify_prefill : one warp per admitted unit; §4 thresholds per token, 16-B loads of 4
//                     tokens per lane, class counts by warp reduction, exclusive (high, low) rank
//                     checkpoints every 256 tokens so the bulk writer can start any segment independently.
#include "dkv_internal.cuh"

namespace dkv {

constexpr int kCT = 128;                   // threads per unit in classify_decode
constexpr int kCV = 4;                     // 16-B score vectors per thread per batch (2048 slots per batch)

// position of section slot s (rare path: ties only)
__device__ __forceinline__ int32_t slot_pos(const PoolDev& p, int cls, int u, int s) {
  int idx;
  const uint8_t* pg = slot_page(p, cls, u, s, idx);
  const int off_pos = cls == DKV_CLS_HIGH ? p.g[1].off_pos : p.g[2].off_pos;
  return __ldg(reinterpret_cast<const int32_t*>(pg + off_pos) + idx);
}

__global__ void __launch_bounds__(kCT)
classify_decode_kernel(PoolDev p, const float* __restrict__ cand_sig, dkv_decision_t* __restrict__ dec) {
  extern __shared__ int32_t s_pid[];                             // page IDs of the scanned section
  __shared__ uint32_t s_wbest[kCT / 32];
  __shared__ int32_t s_wslot[kCT / 32], s_wpos[kCT / 32];
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int u = blockIdx.x;
  if (ld_volatile(&p.ctrl->status) != 0) return;                 // sticky error: no-op
  const int r = u / p.LyH;
  uint8_t tc_class = DKV_CLS_NONE, v_action = DKV_V_NONE, grow = DKV_GROW_NONE, demand = 0;
  int v_slot = -1, tc_slot = -1, v_dst_slot = -1;
  bool scan = false;
  int cls = DKV_CLS_NONE, n = 0, nh = 0, nl = 0;
  float sc = 0.0f, th = 0.0f, tl = 0.0f;
  if (p.req_state[r] == DKV_REQ_ACTIVE) {
    const int N = p.seq_len[r] + 1;                              // Q3: includes this step's token
    const int pc = N - 1 - p.W;                                  // t_c = earliest window token
    if (pc >= 0) {
      sc = cand_sig[u];
      if (!finite_f(sc) || sc < 0.0f) {
        if (tid == 0) set_status(p.ctrl, DKV_ERR_NONFINITE);
      } else {
        sc = canon_zero(sc);
        th = __fdiv_rn(p.alpha_h, (float)N);                     // alpha_h / N
        tl = __fdiv_rn(p.alpha_l, (float)N);                     // alpha_l / N
        cls = sc >= th ? DKV_CLS_HIGH : (sc >= tl ? DKV_CLS_LOW : DKV_CLS_PRUNED);
        tc_class = (uint8_t)cls;
        if (cls != DKV_CLS_PRUNED) {
          nh = p.n_h[u];
          nl = p.n_l[u];
          n = (cls == DKV_CLS_HIGH) ? nh : nl;
          scan = true;
        }
      }
    }
  }
  int vs = -1;                                                   // victim slot, -1 = t_c itself
  uint32_t vb = 0xFFFFFFFFu;
  if (scan && n > 0) {                                           // CTA-uniform
    const int C = cls == DKV_CLS_HIGH ? p.g[1].C : p.g[2].C;
    const int off_score = cls == DKV_CLS_HIGH ? p.g[1].off_score : p.g[2].off_score;
    const bool pow2 = (C & (C - 1)) == 0;
    const int csh = __popc(C - 1);
    const int npages = (n + C - 1) / C;
    const int32_t* row = p.table + (size_t)u * p.L;
    for (int k = tid; k < npages; k += kCT) s_pid[k] = __ldg(row + (cls == DKV_CLS_HIGH ? k : p.L - 1 - k));
    __syncthreads();
    const uint8_t* base_sc = p.pages + off_score;
    // Stored scores are canonical non-negative floats (writers canonicalise -0, Q6): unsigned order of the
    // bit patterns is the float order.
    uint32_t best = 0xFFFFFFFFu;
    int bslot = -1;
    int32_t bpos = -1;                                           // -1 = not loaded yet
    for (int base = 0; base < n; base += 4 * kCT * kCV) {
      uint4 v[kCV];
#pragma unroll
      for (int j = 0; j < kCV; j++) {
        const int s0 = base + j * 4 * kCT + 4 * tid;
        v[j] = make_uint4(0xFFFFFFFFu, 0xFFFFFFFFu, 0xFFFFFFFFu, 0xFFFFFFFFu);
        if (s0 < n) {
          const int pg = pow2 ? (s0 >> csh) : s0 / C;
          const int ix = pow2 ? (s0 & (C - 1)) : s0 % C;
          v[j] = ld_nc_v4(base_sc + (size_t)s_pid[pg] * (size_t)p.page_bytes + 4 * ix);
        }
      }
#pragma unroll
      for (int j = 0; j < kCV; j++) {
        const int s0 = base + j * 4 * kCT + 4 * tid;
        uint32_t e4[4] = {v[j].x, v[j].y, v[j].z, v[j].w};
        if (s0 + 3 >= n) {                                       // tail vector: mask slots >= n
#pragma unroll
          for (int e = 0; e < 4; e++) if (s0 + e >= n) e4[e] = 0xFFFFFFFFu;
        }
        const uint32_t m4 = min(min(e4[0], e4[1]), min(e4[2], e4[3]));
        if (m4 <= best && m4 != 0xFFFFFFFFu) {
#pragma unroll
          for (int e = 0; e < 4; e++) {
            const uint32_t b = e4[e];
            const int s = s0 + e;
            if (b < best) {
              best = b; bslot = s; bpos = -1;
            } else if (b == best) {                              // score tie: older position wins (Q6)
              if (bpos < 0) bpos = slot_pos(p, cls, u, bslot);
              const int32_t ps = slot_pos(p, cls, u, s);
              if (ps < bpos) { bslot = s; bpos = ps; }
            }
          }
        }
      }
    }
    // warp argmin
    const uint32_t m = __reduce_min_sync(kFull, best);
    const bool cand = (best == m) && (bslot >= 0);
    const unsigned tie = __ballot_sync(kFull, cand);
    int wslot = -1;
    int32_t wpos = -1;
    if (tie) {
      int wl;
      if (__popc(tie) == 1) {
        wl = __ffs(tie) - 1;
      } else {
        if (cand && bpos < 0) bpos = slot_pos(p, cls, u, bslot);
        const uint32_t pk = cand ? (uint32_t)bpos : 0xFFFFFFFFu;
        const uint32_t mp = __reduce_min_sync(kFull, pk);
        wl = __ffs(__ballot_sync(kFull, cand && pk == mp)) - 1;
      }
      wslot = __shfl_sync(kFull, bslot, wl);
      wpos = __shfl_sync(kFull, bpos, wl);
    }
    if (lane == 0) { s_wbest[warp] = m; s_wslot[warp] = wslot; s_wpos[warp] = wpos; }
    __syncthreads();
    if (tid == 0) {                                              // CTA argmin over the warp winners
      uint32_t mm = 0xFFFFFFFFu;
#pragma unroll
      for (int w = 0; w < kCT / 32; w++) mm = min(mm, s_wbest[w]);
      int32_t bp = 0x7FFFFFFF;
      int cnt = 0;
#pragma unroll
      for (int w = 0; w < kCT / 32; w++) cnt += (s_wbest[w] == mm && s_wslot[w] >= 0);
#pragma unroll
      for (int w = 0; w < kCT / 32; w++) {
        if (s_wbest[w] != mm || s_wslot[w] < 0) continue;
        if (cnt == 1) { vs = s_wslot[w]; break; }
        const int32_t ps = s_wpos[w] >= 0 ? s_wpos[w] : slot_pos(p, cls, u, s_wslot[w]);
        if (ps < bp) { bp = ps; vs = s_wslot[w]; }
      }
      vb = mm;
    }
  }
  if (tid != 0) return;
  if (scan) {
    // t_c has the largest position, so a stored token wins every score tie with it
    if (vs >= 0 && !(vb <= __float_as_uint(sc))) vs = -1;
    const float sv = __uint_as_float(vb);
    if (cls == DKV_CLS_HIGH) {
      if (vs < 0 || sv >= th) {                                  // t_v stays in KV_h
        v_action = DKV_V_KEEP; grow = DKV_GROW_HIGH; demand = (nh % p.Ch == 0); tc_slot = nh;
      } else if (sv >= tl) {                                     // line requant_high
        v_action = DKV_V_DOWN; grow = DKV_GROW_LOW; demand = (nl % p.Cl == 0);
        v_slot = vs; tc_slot = vs; v_dst_slot = nl;
      } else {                                                   // prune t_v
        v_action = DKV_V_PRUNE; v_slot = vs; tc_slot = vs;
      }
    } else {
      if (vs < 0 || sv >= tl) {
        v_action = DKV_V_KEEP; grow = DKV_GROW_LOW; demand = (nl % p.Cl == 0); tc_slot = nl;
      } else {                                                   // line prune_low
        v_action = DKV_V_PRUNE; v_slot = vs; tc_slot = vs;
      }
    }
  }
  int4 w;
  w.x = (int)((uint32_t)tc_class | ((uint32_t)v_action << 8) | ((uint32_t)grow << 16) | ((uint32_t)demand << 24));
  w.y = v_slot; w.z = tc_slot; w.w = v_dst_slot;
  reinterpret_cast<int4*>(dec)[u] = w;
}

cudaError_t launch_classify_decode(const PoolDev& p, const float* sig, dkv_decision_t* dec, cudaStream_t s) {
  const size_t smem = 4 * (size_t)p.L;
  if (smem > 48 * 1024) {
    cudaError_t e = cudaFuncSetAttribute(classify_decode_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    if (e != cudaSuccess) return e;
  }
  classify_decode_kernel<<<p.U, kCT, smem, s>>>(p, sig, dec);
  return cudaGetLastError();
}

// ------------------------------------------------------------------------------------------- prefill
constexpr int kPrefillWarps = 4;

__device__ __forceinline__ int prompt_class(const PoolDev& p, float s, int t, int T) {
  const float den = (p.prompt_den == 0) ? (float)(t + 1) : (float)T;
  const float th = __fdiv_rn(p.alpha_h, den), tl = __fdiv_rn(p.alpha_l, den);
  return s >= th ? DKV_CLS_HIGH : (s >= tl ? DKV_CLS_LOW : DKV_CLS_PRUNED);
}

// VEC: rows are 16-B aligned (sig_stride % 4 == 0): lane owns 4 consecutive tokens per 128-token step.
template <bool VEC>
__global__ void __launch_bounds__(kPrefillWarps * 32)
classify_prefill_kernel(PoolDev p, int n, const float* __restrict__ sig, int64_t sig_stride, uint8_t* __restrict__ cls_out) {
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int w = blockIdx.x * kPrefillWarps + warp;               // (admitted index, unit-in-request)
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
  constexpr int TPL = VEC ? 4 : 1;                               // tokens per lane per step
  constexpr int STEP = 32 * TPL;
  constexpr int UNR = VEC ? 4 : 8;                               // steps in flight
  for (int tb = 0; tb < T; tb += STEP * UNR) {
    float sv[UNR][TPL];
#pragma unroll
    for (int k = 0; k < UNR; k++) {
      const int t = tb + k * STEP + lane * TPL;
      if constexpr (VEC) {
        float4 f = make_float4(0.f, 0.f, 0.f, 0.f);
        if (t < kept) f = __ldcs(reinterpret_cast<const float4*>(row + t));
        sv[k][0] = f.x; sv[k][1] = f.y; sv[k][2] = f.z; sv[k][3] = f.w;
      } else {
        sv[k][0] = (t < kept) ? __ldcs(row + t) : 0.0f;
      }
    }
#pragma unroll
    for (int k = 0; k < UNR; k++) {
      const int ts = tb + k * STEP;
      if (ts >= T) break;
      if ((ts % kSegTokens) == 0 && lane == 0) {                 // rank checkpoint at segment start
        seg[2 * (ts / kSegTokens)] = nh;
        seg[2 * (ts / kSegTokens) + 1] = nl;
      }
      int ch = 0, cl = 0;
      uint32_t cbytes = 0;
#pragma unroll
      for (int e = 0; e < TPL; e++) {
        const int t = ts + lane * TPL + e;
        int c = DKV_CLS_NONE;
        if (t < kept) {
          float s = sv[k][e];
          if (!finite_f(s) || s < 0.0f) { bad = true; s = 0.0f; }
          c = prompt_class(p, canon_zero(s), t, T);
        }
        ch += c == DKV_CLS_HIGH;
        cl += c == DKV_CLS_LOW;
        cbytes |= (uint32_t)c << (8 * e);
      }
      nh += __reduce_add_sync(kFull, (unsigned)ch);
      nl += __reduce_add_sync(kFull, (unsigned)cl);
      if (crow) {
        const int t = ts + lane * TPL;
        if constexpr (VEC) {
          if (t + 3 < T) *reinterpret_cast<uint32_t*>(crow + t) = cbytes;
          else for (int e = 0; e < 4; e++) if (t + e < T) crow[t + e] = (uint8_t)(cbytes >> (8 * e));
        } else {
          if (t < T) crow[t] = (uint8_t)cbytes;
        }
      }
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
  const int grid = (warps + kPrefillWarps - 1) / kPrefillWarps;
  const bool vec = (sig_stride % 4 == 0) && ((uintptr_t)sig % 16 == 0) && ((uintptr_t)cls % 4 == 0);
  if (vec) classify_prefill_kernel<true><<<grid, kPrefillWarps * 32, 0, s>>>(p, n, sig, sig_stride, cls);
  else classify_prefill_kernel<false><<<grid, kPrefillWarps * 32, 0, s>>>(p, n, sig, sig_stride, cls);
  return cudaGetLastError();
}

}  // namespace dkv
