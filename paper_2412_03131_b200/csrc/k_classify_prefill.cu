// k_classify_prefill.cu — prompt-phase planning (a8): §4 thresholds per token, one warp per
// admitted unit, 16-B loads of 4 tokens per lane, class counts by warp reduction, and exclusive
// (high, low) rank checkpoints every 256 tokens so the bulk writer can start any segment independently.
#include "dkv_internal.cuh"

namespace dkv {

// ------------------------------------------------------------------------------------------- prefill
constexpr int kPrefillWarps = 4;

__device__ __forceinline__ int prompt_class(float ah, float al, int prompt_den, float s, int t, int T, int top = 0,
                                            float at = 0.0f) {
  const float den = (prompt_den == 0) ? (float)(t + 1) : (float)T;
  const float th = __fdiv_rn(ah, den), tl = __fdiv_rn(al, den);
  if (top && s >= __fdiv_rn(at, den)) return DKV_CLS_TOP;       // NEXT-4 (Q38)
  return s >= th ? DKV_CLS_HIGH : (s >= tl ? DKV_CLS_LOW : DKV_CLS_PRUNED);
}

// VEC: rows are 16-B aligned (sig_stride % 4 == 0): lane owns 4 consecutive tokens per 128-token step.
template <bool VEC>
__global__ void __launch_bounds__(kPrefillWarps * 32)
classify_prefill_kernel(PoolDev p, int n, const float* __restrict__ sig, int64_t sig_stride, uint8_t* __restrict__ cls_out) {
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int w = blockIdx.x * kPrefillWarps + warp;               // (admitted index, unit-in-request)
  if (w >= n * p.LyH) return;
  const int i = w / p.LyH, j = w % p.LyH;
  const int r = p.admit[i];
  const int u = r * p.LyH + j;
  const float ah = unit_alpha_h(p, u), al = unit_alpha_l(p, u);  // Q35
  const int T = p.prompt_len[r];
  const int kept = max(T - p.W, 0);
  const float* row = sig + (int64_t)w * sig_stride;
  uint8_t* crow = cls_out ? cls_out + (int64_t)w * sig_stride : nullptr;
  if (ld_volatile(&p.ctrl->status) != 0) {              // sticky error at entry (Q36): no classes, no counts
    if (crow)
      for (int t = lane; t < T; t += 32) crow[t] = DKV_CLS_NONE;
    if (lane == 0) { p.pf_nh[u] = 0; p.pf_nl[u] = 0; if (p.top) p.pf_nt[u] = 0; }
    return;
  }
  int32_t* seg = p.pf_seg + (size_t)u * p.nseg * 2;
  int nh = 0, nl = 0, nt = 0;
  int32_t* seg_t = p.pf_seg_t + (size_t)u * p.nseg;             // NEXT-4 TOP rank checkpoints
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
        if (p.top) seg_t[ts / kSegTokens] = nt;
      }
      int ch = 0, cl = 0, ct = 0;
      uint32_t cbytes = 0;
#pragma unroll
      for (int e = 0; e < TPL; e++) {
        const int t = ts + lane * TPL + e;
        int c = DKV_CLS_NONE;
        if (t < kept) {
          float s = sv[k][e];
          if (!finite_f(s) || s < 0.0f) { bad = true; s = 0.0f; }
          c = prompt_class(ah, al, p.prompt_den, canon_zero(s), t, T, p.top, p.alpha_t);
        }
        ch += c == DKV_CLS_HIGH;
        cl += c == DKV_CLS_LOW;
        ct += c == DKV_CLS_TOP;
        cbytes |= (uint32_t)c << (8 * e);
      }
      nh += __reduce_add_sync(kFull, (unsigned)ch);
      nl += __reduce_add_sync(kFull, (unsigned)cl);
      if (p.top) nt += __reduce_add_sync(kFull, (unsigned)ct);
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
  if (__any_sync(kFull, bad) && lane == 0) set_pending(p.ctrl, DKV_ERR_NONFINITE);   // Q36
  if (lane == 0) { p.pf_nh[u] = nh; p.pf_nl[u] = nl; if (p.top) p.pf_nt[u] = nt; }
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
