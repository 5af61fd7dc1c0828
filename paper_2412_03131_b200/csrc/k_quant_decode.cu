// k_quant_decode.cu — the KV compressor's generation step behind dkv_quant_write(DECODE).
//
// One G-lane group per unit, EPL = d/G consecutive elements of K and of V per lane, so each vector is one
// coalesced row per group and the unit's class (hence its bit widths) is uniform inside the group.  Per
// unit, in the order readings Q8/Q9 fix:
//   1. downgrade the victim t_v (v_action == DOWN): dequantize its K8V4 codes from its KV_h slot and
//      re-quantize at K4V2 into KV_l slot v_dst_slot, carrying its score and position — before t_c
//      overwrites that KV_h slot;
//   2. quantize t_c out of window slot (N-1) mod W == p_c mod W at its class bits into tc_slot,
//      score = s_c, position = p_c;
//   3. write the new token into that same window slot (after its old row has been consumed).
//
// What sets the duration (measured, profiles/): the unit count, not the bytes — each unit is a chain of
// dependent memory round trips, followed by the per-vector scalar work (min/max reduction, two correctly
// rounded divisions) that a group does once for all its lanes (several units per warp amortise it):
//   A. everything indexed by u alone: decision word, the unit's qpid record (dkv_classify recorded the
//      existing pages it touches and the request length, dkv_compact_alloc the granted page — in round 1 this
//      kernel read the pages from the tables and the length from the request state, two more dependent
//      trips), s_c and the new token's K/V;
//   B + C. t_c's window row (its slot follows from the length) and the victim's K8V4 record (downgrades
//      only, addressed by the page ID from A), in flight together.
// The window push is issued only after t_c's row has been consumed: a store issued while the same line's
// load miss is outstanding takes a slow path in L2 (measured: 73 -> 26 us at the Llama-3-8B config).
// Quantizer arithmetic is the oracle's (c.5 / Q16), expressed as in dkv_internal.cuh's quant_h16 /
// quant_chunks_f32: packed half2 NaN-propagating min/max, one mixed-precision subtraction, exact
// round-half-away via two round-down adds.
#include <stdlib.h>

#include "dkv_internal.cuh"

namespace dkv {

#ifndef DKV_QD_THREADS
#define DKV_QD_THREADS 224  // 28 units of 8 lanes: 4 CTAs x 224 threads x 72 registers fill the SM's register file
#endif                      // with no spills, and 592 x 28 >= 16384 units take one pass (256: 64 registers, spills)
constexpr int kQDThreads = DKV_QD_THREADS;
#ifndef DKV_QD_LANES
#define DKV_QD_LANES 8     // lanes per unit; measured best at d = 128 (profiles/r1g_quant_decode_compact_ab.log)
#endif
#ifndef DKV_QD_MINB
#define DKV_QD_MINB 4      // CTAs per SM the register budget is sized for (the persistent grid follows it)
#endif

// EPL codes (low byte of ub[i] = code of element i) -> EPL*bits packed bits, element 0 in the LSBs (Q17)
template <int EPL>
__device__ __forceinline__ uint4 pack_codes(const uint32_t (&ub)[EPL], int bits) {
  uint32_t w[4] = {0u, 0u, 0u, 0u};
  if (bits == 8) {
#pragma unroll
    for (int i = 0; i < EPL / 4; i++) w[i] = pack4_lo_bytes(ub[4 * i], ub[4 * i + 1], ub[4 * i + 2], ub[4 * i + 3]);
  } else if (bits == 4) {
    if constexpr (EPL == 4) {
      w[0] = __byte_perm(ub[0], ub[2], 0x0040) | (__byte_perm(ub[1], ub[3], 0x0040) << 4);
    } else {
#pragma unroll
      for (int i = 0; i < EPL / 8; i++) {
        const uint32_t ev = pack4_lo_bytes(ub[8 * i], ub[8 * i + 2], ub[8 * i + 4], ub[8 * i + 6]);
        const uint32_t od = pack4_lo_bytes(ub[8 * i + 1], ub[8 * i + 3], ub[8 * i + 5], ub[8 * i + 7]);
        w[i] = ev | (od << 4);
      }
    }
  } else {                                               // 2 bits
    if constexpr (EPL == 4) {
      w[0] = (ub[0] & 3u) | ((ub[1] & 3u) << 2) | ((ub[2] & 3u) << 4) | ((ub[3] & 3u) << 6);
    } else if constexpr (EPL == 8) {
      uint32_t acc = 0;
#pragma unroll
      for (int m = 0; m < 4; m++) acc |= __byte_perm(ub[m], ub[m + 4], 0x0040) << (2 * m);
      w[0] = acc;
    } else {
#pragma unroll
      for (int i = 0; i < EPL / 16; i++) {
        uint32_t acc = 0;
#pragma unroll
        for (int m = 0; m < 4; m++)
          acc |= pack4_lo_bytes(ub[16 * i + m], ub[16 * i + m + 4], ub[16 * i + m + 8], ub[16 * i + m + 12]) << (2 * m);
        w[i] = acc;
      }
    }
  }
  return make_uint4(w[0], w[1], w[2], w[3]);
}
// store / load this lane's piece (EPL elements = EPL*bits/8 bytes) of a code row
template <int EPL>
__device__ __forceinline__ void store_codes_lane(uint8_t* row, int q, int bits, uint4 v) {
  const int nb = EPL * bits / 8;
  uint8_t* d = row + q * nb;
  if (nb == 16) *reinterpret_cast<uint4*>(d) = v;
  else if (nb == 8) *reinterpret_cast<uint2*>(d) = make_uint2(v.x, v.y);
  else if (nb == 4) *reinterpret_cast<uint32_t*>(d) = v.x;
  else if (nb == 2) *reinterpret_cast<uint16_t*>(d) = (uint16_t)v.x;
  else *d = (uint8_t)v.x;
}
template <int EPL>
__device__ __forceinline__ uint4 load_codes_lane(const uint8_t* row, int q, int bits) {
  const int nb = EPL * bits / 8;
  const uint8_t* s = row + q * nb;
  if (nb == 16) return *reinterpret_cast<const uint4*>(s);
  if (nb == 8) { const uint2 t = *reinterpret_cast<const uint2*>(s); return make_uint4(t.x, t.y, 0u, 0u); }
  if (nb == 4) return make_uint4(*reinterpret_cast<const uint32_t*>(s), 0u, 0u, 0u);
  if (nb == 2) return make_uint4(*reinterpret_cast<const uint16_t*>(s), 0u, 0u, 0u);
  return make_uint4(*s, 0u, 0u, 0u);
}

// this lane's EPL fp16 elements as EPL/2 half2 words
template <int EPL>
struct HVec {
  uint32_t w[EPL / 2];
};
template <int EPL>
__device__ __forceinline__ HVec<EPL> load_hvec(const uint16_t* row, int q) {
  HVec<EPL> h;
  if constexpr (EPL == 4) {
    const uint2 t = *reinterpret_cast<const uint2*>(row + q * 4);
    h.w[0] = t.x; h.w[1] = t.y;
  } else {
#pragma unroll
    for (int i = 0; i < EPL / 8; i++) {
      const uint4 t = *reinterpret_cast<const uint4*>(row + q * EPL + 8 * i);
      h.w[4 * i] = t.x; h.w[4 * i + 1] = t.y; h.w[4 * i + 2] = t.z; h.w[4 * i + 3] = t.w;
    }
  }
  return h;
}
template <int EPL>
__device__ __forceinline__ HVec<EPL> ldg_hvec(const uint16_t* row, int q) {
  HVec<EPL> h;
  if constexpr (EPL == 4) {
    const uint2 t = __ldg(reinterpret_cast<const uint2*>(row + q * 4));
    h.w[0] = t.x; h.w[1] = t.y;
  } else {
#pragma unroll
    for (int i = 0; i < EPL / 8; i++) {
      const uint4 t = ld_nc_v4(row + q * EPL + 8 * i);
      h.w[4 * i] = t.x; h.w[4 * i + 1] = t.y; h.w[4 * i + 2] = t.z; h.w[4 * i + 3] = t.w;
    }
  }
  return h;
}
template <int EPL>
__device__ __forceinline__ void store_hvec(uint16_t* row, int q, const HVec<EPL>& h) {
  if constexpr (EPL == 4) {
    *reinterpret_cast<uint2*>(row + q * 4) = make_uint2(h.w[0], h.w[1]);
  } else {
#pragma unroll
    for (int i = 0; i < EPL / 8; i++)
      *reinterpret_cast<uint4*>(row + q * EPL + 8 * i) =
          make_uint4(h.w[4 * i], h.w[4 * i + 1], h.w[4 * i + 2], h.w[4 * i + 3]);
  }
}

// this lane's EPL fp16 elements of a row -> shared memory with cp.async (no registers held while in flight)
template <int EPL>
__device__ __forceinline__ void stage_row(uint16_t* sdst, const uint16_t* gsrc) {
  if constexpr (EPL == 4) {
    asm volatile("cp.async.ca.shared.global [%0], [%1], 8;" ::"r"(smem_u32(sdst)), "l"(gsrc) : "memory");
  } else {
#pragma unroll
    for (int i = 0; i < EPL / 8; i++)
      asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(smem_u32(sdst + 8 * i)), "l"(gsrc + 8 * i) : "memory");
  }
}
template <int EPL>
__device__ __forceinline__ HVec<EPL> lds_hvec(const uint16_t* s) {
  HVec<EPL> h;
  if constexpr (EPL == 4) {
    const uint2 t = *reinterpret_cast<const uint2*>(s);
    h.w[0] = t.x; h.w[1] = t.y;
  } else {
#pragma unroll
    for (int i = 0; i < EPL / 8; i++) {
      const uint4 t = *reinterpret_cast<const uint4*>(s + 8 * i);
      h.w[4 * i] = t.x; h.w[4 * i + 1] = t.y; h.w[4 * i + 2] = t.z; h.w[4 * i + 3] = t.w;
    }
  }
  return h;
}

// FP16 input, one vector per G-lane group.
template <int G, int EPL>
__device__ __forceinline__ uint4 quant_h16_lane(const HVec<EPL>& x, int bits, unsigned gmask, uint32_t& meta,
                                                bool& ok) {
  const float Qf = (float)((1 << bits) - 1);
  __half2 lo = *reinterpret_cast<const __half2*>(&x.w[0]), hi = lo;
#pragma unroll
  for (int i = 1; i < EPL / 2; i++) {
    const __half2 v = *reinterpret_cast<const __half2*>(&x.w[i]);
    lo = __hmin2_nan(lo, v);
    hi = __hmax2_nan(hi, v);
  }
  __half2 key = __halves2half2(__hmin_nan(__low2half(lo), __high2half(lo)),
                               __hneg(__hmax_nan(__low2half(hi), __high2half(hi))));
#pragma unroll
  for (int o = G / 2; o > 0; o >>= 1) {
    uint32_t k = *reinterpret_cast<uint32_t*>(&key);
    k = __shfl_xor_sync(gmask, k, o);
    key = __hmin2_nan(key, *reinterpret_cast<__half2*>(&k));
  }
  unsigned short mnb = __half_as_ushort(__low2half(key));
  const unsigned short mxb = __half_as_ushort(__hneg(__high2half(key)));
  if ((mnb & 0x7FFFu) == 0) {                           // group-uniform, rare: which zero is the minimum?
    bool negz = false;
#pragma unroll
    for (int i = 0; i < EPL / 2; i++) negz |= ((x.w[i] & 0xFFFFu) == 0x8000u) | ((x.w[i] >> 16) == 0x8000u);
    mnb = __any_sync(gmask, negz) ? 0x8000u : 0x0000u;
  }
  ok = ((mnb & 0x7C00u) != 0x7C00u) && ((mxb & 0x7C00u) != 0x7C00u);
  const float mn = __half2float(__ushort_as_half(mnb)), mx = __half2float(__ushort_as_half(mxb));
  const float s32 = __fdiv_rn(__fsub_rn(mx, mn), Qf);
  const __half s16 = __float2half_rn(s32);
  meta = (uint32_t)__half_as_ushort(s16) | ((uint32_t)mnb << 16);
  const float sf = __half2float(s16);
  const float inv = __frcp_rn(sf);                      // == fdiv_rn(1, sf)
  const float nz = -mn;                                 // z = min exactly (FP16 input)
  uint32_t ub[EPL];
  if (sf >= 6.103515625e-05f) {                         // group-uniform: s16 normal, t <= Q + 1/8, no clamp / mask
#pragma unroll
    for (int i = 0; i < EPL; i++) {
      const float d = mixed_add_h((i & 1) ? (x.w[i >> 1] >> 16) : (x.w[i >> 1] & 0xFFFFu), nz);
      ub[i] = __float_as_uint(__fadd_rd(__fadd_rd(__fmul_rn(d, inv), 0.5f), 8388608.0f));
    }
  } else {
    const float cap = Qf;                               // clamp for a subnormal s16
    const uint32_t zmask = sf != 0.0f ? 0xFFFFFFFFu : 0u;      // s16 == 0: all codes 0
#pragma unroll
    for (int i = 0; i < EPL; i++) {
      const float d = mixed_add_h((i & 1) ? (x.w[i >> 1] >> 16) : (x.w[i >> 1] & 0xFFFFu), nz);
      const float t = fminf(__fmul_rn(d, inv), cap);
      ub[i] = __float_as_uint(__fadd_rd(__fadd_rd(t, 0.5f), 8388608.0f)) & zmask;
    }
  }
  return pack_codes<EPL>(ub, bits);
}

// FP32 input (a dequantized K8V4 token being downgraded, Q9); as quant_chunks_f32.
template <int G, int EPL>
__device__ __forceinline__ uint4 quant_f32_lane(const float (&x)[EPL], int bits, unsigned gmask, uint32_t& meta) {
  const float Qf = (float)((1 << bits) - 1);
  float mn = x[0], mx = x[0];
#pragma unroll
  for (int i = 1; i < EPL; i++) { mn = fminf(mn, x[i]); mx = fmaxf(mx, x[i]); }
#pragma unroll
  for (int o = G / 2; o > 0; o >>= 1) {
    mn = fminf(mn, __shfl_xor_sync(gmask, mn, o));
    mx = fmaxf(mx, __shfl_xor_sync(gmask, mx, o));
  }
  const float s32 = __fdiv_rn(__fsub_rn(mx, mn), Qf);
  const __half s16 = __float2half_rn(s32), z16 = __float2half_rn(mn);
  meta = (uint32_t)__half_as_ushort(s16) | ((uint32_t)__half_as_ushort(z16) << 16);
  const float sf = __half2float(s16), zf = __half2float(z16);
  const float inv = __frcp_rn(sf);
  const uint32_t zmask = sf != 0.0f ? 0xFFFFFFFFu : 0u;
  uint32_t ub[EPL];
#pragma unroll
  for (int i = 0; i < EPL; i++) {
    const float t = fminf(fmaxf(__fmul_rn(__fsub_rn(x[i], zf), inv), 0.0f), Qf);
    ub[i] = __float_as_uint(__fadd_rd(__fadd_rd(t, 0.5f), 8388608.0f)) & zmask;
  }
  return pack_codes<EPL>(ub, bits);
}

// X^ = s*Q + z for this lane's EPL codes
template <int EPL, int BITS>
__device__ __forceinline__ void dequant_lane_ct(const uint4 c, float sf, float zf, float (&x)[EPL]) {
  const uint32_t w[4] = {c.x, c.y, c.z, c.w};
#pragma unroll
  for (int i = 0; i < EPL; i++) {
    constexpr uint32_t Q = (1u << BITS) - 1u;
    const uint32_t q = (w[(i * BITS) >> 5] >> ((i * BITS) & 31)) & Q;
    x[i] = __fadd_rn(__fmul_rn(sf, __uint_as_float(0x4B000000u | q) - 8388608.0f), zf);
  }
}
template <int EPL>
__device__ __forceinline__ void dequant_lane(const uint4 c, int bits, uint32_t meta, float (&x)[EPL]) {
  const float sf = __half2float(__ushort_as_half((unsigned short)(meta & 0xFFFFu)));
  const float zf = __half2float(__ushort_as_half((unsigned short)(meta >> 16)));
  if (bits == 8) dequant_lane_ct<EPL, 8>(c, sf, zf, x);
  else if (bits == 4) dequant_lane_ct<EPL, 4>(c, sf, zf, x);
  else dequant_lane_ct<EPL, 2>(c, sf, zf, x);
}

// Deferred recycle copy of one freed unit by its G-lane group (decode steps that free requests):
// ring[(end0 + off + k) mod P] = table slot k of the unit in canonical slot order (Q13) — slots [0, ph) then
// [L - pl, L) — and the slot is cleared; {off, ph, freed} were recorded by compact_alloc_kernel in p.rec,
// whose marker (freed != 0) is consumed here.
template <int G>
__device__ __forceinline__ void recycle_unit(const PoolDev& p, int u, int q, unsigned gmask, int64_t end0) {
  const int32_t nfr = p.rec[4 * (size_t)u + 2];
  if (nfr == 0) return;                                  // group-uniform
  const int32_t off = p.rec[4 * (size_t)u], ph = p.rec[4 * (size_t)u + 1], pt = p.rec[4 * (size_t)u + 3];
  const int P = p.P;
  const int64_t ring0 = end0 + off;                      // < 2P
  constexpr int kDepth = 8;
  for (int k0 = 0; k0 < nfr; k0 += G * kDepth) {
    int32_t pid[kDepth];
#pragma unroll
    for (int j = 0; j < kDepth; j++) {
      const int k = k0 + G * j + q;
      pid[j] = k < nfr ? __ldcg(freed_slot(p, u, k, pt, ph, nfr)) : -1;
    }
#pragma unroll
    for (int j = 0; j < kDepth; j++) {
      const int k = k0 + G * j + q;
      if (k < nfr) {
        int64_t pos = ring0 + k;                         // < 3P: two conditional wraps, no division
        pos -= pos >= P ? P : 0;
        pos -= pos >= P ? P : 0;
        p.ring[pos] = pid[j];
        int32_t empty = -1;                              // clear only after the load returned (see the header)
        asm volatile("" : "+r"(empty) : "r"(pid[j]));
        *freed_slot(p, u, k, pt, ph, nfr) = empty;
      }
    }
  }
  __syncwarp(gmask);
  if (q == 0) p.rec[4 * (size_t)u + 2] = 0;
}

// TOP: the pool has the NEXT-4 FP16 tier (its branches compiled out otherwise)
template <int D, int G, bool TOP>
__global__ void __launch_bounds__(kQDThreads, DKV_QD_MINB)
quant_decode_kernel(PoolDev p, const dkv_decision_t* __restrict__ dec, const uint16_t* __restrict__ knew,
                    const uint16_t* __restrict__ vnew, const float* __restrict__ cand_sig, int u0, int u1, int upc) {
  constexpr int EPL = D / G;                             // elements per lane per vector
  // upc <= kQDThreads / G units per CTA per iteration (the launch balances them over the resident CTAs); the
  // groups beyond upc have no unit
  const int gslot = threadIdx.x / G;
  // this lane's part of the new token's K / V rows [0] [1] and of t_c's window K / V rows [2] [3], staged by
  // cp.async so no registers are held across the downgrade while they are in flight
  __shared__ __align__(16) uint16_t s_new[4][kQDThreads * EPL];
  __shared__ int32_t s_status;
  const int lane = threadIdx.x & 31;
  const int q = lane % G;
  const unsigned gmask = G == 32 ? kFull : (((1u << G) - 1u) << (lane & ~(G - 1)));
  __shared__ int32_t s_rec;
  __shared__ int64_t s_end0;
  pdl_wait();                                            // (PDL) everything below reads what compact_alloc wrote
  pdl_trigger();
  if (threadIdx.x == 0) {
    s_status = p.ctrl->qw_status;                        // entry status (Q36), left by dkv_compact_alloc
    s_rec = ld_volatile(&p.ctrl->rec_deferred);          // compact_alloc left this step's recycle copies to us
    s_end0 = ld_volatile(&p.ctrl->rec_end0);
  }
  // the first unit's record and decision are u-indexed: in flight across the barrier
  int ub = blockIdx.x;
  int4 dw = make_int4(0, -1, -1, -1), qp = make_int4(-1, -1, 0, 0);
  {
    const int uf = u0 + ub * upc + gslot;
    if (gslot < upc && uf < u1) { dw = __ldg(reinterpret_cast<const int4*>(dec) + uf); qp = __ldg(p.qpid + uf); }
  }
  __syncthreads();
  const bool dead = s_status != 0;                       // error at entry: no quantization, no window push
  const bool rec_on = s_rec != 0;
  if (dead && !rec_on) return;
  uint16_t* const my_nk = &s_new[0][threadIdx.x * EPL];
  uint16_t* const my_nv = &s_new[1][threadIdx.x * EPL];
  uint16_t* const my_wk = &s_new[2][threadIdx.x * EPL];
  uint16_t* const my_wv = &s_new[3][threadIdx.x * EPL];

  for (; gslot < upc && u0 + ub * upc < u1; ub += gridDim.x) {   // units [u0, u1)
    const int u = u0 + ub * upc + gslot;
    if (u >= u1) break;                                  // whole groups leave together (last block only)
    if (ub != (int)blockIdx.x) { dw = __ldg(reinterpret_cast<const int4*>(dec) + u); qp = __ldg(p.qpid + u); }
    // the request length (already including this step's token: dkv_compact_alloc advanced it), 0 when the
    // request is not ACTIVE — recorded by dkv_classify in the unit's qpid record, so no request state is read
    const int N = qp.z;
    const bool live = N > 0;
    if (!live) {
      // a unit of a request this step's dkv_compact_alloc recycled without copying (decode fast path): its
      // page IDs go to the ring here, at the offsets the scan assigned (Q13 order), and its slots are cleared
      if (rec_on) recycle_unit<G>(p, u, q, gmask, s_end0);
      continue;
    }
    if (dead) continue;

    // ---- A: the loads indexed by u (the decision and the qpid record, above; t_c's significance and the new
    // token, straight to shared memory) and, one round trip later, by the request length: t_c's window row —
    // in flight together with the victim's record (C)
    const float s_in_given = cand_sig ? __ldg(cand_sig + u) : 0.0f;
    stage_row<EPL>(my_nk, knew + (size_t)u * D + q * EPL);
    stage_row<EPL>(my_nv, vnew + (size_t)u * D + q * EPL);
    uint16_t* wk_row = nullptr;
    uint16_t* wv_row = nullptr;
    int ws = 0;
    if (p.W > 0 && live) {
      ws = fmod_(p.div_W, N - 1);
      wk_row = reinterpret_cast<uint16_t*>(p.win_k) + ((size_t)u * p.W + ws) * D;
      wv_row = reinterpret_cast<uint16_t*>(p.win_v) + ((size_t)u * p.W + ws) * D;
      stage_row<EPL>(my_wk, wk_row + q * EPL);
      stage_row<EPL>(my_wv, wv_row + q * EPL);
    }
    cp_async_commit();
    // t_c's significance: given, or (NEXT-2, cand_sig NULL) the running mean kept for its window slot
    const float s_in = cand_sig ? s_in_given : (p.W > 0 && live ? p.win_sig[(size_t)u * p.W + ws] : 0.0f);
    const int pc = N - 1 - p.W;
    const int tc_class = dw.x & 0xFF, v_action = (dw.x >> 8) & 0xFF;
    const int v_slot = dw.y, tc_slot = dw.z, v_dst = dw.w;
    const bool has_tc = live && (tc_class == DKV_CLS_HIGH || tc_class == DKV_CLS_LOW || tc_class == DKV_CLS_TOP);
    const bool down = live && v_action == DKV_V_DOWN;
    const bool tc_high = tc_class == DKV_CLS_HIGH, tc_top = TOP && tc_class == DKV_CLS_TOP;
    const int tc_pg = fdiv(tc_top ? p.div_Ct : (tc_high ? p.div_Ch : p.div_Cl), tc_slot);
    const int pid_tc = qp.x, pid_src = qp.x, pid_dst = qp.y;   // the victim's KV_h slot is t_c's slot (Q8)


    // ---- C + 1. NEXT-4 (Q42): a TOP victim's fp16 rows quantized at the class it moves to (grow)
    if (down && tc_top) {                                // group-uniform
      const ClassGeom gt = p.gt, go = geom_of(p, dw.x >> 16 & 0xFF);
      const int is = fmod_(p.div_Ct, v_slot);
      const int id = fmod_((((dw.x >> 16) & 0xFF) == DKV_GROW_HIGH) ? p.div_Ch : p.div_Cl, v_dst);
      const uint8_t* src = p.pages + (size_t)pid_src * (size_t)p.page_bytes;
      uint8_t* dst = p.pages + (size_t)pid_dst * (size_t)p.page_bytes;
      const HVec<EPL> xk = load_hvec<EPL>(reinterpret_cast<const uint16_t*>(src + gt.off_k + is * gt.k_row), q);
      const HVec<EPL> xv = load_hvec<EPL>(reinterpret_cast<const uint16_t*>(src + gt.off_v + is * gt.v_row), q);
      uint32_t carry = 0;                                // lane 2: score bits, lane 3: position
      if (q == 2) carry = *reinterpret_cast<const uint32_t*>(src + gt.off_score + 4 * is);
      if (q == 3) carry = *reinterpret_cast<const uint32_t*>(src + gt.off_pos + 4 * is);
      uint32_t mk, mv;
      bool fk, fv;                                       // stored TOP rows are finite (Q30 at insertion)
      const uint4 pk = quant_h16_lane<G, EPL>(xk, go.kbits, gmask, mk, fk);
      const uint4 pv = quant_h16_lane<G, EPL>(xv, go.vbits, gmask, mv, fv);
      store_codes_lane<EPL>(dst + go.off_k + id * go.k_row, q, go.kbits, pk);
      store_codes_lane<EPL>(dst + go.off_v + id * go.v_row, q, go.vbits, pv);
      if (q == 0) *reinterpret_cast<uint32_t*>(dst + go.off_kmeta + 4 * id) = mk;
      if (q == 1) *reinterpret_cast<uint32_t*>(dst + go.off_vmeta + 4 * id) = mv;
      if (q == 2) *reinterpret_cast<uint32_t*>(dst + go.off_score + 4 * id) = carry;
      if (q == 3) *reinterpret_cast<uint32_t*>(dst + go.off_pos + 4 * id) = carry;
      __syncwarp(gmask);                                 // every lane's read of t_v precedes t_c's stores
    } else
    // ---- C + 1. downgrade t_v: K8V4 -> K4V2 (Q9)
    if (down) {                                          // group-uniform
      const ClassGeom gh = p.g[1], go = p.g[2];
      const int is = fmod_(p.div_Ch, v_slot), id = fmod_(p.div_Cl, v_dst);
      const uint8_t* src = p.pages + (size_t)pid_src * (size_t)p.page_bytes;
      uint8_t* dst = p.pages + (size_t)pid_dst * (size_t)p.page_bytes;
      const uint4 ck = load_codes_lane<EPL>(src + gh.off_k + is * gh.k_row, q, gh.kbits);
      const uint4 cv = load_codes_lane<EPL>(src + gh.off_v + is * gh.v_row, q, gh.vbits);
      const uint32_t kmeta = *reinterpret_cast<const uint32_t*>(src + gh.off_kmeta + 4 * is);
      const uint32_t vmeta = *reinterpret_cast<const uint32_t*>(src + gh.off_vmeta + 4 * is);
      uint32_t carry = 0;                                // lane 2: score bits, lane 3: position
      if (q == 2) carry = *reinterpret_cast<const uint32_t*>(src + gh.off_score + 4 * is);
      if (q == 3) carry = *reinterpret_cast<const uint32_t*>(src + gh.off_pos + 4 * is);
#pragma unroll 1
      for (int kv = 0; kv < 2; kv++) {
        float x[EPL];
        dequant_lane<EPL>(kv ? cv : ck, kv ? gh.vbits : gh.kbits, kv ? vmeta : kmeta, x);
        uint32_t m2;
        const int db = kv ? go.vbits : go.kbits;
        const uint4 pk = quant_f32_lane<G, EPL>(x, db, gmask, m2);
        store_codes_lane<EPL>(dst + (kv ? go.off_v + id * go.v_row : go.off_k + id * go.k_row), q, db, pk);
        if (q == kv) *reinterpret_cast<uint32_t*>(dst + (kv ? go.off_vmeta : go.off_kmeta) + 4 * id) = m2;
      }
      if (q == 2) *reinterpret_cast<uint32_t*>(dst + go.off_score + 4 * id) = carry;
      if (q == 3) *reinterpret_cast<uint32_t*>(dst + go.off_pos + 4 * id) = carry;
      __syncwarp(gmask);                                 // every lane's read of t_v precedes t_c's stores
    }

    // ---- 2. t_c -> its section slot at its class bits
    cp_async_wait<0>();                                  // this lane's part of the new token and t_c's row are in smem
    bool rejected = false;                               // Q30: a non-finite t_c leaves slot and window as they are
    if (has_tc) {                                        // group-uniform
      const HVec<EPL> wk = lds_hvec<EPL>(p.W == 0 ? my_nk : my_wk);   // W == 0: t_c is the new token
      const HVec<EPL> wv = lds_hvec<EPL>(p.W == 0 ? my_nv : my_wv);
      if (tc_top) {                                      // NEXT-4 (Q40): t_c kept as its fp16 rows
        bool fin = true;
#pragma unroll
        for (int i = 0; i < EPL / 2; i++) {
          fin &= ((wk.w[i] & 0x7C00u) != 0x7C00u) && ((wk.w[i] & 0x7C000000u) != 0x7C000000u);
          fin &= ((wv.w[i] & 0x7C00u) != 0x7C00u) && ((wv.w[i] & 0x7C000000u) != 0x7C000000u);
        }
        if ((__ballot_sync(gmask, !fin) & gmask) != 0u) {                       // Q30: rejected whole
          if (q == 0) set_status(p.ctrl, DKV_ERR_NONFINITE);
          rejected = true;
        } else {
          const ClassGeom gt = p.gt;
          const int idx = tc_slot - tc_pg * gt.C;
          uint8_t* pg = p.pages + (size_t)pid_tc * (size_t)p.page_bytes;
          store_hvec<EPL>(reinterpret_cast<uint16_t*>(pg + gt.off_k + idx * gt.k_row), q, wk);
          store_hvec<EPL>(reinterpret_cast<uint16_t*>(pg + gt.off_v + idx * gt.v_row), q, wv);
          if (q == 2) *reinterpret_cast<float*>(pg + gt.off_score + 4 * idx) = canon_zero(s_in);
          if (q == 3) *reinterpret_cast<int32_t*>(pg + gt.off_pos + 4 * idx) = pc;
        }
      } else {
      const ClassGeom g = geom_of(p, tc_class);
      uint32_t mk, mv;
      bool fk, fv;
      const uint4 pk = quant_h16_lane<G, EPL>(wk, g.kbits, gmask, mk, fk);
      const uint4 pv = quant_h16_lane<G, EPL>(wv, g.vbits, gmask, mv, fv);
      if (!(fk && fv)) {
        if (q == 0) set_status(p.ctrl, DKV_ERR_NONFINITE);
        rejected = true;
      } else {
        const int idx = tc_slot - tc_pg * g.C;
        uint8_t* pg = p.pages + (size_t)pid_tc * (size_t)p.page_bytes;
        store_codes_lane<EPL>(pg + g.off_k + idx * g.k_row, q, g.kbits, pk);
        store_codes_lane<EPL>(pg + g.off_v + idx * g.v_row, q, g.vbits, pv);
        if (q == 0) *reinterpret_cast<uint32_t*>(pg + g.off_kmeta + 4 * idx) = mk;
        if (q == 1) *reinterpret_cast<uint32_t*>(pg + g.off_vmeta + 4 * idx) = mv;
        if (q == 2) *reinterpret_cast<float*>(pg + g.off_score + 4 * idx) = canon_zero(s_in);
        if (q == 3) *reinterpret_cast<int32_t*>(pg + g.off_pos + 4 * idx) = pc;
      }
      }
    }
    // 3. window push, after t_c's row has been consumed
    if (live && q == 0) p.secmin[8 * (size_t)u + 6] = 0;    // section minima of dkv_attend no longer valid
    if (wk_row != nullptr && !rejected) {
      store_hvec<EPL>(wk_row, q, lds_hvec<EPL>(my_nk));
      store_hvec<EPL>(wv_row, q, lds_hvec<EPL>(my_nv));
      if (q == 0) p.win_sig[(size_t)u * p.W + fmod_(p.div_W, N - 1)] = 0.0f;   // the new token (Q33)
    }
  }
}

template <int D, int G, bool TOP>
static cudaError_t launch_qd_t(const PoolDev& p, const dkv_decision_t* dec, const uint16_t* k, const uint16_t* v,
                             const float* sig, int u0, int u1, cudaStream_t s) {
  constexpr int units_per_cta = kQDThreads / G;
  const size_t smem = 0;
  static int cap = 0;                                    // persistent grid (per template instance)
  if (cap == 0) cap = persistent_grid(quant_decode_kernel<D, G, TOP>, kQDThreads, 0);
  if (cap == 0) return cudaErrorUnknown;
  if (u1 <= u0) return cudaSuccess;
  // every resident CTA takes the same number of units (at most units_per_cta): 16384 units over 592 CTAs is 28
  // per CTA and 112 per SM, where full 32-unit CTAs put 128 units on some SMs and 96 on others
  int upc = (u1 - u0 + cap - 1) / cap;
  if (upc > units_per_cta) upc = units_per_cta;
  const int need = (u1 - u0 + upc - 1) / upc;
  return launch_ex(quant_decode_kernel<D, G, TOP>, dim3(need < cap ? need : cap), dim3(kQDThreads), smem, s, p.pdl != 0, p,
                   dec, k, v, sig, u0, u1, upc);
}

template <int D, int G>
static cudaError_t launch_qd(const PoolDev& p, const dkv_decision_t* dec, const uint16_t* k, const uint16_t* v,
                             const float* sig, int u0, int u1, cudaStream_t s) {
  return p.top ? launch_qd_t<D, G, true>(p, dec, k, v, sig, u0, u1, s) : launch_qd_t<D, G, false>(p, dec, k, v, sig, u0, u1, s);
}

cudaError_t launch_quant_decode(const PoolDev& p, const dkv_decision_t* dec, const uint16_t* k, const uint16_t* v,
                                const float* sig, cudaStream_t s, int u0, int u1) {
  if (u1 < 0) u1 = p.U;
  constexpr int g = DKV_QD_LANES;                       // lanes per unit (build-time choice)
  if (p.d == 128) {
    if (g == 32) return launch_qd<128, 32>(p, dec, k, v, sig, u0, u1, s);
    if (g == 8) return launch_qd<128, 8>(p, dec, k, v, sig, u0, u1, s);
    return launch_qd<128, 16>(p, dec, k, v, sig, u0, u1, s);
  }
  if (g == 16) return launch_qd<64, 16>(p, dec, k, v, sig, u0, u1, s);
  if (g == 4) return launch_qd<64, 4>(p, dec, k, v, sig, u0, u1, s);
  return launch_qd<64, 8>(p, dec, k, v, sig, u0, u1, s);
}

}  // namespace dkv
