// k_attend_tc.cu — NEXT-2 on tensor cores: decode attention over the compressed cache (Eq. 1; GQA
// score = max over the group), the running-mean significance update (Q33/Q34) and the section
// minima for the next dkv_classify, with the two contractions (QK^T, PV) on the tensor cores
// (mma.sync.m16n8k16, fp32 accumulation).  Behind dkv_attend_tc; the exact path (k_attend.cu, bit-identical to
// the oracle) stays the parity mode.
//
// The contractions are taken on the integer codes, not on dequantized values, so the tensor-core operands are
// exact and only fp32 accumulation rounds:
//   logit(t, h) = (s_t * sum_f q_hf code_tf + z_t * sum_f q_hf) / sqrt(d)       (X^ = s*Q + z)
//   out(h, f)   = sum_t (a_ht s_t) code_tf + sum_t a_ht z_t
// Codes are < 2^8, so they are exact in fp16; the queries are fp16 inputs (exact); a_ht s_t is an fp32 value,
// scaled by 2^12 and split into fp16 hi + lo (22 significant bits).  The FP16 window (<= W tokens) runs on CUDA
// cores in fp32.
//
// One pass over the pages (round 2, r2n): the heads are the MMA's M dimension, so the QK^T accumulator of a
// 16-token chunk (rows = heads, columns = tokens) is, after the softmax arithmetic, already the A operand of
// that chunk's PV (rows = heads, k = tokens) — no logit round trip through memory between the contractions.
// The softmax is the online (running-max) form: each warp keeps, per head, a running maximum m, sum Z and
// output accumulator rescaled when m grows; the warps' states and the window's are merged at the end.  The
// hi and lo parts of the PV weights are M rows 0-7 and 8-15 of the same MMA (G <= 8), so the split costs no
// extra MMA.  The logits (log2 units) still go to the CTA's scratch slot, once, for the significance pass that
// needs the final per-head maximum and sum.
//
// One CTA per unit (the paper's "one thread block per head") of kTcWarps warps; pages go round-robin to
// the warps, high pages first, then low.  A page's K codes, K meta, V codes and V meta are one
// contiguous prefix of the page (§4 layout) and are staged by ONE bulk copy (TMA, cp.async.bulk, L2
// evict-first) into the warp's ring of kTcStages stages.  The MMA fragments are read straight from the staged
// rows; the paper's tiled K/V layouts (NEXT-3) exist to make per-thread vector loads coalesce in
// global memory — here whole page prefixes are copied (coalesced by construction) and the tiling is a
// permutation of the MMA k / n indices, chosen so that a lane's codes for every k-step are one contiguous run
// of its row (keys: lane tig holds features (d/4) tig + 4g .. 4g+3 of k-step g; values: lane grp holds
// features (d/8) grp + nt of n-tile nt) — the paper's K_vec / V_vec vectorisation at the register level.
#include <type_traits>

#include "dkv_internal.cuh"

namespace dkv {

#ifndef DKV_TC_WARPS
#define DKV_TC_WARPS 4          // warps per CTA (one unit per CTA)
#endif
#ifndef DKV_TC_STAGES
#define DKV_TC_STAGES 2         // pages in flight per warp (measured: 2 beats 3, tools/tc_ab.sh, profiles/r2o_tc_ab.log)
#endif
#ifndef DKV_TC_K8_BIASED
#define DKV_TC_K8_BIASED 0      // K8 key operands left at 1024 + c (the bias folded into z): A/B of precision and time
#endif
#ifndef DKV_TC_MAXNREG
#define DKV_TC_MAXNREG 128   // register cap without a min-blocks hint (4 CTAs/SM all the same): ptxas schedules
#endif                       // it better than __launch_bounds__(128, 4), 2.374 -> 2.350 ms (tools/tc_ab.sh)
#ifndef DKV_TC_MINB
#define DKV_TC_MINB 4           // CTAs per SM the register budget is sized for
#endif
constexpr int kTcWarps = DKV_TC_WARPS;
constexpr int kTcThreads = kTcWarps * 32;
constexpr int kTcStages = DKV_TC_STAGES;
constexpr float kLog2e = 1.4426950408889634f;

template <int I, int N, class F>
__device__ __forceinline__ void static_for(F&& f) {
  if constexpr (I < N) {
    f(std::integral_constant<int, I>{});
    static_for<I + 1, N>(f);
  }
}

__device__ __forceinline__ void mma_f16(float (&d)[4], uint32_t a0, uint32_t a1, uint32_t a2, uint32_t a3, uint32_t b0,
                                        uint32_t b1) {
  asm volatile("mma.sync.aligned.m16n8k16.row.col.f32.f16.f16.f32 {%0,%1,%2,%3}, {%4,%5,%6,%7}, {%8,%9}, "
               "{%0,%1,%2,%3};"
               : "+f"(d[0]), "+f"(d[1]), "+f"(d[2]), "+f"(d[3])
               : "r"(a0), "r"(a1), "r"(a2), "r"(a3), "r"(b0), "r"(b1));
}
__device__ __forceinline__ void mbar_wait_u32(uint32_t bar, uint32_t parity) {
  asm volatile(
      "{\n"
      ".reg .pred P1;\n"
      "WAIT_%=:\n"
      "mbarrier.try_wait.parity.shared::cta.b64 P1, [%0], %1;\n"
      "@!P1 bra WAIT_%=;\n"
      "}\n" ::"r"(bar), "r"(parity) : "memory");
}
__device__ __forceinline__ float ex2(float x) {
  float y;
  asm("ex2.approx.ftz.f32 %0, %1;" : "=f"(y) : "f"(x));
  return y;
}

// Exact code -> fp16 conversion with byte permutes: a w-bit field whose lowest bit sits at mantissa bit b of a
// half with exponent chosen so that that bit weighs exactly 1 (magic M) holds the value M + code; one
// subtraction (exact) leaves the code.  Centred codes: the subtrahend is M + 2^(bits-1), so the operand is the
// code minus half its range (exact in fp16) and the offset moves into z (z' = z + 2^(bits-1) s, tc_zc).  The
// code term and the z term of the output (and of the logit) then no longer nearly cancel — with raw codes both
// are ~|mean V| and their difference is the output, and the tensor core's fp32 accumulation error over a long
// context was amplified into it.
__device__ __forceinline__ uint32_t hsub2_u(uint32_t x, uint32_t m) {
  const __half2 r = __hsub2(*reinterpret_cast<const __half2*>(&x), *reinterpret_cast<const __half2*>(&m));
  return *reinterpret_cast<const uint32_t*>(&r);
}
// (x & MASK) | magic in one LOP3 (the magic lives in a register)
template <uint32_t MASK>
__device__ __forceinline__ uint32_t and_or(uint32_t x, uint32_t magic) {
  uint32_t d;
  asm("lop3.b32 %0, %1, %2, %3, 0xEA;" : "=r"(d) : "r"(x), "n"(MASK), "r"(magic));
  return d;
}
template <int BITS>
__device__ __forceinline__ float tc_zc(float zf, float sf) { return fmaf(sf, (float)(1 << (BITS - 1)), zf); }
// K8: bytes (c0, c1, c2, c3) of x -> fp16x2 (c0, c1) and (c2, c3), centred: (1024 + c) - 1152 = c - 128
__device__ __forceinline__ void k8_pairs(uint32_t x, uint32_t& lo, uint32_t& hi) {
  lo = hsub2_u(__byte_perm(x, 0x64646464u, 0x4140), 0x64806480u);
  hi = hsub2_u(__byte_perm(x, 0x64646464u, 0x4342), 0x64806480u);
}
// K4: the two bytes at byte index KB0 (codes n0 | n1 << 4) and KB0 + 1 (n2 | n3 << 4) of x -> fp16x2 (n0, n1),
// (n2, n3): n0 in bits 0-3 with 0x6400 (1024, ulp 1), n1 in bits 20-23 = bits 4-7 of the high half with 0x5400
// (64, ulp 1/16); centred: c - 8
template <int KB0>
__device__ __forceinline__ void k4_pairs(uint32_t x, uint32_t& lo, uint32_t& hi) {
  constexpr uint32_t s0 = KB0 * 0x1111u, s1 = (KB0 + 1) * 0x1111u;
  lo = hsub2_u(and_or<0x00F0000Fu>(__byte_perm(x, 0u, s0), 0x54006400u), 0x54806408u);
  hi = hsub2_u(and_or<0x00F0000Fu>(__byte_perm(x, 0u, s1), 0x54006400u), 0x54806408u);
}
// V: byte K of x (token j0) and of y (token j1) -> fp16x2 (field of j0, field of j1) for the field at bits
// [SH, SH + VB) of that byte, centred; the magic makes bit SH weigh 1 (fp16, 10 mantissa bits: a value in
// [2^e, 2^(e+1)) has ulp 2^(e-10), so e = 10 - SH: 1024 (0x6400) for SH = 0, 256 (0x5C00) for 2, 64 (0x5400)
// for 4, 16 (0x4C00) for 6)
template <int K, int SH, int VB>
__device__ __forceinline__ uint32_t v_pair(uint32_t x, uint32_t y) {
  constexpr uint32_t sel = K | (K << 4) | ((4 + K) << 8) | ((4 + K) << 12);
  constexpr uint32_t mask = (((1u << VB) - 1u) << SH) * 0x00010001u;
  constexpr uint32_t magic = (SH == 0 ? 0x6400u : SH == 2 ? 0x5C00u : SH == 4 ? 0x5400u : 0x4C00u) * 0x00010001u;
  constexpr uint32_t centre = magic + ((1u << (VB - 1)) << SH) * 0x00010001u;
  return hsub2_u(and_or<mask>(__byte_perm(x, y, sel), magic), centre);
}
// fp32 pair -> fp16x2 hi parts and the fp16x2 of the remainders (x = hi + lo to 22 significant bits)
__device__ __forceinline__ void h2_split(float x0, float x1, uint32_t& hi, uint32_t& lo) {
  const __half2 h = __floats2half2_rn(x0, x1);
  const float2 hf = __half22float2(h);
  const __half2 l = __floats2half2_rn(x0 - hf.x, x1 - hf.y);
  hi = *reinterpret_cast<const uint32_t*>(&h);
  lo = *reinterpret_cast<const uint32_t*>(&l);
}
// The running maximum m moves lazily: only when a chunk's maximum exceeds it by more than kTau (log2 units), so
// p = 2^(l - m) <= 2^kTau (unnormalised: 1/Z is applied at the end).  PV's weights p * s_v are scaled by
// kPvScale = 2^(12 - kTau) before their fp16 split — p * kPvScale <= 2^12 and |s_v| < 2^4 keep them below the
// fp16 maximum, and small probabilities do not sink into fp16 subnormals; the accumulators are scaled back once.
// (An eager rescale on every new maximum ran on ~40 % of the chunks: 36 multiplies each.)
constexpr float kTau = 8.0f;
constexpr float kPvScale = 16.0f, kPvUnscale = 1.0f / 16.0f;

// Compile-time geometry of one precision class (the paper's K8V4 high / K4V2 low pages): tokens per
// page, bit widths, code row bytes, and the offsets of the staged prefix (K codes, K meta, V codes, V meta —
// the §4 page layout, checked by attend_tc_supported).
template <int D, int C_, int KB, int VB>
struct TcCls {
  static constexpr int C = C_, kbits = KB, vbits = VB;
  static constexpr int k_row = D * KB / 8, v_row = D * VB / 8;
  static constexpr int off_kmeta = C * k_row, off_v = off_kmeta + 4 * C, off_vmeta = off_v + C * v_row;
  static constexpr int prefix = off_vmeta + 4 * C;                    // bytes staged per page (16-B multiple)
  static constexpr int rbk = D / 4 * KB / 8, rbv = D / 8 * VB / 8;     // a lane's run per key / value row
};
template <int D>
constexpr int tc_stage_bytes() {
  return (((TcCls<D, 16, 8, 4>::prefix > TcCls<D, 32, 4, 2>::prefix ? TcCls<D, 16, 8, 4>::prefix
                                                                     : TcCls<D, 32, 4, 2>::prefix) + 127) & ~127);
}
// the merge area reuses the stages: [kTcWarps][G][D] fp32 warp partials
__host__ __device__ constexpr int tc_area_bytes(int D, int G, int stage) {
  return kTcWarps * kTcStages * stage > kTcWarps * G * D * 4 ? kTcWarps * kTcStages * stage : kTcWarps * G * D * 4;
}

// `BYTES` contiguous bytes of a staged row at byte `b0` into 32-bit words (BYTES in {2, 4, 8, 16, 32})
template <int BYTES>
__device__ __forceinline__ void lds_run(const uint8_t* p, uint32_t (&w)[(BYTES + 3) / 4]) {
  if constexpr (BYTES >= 16) {
#pragma unroll
    for (int c = 0; c < BYTES / 16; c++) {
      const uint4 v = *reinterpret_cast<const uint4*>(p + 16 * c);
      w[4 * c] = v.x; w[4 * c + 1] = v.y; w[4 * c + 2] = v.z; w[4 * c + 3] = v.w;
    }
  } else if constexpr (BYTES == 8) {
    const uint2 v = *reinterpret_cast<const uint2*>(p);
    w[0] = v.x; w[1] = v.y;
  } else if constexpr (BYTES == 4) {
    w[0] = *reinterpret_cast<const uint32_t*>(p);
  } else {
    w[0] = *reinterpret_cast<const uint16_t*>(p);
  }
}

// Per-warp online-softmax state of one unit, for this lane's heads 2 tig and 2 tig + 1: running maxima (log2
// units), sums of p and of p z' over this lane's tokens, and the output accumulators (PV: M = features, N = heads;
// m-tile mt, rows grp / grp + 8 = features (D/8) grp + 2 mt / + 1, columns 2 tig / 2 tig + 1 = heads)
template <int D>
struct TcState {
  float o[D / 16][4];
  float m[2], z[2], zs[2];
};

__device__ __forceinline__ uint32_t movm_trans(uint32_t x) {
  uint32_t y;
  asm volatile("movmatrix.sync.aligned.m8n8.trans.b16 %0, %1;" : "=r"(y) : "r"(x));
  return y;
}

// The online softmax update and PV of one 16-token chunk, given its logits l (log2 units; [rr][c] = token grp +
// 8 rr, head 2 tig + c; -inf for an absent token or head), each token's V scale svs = s_v * kPvScale and centred
// zero point zv (both 0 for an absent token).  `va(mt, a0, a1, a2, a3)` builds PV's A fragment of m-tile mt
// (m = features (D/8) grp + 2 mt | + 1, k = tokens 2 tig, 2 tig + 1 | + 8).
template <int D, class VA>
__device__ __forceinline__ void tc_softmax_pv(const float (&l)[4], const float (&svs)[2], const float (&zv)[2],
                                              TcState<D>& st, VA&& va) {
  // running maximum of heads 2 tig, 2 tig + 1, moved only by more than kTau: the lane-local test decides whether
  // any lane needs it; only then is the chunk maximum reduced over the 8 lanes (grp) holding each head
  float pm[2] = {fmaxf(l[0], l[2]), fmaxf(l[1], l[3])};
  if (__any_sync(kFull, (pm[0] > st.m[0] + kTau) | (pm[1] > st.m[1] + kTau))) {
#pragma unroll
    for (int c = 0; c < 2; c++) {
      pm[c] = fmaxf(pm[c], __shfl_xor_sync(kFull, pm[c], 4));
      pm[c] = fmaxf(pm[c], __shfl_xor_sync(kFull, pm[c], 8));
      pm[c] = fmaxf(pm[c], __shfl_xor_sync(kFull, pm[c], 16));
    }
    const bool up0 = pm[0] > st.m[0] + kTau, up1 = pm[1] > st.m[1] + kTau;
    const float mn0 = up0 ? pm[0] : st.m[0], mn1 = up1 ? pm[1] : st.m[1];
    const float f0 = ex2(st.m[0] - mn0), f1 = ex2(st.m[1] - mn1);   // 1 when unchanged, 0 from -inf
#pragma unroll
    for (int mt = 0; mt < D / 16; mt++) {
      st.o[mt][0] *= f0; st.o[mt][1] *= f1; st.o[mt][2] *= f0; st.o[mt][3] *= f1;
    }
    st.z[0] *= f0; st.z[1] *= f1;
    st.zs[0] *= f0; st.zs[1] *= f1;
    st.m[0] = mn0; st.m[1] = mn1;
  }
  // weights w = p s_v kPvScale (rows = tokens, columns = heads), split fp16 hi / lo and transposed to PV's B
  // operand (k = tokens 2 tig, 2 tig + 1 | + 8, n = head grp)
  float wv[4];
#pragma unroll
  for (int rr = 0; rr < 2; rr++)
#pragma unroll
    for (int c = 0; c < 2; c++) {
      const float p = ex2(l[2 * rr + c] - st.m[c]);     // 0 for an absent token / head (l = -inf)
      st.z[c] += p;
      st.zs[c] = fmaf(p, zv[rr], st.zs[c]);
      wv[2 * rr + c] = p * svs[rr];
    }
  uint32_t h01, l01, h23, l23;
  h2_split(wv[0], wv[1], h01, l01);                      // token grp: heads (2 tig, 2 tig + 1)
  h2_split(wv[2], wv[3], h23, l23);                      // token grp + 8
  const uint32_t bh0 = movm_trans(h01), bh1 = movm_trans(h23), bl0 = movm_trans(l01), bl1 = movm_trans(l23);
  static_for<0, D / 16>([&](auto mti) {
    uint32_t a0, a1, a2, a3;
    va(mti, a0, a1, a2, a3);
    mma_f16(st.o[decltype(mti)::value], a0, a1, a2, a3, bh0, bh1);
    mma_f16(st.o[decltype(mti)::value], a0, a1, a2, a3, bl0, bl1);
  });
}

// One 16-token chunk of a staged page: QK^T (M = the chunk's tokens, N = heads, K = features), logits to the
// scratch rows, then tc_softmax_pv (PV: M = features, N = heads, K = tokens; its B operand — the weights — is the
// QK accumulator layout transposed in registers by movmatrix).  `lgl` = this lane's logit pointer (row 0, column
// 2 tig); `row0` = the page's first scratch row; `cnt` = valid tokens of the page (tokens 16 ch + i < cnt).
template <int D, int G, int GP, class CL>
__device__ __forceinline__ void tc_chunk(const uint8_t* seg, int ch, int cnt, const uint32_t (&qb)[D / 16][2],
                                         const float (&qsz)[2], float scale2, float* lgl, int row0,
                                         TcState<D>& st, int grp, int tig) {
  constexpr int NG = D / 16;
  constexpr int NWK = CL::rbk / 4, NWV = (CL::rbv + 3) / 4;
  // ---- QK^T: A = key codes (rows = tokens grp, grp + 8; k = features FPK tig + 4g + {0, 1 | 2, 3}),
  // B = queries (k = the same features, n = head grp); two MMA chains (even / odd k-steps)
  float acc2[2][4] = {{0.f, 0.f, 0.f, 0.f}, {0.f, 0.f, 0.f, 0.f}};
  {
    uint32_t w0[NWK], w1[NWK];
    lds_run<CL::rbk>(seg + (16 * ch + grp) * CL::k_row + CL::rbk * tig, w0);
    lds_run<CL::rbk>(seg + (16 * ch + 8 + grp) * CL::k_row + CL::rbk * tig, w1);
    static_for<0, NG>([&](auto gi) {
      constexpr int g = decltype(gi)::value;
      uint32_t a0, a1, a2, a3;
      if constexpr (CL::kbits == 8) {
#if DKV_TC_K8_BIASED
        a0 = __byte_perm(w0[g], 0x64646464u, 0x4140); a2 = __byte_perm(w0[g], 0x64646464u, 0x4342);   // 1024 + c
        a1 = __byte_perm(w1[g], 0x64646464u, 0x4140); a3 = __byte_perm(w1[g], 0x64646464u, 0x4342);
#else
        k8_pairs(w0[g], a0, a2);                         // features 4g .. 4g+3 = word g of the run
        k8_pairs(w1[g], a1, a3);
#endif
      } else {
        static_assert(CL::kbits == 4, "tensor-core path: K8 or K4 keys");
        k4_pairs<2 * (g & 1)>(w0[g >> 1], a0, a2);       // bytes 2g, 2g+1 of the run
        k4_pairs<2 * (g & 1)>(w1[g >> 1], a1, a3);
      }
      mma_f16(acc2[g & 1], a0, a1, a2, a3, qb[g][0], qb[g][1]);
    });
  }
  // logits of (token grp | grp + 8, head 2 tig | 2 tig + 1) = c0, c1 | c2, c3:
  // l2 = (s_k scale2) acc + z'_k (qsum scale2), qsz = qsum scale2 of the lane's two heads (0 beyond G)
  const int t0 = 16 * ch + grp;
  float l[4], svs[2], zv[2];
#pragma unroll
  for (int rr = 0; rr < 2; rr++) {
    const int t = t0 + 8 * rr;
    const bool tok = t < cnt;
    const uint32_t km = *reinterpret_cast<const uint32_t*>(seg + CL::off_kmeta + 4 * t);
    const uint32_t vm = *reinterpret_cast<const uint32_t*>(seg + CL::off_vmeta + 4 * t);
    const float ks = __half2float(__ushort_as_half((unsigned short)(km & 0xFFFFu)));
#if DKV_TC_K8_BIASED
    const float kz = CL::kbits == 8 ? fmaf(ks, -1024.0f, __half2float(__ushort_as_half((unsigned short)(km >> 16))))
                                    : tc_zc<CL::kbits>(__half2float(__ushort_as_half((unsigned short)(km >> 16))), ks);
#else
    const float kz = tc_zc<CL::kbits>(__half2float(__ushort_as_half((unsigned short)(km >> 16))), ks);
#endif
    const float vs = __half2float(__ushort_as_half((unsigned short)(vm & 0xFFFFu)));
    const float vz = tc_zc<CL::vbits>(__half2float(__ushort_as_half((unsigned short)(vm >> 16))), vs);
    svs[rr] = tok ? vs * kPvScale : 0.0f;                // an absent token's stale meta never reaches a product
    zv[rr] = tok ? vz : 0.0f;
    const float kss = ks * scale2;
#pragma unroll
    for (int c = 0; c < 2; c++) {
      const float v = fmaf(kss, acc2[0][2 * rr + c] + acc2[1][2 * rr + c], kz * qsz[c]);
      l[2 * rr + c] = (tok && 2 * tig + c < G) ? v : -INFINITY;
    }
  }
  if (2 * tig < G) {
    float* lr = lgl + (size_t)(row0 + t0) * GP;
    *reinterpret_cast<float2*>(lr) = make_float2(l[0], l[1]);
    *reinterpret_cast<float2*>(lr + 8 * GP) = make_float2(l[2], l[3]);
  }
  // ---- PV: A = value codes (m = features (D/8) grp + 2 mt | + 1, k = tokens), B = weights hi, then lo
  uint32_t vw[4][NWV];                                   // rows 2 tig, 2 tig + 1, 8 + 2 tig, 9 + 2 tig
#pragma unroll
  for (int r = 0; r < 4; r++)
    lds_run<CL::rbv>(seg + CL::off_v + (16 * ch + 2 * tig + (r & 1) + 8 * (r >> 1)) * CL::v_row + CL::rbv * grp, vw[r]);
  tc_softmax_pv<D>(l, svs, zv, st, [&](auto mti, uint32_t& a0, uint32_t& a1, uint32_t& a2, uint32_t& a3) {
    constexpr int mt = decltype(mti)::value;
    constexpr int bit = 2 * mt * CL::vbits;              // features 2 mt, 2 mt + 1 of the lane's run
    constexpr int wi = bit >> 5, kb = (bit >> 3) & 3, sh = bit & 7;
    a0 = v_pair<kb, sh, CL::vbits>(vw[0][wi], vw[1][wi]);
    a1 = v_pair<kb, sh + CL::vbits, CL::vbits>(vw[0][wi], vw[1][wi]);
    a2 = v_pair<kb, sh, CL::vbits>(vw[2][wi], vw[3][wi]);
    a3 = v_pair<kb, sh + CL::vbits, CL::vbits>(vw[2][wi], vw[3][wi]);
  });
}

// One 16-slot chunk of the FP16 window ring (slots 16 c .. 16 c + 15 of [W][D]; slot s is live iff s < nw), straight
// from global memory: the fp16 rows are the MMA operands themselves (s = 1, z = 0).  `wrow0` = the scratch row
// of the oldest window token; slot s holds window token (s - base) mod W, base = (N - nw) mod W.
template <int D, int G, int GP>
__device__ __forceinline__ void tc_window_chunk(const uint16_t* wk, const uint16_t* wv, int c, int nw, int W,
                                                int base, const uint32_t (&qb)[D / 16][2], float scale2,
                                                float* lgl, int wrow0, TcState<D>& st, int grp, int tig) {
  constexpr int NG = D / 16, FPK = D / 4, FPV = D / 8;
  const int s0 = 16 * c + grp, s1 = s0 + 8;
  const bool ok0 = s0 < nw, ok1 = s1 < nw;
  // ---- QK^T: A = the keys' fp16 pairs (features FPK tig + 4g + {0, 1} = word 2g of the lane's run, + {2, 3} =
  // word 2g + 1), in two halves of the k-steps
  float acc2[2][4] = {{0.f, 0.f, 0.f, 0.f}, {0.f, 0.f, 0.f, 0.f}};
  static_for<0, 2>([&](auto hi_) {
    constexpr int hf = decltype(hi_)::value;
    constexpr int NW = FPK / 4;                          // words per half run (FPK/2 fp16 = FPK bytes)
    uint32_t r0[NW], r1[NW];
#pragma unroll
    for (int q4 = 0; q4 < NW / 4; q4++) {
      const uint4 x = ok0 ? ld_nc_v4(wk + (size_t)s0 * D + FPK * tig + hf * (FPK / 2) + 8 * q4) : make_uint4(0u, 0u, 0u, 0u);
      const uint4 y = ok1 ? ld_nc_v4(wk + (size_t)s1 * D + FPK * tig + hf * (FPK / 2) + 8 * q4) : make_uint4(0u, 0u, 0u, 0u);
      r0[4 * q4] = x.x; r0[4 * q4 + 1] = x.y; r0[4 * q4 + 2] = x.z; r0[4 * q4 + 3] = x.w;
      r1[4 * q4] = y.x; r1[4 * q4 + 1] = y.y; r1[4 * q4 + 2] = y.z; r1[4 * q4 + 3] = y.w;
    }
    static_for<0, NG / 2>([&](auto gi) {
      constexpr int gg = decltype(gi)::value, g = hf * (NG / 2) + gg;
      mma_f16(acc2[g & 1], r0[2 * gg], r1[2 * gg], r0[2 * gg + 1], r1[2 * gg + 1], qb[g][0], qb[g][1]);
    });
  });
  float l[4];
  const float svs[2] = {ok0 ? kPvScale : 0.0f, ok1 ? kPvScale : 0.0f}, zv[2] = {0.0f, 0.0f};
#pragma unroll
  for (int rr = 0; rr < 2; rr++)
#pragma unroll
    for (int cc = 0; cc < 2; cc++) {
      const float v = (acc2[0][2 * rr + cc] + acc2[1][2 * rr + cc]) * scale2;
      l[2 * rr + cc] = ((rr ? ok1 : ok0) && 2 * tig + cc < G) ? v : -INFINITY;
    }
  if (2 * tig < G) {
#pragma unroll
    for (int rr = 0; rr < 2; rr++) {
      const int sl = rr ? s1 : s0;
      if (sl < nw) {
        int i = sl - base;
        i += i < 0 ? W : 0;
        *reinterpret_cast<float2*>(lgl + (size_t)(wrow0 + i) * GP) = make_float2(l[2 * rr], l[2 * rr + 1]);
      }
    }
  }
  // ---- PV: A = the values' fp16 (m = features FPV grp + 2 mt | + 1 = the halves of word mt of the lane's run;
  // k = slots 2 tig, 2 tig + 1 | + 8), absent slots zeroed
  uint32_t vw[4][FPV / 2];
#pragma unroll
  for (int r = 0; r < 4; r++) {
    const int sl = 16 * c + 2 * tig + (r & 1) + 8 * (r >> 1);
#pragma unroll
    for (int q4 = 0; q4 < FPV / 8; q4++) {
      const uint4 x = sl < nw ? ld_nc_v4(wv + (size_t)sl * D + FPV * grp + 8 * q4) : make_uint4(0u, 0u, 0u, 0u);
      vw[r][4 * q4] = x.x; vw[r][4 * q4 + 1] = x.y; vw[r][4 * q4 + 2] = x.z; vw[r][4 * q4 + 3] = x.w;
    }
  }
  tc_softmax_pv<D>(l, svs, zv, st, [&](auto mti, uint32_t& a0, uint32_t& a1, uint32_t& a2, uint32_t& a3) {
    constexpr int mt = decltype(mti)::value;
    a0 = __byte_perm(vw[0][mt], vw[1][mt], 0x5410);      // feature 2 mt of slots 2 tig, 2 tig + 1
    a1 = __byte_perm(vw[0][mt], vw[1][mt], 0x7632);      // feature 2 mt + 1
    a2 = __byte_perm(vw[2][mt], vw[3][mt], 0x5410);
    a3 = __byte_perm(vw[2][mt], vw[3][mt], 0x7632);
  });
}

// A unit whose significance pass is still pending (its logits, maxima and sums are final): the pass runs during
// the CTA's next unit, a block of kTcThreads token rows per page iteration of each warp (software pipelining across
// units), so that its dependent loads (page ID -> score / position) overlap that unit's page computation.
struct TcSigUnit {
  int u, N, nh, nl, ph, lo0, wb, nw, Ts, rows, buf;
};

// Persistent: gridDim.x CTAs (the occupancy limit, at most tc_slots) take units blockIdx.x, + gridDim.x, ...  A
// CTA's logits (log2 units) live in its own global scratch slots (p.tc_scratch: two [tc_slot_rows][GP] fp32
// buffers per CTA, alternating between units; rows page-aligned: high page k at 16 k, low page k' at 16 ph + 32 k',
// the window after them), written once in the page pass and read once by the significance pass.
template <int D, int G>
#if DKV_TC_MAXNREG > 0
__global__ void __maxnreg__(DKV_TC_MAXNREG)
#else
__global__ void __launch_bounds__(kTcThreads, DKV_TC_MINB)
#endif
attend_tc_kernel(PoolDev p, const uint16_t* __restrict__ q, float* __restrict__ out, float* __restrict__ probs) {
  constexpr int NG = D / 16, NMT = D / 16, FPK = D / 4, FPV = D / 8, GP = G <= 4 ? 4 : 8;
  constexpr int STG = tc_stage_bytes<D>();
  using HI = TcCls<D, 16, 8, 4>;                                  // K8V4, 16-token pages
  using LO = TcCls<D, 32, 4, 2>;                                  // K4V2, 32-token pages
  extern __shared__ __align__(128) uint8_t tc_smem[];
  __shared__ float s_mw[kTcWarps][8], s_zw[kTcWarps][8], s_zsw[kTcWarps][8];
  __shared__ float s_fw[kTcWarps][8];
  __shared__ float s_C[2][8], s_iZ[2][8];                         // per logit buffer: M + log2 Z per head, and 1/Z
  __shared__ TcSigUnit s_prev;
  __shared__ unsigned long long s_min[2];
  __shared__ int s_slot[2];
  __shared__ __align__(16) float s_sl[2][kTcThreads][GP];         // significance pass: staged logit rows
  __shared__ __align__(8) float s_ss[2][kTcThreads][2];           //   ... and (score, position bits)
  __shared__ unsigned long long s_sa[2][kTcThreads];             //   ... and the score's address
  __shared__ __align__(8) uint64_t s_bar[kTcWarps][kTcStages];   // per-warp stage mbarriers (bulk copies)
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int grp = lane >> 2, tig = lane & 3;
  if (ld_volatile(&p.ctrl->status) != 0) return;                  // sticky error: no-op
  const int L = p.L, W = p.W, R = p.tc_slot_rows, LP = (L + 4) & ~3;
  const ClassGeom gh = p.g[1], gl = p.g[2];
  uint8_t* const stage0 = tc_smem;
  int32_t* const pidb = reinterpret_cast<int32_t*>(tc_smem + tc_area_bytes(D, G, STG));   // [2][LP] page IDs
  uint8_t* const mystage = stage0 + (size_t)warp * kTcStages * STG;
  uint64_t* const bars = s_bar[warp];
  if (tid < kTcWarps * kTcStages) mbar_init(&s_bar[tid / kTcStages][tid % kTcStages], 1);
  if (tid == 0) s_prev.rows = 0;
  fence_mbar_init();
  uint32_t phase = 0;                                             // bit s: parity of stage s's next completion
  const uint32_t bar_s = smem_u32(bars), stage_s = smem_u32(mystage);
  const float scale2 = rsqrtf((float)D) * kLog2e;                 // logits in log2 units: p = 2^(l2 - m2)
  uint64_t pol;
  asm("createpolicy.fractional.L2::evict_first.b64 %0, 1.0;" : "=l"(pol));
  const uint16_t* const wk_all = reinterpret_cast<const uint16_t*>(p.win_k);
  const uint16_t* const wv_all = reinterpret_cast<const uint16_t*>(p.win_v);
  int buf = 0;                                                    // this unit's logit / page-ID buffer

  // ---- the significance pass of the pending unit `sp` (Q33): row block j = rows j * kTcThreads + tid
  // issue: stage the row's logits, score and position with cp.async into slot j & 1 (nothing for a padding row)
  constexpr uint32_t kSsStride = kTcThreads * 8, kSlStride = kTcThreads * GP * 4;
  const uint32_t ss_u32 = smem_u32(&s_ss[0][tid][0]), sl_u32 = smem_u32(&s_sl[0][tid][0]);
  unsigned long long mkey0 = ~0ull, mkey1 = ~0ull;                // this thread's section minima of `sp`
  int mslot0 = -1, mslot1 = -1;
  auto sig_issue = [&](const TcSigUnit& sp, int j) {
    const int row = j * kTcThreads + tid, sl = j & 1;
    if (row >= sp.rows) return;
    const float* lgp = p.tc_scratch + ((size_t)(2 * blockIdx.x + sp.buf) * R + row) * GP;
    if (row < sp.wb) {
      const bool hi = row < sp.lo0;
      const int rr = hi ? row : row - sp.lo0;
      if (rr >= (hi ? sp.nh : sp.nl)) return;                     // a partial page's padding row
      const int k = hi ? row >> 4 : sp.ph + (rr >> 5), j2 = hi ? row & 15 : rr & 31;
      const ClassGeom& gg = hi ? gh : gl;
      const uint8_t* pg = p.pages + (size_t)pidb[sp.buf * LP + k] * (size_t)p.page_bytes;
      s_sa[sl][tid] = reinterpret_cast<unsigned long long>(pg + gg.off_score + 4 * j2);
      asm volatile("cp.async.ca.shared.global [%0], [%1], 4;" ::"r"(ss_u32 + sl * kSsStride), "l"(pg + gg.off_score + 4 * j2) : "memory");
      asm volatile("cp.async.ca.shared.global [%0], [%1], 4;" ::"r"(ss_u32 + sl * kSsStride + 4), "l"(pg + gg.off_pos + 4 * j2) : "memory");
    } else {
      const int pos = sp.N - sp.nw + (row - sp.wb);
      asm volatile("cp.async.ca.shared.global [%0], [%1], 4;" ::"r"(ss_u32 + sl * kSsStride),
                   "l"(p.win_sig + (size_t)sp.u * W + fmod_(p.div_W, pos)) : "memory");
    }
#pragma unroll
    for (int c4 = 0; c4 < GP / 4; c4++)
      asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(sl_u32 + sl * kSlStride + 16 * c4), "l"(lgp + 4 * c4)
                   : "memory");
  };
  // consume: a = max_h 2^(l2 - M) / Z, the running mean written back, probabilities, section minima
  auto sig_consume = [&](const TcSigUnit& sp, int j) {
    const int row = j * kTcThreads + tid, sl = j & 1;
    if (row >= sp.rows) return;
    const bool stored = row < sp.wb, hi = row < sp.lo0;
    const int rr = hi ? row : row - sp.lo0;
    if (stored && rr >= (hi ? sp.nh : sp.nl)) return;
    // a = max_h 2^(l_h - M_h) / Z_h = 2^(max_h (l_h - C_h)), C_h = M_h + log2 Z_h: one exp2 per token
    float xm = -INFINITY;
#pragma unroll
    for (int h = 0; h < G; h++) xm = fmaxf(xm, s_sl[sl][tid][h] - s_C[sp.buf][h]);
    const float a = ex2(xm);
    float sg = s_ss[sl][tid][0];
    const int pos = stored ? __float_as_int(s_ss[sl][tid][1]) : sp.N - sp.nw + (row - sp.wb);
    const int c = sp.N - 2 - pos;
    if (c >= 0) sg = __fdividef(fmaf(sg, (float)c, a), (float)(c + 1));   // (a tolerance path: approximate division)
    if (stored) {
      // the score's address, left by sig_issue in the staging slot (no second page-ID lookup)
      float* sp_addr = reinterpret_cast<float*>(s_sa[sl][tid]);
      if (c >= 0) *sp_addr = sg;
      if (probs) probs[(size_t)sp.u * p.M + (hi ? rr : sp.nh + rr)] = a;
      const unsigned long long key = ((unsigned long long)__float_as_uint(sg) << 32) | (uint32_t)pos;
      if (hi) {
        if (key < mkey0) { mkey0 = key; mslot0 = rr; }
      } else if (key < mkey1) {
        mkey1 = key; mslot1 = rr;
      }
    } else {
      if (c >= 0) p.win_sig[(size_t)sp.u * W + fmod_(p.div_W, pos)] = sg;
      if (probs) probs[(size_t)sp.u * p.M + sp.Ts + (row - sp.wb)] = a;
    }
  };
  // one pipeline step: stage block j + 1, then consume block j
  auto sig_step = [&](const TcSigUnit& sp, int j, int nsig) {
    if (j + 1 < nsig) sig_issue(sp, j + 1);
    cp_async_commit();
    cp_async_wait<1>();
    sig_consume(sp, j);
  };
  // the pending unit's section minima (after every thread has consumed its rows)
  auto sig_finish = [&](const TcSigUnit& sp) {
    if (mkey0 != ~0ull) atomicMin(&s_min[0], mkey0);
    if (mkey1 != ~0ull) atomicMin(&s_min[1], mkey1);
    __syncthreads();
    if (mkey0 != ~0ull && mkey0 == s_min[0]) s_slot[0] = mslot0;
    if (mkey1 != ~0ull && mkey1 == s_min[1]) s_slot[1] = mslot1;
    __syncthreads();
    if (tid == 0) {
      int32_t* m = p.secmin + 8 * (size_t)sp.u;
#pragma unroll
      for (int c = 0; c < 2; c++) {
        m[3 * c] = (int32_t)(uint32_t)(s_min[c] >> 32);
        m[3 * c + 1] = (int32_t)(uint32_t)(s_min[c] & 0xFFFFFFFFull);
        m[3 * c + 2] = s_slot[c];
        s_min[c] = ~0ull;
        s_slot[c] = -1;
      }
      m[6] = 1;
    }
    mkey0 = mkey1 = ~0ull;
    mslot0 = mslot1 = -1;
  };
  if (tid < 2) { s_min[tid] = ~0ull; s_slot[tid] = -1; }

  for (int u = blockIdx.x; u < p.U; u += gridDim.x) {
    const int r = fdiv(p.div_LyH, u);
    if (p.req_state[r] != DKV_REQ_ACTIVE) continue;               // CTA-uniform
    const int N = p.seq_len[r];
    const int nh = p.n_h[u], nl = p.n_l[u];
    const int nw = min(W, N);
    const int ph = (nh + HI::C - 1) / HI::C, pl = (nl + LO::C - 1) / LO::C;
    const int npg = ph + pl;
    const int lo0 = HI::C * ph, wb = lo0 + LO::C * pl;            // first scratch row of the low pages, window
    const int32_t* trow = p.table + (size_t)u * L;
    int32_t* const pid = pidb + buf * LP;
    float* const lg = p.tc_scratch + (size_t)(2 * blockIdx.x + buf) * R * GP;   // this unit's logits [R][GP]
    fence_proxy_async_smem();                                     // the previous unit's generic accesses ...
    __syncthreads();                                              // ... before this unit's bulk fills; s_prev
    const TcSigUnit sp = s_prev;
    const int nsig = (sp.rows + kTcThreads - 1) / kTcThreads;     // the pending unit's row blocks
    for (int k = tid; k < npg; k += kTcThreads) pid[k] = k < ph ? trow[k] : trow[L - 1 - (k - ph)];
    // B fragments of the queries (k = features, permuted as the keys' A fragments; n = head grp): k-step g
    // holds features FPK tig + 4g + {0, 1} (b0) and + {2, 3} (b1) of head grp (zero for grp >= G)
    uint32_t qb[NG][2];
    float qs = 0.0f;                                              // head grp's sum over this lane's features
    {
      const uint16_t* qr = q + ((size_t)u * G + (grp < G ? grp : 0)) * D + FPK * tig;
#pragma unroll
      for (int g = 0; g < NG; g++) {
        uint2 v = make_uint2(0u, 0u);
        if (grp < G) v = *reinterpret_cast<const uint2*>(qr + 4 * g);
        qb[g][0] = v.x; qb[g][1] = v.y;
        const float2 f0 = __half22float2(*reinterpret_cast<const __half2*>(&v.x));
        const float2 f1 = __half22float2(*reinterpret_cast<const __half2*>(&v.y));
        qs += (f0.x + f0.y) + (f1.x + f1.y);
      }
      qs += __shfl_xor_sync(kFull, qs, 1);
      qs += __shfl_xor_sync(kFull, qs, 2);
    }
    // the z' term's per-head sums for this lane's heads 2 tig, 2 tig + 1 (held by grp = 2 tig, 2 tig + 1), x scale2
    const float qsz[2] = {__shfl_sync(kFull, qs, 8 * tig) * scale2, __shfl_sync(kFull, qs, 8 * tig + 4) * scale2};
    __syncthreads();                                              // pid
    float* const lgl = lg + 2 * tig;                              // this lane's logit column

    auto page_ptr = [&](int k) { return p.pages + (size_t)pid[k] * (size_t)p.page_bytes; };
    const int my_n = npg > warp ? (npg - warp + kTcWarps - 1) / kTcWarps : 0;   // this warp's pages
    auto stage = [&](int k, int slot) {
      if (lane != 0) return;
      const uint32_t bytes = k < ph ? HI::prefix : LO::prefix;
      const uint32_t bar = bar_s + 8 * slot;
      asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(bar), "r"(bytes) : "memory");
      asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes.L2::cache_hint [%0], [%1], %2, [%3], %4;"
                   ::"r"(stage_s + slot * STG), "l"(page_ptr(k)), "r"(bytes), "r"(bar), "l"(pol) : "memory");
    };

    // ---- the page pass: each warp its pages (k = warp + i * kTcWarps), kTcStages - 1 copies ahead; page
    // iteration i also runs block i of the pending unit's significance pass
    TcState<D> st;
#pragma unroll
    for (int mt = 0; mt < NMT; mt++) st.o[mt][0] = st.o[mt][1] = st.o[mt][2] = st.o[mt][3] = 0.0f;
#pragma unroll
    for (int c = 0; c < 2; c++) {
      st.m[c] = 2 * tig + c < G ? -INFINITY : 0.0f;
      st.z[c] = 0.0f;
      st.zs[c] = 0.0f;
    }
#pragma unroll
    for (int i = 0; i < kTcStages - 1; i++)
      if (i < my_n) stage(warp + i * kTcWarps, i);
    if (nsig > 0) sig_issue(sp, 0);
    cp_async_commit();
    // page i of this warp sits in stage i mod kTcStages (slot counters, not a modulo; the loop is not unrolled
    // by the stage count — measured: three inlined copies of the chunk code overflowed the instruction cache)
    for (int i = 0, slot = 0, islot = kTcStages - 1; i < my_n; i++) {
      const int k = warp + i * kTcWarps;
      if (i + kTcStages - 1 < my_n) stage(warp + (i + kTcStages - 1) * kTcWarps, islot);
      mbar_wait_u32(bar_s + 8 * slot, (phase >> slot) & 1u);
      phase ^= 1u << slot;
      const uint8_t* seg = mystage + slot * STG;
      if (k < ph) {
        const int t0 = HI::C * k;
        tc_chunk<D, G, GP, HI>(seg, 0, nh - t0, qb, qsz, scale2, lgl, t0, st, grp, tig);
      } else {
        const int kk = k - ph, cnt = nl - LO::C * kk, row = lo0 + LO::C * kk;
        tc_chunk<D, G, GP, LO>(seg, 0, cnt, qb, qsz, scale2, lgl, row, st, grp, tig);
        if (cnt > 16) tc_chunk<D, G, GP, LO>(seg, 1, cnt, qb, qsz, scale2, lgl, row, st, grp, tig);
      }
      // The stage is refilled (by the bulk copy of page i + kTcStages) one iteration later.  No proxy fence: every
      // read of it fed an mma.sync of this iteration, which no lane passes before all lanes have issued it, so
      // the reads have completed before lane 0 can issue that copy (measured: the fence's MEMBAR.CTA per page
      // also waited on the logit stores).
      __syncwarp();
      if (i < nsig) sig_step(sp, i, nsig);
      slot = slot + 1 == kTcStages ? 0 : slot + 1;
      islot = islot + 1 == kTcStages ? 0 : islot + 1;
    }
    // the pending unit's remaining row blocks (a warp with fewer pages than blocks)
    for (int j = my_n; j < nsig; j++) sig_step(sp, j, nsig);
    // the FP16 window: 16-slot chunks of the ring, round-robin over the warps after their pages
    {
      const int wbase = fmod_(p.div_W, N - nw);                   // ring slot of the oldest window token
      for (int c = warp; 16 * c < nw; c += kTcWarps)
        tc_window_chunk<D, G, GP>(wk_all + (size_t)u * W * D, wv_all + (size_t)u * W * D, c, nw, W, wbase, qb,
                                  scale2, lgl, wb, st, grp, tig);
    }
    // the warp's state per head: Z and sum p z' over the 8 lanes (grp) of heads 2 tig, 2 tig + 1
#pragma unroll
    for (int c = 0; c < 2; c++)
#pragma unroll
      for (int o = 4; o < 32; o <<= 1) {
        st.z[c] += __shfl_xor_sync(kFull, st.z[c], o);
        st.zs[c] += __shfl_xor_sync(kFull, st.zs[c], o);
      }
    __syncthreads();                                              // every warp is out of its stages
    if (sp.rows > 0) sig_finish(sp);                              // (two barriers inside)
    float* part = reinterpret_cast<float*>(stage0);               // [kTcWarps][G][D] warp partials (hi + lo)
#pragma unroll
    for (int c = 0; c < 2; c++) {
      const int h = 2 * tig + c;
      if (h < G) {
        if (grp == 0) { s_mw[warp][h] = st.m[c]; s_zw[warp][h] = st.z[c]; s_zsw[warp][h] = st.zs[c]; }
        float* pr = part + ((size_t)warp * G + h) * D + FPV * grp;
#pragma unroll
        for (int mt = 0; mt < NMT; mt++) {
          pr[2 * mt] = st.o[mt][c] * kPvUnscale;
          pr[2 * mt + 1] = st.o[mt][2 + c] * kPvUnscale;
        }
      }
    }
    __syncthreads();
    if (tid < G) {                                                // head tid: the global maximum and sum
      float M = -INFINITY;
      for (int w = 0; w < kTcWarps; w++) M = fmaxf(M, s_mw[w][tid]);
      float Z = 0.0f;
      for (int w = 0; w < kTcWarps; w++) {
        const float f = s_mw[w][tid] == -INFINITY ? 0.0f : ex2(s_mw[w][tid] - M);
        s_fw[w][tid] = f;
        Z = fmaf(f, s_zw[w][tid], Z);
      }
      s_C[buf][tid] = Z > 0.0f ? M + log2f(Z) : INFINITY;
      s_iZ[buf][tid] = Z > 0.0f ? 1.0f / Z : 0.0f;
    }
    if (tid == 0) s_prev = TcSigUnit{u, N, nh, nl, ph, lo0, wb, nw, nh + nl, wb + nw, buf};   // pending now
    __syncthreads();
    // ---- the output: the warps' partials (each with its z term), rescaled to the global maximum
    if (out != nullptr) {
      for (int e = tid; e < G * D / 2; e += kTcThreads) {         // a feature pair per thread
        const int h = e / (D / 2), f = 2 * (e % (D / 2));
        float o0 = 0.0f, o1 = 0.0f;
#pragma unroll
        for (int w = 0; w < kTcWarps; w++) {
          const float fw = s_fw[w][h];
          const float2 pp = *reinterpret_cast<const float2*>(part + ((size_t)w * G + h) * D + f);
          const float zz = s_zsw[w][h];
          o0 = fmaf(fw, pp.x + zz, o0);
          o1 = fmaf(fw, pp.y + zz, o1);
        }
        const float iz = s_iZ[buf][h];
        *reinterpret_cast<float2*>(out + ((size_t)u * G + h) * D + f) = make_float2(o0 * iz, o1 * iz);
      }
    }
    buf ^= 1;
  }
  // the last unit's significance pass, on its own
  __syncthreads();
  const TcSigUnit sp = s_prev;
  if (sp.rows > 0) {
    const int nsig = (sp.rows + kTcThreads - 1) / kTcThreads;
    sig_issue(sp, 0);
    cp_async_commit();
    for (int j = 0; j < nsig; j++) sig_step(sp, j, nsig);
    __syncthreads();
    sig_finish(sp);
  }
}

// ---- Split-sequence form ("split the sequence into segments processed by separate thread blocks, then
// merge"): with few active units one CTA per unit leaves most SMs idle, so each unit gets NS CTAs, CTA s over a
// contiguous range of the unit's pages (the last one also over the window), each writing its partial softmax state
// (per head: maximum M_s, sum Z_s, sum of p z' and the output accumulator, all relative to M_s); a second kernel
// merges the NS states (the same rescaling as the warps' merge) and runs the unit's significance pass.  Scratch
// (U <= kTcSlots): the unit's logit rows in buffer u of tc_scratch, the partial states after buffer kTcSlots.
constexpr int kTcSplitMax = 32;
#ifndef DKV_TC_SPLIT
#define DKV_TC_SPLIT 1      // build-time switch of the split-sequence form (A/B: tools/tc_split_ab.py)
#endif
template <int D, int G>
__host__ __device__ constexpr int tc_partial_floats() { return G * D + 3 * 8 + 8; }   // + minima candidates

template <int D, int G>
#if DKV_TC_MAXNREG > 0
__global__ void __maxnreg__(DKV_TC_MAXNREG)
#else
__global__ void __launch_bounds__(kTcThreads, DKV_TC_MINB)
#endif
attend_tc_split_kernel(PoolDev p, const uint16_t* __restrict__ q, int NS, int slots) {
  constexpr int NG = D / 16, NMT = D / 16, FPK = D / 4, FPV = D / 8, GP = G <= 4 ? 4 : 8;
  constexpr int STG = tc_stage_bytes<D>();
  using HI = TcCls<D, 16, 8, 4>;
  using LO = TcCls<D, 32, 4, 2>;
  extern __shared__ __align__(128) uint8_t tc_smem[];
  __shared__ float s_mw[kTcWarps][8], s_zw[kTcWarps][8], s_zsw[kTcWarps][8];
  __shared__ __align__(8) uint64_t s_bar[kTcWarps][kTcStages];
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int grp = lane >> 2, tig = lane & 3;
  const int u = blockIdx.x, seg = blockIdx.y;
  if (ld_volatile(&p.ctrl->status) != 0) return;
  if (p.req_state[fdiv(p.div_LyH, u)] != DKV_REQ_ACTIVE) return;  // CTA-uniform
  const int L = p.L, W = p.W, R = p.tc_slot_rows;
  const int N = p.seq_len[fdiv(p.div_LyH, u)];
  const int nh = p.n_h[u], nl = p.n_l[u];
  const int nw = min(W, N);
  const int ph = (nh + HI::C - 1) / HI::C, pl = (nl + LO::C - 1) / LO::C, npg = ph + pl;
  const int lo0 = HI::C * ph, wb = lo0 + LO::C * pl;
  const int k0 = (int)((long)seg * npg / NS), k1 = (int)((long)(seg + 1) * npg / NS);   // this CTA's pages
  uint8_t* const stage0 = tc_smem;
  int32_t* const pid = reinterpret_cast<int32_t*>(tc_smem + tc_area_bytes(D, G, STG));
  uint8_t* const mystage = stage0 + (size_t)warp * kTcStages * STG;
  uint64_t* const bars = s_bar[warp];
  if (tid < kTcWarps * kTcStages) mbar_init(&s_bar[tid / kTcStages][tid % kTcStages], 1);
  fence_mbar_init();
  uint32_t phase = 0;
  const uint32_t bar_s = smem_u32(bars), stage_s = smem_u32(mystage);
  const float scale2 = rsqrtf((float)D) * kLog2e;
  uint64_t pol;
  asm("createpolicy.fractional.L2::evict_first.b64 %0, 1.0;" : "=l"(pol));
  const int32_t* trow = p.table + (size_t)u * L;
  for (int k = k0 + tid; k < k1; k += kTcThreads) pid[k - k0] = k < ph ? trow[k] : trow[L - 1 - (k - ph)];
  uint32_t qb[NG][2];
  float qs = 0.0f;
  {
    const uint16_t* qr = q + ((size_t)u * G + (grp < G ? grp : 0)) * D + FPK * tig;
#pragma unroll
    for (int g = 0; g < NG; g++) {
      uint2 v = make_uint2(0u, 0u);
      if (grp < G) v = *reinterpret_cast<const uint2*>(qr + 4 * g);
      qb[g][0] = v.x; qb[g][1] = v.y;
      const float2 f0 = __half22float2(*reinterpret_cast<const __half2*>(&v.x));
      const float2 f1 = __half22float2(*reinterpret_cast<const __half2*>(&v.y));
      qs += (f0.x + f0.y) + (f1.x + f1.y);
    }
    qs += __shfl_xor_sync(kFull, qs, 1);
    qs += __shfl_xor_sync(kFull, qs, 2);
  }
  const float qsz[2] = {__shfl_sync(kFull, qs, 8 * tig) * scale2, __shfl_sync(kFull, qs, 8 * tig + 4) * scale2};
  __syncthreads();                                                // pid, barriers
  float* const lgl = p.tc_scratch + (size_t)u * R * GP + 2 * tig; // the unit's logit buffer, this lane's column
  const int npr = k1 - k0;
  const int my_n = npr > warp ? (npr - warp + kTcWarps - 1) / kTcWarps : 0;
  auto stage = [&](int kl, int slot) {                            // kl: page index within the range
    if (lane != 0) return;
    const int k = k0 + kl;
    const uint32_t bytes = k < ph ? HI::prefix : LO::prefix;
    const uint32_t bar = bar_s + 8 * slot;
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(bar), "r"(bytes) : "memory");
    asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes.L2::cache_hint [%0], [%1], %2, [%3], %4;"
                 ::"r"(stage_s + slot * STG), "l"(p.pages + (size_t)pid[kl] * (size_t)p.page_bytes), "r"(bytes), "r"(bar),
                 "l"(pol) : "memory");
  };
  TcState<D> st;
#pragma unroll
  for (int mt = 0; mt < NMT; mt++) st.o[mt][0] = st.o[mt][1] = st.o[mt][2] = st.o[mt][3] = 0.0f;
#pragma unroll
  for (int c = 0; c < 2; c++) {
    st.m[c] = 2 * tig + c < G ? -INFINITY : 0.0f;
    st.z[c] = 0.0f;
    st.zs[c] = 0.0f;
  }
#pragma unroll
  for (int i = 0; i < kTcStages - 1; i++)
    if (i < my_n) stage(warp + i * kTcWarps, i);
  for (int i = 0, slot = 0, islot = kTcStages - 1; i < my_n; i++) {
    const int kl = warp + i * kTcWarps, k = k0 + kl;
    if (i + kTcStages - 1 < my_n) stage(warp + (i + kTcStages - 1) * kTcWarps, islot);
    mbar_wait_u32(bar_s + 8 * slot, (phase >> slot) & 1u);
    phase ^= 1u << slot;
    const uint8_t* sg = mystage + slot * STG;
    if (k < ph) {
      const int t0 = HI::C * k;
      tc_chunk<D, G, GP, HI>(sg, 0, nh - t0, qb, qsz, scale2, lgl, t0, st, grp, tig);
    } else {
      const int kk = k - ph, cnt = nl - LO::C * kk, row = lo0 + LO::C * kk;
      tc_chunk<D, G, GP, LO>(sg, 0, cnt, qb, qsz, scale2, lgl, row, st, grp, tig);
      if (cnt > 16) tc_chunk<D, G, GP, LO>(sg, 1, cnt, qb, qsz, scale2, lgl, row, st, grp, tig);
    }
    __syncwarp();
    slot = slot + 1 == kTcStages ? 0 : slot + 1;
    islot = islot + 1 == kTcStages ? 0 : islot + 1;
  }
  if (seg == NS - 1) {                                            // the window, by the last segment's CTA
    const uint16_t* wk_all = reinterpret_cast<const uint16_t*>(p.win_k);
    const uint16_t* wv_all = reinterpret_cast<const uint16_t*>(p.win_v);
    const int wbase = fmod_(p.div_W, N - nw);
    for (int c = warp; 16 * c < nw; c += kTcWarps)
      tc_window_chunk<D, G, GP>(wk_all + (size_t)u * W * D, wv_all + (size_t)u * W * D, c, nw, W, wbase, qb, scale2,
                                lgl, wb, st, grp, tig);
  }
#pragma unroll
  for (int c = 0; c < 2; c++)
#pragma unroll
    for (int o = 4; o < 32; o <<= 1) {
      st.z[c] += __shfl_xor_sync(kFull, st.z[c], o);
      st.zs[c] += __shfl_xor_sync(kFull, st.zs[c], o);
    }
  __syncthreads();
  float* part = reinterpret_cast<float*>(stage0);                 // [kTcWarps][G][D]
#pragma unroll
  for (int c = 0; c < 2; c++) {
    const int h = 2 * tig + c;
    if (h < G) {
      if (grp == 0) { s_mw[warp][h] = st.m[c]; s_zw[warp][h] = st.z[c]; s_zsw[warp][h] = st.zs[c]; }
      float* pr = part + ((size_t)warp * G + h) * D + FPV * grp;
#pragma unroll
      for (int mt = 0; mt < NMT; mt++) {
        pr[2 * mt] = st.o[mt][c] * kPvUnscale;
        pr[2 * mt + 1] = st.o[mt][2 + c] * kPvUnscale;
      }
    }
  }
  __syncthreads();
  // the CTA's partial state, relative to its own maximum
  float* ps = p.tc_scratch + (size_t)slots * R * GP + ((size_t)u * NS + seg) * tc_partial_floats<D, G>();
  for (int e = tid; e < G * D; e += kTcThreads) {
    const int h = e / D;
    float M = -INFINITY;
    for (int w = 0; w < kTcWarps; w++) M = fmaxf(M, s_mw[w][h]);
    float o = 0.0f;
    for (int w = 0; w < kTcWarps; w++)
      if (s_mw[w][h] != -INFINITY) o = fmaf(ex2(s_mw[w][h] - M), part[((size_t)w * G + h) * D + (e % D)], o);
    ps[e] = o;
  }
  if (tid < G) {
    float M = -INFINITY, Z = 0.0f, ZS = 0.0f;
    for (int w = 0; w < kTcWarps; w++) M = fmaxf(M, s_mw[w][tid]);
    for (int w = 0; w < kTcWarps; w++)
      if (s_mw[w][tid] != -INFINITY) {
        const float f = ex2(s_mw[w][tid] - M);
        Z = fmaf(f, s_zw[w][tid], Z);
        ZS = fmaf(f, s_zsw[w][tid], ZS);
      }
    ps[G * D + tid] = M;
    ps[G * D + 8 + tid] = Z;
    ps[G * D + 16 + tid] = ZS;
  }
}

// merge + significance: CTA (u, s) combines the unit's NS partial states (every CTA of the unit, so that none
// waits for another; CTA s = 0 writes the output), then runs the significance pass (Q33) of its share of the unit's
// logit rows and leaves its section minima candidates after its partial state; attend_tc_minima_kernel reduces them.
template <int D, int G>
__global__ void __launch_bounds__(kTcThreads)
attend_tc_merge_kernel(PoolDev p, float* __restrict__ out, float* __restrict__ probs, int NS, int slots) {
  constexpr int GP = G <= 4 ? 4 : 8, PF = tc_partial_floats<D, G>();
  using HI = TcCls<D, 16, 8, 4>;
  using LO = TcCls<D, 32, 4, 2>;
  extern __shared__ __align__(16) int32_t tm_pid[];               // [npg] page IDs
  __shared__ float s_f[kTcSplitMax][8], s_C[8], s_iZ[8];
  __shared__ unsigned long long s_min[2];
  __shared__ int s_slot[2];
  const int tid = threadIdx.x, u = blockIdx.x, seg = blockIdx.y;
  if (ld_volatile(&p.ctrl->status) != 0) return;
  const int r = fdiv(p.div_LyH, u);
  if (p.req_state[r] != DKV_REQ_ACTIVE) return;
  const int L = p.L, W = p.W, R = p.tc_slot_rows;
  const ClassGeom gh = p.g[1], gl = p.g[2];
  const int N = p.seq_len[r];
  const int nh = p.n_h[u], nl = p.n_l[u];
  const int nw = min(W, N), Ts = nh + nl;
  const int ph = (nh + HI::C - 1) / HI::C, pl = (nl + LO::C - 1) / LO::C, npg = ph + pl;
  const int lo0 = HI::C * ph, wb = lo0 + LO::C * pl;
  const int32_t* trow = p.table + (size_t)u * L;
  for (int k = tid; k < npg; k += kTcThreads) tm_pid[k] = k < ph ? trow[k] : trow[L - 1 - (k - ph)];
  if (tid < 2) { s_min[tid] = ~0ull; s_slot[tid] = -1; }
  float* const ps0 = p.tc_scratch + (size_t)slots * R * GP + (size_t)u * NS * PF;
  if (tid < G) {
    float M = -INFINITY;
    for (int s = 0; s < NS; s++) M = fmaxf(M, ps0[(size_t)s * PF + G * D + tid]);
    float Z = 0.0f;
    for (int s = 0; s < NS; s++) {
      const float ms = ps0[(size_t)s * PF + G * D + tid];
      const float f = ms == -INFINITY ? 0.0f : ex2(ms - M);
      s_f[s][tid] = f;
      Z = fmaf(f, ps0[(size_t)s * PF + G * D + 8 + tid], Z);
    }
    s_C[tid] = Z > 0.0f ? M + log2f(Z) : INFINITY;
    s_iZ[tid] = Z > 0.0f ? 1.0f / Z : 0.0f;
  }
  __syncthreads();
  if (out != nullptr && seg == 0)
    for (int e = tid; e < G * D; e += kTcThreads) {
      const int h = e / D;
      float o = 0.0f;
      for (int s = 0; s < NS; s++) o = fmaf(s_f[s][h], ps0[(size_t)s * PF + e] + ps0[(size_t)s * PF + G * D + 16 + h], o);
      out[(size_t)u * G * D + e] = o * s_iZ[h];
    }
  // significance (Q33) of this CTA's rows: a thread per row, 4 rows in flight
  const float* lg = p.tc_scratch + (size_t)u * R * GP;
  const int rows = wb + nw, r0 = (int)((long)seg * rows / NS), r1 = (int)((long)(seg + 1) * rows / NS);
  unsigned long long mkey[2] = {~0ull, ~0ull};
  int mslot[2] = {-1, -1};
  constexpr int kB = 4;
  for (int base = r0 + tid; base < r1; base += kB * kTcThreads) {
    float xv[kB], sgv[kB];
    int posv[kB], rrv[kB];
    float* spv[kB];
#pragma unroll
    for (int b = 0; b < kB; b++) {
      const int row = base + b * kTcThreads;
      const bool stored = row < wb, hi = row < lo0;
      const int rr = hi ? row : row - lo0;
      spv[b] = nullptr;
      rrv[b] = rr;
      if (row >= r1 || (stored && rr >= (hi ? nh : nl))) continue;
      float xm = -INFINITY;
#pragma unroll
      for (int h = 0; h < G; h++) xm = fmaxf(xm, lg[(size_t)row * GP + h] - s_C[h]);
      xv[b] = xm;
      if (stored) {
        const int k = hi ? row >> 4 : ph + (rr >> 5), j = hi ? row & 15 : rr & 31;
        const ClassGeom& gg = hi ? gh : gl;
        uint8_t* pg = p.pages + (size_t)tm_pid[k] * (size_t)p.page_bytes;
        posv[b] = *reinterpret_cast<const int32_t*>(pg + gg.off_pos + 4 * j);
        spv[b] = reinterpret_cast<float*>(pg + gg.off_score + 4 * j);
      } else {
        posv[b] = N - nw + (row - wb);
        spv[b] = p.win_sig + (size_t)u * W + fmod_(p.div_W, posv[b]);
      }
      sgv[b] = *spv[b];
    }
#pragma unroll
    for (int b = 0; b < kB; b++) {
      if (spv[b] == nullptr) continue;
      const int row = base + b * kTcThreads, pos = posv[b], rr = rrv[b];
      const float a = ex2(xv[b]);
      float sg = sgv[b];
      const int c = N - 2 - pos;
      if (c >= 0) {
        sg = __fdividef(fmaf(sg, (float)c, a), (float)(c + 1));
        *spv[b] = sg;
      }
      if (row < wb) {
        const bool hi = row < lo0;
        if (probs) probs[(size_t)u * p.M + (hi ? rr : nh + rr)] = a;
        const int cls = hi ? 0 : 1;
        const unsigned long long key = ((unsigned long long)__float_as_uint(sg) << 32) | (uint32_t)pos;
        if (key < mkey[cls]) { mkey[cls] = key; mslot[cls] = rr; }
      } else if (probs) {
        probs[(size_t)u * p.M + Ts + (row - wb)] = a;
      }
    }
  }
#pragma unroll
  for (int c = 0; c < 2; c++)
    if (mkey[c] != ~0ull) atomicMin(&s_min[c], mkey[c]);
  __syncthreads();
#pragma unroll
  for (int c = 0; c < 2; c++)
    if (mkey[c] != ~0ull && mkey[c] == s_min[c]) s_slot[c] = mslot[c];
  __syncthreads();
  if (tid == 0) {                                                 // this CTA's candidates, after its partial state
    uint32_t* mc = reinterpret_cast<uint32_t*>(ps0 + (size_t)seg * PF + G * D + 24);
#pragma unroll
    for (int c = 0; c < 2; c++) {
      mc[3 * c] = (uint32_t)(s_min[c] >> 32);
      mc[3 * c + 1] = (uint32_t)(s_min[c] & 0xFFFFFFFFull);
      mc[3 * c + 2] = (uint32_t)s_slot[c];
    }
  }
}

// the section minima of a split unit: the smallest (significance, position) key over its NS CTAs' candidates
template <int D, int G>
__global__ void attend_tc_minima_kernel(PoolDev p, int NS, int slots) {
  constexpr int GP = G <= 4 ? 4 : 8, PF = tc_partial_floats<D, G>();
  const int u = blockIdx.x, c = threadIdx.x;                      // c: section (0 high, 1 low)
  if (c >= 2 || ld_volatile(&p.ctrl->status) != 0) return;
  if (p.req_state[fdiv(p.div_LyH, u)] != DKV_REQ_ACTIVE) return;
  const float* ps0 = p.tc_scratch + (size_t)slots * p.tc_slot_rows * GP + (size_t)u * NS * PF;
  unsigned long long best = ~0ull;
  int slot = -1;
  for (int s = 0; s < NS; s++) {
    const uint32_t* mc = reinterpret_cast<const uint32_t*>(ps0 + (size_t)s * PF + G * D + 24) + 3 * c;
    const unsigned long long key = ((unsigned long long)mc[0] << 32) | mc[1];
    if (key < best) { best = key; slot = (int)mc[2]; }
  }
  int32_t* m = p.secmin + 8 * (size_t)u;
  m[3 * c] = (int32_t)(uint32_t)(best >> 32);
  m[3 * c + 1] = (int32_t)(uint32_t)(best & 0xFFFFFFFFull);
  m[3 * c + 2] = slot;
  if (c == 0) m[6] = 1;
}

// the kernel is specialised for the paper's classes: K8V4 in 16-token pages, K4V2 in 32-token pages,
// with the §4 segment order (K codes, K meta, V codes, V meta, scores, positions); other geometries take the
// exact path
template <int D>
static bool geom_is(const ClassGeom& g, int C, int kb, int vb) {
  const int kr = D * kb / 8, vr = D * vb / 8;
  return g.C == C && g.kbits == kb && g.vbits == vb && g.k_row == kr && g.v_row == vr && g.off_k == 0 &&
         g.off_kmeta == C * kr && g.off_v == C * kr + 4 * C && g.off_vmeta == C * kr + 4 * C + C * vr;
}
bool attend_tc_supported(const PoolDev& p) {
  if (!(p.G >= 1 && p.G <= 8 && (p.d == 64 || p.d == 128) && p.tc_scratch != nullptr)) return false;
  return p.d == 128 ? geom_is<128>(p.g[1], 16, 8, 4) && geom_is<128>(p.g[2], 32, 4, 2)
                    : geom_is<64>(p.g[1], 16, 8, 4) && geom_is<64>(p.g[2], 32, 4, 2);
}

size_t attend_tc_smem_bytes(const PoolDev& p) {
  const int stg = p.d == 128 ? tc_stage_bytes<128>() : tc_stage_bytes<64>();
  return (size_t)tc_area_bytes(p.d, p.G, stg) + (size_t)2 * ((p.L + 4) & ~3) * 4;
}

template <int D, int G>
static cudaError_t launch_tc(const PoolDev& p, const uint16_t* q, float* out, float* probs, int active_units,
                             int max_len, cudaStream_t s) {
  const size_t smem = attend_tc_smem_bytes(p);
  cudaError_t e = cudaFuncSetAttribute(attend_tc_kernel<D, G>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  if (e != cudaSuccess) return e;
  int dev = 0, sms = 0, per_sm = 0;
  if ((e = cudaGetDevice(&dev)) != cudaSuccess) return e;
  if ((e = cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev)) != cudaSuccess) return e;
  if ((e = cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, attend_tc_kernel<D, G>, kTcThreads, smem)) != cudaSuccess)
    return e;
  int grid = sms * (per_sm > 0 ? per_sm : 1);
  if (grid > p.tc_slots) grid = p.tc_slots;                       // two scratch buffers per CTA slot
  // split-sequence form: at most half as many active units as resident CTAs, long enough to share (>= 2048
  // tokens, >= 8 pages per segment), and the partial states fit the scratch's second half
  const int pages = max_len / 16;
  int NS = 1;
  if (DKV_TC_SPLIT && active_units > 0 && 2 * active_units <= grid && max_len >= 2048 && p.U <= p.tc_slots) {
    NS = grid / active_units;
    if (NS > kTcSplitMax) NS = kTcSplitMax;
    if (NS > pages / 8) NS = pages / 8;
    const long cap = (long)p.tc_slots * p.tc_slot_rows * (G <= 4 ? 4 : 8) / ((long)p.U * tc_partial_floats<D, G>());
    if (NS > cap) NS = (int)cap;
  }
  if (NS >= 2) {
    e = cudaFuncSetAttribute(attend_tc_split_kernel<D, G>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    if (e != cudaSuccess) return e;
    attend_tc_split_kernel<D, G><<<dim3(p.U, NS), kTcThreads, smem, s>>>(p, q, NS, p.tc_slots);
    if ((e = cudaGetLastError()) != cudaSuccess) return e;
    const size_t msm = (size_t)((p.L + 3) & ~3) * 4;
    if (msm > 48 * 1024 &&
        (e = cudaFuncSetAttribute(attend_tc_merge_kernel<D, G>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)msm)) != cudaSuccess)
      return e;
    attend_tc_merge_kernel<D, G><<<dim3(p.U, NS), kTcThreads, msm, s>>>(p, out, probs, NS, p.tc_slots);
    if ((e = cudaGetLastError()) != cudaSuccess) return e;
    attend_tc_minima_kernel<D, G><<<p.U, 32, 0, s>>>(p, NS, p.tc_slots);
    return cudaGetLastError();
  }
  if (grid > p.U) grid = p.U;
  attend_tc_kernel<D, G><<<grid, kTcThreads, smem, s>>>(p, q, out, probs);
  return cudaGetLastError();
}

template <int D>
static cudaError_t launch_tc_d(const PoolDev& p, const uint16_t* q, float* out, float* probs, int au, int ml,
                               cudaStream_t s) {
  switch (p.G) {
    case 1: return launch_tc<D, 1>(p, q, out, probs, au, ml, s);
    case 2: return launch_tc<D, 2>(p, q, out, probs, au, ml, s);
    case 4: return launch_tc<D, 4>(p, q, out, probs, au, ml, s);
    case 5: return launch_tc<D, 5>(p, q, out, probs, au, ml, s);
    case 7: return launch_tc<D, 7>(p, q, out, probs, au, ml, s);
    default: return launch_tc<D, 8>(p, q, out, probs, au, ml, s);
  }
}

// active_units / max_len: the ACTIVE requests' units and longest length (host mirror), which choose the form
cudaError_t launch_attend_tc(const PoolDev& p, const uint16_t* q, float* out, float* probs, int active_units,
                             int max_len, cudaStream_t s) {
  return p.d == 128 ? launch_tc_d<128>(p, q, out, probs, active_units, max_len, s)
                    : launch_tc_d<64>(p, q, out, probs, active_units, max_len, s);
}

}  // namespace dkv
