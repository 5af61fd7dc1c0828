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
// scaled by 2^12, split into fp16 hi + lo (22 significant bits, two MMAs).  The FP16 window (<= W tokens) runs on CUDA
// cores in fp32.
//
// One CTA per unit (the paper's "one thread block per head"), kTcWarps warps; pages go round-robin to
// the warps, high pages first, then low, each staged into shared memory by per-thread 16-B cp.async
// copies (kTcStages pages in flight per warp).  The MMA fragments are read straight from the staged code rows; the paper's
// tiled K/V layouts (NEXT-3) exist to make per-thread vector loads coalesce in global memory — here
// whole page segments are copied (contiguous 1-2 KB runs, coalesced by construction) and the tiling happens in
// shared memory: a 16-B XOR swizzle of each code row so that the fragment reads are bank-conflict free, and a
// permutation of the MMA k index (k = 2j, 2j+1, 2j+8, 2j+9 <-> features / tokens 4j .. 4j+3) so that a thread's
// four codes are adjacent in a row.
//   phase 1: logits of every token (stored pages by MMA, window on CUDA cores) into shared memory;
//   phase 2: per-head max, p = exp(l - max), Z (order-free fp32 sums);
//   phase 3: PV by MMA page by page with a = p / Z, the significance of each stored token (page score
//            segments) and window token, the section minima; the warps' partial outputs are added in a fixed
//            order (deterministic for a given launch).
#include <cuda_bf16.h>

#include "dkv_internal.cuh"

namespace dkv {

#ifndef DKV_TC_MINB
#define DKV_TC_MINB 3           // CTAs per SM the register budget is sized for
#endif
constexpr int kTcWarps = 8;
constexpr int kTcThreads = kTcWarps * 32;
constexpr int kTcStages = 2;                   // pages in flight per warp (cp.async groups)
// bytes per warp per stage: >= C*k_row + 4C (K codes + meta) and C*v_row + 12C + C*GP*4 (V codes, meta, scores,
// positions, the page's probability rows), for both classes at d <= 128
constexpr int tc_stage_bytes(int GP) { return GP == 4 ? 2176 : 2432; }
// the stage area, reused by phase 3's reduction (warp partials, z sums, the staged window values; phase 1 stages the
// window keys there too), rounded to 16 B
__host__ __device__ constexpr int tc_area_bytes(int D, int G, int W, int GP) {
  return ((kTcWarps * kTcStages * tc_stage_bytes(GP) > kTcWarps * G * D * 4 + ((kTcWarps * G + 3) & ~3) * 4 + W * D * 2
               ? kTcWarps * kTcStages * tc_stage_bytes(GP)
               : kTcWarps * G * D * 4 + ((kTcWarps * G + 3) & ~3) * 4 + W * D * 2) + 15) & ~15;
}

__device__ __forceinline__ void mma_f16(float (&d)[4], const uint32_t (&a)[4], uint32_t b0, uint32_t b1) {
  asm volatile("mma.sync.aligned.m16n8k16.row.col.f32.f16.f16.f32 {%0,%1,%2,%3}, {%4,%5,%6,%7}, {%8,%9}, "
               "{%0,%1,%2,%3};"
               : "+f"(d[0]), "+f"(d[1]), "+f"(d[2]), "+f"(d[3])
               : "r"(a[0]), "r"(a[1]), "r"(a[2]), "r"(a[3]), "r"(b0), "r"(b1));
}
__device__ __forceinline__ void mma_bf16(float (&d)[4], const uint32_t (&a)[4], uint32_t b0, uint32_t b1) {
  asm volatile("mma.sync.aligned.m16n8k16.row.col.f32.bf16.bf16.f32 {%0,%1,%2,%3}, {%4,%5,%6,%7}, {%8,%9}, "
               "{%0,%1,%2,%3};"
               : "+f"(d[0]), "+f"(d[1]), "+f"(d[2]), "+f"(d[3])
               : "r"(a[0]), "r"(a[1]), "r"(a[2]), "r"(a[3]), "r"(b0), "r"(b1));
}

// two integer codes (< 1024) -> fp16x2 {c0, c1} exactly: 0x6400 | c = 1024 + c, minus 1024
__device__ __forceinline__ uint32_t h2_codes(uint32_t c0, uint32_t c1) {
  const uint32_t w = c0 | (c1 << 16) | 0x64006400u;
  const __half2 r = __hsub2(*reinterpret_cast<const __half2*>(&w), __halves2half2(__ushort_as_half(0x6400), __ushort_as_half(0x6400)));
  return *reinterpret_cast<const uint32_t*>(&r);
}
// two integer codes (< 256) -> bf16x2 exactly: 0x4300 | c = 128 + c, minus 128
__device__ __forceinline__ uint32_t bf2_codes(uint32_t c0, uint32_t c1) {
  const uint32_t w = c0 | (c1 << 16) | 0x43004300u;
  const uint32_t k = 0x43004300u;
  const __nv_bfloat162 r = __hsub2(*reinterpret_cast<const __nv_bfloat162*>(&w), *reinterpret_cast<const __nv_bfloat162*>(&k));
  return *reinterpret_cast<const uint32_t*>(&r);
}
// fp32 pair -> bf16x2 hi parts and the bf16x2 of the remainders (x = hi + lo to 16 significant bits)
__device__ __forceinline__ void bf2_split(float x0, float x1, uint32_t& hi, uint32_t& lo) {
  const __nv_bfloat162 h = __floats2bfloat162_rn(x0, x1);
  const float2 hf = __bfloat1622float2(h);
  const __nv_bfloat162 l = __floats2bfloat162_rn(x0 - hf.x, x1 - hf.y);
  hi = *reinterpret_cast<const uint32_t*>(&h);
  lo = *reinterpret_cast<const uint32_t*>(&l);
}

// Exact code -> fp16 / bf16 conversion with byte permutes: a w-bit field whose lowest bit sits at mantissa bit b
// of a half with exponent chosen so that that bit weighs exactly 1 (magic M) holds the value M + code; one
// subtraction of M (exact) leaves the code.  x2 = [f0 in the low half | f1 in the high half] after masking.
__device__ __forceinline__ uint32_t hsub2_u(uint32_t x, uint32_t m) {
  const __half2 r = __hsub2(*reinterpret_cast<const __half2*>(&x), *reinterpret_cast<const __half2*>(&m));
  return *reinterpret_cast<const uint32_t*>(&r);
}
__device__ __forceinline__ uint32_t bsub2_u(uint32_t x, uint32_t m) {
  const __nv_bfloat162 r = __hsub2(*reinterpret_cast<const __nv_bfloat162*>(&x), *reinterpret_cast<const __nv_bfloat162*>(&m));
  return *reinterpret_cast<const uint32_t*>(&r);
}
// (x & MASK) | magic in one LOP3 (the compiler splits it into two when both constants are immediates; the magic
// lives in a register)
template <uint32_t MASK>
__device__ __forceinline__ uint32_t and_or(uint32_t x, uint32_t magic) {
  uint32_t d;
  asm("lop3.b32 %0, %1, %2, %3, 0xEA;" : "=r"(d) : "r"(x), "n"(MASK), "r"(magic));
  return d;
}
// K8: bytes (c0, c1, c2, c3) of x -> fp16x2 (c0, c1) and (c2, c3): 0x64XX = 1024 + XX
// The subtraction stays per pair.  Measured alternative (r2v): operands left at M + code with a second MMA whose A
// operand is the constant -M removing the bias after each group — 10 % fewer instructions but slower (3.82 vs
// 3.72 ms: dependent MMA pairs on one accumulator) and outside the Eq. 1 output tolerance (8e-5: the accumulator
// transiently holds M * sum at the tensor core's accumulation precision).
// Centred codes: the subtrahend is M + 2^(bits-1), not M, so the operand is the code minus half its range (exact
// in fp16) and the offset moves into z (z' = z + 2^(bits-1) s, tc_zc).  The code term and the z term of the output
// (and of the logit) then no longer nearly cancel — with raw codes both are ~|mean V| and their difference is the
// output, so the tensor core's fp32 accumulation error over a long context (one rounding per MMA, ~thousands per
// accumulator at 30k tokens) was amplified into the output.
__device__ __forceinline__ uint32_t unbias(uint32_t x, uint32_t m) { return hsub2_u(x, m); }
template <int BITS>
__device__ __forceinline__ float tc_zc(float zf, float sf) { return fmaf(sf, (float)(1 << (BITS - 1)), zf); }
__device__ __forceinline__ void k8_pairs(uint32_t x, uint32_t& lo, uint32_t& hi) {
  lo = unbias(__byte_perm(x, 0x64646464u, 0x4140), 0x64806480u);   // (1024 + c) - 1152 = c - 128
  hi = unbias(__byte_perm(x, 0x64646464u, 0x4342), 0x64806480u);
}
// K4: the two bytes at byte index KB0 (codes n0 | n1 << 4) and KB0 + 1 (n2 | n3 << 4) of x -> fp16x2 (n0, n1),
// (n2, n3): n0 in bits 0-3 with 0x6400 (1024, ulp 1), n1 in bits 20-23 = bits 4-7 of the high half with 0x5400
// (64, ulp 1/16)
template <int KB0>
__device__ __forceinline__ void k4_pairs(uint32_t x, uint32_t& lo, uint32_t& hi) {
  constexpr uint32_t s0 = KB0 * 0x1111u, s1 = (KB0 + 1) * 0x1111u;
  lo = unbias(and_or<0x00F0000Fu>(__byte_perm(x, 0u, s0), 0x54006400u), 0x54806408u);   // c - 8 in both halves
  hi = unbias(and_or<0x00F0000Fu>(__byte_perm(x, 0u, s1), 0x54006400u), 0x54806408u);
}
// V: byte K of x (token j0) and of y (token j1) -> fp16x2 (field of j0, field of j1) for the field at bits
// [SH, SH + VB) of that byte; the magic makes bit SH weigh 1 (fp16, 10 mantissa bits: a value in [2^e, 2^(e+1))
// has ulp 2^(e-10), so e = 10 - SH: 1024 (0x6400) for SH = 0, 256 (0x5C00) for 2, 64 (0x5400) for 4, 16 (0x4C00)
// for 6)
template <int K, int SH, int VB>
__device__ __forceinline__ uint32_t v_pair(uint32_t x, uint32_t y) {
  constexpr uint32_t sel = K | (K << 4) | ((4 + K) << 8) | ((4 + K) << 12);
  constexpr uint32_t mask = (((1u << VB) - 1u) << SH) * 0x00010001u;
  constexpr uint32_t magic = (SH == 0 ? 0x6400u : SH == 2 ? 0x5C00u : SH == 4 ? 0x5400u : 0x4C00u) * 0x00010001u;
  constexpr uint32_t centre = magic + ((1u << (VB - 1)) << SH) * 0x00010001u;   // M + 2^(VB-1): code - half range
  return unbias(and_or<mask>(__byte_perm(x, y, sel), magic), centre);
}

// fp32 pair -> fp16x2 hi parts and the fp16x2 of the remainders (x = hi + lo to 22 significant bits)
__device__ __forceinline__ void h2_split(float x0, float x1, uint32_t& hi, uint32_t& lo) {
  const __half2 h = __floats2half2_rn(x0, x1);
  const float2 hf = __half22float2(h);
  const __half2 l = __floats2half2_rn(x0 - hf.x, x1 - hf.y);
  hi = *reinterpret_cast<const uint32_t*>(&h);
  lo = *reinterpret_cast<const uint32_t*>(&l);
}
// PV's B operand p * s_v (p = exp(l - max) <= 1, unnormalised, so that long contexts' small probabilities do not
// sink into fp16 subnormals; 1/Z is applied to the partials) is scaled by 2^12 before its fp16 split (|s_v| < 2^4
// keeps it below the fp16 maximum); the accumulators are scaled back once
constexpr float kPvScale = 4096.0f, kPvUnscale = 1.0f / 4096.0f;

// Compile-time geometry of one precision class (the paper's K8V4 high / K4V2 low pages): tokens per
// page, bit widths, code row bytes, 16-B chunks per row and the row swizzle shifts of the staged copies.
template <int D, int C_, int KB, int VB>
struct TcCls {
  static constexpr int C = C_, kbits = KB, vbits = VB;
  static constexpr int k_row = D * KB / 8, v_row = D * VB / 8;
  static constexpr int kc = k_row / 16, vc = v_row / 16;               // chunks per row (>= 1 for D >= 64)
  // fragment reads touch rows grp (8 consecutive) at the same byte: shift so those rows' chunks differ
  static constexpr int ksh = k_row >= 128 ? 0 : (k_row == 64 ? 1 : (k_row == 32 ? 2 : 3));
  static constexpr int vsh = 2;                                        // V fragment rows: tokens 4j .. 4j+3
  static_assert(k_row >= 16 && v_row >= 16, "rows of at least one 16-B chunk");
};
template <int KC, int SH>
__device__ __forceinline__ int swz_off(int row, int byte, int row_bytes) {
  return row * row_bytes + ((((byte >> 4) ^ ((row >> SH) & (KC - 1)))) << 4) + (byte & 15);
}

// a page's staged segments: codes (rows swizzled) + 4C-byte segments, per-thread 16-B cp.async
template <int ROW, int KC, int SH, int C>
__device__ __forceinline__ void stage_codes(uint8_t* dst, const uint8_t* src, int lane) {
  constexpr int n = C * KC;
#pragma unroll
  for (int j = lane; j < n; j += 32) {
    const int r = j / KC, c = j % KC;
    cp_async16(dst + r * ROW + ((c ^ ((r >> SH) & (KC - 1))) << 4), src + (size_t)j * 16, true);
  }
}
template <int BYTES>
__device__ __forceinline__ void stage_seg(uint8_t* dst, const uint8_t* src, int lane) {
#pragma unroll
  for (int o = 16 * lane; o < BYTES; o += 512) cp_async16(dst + o, src + o, true);
}

// Loads `BYTES` contiguous bytes of a staged, swizzled row starting at byte `b0` (a multiple of BYTES, BYTES in
// {2, 4, 8, 16, 32}) into 32-bit words.
template <int BYTES, int KC, int SH>
__device__ __forceinline__ void lds_row(const uint8_t* seg, int row, int row_bytes, int b0, uint32_t (&w)[(BYTES + 3) / 4]) {
  if constexpr (BYTES >= 16) {
#pragma unroll
    for (int c = 0; c < BYTES / 16; c++) {
      const uint4 v = *reinterpret_cast<const uint4*>(seg + swz_off<KC, SH>(row, b0 + 16 * c, row_bytes));
      w[4 * c] = v.x; w[4 * c + 1] = v.y; w[4 * c + 2] = v.z; w[4 * c + 3] = v.w;
    }
  } else if constexpr (BYTES == 8) {
    const uint2 v = *reinterpret_cast<const uint2*>(seg + swz_off<KC, SH>(row, b0, row_bytes));
    w[0] = v.x; w[1] = v.y;
  } else if constexpr (BYTES == 4) {
    w[0] = *reinterpret_cast<const uint32_t*>(seg + swz_off<KC, SH>(row, b0, row_bytes));
  } else {
    w[0] = *reinterpret_cast<const uint16_t*>(seg + swz_off<KC, SH>(row, b0, row_bytes));
  }
}

// QK^T of one staged page: logits of its tokens (all G heads) into lg; running max of this lane's two heads.
// MMA k index <-> feature: in group g, lane tig supplies features FPK*tig + 4g + {0,1 | 2,3} (k = 2 tig, 2 tig + 1 |
// 2 tig + 8, 2 tig + 9), FPK = D/4, so a lane's codes for all groups are one contiguous run of its key row.
template <int D, int G, int GP, class CL>
__device__ __forceinline__ void qk_page(const uint8_t* kseg, int t0, int cnt, const uint32_t (&qb)[D / 16][2],
                                        const float* qsum, float scale, float* lg, float (&mx)[2], int grp, int tig) {
  constexpr int FPK = D / 4, RB = FPK * CL::kbits / 8;           // features / bytes per lane per key row
  constexpr int NW = (RB + 3) / 4;
  const uint32_t* kmeta = reinterpret_cast<const uint32_t*>(kseg + CL::C * CL::k_row);
#pragma unroll
  for (int tile = 0; tile < CL::C / 16; tile++) {
    if (tile * 16 >= cnt) break;
    float acc2[2][4] = {{0.f, 0.f, 0.f, 0.f}, {0.f, 0.f, 0.f, 0.f}};   // even / odd groups: two MMA chains
    uint32_t w[2][NW];
    lds_row<RB, 1, 0>(kseg, tile * 16 + grp, CL::k_row, RB * tig, w[0]);
    lds_row<RB, 1, 0>(kseg, tile * 16 + grp + 8, CL::k_row, RB * tig, w[1]);
#pragma unroll
    for (int g = 0; g < D / 16; g++) {
      uint32_t a[4];                                             // a0 / a1: k = 2 tig, 2 tig + 1 (rows grp, grp + 8)
#pragma unroll                                                   // a2 / a3: k = 2 tig + 8, 2 tig + 9
      for (int rr = 0; rr < 2; rr++) {
        if constexpr (CL::kbits == 8) {
          k8_pairs(w[rr][g], a[rr], a[2 + rr]);                  // features 4g .. 4g+3 = word g of the run
        } else {
          static_assert(CL::kbits == 4, "tensor-core path: K8 or K4 keys");
          if (g & 1) k4_pairs<2>(w[rr][g >> 1], a[rr], a[2 + rr]);   // bytes 2g, 2g+1 of the run
          else k4_pairs<0>(w[rr][g >> 1], a[rr], a[2 + rr]);
        }
      }
      mma_f16(acc2[g & 1], a, qb[g][0], qb[g][1]);
    }
    float acc[4];
#pragma unroll
    for (int e = 0; e < 4; e++) acc[e] = acc2[0][e] + acc2[1][e];
#pragma unroll
    for (int hh = 0; hh < 2; hh++) {                             // rows grp, grp + 8
      const int j = tile * 16 + grp + 8 * hh;
      if (j < cnt) {
        const uint32_t km = kmeta[j];
        const float sf = __half2float(__ushort_as_half((unsigned short)(km & 0xFFFFu)));
        const float zf = tc_zc<CL::kbits>(__half2float(__ushort_as_half((unsigned short)(km >> 16))), sf);
#pragma unroll
        for (int c = 0; c < 2; c++) {
          const int h = 2 * tig + c;
          if (h < G) {
            const float l = (sf * acc[2 * hh + c] + zf * qsum[h]) * scale;
            lg[(size_t)(t0 + j) * GP + h] = l;
            mx[c] = fmaxf(mx[c], l);
          }
        }
      }
    }
  }
}

// PV of one staged page into the warp's accumulators + the z term.  MMA m index <-> feature: in m-tile g, row grp
// is feature FPV*grp + 2g and row grp + 8 is FPV*grp + 2g + 1 (FPV = D/8), so a lane's value codes for all
// m-tiles are one contiguous run of each value row; k = tokens 4 tig .. 4 tig + 3; n = head.
template <int D, int G, int GP, class CL>
__device__ __forceinline__ void pv_page(const uint8_t* vseg, int t0, int cnt, const float* lg,
                                        float (&acc)[D / 16][4], float& zsum, int grp, int tig) {
  constexpr int FPV = D / 8, RB = FPV * CL::vbits / 8;           // features / bytes per lane per value row
  constexpr int NW = (RB + 3) / 4;
  const uint32_t* vmeta = reinterpret_cast<const uint32_t*>(vseg + CL::C * CL::v_row);
#pragma unroll
  for (int tile = 0; tile < CL::C / 16; tile++) {
    if (tile * 16 >= cnt) break;
    float bv[4];
#pragma unroll
    for (int jj = 0; jj < 4; jj++) {
      const int j = tile * 16 + tig + 4 * jj;                    // k = 2 tig, 2 tig + 1, +8, +9 <-> tig + 4 jj
      float b = 0.0f;
      if (j < cnt && grp < G) {
        const uint32_t vm = vmeta[j];
        const float sf = __half2float(__ushort_as_half((unsigned short)(vm & 0xFFFFu)));
        const float zf = tc_zc<CL::vbits>(__half2float(__ushort_as_half((unsigned short)(vm >> 16))), sf);
        const float a = lg[(size_t)(t0 + j) * GP + grp];         // unnormalised p = exp(l - max) <= 1
        b = a * sf * kPvScale;
        zsum = fmaf(a, zf, zsum);
      }
      bv[jj] = b;
    }
    uint32_t bh0, bl0, bh1, bl1;
    h2_split(bv[0], bv[1], bh0, bl0);
    h2_split(bv[2], bv[3], bh1, bl1);
    uint32_t w[4][NW];
#pragma unroll
    for (int jj = 0; jj < 4; jj++) lds_row<RB, 1, 0>(vseg, tile * 16 + tig + 4 * jj, CL::v_row, RB * grp, w[jj]);
#pragma unroll
    for (int g = 0; g < D / 16; g++) {
      // features 2g, 2g + 1 of the lane's run: V4 -> byte g (low / high nibble); V2 -> byte g/2, crumbs at bits
      // 4(g&1) and 4(g&1) + 2.  a0 / a2: feature row grp (f0), tokens (4 tig, 4 tig+1) / (4 tig+2, 4 tig+3);
      // a1 / a3: feature row grp + 8 (f0 + 1)
      uint32_t a[4];
      if constexpr (CL::vbits == 4) {
        const int wi = g >> 2;
        switch (g & 3) {
#define DKV_V4(K)                                                                             \
          case K:                                                                             \
            a[0] = v_pair<K, 0, 4>(w[0][wi], w[1][wi]); a[1] = v_pair<K, 4, 4>(w[0][wi], w[1][wi]); \
            a[2] = v_pair<K, 0, 4>(w[2][wi], w[3][wi]); a[3] = v_pair<K, 4, 4>(w[2][wi], w[3][wi]); \
            break;
          DKV_V4(0) DKV_V4(1) DKV_V4(2) DKV_V4(3)
#undef DKV_V4
        }
      } else {
        static_assert(CL::vbits == 2, "tensor-core path: V4 or V2 values");
        const int wi = g >> 3;
        switch (g & 7) {
#define DKV_V2(G8)                                                                                      \
          case G8:                                                                                      \
            a[0] = v_pair<(G8 & 7) / 2, 4 * (G8 & 1), 2>(w[0][wi], w[1][wi]);                          \
            a[1] = v_pair<(G8 & 7) / 2, 4 * (G8 & 1) + 2, 2>(w[0][wi], w[1][wi]);                      \
            a[2] = v_pair<(G8 & 7) / 2, 4 * (G8 & 1), 2>(w[2][wi], w[3][wi]);                          \
            a[3] = v_pair<(G8 & 7) / 2, 4 * (G8 & 1) + 2, 2>(w[2][wi], w[3][wi]);                      \
            break;
          DKV_V2(0) DKV_V2(1) DKV_V2(2) DKV_V2(3) DKV_V2(4) DKV_V2(5) DKV_V2(6) DKV_V2(7)
#undef DKV_V2
        }
      }
      mma_f16(acc[g], a, bh0, bh1);
      mma_f16(acc[g], a, bl0, bl1);
    }
  }
}

// Persistent: gridDim.x CTAs (the occupancy limit, at most kTcSlots) take units blockIdx.x, + gridDim.x, ...  A
// CTA's logits live in its own global scratch slot (p.tc_scratch: [tc_slot_rows][GP] fp32; the slots of the
// resident CTAs, ~70 MB at configs[1], stay in L2), so shared memory holds only the page stages and the per-unit
// reduction area and three CTAs fit per SM (logits in shared memory allowed two).  Phase 3 stages each page's
// probability rows together with its value segments (bulk copies).
template <int D, int G>
__global__ void __launch_bounds__(kTcThreads, DKV_TC_MINB)
attend_tc_kernel(PoolDev p, const uint16_t* __restrict__ q, float* __restrict__ out, float* __restrict__ probs) {
  constexpr int GP = G <= 4 ? 4 : 8;                             // logit row: GP floats per token
  constexpr int NG = D / 16;                                      // 16-feature groups (QK k-steps, PV m-tiles)
  constexpr int STG = tc_stage_bytes(GP);                         // bytes per warp per stage
  using HI = TcCls<D, 16, 8, 4>;                                  // K8V4, 16-token pages
  using LO = TcCls<D, 32, 4, 2>;                                  // K4V2, 32-token pages
  extern __shared__ __align__(16) uint8_t tc_smem[];
  __shared__ float s_q[G][D];
  __shared__ float s_qsum[G], s_m[G], s_iz[G];
  __shared__ float s_red[kTcWarps][G];
  __shared__ unsigned long long s_min[2];
  __shared__ int s_slot[2];
  __shared__ __align__(8) uint64_t s_bar[kTcWarps][kTcStages];   // per-warp stage mbarriers (bulk copies)
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int grp = lane >> 2, tig = lane & 3;
  if (ld_volatile(&p.ctrl->status) != 0) return;                  // sticky error: no-op
  const int L = p.L, W = p.W;
  const ClassGeom gh = p.g[1], gl = p.g[2];                       // segment offsets inside a page
  float* const lg = p.tc_scratch + (size_t)blockIdx.x * p.tc_slot_rows * GP;   // this CTA's logits [rows][GP]
  // dynamic shared memory: the stage / reduction area first (a compile-time base), then the page IDs and the
  // window's probability rows
  uint8_t* stage0 = tc_smem;
  int32_t* pid = reinterpret_cast<int32_t*>(tc_smem + tc_area_bytes(D, G, W, GP));
  float* wprob = reinterpret_cast<float*>(pid + ((L + 4) & ~3));     // [W][GP] window probabilities (phase 3)
  uint8_t* mystage = stage0 + (size_t)warp * kTcStages * STG;
  uint64_t* bars = s_bar[warp];
  if (tid < kTcWarps * kTcStages) mbar_init(&s_bar[tid / kTcStages][tid % kTcStages], 1);
  fence_mbar_init();
  uint32_t phase = 0;                                             // bit s: parity of stage s's next completion
  const uint32_t bar_s = smem_u32(bars), stage_s = smem_u32(mystage);
  const float scale = rsqrtf((float)D);
  const uint16_t* const wk_all = reinterpret_cast<const uint16_t*>(p.win_k);
  const uint16_t* const wv_all = reinterpret_cast<const uint16_t*>(p.win_v);

  for (int u = blockIdx.x; u < p.U; u += gridDim.x) {
    const int r = fdiv(p.div_LyH, u);
    if (p.req_state[r] != DKV_REQ_ACTIVE) continue;               // CTA-uniform
    const int N = p.seq_len[r];
    const int nh = p.n_h[u], nl = p.n_l[u];
    const int nw = min(W, N);
    const int Ts = nh + nl, T = Ts + nw;                          // logit rows: stored tokens, then the window
    const int ph = ceil_div(nh, HI::C), pl = ceil_div(nl, LO::C);
    const int npg = ph + pl;
    const int32_t* trow = p.table + (size_t)u * L;
    __syncthreads();                                              // the previous unit's readers are done
    for (int k = tid; k < npg; k += kTcThreads) pid[k] = k < ph ? trow[k] : trow[L - 1 - (k - ph)];
    for (int k = tid; k < G * D; k += kTcThreads)
      s_q[k / D][k % D] = __half2float(__ushort_as_half(q[(size_t)u * G * D + k]));
    if (tid < 2) { s_min[tid] = ~0ull; s_slot[tid] = -1; }
    __syncthreads();
    if (tid < G) {
      float sacc = 0.0f;
      for (int f = 0; f < D; f++) sacc += s_q[tid][f];
      s_qsum[tid] = sacc;
    }
    // B fragments of the queries (k = features, permuted as in qk_page; n = head = grp): group g, b0 = features
    // (D/4) tig + 4g + {0, 1}, b1 = + {2, 3} of head grp
    uint32_t qb[NG][2];
#pragma unroll
    for (int g = 0; g < NG; g++) {
      uint32_t w0 = 0, w1 = 0;
      if (grp < G) {
        const uint2 v = *reinterpret_cast<const uint2*>(q + ((size_t)u * G + grp) * D + (D / 4) * tig + 4 * g);
        w0 = v.x; w1 = v.y;
      }
      qb[g][0] = w0; qb[g][1] = w1;
    }
    __syncthreads();

    auto page_ptr = [&](int k) { return p.pages + (size_t)pid[k] * (size_t)p.page_bytes; };
    const int my_n = npg > warp ? (npg - warp + kTcWarps - 1) / kTcWarps : 0;   // this warp's pages

    // ---- phase 1: logits.  Stored pages: each warp its pages (k = warp + i * kTcWarps), K codes + K meta staged
    // kTcStages - 1 pages ahead by bulk copies (lanes 0 and 1: codes, meta, one warp instruction)
    float mx[2] = {-INFINITY, -INFINITY};                         // heads 2 tig, 2 tig + 1
    auto stage_k = [&](int k, int slot) {
      if (lane >= 2) return;
      const bool hi = k < ph;
      const int C = hi ? HI::C : LO::C, krow = hi ? HI::k_row : LO::k_row;
      const uint32_t bar = bar_s + 8 * slot;
      if (lane == 0)
        asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(bar), "r"((uint32_t)(C * krow + 4 * C))
                     : "memory");
      const int off = lane == 0 ? (hi ? gh.off_k : gl.off_k) : (hi ? gh.off_kmeta : gl.off_kmeta);
      const uint32_t dst = stage_s + slot * STG + (lane == 0 ? 0 : C * krow);
      const uint32_t bytes = lane == 0 ? C * krow : 4 * C;
      asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];"
                   ::"r"(dst), "l"(page_ptr(k) + off), "r"(bytes), "r"(bar) : "memory");
    };
    auto stage_wait = [&](int slot) {
      mbar_wait(&bars[slot], (phase >> slot) & 1u);
      phase ^= 1u << slot;
    };
    {
#pragma unroll
      for (int i = 0; i < kTcStages - 1; i++)
        if (i < my_n) stage_k(warp + i * kTcWarps, i);
      for (int i = 0; i < my_n; i++) {
        const int k = warp + i * kTcWarps, slot = i % kTcStages;
        if (i + kTcStages - 1 < my_n) stage_k(warp + (i + kTcStages - 1) * kTcWarps, (i + kTcStages - 1) % kTcStages);
        stage_wait(slot);
        const uint8_t* kseg = mystage + slot * STG;
        if (k < ph) {
          const int t0 = k * HI::C;
          qk_page<D, G, GP, HI>(kseg, t0, min(HI::C, nh - t0), qb, s_qsum, scale, lg, mx, grp, tig);
        } else {
          const int t0 = nh + (k - ph) * LO::C;
          qk_page<D, G, GP, LO>(kseg, t0, min(LO::C, Ts - t0), qb, s_qsum, scale, lg, mx, grp, tig);
        }
        fence_proxy_async_smem();                                 // this stage's reads before its next bulk fill
        __syncwarp();
      }
    }
    // window tokens (FP16 keys): rows staged into shared memory (the page stages are free now), then one
    // (token, head) dot product per thread on CUDA cores
    __syncthreads();
    const uint16_t* wkg = wk_all + (size_t)u * W * D;
    const uint16_t* wvg = wv_all + (size_t)u * W * D;
    uint16_t* wks = reinterpret_cast<uint16_t*>(stage0);          // [nw][D] fp16, oldest first
    for (int c = tid; c < nw * (D / 8); c += kTcThreads) {
      const int i = c / (D / 8), e = c % (D / 8);
      cp_async16(wks + (size_t)i * D + 8 * e, wkg + (size_t)fmod_(p.div_W, N - nw + i) * D + 8 * e, true);
    }
    cp_async_commit();
    cp_async_wait<0>();
    __syncthreads();
    float wmx[G];
#pragma unroll
    for (int h = 0; h < G; h++) wmx[h] = -INFINITY;
    for (int x = tid; x < nw * G; x += kTcThreads) {
      const int i = x / G, h = x % G;
      const __half2* kr = reinterpret_cast<const __half2*>(wks + (size_t)i * D);
      float acc0 = 0.0f, acc1 = 0.0f;
#pragma unroll 8
      for (int e = 0; e < D / 2; e++) {
        const float2 kv = __half22float2(kr[e]);
        acc0 = fmaf(s_q[h][2 * e], kv.x, acc0);
        acc1 = fmaf(s_q[h][2 * e + 1], kv.y, acc1);
      }
      const float l = (acc0 + acc1) * scale;
      lg[(size_t)(Ts + i) * GP + h] = l;
#pragma unroll
      for (int hh = 0; hh < G; hh++)
        if (hh == h) wmx[hh] = fmaxf(wmx[hh], l);
    }
    // ---- phase 2: per-head max, p = exp(l - max), Z (thread per logit row of the CTA's global slot)
    fence_proxy_async_smem();                                     // the window rows' reads before phase 3's bulk fills
    {
#pragma unroll
      for (int c = 0; c < 2; c++) {
        float v = mx[c];                                          // reduce over the 8 lanes of this tig
#pragma unroll
        for (int o = 4; o < 32; o <<= 1) v = fmaxf(v, __shfl_xor_sync(kFull, v, o));
        mx[c] = v;
      }
#pragma unroll
      for (int h = 0; h < G; h++) {
        // head h's MMA maximum is held by the lanes with tig == h / 2
        float v = fmaxf(wmx[h], __shfl_sync(kFull, mx[h & 1], (h >> 1) & 3));
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) v = fmaxf(v, __shfl_xor_sync(kFull, v, o));
        if (lane == 0) s_red[warp][h] = v;
      }
      __syncthreads();                                            // also: every logit row is written
      if (tid < G) {
        float v = -INFINITY;
        for (int w = 0; w < kTcWarps; w++) v = fmaxf(v, s_red[w][tid]);
        s_m[tid] = v;
      }
      __syncthreads();
      float m[G], zs[G];
#pragma unroll
      for (int h = 0; h < G; h++) { m[h] = s_m[h]; zs[h] = 0.0f; }
      for (int i = tid; i < T; i += kTcThreads) {
        float4* row = reinterpret_cast<float4*>(lg + (size_t)i * GP);
#pragma unroll
        for (int c4 = 0; c4 < GP / 4; c4++) {
          float4 v = row[c4];
          float e[4] = {v.x, v.y, v.z, v.w};
#pragma unroll
          for (int j = 0; j < 4; j++) {
            const int h = 4 * c4 + j;
            if (h < G) { e[j] = __expf(e[j] - m[h]); zs[h] += e[j]; }
          }
          row[c4] = make_float4(e[0], e[1], e[2], e[3]);
        }
      }
      // the probability rows are read by phase 3's bulk copies (async proxy) after the barrier below
      asm volatile("fence.proxy.async.global;" ::: "memory");
#pragma unroll
      for (int h = 0; h < G; h++) {
        float v = zs[h];
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(kFull, v, o);
        if (lane == 0) s_red[warp][h] = v;
      }
      __syncthreads();
      if (tid < G) {
        float v = 0.0f;
        for (int w = 0; w < kTcWarps; w++) v += s_red[w][tid];
        s_iz[tid] = 1.0f / v;
      }
      __syncthreads();
    }
    // ---- phase 3: PV by MMA (A = value codes^T: m = features f0 = 16g + 2 grp, f0 + 1; k = tokens 4 tig .. +3;
    // B = 2^12 p * s_v split fp16 hi / lo, p = exp(l - max) unnormalised (1/Z applied to the partials): k = tokens,
    // n = head grp), significance + minima, page by page
    float acc[NG][4];
#pragma unroll
    for (int g = 0; g < NG; g++) acc[g][0] = acc[g][1] = acc[g][2] = acc[g][3] = 0.0f;
    float zsum = 0.0f;                                            // sum_t a_t z_t of head grp (this lane's tokens)
    unsigned long long mkey[2] = {~0ull, ~0ull};
    int mslot[2] = {-1, -1};
    float izr[G];
#pragma unroll
    for (int h = 0; h < G; h++) izr[h] = s_iz[h];
    // lanes 0-4 issue the five segment copies (V codes, V meta, scores, positions, the page's probability rows
    // from the scratch slot) as one warp instruction
    auto stage_v = [&](int k, int slot) {
      if (lane >= 5) return;
      const bool hi = k < ph;
      const ClassGeom& gg = hi ? gh : gl;
      const int C = hi ? HI::C : LO::C, vrow = hi ? HI::v_row : LO::v_row;
      const int t0 = hi ? k * HI::C : nh + (k - ph) * LO::C;
      const uint32_t bar = bar_s + 8 * slot;
      if (lane == 0)
        asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(bar),
                     "r"((uint32_t)(C * vrow + 12 * C + C * GP * 4)) : "memory");
      const uint8_t* src = lane == 4 ? reinterpret_cast<const uint8_t*>(lg + (size_t)t0 * GP)
                                     : page_ptr(k) + (lane == 0 ? gg.off_v : (lane == 1 ? gg.off_vmeta
                                                                  : (lane == 2 ? gg.off_score : gg.off_pos)));
      const uint32_t dst = stage_s + slot * STG + (lane == 0 ? 0 : C * vrow + 4 * C * (lane - 1));
      const uint32_t bytes = lane == 0 ? C * vrow : (lane == 4 ? C * GP * 4 : 4 * C);
      asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];"
                   ::"r"(dst), "l"(src), "r"(bytes), "r"(bar) : "memory");
    };
    {
#pragma unroll
      for (int i = 0; i < kTcStages - 1; i++)
        if (i < my_n) stage_v(warp + i * kTcWarps, i);
      for (int i = 0; i < my_n; i++) {
        const int k = warp + i * kTcWarps, slot = i % kTcStages;
        if (i + kTcStages - 1 < my_n) stage_v(warp + (i + kTcStages - 1) * kTcWarps, (i + kTcStages - 1) % kTcStages);
        stage_wait(slot);
        const uint8_t* vseg = mystage + slot * STG;
        const bool hi = k < ph;
        const int C = hi ? HI::C : LO::C;
        const int t0 = hi ? k * HI::C : nh + (k - ph) * LO::C;
        const int cnt = min(C, (hi ? nh : Ts) - t0);
        const int vrow = hi ? HI::v_row : LO::v_row;
        const float* prow = reinterpret_cast<const float*>(vseg + C * vrow + 12 * C);   // [C][GP] probabilities
        if (hi) pv_page<D, G, GP, HI>(vseg, 0, cnt, prow, acc, zsum, grp, tig);
        else pv_page<D, G, GP, LO>(vseg, 0, cnt, prow, acc, zsum, grp, tig);
        // significance (Q33) of the page's tokens: a lane per token
        const float* ssc = reinterpret_cast<const float*>(vseg + C * vrow + 4 * C);
        const int32_t* spos = reinterpret_cast<const int32_t*>(vseg + C * vrow + 8 * C);
        float* gsc = reinterpret_cast<float*>(page_ptr(k) + (hi ? gh.off_score : gl.off_score));
        for (int j = lane; j < cnt; j += 32) {
          const int i2 = t0 + j;                                  // token index (Q31 order)
          const float* row = prow + (size_t)j * GP;
          float a = 0.0f;
#pragma unroll
          for (int h = 0; h < G; h++) a = fmaxf(a, row[h] * izr[h]);
          if (probs) probs[(size_t)u * p.M + i2] = a;
          const int pos = spos[j];
          float sg = ssc[j];
          const int c = N - 2 - pos;
          if (c >= 0) {
            sg = (sg * (float)c + a) * __frcp_rn((float)(c + 1));
            gsc[j] = sg;
          }
          const int cls = hi ? 0 : 1;
          const int slotj = hi ? t0 + j : t0 - nh + j;
          const unsigned long long key = ((unsigned long long)__float_as_uint(sg) << 32) | (uint32_t)pos;
          if (key < mkey[cls]) { mkey[cls] = key; mslot[cls] = slotj; }
        }
        fence_proxy_async_smem();                                 // this stage's reads before its next bulk fill
        __syncwarp();
      }
    }
    __syncthreads();                                              // staging areas are free: reuse for the reduction
    float* part = reinterpret_cast<float*>(stage0);               // [kTcWarps][G][D] MMA partials
    float* zred = part + kTcWarps * G * D;                        // [kTcWarps][G]
    uint16_t* wvs = reinterpret_cast<uint16_t*>(zred + ((kTcWarps * G + 3) & ~3));   // [nw][D] window values
    for (int c = tid; c < nw * (D / 8); c += kTcThreads) {
      const int i = c / (D / 8), e = c % (D / 8);
      cp_async16(wvs + (size_t)i * D + 8 * e, wvg + (size_t)fmod_(p.div_W, N - nw + i) * D + 8 * e, true);
    }
    cp_async_commit();
    // window: significance on CUDA cores; its normalised probabilities staged for the output below
    for (int i = tid; i < nw; i += kTcThreads) {
      const int pos = N - nw + i;
      const float* row = lg + (size_t)(Ts + i) * GP;
      float a = 0.0f;
#pragma unroll
      for (int h = 0; h < G; h++) {
        const float ah = row[h] * izr[h];
        wprob[i * GP + h] = ah;
        a = fmaxf(a, ah);
      }
      if (probs) probs[(size_t)u * p.M + Ts + i] = a;
      const int c = N - 2 - pos;
      float* sp = p.win_sig + (size_t)u * W + fmod_(p.div_W, pos);
      if (c >= 0) *sp = (*sp * (float)c + a) * __frcp_rn((float)(c + 1));
    }
#pragma unroll
    for (int gg = 0; gg < NG; gg++) {
#pragma unroll
      for (int c = 0; c < 4; c++) {
        const int h = 2 * tig + (c & 1);
        const int f = (D / 8) * grp + 2 * gg + (c >> 1);        // pv_page's feature mapping
        if (h < G) part[((size_t)warp * G + h) * D + f] = acc[gg][c] * kPvUnscale * s_iz[h];
      }
    }
    {
      float v = zsum;                                             // lanes of head grp: tig = 0..3
      v += __shfl_xor_sync(kFull, v, 1);
      v += __shfl_xor_sync(kFull, v, 2);
      if (tig == 0 && grp < G) zred[warp * G + grp] = v * s_iz[grp];
    }
    cp_async_wait<0>();
    __syncthreads();
    if (out != nullptr) {
      for (int e = tid; e < G * D / 2; e += kTcThreads) {          // a feature pair per thread
        const int h = e / (D / 2), f = 2 * (e % (D / 2));
        float o0 = 0.0f, o1 = 0.0f, z = 0.0f;
        for (int w = 0; w < kTcWarps; w++) {
          const float2 pp = *reinterpret_cast<const float2*>(part + ((size_t)w * G + h) * D + f);
          o0 += pp.x; o1 += pp.y; z += zred[w * G + h];
        }
        float w0 = 0.0f, w1 = 0.0f;                                // the window's values (FP16) on CUDA cores
        for (int i = 0; i < nw; i++) {
          const float a = wprob[i * GP + h];
          const float2 vv = __half22float2(*reinterpret_cast<const __half2*>(wvs + (size_t)i * D + f));
          w0 = fmaf(a, vv.x, w0);
          w1 = fmaf(a, vv.y, w1);
        }
        *reinterpret_cast<float2*>(out + ((size_t)u * G + h) * D + f) = make_float2(o0 + z + w0, o1 + z + w1);
      }
    }
    // section minima (stored sections only; keys are unique: positions differ)
#pragma unroll
    for (int c = 0; c < 2; c++)
      if (mkey[c] != ~0ull) atomicMin(&s_min[c], mkey[c]);
    __syncthreads();
#pragma unroll
    for (int c = 0; c < 2; c++)
      if (mkey[c] != ~0ull && mkey[c] == s_min[c]) s_slot[c] = mslot[c];
    __syncthreads();
    if (tid == 0) {
      int32_t* m = p.secmin + 8 * (size_t)u;
#pragma unroll
      for (int c = 0; c < 2; c++) {
        m[3 * c] = (int32_t)(uint32_t)(s_min[c] >> 32);
        m[3 * c + 1] = (int32_t)(uint32_t)(s_min[c] & 0xFFFFFFFFull);
        m[3 * c + 2] = s_slot[c];
      }
      m[6] = 1;
    }
  }
}

// the kernel is specialised for the paper's classes: K8V4 in 16-token pages, K4V2 in 32-token pages;
// other geometries take the exact path
bool attend_tc_supported(const PoolDev& p) {
  const ClassGeom &h = p.g[1], &l = p.g[2];
  return h.C == 16 && h.kbits == 8 && h.vbits == 4 && l.C == 32 && l.kbits == 4 && l.vbits == 2 && p.G >= 1 &&
         p.G <= 8 && (p.d == 64 || p.d == 128) && p.tc_scratch != nullptr;
}

size_t attend_tc_smem_bytes(const PoolDev& p) {
  const int GP = p.G <= 4 ? 4 : 8;
  return (size_t)tc_area_bytes(p.d, p.G, p.W, GP) + (size_t)((p.L + 4) & ~3) * 4 + (size_t)p.W * GP * 4;
}

template <int D, int G>
static cudaError_t launch_tc(const PoolDev& p, const uint16_t* q, float* out, float* probs, cudaStream_t s) {
  const size_t smem = attend_tc_smem_bytes(p);
  cudaError_t e = cudaFuncSetAttribute(attend_tc_kernel<D, G>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  if (e != cudaSuccess) return e;
  int dev = 0, sms = 0, per_sm = 0;
  if ((e = cudaGetDevice(&dev)) != cudaSuccess) return e;
  if ((e = cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev)) != cudaSuccess) return e;
  if ((e = cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, attend_tc_kernel<D, G>, kTcThreads, smem)) != cudaSuccess)
    return e;
  int grid = sms * (per_sm > 0 ? per_sm : 1);
  if (grid > p.tc_slots) grid = p.tc_slots;                       // one scratch slot per CTA
  if (grid > p.U) grid = p.U;
  attend_tc_kernel<D, G><<<grid, kTcThreads, smem, s>>>(p, q, out, probs);
  return cudaGetLastError();
}

template <int D>
static cudaError_t launch_tc_d(const PoolDev& p, const uint16_t* q, float* out, float* probs, cudaStream_t s) {
  switch (p.G) {
    case 1: return launch_tc<D, 1>(p, q, out, probs, s);
    case 2: return launch_tc<D, 2>(p, q, out, probs, s);
    case 4: return launch_tc<D, 4>(p, q, out, probs, s);
    case 5: return launch_tc<D, 5>(p, q, out, probs, s);
    case 7: return launch_tc<D, 7>(p, q, out, probs, s);
    default: return launch_tc<D, 8>(p, q, out, probs, s);
  }
}

cudaError_t launch_attend_tc(const PoolDev& p, const uint16_t* q, float* out, float* probs, cudaStream_t s) {
  return p.d == 128 ? launch_tc_d<128>(p, q, out, probs, s) : launch_tc_d<64>(p, q, out, probs, s);
}

}  // namespace dkv
