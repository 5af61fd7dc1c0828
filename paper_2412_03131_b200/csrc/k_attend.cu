// k_attend.cu — NEXT-2: decode attention over the compressed cache with the significance update and the
// victim search of the next step fused into its epilogue (readings Q31-Q34).
//
// One CTA per unit (request, layer, KV head), the paper's "one thread block per (head, sequence)".
// The unit's tokens are taken in the normative order of Q31 — high section slots, low section slots, the
// FP16 window oldest first — and every floating-point result is fixed by Q31-Q34, so the kernel matches the
// oracle bit for bit:
//   1. logits: one thread per token dequantizes its key (X^ = s*Q + z) and accumulates the G dot
//      products serially over the d elements; logit = dot * (1/sqrt(d));
//   2. softmax: max per head (order-free), p = dkv_exp(logit - max), Z = pages summed in order of their
//      serial in-page sums (the window as pages of C_h tokens), a = p / Z, score = max over the G heads;
//   3. significance: sig' = (sig * c + score) / (c + 1), c = N - 2 - position (Q33), written in place
//      (page score segment / window array, Q34); each section's (sig', position) minimum goes to the unit's
//      secmin record, which lets the next dkv_classify(DECODE) pick its victim without a scan;
//   4. output (optional): pages in order of their in-page fma chains; a warp per page, a lane per element
//      set with all G heads, partials added in page order by (head, element) threads.
// Logits / probabilities live in shared memory: q_per_kv floats per token, sized by the longest ACTIVE request
// (the host mirror knows every request's length; a unit holds at most that many tokens).
#include <algorithm>

#include "dkv_internal.cuh"

namespace dkv {

#ifndef DKV_ATT_THREADS
#define DKV_ATT_THREADS 512
#endif
constexpr int kAttThreads = DKV_ATT_THREADS;                      // 2 CTAs per SM (launch bounds)
// output pages per round: one per warp, at most 16 (G <= 4) / 8 page partials of [G][D] floats
__host__ __device__ constexpr int att_ppr(int G) {
  return (G <= 4 ? 16 : 8) < kAttThreads / 32 ? (G <= 4 ? 16 : 8) : kAttThreads / 32;
}

// Q32: exp for x <= 0 — 2^t, t = x*log2(e), n = rint(t), f = t - n, degree-6 Taylor polynomial of 2^f in
// Horner form, times 2^n; 0 below t = -125.  Every step one IEEE binary32 operation (as the oracle's orc_exp).
__device__ __forceinline__ float dkv_exp(float x) {
  const float t = __fmul_rn(x, 1.44269504088896341f);
  if (t < -125.0f) return 0.0f;
  const float n = rintf(t);
  const float f = __fsub_rn(t, n);
  float r = 1.54035304e-4f;
  r = __fadd_rn(__fmul_rn(r, f), 1.33335581e-3f);
  r = __fadd_rn(__fmul_rn(r, f), 9.61812911e-3f);
  r = __fadd_rn(__fmul_rn(r, f), 5.55041087e-2f);
  r = __fadd_rn(__fmul_rn(r, f), 2.40226507e-1f);
  r = __fadd_rn(__fmul_rn(r, f), 6.93147181e-1f);
  r = __fadd_rn(__fmul_rn(r, f), 1.0f);
  return __fmul_rn(r, __int_as_float(((int)n + 127) << 23));
}

// X^ = s*Q + z.  s is binary16 and Q < 2^8, so s*Q is exact in binary32 and fma(s, Q, z) rounds once,
// exactly like the oracle's fadd(fmul(s, Q), z).
__device__ __forceinline__ float dq(uint32_t code, float sf, float zf) {
  return __fmaf_rn(sf, __uint_as_float(0x4B000000u | code) - 8388608.0f, zf);
}

// one output warp's shared-memory area: a page's value codes + value (s, z) pairs (the contiguous span from
// off_v), later overwritten by the warp's [G][D] fp32 page partial
// (long-context form: followed by the page's probabilities, staged from the HBM logit slot)
__host__ __device__ inline int attend_span(const ClassGeom& a, const ClassGeom& b) {
  const int sa = a.off_vmeta - a.off_v + 4 * a.C, sb = b.off_vmeta - b.off_v + 4 * b.C;
  return ((sa > sb ? sa : sb) + 15) & ~15;
}
__host__ __device__ inline int attend_warp_area(const ClassGeom& a, const ClassGeom& b, int G, int D) {
  const int GP = (G + 3) / 4 * 4, C = a.C > b.C ? a.C : b.C;
  const int staged = attend_span(a, b) + 4 * GP * C;
  return staged > 4 * G * D ? staged : 4 * G * D;
}

template <int G>
constexpr int padded_heads() { return (G + 3) / 4 * 4; }          // lg row stride: 16-B aligned per token

struct AttShared {
  float* qf;        // [G][D]
  float* lg;        // [M][GP] logits -> exp -> probabilities, token-major (one 16-B load per 4 heads)
  float* part;      // [G][npage]
  int32_t* pid;     // [ph + pl] page IDs, section order
};

// Accumulate the G dot products of the query heads with one stored key of BITS-bit codes: the whole code
// row is loaded first, then one fma chain per head over e = 0..d-1 (Q31).
template <int D, int G, int BITS>
__device__ __forceinline__ void dot_stored(const float* __restrict__ qf, const uint8_t* row, uint32_t kmeta,
                                           float (&acc)[G]) {
  const float sf = __half2float(__ushort_as_half((unsigned short)(kmeta & 0xFFFFu)));
  const float zf = __half2float(__ushort_as_half((unsigned short)(kmeta >> 16)));
  constexpr int PER = 32 / BITS;                                  // codes per 32-bit word
  constexpr int NW = D / PER;                                     // words per row
  constexpr uint32_t Q = (1u << BITS) - 1u;
  uint32_t w[NW];
#pragma unroll
  for (int k = 0; k < NW / 4; k++) {
    const uint4 v = *reinterpret_cast<const uint4*>(row + 16 * k);
    w[4 * k] = v.x; w[4 * k + 1] = v.y; w[4 * k + 2] = v.z; w[4 * k + 3] = v.w;
  }
  constexpr int PB = 8 / BITS;                                    // codes per byte
  constexpr uint32_t MB = Q * (0x01010101u);                      // the code mask in every byte
#pragma unroll
  for (int k = 0; k < NW; k++) {
    // part[i] byte b = code (b * PB + i) of the word (Q17: lowest element in the least-significant bits); one
    // byte permute then yields the float 2^23 + code (exact), and the subtraction of 2^23 is exact too
    uint32_t part[PB];
#pragma unroll
    for (int i = 0; i < PB; i++) part[i] = (w[k] >> (i * BITS)) & MB;
#pragma unroll
    for (int j = 0; j < PER; j += 4) {
      float x[4];
#pragma unroll
      for (int jj = 0; jj < 4; jj++) {
        const int e = j + jj;
        const float c = __uint_as_float(__byte_perm(part[e % PB], 0x4B000000u, 0x7540u | (uint32_t)(e / PB)));
        x[jj] = __fmaf_rn(sf, __fsub_rn(c, 8388608.0f), zf);
      }
      const int e = k * PER + j;
#pragma unroll
      for (int g = 0; g < G; g++) {
        const float4 qv = *reinterpret_cast<const float4*>(qf + g * D + e);
        acc[g] = __fmaf_rn(qv.x, x[0], acc[g]);
        acc[g] = __fmaf_rn(qv.y, x[1], acc[g]);
        acc[g] = __fmaf_rn(qv.z, x[2], acc[g]);
        acc[g] = __fmaf_rn(qv.w, x[3], acc[g]);
      }
    }
  }
}

// The output chains of one staged page (Q32): for each of its cnt tokens in slot order, this lane's EPL
// consecutive value elements (EPL * VB bits of one aligned shared word) dequantized with the token's (s, z)
// and accumulated into the G heads' chains.  Codes become floats as in dot_stored (byte permute, exact).
template <int D, int G, int VB>
__device__ __forceinline__ void value_tokens(const uint8_t* seg, int mbase, int v_row, int lane, const float* lg,
                                             int cnt, float (&acc)[D / 32][G]) {
  constexpr int EPL = D / 32, GP = padded_heads<G>();
  constexpr int PB = 8 / VB;
  constexpr uint32_t MB = ((1u << VB) - 1u) * 0x01010101u;
  const int bit0 = lane * EPL * VB;
  const uint8_t* wp = seg + ((bit0 >> 5) << 2);
  const int sh = bit0 & 31;
  for (int j = 0; j < cnt; j++) {
    const uint32_t vm = *reinterpret_cast<const uint32_t*>(seg + mbase + 4 * j);
    const float sf = __half2float(__ushort_as_half((unsigned short)(vm & 0xFFFFu)));
    const float zf = __half2float(__ushort_as_half((unsigned short)(vm >> 16)));
    float av[G];
#pragma unroll
    for (int g4 = 0; g4 < GP; g4 += 4) {
      const float4 a4 = *reinterpret_cast<const float4*>(lg + (size_t)j * GP + g4);
      if (g4 < G) av[g4] = a4.x;
      if (g4 + 1 < G) av[g4 + 1] = a4.y;
      if (g4 + 2 < G) av[g4 + 2] = a4.z;
      if (g4 + 3 < G) av[g4 + 3] = a4.w;
    }
    // the lane's EPL * VB code bits: a byte / half-word / word load when they are byte-aligned (no shift)
    constexpr int LB = EPL * VB;
    uint32_t word;
    if constexpr (LB == 8) word = seg[j * v_row + (bit0 >> 3)];
    else if constexpr (LB == 16) word = *reinterpret_cast<const uint16_t*>(seg + j * v_row + (bit0 >> 3));
    else if constexpr (LB == 32) word = *reinterpret_cast<const uint32_t*>(seg + j * v_row + (bit0 >> 3));
    else word = *reinterpret_cast<const uint32_t*>(wp + j * v_row) >> sh;
    uint32_t part[PB];
    if constexpr (VB != 2) {
#pragma unroll
      for (int i = 0; i < PB; i++) part[i] = (word >> (i * VB)) & MB;
    }
#pragma unroll
    for (int x = 0; x < EPL; x++) {
      // 2-bit codes: shift + one LOP3 ((w >> s) & 3 | 2^23 bits) per code beats four byte-wise masks
      const float c = VB == 2 ? __uint_as_float(((word >> (2 * x)) & 3u) | 0x4B000000u)
                              : __uint_as_float(__byte_perm(part[x % PB], 0x4B000000u, 0x7540u | (uint32_t)(x / PB)));
      const float v = __fmaf_rn(sf, __fsub_rn(c, 8388608.0f), zf);
#pragma unroll
      for (int g = 0; g < G; g++) acc[x][g] = __fmaf_rn(av[g], v, acc[x][g]);
    }
  }
}

// One unit.  LONG: the logits and (s, z) pairs live in a per-CTA slot of HBM scratch instead of shared memory
// (contexts whose q_per_kv * length floats exceed shared memory; the kernel is then persistent).
template <int D, int G, bool LONG>
__device__ __forceinline__ void attend_unit(const PoolDev& p, const uint16_t* __restrict__ q, float* __restrict__ out,
                                            float* __restrict__ probs, int TS, int u, float* g_lg) {
  extern __shared__ __align__(16) float att_smem[];
  __shared__ float s_red[kAttThreads / 32][G];
  __shared__ float s_m[G], s_Z[G];
  __shared__ unsigned long long s_min[2];
  __shared__ int s_slot[2];
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  if (ld_volatile(&p.ctrl->status) != 0) return;                  // sticky error: no-op
  const int r = fdiv(p.div_LyH, u);
  if (p.req_state[r] != DKV_REQ_ACTIVE) return;
  const int M = TS, L = p.L, W = p.W;                            // M: per-head logit stride in shared memory
  const int N = p.seq_len[r];                                     // includes the newest token
  const int nh = p.n_h[u], nl = p.n_l[u];
  const int nw = min(W, N);
  const int T = nh + nl + nw;
  const int Ch = p.g[1].C, Cl = p.g[2].C;
  const int ph = ceil_div(nh, Ch), pl = ceil_div(nl, Cl);
  const int npage = ph + pl + ceil_div(nw, Ch);                  // Q32: the window as pages of C_h tokens
  const int PS = L + ceil_div(W, Ch);                            // page-partial stride (pages a unit can have)
  AttShared S;
  constexpr int GP = padded_heads<G>();
  // every region is carved by float offsets from the shared base (keeps the compiler on shared-space loads)
  const int off_lg = G * D;                                       // multiple of 4 floats
  const int off_part = off_lg + (LONG ? 0 : GP * M);
  const int off_pid = off_part + G * PS;
  S.qf = att_smem;
  S.lg = LONG ? g_lg : att_smem + off_lg;
  S.part = att_smem + off_part;
  S.pid = reinterpret_cast<int32_t*>(att_smem + off_pid);
  const int32_t* row = p.table + (size_t)u * L;
  for (int k = tid; k < ph + pl; k += kAttThreads) S.pid[k] = k < ph ? row[k] : row[L - 1 - (k - ph)];
  for (int k = tid; k < G * D; k += kAttThreads)
    S.qf[k] = __half2float(__ushort_as_half(q[(size_t)u * G * D + k]));
  if (tid < 2) { s_min[tid] = ~0ull; s_slot[tid] = -1; }
  __syncthreads();
  const float scale = __fdiv_rn(1.0f, __fsqrt_rn((float)D));
  const ClassGeom gh = p.g[1], gl = p.g[2];

  // a token's GP-float logit / probability row (G heads + zero padding) moves as 16-B vectors
  auto store_row = [&](int i, const float (&row)[GP]) {
#pragma unroll
    for (int g4 = 0; g4 < GP; g4 += 4)
      *reinterpret_cast<float4*>(S.lg + (size_t)i * GP + g4) = make_float4(row[g4], row[g4 + 1], row[g4 + 2], row[g4 + 3]);
  };
  auto load_row = [&](int i, float (&row)[GP]) {
#pragma unroll
    for (int g4 = 0; g4 < GP; g4 += 4) {
      const float4 v = *reinterpret_cast<const float4*>(S.lg + (size_t)i * GP + g4);
      row[g4] = v.x; row[g4 + 1] = v.y; row[g4 + 2] = v.z; row[g4 + 3] = v.w;
    }
  };
  // ---- 1. logits (Q31)
  float mx[G];
#pragma unroll
  for (int g = 0; g < G; g++) mx[g] = -INFINITY;
  for (int i = tid; i < T; i += kAttThreads) {
    float acc[G];
#pragma unroll
    for (int g = 0; g < G; g++) acc[g] = 0.0f;
    if (i < nh + nl) {
      const bool hi = i < nh;
      const ClassGeom& gg = hi ? gh : gl;
      const int s = hi ? i : i - nh;
      const int pg = hi ? fdiv(p.div_Ch, s) : ph + fdiv(p.div_Cl, s);
      const int idx = hi ? s - (pg * Ch) : s - (pg - ph) * Cl;
      const uint8_t* page = p.pages + (size_t)S.pid[pg] * (size_t)p.page_bytes;
      const uint32_t km = *reinterpret_cast<const uint32_t*>(page + gg.off_kmeta + 4 * idx);
      const uint8_t* krow = page + gg.off_k + idx * gg.k_row;
      if (gg.kbits == 8) dot_stored<D, G, 8>(S.qf, krow, km, acc);
      else if (gg.kbits == 4) dot_stored<D, G, 4>(S.qf, krow, km, acc);
      else dot_stored<D, G, 2>(S.qf, krow, km, acc);
    } else {
      const int pos = N - nw + (i - nh - nl);
      const uint16_t* wk = reinterpret_cast<const uint16_t*>(p.win_k) + ((size_t)u * W + fmod_(p.div_W, pos)) * D;
#pragma unroll 2
      for (int e0 = 0; e0 < D; e0 += 8) {
        const uint4 v = *reinterpret_cast<const uint4*>(wk + e0);
        const uint32_t hw[4] = {v.x, v.y, v.z, v.w};
#pragma unroll
        for (int k = 0; k < 8; k++) {
          const float x = __half2float(__ushort_as_half((unsigned short)(hw[k >> 1] >> (16 * (k & 1)))));
#pragma unroll
          for (int g = 0; g < G; g++) acc[g] = __fmaf_rn(S.qf[g * D + e0 + k], x, acc[g]);
        }
      }
    }
    float row[GP];
#pragma unroll
    for (int g = 0; g < GP; g++) {
      row[g] = 0.0f;
      if (g < G) {
        row[g] = __fmul_rn(acc[g], scale);
        mx[g] = fmaxf(mx[g], row[g]);
      }
    }
    store_row(i, row);
  }
  // the output phase reads the unit's FP16 window value rows last: pull them into L2 now
  if (out != nullptr) {
    const char* wv = reinterpret_cast<const char*>(p.win_v + (size_t)u * W * D);
    for (int o = tid * 128; o < W * D * 2; o += kAttThreads * 128)
      asm volatile("prefetch.global.L2 [%0];" ::"l"(wv + o));
  }
  // ---- 2. softmax (Q32)
#pragma unroll
  for (int g = 0; g < G; g++) {
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) mx[g] = fmaxf(mx[g], __shfl_xor_sync(kFull, mx[g], o));
    if (lane == 0) s_red[warp][g] = mx[g];
  }
  __syncthreads();
  if (tid < G) {
    float m = -INFINITY;
    for (int w = 0; w < kAttThreads / 32; w++) m = fmaxf(m, s_red[w][tid]);
    s_m[tid] = m;
  }
  __syncthreads();
  for (int i = tid; i < T; i += kAttThreads) {
    float row[GP];
    load_row(i, row);
#pragma unroll
    for (int g = 0; g < G; g++) row[g] = dkv_exp(__fsub_rn(row[g], s_m[g]));
    store_row(i, row);
  }
  __syncthreads();
  auto page_range = [&](int k, int& t0, int& t1) {
    if (k < ph) { t0 = k * Ch; t1 = min(t0 + Ch, nh); }
    else if (k < ph + pl) { t0 = nh + (k - ph) * Cl; t1 = min(t0 + Cl, nh + nl); }
    else { t0 = nh + nl + (k - ph - pl) * Ch; t1 = min(t0 + Ch, T); }
  };
  if (LONG) {                                                     // serial in-page sums, a thread per page:
    for (int k = tid; k < npage; k += kAttThreads) {              // whole rows from the HBM slot, G chains
      int t0, t1;
      page_range(k, t0, t1);
      float sum[GP];
#pragma unroll
      for (int g = 0; g < GP; g++) sum[g] = 0.0f;
#pragma unroll 4
      for (int i = t0; i < t1; i++) {
        float row[GP];
        load_row(i, row);
#pragma unroll
        for (int g = 0; g < G; g++) sum[g] = __fadd_rn(sum[g], row[g]);
      }
#pragma unroll
      for (int g = 0; g < G; g++) S.part[g * PS + k] = sum[g];
    }
  } else {
    for (int it = tid; it < G * npage; it += kAttThreads) {        // serial in-page sums
      const int g = it / npage, k = it % npage;
      int t0, t1;
      page_range(k, t0, t1);
      float sum = 0.0f;
      for (int i = t0; i < t1; i++) sum = __fadd_rn(sum, S.lg[(size_t)i * GP + g]);
      S.part[g * PS + k] = sum;
    }
  }
  __syncthreads();
  if (tid < G) {                                                  // pages in order
    float Z = 0.0f;
    for (int k = 0; k < npage; k++) Z = __fadd_rn(Z, S.part[tid * PS + k]);
    s_Z[tid] = Z;
  }
  __syncthreads();

  // ---- 3. scores, significance (Q33, Q34), section minima.  Two tokens per trip so their score / position
  // loads overlap; each thread keeps its running (sig, position) minimum and slot per section, so the section
  // minimum's slot is found without a second pass over the positions.
  unsigned long long mkey[2] = {~0ull, ~0ull};
  int mslot[2] = {-1, -1};
  auto locate = [&](int i, float*& sp, int& pos, int& cls, int& slot) {
    if (i < nh + nl) {
      const bool hi = i < nh;
      const ClassGeom& gg = hi ? gh : gl;
      slot = hi ? i : i - nh;
      const int pg = hi ? fdiv(p.div_Ch, slot) : ph + fdiv(p.div_Cl, slot);
      const int idx = hi ? slot - pg * Ch : slot - (pg - ph) * Cl;
      uint8_t* page = p.pages + (size_t)S.pid[pg] * (size_t)p.page_bytes;
      sp = reinterpret_cast<float*>(page + gg.off_score + 4 * idx);
      pos = *reinterpret_cast<const int32_t*>(page + gg.off_pos + 4 * idx);
      cls = hi ? 1 : 2;
    } else {
      pos = N - nw + (i - nh - nl);
      sp = p.win_sig + (size_t)u * W + fmod_(p.div_W, pos);
      cls = 0; slot = 0;
    }
  };
  auto update = [&](int i, float* sp, int pos, int cls, int slot, float sg) {
    float a = 0.0f, row[GP];
    load_row(i, row);
#pragma unroll
    for (int g = 0; g < G; g++) {
      row[g] = __fdiv_rn(row[g], s_Z[g]);
      a = fmaxf(a, row[g]);                                       // GQA: max over the group
    }
    store_row(i, row);
    if (probs) probs[(size_t)u * p.M + i] = a;
    const int c = N - 2 - pos;                                    // later queries so far
    if (c >= 0) {
      sg = __fdiv_rn(__fadd_rn(__fmul_rn(sg, (float)c), a), (float)(c + 1));
      *sp = sg;
    }
    if (cls) {
      const unsigned long long key = ((unsigned long long)__float_as_uint(sg) << 32) | (uint32_t)pos;
      if (key < mkey[cls - 1]) { mkey[cls - 1] = key; mslot[cls - 1] = slot; }
    }
  };
  for (int i = tid; i < T; i += 2 * kAttThreads) {
    const int i2 = i + kAttThreads;
    float *sp1, *sp2 = nullptr;
    int pos1, cls1, slot1, pos2 = 0, cls2 = 0, slot2 = 0;
    locate(i, sp1, pos1, cls1, slot1);
    if (i2 < T) locate(i2, sp2, pos2, cls2, slot2);
    const float sg1 = *sp1;
    const float sg2 = i2 < T ? *sp2 : 0.0f;
    update(i, sp1, pos1, cls1, slot1, sg1);
    if (i2 < T) update(i2, sp2, pos2, cls2, slot2, sg2);
  }
#pragma unroll
  for (int c = 0; c < 2; c++)
    if (mkey[c] != ~0ull) atomicMin(&s_min[c], mkey[c]);
  __syncthreads();
#pragma unroll
  for (int c = 0; c < 2; c++)
    if (mkey[c] != ~0ull && mkey[c] == s_min[c]) s_slot[c] = mslot[c];   // positions are unique: one winner
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
  // ---- 4. output (Q32): pages in order, each page's partial a fma chain over its tokens.  Rounds of PPR
  // pages: warp w < PPR computes page (round * PPR + w) for every (element, head) — lane owns EPL elements and
  // all heads, so its 16-32 chains are independent — from the page's value codes and value (s, z) pairs (one
  // contiguous span of the page) staged in the warp's shared-memory area; the warp then overwrites that area
  // with its [G][D] page partial, and thread (head, element) adds the round's partials to its running sum in
  // page order.  A lane owns EPL consecutive elements, so one aligned 32-bit shared load yields all of its
  // codes of a token.
  if (out != nullptr) {
    constexpr int PPR = att_ppr(G);                               // pages per round
    constexpr int EPL = D / 32;                                   // elements per lane
    const int wbytes = attend_warp_area(gh, gl, G, D);
    uint8_t* seg0 = reinterpret_cast<uint8_t*>(att_smem + ((off_pid + L + 1 + 3) & ~3));   // PPR warp areas
    uint8_t* seg = seg0 + (size_t)warp * wbytes;
    float* part4 = reinterpret_cast<float*>(seg);                 // [G][D], after the page is consumed
    float run[(G * D + kAttThreads - 1) / kAttThreads];
#pragma unroll
    for (int j = 0; j < (G * D + kAttThreads - 1) / kAttThreads; j++) run[j] = 0.0f;
    for (int r0 = 0; r0 < npage; r0 += PPR) {
      const int k = r0 + warp;
      {                                                           // pull the next round's value span into L2
        const int kn = k + PPR;
        if (warp < PPR && kn < ph + pl) {
          const ClassGeom& gn = kn < ph ? gh : gl;
          const int span = gn.off_vmeta - gn.off_v + 4 * gn.C;
          const char* src = reinterpret_cast<const char*>(p.pages + (size_t)S.pid[kn] * (size_t)p.page_bytes + gn.off_v);
          if (lane * 128 < span) asm volatile("prefetch.global.L2 [%0];" ::"l"(src + lane * 128));
        }
      }
      if (warp < PPR && k < npage) {
        float acc[EPL][G];
#pragma unroll
        for (int x = 0; x < EPL; x++)
#pragma unroll
          for (int g = 0; g < G; g++) acc[x][g] = 0.0f;
        if (k < ph + pl) {                                        // a stored page
          const bool hi = k < ph;
          const ClassGeom& gg = hi ? gh : gl;
          const int t0 = hi ? k * Ch : nh + (k - ph) * Cl;
          const int cnt = min(hi ? Ch : Cl, (hi ? nh : nh + nl) - t0);
          const uint8_t* src = p.pages + (size_t)S.pid[k] * (size_t)p.page_bytes + gg.off_v;
          const int mbase = gg.off_vmeta - gg.off_v;              // value (s, z) pairs follow the codes
          const int nbytes = mbase + 4 * cnt;
          for (int o = 16 * lane; o < nbytes; o += 512)
            *reinterpret_cast<uint4*>(seg + o) = *reinterpret_cast<const uint4*>(src + o);
          const float* lgp = S.lg + (size_t)t0 * GP;
          if (LONG) {                                             // the page's probabilities, HBM slot -> shared
            float* sa = reinterpret_cast<float*>(seg + attend_span(gh, gl));
            for (int o = 4 * lane; o < cnt * GP; o += 128)
              *reinterpret_cast<float4*>(sa + o) = *reinterpret_cast<const float4*>(lgp + o);
            lgp = sa;
          }
          __syncwarp();
          if (gg.vbits == 4) value_tokens<D, G, 4>(seg, mbase, gg.v_row, lane, lgp, cnt, acc);
          else if (gg.vbits == 2) value_tokens<D, G, 2>(seg, mbase, gg.v_row, lane, lgp, cnt, acc);
          else value_tokens<D, G, 8>(seg, mbase, gg.v_row, lane, lgp, cnt, acc);
          __syncwarp();                                           // seg now takes the page partial
        } else {                                                  // a window page (C_h tokens, oldest first)
          constexpr int WB = 8;                                   // window rows in flight per lane
          const int w0 = nh + nl + (k - ph - pl) * Ch, w1 = min(w0 + Ch, T);   // this window page
          for (int i0 = w0; i0 < w1; i0 += WB) {
            uint32_t raw[WB][EPL / 2];
#pragma unroll
            for (int b = 0; b < WB; b++) {
              const int pos = N - nw + (i0 + b - nh - nl);
              if (i0 + b < w1) {
                const uint32_t* vr = reinterpret_cast<const uint32_t*>(
                    p.win_v + ((size_t)u * W + fmod_(p.div_W, pos)) * D) + lane * (EPL / 2);
                if constexpr (EPL == 4) {
                  const uint2 t2 = *reinterpret_cast<const uint2*>(vr);
                  raw[b][0] = t2.x; raw[b][EPL / 2 - 1] = t2.y;
                } else {
                  raw[b][0] = vr[0];
                }
              }
            }
#pragma unroll
            for (int b = 0; b < WB; b++) {
              const int i = i0 + b;
              if (i < w1) {
                float av[G];
#pragma unroll
                for (int g = 0; g < G; g++) av[g] = S.lg[(size_t)i * GP + g];
#pragma unroll
                for (int x = 0; x < EPL; x++) {
                  const float v = __half2float(__ushort_as_half((unsigned short)(raw[b][x >> 1] >> (16 * (x & 1)))));
#pragma unroll
                  for (int g = 0; g < G; g++) acc[x][g] = __fmaf_rn(av[g], v, acc[x][g]);
                }
              }
            }
          }
        }
#pragma unroll
        for (int x = 0; x < EPL; x++)
#pragma unroll
          for (int g = 0; g < G; g++) part4[g * D + EPL * lane + x] = acc[x][g];
      }
      __syncthreads();
#pragma unroll
      for (int j = 0; j < (G * D + kAttThreads - 1) / kAttThreads; j++) {
        const int t = tid + j * kAttThreads;                      // (head, element) = (t / D, t % D)
        if (t < G * D) {
          const float* pp = reinterpret_cast<const float*>(seg0) + t;
          const int ws = wbytes / 4;
          if (r0 + PPR <= npage) {                                // full round: all loads first, then the chain
            float v[PPR];
#pragma unroll
            for (int w = 0; w < PPR; w++) v[w] = pp[w * ws];
#pragma unroll
            for (int w = 0; w < PPR; w++) run[j] = __fadd_rn(run[j], v[w]);
          } else {
            for (int w = 0; r0 + w < npage; w++) run[j] = __fadd_rn(run[j], pp[w * ws]);
          }
        }
      }
      __syncthreads();                                            // partials are rewritten next round
    }
#pragma unroll
    for (int j = 0; j < (G * D + kAttThreads - 1) / kAttThreads; j++) {
      const int t = tid + j * kAttThreads;
      if (t < G * D) out[(size_t)u * G * D + t] = run[j];
    }
  }
}

template <int D, int G>
__global__ void __launch_bounds__(kAttThreads, 2)
attend_kernel(PoolDev p, const uint16_t* __restrict__ q, float* __restrict__ out, float* __restrict__ probs, int TS) {
  attend_unit<D, G, false>(p, q, out, probs, TS, blockIdx.x, nullptr);
}

// persistent form for long contexts: CTA b owns scratch slot b and walks units b, b + grid, ...
template <int D, int G>
__global__ void __launch_bounds__(kAttThreads, 2)
attend_long_kernel(PoolDev p, const uint16_t* __restrict__ q, float* __restrict__ out, float* __restrict__ probs,
                   int TS) {
  constexpr int GP = padded_heads<G>();
  float* lg = p.att_scratch + (size_t)blockIdx.x * (GP + 2) * (size_t)TS;
  for (int u = blockIdx.x; u < p.U; u += gridDim.x) {
    attend_unit<D, G, true>(p, q, out, probs, TS, u, lg);
    __syncthreads();                                              // shared state is reused by the next unit
  }
}

// bytes of shared memory per unit besides the logits: q, Z page partials, page IDs (+ alignment), and PPR warp
// areas, each holding one page's value codes + (s, z) pairs, then that page's [G][D] output partial
static size_t attend_fixed_bytes(const PoolDev& p) {
  const size_t G = p.G > 0 ? p.G : 1, PPR = att_ppr((int)G);
  const size_t PS = (size_t)p.L + (size_t)((p.W + p.g[1].C - 1) / p.g[1].C);   // page partials per head
  return 4 * (G * p.d + G * PS + (size_t)p.L + 1 + 3) +
         PPR * (size_t)attend_warp_area(p.g[1], p.g[2], (int)G, p.d);
}

size_t attend_long_smem_bytes(const PoolDev& p) { return attend_fixed_bytes(p); }

size_t attend_smem_bytes(const PoolDev& p, int TS) {
  const size_t G = p.G > 0 ? p.G : 1, GP = (G + 3) / 4 * 4;
  return attend_fixed_bytes(p) + 4 * GP * (size_t)TS;             // + the logits, token-major
}

template <int D, int G>
static cudaError_t launch_att(const PoolDev& p, const uint16_t* q, float* out, float* probs, int TS, cudaStream_t s) {
  if (TS < 0) {                                                   // long-context form (scratch slots in HBM)
    const int ts = -TS;
    const size_t smem = attend_long_smem_bytes(p);
    cudaError_t e = cudaFuncSetAttribute(attend_long_kernel<D, G>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                         (int)smem);
    if (e != cudaSuccess) return e;
    const int grid = p.U < p.att_slots ? p.U : p.att_slots;
    attend_long_kernel<D, G><<<grid, kAttThreads, smem, s>>>(p, q, out, probs, ts);
    return cudaGetLastError();
  }
  const size_t smem = attend_smem_bytes(p, TS);
  cudaError_t e = cudaFuncSetAttribute(attend_kernel<D, G>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  if (e != cudaSuccess) return e;
  attend_kernel<D, G><<<p.U, kAttThreads, smem, s>>>(p, q, out, probs, TS);
  return cudaGetLastError();
}

template <int D>
static cudaError_t launch_att_d(const PoolDev& p, const uint16_t* q, float* out, float* probs, int TS, cudaStream_t s) {
  switch (p.G) {
    case 1: return launch_att<D, 1>(p, q, out, probs, TS, s);
    case 2: return launch_att<D, 2>(p, q, out, probs, TS, s);
    case 4: return launch_att<D, 4>(p, q, out, probs, TS, s);
    case 5: return launch_att<D, 5>(p, q, out, probs, TS, s);
    case 7: return launch_att<D, 7>(p, q, out, probs, TS, s);
    case 8: return launch_att<D, 8>(p, q, out, probs, TS, s);
    default: return cudaErrorInvalidValue;
  }
}

cudaError_t launch_attend(const PoolDev& p, const uint16_t* q, float* out, float* probs, int TS, cudaStream_t s) {
  return p.d == 128 ? launch_att_d<128>(p, q, out, probs, TS, s) : launch_att_d<64>(p, q, out, probs, TS, s);
}

}  // namespace dkv
