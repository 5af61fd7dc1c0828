// dkv_internal.cuh — device-side structures and primitives shared by the sm_100a kernels.
// Product code: never includes or links anything under oracle/.
#pragma once
#include <cuda_fp16.h>
#include <cuda_runtime.h>
#include <stdint.h>

#include "../../include/dkv.h"

namespace dkv {

constexpr int kSegTokens = 256;         // prefill rank checkpoint granularity (tokens per segment)
constexpr unsigned kFull = 0xFFFFFFFFu;

// Device control block at arena offset 0 (256 B).
struct Ctrl {
  int64_t start;                 // ring index of the first free page (allocation pointer)
  int64_t free;                  // free pages; end = (start + free) mod P (recycling pointer, Q1)
  int32_t status;                // sticky device status, first error wins
  int32_t oom_count;
  unsigned long long ticket;     // dynamic tile tickets of compact_alloc (monotonic)
  unsigned long long arrive;     // grid-barrier arrivals of compact_alloc (monotonic)
  int64_t last_demand, last_freed;
  int64_t total_dem, total_fr;   // published by the last scan tile before the barrier
  unsigned long long bar_epoch;  // grid barriers crossed (only calls that take the barrier path)
  int64_t rec_end0;              // end pointer at entry of the last compact_alloc (deferred recycle)
  int32_t rec_deferred;          // 1: the last compact_alloc left its recycle copies to recycle_kernel
  // Status snapshots (reading Q36: every call takes the status once, at entry).  dkv_classify's kernels
  // never write `status` (their errors go to `pending`), so every classify warp sees the same entry value;
  // dkv_compact_alloc merges `pending` into `status` and leaves its final status in `qw_status`, the entry
  // status of the following dkv_quant_write, whose kernels read only that word.
  int32_t pending;
  int32_t qw_status;
  int32_t pad32;
  // decode tile sums (classify → compact_alloc): the epoch whose sums dkv_classify(DECODE) accumulated in tsum,
  // and the tiles of each compact_alloc call that have read their entry state (monotonic, num_tiles per call)
  unsigned long long tsum_ticket;
  unsigned long long arrive2;
};
static_assert(sizeof(Ctrl) <= 256, "ctrl block");

struct ClassGeom {
  int32_t C, kbits, vbits, k_row, v_row, off_k, off_kmeta, off_v, off_vmeta, off_score, off_pos;
};

// n / d and n % d for 0 <= n < 2^31 by multiply-high (Granlund-Montgomery): mul = ceil(2^(31+l) / d),
// l = ceil(log2 d); d = 1 is mul = 0.  Built on the host (make_fastdiv), checked there over every n a
// kernel can pass (fastdiv_check).
struct FastDiv {
  int32_t d;
  uint32_t mul;
  int32_t shr;
};
__host__ __device__ __forceinline__ int32_t fdiv(const FastDiv& f, int32_t n) {
#ifdef __CUDA_ARCH__
  return f.mul == 0 ? n : (int32_t)(__umulhi((uint32_t)n, f.mul) >> f.shr);
#else
  return f.mul == 0 ? n : (int32_t)((((uint64_t)(uint32_t)n * f.mul) >> 32) >> f.shr);
#endif
}
__host__ __device__ __forceinline__ int32_t fmod_(const FastDiv& f, int32_t n) { return n - fdiv(f, n) * f.d; }
inline FastDiv make_fastdiv(int32_t d) {
  FastDiv f;
  f.d = d;
  if (d <= 1) { f.mul = 0; f.shr = 0; return f; }
  int l = 0;
  while ((1ll << l) < d) l++;
  f.mul = (uint32_t)((((uint64_t)1 << (31 + l)) + (uint64_t)d - 1) / (uint64_t)d);
  f.shr = l - 1;
  return f;
}
inline bool fastdiv_check(const FastDiv& f, int64_t n_max) {
  for (int64_t n = 0; n <= n_max && n < ((int64_t)1 << 31); n++)
    if (fdiv(f, (int32_t)n) != (int32_t)(n / f.d)) return false;
  return true;
}

// Everything a kernel needs, passed by value.
struct PoolDev {
  int32_t R, Ly, H, LyH, U, d, M, W, L, P, page_bytes, Ch, Cl;
  int32_t prompt_den, num_tiles, tile_units, nseg;
  float alpha_h, alpha_l;
  ClassGeom g[3];
  Ctrl* ctrl;
  unsigned long long* tile_status;
  int32_t* ring;
  int32_t* table;
  int32_t* n_h;
  int32_t* n_l;
  int8_t* req_state;
  int32_t* seq_len;
  int32_t* prompt_len;
  int32_t* admit;
  int32_t* pf_nh;
  int32_t* pf_nl;
  int32_t* pf_seg;      // [U][nseg][2] exclusive (high, low) ranks at each segment start
  __half* win_k;
  __half* win_v;
  uint8_t* pages;
  int64_t* stats;       // int64[4] admission counters
  FastDiv div_LyH, div_W, div_Ch, div_Cl;   // u -> request, position -> window slot, slot -> (page, index)
  int64_t* tile_sums;   // [num_tiles][3] prompt-workflow scan scratch
  uint32_t* tsum;       // [2][num_tiles][2] decode tile sums {demand, freed pages} by ticket parity (classify)
  int32_t* rec;         // [U][3] deferred recycle: {ring offset from the end pointer, ph, freed pages}
  float* win_sig;       // [U][W] significance of the window tokens (NEXT-2)
  int32_t* secmin;      // [U][8] {sig_h, pos_h, slot_h, sig_l, pos_l, slot_l, valid, 0} from dkv_attend
  int32_t G;            // q_per_kv
  float* head_alpha;    // [LyH][2] per-head (alpha_h, alpha_l) (NEXT-4)
  float* att_scratch;   // [att_slots][GP + 2][M] long-context attention scratch (NEXT-2), or null
  int32_t att_slots;
  float* tc_scratch;    // [tc_slots][tc_slot_rows][GP] logits of the persistent tensor-core attention CTAs, or null
  int32_t tc_slots, tc_slot_rows;
  int32_t use_head_alpha;   // 1: head_alpha replaces alpha_h / alpha_l
  int32_t prefill_wf;   // dkv_config_t.prefill_workflow
  int4* qpid;           // [U] {t_c's page, downgraded victim's KV_l page, N if the request is ACTIVE else 0, 0}
                        // for dkv_quant_write(DECODE), written by dkv_classify(DECODE) (+ granted pages by compact)
  int32_t pdl;          // launch option: 1 = programmatic dependent launch (decode-step CUDA graphs)
  // NEXT-4 three-level tier FP16-K8V4-K4V2 (readings Q38-Q44)
  int32_t top;          // 1: the FP16 class TOP above High
  float alpha_t;
  int32_t Lt, Ct;       // TOP table slots per unit, tokens per TOP page
  ClassGeom gt;         // TOP page geometry: fp16 K / V rows (k_row = v_row = 2d), no metadata
  int32_t* ttable;      // [U][Lt] TOP page table, left to right
  int32_t* n_t;         // [U] stored TOP tokens
  int32_t* pf_nt;       // [U] prompt TOP counts
  int32_t* pf_seg_t;    // [U][nseg] exclusive TOP rank at each segment start
  FastDiv div_Ct;
};

// Deferred-recycle record of a freed unit (p.rec, 4 ints): {ring offset from the end pointer, ph, freed pages,
// pt}.  The unit's freed slots as one flat list: TOP table slots [0, pt), then bidirectional slots [0, ph) and
// [L - pl, L) (Q13, Q41).
__device__ __forceinline__ int32_t* freed_slot(const PoolDev& p, int u, int k, int pt, int ph, int nfr) {
  if (k < pt) return p.ttable + (size_t)u * p.Lt + k;
  const int kk = k - pt;
  return p.table + (size_t)u * p.L + (kk < ph ? kk : p.L - (nfr - pt) + kk);
}

// kernel launch with optional programmatic dependent launch (cudaLaunchKernelEx)
template <typename... KArgs, typename... Args>
inline cudaError_t launch_ex(void (*k)(KArgs...), dim3 grid, dim3 block, size_t smem, cudaStream_t s, bool pdl,
                             Args... args) {
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = grid;
  cfg.blockDim = block;
  cfg.dynamicSmemBytes = smem;
  cfg.stream = s;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  attr[0].val.programmaticStreamSerializationAllowed = 1;
  cfg.attrs = attr;
  cfg.numAttrs = pdl ? 1 : 0;
  return cudaLaunchKernelEx(&cfg, k, args...);
}

// ------------------------------------------------------------------------------------- memory ops
__device__ __forceinline__ int32_t ld_volatile(const int32_t* p) { return *(volatile const int32_t*)p; }
__device__ __forceinline__ int64_t ld_volatile(const int64_t* p) { return *(volatile const int64_t*)p; }

__device__ __forceinline__ unsigned long long ld_acquire(const unsigned long long* p) {
  unsigned long long v;
  asm volatile("ld.acquire.gpu.global.u64 %0, [%1];" : "=l"(v) : "l"(p) : "memory");
  return v;
}
__device__ __forceinline__ void st_release(unsigned long long* p, unsigned long long v) {
  asm volatile("st.release.gpu.global.u64 [%0], %1;" ::"l"(p), "l"(v) : "memory");
}
__device__ __forceinline__ uint32_t ld_nc_u32(const void* p) {
  uint32_t v;
  asm volatile("ld.global.nc.L1::no_allocate.u32 %0, [%1];" : "=r"(v) : "l"(p));
  return v;
}
__device__ __forceinline__ uint4 ld_nc_v4(const void* p) {
  uint4 v;
  asm volatile("ld.global.nc.L1::no_allocate.v4.u32 {%0,%1,%2,%3}, [%4];"
               : "=r"(v.x), "=r"(v.y), "=r"(v.z), "=r"(v.w)
               : "l"(p));
  return v;
}
// same, with the L2 fetch limited to the 64-B sector pair the load touches (.L2::64B prefetch size)
__device__ __forceinline__ uint4 ld_nc_v4_64(const void* p) {
  uint4 v;
  asm volatile("ld.global.nc.L1::no_allocate.L2::64B.v4.u32 {%0,%1,%2,%3}, [%4];"
               : "=r"(v.x), "=r"(v.y), "=r"(v.z), "=r"(v.w)
               : "l"(p));
  return v;
}
// streaming loads of inputs read exactly once
__device__ __forceinline__ uint4 ld_stream_v4(const void* p) {
  uint4 v;
  asm volatile("ld.global.cs.v4.u32 {%0,%1,%2,%3}, [%4];"
               : "=r"(v.x), "=r"(v.y), "=r"(v.z), "=r"(v.w)
               : "l"(p));
  return v;
}

__device__ __forceinline__ void set_status(Ctrl* c, int32_t st) { atomicCAS(&c->status, 0, st); }
// an error found by a dkv_classify kernel (Q36): merged into `status` by the next dkv_compact_alloc
__device__ __forceinline__ void set_pending(Ctrl* c, int32_t st) { atomicCAS(&c->pending, 0, st); }

// Programmatic dependent launch (sm_90+): a kernel launched with the programmatic-serialization attribute
// may start while its predecessor runs; pdl_wait() blocks until the predecessor grid has completed and its
// writes are visible, pdl_trigger() lets the successor launch.  Both are no-ops without the attribute.  Every
// kernel of the decode step triggers only after its own wait, so when a kernel starts, the kernel two back
// has completed: code before pdl_wait() may read anything the immediate predecessor does not write.
__device__ __forceinline__ void pdl_wait() { asm volatile("griddepcontrol.wait;" ::: "memory"); }
__device__ __forceinline__ void pdl_trigger() { asm volatile("griddepcontrol.launch_dependents;" ::: "memory"); }

// ------------------------------------------------------------------------------------- async bulk copies
// 1-D TMA (cp.async.bulk) global -> shared with mbarrier transaction counting (sm_90+ / sm_100a).
__device__ __forceinline__ uint32_t smem_u32(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }
__device__ __forceinline__ void mbar_init(uint64_t* bar, uint32_t count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count) : "memory");
}
__device__ __forceinline__ void fence_mbar_init() {
  asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
}
__device__ __forceinline__ void fence_proxy_async_smem() {
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
}
__device__ __forceinline__ void mbar_arrive_expect_tx(uint64_t* bar, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)), "r"(bytes) : "memory");
}
__device__ __forceinline__ void bulk_g2s(void* dst, const void* src, uint32_t bytes, uint64_t* bar) {
  asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];"
               ::"r"(smem_u32(dst)), "l"(src), "r"(bytes), "r"(smem_u32(bar)) : "memory");
}
// Ampere-style per-thread 16-byte async copies (LDGSTS), L2-only (.cg).
__device__ __forceinline__ void cp_async16(void* dst, const void* src, bool pred) {
  asm volatile(
      "{\n"
      ".reg .pred p;\n"
      "setp.ne.b32 p, %2, 0;\n"
      "@p cp.async.cg.shared.global [%0], [%1], 16;\n"
      "}\n" ::"r"(smem_u32(dst)), "l"(src), "r"((int)pred) : "memory");
}
__device__ __forceinline__ void cp_async_commit() { asm volatile("cp.async.commit_group;" ::: "memory"); }
template <int N>
__device__ __forceinline__ void cp_async_wait() { asm volatile("cp.async.wait_group %0;" ::"n"(N) : "memory"); }

__device__ __forceinline__ void mbar_wait(uint64_t* bar, uint32_t parity) {
  asm volatile(
      "{\n"
      ".reg .pred P1;\n"
      "WAIT_%=:\n"
      "mbarrier.try_wait.parity.shared::cta.b64 P1, [%0], %1;\n"
      "@!P1 bra WAIT_%=;\n"
      "}\n" ::"r"(smem_u32(bar)), "r"(parity) : "memory");
}

// ------------------------------------------------------------------------------------- float helpers
// Total order on finite floats with -0 < +0 (Q16): monotone unsigned key.
__device__ __forceinline__ uint32_t total_key(float f) {
  uint32_t b = __float_as_uint(f);
  return (b & 0x80000000u) ? ~b : (b | 0x80000000u);
}
__device__ __forceinline__ float key_to_float(uint32_t k) {
  return __uint_as_float((k & 0x80000000u) ? (k & 0x7FFFFFFFu) : ~k);
}
__device__ __forceinline__ bool finite_f(float x) { return (__float_as_uint(x) & 0x7F800000u) != 0x7F800000u; }
__device__ __forceinline__ float canon_zero(float x) { return x == 0.0f ? 0.0f : x; }

__device__ __forceinline__ void unpack_h8(const uint4& v, float x[8]) {
  const __half2* h = reinterpret_cast<const __half2*>(&v);
#pragma unroll
  for (int i = 0; i < 4; i++) {
    float2 f = __half22float2(h[i]);
    x[2 * i] = f.x;
    x[2 * i + 1] = f.y;
  }
}

// Quantize the 8 values each lane of a group of `gl` lanes holds (one d-vector per group) at `bits`
// (Q16).  Returns the packed codes of this lane's 8 elements (8*bits bits, lowest element in
// the LSBs, Q17) and the group's fp16 (s, z) as one u32 {s16 | z16 << 16}.  `ok` = all finite.
template <int GL>
__device__ __forceinline__ uint64_t quantize8(const float x[8], int bits, uint32_t& meta, bool& ok) {
  uint32_t kmin = 0xFFFFFFFFu, kmax = 0u;
  bool fin = true;
#pragma unroll
  for (int i = 0; i < 8; i++) {
    fin &= finite_f(x[i]);
    uint32_t k = total_key(x[i]);
    kmin = min(kmin, k);
    kmax = max(kmax, k);
  }
#pragma unroll
  for (int o = GL / 2; o > 0; o >>= 1) {
    kmin = min(kmin, __shfl_xor_sync(kFull, kmin, o));
    kmax = max(kmax, __shfl_xor_sync(kFull, kmax, o));
  }
  unsigned allfin = __ballot_sync(kFull, fin);
  const int lane = threadIdx.x & 31;
  const unsigned gmask = ((GL == 32) ? kFull : ((1u << GL) - 1u)) << (lane & ~(GL - 1) & 31);
  ok = (allfin & gmask) == gmask;
  const float mn = key_to_float(kmin), mx = key_to_float(kmax);
  const int Q = (1 << bits) - 1;
  float s32 = __fdiv_rn(__fsub_rn(mx, mn), (float)Q);
  __half s16 = __float2half_rn(s32), z16 = __float2half_rn(mn);
  const float sf = __half2float(s16), zf = __half2float(z16);
  meta = (uint32_t)__half_as_ushort(s16) | ((uint32_t)__half_as_ushort(z16) << 16);
  uint64_t packed = 0;
  if (sf != 0.0f) {
    const float inv = __fdiv_rn(1.0f, sf);
#pragma unroll
    for (int i = 0; i < 8; i++) {
      float t = __fmul_rn(__fsub_rn(x[i], zf), inv);
      float r = roundf(t);                       // round half away from zero
      r = fminf(fmaxf(r, 0.0f), (float)Q);
      packed |= (uint64_t)(uint32_t)r << (i * bits);
    }
  }
  return packed;
}

// ------------------------------------------------------------------------------------- fast fp16 quantizer
// Same arithmetic as quantize8 (and the oracle) for FP16 inputs, with far fewer instructions:
//  * min / max on packed half2 with NaN propagation (min.NaN / max.NaN), reduced across the group as one
//    half2 {min, -max}; a NaN or Inf input makes min or max non-finite -> ok = false;
//  * the sign of a zero minimum is fixed up exactly (total order -0 < +0, Q16) in a rare warp-uniform path;
//  * x - z with one mixed-precision add (add.rn.f32.f16: fp16 operand, fp32 result, one RN rounding —
//    identical to fsub_rn(float(x), z) since float(x) is exact);
//  * t >= 0 always (z = min exactly), so round-half-away(t) = floor(t + 1/2), computed exactly as
//    RD(RD(t + 1/2) + 2^23): the code lands in the low mantissa bits, no float->int conversion;
//  * t <= Q + 1/8 when s16 is a normal binary16 number, so the clamp is only applied when s16 is subnormal.
__device__ __forceinline__ float mixed_add_h(uint32_t h16, float c) {
  float r;
  asm("add.rn.f32.f16 %0, %1, %2;" : "=f"(r) : "h"((unsigned short)h16), "f"(c));
  return r;
}
__device__ __forceinline__ uint32_t pack4_lo_bytes(uint32_t a, uint32_t b, uint32_t c, uint32_t d) {
  return __byte_perm(__byte_perm(a, b, 0x0040), __byte_perm(c, d, 0x0040), 0x5410);
}

// Each lane of a G-lane group holds NW half2 words (elements [2*NW*gl, 2*NW*(gl+1)) of the vector).
// Writes NW*2*BITS/32 packed code words (lowest element in the LSBs, Q17) and meta = s16 | z16 << 16.
template <int G, int NW, int BITS>
__device__ __forceinline__ void quant_h16(const uint32_t (&x)[NW], uint32_t (&cw)[(NW * 2 * BITS) / 32],
                                          uint32_t& meta, bool& ok) {
  constexpr int NCW = (NW * 2 * BITS) / 32;
  constexpr float Qf = (float)((1 << BITS) - 1);
  __half2 lo = *reinterpret_cast<const __half2*>(&x[0]), hi = lo;
#pragma unroll
  for (int i = 1; i < NW; i++) {
    const __half2 v = *reinterpret_cast<const __half2*>(&x[i]);
    lo = __hmin2_nan(lo, v);
    hi = __hmax2_nan(hi, v);
  }
  __half2 key = __halves2half2(__hmin_nan(__low2half(lo), __high2half(lo)),
                               __hneg(__hmax_nan(__low2half(hi), __high2half(hi))));
#pragma unroll
  for (int o = G / 2; o > 0; o >>= 1) {
    uint32_t k = *reinterpret_cast<uint32_t*>(&key);
    k = __shfl_xor_sync(kFull, k, o);
    key = __hmin2_nan(key, *reinterpret_cast<__half2*>(&k));
  }
  unsigned short mnb = __half_as_ushort(__low2half(key));
  const unsigned short mxb = __half_as_ushort(__hneg(__high2half(key)));
  const bool zmin = (mnb & 0x7FFFu) == 0;
  if (__any_sync(kFull, zmin)) {                        // rare: which zero is the minimum?
    bool negz = false;
#pragma unroll
    for (int i = 0; i < NW; i++) negz |= ((x[i] & 0xFFFFu) == 0x8000u) | ((x[i] >> 16) == 0x8000u);
    const unsigned b = __ballot_sync(kFull, negz);
    const int lane = threadIdx.x & 31;
    const unsigned gmask = ((G == 32) ? kFull : ((1u << G) - 1u)) << (lane & ~(G - 1) & 31);
    if (zmin) mnb = (b & gmask) ? 0x8000u : 0x0000u;
  }
  ok = ((mnb & 0x7C00u) != 0x7C00u) && ((mxb & 0x7C00u) != 0x7C00u);
  const float mn = __half2float(__ushort_as_half(mnb)), mx = __half2float(__ushort_as_half(mxb));
  const float s32 = __fdiv_rn(__fsub_rn(mx, mn), Qf);
  const __half s16 = __float2half_rn(s32);
  meta = (uint32_t)__half_as_ushort(s16) | ((uint32_t)mnb << 16);
  const float sf = __half2float(s16);
  if (sf == 0.0f) {
#pragma unroll
    for (int w = 0; w < NCW; w++) cw[w] = 0u;
    return;
  }
  const float inv = __fdiv_rn(1.0f, sf);
  const float nz = -mn;                                  // z = min exactly (FP16 input)
  const float cap = (sf >= 6.103515625e-05f) ? 3.0e38f : Qf;   // clamp only for subnormal s16
  uint32_t ub[NW * 2];
#pragma unroll
  for (int i = 0; i < NW; i++) {
#pragma unroll
    for (int hh = 0; hh < 2; hh++) {
      const float d = mixed_add_h(hh ? (x[i] >> 16) : (x[i] & 0xFFFFu), nz);
      float t = __fmul_rn(d, inv);
      t = fminf(t, cap);
      const float a = __fadd_rd(t, 0.5f);
      ub[2 * i + hh] = __float_as_uint(__fadd_rd(a, 8388608.0f));
    }
  }
#pragma unroll
  for (int w = 0; w < NCW; w++) {
    if constexpr (BITS == 8) {
      cw[w] = pack4_lo_bytes(ub[4 * w], ub[4 * w + 1], ub[4 * w + 2], ub[4 * w + 3]);
    } else if constexpr (BITS == 4) {
      const uint32_t ev = pack4_lo_bytes(ub[8 * w], ub[8 * w + 2], ub[8 * w + 4], ub[8 * w + 6]);
      const uint32_t od = pack4_lo_bytes(ub[8 * w + 1], ub[8 * w + 3], ub[8 * w + 5], ub[8 * w + 7]);
      cw[w] = ev | (od << 4);
    } else {
      uint32_t acc = 0;
#pragma unroll
      for (int m = 0; m < 4; m++)
        acc |= pack4_lo_bytes(ub[16 * w + m], ub[16 * w + m + 4], ub[16 * w + m + 8], ub[16 * w + m + 12]) << (2 * m);
      cw[w] = acc;
    }
  }
}

template <int N>
__device__ __forceinline__ void store_words(uint8_t* dst, const uint32_t (&w)[N]) {
  if constexpr (N % 4 == 0) {
#pragma unroll
    for (int i = 0; i < N; i += 4) reinterpret_cast<uint4*>(dst)[i / 4] = make_uint4(w[i], w[i + 1], w[i + 2], w[i + 3]);
  } else if constexpr (N == 2) {
    *reinterpret_cast<uint2*>(dst) = make_uint2(w[0], w[1]);
  } else {
    *reinterpret_cast<uint32_t*>(dst) = w[0];
  }
}

// ---- chunk-interleaved quantizer.  A d-vector is spread over a G-lane group in 8-element (16-B) chunks,
// lane q holding chunks q, q+G, q+2G, ... so that each warp-wide 16-B load / code store of the group
// touches contiguous bytes.  Chunk c's codes occupy bytes [c*bits, (c+1)*bits) of the code row.
__device__ __forceinline__ uint2 pack8_codes(const uint32_t (&ub)[8], int bits) {
  if (bits == 8)
    return make_uint2(pack4_lo_bytes(ub[0], ub[1], ub[2], ub[3]), pack4_lo_bytes(ub[4], ub[5], ub[6], ub[7]));
  if (bits == 4) {
    const uint32_t ev = pack4_lo_bytes(ub[0], ub[2], ub[4], ub[6]);
    const uint32_t od = pack4_lo_bytes(ub[1], ub[3], ub[5], ub[7]);
    return make_uint2(ev | (od << 4), 0u);
  }
  uint32_t acc = 0;
#pragma unroll
  for (int m = 0; m < 4; m++) acc |= __byte_perm(ub[m], ub[m + 4], 0x0040) << (2 * m);
  return make_uint2(acc & 0xFFFFu, 0u);
}

__device__ __forceinline__ void store_chunk_codes(uint8_t* row, int chunk, int bits, uint2 v) {
  uint8_t* d = row + chunk * bits;
  if (bits == 8) *reinterpret_cast<uint2*>(d) = v;
  else if (bits == 4) *reinterpret_cast<uint32_t*>(d) = v.x;
  else *reinterpret_cast<uint16_t*>(d) = (uint16_t)v.x;
}

// FP16 input (x[c][w] = half2 word w of this lane's chunk c), runtime bits, group-masked collectives.
// Arithmetic identical to quant_h16 / the oracle.
template <int G, int NCH>
__device__ __forceinline__ void quant_chunks_h16(const uint32_t (&x)[NCH][4], int bits, unsigned gmask,
                                                 uint2 (&pk)[NCH], uint32_t& meta, bool& ok) {
  const float Qf = (float)((1 << bits) - 1);
  __half2 lo = *reinterpret_cast<const __half2*>(&x[0][0]), hi = lo;
#pragma unroll
  for (int c = 0; c < NCH; c++)
#pragma unroll
    for (int w = 0; w < 4; w++) {
      if (c == 0 && w == 0) continue;
      const __half2 v = *reinterpret_cast<const __half2*>(&x[c][w]);
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
  if ((mnb & 0x7FFFu) == 0) {                           // group-uniform: which zero is the minimum?
    bool negz = false;
#pragma unroll
    for (int c = 0; c < NCH; c++)
#pragma unroll
      for (int w = 0; w < 4; w++) negz |= ((x[c][w] & 0xFFFFu) == 0x8000u) | ((x[c][w] >> 16) == 0x8000u);
    mnb = (__ballot_sync(gmask, negz) & gmask) ? 0x8000u : 0x0000u;
  }
  ok = ((mnb & 0x7C00u) != 0x7C00u) && ((mxb & 0x7C00u) != 0x7C00u);
  const float mn = __half2float(__ushort_as_half(mnb)), mx = __half2float(__ushort_as_half(mxb));
  const float s32 = __fdiv_rn(__fsub_rn(mx, mn), Qf);
  const __half s16 = __float2half_rn(s32);
  meta = (uint32_t)__half_as_ushort(s16) | ((uint32_t)mnb << 16);
  const float sf = __half2float(s16);
  const float inv = __fdiv_rn(1.0f, sf);
  const float nz = -mn;
  const float cap = (sf >= 6.103515625e-05f) ? 3.0e38f : Qf;
  const uint32_t zmask = sf != 0.0f ? 0xFFFFFFFFu : 0u;  // s16 == 0: all codes 0
#pragma unroll
  for (int c = 0; c < NCH; c++) {
    uint32_t ub[8];
#pragma unroll
    for (int w = 0; w < 4; w++)
#pragma unroll
      for (int hh = 0; hh < 2; hh++) {
        const float d = mixed_add_h(hh ? (x[c][w] >> 16) : (x[c][w] & 0xFFFFu), nz);
        float t = __fmul_rn(d, inv);
        t = fminf(t, cap);
        const float a = __fadd_rd(t, 0.5f);
        ub[2 * w + hh] = __float_as_uint(__fadd_rd(a, 8388608.0f)) & zmask;
      }
    pk[c] = pack8_codes(ub, bits);
  }
}

template <int BITS>
__device__ __forceinline__ uint2 pack8_codes_ct(const uint32_t (&ub)[8]) {
  if constexpr (BITS == 8) {
    return make_uint2(pack4_lo_bytes(ub[0], ub[1], ub[2], ub[3]), pack4_lo_bytes(ub[4], ub[5], ub[6], ub[7]));
  } else if constexpr (BITS == 4) {
    const uint32_t ev = pack4_lo_bytes(ub[0], ub[2], ub[4], ub[6]);
    const uint32_t od = pack4_lo_bytes(ub[1], ub[3], ub[5], ub[7]);
    return make_uint2(ev | (od << 4), 0u);
  } else {
    uint32_t acc = 0;
#pragma unroll
    for (int m = 0; m < 4; m++) acc |= __byte_perm(ub[m], ub[m + 4], 0x0040) << (2 * m);
    return make_uint2(acc & 0xFFFFu, 0u);
  }
}

template <int BITS>
__device__ __forceinline__ void store_chunk_codes_ct(uint8_t* row, int chunk, uint2 v) {
  uint8_t* d = row + chunk * BITS;
  if constexpr (BITS == 8) *reinterpret_cast<uint2*>(d) = v;
  else if constexpr (BITS == 4) *reinterpret_cast<uint32_t*>(d) = v.x;
  else *reinterpret_cast<uint16_t*>(d) = (uint16_t)v.x;
}

// Compile-time bit width, called by ALL 32 lanes of the warp (warp-uniform fast path): as
// quant_chunks_h16, but the clamp (subnormal s16) and the s16 == 0 masking run only when some group of
// the warp needs them.
template <int G, int NCH, int BITS>
__device__ __forceinline__ void quant_chunks_h16_ct(const uint32_t (&x)[NCH][4], unsigned gmask, uint2 (&pk)[NCH],
                                                    uint32_t& meta, bool& ok) {
  constexpr float Qf = (float)((1 << BITS) - 1);
  __half2 lo = *reinterpret_cast<const __half2*>(&x[0][0]), hi = lo;
#pragma unroll
  for (int c = 0; c < NCH; c++)
#pragma unroll
    for (int w = 0; w < 4; w++) {
      if (c == 0 && w == 0) continue;
      const __half2 v = *reinterpret_cast<const __half2*>(&x[c][w]);
      lo = __hmin2_nan(lo, v);
      hi = __hmax2_nan(hi, v);
    }
  __half2 key = __halves2half2(__hmin_nan(__low2half(lo), __high2half(lo)),
                               __hneg(__hmax_nan(__low2half(hi), __high2half(hi))));
#pragma unroll
  for (int o = G / 2; o > 0; o >>= 1) {
    uint32_t k = *reinterpret_cast<uint32_t*>(&key);
    k = __shfl_xor_sync(kFull, k, o);
    key = __hmin2_nan(key, *reinterpret_cast<__half2*>(&k));
  }
  unsigned short mnb = __half_as_ushort(__low2half(key));
  const unsigned short mxb = __half_as_ushort(__hneg(__high2half(key)));
  const bool zmin = (mnb & 0x7FFFu) == 0;
  if (__any_sync(kFull, zmin)) {                        // rare: which zero is the minimum?
    bool negz = false;
#pragma unroll
    for (int c = 0; c < NCH; c++)
#pragma unroll
      for (int w = 0; w < 4; w++) negz |= ((x[c][w] & 0xFFFFu) == 0x8000u) | ((x[c][w] >> 16) == 0x8000u);
    const unsigned b = __ballot_sync(kFull, negz);
    if (zmin) mnb = (b & gmask) ? 0x8000u : 0x0000u;
  }
  ok = ((mnb & 0x7C00u) != 0x7C00u) && ((mxb & 0x7C00u) != 0x7C00u);
  const float mn = __half2float(__ushort_as_half(mnb)), mx = __half2float(__ushort_as_half(mxb));
  const float s32 = __fdiv_rn(__fsub_rn(mx, mn), Qf);
  const __half s16 = __float2half_rn(s32);
  meta = (uint32_t)__half_as_ushort(s16) | ((uint32_t)mnb << 16);
  const float sf = __half2float(s16);
  const float inv = __fdiv_rn(1.0f, sf);
  const float nz = -mn;
  if (!__any_sync(kFull, !(sf >= 6.103515625e-05f))) {  // every s16 normal: t <= Q + 1/8, no clamp needed
#pragma unroll
    for (int c = 0; c < NCH; c++) {
      uint32_t ub[8];
#pragma unroll
      for (int w = 0; w < 4; w++)
#pragma unroll
        for (int hh = 0; hh < 2; hh++) {
          const float d = mixed_add_h(hh ? (x[c][w] >> 16) : (x[c][w] & 0xFFFFu), nz);
          const float a = __fadd_rd(__fmul_rn(d, inv), 0.5f);
          ub[2 * w + hh] = __float_as_uint(__fadd_rd(a, 8388608.0f));
        }
      pk[c] = pack8_codes_ct<BITS>(ub);
    }
  } else {
    const float cap = (sf >= 6.103515625e-05f) ? 3.0e38f : Qf;
    const uint32_t zmask = sf != 0.0f ? 0xFFFFFFFFu : 0u;
#pragma unroll
    for (int c = 0; c < NCH; c++) {
      uint32_t ub[8];
#pragma unroll
      for (int w = 0; w < 4; w++)
#pragma unroll
        for (int hh = 0; hh < 2; hh++) {
          const float d = mixed_add_h(hh ? (x[c][w] >> 16) : (x[c][w] & 0xFFFFu), nz);
          const float t = fminf(__fmul_rn(d, inv), cap);
          const float a = __fadd_rd(t, 0.5f);
          ub[2 * w + hh] = __float_as_uint(__fadd_rd(a, 8388608.0f)) & zmask;
        }
      pk[c] = pack8_codes_ct<BITS>(ub);
    }
  }
}

// The same quantizer split in two so a caller can validate both vectors of a token before storing
// either (Q30): qstats_h16_ct = min/max, group reduction, s, z, metadata, finiteness; qencode_h16_ct =
// the codes.  Arithmetic identical to quant_chunks_h16_ct.
struct QStats {
  float nz, inv, cap;
  uint32_t zmask, meta;
  bool ok, all_normal;      // all_normal is warp-uniform
};
template <int G, int NCH, int BITS>
__device__ __forceinline__ QStats qstats_h16_ct(const uint32_t (&x)[NCH][4], unsigned gmask) {
  constexpr float Qf = (float)((1 << BITS) - 1);
  __half2 lo = *reinterpret_cast<const __half2*>(&x[0][0]), hi = lo;
#pragma unroll
  for (int c = 0; c < NCH; c++)
#pragma unroll
    for (int w = 0; w < 4; w++) {
      if (c == 0 && w == 0) continue;
      const __half2 v = *reinterpret_cast<const __half2*>(&x[c][w]);
      lo = __hmin2_nan(lo, v);
      hi = __hmax2_nan(hi, v);
    }
  __half2 key = __halves2half2(__hmin_nan(__low2half(lo), __high2half(lo)),
                               __hneg(__hmax_nan(__low2half(hi), __high2half(hi))));
#pragma unroll
  for (int o = G / 2; o > 0; o >>= 1) {
    uint32_t k = *reinterpret_cast<uint32_t*>(&key);
    k = __shfl_xor_sync(kFull, k, o);
    key = __hmin2_nan(key, *reinterpret_cast<__half2*>(&k));
  }
  unsigned short mnb = __half_as_ushort(__low2half(key));
  const unsigned short mxb = __half_as_ushort(__hneg(__high2half(key)));
  const bool zmin = (mnb & 0x7FFFu) == 0;
  if (__any_sync(kFull, zmin)) {                        // rare: which zero is the minimum?
    bool negz = false;
#pragma unroll
    for (int c = 0; c < NCH; c++)
#pragma unroll
      for (int w = 0; w < 4; w++) negz |= ((x[c][w] & 0xFFFFu) == 0x8000u) | ((x[c][w] >> 16) == 0x8000u);
    const unsigned b = __ballot_sync(kFull, negz);
    if (zmin) mnb = (b & gmask) ? 0x8000u : 0x0000u;
  }
  QStats st;
  st.ok = ((mnb & 0x7C00u) != 0x7C00u) && ((mxb & 0x7C00u) != 0x7C00u);
  const float mn = __half2float(__ushort_as_half(mnb)), mx = __half2float(__ushort_as_half(mxb));
  const float s32 = __fdiv_rn(__fsub_rn(mx, mn), Qf);
  const __half s16 = __float2half_rn(s32);
  st.meta = (uint32_t)__half_as_ushort(s16) | ((uint32_t)mnb << 16);
  const float sf = __half2float(s16);
  st.inv = __fdiv_rn(1.0f, sf);
  st.nz = -mn;
  st.all_normal = !__any_sync(kFull, !(sf >= 6.103515625e-05f));
  st.cap = (sf >= 6.103515625e-05f) ? 3.0e38f : Qf;
  st.zmask = sf != 0.0f ? 0xFFFFFFFFu : 0u;
  return st;
}
template <int NCH, int BITS>
__device__ __forceinline__ void qencode_h16_ct(const uint32_t (&x)[NCH][4], const QStats& st, uint2 (&pk)[NCH]) {
  if (st.all_normal) {                                  // every s16 normal: t <= Q + 1/8, no clamp needed
#pragma unroll
    for (int c = 0; c < NCH; c++) {
      uint32_t ub[8];
#pragma unroll
      for (int w = 0; w < 4; w++)
#pragma unroll
        for (int hh = 0; hh < 2; hh++) {
          const float d = mixed_add_h(hh ? (x[c][w] >> 16) : (x[c][w] & 0xFFFFu), st.nz);
          const float a = __fadd_rd(__fmul_rn(d, st.inv), 0.5f);
          ub[2 * w + hh] = __float_as_uint(__fadd_rd(a, 8388608.0f));
        }
      pk[c] = pack8_codes_ct<BITS>(ub);
    }
  } else {
#pragma unroll
    for (int c = 0; c < NCH; c++) {
      uint32_t ub[8];
#pragma unroll
      for (int w = 0; w < 4; w++)
#pragma unroll
        for (int hh = 0; hh < 2; hh++) {
          const float d = mixed_add_h(hh ? (x[c][w] >> 16) : (x[c][w] & 0xFFFFu), st.nz);
          const float t = fminf(__fmul_rn(d, st.inv), st.cap);
          const float a = __fadd_rd(t, 0.5f);
          ub[2 * w + hh] = __float_as_uint(__fadd_rd(a, 8388608.0f)) & st.zmask;
        }
      pk[c] = pack8_codes_ct<BITS>(ub);
    }
  }
}

// FP32 input (a dequantized K8V4 token being downgraded, Q9): x[c][e] = element e of chunk c.
// min/max with fminf/fmaxf (IEEE minimum/maximum, -0 < +0 on sm_100 as the oracle's total order);
// z = f16(min) may exceed some inputs, so t is clamped to [0, Q] before the exact RD rounding — equal to
// clamp(round_half_away(t), 0, Q).
template <int G, int NCH>
__device__ __forceinline__ void quant_chunks_f32(const float (&x)[NCH][8], int bits, unsigned gmask,
                                                 uint2 (&pk)[NCH], uint32_t& meta) {
  const float Qf = (float)((1 << bits) - 1);
  float mn = x[0][0], mx = x[0][0];
#pragma unroll
  for (int c = 0; c < NCH; c++)
#pragma unroll
    for (int e = 0; e < 8; e++) { mn = fminf(mn, x[c][e]); mx = fmaxf(mx, x[c][e]); }
#pragma unroll
  for (int o = G / 2; o > 0; o >>= 1) {
    mn = fminf(mn, __shfl_xor_sync(gmask, mn, o));
    mx = fmaxf(mx, __shfl_xor_sync(gmask, mx, o));
  }
  const float s32 = __fdiv_rn(__fsub_rn(mx, mn), Qf);
  const __half s16 = __float2half_rn(s32), z16 = __float2half_rn(mn);
  meta = (uint32_t)__half_as_ushort(s16) | ((uint32_t)__half_as_ushort(z16) << 16);
  const float sf = __half2float(s16), zf = __half2float(z16);
  const float inv = __fdiv_rn(1.0f, sf);
  const uint32_t zmask = sf != 0.0f ? 0xFFFFFFFFu : 0u;
#pragma unroll
  for (int c = 0; c < NCH; c++) {
    uint32_t ub[8];
#pragma unroll
    for (int e = 0; e < 8; e++) {
      float t = __fmul_rn(__fsub_rn(x[c][e], zf), inv);
      t = fminf(fmaxf(t, 0.0f), Qf);
      const float a = __fadd_rd(t, 0.5f);
      ub[e] = __float_as_uint(__fadd_rd(a, 8388608.0f)) & zmask;
    }
    pk[c] = pack8_codes(ub, bits);
  }
}

// Dequantize one 8-element chunk (its `bits`-byte code piece) -> fp32 (X^ = s*Q + z).
__device__ __forceinline__ void dequant_chunk(const uint8_t* row, int chunk, int bits, uint32_t meta, float (&x)[8]) {
  const float sf = __half2float(__ushort_as_half((unsigned short)(meta & 0xFFFFu)));
  const float zf = __half2float(__ushort_as_half((unsigned short)(meta >> 16)));
  const uint8_t* s = row + chunk * bits;
  uint64_t v;
  if (bits == 8) { const uint2 t = *reinterpret_cast<const uint2*>(s); v = (uint64_t)t.x | ((uint64_t)t.y << 32); }
  else if (bits == 4) v = *reinterpret_cast<const uint32_t*>(s);
  else v = *reinterpret_cast<const uint16_t*>(s);
  const uint32_t Q = (1u << bits) - 1u;
#pragma unroll
  for (int e = 0; e < 8; e++) {
    const uint32_t q = (uint32_t)(v >> (e * bits)) & Q;
    x[e] = __fadd_rn(__fmul_rn(sf, __uint_as_float(0x4B000000u | q) - 8388608.0f), zf);
  }
}

// ---- runtime-bit-width variants for kernels whose lanes groups hold different classes (decode): the
// arithmetic is the same; only Q and the packing depend on `bits`; collectives use the group mask.
template <int E>
__device__ __forceinline__ int pack_codes_rt(const uint32_t (&ub)[E], int bits, uint32_t (&cw)[E / 4]) {
  if (bits == 8) {
#pragma unroll
    for (int w = 0; w < E / 4; w++) cw[w] = pack4_lo_bytes(ub[4 * w], ub[4 * w + 1], ub[4 * w + 2], ub[4 * w + 3]);
    return E / 4;
  }
  if (bits == 4) {
#pragma unroll
    for (int w = 0; w < E / 8; w++) {
      const uint32_t ev = pack4_lo_bytes(ub[8 * w], ub[8 * w + 2], ub[8 * w + 4], ub[8 * w + 6]);
      const uint32_t od = pack4_lo_bytes(ub[8 * w + 1], ub[8 * w + 3], ub[8 * w + 5], ub[8 * w + 7]);
      cw[w] = ev | (od << 4);
    }
    return E / 8;
  }
#pragma unroll
  for (int w = 0; w < E / 16; w++) {
    uint32_t acc = 0;
#pragma unroll
    for (int m = 0; m < 4; m++)
      acc |= pack4_lo_bytes(ub[16 * w + m], ub[16 * w + m + 4], ub[16 * w + m + 8], ub[16 * w + m + 12]) << (2 * m);
    cw[w] = acc;
  }
  return E / 16;
}

template <int NC>
__device__ __forceinline__ void store_words_rt(uint8_t* dst, const uint32_t (&w)[NC], int n) {
  if (n >= 4) {
#pragma unroll
    for (int i = 0; i < NC; i += 4)
      if (i < n) reinterpret_cast<uint4*>(dst)[i / 4] = make_uint4(w[i], w[i + 1], w[i + 2], w[i + 3]);
  } else if (n == 2) {
    *reinterpret_cast<uint2*>(dst) = make_uint2(w[0], w[1]);
  } else {
    *reinterpret_cast<uint32_t*>(dst) = w[0];
  }
}

// FP16 input, runtime bits, group-masked collectives.  Same arithmetic as quant_h16.
template <int G, int NW>
__device__ __forceinline__ int quant_h16_rt(const uint32_t (&x)[NW], int bits, unsigned gmask,
                                            uint32_t (&cw)[NW / 2], uint32_t& meta, bool& ok) {
  const float Qf = (float)((1 << bits) - 1);
  __half2 lo = *reinterpret_cast<const __half2*>(&x[0]), hi = lo;
#pragma unroll
  for (int i = 1; i < NW; i++) {
    const __half2 v = *reinterpret_cast<const __half2*>(&x[i]);
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
  if ((mnb & 0x7FFFu) == 0) {                           // group-uniform: which zero is the minimum?
    bool negz = false;
#pragma unroll
    for (int i = 0; i < NW; i++) negz |= ((x[i] & 0xFFFFu) == 0x8000u) | ((x[i] >> 16) == 0x8000u);
    mnb = (__ballot_sync(gmask, negz) & gmask) ? 0x8000u : 0x0000u;
  }
  ok = ((mnb & 0x7C00u) != 0x7C00u) && ((mxb & 0x7C00u) != 0x7C00u);
  const float mn = __half2float(__ushort_as_half(mnb)), mx = __half2float(__ushort_as_half(mxb));
  const float s32 = __fdiv_rn(__fsub_rn(mx, mn), Qf);
  const __half s16 = __float2half_rn(s32);
  meta = (uint32_t)__half_as_ushort(s16) | ((uint32_t)mnb << 16);
  const float sf = __half2float(s16);
  const float inv = __fdiv_rn(1.0f, sf);
  const float nz = -mn;
  const float cap = (sf >= 6.103515625e-05f) ? 3.0e38f : Qf;
  uint32_t ub[NW * 2];
#pragma unroll
  for (int i = 0; i < NW; i++) {
#pragma unroll
    for (int hh = 0; hh < 2; hh++) {
      const float d = mixed_add_h(hh ? (x[i] >> 16) : (x[i] & 0xFFFFu), nz);
      float t = __fmul_rn(d, inv);
      t = fminf(t, cap);
      const float a = __fadd_rd(t, 0.5f);
      ub[2 * i + hh] = sf != 0.0f ? __float_as_uint(__fadd_rd(a, 8388608.0f)) : 0u;
    }
  }
  return pack_codes_rt<NW * 2>(ub, bits, cw);
}

// FP32 input (a dequantized K8V4 token being downgraded, Q9), runtime bits, group-masked collectives.
// min/max with fminf/fmaxf (IEEE minimum/maximum: -0 < +0 on sm_100, as the oracle's total order);
// z = f16(min) may exceed some inputs, so t is clamped to [0, Q] before the exact RD rounding — the same
// result as clamp(round_half_away(t), 0, Q).
template <int G, int E>
__device__ __forceinline__ int quant_f32_rt(const float (&x)[E], int bits, unsigned gmask, uint32_t (&cw)[E / 4],
                                            uint32_t& meta) {
  const float Qf = (float)((1 << bits) - 1);
  float mn = x[0], mx = x[0];
#pragma unroll
  for (int i = 1; i < E; i++) { mn = fminf(mn, x[i]); mx = fmaxf(mx, x[i]); }
#pragma unroll
  for (int o = G / 2; o > 0; o >>= 1) {
    mn = fminf(mn, __shfl_xor_sync(gmask, mn, o));
    mx = fmaxf(mx, __shfl_xor_sync(gmask, mx, o));
  }
  const float s32 = __fdiv_rn(__fsub_rn(mx, mn), Qf);
  const __half s16 = __float2half_rn(s32), z16 = __float2half_rn(mn);
  meta = (uint32_t)__half_as_ushort(s16) | ((uint32_t)__half_as_ushort(z16) << 16);
  const float sf = __half2float(s16), zf = __half2float(z16);
  const float inv = __fdiv_rn(1.0f, sf);
  uint32_t ub[E];
#pragma unroll
  for (int i = 0; i < E; i++) {
    float t = __fmul_rn(__fsub_rn(x[i], zf), inv);
    t = fminf(fmaxf(t, 0.0f), Qf);
    const float a = __fadd_rd(t, 0.5f);
    ub[i] = sf != 0.0f ? __float_as_uint(__fadd_rd(a, 8388608.0f)) : 0u;
  }
  return pack_codes_rt<E>(ub, bits, cw);
}

// Dequantize E codes (bits each, packed LSB-first in words) -> fp32 (X^ = s*Q + z).
template <int E>
__device__ __forceinline__ void dequant_rt(const uint32_t* w, int bits, uint32_t meta, float (&x)[E]) {
  const float sf = __half2float(__ushort_as_half((unsigned short)(meta & 0xFFFFu)));
  const float zf = __half2float(__ushort_as_half((unsigned short)(meta >> 16)));
  const uint32_t Q = (1u << bits) - 1u;
#pragma unroll
  for (int i = 0; i < E; i++) {
    const int bit = i * bits;
    const uint32_t q = (w[bit >> 5] >> (bit & 31)) & Q;
    x[i] = __fadd_rn(__fmul_rn(sf, __uint_as_float(0x4B000000u | q) - 8388608.0f), zf);
  }
}

// Dequantize this lane's 8 codes (X^ = s*Q + z).
__device__ __forceinline__ void dequant8(uint64_t packed, int bits, uint32_t meta, float x[8]) {
  const float sf = __half2float(__ushort_as_half((unsigned short)(meta & 0xFFFFu)));
  const float zf = __half2float(__ushort_as_half((unsigned short)(meta >> 16)));
  const uint32_t Q = (1u << bits) - 1u;
#pragma unroll
  for (int i = 0; i < 8; i++) {
    uint32_t q = (uint32_t)(packed >> (i * bits)) & Q;
    x[i] = __fadd_rn(__fmul_rn(sf, (float)q), zf);
  }
}

__device__ __forceinline__ void store_codes(uint8_t* dst, uint64_t packed, int bits) {
  if (bits == 8) *reinterpret_cast<uint2*>(dst) = make_uint2((uint32_t)packed, (uint32_t)(packed >> 32));
  else if (bits == 4) *reinterpret_cast<uint32_t*>(dst) = (uint32_t)packed;
  else *reinterpret_cast<uint16_t*>(dst) = (uint16_t)packed;
}
__device__ __forceinline__ uint64_t load_codes(const uint8_t* src, int bits) {
  if (bits == 8) {
    uint2 v = *reinterpret_cast<const uint2*>(src);
    return (uint64_t)v.x | ((uint64_t)v.y << 32);
  }
  if (bits == 4) return *reinterpret_cast<const uint32_t*>(src);
  return *reinterpret_cast<const uint16_t*>(src);
}

// Geometry of class `cls` selected field by field (a runtime index into the kernel-parameter struct
// would force a local-memory copy of it).
__device__ __forceinline__ ClassGeom geom_of(const PoolDev& p, int cls) {
  const bool h = cls == DKV_CLS_HIGH;
  ClassGeom g;
  g.C = h ? p.g[1].C : p.g[2].C;
  g.kbits = h ? p.g[1].kbits : p.g[2].kbits;
  g.vbits = h ? p.g[1].vbits : p.g[2].vbits;
  g.k_row = h ? p.g[1].k_row : p.g[2].k_row;
  g.v_row = h ? p.g[1].v_row : p.g[2].v_row;
  g.off_k = h ? p.g[1].off_k : p.g[2].off_k;
  g.off_kmeta = h ? p.g[1].off_kmeta : p.g[2].off_kmeta;
  g.off_v = h ? p.g[1].off_v : p.g[2].off_v;
  g.off_vmeta = h ? p.g[1].off_vmeta : p.g[2].off_vmeta;
  g.off_score = h ? p.g[1].off_score : p.g[2].off_score;
  g.off_pos = h ? p.g[1].off_pos : p.g[2].off_pos;
  return g;
}

// Section slot s of class cls of unit u -> (page pointer, index in page)  (c.1)
__device__ __forceinline__ uint8_t* slot_page(const PoolDev& p, int cls, int u, int s, int& idx) {
  const int C = cls == DKV_CLS_HIGH ? p.g[1].C : p.g[2].C;
  const int k = (cls == DKV_CLS_HIGH) ? s / C : p.L - 1 - s / C;
  const int pid = p.table[(size_t)u * p.L + k];
  idx = s % C;
  return p.pages + (size_t)pid * (size_t)p.page_bytes;
}

__device__ __forceinline__ int ceil_div(int a, int b) { return (a + b - 1) / b; }

// Q35 (NEXT-4): the thresholds of unit u's (layer, head)
__device__ __forceinline__ float unit_alpha_h(const PoolDev& p, int u) {
  return p.use_head_alpha ? p.head_alpha[2 * fmod_(p.div_LyH, u)] : p.alpha_h;
}
__device__ __forceinline__ float unit_alpha_l(const PoolDev& p, int u) {
  return p.use_head_alpha ? p.head_alpha[2 * fmod_(p.div_LyH, u) + 1] : p.alpha_l;
}

// ---- per-CTA copy of the per-request arrays.  Every unit of a request reads the same state / length
// word, so thousands of warps loading them (or the control block) directly all queue on the same few L2
// lines at one slice — measured to dominate the decode kernels.  Persistent CTAs copy the arrays into
// shared memory once instead (one coalesced pass per CTA).  Above kReqSmemMax requests the kernels read
// global memory directly.
constexpr int kReqSmemMax = 4096;
__host__ __device__ __forceinline__ size_t req_cache_bytes(int R) {
  return R <= kReqSmemMax ? (size_t)R * 4 + (((size_t)R + 15) & ~(size_t)15) : 0;
}
struct ReqCache {
  const int32_t* len;
  const int8_t* st;
};
// smem: [R] int32 committed lengths, then [R] int8 states (caller provides req_cache_bytes(R) bytes)
__device__ __forceinline__ ReqCache load_req_cache(const PoolDev& p, void* smem) {
  ReqCache c;
  if (p.R <= kReqSmemMax) {
    int32_t* len = reinterpret_cast<int32_t*>(smem);
    int8_t* st = reinterpret_cast<int8_t*>(len + p.R);
    for (int i = threadIdx.x; i < p.R; i += blockDim.x) { len[i] = p.seq_len[i]; st[i] = p.req_state[i]; }
    c.len = len;
    c.st = st;
  } else {
    c.len = p.seq_len;
    c.st = p.req_state;
  }
  return c;                                            // caller: __syncthreads() before use
}

// CTAs of a persistent kernel: resident CTAs per SM x SMs (cached per kernel by the caller)
template <typename K>
inline int persistent_grid(K kernel, int threads, size_t smem) {
  int dev = 0, sms = 0, per_sm = 0;
  if (cudaGetDevice(&dev) != cudaSuccess) return 0;
  if (cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev) != cudaSuccess) return 0;
  if (cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, kernel, threads, smem) != cudaSuccess) return 0;
  return sms * (per_sm > 0 ? per_sm : 1);
}

// ------------------------------------------------------------------------------------- launchers
// Each returns a cudaError_t from the launch.
cudaError_t launch_init(const PoolDev& p, cudaStream_t s);
cudaError_t launch_set_requests(const PoolDev& p, const int32_t* req, const int32_t* len, int n, int mode,
                                cudaStream_t s);
cudaError_t launch_clear_status(const PoolDev& p, cudaStream_t s);
cudaError_t launch_classify_decode(const PoolDev& p, const float* sig, dkv_decision_t* dec, int max_len, cudaStream_t s);
cudaError_t launch_classify_prefill(const PoolDev& p, int n, const float* sig, int64_t sig_stride, uint8_t* cls,
                                    int max_len, cudaStream_t s);
cudaError_t launch_compact_alloc(const PoolDev& p, const dkv_decision_t* dec, int phase, cudaStream_t s,
                                 bool alloc = true, bool defer_recycle = false);
cudaError_t launch_recycle(const PoolDev& p, const int32_t* req, int n, cudaStream_t s);
cudaError_t launch_attend(const PoolDev& p, const uint16_t* q, float* out, float* probs, int TS, cudaStream_t s);
size_t attend_smem_bytes(const PoolDev& p, int TS);
size_t attend_long_smem_bytes(const PoolDev& p);
cudaError_t launch_attend_tc(const PoolDev& p, const uint16_t* q, float* out, float* probs, int active_units, int max_len,
                             cudaStream_t s);
constexpr int kAuditResults = 8;
cudaError_t launch_audit(const PoolDev& p, uint32_t* hist, int64_t* res, cudaStream_t s);
size_t attend_tc_smem_bytes(const PoolDev& p);
bool attend_tc_supported(const PoolDev& p);
cudaError_t launch_prefill_conservative(const PoolDev& p, cudaStream_t s);
// units [u0, u1) (u1 < 0: all U)
cudaError_t launch_quant_decode(const PoolDev& p, const dkv_decision_t* dec, const uint16_t* k, const uint16_t* v,
                                const float* sig, cudaStream_t s, int u0 = 0, int u1 = -1);
cudaError_t launch_quant_prefill(const PoolDev& p, int n, const uint16_t* k, const uint16_t* v, int64_t kv_stride,
                                 const float* sig, int64_t sig_stride, int max_len, cudaStream_t s);
int compact_max_coresident(int tile_units);

}  // namespace dkv
