// k_classify_decode.cu — generation-phase planning (a1-a2; "each attention head independently
// determines its memory allocation requirements ... perfectly parallelizable").
//
// One warp per unit.  Algorithm 1: the class of t_c from the thresholds alpha/N, then the
// victim t_v = lexicographic (score, position) argmin over the section t_c joins (Q6, Q7).  The section's
// page IDs are staged in shared memory with one coalesced pass over its table row, then each lane issues
// kCV 16-B score loads (4 slots each) at once, so a unit costs two dependent memory round trips.  The scan
// keeps a running unsigned minimum (stored scores are canonical non-negative floats, so bit order is float
// order) with a tiny update path; whenever the minimum score may be shared by several slots, an exact pass
// re-reads the section (batched, with the positions of the vectors holding the minimum) and breaks the tie on
// positions (oldest wins).
#include <stdlib.h>

#include "dkv_internal.cuh"

namespace dkv {

#ifndef DKV_CD_WARPS
#define DKV_CD_WARPS 4
#endif
#ifndef DKV_CD_SPEC
#define DKV_CD_SPEC 1      // u-addressed loads (status, section minima, first table entries) in one round trip
#endif
#ifndef DKV_CD_MINB
#define DKV_CD_MINB 10     // 10 CTAs (40 warps) per SM: 48 registers, a few spilled
#endif
#ifndef DKV_CD_PREFETCH
#define DKV_CD_PREFETCH 0  // L2 prefetch of what dkv_quant_write(DECODE) reads: t_c's window rows, the victim's record
#endif
#ifndef DKV_CD_KCV
#define DKV_CD_KCV 8
#endif
#ifndef DKV_CD_KCV_LONG
#define DKV_CD_KCV_LONG 8   // the same for the full-register form (measured: 16 and 24 lose, profiles/r2t_classify_long_ab.log)
#endif
constexpr int kCDWarps = DKV_CD_WARPS;     // units (warps) per CTA
constexpr int kCV = DKV_CD_KCV;            // 16-B score vectors per lane per batch (1024 slots per batch)
constexpr int kXV = 4;                     // the same for the exact (tie-breaking) pass, which also holds positions

// Build knobs, measured by tools/classify_ab.sh at the Llama-3-8B config (classify scan µs, two runs each):
// baseline 44.5; DKV_CD_64B 43.6; DKV_CD_SPEC 42.8; SPEC + 64B 42.4; SPEC + MINB 10 40.8; kCV 16 59.8;
// kCV 4 45.2; 8 warps per CTA 49.6 — the scan is latency-bound, so fewer dependent round trips and more
// resident warps win, and more loads in flight per warp (at the cost of occupancy) lose.
#ifndef DKV_CD_64B
#define DKV_CD_64B 1
#endif
#if DKV_CD_64B      // limit the L2 fetch of a score load to the 64-B segment it touches
#define CD_LD ld_nc_v4_64
#else
#define CD_LD ld_nc_v4
#endif

// TOP: the pool has the NEXT-4 FP16 tier (compiled out otherwise: its branches cost registers at the 10-CTA budget)
template <int MINB, bool TOP>
__global__ void __launch_bounds__(kCDWarps * 32, MINB)
classify_decode_kernel(PoolDev p, const float* __restrict__ cand_sig, dkv_decision_t* __restrict__ dec) {
  extern __shared__ int32_t s_pid_all[];                         // [kCDWarps][L] page IDs of the scanned sections
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int u = blockIdx.x * kCDWarps + warp;
  if (u >= p.U) return;                                          // whole warps exit together
  pdl_wait();                                                    // (PDL) the previous quant_write's writes
  pdl_trigger();
  const int LP = TOP && p.Lt > p.L ? p.Lt : p.L;                 // page IDs a scanned section can have
  int32_t* s_pid = s_pid_all + warp * LP;
#if DKV_CD_SPEC
  // One round trip for everything u alone addresses: the sticky status (read through L1 — 16k warps reading
  // the word at one L2 slice queue there; a status set during this call is seen or not, as before), the
  // section minima of dkv_attend, and the first table entries at both ends of the row (64 high pages, 32 low
  // pages: the first scan batch's page IDs whichever class t_c takes)
  const int32_t* row = p.table + (size_t)u * p.L;
  const int32_t sm_w = lane < 8 ? __ldg(p.secmin + 8 * (size_t)u + lane) : 0;
  const int32_t sp_h0 = lane < p.L ? __ldg(row + lane) : 0;
  const int32_t sp_h1 = lane + 32 < p.L ? __ldg(row + lane + 32) : 0;
  const int32_t sp_l0 = lane < p.L ? __ldg(row + p.L - 1 - lane) : 0;
  const bool dead = __ldg(&p.ctrl->status) != 0;
  const unsigned long long tk = __ldg(&p.ctrl->ticket);         // the following compact_alloc's call counter
#else
  const bool dead = ld_volatile(&p.ctrl->status) != 0;
  const unsigned long long tk = *(volatile const unsigned long long*)&p.ctrl->ticket;
#endif
  // sticky error at entry (Q36: one snapshot per call; classify kernels never write `status`): the unit's
  // decision is the empty one, nothing else happens
  if (dead) {
    if (lane == 0) {
      reinterpret_cast<int4*>(dec)[u] = make_int4(0, -1, -1, -1);
      p.qpid[u] = make_int4(-1, -1, 0, 0);
    }
    return;
  }
  if (u < (p.U + 31) / 32 && lane == 0) {
    // warm L2 with the ring window the following dkv_compact_alloc grants from: [start, start + U) holds
    // every page a decode step can demand (one per unit); one 128-B line per warp
    const int64_t idx = (ld_volatile(&p.ctrl->start) + 32 * (int64_t)u) % p.P;
    asm volatile("prefetch.global.L2 [%0];" ::"l"(p.ring + idx));
  }
  const int r = u / p.LyH;
  uint8_t tc_class = DKV_CLS_NONE, v_action = DKV_V_NONE, grow = DKV_GROW_NONE, demand = 0;
  int v_slot = -1, tc_slot = -1, v_dst_slot = -1;
  bool scan = false;
  int cls = DKV_CLS_NONE, n = 0, nh = 0, nl = 0;
  float sc = 0.0f, th = 0.0f, tl = 0.0f, tt = 0.0f;
  int nlive = 0;                                                 // N if the request is ACTIVE (for quant_write)
  int frp = 0;                                                   // pages a freed request's unit returns (a3)
  {
    const int8_t st = p.req_state[r];
    const int N = p.seq_len[r] + 1;                              // Q3: includes this step's token
    nlive = st == DKV_REQ_ACTIVE ? N : 0;
    // t_c's significance: given, or (NEXT-2, cand_sig NULL) the running mean kept for its window slot
    const float s_in = cand_sig ? cand_sig[u]
                                : (p.W > 0 && N - 1 - p.W >= 0 ? p.win_sig[(size_t)u * p.W + (N - 1 - p.W) % p.W] : 0.0f);
    const int nh_in = p.n_h[u], nl_in = p.n_l[u];
    const int nt_in = TOP ? p.n_t[u] : 0;
    if (st == DKV_REQ_PENDING_FREE)
      frp = (TOP ? (nt_in + p.Ct - 1) / p.Ct : 0) + (nh_in + p.Ch - 1) / p.Ch + (nl_in + p.Cl - 1) / p.Cl;
    const int pc = N - 1 - p.W;                                  // t_c = earliest window token
    if (st == DKV_REQ_ACTIVE && pc >= 0) {
#if DKV_CD_PREFETCH
      // warm L2 with t_c's window rows (slot p_c mod W), which the following dkv_quant_write reads first
      const int lines = (p.d * 2 + 127) >> 7;
      if (p.W > 0 && lane < 2 * lines) {
        const __half* wrow = (lane < lines ? p.win_k : p.win_v) + ((size_t)u * p.W + (N - 1) % p.W) * p.d;
        asm volatile("prefetch.global.L2 [%0];" ::"l"(reinterpret_cast<const uint8_t*>(wrow) + 128 * (lane % lines)));
      }
#endif
      if (!finite_f(s_in) || s_in < 0.0f) {
        if (lane == 0) set_pending(p.ctrl, DKV_ERR_NONFINITE);   // Q36: merged by compact_alloc
      } else {
        sc = canon_zero(s_in);
        th = __fdiv_rn(unit_alpha_h(p, u), (float)N);            // alpha_h / N (per head: Q35)
        tl = __fdiv_rn(unit_alpha_l(p, u), (float)N);            // alpha_l / N
        cls = sc >= th ? DKV_CLS_HIGH : (sc >= tl ? DKV_CLS_LOW : DKV_CLS_PRUNED);
        if (TOP) {                                               // NEXT-4 (Q38): the FP16 tier above High
          tt = __fdiv_rn(p.alpha_t, (float)N);
          if (sc >= tt) cls = DKV_CLS_TOP;
        }
        tc_class = (uint8_t)cls;
        if (cls != DKV_CLS_PRUNED) {
          nh = nh_in;
          nl = nl_in;
          n = (TOP && cls == DKV_CLS_TOP) ? nt_in : ((cls == DKV_CLS_HIGH) ? nh : nl);
          scan = true;
        }
      }
    }
  }
  int vs = -1;                                                   // victim slot, -1 = t_c itself
  uint32_t vb = 0xFFFFFFFFu;
  // NEXT-2: dkv_attend recorded each section's (significance, position) minimum after its update and no
  // section changed since (quant_write clears the flag): the victim needs no scan
#if DKV_CD_SPEC
  const bool fused = scan && n > 0 && cls != DKV_CLS_TOP && __shfl_sync(kFull, sm_w, 6) == 1;
  if (fused) {
    const int b = cls == DKV_CLS_HIGH ? 0 : 3;
    vb = (uint32_t)__shfl_sync(kFull, sm_w, b);
    vs = __shfl_sync(kFull, sm_w, b + 2);
  } else if
#else
  const bool fused = scan && n > 0 && cls != DKV_CLS_TOP && p.secmin[8 * (size_t)u + 6] == 1;
  if (fused) {
    const int b = cls == DKV_CLS_HIGH ? 0 : 3;
    vb = (uint32_t)p.secmin[8 * (size_t)u + b];
    vs = p.secmin[8 * (size_t)u + b + 2];
  } else if
#endif
  (scan && n > 0) {                                    // warp-uniform
    const int C = (TOP && cls == DKV_CLS_TOP) ? p.gt.C : (cls == DKV_CLS_HIGH ? p.g[1].C : p.g[2].C);
    const int off_score = (TOP && cls == DKV_CLS_TOP) ? p.gt.off_score : (cls == DKV_CLS_HIGH ? p.g[1].off_score : p.g[2].off_score);
    const bool pow2 = (C & (C - 1)) == 0;
    const int csh = __popc(C - 1);
    const int npages = (n + C - 1) / C;
#if DKV_CD_SPEC
    // the first scan batch's pages (1024 slots: 64 high / 32 low pages) come from the first round trip's
    // registers; the rest of the row is copied into shared memory asynchronously (cp.async) and waited for only
    // before the second batch, so that batch 1's score loads do not wait on it
    for (int k = lane; k < npages; k += 32) {
      if (TOP && cls == DKV_CLS_TOP) {
        s_pid[k] = __ldg(p.ttable + (size_t)u * p.Lt + k);     // NEXT-4 (Q41)
      } else if (cls == DKV_CLS_HIGH) {
        if (k < 64) s_pid[k] = k < 32 ? sp_h0 : sp_h1;
        else asm volatile("cp.async.ca.shared.global [%0], [%1], 4;" ::"r"(smem_u32(s_pid + k)), "l"(row + k) : "memory");
      } else {
        if (k < 32) s_pid[k] = sp_l0;
        else asm volatile("cp.async.ca.shared.global [%0], [%1], 4;" ::"r"(smem_u32(s_pid + k)), "l"(row + p.L - 1 - k)
                          : "memory");
      }
    }
    cp_async_commit();
#else
    const int32_t* row = p.table + (size_t)u * p.L;
    for (int k = lane; k < npages; k += 32)
      s_pid[k] = (TOP && cls == DKV_CLS_TOP) ? __ldg(p.ttable + (size_t)u * p.Lt + k) : __ldg(row + (cls == DKV_CLS_HIGH ? k : p.L - 1 - k));
#endif
    __syncwarp();
    const uint8_t* base_sc = p.pages + off_score;
    auto vec_addr = [&](int s0) {
      const int pg = pow2 ? (s0 >> csh) : s0 / C;
      const int ix = pow2 ? (s0 & (C - 1)) : s0 % C;
      return base_sc + (size_t)s_pid[pg] * (size_t)p.page_bytes + 4 * ix;
    };
    uint32_t best = 0xFFFFFFFFu;
    int bslot = -1;
    bool tie = false;                                            // best may be held by more than one slot
    // long-section / tie-heavy form (the full-register instantiation): which of this lane's vectors (by
    // iteration index, 128 per lane at most) hold its running minimum, so that the tie-breaking pass reloads
    // only those — one round trip instead of a second pass over the whole section
    constexpr bool kMask = MINB == 1;
    constexpr int KV = MINB == 1 ? DKV_CD_KCV_LONG : kCV;        // score vectors per lane per batch
    uint64_t tlo = 0, thi = 0;
    bool ovf = false;
    int it0 = 0;
    for (int base = 0; base < n; base += 128 * KV, it0 += KV) {
      if (base == 128 * KV) {                                    // batch 2 reads the asynchronously copied IDs
        cp_async_wait<0>();
        __syncwarp();
      }
      uint4 v[KV];
#pragma unroll
      for (int j = 0; j < KV; j++) {
        const int s0 = base + j * 128 + 4 * lane;
        v[j] = make_uint4(0xFFFFFFFFu, 0xFFFFFFFFu, 0xFFFFFFFFu, 0xFFFFFFFFu);
        if (s0 < n) v[j] = CD_LD(vec_addr(s0));
      }
#pragma unroll
      for (int j = 0; j < KV; j++) {
        const int s0 = base + j * 128 + 4 * lane;
        uint32_t a = v[j].x, b = v[j].y, c = v[j].z, d = v[j].w;
        if (s0 + 3 >= n) {                                       // tail vector: mask slots >= n
          a = s0 < n ? a : 0xFFFFFFFFu;
          b = s0 + 1 < n ? b : 0xFFFFFFFFu;
          c = s0 + 2 < n ? c : 0xFFFFFFFFu;
          d = 0xFFFFFFFFu;
        }
        const uint32_t m4 = min(min(a, b), min(c, d));
        if (m4 <= best && m4 != 0xFFFFFFFFu) {                   // rare after the first steps
          if constexpr (kMask) {
            const int it = it0 + j;
            const uint64_t blo = it < 64 ? 1ull << (it & 63) : 0ull, bhi = it >= 64 && it < 128 ? 1ull << (it & 63) : 0ull;
            ovf = ovf || it >= 128;
            if (m4 == best) { tlo |= blo; thi |= bhi; }
            else { tlo = blo; thi = bhi; }
          }
          if (m4 == best) {
            tie = true;
          } else {
            best = m4;
            bslot = s0 + (a == m4 ? 0 : (b == m4 ? 1 : (c == m4 ? 2 : 3)));
            tie = ((a == m4) + (b == m4) + (c == m4) + (d == m4)) > 1;
          }
        }
      }
    }
    cp_async_wait<0>();                                          // every page ID is in shared memory
    __syncwarp();
    const uint32_t m = __reduce_min_sync(kFull, best);
    const unsigned holders = __ballot_sync(kFull, best == m);
    const bool any_tie = __any_sync(kFull, best == m && tie);
    if (__popc(holders) == 1 && !any_tie) {
      vs = __shfl_sync(kFull, bslot, __ffs(holders) - 1);
    } else if (kMask && !__any_sync(kFull, ovf)) {
      // tie-breaking from the recorded vectors: each holder lane reloads its vectors that hold m (scores and
      // the same 4 slots' positions, 4 vectors in flight at a time); the oldest position wins (Q6)
      const int off_pos = (TOP && cls == DKV_CLS_TOP) ? p.gt.off_pos : (cls == DKV_CLS_HIGH ? p.g[1].off_pos : p.g[2].off_pos);
      uint64_t mlo = best == m ? tlo : 0ull, mhi = best == m ? thi : 0ull;
      int32_t bp = 0x7FFFFFFF;
      int bs = -1;
      while (__any_sync(kFull, (mlo | mhi) != 0ull)) {
        int s0k[4];
        uint4 v[4], q[4];
#pragma unroll
        for (int k = 0; k < 4; k++) {
          int it = -1;
          if (mlo) { it = __ffsll((long long)mlo) - 1; mlo &= mlo - 1; }
          else if (mhi) { it = 64 + __ffsll((long long)mhi) - 1; mhi &= mhi - 1; }
          s0k[k] = it < 0 ? -1 : (it / KV) * (128 * KV) + (it % KV) * 128 + 4 * lane;
        }
#pragma unroll
        for (int k = 0; k < 4; k++)
          if (s0k[k] >= 0) { v[k] = CD_LD(vec_addr(s0k[k])); q[k] = ld_nc_v4(vec_addr(s0k[k]) - off_score + off_pos); }
#pragma unroll
        for (int k = 0; k < 4; k++) {
          if (s0k[k] < 0) continue;
          const uint32_t e4[4] = {v[k].x, v[k].y, v[k].z, v[k].w};
          const int32_t p4[4] = {(int32_t)q[k].x, (int32_t)q[k].y, (int32_t)q[k].z, (int32_t)q[k].w};
#pragma unroll
          for (int e = 0; e < 4; e++)
            if (s0k[k] + e < n && e4[e] == m && p4[e] < bp) { bp = p4[e]; bs = s0k[k] + e; }
        }
      }
      const uint32_t mp = __reduce_min_sync(kFull, (uint32_t)bp);
      vs = __shfl_sync(kFull, bs, __ffs(__ballot_sync(kFull, (uint32_t)bp == mp && bs >= 0)) - 1);
    } else {
      // exact pass: among the slots scoring m, the oldest position wins (Q6).  Batched: kXV score vectors
      // in flight per lane, then one 16-B position vector (the same 4 slots' positions, contiguous in the
      // page) for every score vector holding m — a section whose minimum is shared by hundreds of slots
      // (exact zeros when nothing is pruned) costs two round trips per batch, not one per tied slot
      const int off_pos = (TOP && cls == DKV_CLS_TOP) ? p.gt.off_pos : (cls == DKV_CLS_HIGH ? p.g[1].off_pos : p.g[2].off_pos);
      int32_t bp = 0x7FFFFFFF;
      int bs = -1;
      for (int base = 0; base < n; base += 128 * kXV) {
        uint4 v[kXV], q[kXV];
#pragma unroll
        for (int j = 0; j < kXV; j++) {
          const int s0 = base + j * 128 + 4 * lane;
          v[j] = make_uint4(0xFFFFFFFFu, 0xFFFFFFFFu, 0xFFFFFFFFu, 0xFFFFFFFFu);
          if (s0 < n) v[j] = CD_LD(vec_addr(s0));
        }
#pragma unroll
        for (int j = 0; j < kXV; j++) {
          const int s0 = base + j * 128 + 4 * lane;
          if (v[j].x == m || v[j].y == m || v[j].z == m || v[j].w == m)
            q[j] = ld_nc_v4(vec_addr(s0) - off_score + off_pos);
        }
#pragma unroll
        for (int j = 0; j < kXV; j++) {
          const int s0 = base + j * 128 + 4 * lane;
          const uint32_t e4[4] = {v[j].x, v[j].y, v[j].z, v[j].w};
          const int32_t p4[4] = {(int32_t)q[j].x, (int32_t)q[j].y, (int32_t)q[j].z, (int32_t)q[j].w};
#pragma unroll
          for (int e = 0; e < 4; e++)
            if (s0 + e < n && e4[e] == m && p4[e] < bp) { bp = p4[e]; bs = s0 + e; }
        }
      }
      const uint32_t mp = __reduce_min_sync(kFull, (uint32_t)bp);
      vs = __shfl_sync(kFull, bs, __ffs(__ballot_sync(kFull, (uint32_t)bp == mp && bs >= 0)) - 1);
    }
    vb = m;
  }
  if (lane != 0) return;
  if (scan) {
    // t_c has the largest position, so a stored token wins every score tie with it
    if (vs >= 0 && !(vb <= __float_as_uint(sc))) vs = -1;
    const float sv = __uint_as_float(vb);
    if (TOP && cls == DKV_CLS_TOP) {                                      // NEXT-4 (Q39): Algorithm 1 one level up
      if (vs < 0 || sv >= tt) {                                  // t_v stays in KV_t
        v_action = DKV_V_KEEP; grow = DKV_GROW_TOP; demand = (n % p.Ct == 0); tc_slot = n;
      } else if (sv >= th) {                                     // t_v moves to KV_h
        v_action = DKV_V_DOWN; grow = DKV_GROW_HIGH; demand = (nh % p.Ch == 0);
        v_slot = vs; tc_slot = vs; v_dst_slot = nh;
      } else if (sv >= tl) {                                     // t_v moves to KV_l
        v_action = DKV_V_DOWN; grow = DKV_GROW_LOW; demand = (nl % p.Cl == 0);
        v_slot = vs; tc_slot = vs; v_dst_slot = nl;
      } else {                                                   // prune t_v
        v_action = DKV_V_PRUNE; v_slot = vs; tc_slot = vs;
      }
    } else if (cls == DKV_CLS_HIGH) {
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
  // the following dkv_compact_alloc's tile sums (demand, freed pages per scan tile), by the parity of its call
  // counter: with them it needs no look-back across tiles (k_compact.cu)
  {
    if (demand | frp) {                                          // tile_units is a power of two
      uint32_t* ts = p.tsum + 2 * ((size_t)(tk & 1ull) * p.num_tiles + (u >> (__ffs(p.tile_units) - 1)));
      if (demand) atomicAdd(ts, 1u);
      if (frp) atomicAdd(ts + 1, (uint32_t)frp);
    }
    if (u == 0) p.ctrl->tsum_ticket = tk;
  }
  // The page IDs dkv_quant_write(DECODE) will touch, so that it reads no table: t_c's page (which is also the
  // victim's KV_h page when the victim is downgraded, since t_c takes its slot, Q8) and the KV_l page a
  // downgraded victim moves to.  A page the growing section receives this step is not known yet: -1 here,
  // written by dkv_compact_alloc when it grants it.  The scanned section's IDs are in shared memory already.
  // The record also carries the request length (0: not ACTIVE), so quant_write reads no request state.
  if (!scan) p.qpid[u] = make_int4(-1, -1, nlive, 0);
  if (scan) {
    const bool hi = cls == DKV_CLS_HIGH, top = TOP && cls == DKV_CLS_TOP;
    const int C = top ? p.Ct : (hi ? p.Ch : p.Cl);
    const int32_t* trow = p.table + (size_t)u * p.L;
    const bool have = n > 0 && !fused;                          // s_pid holds the section's pages
    int pa = -1, pb = -1;
    if (!(v_action == DKV_V_KEEP && demand)) {
      const int k = tc_slot / C;
      pa = have ? s_pid[k] : (top ? __ldg(p.ttable + (size_t)u * p.Lt + k) : __ldg(trow + (hi ? k : p.L - 1 - k)));
    }
    if (v_action == DKV_V_DOWN && !demand)                      // the destination section's tail page
      pb = grow == DKV_GROW_HIGH ? __ldg(trow + nh / p.Ch) : __ldg(trow + p.L - 1 - nl / p.Cl);
    p.qpid[u] = make_int4(pa, pb, nlive, 0);
#if DKV_CD_PREFETCH
    if (v_action == DKV_V_DOWN) {                                // warm L2 with the victim's record (read by quant_write)
      const ClassGeom g = top ? p.gt : p.g[1];
      const uint8_t* pg = p.pages + (size_t)pa * (size_t)p.page_bytes;
      const int is = vs - (vs / C) * C;
      for (int o = 0; o < g.k_row; o += 128) asm volatile("prefetch.global.L2 [%0];" ::"l"(pg + g.off_k + is * g.k_row + o));
      for (int o = 0; o < g.v_row; o += 128) asm volatile("prefetch.global.L2 [%0];" ::"l"(pg + g.off_v + is * g.v_row + o));
      if (!top) {
        asm volatile("prefetch.global.L2 [%0];" ::"l"(pg + g.off_kmeta + 4 * is));
        asm volatile("prefetch.global.L2 [%0];" ::"l"(pg + g.off_vmeta + 4 * is));
      }
      asm volatile("prefetch.global.L2 [%0];" ::"l"(pg + g.off_score + 4 * is));
      asm volatile("prefetch.global.L2 [%0];" ::"l"(pg + g.off_pos + 4 * is));
    }
#endif
  }
}

#ifndef DKV_CD_LONG_LEN
#define DKV_CD_LONG_LEN 12288   // longest active request above which the full-register instantiation runs
#endif

template <int MINB, bool TOP>
static cudaError_t launch_cd_t(const PoolDev& p, const float* sig, dkv_decision_t* dec, cudaStream_t s) {
  const size_t smem = 4 * (size_t)(TOP && p.Lt > p.L ? p.Lt : p.L) * kCDWarps;
  if (smem > 48 * 1024) {
    cudaError_t e = cudaFuncSetAttribute(classify_decode_kernel<MINB, TOP>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    if (e != cudaSuccess) return e;
  }
  return launch_ex(classify_decode_kernel<MINB, TOP>, dim3((p.U + kCDWarps - 1) / kCDWarps), dim3(kCDWarps * 32), smem, s,
                   p.pdl != 0, p, sig, dec);
}

template <int MINB>
static cudaError_t launch_cd(const PoolDev& p, const float* sig, dkv_decision_t* dec, cudaStream_t s) {
  return p.top ? launch_cd_t<MINB, true>(p, sig, dec, s) : launch_cd_t<MINB, false>(p, sig, dec, s);
}

// max_len: the longest ACTIVE request (host mirror).  Long sections run the instantiation with the full
// register budget: their scans take many batches and, when the minimum is shared, the exact pass, which
// spills at the 10-CTA budget (measured: profiles/r1j_classify_long_ab.log)
cudaError_t launch_classify_decode(const PoolDev& p, const float* sig, dkv_decision_t* dec, int max_len, cudaStream_t s) {
  // the full-register form also when nothing is pruned (alpha_l = 0): the low sections then hold many exact-zero
  // significances, a shared minimum, and that form breaks the tie from the vectors it recorded
  if (max_len > DKV_CD_LONG_LEN || (p.alpha_l == 0.0f && !p.use_head_alpha)) return launch_cd<1>(p, sig, dec, s);
  return launch_cd<DKV_CD_MINB>(p, sig, dec, s);
}

}  // namespace dkv
