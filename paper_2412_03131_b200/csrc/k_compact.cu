// k_compact.cu — coordination: recycle (stream compaction into the circular free list) + allocation
// (exclusive scan of per-head demand, all-or-nothing grant, bidirectional table write) in ONE kernel.
//
// "after each head determines the number of pages to be allocated or freed, a parallel prefix
// sum operation computes a unique offset for each head relative to the start or end pointer ... each head
// concurrently retrieves its new page IDs from its designated region in the list, with the start pointer
// incremented by the cumulative number of pages required ... for memory recycling, each head writes freed
// page IDs to its designated region, with the end pointer incremented by the total number of pages
// released."
//
// One CTA = one tile of `tile_units` consecutive units (one thread per unit).  Both scans (demand, freed
// pages) run in a single pass: warp ballot/popc (0/1 decode demand) or shuffle scans, a shared-memory
// scan of warp totals, then a decoupled look-back across tiles on one 64-bit status word per tile
// {tag:6 | flag:2 | freed:28 | demand:28} published with st.release.gpu / read with ld.acquire.gpu; tile
// order comes from a ticket counter and the epoch tag is the ticket quotient, so status words never need
// resetting.  Recycled IDs are written right after the look-back.  All-or-nothing allocation (Q15) needs
// the grid-wide demand before any grant, and grants may read ring slots recycled by other tiles in this
// call (Q14), so the kernel then crosses one software grid barrier (arrival counter; the launch is
// cooperative, which guarantees co-residency) and grants.
#include <stdlib.h>

#include "dkv_internal.cuh"

namespace dkv {

constexpr uint64_t kFlagAgg = 1, kFlagPre = 2;
constexpr uint32_t kValMask = (1u << 28) - 1u;

__device__ __forceinline__ unsigned long long pack_status(uint32_t tag, uint64_t flag, uint32_t fr, uint32_t dem) {
  return ((unsigned long long)(tag & 63u) << 58) | (flag << 56) | ((unsigned long long)(fr & kValMask) << 28) |
         (unsigned long long)(dem & kValMask);
}
__device__ __forceinline__ uint32_t st_tag(unsigned long long w) { return (uint32_t)(w >> 58); }
__device__ __forceinline__ uint32_t st_flag(unsigned long long w) { return (uint32_t)(w >> 56) & 3u; }
__device__ __forceinline__ uint32_t st_fr(unsigned long long w) { return (uint32_t)(w >> 28) & kValMask; }
__device__ __forceinline__ uint32_t st_dem(unsigned long long w) { return (uint32_t)w & kValMask; }

__device__ __forceinline__ uint32_t warp_incl_scan(uint32_t v, int lane) {
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    uint32_t y = __shfl_up_sync(kFull, v, o);
    if (lane >= o) v += y;
  }
  return v;
}

#ifndef DKV_CA_TRACE
#define DKV_CA_TRACE 0      // debug builds: globaltimer marks of the last tile's phases into rec[0..11] (tools/ca_trace.py)
#endif
__device__ __forceinline__ void ca_mark(const PoolDev& p, int idx) {
#if DKV_CA_TRACE
  if (threadIdx.x == 0 && blockIdx.x == gridDim.x - 1) {
    unsigned long long t;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
    reinterpret_cast<unsigned long long*>(p.rec)[idx] = t;
  }
#else
  (void)p; (void)idx;
#endif
}

template <int TU>
__global__ void __launch_bounds__(TU) compact_alloc_kernel(PoolDev p, const dkv_decision_t* __restrict__ dec, int phase, int alloc, int defer_rec) {
  constexpr int NW = TU / 32;
  __shared__ unsigned long long s_epoch;
  __shared__ int64_t s_start0, s_free0, s_D, s_F;
  __shared__ int s_status0;
  __shared__ unsigned long long s_tst;
  __shared__ uint32_t s_wdem[NW], s_wfr[NW];
  __shared__ uint32_t s_exdem, s_exfr, s_incdem, s_incfr;

  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  Ctrl* ctrl = p.ctrl;
  // The launch is cooperative (all tiles co-resident), so tiles take their index from blockIdx and the
  // look-back always waits on running or finished tiles.  The call's epoch (status-word tag and barrier
  // target) is ctrl->ticket, which only tile 0 advances, after the barrier every tile crossed having read it.
  const int tile = blockIdx.x;
  // per-unit loads do not depend on the control block: issue them before the first barrier; the request
  // state and counts are not written by dkv_classify, so they may be read before the PDL wait
  const int u = tile * TU + tid;
  ca_mark(p, 0);
  int st = -1, r = 0, nh = 0, nl = 0, nt = 0;
  uint32_t dword = 0;
  int pfh = 0, pfl = 0, pft = 0;
  if (u < p.U) {
    r = u / p.LyH;
    st = p.req_state[r];
    nh = p.n_h[u];
    nl = p.n_l[u];
    if (p.top) nt = p.n_t[u];                          // NEXT-4 TOP section
  }
  pdl_wait();                                        // (PDL) the decisions and classify's pending error
  pdl_trigger();
  if (tid == 0) s_epoch = *(volatile unsigned long long*)&ctrl->ticket;
  if (tid == 32) s_start0 = ld_volatile(&ctrl->start);
  if (tid == 64) s_free0 = ld_volatile(&ctrl->free);
  if (tid == 96) {                                   // entry status (Q36): sticky status, else classify's error
    const int a = ld_volatile(&ctrl->status);
    s_status0 = a != 0 ? a : ld_volatile(&ctrl->pending);
  }
  if (tid == 128) s_tst = *(volatile unsigned long long*)&ctrl->tsum_ticket;
  // decode tile sums left by dkv_classify for both ticket parities (the parity is known after the barrier)
  uint2 ts0 = make_uint2(0u, 0u), ts1 = ts0;
  if (phase == DKV_PHASE_DECODE && lane < p.num_tiles) {      // every warp (lane = tile)
    ts0 = __ldcg(reinterpret_cast<const uint2*>(p.tsum) + lane);
    ts1 = __ldcg(reinterpret_cast<const uint2*>(p.tsum) + p.num_tiles + lane);
  }
  if (u < p.U) {
    if (phase == DKV_PHASE_DECODE) dword = __ldg(reinterpret_cast<const uint32_t*>(dec + u));
    else { pfh = p.pf_nh[u]; pfl = p.pf_nl[u]; if (p.top) pft = p.pf_nt[u]; }
  }
  // the request state has arrived in every thread before the barrier, so that the arrival count below orders
  // every read of it before a rewrite by another tile
  asm volatile("" ::"r"((int)st));
  __syncthreads();
  ca_mark(p, 1);
  const unsigned long long epoch = s_epoch;
  const uint32_t tag = (uint32_t)(epoch & 63ull);
  const int64_t start0 = s_start0, free0 = s_free0;
  const int status0 = s_status0;
  const int P = p.P, L = p.L;
  // every tile has read its entry state (ctrl, request states): counted for the tile that rewrites them
  if (tid == 0) atomicAdd(&ctrl->arrive2, 1ull);
  // this call's tile-sum buffer is tsum[epoch & 1]; the other one is the next classify's: cleared here
  if (tid == 32) reinterpret_cast<uint2*>(p.tsum)[(size_t)((epoch & 1ull) ^ 1ull) * p.num_tiles + tile] = make_uint2(0u, 0u);
  // Tile sums instead of the look-back (decode, no error, the fast path's free region, and sums this step's
  // dkv_classify accumulated for this very call): every tile's exclusive demand / freed offsets follow from
  // the sums directly, with no wait on another tile
  const bool use_ts = phase == DKV_PHASE_DECODE && alloc && status0 == 0 && free0 >= (int64_t)p.U &&
                      s_tst == epoch && p.num_tiles <= 32;

  // ---- per-unit demand and freed pages (planning results)
  int grow = 0;
  uint32_t dem = 0, fr = 0;
  if (u < p.U) {
    const int pt = p.top ? ceil_div(nt, p.Ct) : 0;
    if (st == DKV_REQ_PENDING_FREE) fr = pt + ceil_div(nh, p.Ch) + ceil_div(nl, p.Cl);
    if (status0 == 0) {
      if (phase == DKV_PHASE_DECODE) {
        if (st == DKV_REQ_ACTIVE) {
          dem = dword >> 24;
          grow = (dword >> 16) & 0xFF;
        }
      } else if (st == DKV_REQ_ADMITTING && alloc) {
        dem = ceil_div(pfh, p.Ch) + ceil_div(pfl, p.Cl) + (p.top ? ceil_div(pft, p.Ct) : 0);   // Q43
      }
    }
  }

  // ---- tile-local exclusive scans
  uint32_t inc_dem;
  if (phase == DKV_PHASE_DECODE) {                               // demand is 0/1: ballot + popc
    const unsigned m = __ballot_sync(kFull, dem != 0);
    inc_dem = __popc(m & (0xFFFFFFFFu >> (31 - lane)));
  } else {
    inc_dem = warp_incl_scan(dem, lane);
  }
  const uint32_t inc_fr = warp_incl_scan(fr, lane);
  if (lane == 31) { s_wdem[warp] = inc_dem; s_wfr[warp] = inc_fr; }
  __syncthreads();
  ca_mark(p, 2);
  uint32_t off_dem, off_fr, tile_ex_fr, tile_inc_fr, tile_inc_dem;
  unsigned long long a2_early = 0ull;                            // the finalizer's first look at arrive2
  if (use_ts) {
    // every warp on its own: the warps before it from the shared warp totals, the tiles before it from the
    // tile sums — no warp-0 pass and no further barrier
    const uint2 t = (epoch & 1ull) ? ts1 : ts0;                    // lane = tile
    const uint32_t wd = __reduce_add_sync(kFull, lane < warp ? s_wdem[lane] : 0u);
    const uint32_t wf = __reduce_add_sync(kFull, lane < warp ? s_wfr[lane] : 0u);
    const uint32_t ex_d = __reduce_add_sync(kFull, lane < tile ? t.x : 0u);
    const uint32_t ex_f = __reduce_add_sync(kFull, lane < tile ? t.y : 0u);
    const uint2 mine = make_uint2(__shfl_sync(kFull, t.x, tile & 31), __shfl_sync(kFull, t.y, tile & 31));
    off_dem = ex_d + wd + inc_dem - (dem != 0);
    off_fr = ex_f + wf + inc_fr - fr;
    tile_ex_fr = ex_f; tile_inc_fr = ex_f + mine.y; tile_inc_dem = ex_d + mine.x;
    if (tid == 0 && tile == p.num_tiles - 1) a2_early = *(volatile unsigned long long*)&ctrl->arrive2;   // no stall
  } else {
    if (warp == 0) {
      uint32_t a = lane < NW ? s_wdem[lane] : 0u, b = lane < NW ? s_wfr[lane] : 0u;
      const uint32_t ia = warp_incl_scan(a, lane), ib = warp_incl_scan(b, lane);
      if (lane < NW) { s_wdem[lane] = ia - a; s_wfr[lane] = ib - b; }
      const uint32_t tot_dem = __shfl_sync(kFull, ia, 31), tot_fr = __shfl_sync(kFull, ib, 31);
      // ---- decoupled look-back across tiles (or the tile sums)
      unsigned long long* stat = p.tile_status;
      uint32_t ex_d = 0, ex_f = 0;
      if (use_ts) {
        const uint2 t = (epoch & 1ull) ? ts1 : ts0;                  // lane = tile
        ex_d = __reduce_add_sync(kFull, lane < tile ? t.x : 0u);
        ex_f = __reduce_add_sync(kFull, lane < tile ? t.y : 0u);
      } else if (tile == 0) {
        if (lane == 0) st_release(&stat[0], pack_status(tag, kFlagPre, tot_fr, tot_dem));
      } else {
        if (lane == 0) st_release(&stat[tile], pack_status(tag, kFlagAgg, tot_fr, tot_dem));
        int look = tile - 1;
        while (true) {
          const int idx = look - lane;
          const unsigned long long w = idx >= 0 ? ld_acquire(&stat[idx]) : pack_status(tag, kFlagPre, 0, 0);
          const bool valid = st_tag(w) == tag && st_flag(w) != 0;
          const unsigned vm = __ballot_sync(kFull, valid);
          const unsigned pm = __ballot_sync(kFull, valid && st_flag(w) == kFlagPre);
          if (pm) {
            const int jl = __ffs(pm) - 1;
            const unsigned need = (jl == 31) ? kFull : ((2u << jl) - 1u);
            if ((vm & need) != need) continue;                     // a nearer predecessor not published yet
            ex_d += __reduce_add_sync(kFull, lane <= jl ? st_dem(w) : 0u);
            ex_f += __reduce_add_sync(kFull, lane <= jl ? st_fr(w) : 0u);
            break;
          }
          if (vm == kFull) {
            ex_d += __reduce_add_sync(kFull, st_dem(w));
            ex_f += __reduce_add_sync(kFull, st_fr(w));
            look -= 32;
          }
        }
        if (lane == 0) st_release(&stat[tile], pack_status(tag, kFlagPre, ex_f + tot_fr, ex_d + tot_dem));
      }
      if (lane == 0) { s_exdem = ex_d; s_exfr = ex_f; s_incdem = ex_d + tot_dem; s_incfr = ex_f + tot_fr; }
    }
    __syncthreads();
    off_dem = s_exdem + s_wdem[warp] + inc_dem - (phase == DKV_PHASE_DECODE ? (dem != 0) : dem);
    off_fr = s_exfr + s_wfr[warp] + inc_fr - fr;
    tile_ex_fr = s_exfr; tile_inc_fr = s_incfr; tile_inc_dem = s_incdem;
  }
  ca_mark(p, 3);

  // ---- recycle: freed IDs -> ring[(end + off + k) mod P], canonical slot order (Q13).  The tile's freed
  // slots form one flat list (k = tile-local exclusive scan of the freed counts + slot rank), cut into one
  // contiguous chunk per warp; lane l of a warp takes k = base + 32 j + l (coalesced table reads and ring
  // writes), finds its first unit by binary search and then only walks forward.  kRecDepth loads per lane
  // are in flight before the dependent ring / table stores.  A whole finished request (its units sit in one
  // or two tiles) is copied by every warp of those tiles at once.
  {
    constexpr int kRecDepth = 8;
    __shared__ uint32_t s_loc[TU];                               // tile-local exclusive freed offset
    __shared__ int s_nfr[TU], s_ph[TU], s_pt[TU];
    const uint32_t tile_ex = tile_ex_fr;
    const uint32_t Ft = tile_inc_fr - tile_ex;                   // freed slots in this tile
    // deferred: in the decode fast path (grants never read a slot recycled in this call) the copy is left to
    // the following dkv_quant_write(DECODE) (quant_decode_kernel, over all SMs — here it would run on the one
    // or two CTAs whose tile holds the request); this kernel records each freed unit's offset from the end
    // pointer
    const bool defer = defer_rec && phase == DKV_PHASE_DECODE && status0 == 0 && free0 >= (int64_t)p.U;
    if (defer && fr != 0) {
      p.rec[4 * (size_t)u] = (int32_t)off_fr;
      p.rec[4 * (size_t)u + 1] = ceil_div(nh, p.Ch);
      p.rec[4 * (size_t)u + 3] = p.top ? ceil_div(nt, p.Ct) : 0;
      p.rec[4 * (size_t)u + 2] = (int32_t)fr;                    // the marker (non-zero) last
    }
    if (tid == 0 && tile == 0 && defer_rec) {
      int64_t e0 = start0 + free0;
      ctrl->rec_end0 = e0 >= P ? e0 - P : e0;
      ctrl->rec_deferred = defer ? 1 : 0;
    }
    if (Ft > 0 && !defer) {                                      // tile-uniform
      int64_t ring0 = start0 + free0;                            // end pointer + this tile's offset
      ring0 -= ring0 >= P ? P : 0;
      ring0 += tile_ex;
      s_loc[tid] = off_fr - tile_ex; s_nfr[tid] = (int)fr; s_ph[tid] = ceil_div(nh, p.Ch);
      s_pt[tid] = p.top ? ceil_div(nt, p.Ct) : 0;
      __syncthreads();
      const uint32_t per = ((Ft + NW - 1) / NW + 31) & ~31u;     // per-warp chunk, a multiple of 32
      const uint32_t w0 = (uint32_t)warp * per, w1 = min(w0 + per, Ft);
      int t = 0;
      if (w0 + lane < w1) {                                      // last t with s_loc[t] <= k
        const uint32_t k = w0 + lane;
        int lo = 0, hi = TU;
        while (hi - lo > 1) {
          const int mid = (lo + hi) >> 1;
          if (s_loc[mid] <= k) lo = mid; else hi = mid;
        }
        t = lo;
      }
      for (uint32_t base = w0; base < w1; base += 32 * kRecDepth) {
        int32_t* tix[kRecDepth];                                 // the freed slot (TOP table or bidirectional)
#pragma unroll
        for (int j = 0; j < kRecDepth; j++) {
          const uint32_t k = base + 32 * j + lane;
          tix[j] = nullptr;
          if (k < w1) {
            while (k >= s_loc[t] + (uint32_t)s_nfr[t]) t++;
            // [0, pt) of the TOP table, then [0, ph) and [L - pl, L) of the bidirectional one (Q13, Q41)
            tix[j] = freed_slot(p, tile * TU + t, (int)(k - s_loc[t]), s_pt[t], s_ph[t], s_nfr[t]);
          }
        }
        int32_t pid[kRecDepth];
#pragma unroll
        for (int j = 0; j < kRecDepth; j++) pid[j] = tix[j] != nullptr ? __ldcg(tix[j]) : -1;
#pragma unroll
        for (int j = 0; j < kRecDepth; j++) {
          if (tix[j] != nullptr) {
            int64_t pos = ring0 + base + 32 * j + lane;            // < 3P: two conditional wraps, no division
            pos -= pos >= P ? P : 0;
            pos -= pos >= P ? P : 0;
            p.ring[pos] = pid[j];
            // clear the slot only once its load has returned: a store issued while the same line's load
            // miss is outstanding takes a slow path in L2 (see k_quant_decode.cu)
            int32_t empty = -1;
            asm volatile("" : "+r"(empty) : "r"(pid[j]));
            *tix[j] = empty;
          }
        }
      }
    }
    if (fr != 0) { p.n_h[u] = 0; p.n_l[u] = 0; if (p.top) p.n_t[u] = 0; }
    // a request freed after this step's dkv_classify (the OOM recovery of dkv.h) is no longer live for the
    // following dkv_quant_write, which takes liveness from the unit's qpid record
    if (phase == DKV_PHASE_DECODE && st == DKV_REQ_PENDING_FREE) reinterpret_cast<int32_t*>(p.qpid + u)[2] = 0;
  }

  // ---- Fast path (no grid barrier): with an error pending nothing is granted; in a decode step every unit
  // demands at most one page, so if the free region at entry already holds >= U pages the
  // all-or-nothing check cannot fail and every grant reads a ring slot of that region, never one recycled
  // in this call.  Both conditions are read at entry and identical in every tile.
  const bool fast = (status0 != 0) || (phase == DKV_PHASE_DECODE && free0 >= (int64_t)p.U);
  // the recycle copies above are complete before a grant (or the grid barrier) — a barrier needed only when
  // this tile copied in place: a deferred (decode fast path) recycle writes no ring slot here
  if (!fast || (tile_inc_fr - tile_ex_fr > 0 && !(defer_rec && phase == DKV_PHASE_DECODE && status0 == 0 && free0 >= (int64_t)p.U)))
    __syncthreads();
  bool ok;
  int64_t D = 0, F = 0;
  if (fast) {
    ok = status0 == 0;
  } else {
    // grid barrier: every tile's recycle writes are visible and the totals are known
    if (tid == 0) {
      if (tile == p.num_tiles - 1) { ctrl->total_dem = s_incdem; ctrl->total_fr = s_incfr; }
      const unsigned long long bep = *(volatile unsigned long long*)&ctrl->bar_epoch;
      __threadfence();
      atomicAdd(&ctrl->arrive, 1ull);
      const unsigned long long target = (bep + 1ull) * (unsigned long long)p.num_tiles;
      while (ld_acquire(&ctrl->arrive) < target) __nanosleep(40);
      s_D = ld_volatile(&ctrl->total_dem);
      s_F = ld_volatile(&ctrl->total_fr);
    }
    __syncthreads();
    D = s_D;
    F = s_F;
    ok = (status0 == 0) && (D <= free0 + F);
  }

  // ---- grant + bidirectional table write + counts
  if (ok) {
    if (phase == DKV_PHASE_DECODE) {
      if (dem) {
        const int ph = ceil_div(nh, p.Ch), pl = ceil_div(nl, p.Cl);
        const bool top = grow == DKV_GROW_TOP;                   // NEXT-4: the TOP table, left to right
        if (top ? nt / p.Ct >= p.Lt : ph + pl + 1 > L) {
          set_status(ctrl, DKV_ERR_OVERFLOW);
        } else {
          int32_t* slotp = top ? p.ttable + (size_t)u * p.Lt + nt / p.Ct
                               : p.table + (size_t)u * L + ((grow == DKV_GROW_HIGH) ? nh / p.Ch : L - 1 - nl / p.Cl);
          int64_t pos = start0 + off_dem;                        // < 2P (off_dem < D <= free)
          pos -= pos >= P ? P : 0;
          const int32_t pid = __ldcg(p.ring + pos);
          *slotp = pid;
          // for dkv_quant_write: the granted page is t_c's (KEEP) or the downgraded victim's KV_l page (DOWN)
          reinterpret_cast<int32_t*>(p.qpid + u)[((dword >> 8) & 0xFF) == DKV_V_DOWN ? 1 : 0] = pid;
        }
      }
      if (st == DKV_REQ_ACTIVE) {
        if (grow == DKV_GROW_HIGH) p.n_h[u] = nh + 1;
        if (grow == DKV_GROW_LOW) p.n_l[u] = nl + 1;             // DOWN: n_h unchanged, n_l + 1
        if (grow == DKV_GROW_TOP) p.n_t[u] = nt + 1;
      }
    } else {
      unsigned gm = __ballot_sync(kFull, dem != 0);
      while (gm) {
        const int src = __ffs(gm) - 1;
        gm &= gm - 1;
        const int uu = __shfl_sync(kFull, u, src);
        const uint32_t off = __shfl_sync(kFull, off_dem, src);
        const int nd = (int)__shfl_sync(kFull, dem, src);
        const int ph = ceil_div(p.pf_nh[uu], p.Ch);
        const int pt = p.top ? ceil_div(p.pf_nt[uu], p.Ct) : 0;   // Q43: a unit's TOP pages first
        if (nd - pt > L || pt > p.Lt) {
          if (lane == 0) set_status(ctrl, DKV_ERR_OVERFLOW);
          continue;
        }
        int32_t* row = p.table + (size_t)uu * L;
        int32_t* trow = p.ttable + (size_t)uu * p.Lt;
        for (int k = lane; k < nd; k += 32) {
          const int kk = k - pt;                                 // high left-to-right, low right-to-left
          int32_t* slotp = kk < 0 ? trow + k : row + (kk < ph ? kk : L - 1 - (kk - ph));
          int64_t pos = start0 + off + k;                        // < 2P
          pos -= pos >= P ? P : 0;
          *slotp = __ldcg(p.ring + pos);
        }
      }
      if (st == DKV_REQ_ADMITTING && alloc) {
        p.n_h[u] = p.pf_nh[u]; p.n_l[u] = p.pf_nl[u];
        if (p.top) p.n_t[u] = p.pf_nt[u];
      }
    }
  }
  ca_mark(p, 4);
  // ---- request-level transitions, by the tile owning the request's LAST unit: every other tile holding
  // units of the request is a predecessor, and has read req_state before publishing its look-back status
  // (with the tile sums there is no look-back: the tile waits for every tile's entry reads instead; only a
  // freed request's state is read by other tiles — compact_alloc never reads seq_len)
  const unsigned long long all_read = (epoch + 1ull) * (unsigned long long)p.num_tiles;
  if (u < p.U && u % p.LyH == p.LyH - 1) {
    if (st == DKV_REQ_PENDING_FREE) {
      if (use_ts)
        while (ld_acquire(&ctrl->arrive2) < all_read) __nanosleep(32);
      p.req_state[r] = DKV_REQ_IDLE; p.seq_len[r] = 0; p.prompt_len[r] = 0;
    } else if (ok && phase == DKV_PHASE_DECODE && st == DKV_REQ_ACTIVE) {
      p.seq_len[r] += 1;
    } else if (ok && alloc && phase == DKV_PHASE_PREFILL && st == DKV_REQ_ADMITTING) {
      p.seq_len[r] = p.prompt_len[r];
    }
  }
  // ---- pointers: every tile read them before publishing its look-back status, so the last tile (whose
  // inclusive prefix holds the totals) may write them in the fast path; tile 0 after the barrier otherwise
  if (tid == 0 && (fast ? tile == p.num_tiles - 1 : tile == 0)) {
    if (use_ts && a2_early < all_read)                           // every tile has read the pointers and ticket
      while (ld_acquire(&ctrl->arrive2) < all_read) __nanosleep(32);
    if (fast) { D = tile_inc_dem; F = tile_inc_fr; }
    const int64_t free_avail = free0 + F;
    if (status0 != 0) set_status(ctrl, status0);      // classify's pending error becomes the sticky status
    ctrl->pending = 0;
    if (status0 == 0 && !ok) { set_status(ctrl, DKV_ERR_OOM); ctrl->oom_count += 1; }
    const int64_t ns = ok ? (start0 + D) % P : start0;
    const int64_t nf = ok ? free_avail - D : free_avail;
    ctrl->start = ns;
    ctrl->free = nf;
    ctrl->last_demand = status0 == 0 ? D : 0;
    ctrl->last_freed = F;
    ctrl->ticket = epoch + 1ull;                       // next call's epoch
    if (!fast) ctrl->bar_epoch = ctrl->bar_epoch + 1ull;   // every tile read it before arriving
    p.stats[0] = nf;
    p.stats[1] = -(status0 == 0 ? D : 0);
    p.stats[2] = -((int64_t)P - nf);
    const int fin = ld_volatile(&ctrl->status);
    ctrl->qw_status = fin;                             // entry status of the following dkv_quant_write (Q36)
    p.stats[3] = (int64_t)fin;                         // <= 0: the MIN over GPUs shows any error
  }
  ca_mark(p, 5);
}

template <int TU>
static cudaError_t launch_tu(const PoolDev& p, const dkv_decision_t* dec, int phase, cudaStream_t s, int alloc,
                             int defer) {
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3(p.num_tiles);
  cfg.blockDim = dim3(TU);
  cfg.dynamicSmemBytes = 0;
  cfg.stream = s;
  cudaLaunchAttribute attr[2];
  attr[0].id = cudaLaunchAttributeCooperative;         // always cooperative: the grid barrier needs co-residency
  attr[0].val.cooperative = 1;
  attr[1].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  attr[1].val.programmaticStreamSerializationAllowed = 1;
  cfg.attrs = attr;
  cfg.numAttrs = p.pdl ? 2 : 1;
  return cudaLaunchKernelEx(&cfg, compact_alloc_kernel<TU>, p, dec, phase, alloc, defer);
}

cudaError_t launch_compact_alloc(const PoolDev& p, const dkv_decision_t* dec, int phase, cudaStream_t s, bool alloc,
                                 bool defer_recycle) {
  const int a = alloc ? 1 : 0, d = defer_recycle ? 1 : 0;
  switch (p.tile_units) {
    case 256: return launch_tu<256>(p, dec, phase, s, a, d);
    case 512: return launch_tu<512>(p, dec, phase, s, a, d);
    default: return launch_tu<1024>(p, dec, phase, s, a, d);
  }
}

int compact_max_coresident(int tile_units) {
  int dev = 0, sms = 0, per = 0;
  if (cudaGetDevice(&dev) != cudaSuccess) return 0;
  if (cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev) != cudaSuccess) return 0;
  cudaError_t e;
  switch (tile_units) {
    case 256: e = cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per, compact_alloc_kernel<256>, 256, 0); break;
    case 512: e = cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per, compact_alloc_kernel<512>, 512, 0); break;
    default: e = cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per, compact_alloc_kernel<1024>, 1024, 0); break;
  }
  if (e != cudaSuccess) return 0;
  return per * sms;
}

// ---- deferred recycle copy, eager form (dkv_compact_alloc of a decode step that frees requests): one warp per
// unit of the freed requests (host list), ring[(end0 + off + k) mod P] = table slot k of the unit in canonical
// slot order (Q13), then the slot is cleared and the unit's marker consumed — so the pool state is complete when
// dkv_compact_alloc returns.  Inside a decode-step CUDA graph (no host list) the following quant_write kernel
// does the same copies from the markers instead (k_quant_decode.cu).  A no-op if the scan took the barrier path
// (it then copied in place and left no marker).
constexpr int kRecMaxReq = 64;
struct RecList {
  int32_t n;
  int32_t req[kRecMaxReq];
};

__global__ void __launch_bounds__(256) recycle_kernel(PoolDev p, RecList l) {
  const int lane = threadIdx.x & 31;
  const int wu = (blockIdx.x * 256 + threadIdx.x) >> 5;         // index over the freed requests' units
  if (wu >= l.n * p.LyH) return;
  const int u = l.req[wu / p.LyH] * p.LyH + wu % p.LyH;
  const int32_t nfr = p.rec[4 * (size_t)u + 2];
  if (nfr == 0) return;                                         // warp-uniform
  const int32_t off = p.rec[4 * (size_t)u], ph = p.rec[4 * (size_t)u + 1], pt = p.rec[4 * (size_t)u + 3];
  const int P = p.P;
  const int64_t ring0 = p.ctrl->rec_end0 + off;                  // < 2P
  for (int k0 = 0; k0 < nfr; k0 += 32 * 8) {
    int32_t pid[8];
#pragma unroll
    for (int j = 0; j < 8; j++) {
      const int k = k0 + 32 * j + lane;
      pid[j] = k < nfr ? __ldcg(freed_slot(p, u, k, pt, ph, nfr)) : -1;
    }
#pragma unroll
    for (int j = 0; j < 8; j++) {
      const int k = k0 + 32 * j + lane;
      if (k < nfr) {
        int64_t pos = ring0 + k;                                 // < 3P
        pos -= pos >= P ? P : 0;
        pos -= pos >= P ? P : 0;
        p.ring[pos] = pid[j];
        int32_t empty = -1;                                      // clear only after the load returned
        asm volatile("" : "+r"(empty) : "r"(pid[j]));
        *freed_slot(p, u, k, pt, ph, nfr) = empty;
      }
    }
  }
  __syncwarp();
  if (lane == 0) p.rec[4 * (size_t)u + 2] = 0;                  // marker consumed
}

cudaError_t launch_recycle(const PoolDev& p, const int32_t* req, int n, cudaStream_t s) {
  for (int i0 = 0; i0 < n; i0 += kRecMaxReq) {
    RecList l;
    l.n = n - i0 < kRecMaxReq ? n - i0 : kRecMaxReq;
    for (int i = 0; i < l.n; i++) l.req[i] = req[i0 + i];
    const long warps = (long)l.n * p.LyH;
    recycle_kernel<<<(unsigned)((warps + 7) / 8), 256, 0, s>>>(p, l);
    cudaError_t e = cudaGetLastError();
    if (e != cudaSuccess) return e;
  }
  return cudaSuccess;
}

}  // namespace dkv
