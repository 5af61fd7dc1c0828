// k_prefill_conservative.cu — the paper's prompt-phase workflow (NEXT-1, fig:memory_management_flow)
// behind dkv_compact_alloc(PREFILL) when dkv_config_t.prefill_workflow = 1.  Runs after the recycle-only
// pass of compact_alloc_kernel, so start / free already include this call's recycled pages (Q14).
//
//   "memory pages are conservatively allocated for each head, assuming all tokens are stored at high
//    precision": head u gets a block of c_u = ceil(kept/C_h) pages, kept = prompt tokens outside
//    the window, from the allocation pointer (Q1) — exclusive scan of c over canonical units;
//   the planning phase (dkv_classify(PREFILL), already run) fixed ph = ceil(n_h/C_h), pl = ceil(n_l/C_l)
//    (P:525-526); a head whose plan needs one page more than its block (Q29) takes one top-up page,
//    granted after every block (exclusive scan of e);
//   "each head retains the high-precision pages from the left and the low-precision pages from the right
//    ... pages in between are reclaimed and appended at the end pointer via a parallel prefix-sum"
//     — exclusive scan of the middle counts m, ring[end + off_m + k].
// All three scans are one pass: block scans, per-tile totals in pool scratch, a grid barrier, and every
// tile summing its predecessors' totals.  Blocks and top-ups are one all-or-nothing allocation (Q15).  A
// second grid barrier separates every read of a granted ring slot from the reclaim writes (which may wrap
// onto granted slots when the free region ends at the start pointer); the middle page IDs wait in their
// own (empty) table slots in between.  The launch is cooperative (co-residency of every tile).
#include "dkv_internal.cuh"

namespace dkv {

__device__ __forceinline__ uint32_t warp_incl_scan_u32(uint32_t v, int lane) {
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    const uint32_t y = __shfl_up_sync(kFull, v, o);
    if (lane >= o) v += y;
  }
  return v;
}

__device__ __forceinline__ void grid_barrier(Ctrl* ctrl, unsigned long long target) {
  __syncthreads();
  if (threadIdx.x == 0) {
    __threadfence();
    atomicAdd(&ctrl->arrive, 1ull);
    while (ld_acquire(&ctrl->arrive) < target) __nanosleep(40);
    __threadfence();
  }
  __syncthreads();
}

template <int TU>
__global__ void __launch_bounds__(TU) prefill_conservative_kernel(PoolDev p) {
  constexpr int NW = TU / 32;
  __shared__ int64_t s_start0, s_free0;
  __shared__ int s_status0;
  __shared__ unsigned long long s_bep;
  __shared__ uint32_t s_w[3][NW];
  __shared__ int64_t s_ex[3], s_tot[3];
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5, tile = blockIdx.x;
  Ctrl* ctrl = p.ctrl;
  if (tid == 0) {
    s_start0 = ctrl->start;
    s_free0 = ctrl->free;
    s_status0 = ctrl->status;
    s_bep = *(volatile unsigned long long*)&ctrl->bar_epoch;   // only this kernel's last tile 0 moves it
  }
  const int u = tile * TU + tid;
  int r = 0, cu = 0, eu = 0, mu = 0, ph = 0, pl = 0;
  bool adm = false;
  if (u < p.U) {
    r = fdiv(p.div_LyH, u);
    adm = p.req_state[r] == DKV_REQ_ADMITTING;
  }
  __syncthreads();
  const int status0 = s_status0;
  const int64_t start0 = s_start0, free0 = s_free0;
  const int P = p.P, L = p.L;
  adm = adm && status0 == 0;
  if (adm) {
    const int kept = max(p.prompt_len[r] - p.W, 0);
    cu = ceil_div(kept, p.Ch);                                   // "assuming all tokens ... high precision"
    ph = ceil_div(p.pf_nh[u], p.Ch);
    pl = ceil_div(p.pf_nl[u], p.Cl);
    eu = ph + pl > cu ? 1 : 0;                                   // Q29 top-up
    mu = cu + eu - ph - pl;                                      // the reclaimed middle
  }

  // ---- three exclusive scans over canonical units: block (c), top-up (e), middle (m)
  const uint32_t ic = warp_incl_scan_u32((uint32_t)cu, lane);
  const uint32_t ie = __popc(__ballot_sync(kFull, eu != 0) & (0xFFFFFFFFu >> (31 - lane)));
  const uint32_t im = warp_incl_scan_u32((uint32_t)mu, lane);
  if (lane == 31) { s_w[0][warp] = ic; s_w[1][warp] = ie; s_w[2][warp] = im; }
  __syncthreads();
  if (warp == 0) {
#pragma unroll
    for (int k = 0; k < 3; k++) {
      const uint32_t a = lane < NW ? s_w[k][lane] : 0u;
      const uint32_t ia = warp_incl_scan_u32(a, lane);
      if (lane < NW) s_w[k][lane] = ia - a;
      if (lane == 31) p.tile_sums[(size_t)tile * 3 + k] = (int64_t)ia;
    }
  }
  const unsigned long long T = (unsigned long long)gridDim.x;
  grid_barrier(ctrl, (s_bep + 1ull) * T);
  if (warp == 0) {
    int64_t ex[3] = {0, 0, 0}, tot[3] = {0, 0, 0};
    for (int t = lane; t < (int)gridDim.x; t += 32) {
#pragma unroll
      for (int k = 0; k < 3; k++) {
        const int64_t v = __ldcg(p.tile_sums + (size_t)t * 3 + k);
        tot[k] += v;
        if (t < tile) ex[k] += v;
      }
    }
#pragma unroll
    for (int k = 0; k < 3; k++) {
#pragma unroll
      for (int o = 16; o > 0; o >>= 1) {
        ex[k] += __shfl_xor_sync(kFull, ex[k], o);
        tot[k] += __shfl_xor_sync(kFull, tot[k], o);
      }
    }
    if (lane == 0) {
#pragma unroll
      for (int k = 0; k < 3; k++) { s_ex[k] = ex[k]; s_tot[k] = tot[k]; }
    }
  }
  __syncthreads();
  const int64_t off_c = s_ex[0] + s_w[0][warp] + ic - (uint32_t)cu;
  const int64_t off_e = s_ex[1] + s_w[1][warp] + ie - (uint32_t)eu;
  const int64_t off_m = s_ex[2] + s_w[2][warp] + im - (uint32_t)mu;
  const int64_t D = s_tot[0] + s_tot[1], M = s_tot[2];
  const bool ok = status0 == 0 && D <= free0;
  const int64_t end0 = (start0 + free0) % P;

  // ---- grant: block'[k] = ring[start + off_c + k] (k < c), the top-up ring[start + sum(c) + off_e];
  // high pages left to right, low pages right to left; the middle waits in its own slots
  if (ok) {
    unsigned gm = __ballot_sync(kFull, adm);
    while (gm) {
      const int src = __ffs(gm) - 1;
      gm &= gm - 1;
      const int uu = __shfl_sync(kFull, u, src);
      const int c_ = __shfl_sync(kFull, cu, src), e_ = __shfl_sync(kFull, eu, src);
      const int ph_ = __shfl_sync(kFull, ph, src), pl_ = __shfl_sync(kFull, pl, src);
      const int64_t bc = start0 + __shfl_sync(kFull, off_c, src);
      const int64_t pe = start0 + s_tot[0] + __shfl_sync(kFull, off_e, src);
      const int nb = c_ + e_;
      if (ph_ + pl_ > L || nb > L) {                             // unreachable (Q12)
        if (lane == 0) set_status(ctrl, DKV_ERR_OVERFLOW);
        continue;
      }
      int32_t* row = p.table + (size_t)uu * L;
      for (int k = lane; k < nb - pl_; k += 32)                  // high pages + the middle (staged)
        row[k] = __ldcg(p.ring + (k < c_ ? bc + k : pe) % P);
      for (int k = lane; k < pl_; k += 32) {                     // low pages: block'[nb-1-k] -> slot L-1-k
        const int b = nb - 1 - k;
        row[L - 1 - k] = __ldcg(p.ring + (b < c_ ? bc + b : pe) % P);
      }
    }
  }
  grid_barrier(ctrl, (s_bep + 2ull) * T);

  // ---- reclaim the middles at the end pointer, canonical order
  if (ok) {
    unsigned gm = __ballot_sync(kFull, adm && mu > 0);
    while (gm) {
      const int src = __ffs(gm) - 1;
      gm &= gm - 1;
      const int uu = __shfl_sync(kFull, u, src);
      const int m_ = __shfl_sync(kFull, mu, src), ph_ = __shfl_sync(kFull, ph, src);
      const int64_t om = __shfl_sync(kFull, off_m, src);
      int32_t* row = p.table + (size_t)uu * L;
      for (int k = lane; k < m_; k += 32) {
        const int32_t pid = __ldcg(row + ph_ + k);
        p.ring[(end0 + om + k) % P] = pid;
        int32_t empty = -1;                                      // clear only after the load returned
        asm volatile("" : "+r"(empty) : "r"(pid));
        row[ph_ + k] = empty;
      }
    }
    if (adm) { p.n_h[u] = p.pf_nh[u]; p.n_l[u] = p.pf_nl[u]; }
    if (adm && fmod_(p.div_LyH, u) == p.LyH - 1) p.seq_len[r] = p.prompt_len[r];
  }
  if (tile == 0 && tid == 0) {
    if (status0 == 0 && !ok) { set_status(ctrl, DKV_ERR_OOM); ctrl->oom_count += 1; }
    const int64_t ns = ok ? (start0 + D) % P : start0;
    const int64_t nf = ok ? free0 - D + M : free0;
    ctrl->start = ns;
    ctrl->free = nf;
    ctrl->last_demand = status0 == 0 ? D : 0;
    ctrl->bar_epoch = s_bep + 2ull;                              // every tile read it before arriving
    p.stats[0] = nf;
    p.stats[1] = -(status0 == 0 ? D : 0);
    p.stats[2] = -((int64_t)P - nf);
    const int fin = ld_volatile(&ctrl->status);
    ctrl->qw_status = fin;                             // entry status of the following dkv_quant_write (Q36)
    p.stats[3] = (int64_t)fin;                         // <= 0: the MIN over GPUs shows any error
  }
}

template <int TU>
static cudaError_t launch_pc(const PoolDev& p, cudaStream_t s) {
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3(p.num_tiles);
  cfg.blockDim = dim3(TU);
  cfg.stream = s;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeCooperative;
  attr[0].val.cooperative = 1;
  cfg.attrs = attr;
  cfg.numAttrs = 1;
  return cudaLaunchKernelEx(&cfg, prefill_conservative_kernel<TU>, p);
}

cudaError_t launch_prefill_conservative(const PoolDev& p, cudaStream_t s) {
  switch (p.tile_units) {
    case 256: return launch_pc<256>(p, s);
    case 512: return launch_pc<512>(p, s);
    default: return launch_pc<1024>(p, s);
  }
}

}  // namespace dkv
