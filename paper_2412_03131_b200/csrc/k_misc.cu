// k_misc.cu — pool initialisation and request-state transitions.
#include "dkv_internal.cuh"

namespace dkv {

// a0: ring = iota, start = 0, free = P; tables = -1; counts, request state, scratch = 0.
__global__ void init_kernel(PoolDev p) {
  const size_t tid = (size_t)blockIdx.x * blockDim.x + threadIdx.x;
  const size_t nth = (size_t)gridDim.x * blockDim.x;
  for (size_t i = tid; i < (size_t)p.P; i += nth) p.ring[i] = (int32_t)i;
  const size_t UL = (size_t)p.U * p.L;
  for (size_t i = tid; i < UL; i += nth) p.table[i] = -1;
  const size_t ULt = (size_t)p.U * p.Lt;                    // NEXT-4 TOP table
  for (size_t i = tid; i < ULt; i += nth) p.ttable[i] = -1;
  for (size_t i = tid; i < (size_t)p.U; i += nth) {
    p.n_h[i] = 0; p.n_l[i] = 0; p.pf_nh[i] = 0; p.pf_nl[i] = 0;
  }
  for (size_t i = tid; i < (size_t)p.R; i += nth) {
    p.req_state[i] = DKV_REQ_IDLE; p.seq_len[i] = 0; p.prompt_len[i] = 0; p.admit[i] = 0;
  }
  for (size_t i = tid; i < (size_t)p.num_tiles; i += nth) p.tile_status[i] = 0ull;
  for (size_t i = tid; i < 4 * (size_t)p.num_tiles; i += nth) p.tsum[i] = 0u;
  if (tid == 0) {
    Ctrl* c = p.ctrl;
    c->start = 0; c->free = p.P; c->status = 0; c->oom_count = 0;
    c->ticket = 0ull; c->arrive = 0ull; c->last_demand = 0; c->last_freed = 0;
    c->total_dem = 0; c->total_fr = 0; c->bar_epoch = 0ull;
    c->tsum_ticket = ~0ull; c->arrive2 = 0ull;
    p.stats[0] = p.P; p.stats[1] = 0; p.stats[2] = 0; p.stats[3] = 0;
  }
}

cudaError_t launch_init(const PoolDev& p, cudaStream_t s) {
  init_kernel<<<148 * 4, 256, 0, s>>>(p);
  return cudaGetLastError();
}

// Request-state transitions carried in kernel parameters (captured at launch, no host buffer lifetime).
constexpr int kMaxReqPerLaunch = 240;
struct ReqList {
  int32_t n, mode;
  int32_t req[kMaxReqPerLaunch];
  int32_t len[kMaxReqPerLaunch];
  int32_t base;   // index of req[0] in the admission order
};

// mode 0: admit (IDLE -> ADMITTING, prompt_len, admission order); mode 1: free (ACTIVE -> PENDING_FREE)
__global__ void set_requests_kernel(PoolDev p, ReqList l) {
  const int i = threadIdx.x;
  if (i >= l.n) return;
  const int r = l.req[i];
  if (l.mode == 0) {
    p.req_state[r] = DKV_REQ_ADMITTING;
    p.prompt_len[r] = l.len[i];
    p.admit[l.base + i] = r;
  } else if (p.req_state[r] == DKV_REQ_ACTIVE) {      // an admission rolled back on the device (Q37) stays IDLE
    p.req_state[r] = DKV_REQ_PENDING_FREE;
  }
}

cudaError_t launch_set_requests(const PoolDev& p, const int32_t* req, const int32_t* len, int n, int mode,
                                cudaStream_t s) {
  for (int b = 0; b < n; b += kMaxReqPerLaunch) {
    ReqList l;
    l.n = n - b < kMaxReqPerLaunch ? n - b : kMaxReqPerLaunch;
    l.mode = mode;
    l.base = b;
    for (int i = 0; i < l.n; i++) {
      l.req[i] = req[b + i];
      l.len[i] = len ? len[b + i] : 0;
    }
    set_requests_kernel<<<1, kMaxReqPerLaunch, 0, s>>>(p, l);
    cudaError_t e = cudaGetLastError();
    if (e != cudaSuccess) return e;
  }
  return cudaSuccess;
}

__global__ void clear_status_kernel(PoolDev p) {
  p.ctrl->status = 0;
  p.ctrl->pending = 0;
  p.ctrl->qw_status = 0;
}

cudaError_t launch_clear_status(const PoolDev& p, cudaStream_t s) {
  clear_status_kernel<<<1, 1, 0, s>>>(p);
  return cudaGetLastError();
}

}  // namespace dkv
