// k_audit.cu — debug audit of the pool's invariants on the device (SURVEY §8 "Proposed build kernels", audit row;
// the oracle's PIN-10 invariants I1-I4 checked on the GPU's own state), behind dkv_audit.
//
// The invariants follow from the paper's memory layout: every page of the unified pool is either in
// the circular free list's free region [start, start + free) or in exactly one occupied page-table slot; a unit's
// high-precision pages fill its table row left to right and its low-precision pages right to left, so
// its occupied slots are exactly [0, ceil(n_h / C_h)) and [L - ceil(n_l / C_l), L) (and [0, ceil(n_t / C_t)) of the
// NEXT-4 TOP table, Q41); every other slot is empty (-1); and a stored token is one the model has seen and left the
// recent window, so its position is below N - W and unique within its unit.
//
// Four kernels on the caller's stream: zero the per-page histogram (caller-owned, P words) and the result; count
// the free region's pages; a warp per unit counts its occupied slots' pages, checks the empty slots and, for an
// ACTIVE request, the stored positions (a shared-memory bitmap per warp); a grid-stride pass over the histogram
// counts pages owned twice or more and pages owned by nobody.
#include "dkv_internal.cuh"

namespace dkv {

constexpr int kAuditWarps = 4;

__device__ __forceinline__ void audit_add(int64_t* res, int i, unsigned long long v) {
  if (v) atomicAdd(reinterpret_cast<unsigned long long*>(res + i), v);
}

__global__ void audit_zero_kernel(PoolDev p, uint32_t* hist, int64_t* res) {
  const size_t tid = (size_t)blockIdx.x * blockDim.x + threadIdx.x, nth = (size_t)gridDim.x * blockDim.x;
  for (size_t i = tid; i < (size_t)p.P; i += nth) hist[i] = 0u;
  if (tid < kAuditResults) res[tid] = 0;
}

// the free region [start, start + free) of the ring
__global__ void audit_ring_kernel(PoolDev p, uint32_t* hist, int64_t* res) {
  const int64_t start = ld_volatile(&p.ctrl->start), fr = ld_volatile(&p.ctrl->free);
  const size_t tid = (size_t)blockIdx.x * blockDim.x + threadIdx.x, nth = (size_t)gridDim.x * blockDim.x;
  unsigned long long bad = 0;
  for (size_t i = tid; i < (size_t)fr; i += nth) {
    int64_t pos = start + (int64_t)i;
    pos -= pos >= p.P ? p.P : 0;
    const int32_t id = p.ring[pos];
    if (id < 0 || id >= p.P) bad++;
    else atomicAdd(hist + id, 1u);
  }
  audit_add(res, 2, bad);
  if (tid == 0) res[4] = fr;
}

// a warp per unit: page-table slots and (ACTIVE requests) stored positions
__global__ void __launch_bounds__(kAuditWarps * 32) audit_units_kernel(PoolDev p, uint32_t* hist, int64_t* res) {
  extern __shared__ uint32_t s_bits[];                     // [kAuditWarps][ceil(M / 32)] seen positions
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int u = blockIdx.x * kAuditWarps + warp;
  if (u >= p.U) return;
  const int MW = (p.M + 31) / 32;
  uint32_t* bits = s_bits + (size_t)warp * MW;
  const int nh = p.n_h[u], nl = p.n_l[u], nt = p.top ? p.n_t[u] : 0;
  const int ph = (nh + p.Ch - 1) / p.Ch, pl = (nl + p.Cl - 1) / p.Cl, pt = p.top ? (nt + p.Ct - 1) / p.Ct : 0;
  unsigned long long bad = 0, used = 0, dup = 0, out = 0, over = 0;
  if (ph + pl > p.L || pt > p.Lt) over = 1;
  const int32_t* row = p.table + (size_t)u * p.L;
  for (int k = lane; k < p.L; k += 32) {
    const int32_t id = row[k];
    const bool occ = k < ph || k >= p.L - pl;
    if (occ) {
      if (id < 0 || id >= p.P) bad++;
      else { atomicAdd(hist + id, 1u); used++; }
    } else if (id != -1) {
      bad++;
    }
  }
  if (p.top) {
    const int32_t* trow = p.ttable + (size_t)u * p.Lt;
    for (int k = lane; k < p.Lt; k += 32) {
      const int32_t id = trow[k];
      if (k < pt) {
        if (id < 0 || id >= p.P) bad++;
        else { atomicAdd(hist + id, 1u); used++; }
      } else if (id != -1) {
        bad++;
      }
    }
  }
  // stored positions of an ACTIVE request: in [0, N - W), unique within the unit
  const int r = u / p.LyH;
  if (p.req_state[r] == DKV_REQ_ACTIVE && over == 0) {
    const int lim = p.seq_len[r] - p.W;
    for (int i = lane; i < MW; i += 32) bits[i] = 0u;
    __syncwarp();
    for (int cls = 0; cls < 3; cls++) {
      const int n = cls == 0 ? nh : (cls == 1 ? nl : nt);
      const ClassGeom g = cls == 0 ? p.g[1] : (cls == 1 ? p.g[2] : p.gt);
      for (int s = lane; s < n; s += 32) {
        const int k = s / g.C, idx = s - k * g.C;
        const int32_t id = cls == 0 ? row[k] : (cls == 1 ? row[p.L - 1 - k] : p.ttable[(size_t)u * p.Lt + k]);
        if (id < 0 || id >= p.P) continue;                  // counted above
        const int32_t pos = *reinterpret_cast<const int32_t*>(p.pages + (size_t)id * p.page_bytes + g.off_pos + 4 * idx);
        if (pos < 0 || pos >= lim || pos >= p.M) { out++; continue; }
        const uint32_t m = 1u << (pos & 31);
        if (atomicOr(bits + (pos >> 5), m) & m) dup++;
      }
    }
  }
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) {
    bad += __shfl_xor_sync(kFull, bad, o);
    used += __shfl_xor_sync(kFull, used, o);
    dup += __shfl_xor_sync(kFull, dup, o);
    out += __shfl_xor_sync(kFull, out, o);
  }
  if (lane == 0) {
    audit_add(res, 2, bad);
    audit_add(res, 3, used);
    audit_add(res, 5, dup);
    audit_add(res, 6, out);
    audit_add(res, 7, over);
  }
}

// every page is owned exactly once (free region or one occupied slot)
__global__ void audit_count_kernel(PoolDev p, const uint32_t* hist, int64_t* res) {
  const size_t tid = (size_t)blockIdx.x * blockDim.x + threadIdx.x, nth = (size_t)gridDim.x * blockDim.x;
  unsigned long long twice = 0, none = 0;
  for (size_t i = tid; i < (size_t)p.P; i += nth) {
    const uint32_t c = hist[i];
    twice += c >= 2u;
    none += c == 0u;
  }
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) {
    twice += __shfl_xor_sync(kFull, twice, o);
    none += __shfl_xor_sync(kFull, none, o);
  }
  if ((threadIdx.x & 31) == 0) {
    audit_add(res, 0, twice);
    audit_add(res, 1, none);
  }
}

cudaError_t launch_audit(const PoolDev& p, uint32_t* hist, int64_t* res, cudaStream_t s) {
  audit_zero_kernel<<<148 * 4, 256, 0, s>>>(p, hist, res);
  audit_ring_kernel<<<148 * 4, 256, 0, s>>>(p, hist, res);
  const size_t smem = (size_t)kAuditWarps * ((p.M + 31) / 32) * 4;
  cudaError_t e = cudaGetLastError();
  if (e != cudaSuccess) return e;
  if (smem > 48 * 1024) {
    e = cudaFuncSetAttribute(audit_units_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    if (e != cudaSuccess) return e;
  }
  audit_units_kernel<<<(p.U + kAuditWarps - 1) / kAuditWarps, kAuditWarps * 32, smem, s>>>(p, hist, res);
  audit_count_kernel<<<148 * 4, 256, 0, s>>>(p, hist, res);
  return cudaGetLastError();
}

}  // namespace dkv
