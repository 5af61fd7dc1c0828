// k_quant_decode.cu — the KV compressor's generation step behind dkv_quant_write(DECODE).
//
// Four lanes per unit, eight units per warp.  A d-vector is handled as d/8 16-byte chunks; lane q of a
// group owns chunks q, q+4, q+8, ... so each warp-wide 16-B access of a group covers 64 contiguous bytes.
// Per unit, in the order readings Q8/Q9 fix:
//   1. downgrade the victim t_v (v_action == DOWN): dequantize its K8V4 codes from its KV_h slot and
//      re-quantize at K4V2 (quant_chunks_f32) into KV_l slot v_dst_slot, carrying its score and position —
//      before t_c overwrites that KV_h slot;
//   2. quantize t_c out of window slot (N-1) mod W == p_c mod W at its class bits (quant_chunks_h16) into
//      tc_slot, score = s_c, position = p_c;
//   3. write the new token into that same window slot (its old row was read into registers first).
// Every collective is group-masked, so units with different classes / actions in one warp are independent.
#include <stdlib.h>

#include "dkv_internal.cuh"

namespace dkv {

constexpr int kQDWarps = 4;

template <int D, int kQDG>                               // kQDG lanes per unit
__global__ void __launch_bounds__(kQDWarps * 32)
quant_decode_kernel(PoolDev p, const dkv_decision_t* __restrict__ dec, const uint16_t* __restrict__ knew,
                    const uint16_t* __restrict__ vnew, const float* __restrict__ cand_sig) {
  constexpr int NCH = D / (8 * kQDG);                    // chunks per lane
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int grp = lane / kQDG, q = lane % kQDG;
  const unsigned gmask = ((1u << kQDG) - 1u) << (grp * kQDG);
  const int u = (blockIdx.x * kQDWarps + warp) * (32 / kQDG) + grp;
  if (u >= p.U) return;                                  // whole groups exit together
  if (ld_volatile(&p.ctrl->status) != 0) return;
  const int r = u / p.LyH;
  if (p.req_state[r] != DKV_REQ_ACTIVE) return;
  const int N = p.seq_len[r];                            // already includes this step's token (compact_alloc)
  const int pc = N - 1 - p.W;
  const int4 dw = reinterpret_cast<const int4*>(dec)[u];
  const int tc_class = dw.x & 0xFF, v_action = (dw.x >> 8) & 0xFF;
  const int v_slot = dw.y, tc_slot = dw.z, v_dst = dw.w;

  // window row of t_c and the new token (16 x 16 B per lane in flight at d = 128)
  uint32_t wk[NCH][4], wv[NCH][4], nk[NCH][4], nv[NCH][4];
  const int ws = p.W > 0 ? (N - 1) % p.W : 0;
  uint4* wk_row = reinterpret_cast<uint4*>(p.win_k + ((size_t)u * p.W + ws) * D);
  uint4* wv_row = reinterpret_cast<uint4*>(p.win_v + ((size_t)u * p.W + ws) * D);
  const uint4* nk_row = reinterpret_cast<const uint4*>(knew + (size_t)u * D);
  const uint4* nv_row = reinterpret_cast<const uint4*>(vnew + (size_t)u * D);
#pragma unroll
  for (int c = 0; c < NCH; c++) {
    const int ch = q + kQDG * c;
    const uint4 a = __ldg(nk_row + ch), b = __ldg(nv_row + ch);
    nk[c][0] = a.x; nk[c][1] = a.y; nk[c][2] = a.z; nk[c][3] = a.w;
    nv[c][0] = b.x; nv[c][1] = b.y; nv[c][2] = b.z; nv[c][3] = b.w;
    uint4 x = a, y = b;                                  // W = 0: t_c is the new token itself
    if (p.W > 0) { x = wk_row[ch]; y = wv_row[ch]; }
    wk[c][0] = x.x; wk[c][1] = x.y; wk[c][2] = x.z; wk[c][3] = x.w;
    wv[c][0] = y.x; wv[c][1] = y.y; wv[c][2] = y.z; wv[c][3] = y.w;
  }
  // 3. window push, issued early: t_c's row is already in registers (same lanes, same addresses, program order)
  if (p.W > 0) {
#pragma unroll
    for (int c = 0; c < NCH; c++) {
      const int ch = q + kQDG * c;
      wk_row[ch] = make_uint4(nk[c][0], nk[c][1], nk[c][2], nk[c][3]);
      wv_row[ch] = make_uint4(nv[c][0], nv[c][1], nv[c][2], nv[c][3]);
    }
  }

  // 1. downgrade t_v: K8V4 -> K4V2 (Q9)
  if (v_action == DKV_V_DOWN) {
    const ClassGeom gh = geom_of(p, DKV_CLS_HIGH), go = geom_of(p, DKV_CLS_LOW);
    int is, id;
    const uint8_t* src = slot_page(p, DKV_CLS_HIGH, u, v_slot, is);
    uint8_t* dst = slot_page(p, DKV_CLS_LOW, u, v_dst, id);
#pragma unroll 1
    for (int kvsel = 0; kvsel < 2; kvsel++) {
      const int sb = kvsel ? gh.vbits : gh.kbits, db = kvsel ? go.vbits : go.kbits;
      const uint8_t* srow = src + (kvsel ? gh.off_v + is * gh.v_row : gh.off_k + is * gh.k_row);
      uint8_t* drow = dst + (kvsel ? go.off_v + id * go.v_row : go.off_k + id * go.k_row);
      const uint32_t meta = *reinterpret_cast<const uint32_t*>(src + (kvsel ? gh.off_vmeta : gh.off_kmeta) + 4 * is);
      float x[NCH][8];
#pragma unroll
      for (int c = 0; c < NCH; c++) dequant_chunk(srow, q + kQDG * c, sb, meta, x[c]);
      uint2 pk[NCH];
      uint32_t m2;
      quant_chunks_f32<kQDG, NCH>(x, db, gmask, pk, m2);
#pragma unroll
      for (int c = 0; c < NCH; c++) store_chunk_codes(drow, q + kQDG * c, db, pk[c]);
      if (q == kvsel) *reinterpret_cast<uint32_t*>(dst + (kvsel ? go.off_vmeta : go.off_kmeta) + 4 * id) = m2;
    }
    if (q == 2) *reinterpret_cast<uint32_t*>(dst + go.off_score + 4 * id) =
        *reinterpret_cast<const uint32_t*>(src + gh.off_score + 4 * is);
    if (q == 3) *reinterpret_cast<int32_t*>(dst + go.off_pos + 4 * id) =
        *reinterpret_cast<const int32_t*>(src + gh.off_pos + 4 * is);
  }

  // 2. t_c -> its section slot at its class bits
  if (tc_class == DKV_CLS_HIGH || tc_class == DKV_CLS_LOW) {
    const ClassGeom g = geom_of(p, tc_class);
    uint2 pkk[NCH], pkv[NCH];
    uint32_t mk, mv;
    bool fk, fv;
    quant_chunks_h16<kQDG, NCH>(wk, g.kbits, gmask, pkk, mk, fk);
    quant_chunks_h16<kQDG, NCH>(wv, g.vbits, gmask, pkv, mv, fv);
    if (!(fk && fv)) {
      if (q == 0) set_status(p.ctrl, DKV_ERR_NONFINITE);
    } else {
      int idx;
      uint8_t* pg = slot_page(p, tc_class, u, tc_slot, idx);
      uint8_t* krow = pg + g.off_k + idx * g.k_row;
      uint8_t* vrow = pg + g.off_v + idx * g.v_row;
#pragma unroll
      for (int c = 0; c < NCH; c++) {
        store_chunk_codes(krow, q + kQDG * c, g.kbits, pkk[c]);
        store_chunk_codes(vrow, q + kQDG * c, g.vbits, pkv[c]);
      }
      if (q == 0) *reinterpret_cast<uint32_t*>(pg + g.off_kmeta + 4 * idx) = mk;
      if (q == 1) *reinterpret_cast<uint32_t*>(pg + g.off_vmeta + 4 * idx) = mv;
      if (q == 2) *reinterpret_cast<float*>(pg + g.off_score + 4 * idx) = canon_zero(cand_sig[u]);
      if (q == 3) *reinterpret_cast<int32_t*>(pg + g.off_pos + 4 * idx) = pc;
    }
  }
}

template <int D, int G>
static cudaError_t launch_qd(const PoolDev& p, const dkv_decision_t* dec, const uint16_t* k, const uint16_t* v,
                             const float* sig, cudaStream_t s) {
  const int units_per_cta = kQDWarps * (32 / G);
  const int grid = (p.U + units_per_cta - 1) / units_per_cta;
  quant_decode_kernel<D, G><<<grid, kQDWarps * 32, 0, s>>>(p, dec, k, v, sig);
  return cudaGetLastError();
}

cudaError_t launch_quant_decode(const PoolDev& p, const dkv_decision_t* dec, const uint16_t* k, const uint16_t* v,
                                const float* sig, cudaStream_t s) {
  static const int g = getenv("DKV_QD_G") ? atoi(getenv("DKV_QD_G")) : 4;   // tuning knob
  if (p.d == 128) {
    if (g == 16) return launch_qd<128, 16>(p, dec, k, v, sig, s);
    return g == 4 ? launch_qd<128, 4>(p, dec, k, v, sig, s) : launch_qd<128, 8>(p, dec, k, v, sig, s);
  }
  return g == 4 ? launch_qd<64, 4>(p, dec, k, v, sig, s) : launch_qd<64, 8>(p, dec, k, v, sig, s);
}

}  // namespace dkv
