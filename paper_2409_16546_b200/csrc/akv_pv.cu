// output_aligned for every (unit, q-head).
//
// Per-warp TMA ring: every warp owns a balanced contiguous range of
// (unit, page, head-pass) items and streams them through a private 2-slot
// shared-memory ring.  Lane 0 issues one cp.async.bulk per 64-row stage of V
// head rows (8 KB, token-major; uniform tiers: 32 rows + their mid / low rows)
// and, with a page's first stage, the page's p_t, selection words and the
// q-heads' need-mid / need-low words (akv_softmax_select's RowMax superset
// rule); everything completes on the slot's mbarrier.  The warp
// computes one stage while the next is in flight; no cross-warp sync.
// Lane = (row r4 = lane / 8, 16-channel group cg = lane % 8): one LDS.128
// reads four rows; a batch is 16 rows.
//
// A batch with no row in the union fetch plan (the common case) takes the
// branch-free path: T8 words by PRMT (midpoint fill, HB:160-179), fp16 ->
// fp32 by HADD2.F32, p_t * V~ by the packed FFMA2 into fp32.
// Selected rows carry p = 0 here (D6: their T16 contribution is o_est).
// Other rows fetch the needed 64 B nibble rows (LDG) and apply each q-head's
// rule: unknown target_r -> T16 (p_t = 0 included), else p_t = 0 -> T8 (D5);
// ELEMENT: keep mid iff max(bexp,1) + e(p_t) >
// 17 + target_r - margin, low iff > that + 4 (D4); row strategy: the row tier
// (D7); forced / baseline tiers.  Truncation is applied after the fetch, so
// the masks equal the oracle's bit for bit.  The page's partial output goes to
// o_partial[h][page]; akv_combine adds o_est and the partials in a fixed order
// (deterministic).
#include <algorithm>
#include <cstdlib>
#include <cstring>

#include <cuda.h>

#include "akv_common.cuh"

namespace akv {

// One 16-row batch as the row code sees it (filled from the stage in shared
// memory).  Aligned mode stages only head rows (nibble rows are rare and are
// fetched on demand by the generic path); uniform tiers (forced / baseline)
// stage the nibble rows too.
template <int HG, bool NIB>
struct VBatch {
  uint4 h[4];                        // head bytes: row 16b + 4i + r4, channels 16cg .. +15
  uint2 m[NIB ? 4 : 1], l[NIB ? 4 : 1];  // mid / low nibble words of the same (uniform tiers)
  float p[HG];                       // lanes 0..15: p of row 16b + lane (0 beyond n)
  uint32_t sel[HG];                  // selection word of the batch's 32-row chunk (warp-uniform)
};

__device__ __forceinline__ void t8_words16(const uint4& h, uint32_t w[8]) {
  const uint32_t c80 = 0x80808080u;
  const uint32_t hv[4] = {h.x, h.y, h.z, h.w};
#pragma unroll
  for (int r = 0; r < 4; ++r) {
    w[2 * r] = prmt(hv[r], c80, 0x1404);
    w[2 * r + 1] = prmt(hv[r], c80, 0x3424);
  }
}

struct PvCtx {
  const uint8_t* vb;  // page base (V pool)
  int rows;           // valid rows of the page
  int pg, u, cap;
  uint32_t nwu;       // lanes 0..7: union need-mid word of chunk lane; lanes 8..15: need-low word of chunk lane-8
};

template <int HG>
struct VGen {  // contributions of the aligned generic path (returned by value: keeps the caller's
  float2 acc[HG][8];  // accumulators in registers)
  int adj[HG][3];
};
template <int HG>
struct VRowP {
  float v[HG][4];
};

// One aligned row in the union fetch plan (this lane's 16 channels): per q-head mode
// (selected -> skip, no need bit -> T8, row strategy -> row tier, element strategy ->
// per-element rule D4) applied to the fetched nibbles; contributions into out.
// selw[jj]: the row's 32-row selection word; vt_row: export pointer of the row (or null).
template <int G, int HG, bool EXPORT>
__device__ __forceinline__ void v_row_generic(VGen<HG>& out, const uint4& hv, uint2 mw, uint2 lw, int row, bool valid,
                                              const PvCtx& c, int j0, const akv_cfg_t& cfg, const akv_step_t& st,
                                              const float (&pvj)[HG], const uint32_t (&selw)[HG], uint8_t* vt_row) {
  const int lane = threadIdx.x & 31, cg = lane & 7;
  const int capw = c.cap >> 5, ch = row >> 5;
#pragma unroll
  for (int jj = 0; jj < HG; ++jj) {
    const size_t h = (size_t)c.u * G + j0 + jj;
    const float pv = pvj[jj];
    int mode;  // 0 skip, 1 element, 8/12/16 tier
    if ((selw[jj] >> (row & 31)) & 1u) {
      mode = 0;
    } else {
      const uint32_t nm = st.need_bits[h * 2 * capw + c.pg * 8 + ch];
      if (!((nm >> (row & 31)) & 1u)) {
        mode = 8;  // p == 0 rows are outside the plan unless some target is unknown (D5)
      } else if (cfg.strategy == 1) {
        const uint32_t nl = st.need_bits[h * 2 * capw + capw + c.pg * 8 + ch];
        mode = ((nl >> (row & 31)) & 1u) ? 16 : 12;
      } else {
        mode = 1;
      }
    }
    if (!valid) mode = 0;
    uint32_t w[8];
    uint32_t cds[4] = {0u, 0u, 0u, 0u};
    if (mode == 0) {
      if (EXPORT && vt_row && valid)
        *reinterpret_cast<uint4*>(vt_row + (size_t)(j0 + jj) * c.cap * D) =
            make_uint4(0x10101010u, 0x10101010u, 0x10101010u, 0x10101010u);
      continue;
    }
    if (mode == 8) {
      t8_words16(hv, w);
      if (EXPORT) cds[0] = cds[1] = cds[2] = cds[3] = 0x08080808u;
    } else if (mode != 1) {
      const TierMask tm = tier_mask(mode);
      assemble8(hv.x, hv.y, bsel(tm.mk, mw.x, 0x88888888u), bsel(tm.lk, lw.x, tm.lf), w);
      assemble8(hv.z, hv.w, bsel(tm.mk, mw.y, 0x88888888u), bsel(tm.lk, lw.y, tm.lf), w + 4);
      out.adj[jj][0] -= 16;
      out.adj[jj][mode == 12 ? 1 : 2] += 16;
      if (EXPORT) cds[0] = cds[1] = cds[2] = cds[3] = (uint32_t)mode * 0x01010101u;
    } else {
      assemble8(hv.x, hv.y, mw.x, lw.x, w);
      assemble8(hv.z, hv.w, mw.y, lw.y, w + 4);
      const int ep = pv > 0.f ? floor_log2f(pv) : -30000;
      const int4* tp = reinterpret_cast<const int4*>(st.targets + h * D + cg * 16);
      int tg[16];
#pragma unroll
      for (int q4 = 0; q4 < 4; ++q4) {
        const int4 t = tp[q4];
        tg[4 * q4] = t.x;
        tg[4 * q4 + 1] = t.y;
        tg[4 * q4 + 2] = t.z;
        tg[4 * q4 + 3] = t.w;
      }
      const uint32_t hb[4] = {hv.x, hv.y, hv.z, hv.w};
#pragma unroll
      for (int e = 0; e < 16; ++e) {
        const int g = tg[e] == AKV_TARGET_UNKNOWN ? -(1 << 20) : 17 + tg[e] - cfg.margin_bits;
        const uint32_t hbyte = (hb[e >> 2] >> (8 * (e & 3))) & 0xFFu;
        const int E = max((int)((hbyte >> 2) & 31u), 1) + ep;
        const bool km = E > g, kl = E > g + 4;
        const int sh = 16 * (e & 1);
        uint32_t w16 = (w[e >> 1] >> sh) & 0xFFFFu;
        w16 = kl ? w16 : (km ? ((w16 & 0xFFF0u) | 0x8u) : ((w16 & 0xFF00u) | 0x80u));
        w[e >> 1] = (w[e >> 1] & ~(0xFFFFu << sh)) | (w16 << sh);
        out.adj[jj][0] -= km ? 1 : 0;
        out.adj[jj][1] += (km && !kl) ? 1 : 0;
        out.adj[jj][2] += kl ? 1 : 0;
        if (EXPORT) cds[e >> 2] |= (kl ? 16u : (km ? 12u : 8u)) << (8 * (e & 3));
      }
    }
#pragma unroll
    for (int k = 0; k < 8; ++k) out.acc[jj][k] = ffma2_scalar(half2_bits_to_float2(w[k]), pv, out.acc[jj][k]);
    if (EXPORT && vt_row)
      *reinterpret_cast<uint4*>(vt_row + (size_t)(j0 + jj) * c.cap * D) = make_uint4(cds[0], cds[1], cds[2], cds[3]);
  }
}

template <int HG>
__device__ __forceinline__ void vgen_zero(VGen<HG>& out) {
#pragma unroll
  for (int jj = 0; jj < HG; ++jj) {
    out.adj[jj][0] = out.adj[jj][1] = out.adj[jj][2] = 0;
#pragma unroll
    for (int q = 0; q < 8; ++q) out.acc[jj][q] = make_float2(0.f, 0.f);
  }
}

// Aligned rows of a batch in the union fetch plan (quads in qmask), nibble rows fetched
// here.  Rare on the hot path, so kept out of line (I-cache).
template <int G, int HG, bool EXPORT>
__device__ __noinline__ VGen<HG> v_generic_aligned(VBatch<HG, false> X, PvCtx c, int b, int j0, akv_cfg_t cfg,
                                                   const akv_step_t* stp, VRowP<HG> p, uint32_t um, uint32_t qmask) {
  const akv_step_t& st = *stp;
  const int lane = threadIdx.x & 31, r4 = lane >> 3, cg = lane & 7;
  const int nvalid = min(max(c.rows - 16 * b, 0), 16);
  VGen<HG> out;
  vgen_zero(out);
  uint8_t* vt = nullptr;
  if (EXPORT && st.v_tiers) vt = st.v_tiers + ((size_t)c.u * G * c.cap + (size_t)c.pg * P + 16 * b) * D + cg * 16;
  const uint32_t ul = __shfl_sync(0xFFFFFFFFu, c.nwu, 8 + (b >> 1));
  const uint64_t pol = evict_first_policy();
#pragma unroll 1
  for (int i = 0; i < 4; ++i) {
    if (!((qmask >> i) & 1u)) continue;  // quad handled by the caller's T8 path
    const int rr = 4 * i + r4, row = 16 * b + rr;
    const bool valid = rr < nvalid;
    const uint4 hv = i == 0 ? X.h[0] : (i == 1 ? X.h[1] : (i == 2 ? X.h[2] : X.h[3]));
    uint2 mw = make_uint2(0u, 0u), lw = make_uint2(0u, 0u);
    if (valid && ((um >> (row & 31)) & 1u)) mw = ld_stream_u64(c.vb + MID + row * (D / 2) + cg * 8, pol);
    if (valid && ((ul >> (row & 31)) & 1u)) lw = ld_stream_u64(c.vb + LOW + row * (D / 2) + cg * 8, pol);
    float pvj[HG];
    uint32_t selw[HG];
#pragma unroll
    for (int jj = 0; jj < HG; ++jj) {
      pvj[jj] = i == 0 ? p.v[jj][0] : (i == 1 ? p.v[jj][1] : (i == 2 ? p.v[jj][2] : p.v[jj][3]));
      selw[jj] = X.sel[jj];
    }
    v_row_generic<G, HG, EXPORT>(out, hv, mw, lw, row, valid, c, j0, cfg, st, pvj, selw,
                                 vt ? vt + (size_t)rr * D : nullptr);
  }
  return out;
}

// One quad (this lane's row) of a wide-group stage in the fetch plan; out of line.
template <int G, int HG>
__device__ __noinline__ VGen<HG> v_quad_generic(uint4 hv, int row, bool valid, PvCtx c, int j0, akv_cfg_t cfg,
                                                const akv_step_t* stp, VRowP<HG> p, const uint32_t* ss) {
  const int lane = threadIdx.x & 31, cg = lane & 7;
  VGen<HG> out;
  vgen_zero(out);
  const uint32_t um = __shfl_sync(0xFFFFFFFFu, c.nwu, row >> 5 & 7);
  const uint32_t ul = __shfl_sync(0xFFFFFFFFu, c.nwu, 8 + ((row >> 5) & 7));
  const uint64_t pol = evict_first_policy();
  uint2 mw = make_uint2(0u, 0u), lw = make_uint2(0u, 0u);
  if (valid && ((um >> (row & 31)) & 1u)) mw = ld_stream_u64(c.vb + MID + row * (D / 2) + cg * 8, pol);
  if (valid && ((ul >> (row & 31)) & 1u)) lw = ld_stream_u64(c.vb + LOW + row * (D / 2) + cg * 8, pol);
  float pvj[HG];
  uint32_t selw[HG];
#pragma unroll
  for (int jj = 0; jj < HG; ++jj) {
    pvj[jj] = p.v[jj][0];
    selw[jj] = ss[jj * 8 + (row >> 5)];
  }
  v_row_generic<G, HG, false>(out, hv, mw, lw, row, valid, c, j0, cfg, *stp, pvj, selw, nullptr);
  return out;
}

template <int G, int HG, bool TRUNC, bool EXPORT, bool UNIFORM>
__device__ __forceinline__ void v_compute(const VBatch<HG, UNIFORM>& X, const PvCtx& c, int b, int j0, const akv_cfg_t& cfg,
                                          const akv_step_t& st, float2 (&acc)[HG][8], int (&adj)[HG][3],
                                          int (&base)[HG], uint32_t tkm, uint32_t tf) {
  const int lane = threadIdx.x & 31, r4 = lane >> 3, cg = lane & 7;
  constexpr bool aligned = !UNIFORM;
  const int uni = TRUNC ? 16 : cfg.force_tier;
  const int ch = b >> 1, sh16 = 16 * (b & 1);
  const int nvalid = min(max(c.rows - 16 * b, 0), 16);
  const uint32_t vmask16 = nvalid >= 16 ? 0xFFFFu : ((1u << nvalid) - 1u);
  const uint32_t um = __shfl_sync(0xFFFFFFFFu, c.nwu, ch);
  // p of this lane's 4 rows per head; the selection (D6) and the page end fold into p = 0
  VRowP<HG> p;
#pragma unroll
  for (int jj = 0; jj < HG; ++jj) {
    const uint32_t selb = aligned ? ((X.sel[jj] >> sh16) & vmask16) : 0u;
    base[jj] += nvalid - __popc(selb);  // rows counted at T8 (aligned) / the uniform tier
#pragma unroll
    for (int i = 0; i < 4; ++i) {
      const int rr = 4 * i + r4;
      const float pv = __shfl_sync(0xFFFFFFFFu, X.p[jj], rr);
      p.v[jj][i] = ((selb >> rr) & 1u) || rr >= nvalid ? 0.f : pv;
    }
  }
  uint8_t* vt = nullptr;
  if (EXPORT && st.v_tiers) vt = st.v_tiers + ((size_t)c.u * G * c.cap + (size_t)c.pg * P + 16 * b) * D + cg * 16;

  if (UNIFORM) {
    // forced / baseline tier: one mask for every valid row
    const TierMask tm = tier_mask(uni);
#pragma unroll
    for (int i = 0; i < 4; ++i) {
      uint32_t w[8];
      const uint2 mw = X.m[UNIFORM ? i : 0], lw = X.l[UNIFORM ? i : 0];
      assemble8(X.h[i].x, X.h[i].y, bsel(tm.mk, mw.x, 0x88888888u), bsel(tm.lk, lw.x, tm.lf), w);
      assemble8(X.h[i].z, X.h[i].w, bsel(tm.mk, mw.y, 0x88888888u), bsel(tm.lk, lw.y, tm.lf), w + 4);
      if (TRUNC) {
#pragma unroll
        for (int k = 0; k < 8; ++k) w[k] = (w[k] & tkm) | tf;
      }
      float2 f[8];
#pragma unroll
      for (int k = 0; k < 8; ++k) f[k] = half2_bits_to_float2(w[k]);
#pragma unroll
      for (int jj = 0; jj < HG; ++jj)
#pragma unroll
        for (int k = 0; k < 8; ++k) acc[jj][k] = ffma2_scalar(f[k], p.v[jj][i], acc[jj][k]);
      if (EXPORT && vt && 4 * i + r4 < nvalid) {
        const uint32_t cd = (uint32_t)uni * 0x01010101u;
#pragma unroll
        for (int jj = 0; jj < HG; ++jj)
          *reinterpret_cast<uint4*>(vt + (size_t)(j0 + jj) * c.cap * D + (size_t)(4 * i + r4) * D) =
              make_uint4(cd, cd, cd, cd);
      }
    }
    return;
  }
  if (((um >> sh16) & vmask16) == 0u) {
    // fast batch: every row is T8 (or p = 0) for every q-head
#pragma unroll
    for (int i = 0; i < 4; ++i) {
      uint32_t w[8];
      t8_words16(X.h[i], w);
      float2 f[8];
#pragma unroll
      for (int k = 0; k < 8; ++k) f[k] = half2_bits_to_float2(w[k]);
#pragma unroll
      for (int jj = 0; jj < HG; ++jj)
#pragma unroll
        for (int k = 0; k < 8; ++k) acc[jj][k] = ffma2_scalar(f[k], p.v[jj][i], acc[jj][k]);
      if (EXPORT && vt) {
        const int rr = 4 * i + r4;
        if (rr < nvalid) {
#pragma unroll
          for (int jj = 0; jj < HG; ++jj) {
            const bool sel = (X.sel[jj] >> (sh16 + rr)) & 1u;
            const uint32_t cd = sel ? 0x10101010u : 0x08080808u;
            *reinterpret_cast<uint4*>(vt + (size_t)(j0 + jj) * c.cap * D + (size_t)rr * D) = make_uint4(cd, cd, cd, cd);
          }
        }
      }
    }
    return;
  }
  if constexpr (!UNIFORM) {
    // quads (4 rows) with no row in the fetch plan take the T8 path inline; the rest go
    // through the out-of-line per-element rule
    uint32_t gq = 0u;
#pragma unroll
    for (int i = 0; i < 4; ++i)
      if ((um >> (sh16 + 4 * i)) & 0xFu & (vmask16 >> (4 * i))) gq |= 1u << i;
#pragma unroll
    for (int i = 0; i < 4; ++i) {
      if ((gq >> i) & 1u) continue;
      uint32_t w[8];
      t8_words16(X.h[i], w);
      float2 f[8];
#pragma unroll
      for (int k = 0; k < 8; ++k) f[k] = half2_bits_to_float2(w[k]);
#pragma unroll
      for (int jj = 0; jj < HG; ++jj)
#pragma unroll
        for (int k = 0; k < 8; ++k) acc[jj][k] = ffma2_scalar(f[k], p.v[jj][i], acc[jj][k]);
      if (EXPORT && vt) {
        const int rr = 4 * i + r4;
        if (rr < nvalid) {
#pragma unroll
          for (int jj = 0; jj < HG; ++jj) {
            const bool sel = (X.sel[jj] >> (sh16 + rr)) & 1u;
            const uint32_t cd = sel ? 0x10101010u : 0x08080808u;
            *reinterpret_cast<uint4*>(vt + (size_t)(j0 + jj) * c.cap * D + (size_t)rr * D) = make_uint4(cd, cd, cd, cd);
          }
        }
      }
    }
    if (!gq) return;
    const VGen<HG> gen = v_generic_aligned<G, HG, EXPORT>(X, c, b, j0, cfg, &st, p, um, gq);
#pragma unroll
    for (int jj = 0; jj < HG; ++jj) {
#pragma unroll
      for (int k = 0; k < 8; ++k) {
        acc[jj][k].x += gen.acc[jj][k].x;
        acc[jj][k].y += gen.acc[jj][k].y;
      }
      adj[jj][0] += gen.adj[jj][0];
      adj[jj][1] += gen.adj[jj][1];
      adj[jj][2] += gen.adj[jj][2];
    }
  }
}

// ---------------------------------------------------------------------------
// pv v3: per-warp TMA ring.  Every warp streams its own (unit, page, head-pass)
// items through a private NS-slot shared-memory ring: lane 0 issues one
// cp.async.bulk per 64-row stage of head rows (8 KB; uniform tiers add the
// stage's mid / low rows) plus the stage's p_t and selection words, completing
// on the slot's mbarrier; the warp computes from shared memory with the same
// row code as the register-pipelined kernel.  In-flight data lives in shared
// memory (NS-1 stages ahead), not registers.
// ---------------------------------------------------------------------------
template <int G, bool UNIFORM>
struct Pv3Shape {
  static constexpr int HG = G < 4 ? G : 4;  // q-heads per pass (accumulator budget); passes re-read the page from L2
  static constexpr int NPASS = G / HG;
#ifndef AKV_PV_ROWS
#define AKV_PV_ROWS 64
#endif
  static constexpr int ROWS = UNIFORM ? 32 : AKV_PV_ROWS;        // rows per stage
  static constexpr int HEAD = ROWS * D;                          // head bytes per stage
  static constexpr int NIB = UNIFORM ? ROWS * (D / 2) : 0;       // mid (= low) bytes per stage
  static constexpr int SLOT = HEAD + 2 * NIB;                    // 8 KB
  // per-page metadata (issued with the page's first stage): p[HG][P], sel[HG][8], need[G][2][8]
  static constexpr int M_P = 0, M_SEL = HG * P * 4, M_NEED = M_SEL + HG * 32;
  static constexpr int META = M_NEED + G * 64;
#ifndef AKV_PV_NS
#define AKV_PV_NS 2
#endif
  static constexpr int NS = UNIFORM ? 2 : AKV_PV_NS;  // stages per warp ring (NS-1 in flight while one is computed)
  static constexpr int WARPS = 4;
  static constexpr int PER_WARP = (NS * SLOT + 2 * META + NS * 8 + 127) & ~127;  // bulk-copy destinations stay 16 B aligned
  static constexpr int SMEM = WARPS * PER_WARP;
  static constexpr int MINB = G == 1 ? 3 : 2;
};

struct PvCursor {
  long long item;     // (unit * npg + page) * npass + pass
  int sub;            // stage within the page
  int u, pg, pass, rows, nsub, npage;  // npage: pages started by this cursor (meta buffer parity)
  size_t pid;
  UnitPages up;
};

// (unit, page, pass) advanced incrementally (no 64-bit division per page); the pages past
// a unit's length are skipped as a block.
template <int ROWS>
__device__ __forceinline__ bool pv_cursor_seek(PvCursor& c, long long i1, const akv_store_t& s, int npg_max,
                                               int npass) {
  while (c.item < i1) {
    if (c.u != c.up.u) unit_pages_fetch(c.up, s, c.u);
    if (c.pg * P >= c.up.n) {
      c.item += (long long)(npg_max - c.pg) * npass - c.pass;
      c.pg = 0;
      c.pass = 0;
      ++c.u;
      continue;
    }
    c.rows = min(c.up.n - c.pg * P, P);
    c.nsub = (c.rows + ROWS - 1) / ROWS;
    c.sub = 0;
    c.pid = unit_page(c.up, s, c.pg);
    ++c.npage;
    return true;
  }
  return false;
}

template <int ROWS>
__device__ __forceinline__ bool pv_cursor_next(PvCursor& c, long long i1, const akv_store_t& s, int npg_max,
                                               int npass) {
  if (c.sub + 1 < c.nsub) {
    ++c.sub;
    return true;
  }
  ++c.item;
  if (++c.pass == npass) {
    c.pass = 0;
    if (++c.pg == npg_max) {
      c.pg = 0;
      ++c.u;
    }
  }
  return pv_cursor_seek<ROWS>(c, i1, s, npg_max, npass);
}

template <int G, bool UNIFORM>
__device__ __forceinline__ void pv3_issue(uint8_t* slot, uint8_t* meta, uint64_t* bar, const PvCursor& c,
                                          const akv_store_t& s, const akv_step_t& st, int cap) {
  using S = Pv3Shape<G, UNIFORM>;
  const uint8_t* vb = s.v_pool + c.pid * PAGE;
  const int r0 = c.sub * S::ROWS;
  const int capw = cap >> 5;
  const bool first = c.sub == 0;
  const uint32_t mbytes = first ? S::HG * P * 4 + (UNIFORM ? 0 : S::HG * 32 + G * 64) : 0;
  mbar_arrive_expect_tx(bar, S::SLOT + mbytes);
  bulk_g2s(slot, vb + r0 * D, S::HEAD, bar);
  if (UNIFORM) {
    bulk_g2s(slot + S::HEAD, vb + MID + r0 * (D / 2), S::NIB, bar);
    bulk_g2s(slot + S::HEAD + S::NIB, vb + LOW + r0 * (D / 2), S::NIB, bar);
  }
  if (first) {
#pragma unroll
    for (int jj = 0; jj < S::HG; ++jj) {
      const size_t h = (size_t)c.u * G + c.pass * S::HG + jj;
      bulk_g2s(meta + S::M_P + jj * P * 4, st.probs + h * cap + (size_t)c.pg * P, P * 4, bar);
      if (!UNIFORM) bulk_g2s(meta + S::M_SEL + jj * 32, st.sel_bits + h * capw + c.pg * 8, 32, bar);
    }
    if (!UNIFORM) {
#pragma unroll
      for (int j = 0; j < G; ++j) {
        const uint32_t* nb = st.need_bits + ((size_t)c.u * G + j) * 2 * capw + c.pg * 8;
        bulk_g2s(meta + S::M_NEED + j * 64, nb, 32, bar);
        bulk_g2s(meta + S::M_NEED + j * 64 + 32, nb + capw, 32, bar);
      }
    }
  }
}

template <int G, bool TRUNC, bool EXPORT, bool UNIFORM>
__global__ void __launch_bounds__(32 * Pv3Shape<G, UNIFORM>::WARPS, Pv3Shape<G, UNIFORM>::MINB)
    pv3_kernel(akv_store_t s, akv_cfg_t cfg, akv_step_t st, int cap, int npg_max) {
  using S = Pv3Shape<G, UNIFORM>;
  constexpr int HG = S::HG, NS = S::NS;
  extern __shared__ __align__(128) uint8_t pv3_smem[];
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int r4 = lane >> 3, cg = lane & 7;
  uint8_t* ring = pv3_smem + warp * S::PER_WARP;
  uint8_t* metab = ring + NS * S::SLOT;
  uint64_t* full = reinterpret_cast<uint64_t*>(metab + 2 * S::META);
  if (lane == 0) {
    for (int i = 0; i < NS; ++i) mbar_init(&full[i], 1);
    mbar_fence_init();
  }
  __syncwarp();
  pdl_trigger();
  pdl_wait();
  constexpr bool aligned = !UNIFORM;
  const int uni = TRUNC ? 16 : cfg.force_tier;
  uint32_t tkm = 0xFFFFFFFFu, tf = 0u;
  if (TRUNC) {
    const int kb = cfg.trunc_bits - 6;
    const uint32_t km = (0xFFFFu << (10 - kb)) & 0xFFFFu;
    const uint32_t fill = kb < 10 ? (1u << (9 - kb)) : 0u;
    tkm = km | (km << 16);
    tf = fill | (fill << 16);
  }
  const long long total = (long long)s.n_units * npg_max * S::NPASS;
  const long long nw = (long long)gridDim.x * S::WARPS, gw = (long long)blockIdx.x * S::WARPS + warp;
  const long long i0 = total * gw / nw, i1 = total * (gw + 1) / nw;

  PvCursor ic, cc;  // issue / consume cursors
  ic.item = i0;
  ic.pass = (int)(i0 % S::NPASS);
  ic.u = (int)(i0 / S::NPASS / npg_max);
  ic.pg = (int)(i0 / S::NPASS % npg_max);
  ic.up.u = -1;
  ic.up.n = 0;
  ic.npage = 0;
  bool iv = pv_cursor_seek<S::ROWS>(ic, i1, s, npg_max, S::NPASS);
  cc = ic;
  bool cv = iv;
  int kiss = 0;
  for (; kiss < NS - 1 && iv; ++kiss) {
    if (lane == 0)
      pv3_issue<G, UNIFORM>(ring + (kiss % NS) * S::SLOT, metab + (ic.npage & 1) * S::META, &full[kiss % NS], ic, s,
                            st, cap);
    iv = pv_cursor_next<S::ROWS>(ic, i1, s, npg_max, S::NPASS);
  }

  float2 acc[HG][8];
  int adj[HG][3], base[HG];
  PvCtx c;
  for (int k = 0; cv; ++k) {
    // keep NS-1 stages ahead: the slot being refilled was consumed at k-1 by this warp
    __syncwarp();
    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
    if (iv) {
      if (lane == 0)
        pv3_issue<G, UNIFORM>(ring + (kiss % NS) * S::SLOT, metab + (ic.npage & 1) * S::META, &full[kiss % NS], ic,
                              s, st, cap);
      ++kiss;
      iv = pv_cursor_next<S::ROWS>(ic, i1, s, npg_max, S::NPASS);
    }
    const int slot = k % NS;
    mbar_wait(&full[slot], (k / NS) & 1);
    const uint8_t* sd = ring + slot * S::SLOT;
    const uint8_t* md = metab + (cc.npage & 1) * S::META;
    const int j0 = cc.pass * HG;
    if (cc.sub == 0) {
      // page start: accumulators, fetch plan (union need words of every q-head) from the page metadata
#pragma unroll
      for (int jj = 0; jj < HG; ++jj) {
        adj[jj][0] = adj[jj][1] = adj[jj][2] = 0;
        base[jj] = 0;
#pragma unroll
        for (int q = 0; q < 8; ++q) acc[jj][q] = make_float2(0.f, 0.f);
      }
      c.vb = s.v_pool + cc.pid * PAGE;
      c.rows = cc.rows;
      c.pg = cc.pg;
      c.u = cc.u;
      c.cap = cap;
      uint32_t w = 0u;
      if (lane < 16) {
        const int chk = lane & 7;
        const int valid = min(max(c.rows - 32 * chk, 0), 32);
        const uint32_t vm = valid >= 32 ? 0xFFFFFFFFu : ((1u << valid) - 1u);
        if (!aligned) {
          w = (lane < 8 ? uni >= 12 : uni >= 16) ? vm : 0u;
        } else {
          const uint32_t* nw8 = reinterpret_cast<const uint32_t*>(md + S::M_NEED);
#pragma unroll
          for (int j = 0; j < G; ++j) w |= nw8[j * 16 + (lane >> 3) * 8 + chk];
          w &= vm;
        }
      }
      c.nwu = w;
      if (cc.pass == 0) {
        const int nib = warp_sum_i(__popc(w));
        if (lane == 0)
          atomicAdd(reinterpret_cast<unsigned long long*>(st.unit_bytes + (size_t)cc.u * 4 + 1),
                    (unsigned long long)c.rows * D + (unsigned long long)nib * (D / 2));
      }
    }
    const float* sp = reinterpret_cast<const float*>(md + S::M_P);
    const uint32_t* ss = reinterpret_cast<const uint32_t*>(md + S::M_SEL);
    if (!UNIFORM && cc.sub == 0 && !EXPORT) {
      // page start: fold the selection (D6) and the page end into the staged p (p = 0 there),
      // so the stage fast path below reads p without masks
      float* spw = reinterpret_cast<float*>(metab + (cc.npage & 1) * S::META + S::M_P);
#pragma unroll
      for (int jj = 0; jj < HG; ++jj)
#pragma unroll
        for (int r = lane; r < P; r += 32)
          if (r >= c.rows || ((ss[jj * 8 + (r >> 5)] >> (r & 31)) & 1u)) spw[jj * P + r] = 0.f;
      __syncwarp();
    }
    const int r0s = cc.sub * S::ROWS;
    constexpr int SW = S::ROWS / 32;  // 32-row chunks per stage
    uint32_t um_stage = 0u;
#pragma unroll
    for (int w = 0; w < SW; ++w) um_stage |= __shfl_sync(0xFFFFFFFFu, c.nwu, (r0s >> 5) + w);
    if (!UNIFORM && !EXPORT && r0s + S::ROWS <= c.rows && um_stage == 0u) {
      // stage fast path: full rows, none in the fetch plan -> every row is T8 (or p = 0)
#pragma unroll
      for (int jj = 0; jj < HG; ++jj) {
        int ns = 0;
#pragma unroll
        for (int w = 0; w < SW; ++w) ns += __popc(ss[jj * 8 + (r0s >> 5) + w]);
        base[jj] += S::ROWS - ns;
      }
#pragma unroll 4
      for (int q = 0; q < S::ROWS / 4; ++q) {
        const int rl = 4 * q + r4;
        const uint4 hv = *reinterpret_cast<const uint4*>(sd + rl * D + cg * 16);
        uint32_t w[8];
        t8_words16(hv, w);
        float2 f[8];
#pragma unroll
        for (int k = 0; k < 8; ++k) f[k] = half2_bits_to_float2(w[k]);
#pragma unroll
        for (int jj = 0; jj < HG; ++jj) {
          const float pv = sp[jj * P + r0s + rl];
#pragma unroll
          for (int k = 0; k < 8; ++k) acc[jj][k] = ffma2_scalar(f[k], pv, acc[jj][k]);
        }
      }
    } else if (!UNIFORM && !EXPORT && G >= 4) {
      // wide groups: 4-row quads; quads without rows in the fetch plan take the T8 path
      // inline (p is pre-zeroed for selected rows / the page end), the rest go out of line
      const int nvs = min(S::ROWS, c.rows - r0s);
#pragma unroll
      for (int jj = 0; jj < HG; ++jj) {
        int ns = 0;
#pragma unroll
        for (int w = 0; w < SW; ++w) {
          const int valid = min(max(nvs - 32 * w, 0), 32);
          const uint32_t vm = valid >= 32 ? 0xFFFFFFFFu : ((1u << valid) - 1u);
          ns += __popc(ss[jj * 8 + (r0s >> 5) + w] & vm);
        }
        base[jj] += nvs - ns;
      }
#pragma unroll 1
      for (int q = 0; 4 * q < nvs; ++q) {
        const int rl = 4 * q + r4, row = r0s + rl;
        const bool valid = rl < nvs;
        const int qr = r0s + 4 * q;  // first row of the quad (quads never straddle a 32-row chunk)
        const uint32_t fl = (__shfl_sync(0xFFFFFFFFu, c.nwu, qr >> 5) >> (qr & 31)) & 0xFu;
        const uint4 hv = valid ? *reinterpret_cast<const uint4*>(sd + rl * D + cg * 16) : make_uint4(0u, 0u, 0u, 0u);
        if (!fl) {
          uint32_t w[8];
          t8_words16(hv, w);
          float2 f[8];
#pragma unroll
          for (int k = 0; k < 8; ++k) f[k] = half2_bits_to_float2(w[k]);
#pragma unroll
          for (int jj = 0; jj < HG; ++jj) {
            const float pv = valid ? sp[jj * P + row] : 0.f;
#pragma unroll
            for (int k = 0; k < 8; ++k) acc[jj][k] = ffma2_scalar(f[k], pv, acc[jj][k]);
          }
        } else {
          VRowP<HG> pq;
#pragma unroll
          for (int jj = 0; jj < HG; ++jj) {
            pq.v[jj][0] = valid ? sp[jj * P + row] : 0.f;
            pq.v[jj][1] = pq.v[jj][2] = pq.v[jj][3] = 0.f;
          }
          const VGen<HG> g = v_quad_generic<G, HG>(hv, row, valid, c, j0, cfg, &st, pq, ss);
#pragma unroll
          for (int jj = 0; jj < HG; ++jj) {
#pragma unroll
            for (int k = 0; k < 8; ++k) {
              acc[jj][k].x += g.acc[jj][k].x;
              acc[jj][k].y += g.acc[jj][k].y;
            }
            adj[jj][0] += g.adj[jj][0];
            adj[jj][1] += g.adj[jj][1];
            adj[jj][2] += g.adj[jj][2];
          }
        }
      }
    } else
#pragma unroll(G == 1 ? S::ROWS / 16 : 1)
    for (int bb = 0; bb < S::ROWS / 16; ++bb) {
      const int b = cc.sub * (S::ROWS / 16) + bb;  // 16-row batch index inside the page
      if (16 * b >= c.rows) break;
      VBatch<HG, UNIFORM> X;
#pragma unroll
      for (int i = 0; i < 4; ++i) {
        const int rl = 16 * bb + 4 * i + r4;  // row inside the stage
        const bool valid = 16 * b + 4 * i + r4 < c.rows;
        X.h[i] = valid ? *reinterpret_cast<const uint4*>(sd + rl * D + cg * 16) : make_uint4(0u, 0u, 0u, 0u);
        if (UNIFORM) {
          X.m[i] = valid ? *reinterpret_cast<const uint2*>(sd + S::HEAD + rl * (D / 2) + cg * 8) : make_uint2(0u, 0u);
          X.l[i] = valid ? *reinterpret_cast<const uint2*>(sd + S::HEAD + S::NIB + rl * (D / 2) + cg * 8)
                         : make_uint2(0u, 0u);
        }
      }
#pragma unroll
      for (int jj = 0; jj < HG; ++jj) {
        const int row = 16 * b + (lane & 15);
        X.p[jj] = (lane < 16 && row < c.rows) ? sp[jj * P + row] : 0.f;
        X.sel[jj] = UNIFORM ? 0u : ss[jj * 8 + (b >> 1)];
      }
      v_compute<G, HG, TRUNC, EXPORT, UNIFORM>(X, c, b, j0, cfg, st, acc, adj, base, tkm, tf);
    }
    if (cc.sub + 1 == cc.nsub) {
      // page end: fold the four row groups, lanes 0..7 write 16 channels each; element counts
#pragma unroll
      for (int jj = 0; jj < HG; ++jj) {
#pragma unroll
        for (int q = 0; q < 8; ++q) {
          acc[jj][q].x += __shfl_xor_sync(0xFFFFFFFFu, acc[jj][q].x, 8);
          acc[jj][q].y += __shfl_xor_sync(0xFFFFFFFFu, acc[jj][q].y, 8);
          acc[jj][q].x += __shfl_xor_sync(0xFFFFFFFFu, acc[jj][q].x, 16);
          acc[jj][q].y += __shfl_xor_sync(0xFFFFFFFFu, acc[jj][q].y, 16);
        }
        const size_t h = (size_t)cc.u * G + j0 + jj;
        if (r4 == 0) {
          float4* dst = reinterpret_cast<float4*>(st.o_partial + (h * (cap / P) + cc.pg) * D + cg * 16);
#pragma unroll
          for (int q4 = 0; q4 < 4; ++q4)
            dst[q4] = make_float4(acc[jj][2 * q4].x, acc[jj][2 * q4].y, acc[jj][2 * q4 + 1].x, acc[jj][2 * q4 + 1].y);
        }
        const int a = warp_sum_i(adj[jj][0]), b1 = warp_sum_i(adj[jj][1]), c2 = warp_sum_i(adj[jj][2]);
        if (lane == 0) {
          unsigned long long* ct = reinterpret_cast<unsigned long long*>(st.counters + h * 8 + 3);
          long long t8 = a, t12 = b1, t16 = c2;
          const long long bs = (long long)base[jj] * D;
          if (aligned || uni == 8) t8 += bs;
          else if (uni == 12) t12 += bs;
          else t16 += bs;
          if (t8) atomicAdd(ct + 0, (unsigned long long)t8);
          if (t12) atomicAdd(ct + 1, (unsigned long long)t12);
          if (t16) atomicAdd(ct + 2, (unsigned long long)t16);
        }
      }
    }
    cv = pv_cursor_next<S::ROWS>(cc, i1, s, npg_max, S::NPASS);
  }
}

// o = o_est + sum over the unit's pages of o_partial, fixed order (deterministic):
// groups of four pages, then the rest.  All partials of a 32-page window are
// loaded before they are summed (one memory round trip per window).
__global__ void __launch_bounds__(128) combine_kernel(akv_store_t s, akv_cfg_t cfg, akv_step_t st) {
  pdl_trigger();
  pdl_wait();
  const int h = blockIdx.x;
  const int u = h / cfg.group;
  const int n = s.lengths[u];
  const int npg = (n + P - 1) / P;
  const float* part = st.o_partial + (size_t)h * s.max_pages * D + threadIdx.x;
  float acc = st.o_est[(size_t)h * D + threadIdx.x];
  constexpr int WIN = 32;
  for (int w0 = 0; w0 < npg; w0 += WIN) {
    float v[WIN];
#pragma unroll
    for (int i = 0; i < WIN; ++i) v[i] = w0 + i < npg ? part[(w0 + i) * D] : 0.f;
    const int m = min(npg - w0, WIN);
    int i = 0;
#pragma unroll
    for (int g = 0; g < WIN / 4; ++g)
      if (i + 4 <= m) {
        acc += ((v[4 * g] + v[4 * g + 1]) + (v[4 * g + 2] + v[4 * g + 3]));
        i += 4;
      }
#pragma unroll
    for (int r = 0; r < WIN; ++r)
      if (r >= i && r < m) acc += v[r];
  }
  st.o[(size_t)h * D + threadIdx.x] = acc;
}

template <int G, bool TRUNC, bool EXPORT, bool UNIFORM>
static void launch_pv3_t(const akv_store_t& s, const akv_cfg_t& cfg, const akv_step_t& st, int max_len,
                         cudaStream_t stream) {
  using S = Pv3Shape<G, UNIFORM>;
  const int resident = resident_ctas<pv3_kernel<G, TRUNC, EXPORT, UNIFORM>>(32 * S::WARPS, S::SMEM);
  const int cap = s.max_pages * P;
  const int npg = (max_len + P - 1) / P;
  const long long items = (long long)s.n_units * npg * S::NPASS;
  const int grid = (int)std::min<long long>(resident, std::max<long long>((items + S::WARPS - 1) / S::WARPS, 1));
  launch_pdl(PDL_PV, pv3_kernel<G, TRUNC, EXPORT, UNIFORM>, dim3(grid), dim3(32 * S::WARPS), (size_t)S::SMEM, stream, s, cfg, st, cap, npg);
}

}  // namespace akv

#include "akv_pv4.cuh"
#include "akv_pv5.cuh"
#include "akv_pv6.cuh"

namespace akv {

// AKV_PV_KERNEL=pv3 / pv4 / pv5 select the round-1 kernel / the CUDA-core ring kernel /
// the fixed-slot tensor-core kernel for A/B measurements.  Default: pv6 (variable-size
// ring, T8 stages on the tensor cores, dense stages through the SIMD element rule) for
// every aligned mode (serving and V-mask export), pv4 for the uniform-tier (forced /
// baseline) modes.
static int pv_choice() {
  static const int v = [] {
    const char* e = getenv("AKV_PV_KERNEL");
    if (e && strcmp(e, "pv3") == 0) return 3;
    if (e && strcmp(e, "pv4") == 0) return 4;
    if (e && strcmp(e, "pv5") == 0) return 5;
    return 6;
  }();
  return v;
}
static bool pv_legacy() { return pv_choice() == 3; }

template <int G>
static void launch_pv_g(const akv_store_t& s, const akv_cfg_t& cfg, const akv_step_t& st, int max_len,
                        cudaStream_t stream) {
  const bool ex = st.v_tiers != nullptr;
  if (!pv_legacy()) {
    if (cfg.trunc_bits) {
      if (ex) launch_pv4_t<G, true, true, true>(s, cfg, st, max_len, stream);
      else launch_pv4_t<G, true, false, true>(s, cfg, st, max_len, stream);
    } else if (cfg.force_tier) {
      if (ex) launch_pv4_t<G, false, true, true>(s, cfg, st, max_len, stream);
      else launch_pv4_t<G, false, false, true>(s, cfg, st, max_len, stream);
    } else if (pv_choice() == 6 && (ex ? launch_pv6_t<G, true>(s, cfg, st, max_len, stream)
                                        : launch_pv6_t<G, false>(s, cfg, st, max_len, stream))) {
    } else if (ex) {
      launch_pv4_t<G, false, true, false>(s, cfg, st, max_len, stream);
    } else if (pv_choice() == 4 || !launch_pv5_t<G>(s, cfg, st, max_len, stream)) {
      launch_pv4_t<G, false, false, false>(s, cfg, st, max_len, stream);
    }
    return;
  }
  if (cfg.trunc_bits) {
    if (ex) launch_pv3_t<G, true, true, true>(s, cfg, st, max_len, stream);
    else launch_pv3_t<G, true, false, true>(s, cfg, st, max_len, stream);
  } else if (cfg.force_tier) {
    if (ex) launch_pv3_t<G, false, true, true>(s, cfg, st, max_len, stream);
    else launch_pv3_t<G, false, false, true>(s, cfg, st, max_len, stream);
  } else {
    if (ex) launch_pv3_t<G, false, true, false>(s, cfg, st, max_len, stream);
    else launch_pv3_t<G, false, false, false>(s, cfg, st, max_len, stream);
  }
}

void launch_pv(const akv_store_t& s, const akv_cfg_t& cfg, const akv_step_t& st, int max_len, cudaStream_t stream) {
  switch (cfg.group) {
    case 1: launch_pv_g<1>(s, cfg, st, max_len, stream); break;
    case 2: launch_pv_g<2>(s, cfg, st, max_len, stream); break;
    case 4: launch_pv_g<4>(s, cfg, st, max_len, stream); break;
    case 8: launch_pv_g<8>(s, cfg, st, max_len, stream); break;
  }
}

void launch_combine(const akv_store_t& s, const akv_cfg_t& cfg, const akv_step_t& st, cudaStream_t stream) {
  launch_pdl(PDL_COMBINE, combine_kernel, dim3(s.n_units * cfg.group), dim3(D), 0, stream, s, cfg, st);
}

}  // namespace akv
