// qk8: scores_aligned for every G from a per-warp bulk-copy ring.
// Included by akv_qk.cu (shares k_rule1, fma_hh).
//
// Layout fact it exploits: a K page's head plane is channel-major [d][P], so the
// head rows of any run of consecutive channels are one contiguous block, and each
// channel's mid / low nibbles for the page are one 128 B row.  Per unit the warp
// evaluates Rule 1 once (k_rule1) and cuts the channels into RUNS: each group of
// 16 consecutive channels that is not entirely SKIP is one run when its bytes
// (16 x 256 B head rows + the 128 B nibble rows of its T12 / T16 channels) fit a
// 6 KB slot, else two runs of 8 channels.  Per (page, run) the warp's lanes issue
// one cp.async.bulk (UBLKCP) of the run's head rows plus one 128 B bulk copy per
// nibble row the run's tiers need, into the next slot of a private NS-slot ring
// completing on the slot's mbarrier; the ring runs NS-1 stages ahead of the math,
// continuously across the pages of a unit and across units (the per-unit state is
// double-buffered, so a unit change never drains the ring).
//
// Math: lane l owns tokens 8l .. 8l+7 of the page, so a channel is one LDS.64 of
// head bytes (+ one LDS.32 per nibble row) per lane, rebuilt to fp16 words with
// PRMT / LOP3 (midpoint fill, HB:160-179), masked down to each q-head's tier, and
// accumulated with the mixed-precision FHFMA (exact fp16 products, fp32 sums,
// SPEC.md:318,379; channel order fixed, so results do not depend on the grid).
// Lanes hold complete token sums: the page finish (x 1/sqrt(d), SPEC.md:381;
// scores; per-32-token (max, sum exp)) needs no cross-lane fold beyond the chunk.

namespace akv {

constexpr int Q8_SLOT = 6144;
constexpr int Q8_MAXRUN = 16;  // 8 groups of 16 channels, each one or two runs

template <int G>
struct alignas(16) Qk8Unit {
  uint16_t q[D][G];        // channel c, head j: q_jc as fp16 bits, 0 where head j reads nothing (SKIP)
  uint32_t hc[D];          // channel c: bits 2j..2j+1 = head j's tier index (0 SKIP, 1 T8, 2 T12, 3 T16);
                           //            bits 16..23 = union code
  uint32_t noff[D];        // channel c: offset of its mid row | offset of its low row << 16 in the slot
                           //            (0 = the head rows: a harmless address, the word is not used)
  uint32_t copies[2 * D];  // the unit's nibble copies: src / 128 (bits 0..8, within the page) |
                           //   dst / 128 (bits 9..15, within the slot) | 128 B rows (bits 16..20)
  uint16_t run_cp[Q8_MAXRUN + 1];  // run r's copies: [run_cp[r], run_cp[r+1])
  uint16_t run_bytes[Q8_MAXRUN];
  uint8_t run_c0[Q8_MAXRUN], run_c1[Q8_MAXRUN];
  int nrun, unit, n, pad;
};

template <int G>
struct Qk8Shape {
  static constexpr int WARPS = 4;
  static constexpr int NS = 3;
  static constexpr int UNIT = (sizeof(Qk8Unit<G>) + 127) & ~127;
  static constexpr int PER_WARP = NS * Q8_SLOT + 2 * UNIT + 128;  // ring | 2 unit states | mbarriers
  static constexpr int SMEM = WARPS * PER_WARP;
  static constexpr int MINB = 2;
};

__device__ __forceinline__ uint32_t tier_index(int code) { return code == 0 ? 0u : (uint32_t)((code - 4) >> 2); }

// Rule 1 for unit u (k_rule1), the unit's runs and their copy lists, into U.
template <int G, bool TRUNC>
__device__ void q8_prologue(Qk8Unit<G>& U, const akv_store_t& s, const akv_cfg_t& cfg, const akv_step_t& st, int u,
                            int n, bool book) {
  const int lane = threadIdx.x & 31;
  uint32_t qw[G][4];
  int code[G][4], ucode[4];
  k_rule1<G, TRUNC>(s, cfg, st, u, n, book, qw, code, ucode);
#pragma unroll
  for (int k = 0; k < 4; ++k) {  // lane l owns channels l + 32k
    const int c = lane + 32 * k;
    uint32_t hc = (uint32_t)ucode[k] << 16;
#pragma unroll
    for (int j = 0; j < G; ++j) {
      U.q[c][j] = code[j][k] ? (uint16_t)(qw[j][k] & 0xFFFFu) : (uint16_t)0;
      hc |= tier_index(code[j][k]) << (2 * j);
    }
    U.hc[c] = hc;
  }
  __syncwarp();
  // Runs.  Lane 2p + h (p < 8) looks at channels [16p + 8h, 16p + 8h + 8); a group of 16 is
  // one run if its head rows + nibble rows fit a slot (head rows of SKIP channels inside a
  // run are copied too), else two runs of 8 (an all-SKIP half is dropped).
  const int p = (lane >> 1) & 7, hlf = lane & 1;
  const bool act = lane < 16;
  uint32_t uc8[8];
  int any8 = 0, nm8 = 0, nl8 = 0;
#pragma unroll
  for (int i = 0; i < 8; ++i) {
    const uint32_t uc = act ? (U.hc[16 * p + 8 * hlf + i] >> 16) & 0xFFu : 0u;
    uc8[i] = uc;
    any8 |= uc != 0;
    nm8 += uc >= 12;
    nl8 += uc == 16;
  }
  const int any_o = __shfl_xor_sync(0xFFFFFFFFu, any8, 1);
  const int nm_o = __shfl_xor_sync(0xFFFFFFFFu, nm8, 1), nl_o = __shfl_xor_sync(0xFFFFFFFFu, nl8, 1);
  const bool whole = (any8 || any_o) && 16 * P + (nm8 + nm_o + nl8 + nl_o) * (P / 2) <= Q8_SLOT;
  const bool mine = whole ? hlf == 0 : any8 != 0;
  // slot layout of a run: [head rows][mid rows of its T12/T16 channels][low rows of its T16 channels]
  // (channel order inside each block, so consecutive channels' rows coalesce into one copy)
  int head = whole ? 16 * P : 8 * P;
  int mid0 = head + (whole && hlf ? nm_o : 0) * (P / 2);
  int nmr = whole ? nm8 + nm_o : nm8;
  int low0 = head + nmr * (P / 2) + (whole && hlf ? nl_o : 0) * (P / 2);
  // copies of my half: maximal runs of consecutive channels needing the mid (low) row
  int ncp = 0;
  {
    int mo = mid0, lo = low0;
#pragma unroll
    for (int i = 0; i < 8; ++i) {
      const int c = 16 * p + 8 * hlf + i;
      const bool f = uc8[i] >= 12, t = uc8[i] == 16;
      if (act) U.noff[c] = (f ? (uint32_t)mo : 0u) | ((t ? (uint32_t)lo : 0u) << 16);
      const bool fs = f && (i == 0 || uc8[i - 1] < 12), ts = t && (i == 0 || uc8[i - 1] != 16);
      ncp += fs + ts;
      mo += f ? P / 2 : 0;
      lo += t ? P / 2 : 0;
    }
  }
  // the copy list is laid out run by run (a whole group's two halves are adjacent)
  int before = ncp;
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    const int y = __shfl_up_sync(0xFFFFFFFFu, before, o);
    if (lane >= o) before += y;
  }
  before -= ncp;  // exclusive prefix over lanes
  if (act) {
    int k = before, mo = mid0, lo = low0;
    // mid copies, then low copies (dst blocks are separate)
#pragma unroll
    for (int pass = 0; pass < 2; ++pass) {
      int start = -1, dst = 0;
#pragma unroll
      for (int i = 0; i <= 8; ++i) {
        const bool need = i < 8 && (pass ? uc8[i] == 16 : uc8[i] >= 12);
        const int c = 16 * p + 8 * hlf + i;
        if (need && start < 0) {
          start = c;
          dst = pass ? lo : mo;
        }
        if (!need && start >= 0) {
          const int src = (pass ? LOW : MID) + start * (P / 2);
          U.copies[k++] = (uint32_t)(src >> 7) | ((uint32_t)(dst >> 7) << 9) | ((uint32_t)(c - start) << 16);
          start = -1;
        }
        if (need) {
          if (pass) lo += P / 2;
          else mo += P / 2;
        }
      }
    }
  }
  const unsigned bm = __ballot_sync(0xFFFFFFFFu, mine);
  const int slot = __popc(bm & ((1u << lane) - 1u));
  // a whole group's run spans both halves' copies: [before(2p), before(2p) + ncp(2p) + ncp(2p+1))
  const int ncp_o = __shfl_xor_sync(0xFFFFFFFFu, ncp, 1);
  if (mine) {
    U.run_c0[slot] = (uint8_t)(whole ? 16 * p : 16 * p + 8 * hlf);
    U.run_c1[slot] = (uint8_t)(whole ? 16 * p + 16 : 16 * p + 8 * hlf + 8);
    U.run_bytes[slot] = (uint16_t)(head + (nmr + (whole ? nl8 + nl_o : nl8)) * (P / 2));
    U.run_cp[slot] = (uint16_t)before;
    U.run_cp[slot + 1] = (uint16_t)(before + ncp + (whole ? ncp_o : 0));
  }
  int nrun = __popc(bm);
  __syncwarp();
  if (nrun == 0) {  // every channel SKIP for every head: one run over channels 0..7 (q = 0 everywhere)
    if (lane == 0) {
      U.run_c0[0] = 0;
      U.run_c1[0] = 8;
      U.run_bytes[0] = 8 * P;
      U.run_cp[0] = U.run_cp[1] = 0;
    }
    nrun = 1;
  }
  if (lane == 0) {
    U.nrun = nrun;
    U.unit = u;
    U.n = n;
  }
  __syncwarp();
}

// Issue run r of page base into slot dst: one copy of the run's head rows, then the run's
// nibble copies, all from lane 0 (bulk-copy operands are warp-uniform registers).
template <int G>
__device__ __forceinline__ void q8_issue(uint8_t* dst, uint64_t* bar, const Qk8Unit<G>& U, int r, const uint8_t* base) {
  if ((threadIdx.x & 31) == 0) {
    const int c0 = U.run_c0[r], c1 = U.run_c1[r];
    mbar_arrive_expect_tx(bar, U.run_bytes[r]);
    bulk_g2s(dst, base + c0 * P, (uint32_t)(c1 - c0) * P, bar);
    const int k1 = U.run_cp[r + 1];
    for (int k = U.run_cp[r]; k < k1; ++k) {
      const uint32_t e = U.copies[k];
      bulk_g2s(dst + ((e >> 9) & 0x7F) * 128, base + (e & 0x1FF) * 128, (e >> 16) * 128, bar);
    }
  }
}

// Four channels c .. c+3 of the run in slot sd (branch-free: a T8 channel is rebuilt with
// the T8 fill words, mid 0x8 / low 0x0 nibbles; T12 with low 0x8, HB:160-179).
template <int G, bool TRUNC>
__device__ __forceinline__ void q8_four(const uint8_t* sd, const Qk8Unit<G>& U, int c, int c0, float (&acc)[G][8],
                                        uint32_t tkm, uint32_t tf) {
  const int lane = threadIdx.x & 31;
  const uint4 hc4 = *reinterpret_cast<const uint4*>(&U.hc[c]);
  const uint4 no4 = *reinterpret_cast<const uint4*>(&U.noff[c]);
  const uint32_t hcv[4] = {hc4.x, hc4.y, hc4.z, hc4.w};
  const uint32_t nov[4] = {no4.x, no4.y, no4.z, no4.w};
  uint32_t qv[4][(G + 1) / 2];  // q pairs of the 4 channels
  if constexpr (G == 1) {
    const uint2 t = *reinterpret_cast<const uint2*>(&U.q[c][0]);
    qv[0][0] = t.x & 0xFFFFu;
    qv[1][0] = t.x >> 16;
    qv[2][0] = t.y & 0xFFFFu;
    qv[3][0] = t.y >> 16;
  } else {
#pragma unroll
    for (int i = 0; i < 4; ++i) {
      if constexpr (G == 2) {
        qv[i][0] = *reinterpret_cast<const uint32_t*>(&U.q[c + i][0]);
      } else if constexpr (G == 4) {
        const uint2 t = *reinterpret_cast<const uint2*>(&U.q[c + i][0]);
        qv[i][0] = t.x;
        qv[i][1] = t.y;
      } else {
        const uint4 t = *reinterpret_cast<const uint4*>(&U.q[c + i][0]);
        qv[i][0] = t.x;
        qv[i][1] = t.y;
        qv[i][2] = t.z;
        qv[i][3] = t.w;
      }
    }
  }
  uint2 hv[4];
  uint32_t mw[4], lw[4];
#pragma unroll
  for (int i = 0; i < 4; ++i) {
    hv[i] = *reinterpret_cast<const uint2*>(sd + (c - c0 + i) * P + lane * 8);
    mw[i] = *reinterpret_cast<const uint32_t*>(sd + (nov[i] & 0xFFFFu) + lane * 4);
    lw[i] = *reinterpret_cast<const uint32_t*>(sd + (nov[i] >> 16) + lane * 4);
  }
#pragma unroll
  for (int i = 0; i < 4; ++i) {
    const uint32_t uc = (hcv[i] >> 16) & 0xFFu;
    const uint32_t mid = uc >= 12 ? mw[i] : 0x88888888u;
    const uint32_t low = uc == 16 ? lw[i] : (uc == 12 ? 0x88888888u : 0u);
    uint32_t w[4];
    assemble8(hv[i].x, hv[i].y, mid, low, w);
    if (TRUNC) {
#pragma unroll
      for (int k = 0; k < 4; ++k) w[k] = (w[k] & tkm) | tf;
    }
    const uint32_t uti = tier_index((int)uc);
#pragma unroll
    for (int j = 0; j < G; ++j) {
      uint32_t wj[4];
      const uint32_t tj = (hcv[i] >> (2 * j)) & 3u;
      if (G > 1 && tj != uti && tj != 0) {  // head j reads a lower tier than the union: mask + fill
        const uint32_t km = tj == 2 ? 0xFFF0FFF0u : 0xFF00FF00u, kf = tj == 2 ? 0x00080008u : 0x00800080u;
#pragma unroll
        for (int k = 0; k < 4; ++k) wj[k] = (w[k] & km) | kf;
      } else {
#pragma unroll
        for (int k = 0; k < 4; ++k) wj[k] = w[k];
      }
      const uint32_t qp = (j & 1) ? (qv[i][j >> 1] >> 16) : qv[i][j >> 1];  // 0 for SKIP heads / channels
#pragma unroll
      for (int k = 0; k < 4; ++k) {
        acc[j][2 * k] = fma_hh<0, 0>(wj[k], qp, acc[j][2 * k]);
        acc[j][2 * k + 1] = fma_hh<1, 0>(wj[k], qp, acc[j][2 * k + 1]);
      }
    }
  }
}

// Scale, store and summarise this lane's 8 tokens (8l .. 8l+7 of the page) for one head.
__device__ __forceinline__ void q8_finish(const float (&raw)[8], int tok0, int n, float* scores_h, float* stats_h,
                                          float isd) {
  const int lane = threadIdx.x & 31;
  const int nv = min(max(n - tok0, 0), 8);
  float sv[8];
  float m = -INFINITY;
#pragma unroll
  for (int e = 0; e < 8; ++e) {
    sv[e] = raw[e] * isd;
    if (e < nv) m = fmaxf(m, sv[e]);
  }
  m = fmaxf(m, __shfl_xor_sync(0xFFFFFFFFu, m, 1));
  m = fmaxf(m, __shfl_xor_sync(0xFFFFFFFFu, m, 2));
  float l = 0.f;  // MUFU exp2 of (s - m) log2(e): the max term is exactly 1 (see k5_finish)
#pragma unroll
  for (int e = 0; e < 8; ++e)
    if (e < nv) {
      float ex;
      asm("ex2.approx.ftz.f32 %0, %1;" : "=f"(ex) : "f"((sv[e] - m) * 1.4426950408889634f));
      l += ex;
    }
  l += __shfl_xor_sync(0xFFFFFFFFu, l, 1);
  l += __shfl_xor_sync(0xFFFFFFFFu, l, 2);
  float* out = scores_h + tok0;
  if (nv == 8) {
    reinterpret_cast<float4*>(out)[0] = make_float4(sv[0], sv[1], sv[2], sv[3]);
    reinterpret_cast<float4*>(out)[1] = make_float4(sv[4], sv[5], sv[6], sv[7]);
  } else {
#pragma unroll
    for (int e = 0; e < 8; ++e)
      if (e < nv) out[e] = sv[e];
  }
  if ((lane & 3) == 0 && tok0 < n) {  // lanes 4c own 32-token chunk c
    float* ps = stats_h + (tok0 >> 5) * 2;
    ps[0] = m;
    ps[1] = l;
  }
}

struct Q8Cur {
  long long i;  // item = unit * npg + page
  int u, pg, r, seq;
  UnitPages up;
};

template <int G, bool TRUNC>
__global__ void __launch_bounds__(32 * Qk8Shape<G>::WARPS, Qk8Shape<G>::MINB)
    qk8_kernel(akv_store_t s, akv_cfg_t cfg, akv_step_t st, int cap, float isd, int npg_max) {
  using S = Qk8Shape<G>;
  constexpr int NS = S::NS;
  extern __shared__ __align__(128) uint8_t q8_smem[];
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  uint8_t* ring = q8_smem + warp * S::PER_WARP;
  Qk8Unit<G>* ust = reinterpret_cast<Qk8Unit<G>*>(ring + NS * Q8_SLOT);  // [2]
  uint64_t* full = reinterpret_cast<uint64_t*>(ring + NS * Q8_SLOT + 2 * S::UNIT);
  if (lane == 0) {
    for (int i = 0; i < NS; ++i) mbar_init(&full[i], 1);
    mbar_fence_init();
  }
  __syncwarp();
  pdl_trigger();
  pdl_wait();
  uint32_t tkm = 0xFFFFFFFFu, tf = 0u;
  if (TRUNC) {
    const int kb = cfg.trunc_bits - 6;
    const uint32_t km = (0xFFFFu << (10 - kb)) & 0xFFFFu;
    const uint32_t fill = kb < 10 ? (1u << (9 - kb)) : 0u;
    tkm = km | (km << 16);
    tf = fill | (fill << 16);
  }
  const long long total = (long long)s.n_units * npg_max;
  const long long nw = (long long)gridDim.x * S::WARPS, gw = (long long)blockIdx.x * S::WARPS + warp;
  const long long i0 = total * gw / nw, i1 = total * (gw + 1) / nw;
  const int cap_chunks = s.max_pages * (P / 32);

  // first valid item at or after c (pages past a unit's length are skipped as a block)
  auto seek = [&](Q8Cur& c) {
    while (c.i < i1) {
      if (c.u != c.up.u) unit_pages_fetch(c.up, s, c.u);
      if (c.pg * P < c.up.n) return;
      c.i += npg_max - c.pg;
      c.pg = 0;
      ++c.u;
    }
  };
  Q8Cur ic;
  ic.i = i0;
  ic.u = (int)(i0 / npg_max);
  ic.pg = (int)(i0 % npg_max);
  ic.r = 0;
  ic.seq = 0;
  ic.up.u = -1;
  ic.up.n = 0;
  seek(ic);
  if (ic.i >= i1) return;
  q8_prologue<G, TRUNC>(ust[0], s, cfg, st, ic.u, ic.up.n, ic.pg == 0);
  Q8Cur cc = ic;
  const uint8_t* ibase = s.k_pool + unit_page(ic.up, s, ic.pg) * PAGE;
  bool ivalid = true, iblocked = false;

  // advance the issue cursor by one stage; entering a new unit builds its state in the
  // other buffer unless the compute cursor still uses that buffer (then block)
  auto iadvance = [&]() {
    if (++ic.r < ust[ic.seq & 1].nrun) return;
    ic.r = 0;
    const int pu = ic.u;
    ++ic.i;
    if (++ic.pg == npg_max) {
      ic.pg = 0;
      ++ic.u;
    }
    seek(ic);
    if (ic.i >= i1) {
      ivalid = false;
      return;
    }
    if (ic.u != pu) {
      if (cc.seq != ic.seq) {  // the other buffer is still in use: wait for the compute cursor
        iblocked = true;
        return;
      }
      ++ic.seq;
      q8_prologue<G, TRUNC>(ust[ic.seq & 1], s, cfg, st, ic.u, ic.up.n, ic.pg == 0);
    }
    ibase = s.k_pool + unit_page(ic.up, s, ic.pg) * PAGE;
  };
  auto try_unblock = [&]() {
    if (iblocked && cc.seq == ic.seq) {
      iblocked = false;
      ++ic.seq;
      q8_prologue<G, TRUNC>(ust[ic.seq & 1], s, cfg, st, ic.u, ic.up.n, ic.pg == 0);
      ibase = s.k_pool + unit_page(ic.up, s, ic.pg) * PAGE;
    }
  };

  int kiss = 0;
  for (; kiss < NS - 1 && ivalid && !iblocked; ++kiss) {
    q8_issue<G>(ring + (kiss % NS) * Q8_SLOT, &full[kiss % NS], ust[ic.seq & 1], ic.r, ibase);
    iadvance();
  }

  float acc[G][8];
#pragma unroll
  for (int j = 0; j < G; ++j)
#pragma unroll
    for (int e = 0; e < 8; ++e) acc[j][e] = 0.f;

  for (int k = 0;; ++k) {
    // refill the slot computed in the previous iteration (every lane is past it)
    __syncwarp();
    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
    try_unblock();
    if (ivalid && !iblocked) {
      q8_issue<G>(ring + (kiss % NS) * Q8_SLOT, &full[kiss % NS], ust[ic.seq & 1], ic.r, ibase);
      ++kiss;
      iadvance();
    }
    const int slot = k % NS;
    mbar_wait(&full[slot], (uint32_t)(k / NS) & 1u);
    const uint8_t* sd = ring + slot * Q8_SLOT;
    const Qk8Unit<G>& U = ust[cc.seq & 1];
    const int c0 = U.run_c0[cc.r], c1 = U.run_c1[cc.r];
#pragma unroll 1
    for (int c = c0; c < c1; c += 4) q8_four<G, TRUNC>(sd, U, c, c0, acc, tkm, tf);
    if (cc.r + 1 < U.nrun) {
      ++cc.r;
      continue;
    }
    // page done: lane l holds tokens 8l .. 8l+7 of every head
    const int u = cc.u, pg = cc.pg, n = cc.up.n;
#pragma unroll
    for (int j = 0; j < G; ++j) {
      const size_t h = (size_t)u * G + j;
      q8_finish(acc[j], pg * P + 8 * lane, n, st.scores + h * cap, st.page_stats + h * cap_chunks * 2, isd);
#pragma unroll
      for (int e = 0; e < 8; ++e) acc[j][e] = 0.f;
    }
    cc.r = 0;
    ++cc.i;
    if (++cc.pg == npg_max) {
      cc.pg = 0;
      ++cc.u;
    }
    const int pu = cc.u;
    seek(cc);
    if (cc.i >= i1) break;
    if (cc.u != u) ++cc.seq;
    (void)pu;
  }
}

template <int G, bool TRUNC>
static void launch_qk8_t(const akv_store_t& s, const akv_cfg_t& cfg, const akv_step_t& st, int max_len,
                         cudaStream_t stream) {
  using S = Qk8Shape<G>;
  const int resident = resident_ctas<qk8_kernel<G, TRUNC>>(32 * S::WARPS, S::SMEM);
  const int cap = s.max_pages * P;
  const int npg = (max_len + P - 1) / P;
  const long long items = (long long)s.n_units * npg;
  const int grid = (int)std::min<long long>(resident, std::max<long long>((items + S::WARPS - 1) / S::WARPS, 1));
  const float isd = (float)(1.0 / 11.313708498984761);  // 1/sqrt(128)
  launch_pdl(PDL_QK, qk8_kernel<G, TRUNC>, dim3(grid), dim3(32 * S::WARPS), (size_t)S::SMEM, stream, s, cfg, st, cap, isd, npg);
}

}  // namespace akv
