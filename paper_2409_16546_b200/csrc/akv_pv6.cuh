// pv6: output_aligned for the aligned modes (element and row strategy,
// with or without the V-mask export).  Included by akv_pv.cu after akv_pv5.cuh (shares
// PvCursor, the V head-row tensor map and the mma helpers).
//
// Per-warp variable-size ring.  A stage is 32 token rows of one page:
//   [V head rows, 4 KB, TMA 2-D box with 128 B swizzle]
//   [the stage's mid nibble rows in the union fetch plan, 64 B each, compacted]
//   [the stage's low nibble rows in the union fetch plan, compacted]
// rounded up to 1 KB, so a stage is 4 KB when no row of it is in the plan (SPEC
// generator at scale 2^U[-4,4]) and 8 KB when every row is (paper-like scales).  The ring
// (16 KB per warp) holds up to four sparse stages or two dense ones: the bytes in flight
// follow the bytes the plan reads.  The issuer knows a stage's plan before it copies it:
// the page's selection / fetch-plan words ([3][G][8] words: sel, need-mid, need-low, from
// akv_softmax_select) are bulk-copied one page ahead into a 3-slot page-meta ring.
// Nibble rows are copied as maximal runs of consecutive plan rows, one bulk copy per run,
// issued by the lane at the run's first row.
//
// Compute per stage:
//  * no row in the plan (and no export): the T8 words of all 32 rows go through the
//    tensor cores exactly as in pv5 (mma.sync m16n8k16, V as A via ldmatrix.trans, p as
//    hi/lo fp16 pairs in B, 4 q-heads per n-tile); selected rows and rows past the length
//    carry p = 0;
//  * otherwise the dense path: lane = (row half, 8 channels), every row through the
//    per-element rule in 16-bit SIMD form.  For one row and head, with ep = floor(log2 p_t)
//    and g_c = 17 + target_c - margin:
//        keep mid  <=>  max(bexp, 1) + ep > g_c   <=>  max(bexp, 1) >= G1_c - ep,  G1_c = g_c + 1
//        keep low  <=>  max(bexp, 1) >= G1_c - ep + 4                              (D4)
//    max(bexp, 1) of an element pair is ((|w| max 0x0400) >> 10) per half (VIMNMX, SHF, LOP);
//    the thresholds are min(max(G1 + (-ep), 0), 31) per half (one VIADDMNMX.RELU each), and
//    the compares are HSET2.GE on the small integers as fp16 patterns (positive subnormals
//    order like integers), giving 0xFFFF / 0 half masks.  The word is then
//    bsel(mm, bsel(ml, w, T12 word), T8 word) (midpoint fill, HB:160-179) and the element
//    counts are the masks summed with VIADDMNMX (a mask half is -1).  Unknown targets
//    (o_est_r == 0) carry G1 = -16384: always kept, p_t == 0 included; p_t == 0
//    with a known target and rows outside the head's plan use -ep = 16000: never kept (D5).
//    The row strategy (D7) takes the row tier from the need words.  Contributions are
//    folded into the mma accumulators through shared memory.
// Per-page partials go to o_partial; akv_combine adds o_est and the partials in a fixed
// order (deterministic).

namespace akv {

template <int G>
struct Pv6Shape {
  static constexpr int R = 32;                    // rows per stage
  static constexpr int HEAD = R * D;              // 4 KB
  // G <= 4: the rule rows accumulate into page-persistent registers (one fold per page);
  // G = 8: passes of 2 q-heads folded per stage (register budget)
  // (G = 4 keeps 12 warps / SM with a 12 KB ring and per-stage folds: measured faster at c3
  // than 8 warps with page accumulators, 85.9 vs 91.3 us)
  static constexpr bool PAGEACC = G <= 2;
  static constexpr int HC = PAGEACC ? G : 2;      // q-heads per rule pass
  static constexpr int WARPS = G == 2 ? 5 : 4;
  static constexpr int MINB = (G == 1 || G == 4) ? 3 : 2;  // warps / SM: G = 1, 4: 12, G = 2: 10, G = 8: 8
  static constexpr int RING = G == 4 ? 12288 : 16384;       // per-warp stage ring
  static constexpr int MAXS = RING / HEAD;        // stages in flight at most
  static constexpr int PB = G * R * 4;            // p block [G][R] per stage
  static constexpr int NMETA = 4;                 // page-meta slots
  static constexpr int SEL_B = (32 * G + 127) & ~127;   // sel [G][8] words (TMA box 8 x G)
  static constexpr int NEED_B = (64 * G + 127) & ~127;  // need [G][mid, low][8] words (TMA box 8 x 2G)
  static constexpr int META = SEL_B + NEED_B;
  static constexpr int SCR = HC * D * 4;         // fold scratch of one dense pass
  static constexpr int OFF_PB = 0;
  static constexpr int OFF_META = OFF_PB + MAXS * PB;
  static constexpr int OFF_G1 = OFF_META + NMETA * META;  // [G][64] threshold words of the current unit
  static constexpr int OFF_SCR = OFF_G1 + G * 256;
  static constexpr int OFF_NE = OFF_SCR + SCR;            // [G][R] packed -ep words of the stage's rows
  static constexpr int OFF_BAR = OFF_NE + G * R * 4;
  static constexpr int DENSE_MIN = 20;
  static constexpr bool USE_DENSE = G <= 2;               // G >= 4: registers (the SPARSE path takes every plan row)
  static constexpr int RULE_UNROLL = G >= 2 ? 1 : 2;     // rule-loop unroll (register budget)                    // plan rows from which a full stage goes DENSE
  static constexpr int MISC = (OFF_BAR + (MAXS + NMETA) * 8 + 127) & ~127;
  static constexpr int SMEM = WARPS * (RING + MISC) + 1024;  // + 1 KB alignment slack
};

// bytes of a stage with nm mid and nl low nibble rows, rounded to 1 KB (the next stage's
// head rows must stay 1 KB aligned for the 128 B swizzle)
__device__ __forceinline__ int pv6_stage_bytes(int nm, int nl) { return (4096 + 64 * (nm + nl) + 1023) & ~1023; }

__device__ __forceinline__ uint32_t hset2_ge(uint32_t a, uint32_t b) {
  uint32_t d;
  asm("set.ge.u32.f16x2 %0, %1, %2;" : "=r"(d) : "r"(a), "r"(b));
  return d;
}

// maximal runs of set bits: the lane at a run's first bit copies the run
__device__ __forceinline__ void pv6_copy_runs(uint32_t m, uint8_t* dst0, const uint8_t* src0, uint64_t* bar) {
  const int lane = threadIdx.x & 31;
  const uint32_t sh = m >> lane;
  const bool start = (sh & 1u) && (lane == 0 || !((m >> (lane - 1)) & 1u));
  if (start) {
    const uint32_t x = ~sh;
    const int len = x ? __ffs(x) - 1 : 32 - lane;
    bulk_g2s(dst0 + 64 * __popc(m & ((1u << lane) - 1u)), src0 + 64 * lane, (uint32_t)(64 * len), bar);
  }
}

// Decode a packed element count accumulated by 32-bit adds of 0xFFFF / 0 half masks:
// S = 2^16 (B - A) - B (mod 2^32) for A high-half and B low-half hits (each < 2^15).
__device__ __forceinline__ int pv6_mask_count(uint32_t S) {
  const uint32_t b = (0u - S) & 0xFFFFu;
  const int d = (int)(S + b) >> 16;  // B - A
  return 2 * (int)b - d;
}

// Rule-path partials of HC q-heads (heads p0 ..): element counts into adj, the two row
// halves folded, and the sums added into the mma accumulators (their channel layout)
// through shared memory.
template <int G, int HC, int NT>
__device__ __forceinline__ void pv6_fold(float2 (&ad)[HC][4], const uint32_t (&cmk)[HC], const uint32_t (&clk)[HC],
                                         int p0, float* scr, float (&acc)[NT][8][4], int (&adj)[G][3]) {
  const int lane = threadIdx.x & 31, half = lane >> 4, cg = lane & 15, g = lane >> 2, t = lane & 3;
#pragma unroll
  for (int jj = 0; jj < HC; ++jj) {
    const int cm = pv6_mask_count(cmk[jj]);
    const int cl = pv6_mask_count(clk[jj]);
    adj[p0 + jj][0] -= cm;
    adj[p0 + jj][1] += cm - cl;
    adj[p0 + jj][2] += cl;
#pragma unroll
    for (int k = 0; k < 4; ++k) {
      ad[jj][k].x += __shfl_xor_sync(0xFFFFFFFFu, ad[jj][k].x, 16);
      ad[jj][k].y += __shfl_xor_sync(0xFFFFFFFFu, ad[jj][k].y, 16);
    }
  }
  __syncwarp();
  if (half == 0) {
#pragma unroll
    for (int jj = 0; jj < HC; ++jj) {
      float4* d4 = reinterpret_cast<float4*>(scr + jj * D + 8 * cg);
      d4[0] = make_float4(ad[jj][0].x, ad[jj][0].y, ad[jj][1].x, ad[jj][1].y);
      d4[1] = make_float4(ad[jj][2].x, ad[jj][2].y, ad[jj][3].x, ad[jj][3].y);
    }
  }
  __syncwarp();
#pragma unroll
  for (int nt = 0; nt < NT; ++nt) {
    const int j = 4 * nt + t;
    if (j >= p0 && j < p0 + HC) {
#pragma unroll
      for (int ti = 0; ti < 8; ++ti) {
        const float2 v = *reinterpret_cast<const float2*>(scr + (j - p0) * D + 16 * ti + 2 * g);
        acc[nt][ti][0] += v.x * 16384.f;
        acc[nt][ti][2] += v.y * 16384.f;
      }
    }
  }
  __syncwarp();
}

// Operands of the CUDA-core rule path for one stage (registers after inlining).
template <int G>
struct Pv6Rule {
  const uint8_t* hd;       // the stage: head rows (swizzled) | mid rows | low rows
  const float* pb;         // p block [G][R]
  uint32_t* neb;           // [G][R] packed -ep words
  const uint32_t* g1s;     // [G][64] packed G1 + 8 words of the unit
  float* scr;              // fold scratch [HC][D]
  uint8_t* vt;             // V-mask export base of head 0, row r0 (EXPORT), else null
  size_t vt_head;          // export stride between heads (cap * D)
  uint32_t rm, um, ul;     // rule rows, union mid / low plan rows
  int nm;
  uint32_t selw[G], nmw[G], nlw[G];
};

// The per-element rule (ROWS = false, D4, SPEC.md:169 for unknown targets, D5) or the row
// tier (ROWS = true, D7); contributions folded into the mma accumulators, element counts
// into adj.  SPARSE (DENSE = false): the rows of c.rm, split between the two half-warps by
// the parity of their rank.  DENSE: all 32 rows of a full stage, row 2 it + half (no
// per-row branches): rows outside a head's plan and selected rows go through the rule with
// a threshold that never keeps (selected rows with p = 0: their T16 term is o_est, D6).
// lane = (half, 8 channels).  With e = max(bexp, 1) and X = G1 - ep (G1 = 18 + target -
// margin): keep mid <=> e >= clamp(X, 0, 31), keep low <=> e >= clamp(X + 4, 0, 31); both
// compares share one threshold T = clamp(X + 8, 0, 63): mid <=> e + 8 >= T, low <=> e + 4
// >= T (HSET2 on the small integers as fp16 patterns).  Element counts: the masks summed
// by 32-bit adds (pv6_mask_count).
template <int G, bool EXPORT, bool ROWS, bool DENSE, int NT>
__device__ __forceinline__ void pv6_rule_rows(const Pv6Rule<G>& c, float (&acc)[NT][8][4], int (&adj)[G][3],
                                              float2 (&pad)[Pv6Shape<G>::HC][4], uint32_t (&pcm)[Pv6Shape<G>::HC],
                                              uint32_t (&pcl)[Pv6Shape<G>::HC]) {
  using S = Pv6Shape<G>;
  constexpr int R = S::R, HC = S::HC;
  const int lane = threadIdx.x & 31, half = lane >> 4, cg = lane & 15;
  const uint32_t even = __ballot_sync(0xFFFFFFFFu, ((c.rm >> lane) & 1u) && !(__popc(c.rm & ((1u << lane) - 1u)) & 1));
  const uint32_t mine0 = half ? (c.rm & ~even) : even;
  if (!ROWS || DENSE) {
    // lane = row: -ep = -floor(log2 p) for rows in the head's plan with p > 0; 16000 (kept only
    // for an unknown target) otherwise; 20000 (never) for selected rows (DENSE)
#pragma unroll
    for (int j = 0; j < G; ++j) {
      const float p = c.pb[j * R + lane];
      const bool sel = (c.selw[j] >> lane) & 1u;
      int ne = (((c.nmw[j] >> lane) & 1u) && p > 0.f) ? -floor_log2f(p) : 16000;
      if (DENSE && sel) ne = 20000;
      c.neb[j * R + lane] = (uint32_t)ne * 0x00010001u;
    }
    __syncwarp();
  }
  const uint8_t* nibm = c.hd + S::HEAD;
  const uint8_t* nibl = c.hd + S::HEAD + 64 * c.nm;
  const uint32_t c8 = 0x00800080u, c12 = 0x00080008u;
#pragma unroll
  for (int p0 = 0; p0 < G; p0 += HC) {
    float2 adl[HC][4];
    uint32_t cml[HC], cll[HC], g1[HC][4];
    // page-persistent accumulators (PAGEACC: one pass, folded at the page end) or per-pass ones
    float2 (&ad)[HC][4] = S::PAGEACC ? pad : adl;
    uint32_t (&cmk)[HC] = S::PAGEACC ? pcm : cml;
    uint32_t (&clk)[HC] = S::PAGEACC ? pcl : cll;
#pragma unroll
    for (int jj = 0; jj < HC; ++jj) {
      if (!S::PAGEACC) {
        cmk[jj] = clk[jj] = 0u;
#pragma unroll
        for (int k = 0; k < 4; ++k) ad[jj][k] = make_float2(0.f, 0.f);
      }
      if (!ROWS) {
        const uint4 gv = *reinterpret_cast<const uint4*>(c.g1s + (p0 + jj) * 64 + 4 * cg);
        g1[jj][0] = gv.x;
        g1[jj][1] = gv.y;
        g1[jj][2] = gv.z;
        g1[jj][3] = gv.w;
      }
    }
    uint32_t mine = mine0;
    int it = 0;
#pragma unroll(S::RULE_UNROLL)
    for (; DENSE ? it < 16 : mine != 0u; ++it) {
      const int rr = DENSE ? 2 * it + half : __ffs(mine) - 1;
      if (!DENSE) mine &= mine - 1u;
      const uint32_t bit = 1u << rr, below = bit - 1u;
      const uint2 hv = *reinterpret_cast<const uint2*>(c.hd + rr * D + (((cg >> 1) ^ (rr & 7)) << 4) + (cg & 1) * 8);
      uint32_t mw = 0u, lw = 0u;
      if (c.um & bit) mw = *reinterpret_cast<const uint32_t*>(nibm + 64 * __popc(c.um & below) + 4 * cg);
      if (c.ul & bit) lw = *reinterpret_cast<const uint32_t*>(nibl + 64 * __popc(c.ul & below) + 4 * cg);
      uint32_t w[4], e8[4], e4[4], w8[4], w12[4];
      assemble8(hv.x, hv.y, mw, lw, w);
#pragma unroll
      for (int k = 0; k < 4; ++k) {
        if (!ROWS) {
          // max(bexp, 1) + 8 and + 4 per half (for HC >= 2 the + 4 is formed per use: registers)
          e8[k] = __viaddmax_u16x2((w[k] & 0x7C007C00u) >> 10, 0x00080008u, 0x00090009u);
          if (HC == 1) e4[k] = e8[k] - 0x00040004u;
        }
        w8[k] = (w[k] & 0xFF00FF00u) | c8;
        w12[k] = (w[k] & 0xFFF0FFF0u) | c12;
      }
#pragma unroll
      for (int jj = 0; jj < HC; ++jj) {
        const int j = p0 + jj;
        uint8_t* vt = EXPORT && c.vt ? c.vt + (size_t)j * c.vt_head + (size_t)rr * D + cg * 8 : nullptr;
        if ((!DENSE || EXPORT) && (c.selw[j] & bit)) {  // selected (D6): its T16 term is o_est
          if (EXPORT && vt) *reinterpret_cast<uint2*>(vt) = make_uint2(0x10101010u, 0x10101010u);
          continue;
        }
        const float p = DENSE && ((c.selw[j] >> rr) & 1u) ? 0.f : c.pb[j * R + rr];
        uint32_t mm[4], ml[4];
        if (ROWS) {
          const bool row_ok = !DENSE || !((c.selw[j] >> rr) & 1u);
          const uint32_t a = row_ok && (c.nmw[j] & bit) ? 0xFFFFFFFFu : 0u;
          const uint32_t b = row_ok && (c.nlw[j] & bit) ? 0xFFFFFFFFu : 0u;
#pragma unroll
          for (int k = 0; k < 4; ++k) {
            mm[k] = a;
            ml[k] = b;
          }
        } else {
          const uint32_t nE = c.neb[j * R + rr];
#pragma unroll
          for (int k = 0; k < 4; ++k) {
            const uint32_t T = __viaddmin_s16x2_relu(g1[jj][k], nE, 0x003F003Fu);
            mm[k] = hset2_ge(e8[k], T);
            ml[k] = hset2_ge(HC == 1 ? e4[k] : e8[k] - 0x00040004u, T);
          }
        }
        uint32_t cds[2] = {0u, 0u};
#pragma unroll
        for (int k = 0; k < 4; ++k) {
          const uint32_t wj = bsel(mm[k], bsel(ml[k], w[k], w12[k]), w8[k]);
          ad[jj][k] = ffma2_scalar(half2_bits_to_float2(wj), p, ad[jj][k]);
          if (EXPORT) {
            const uint32_t c2 = 0x00080008u + (mm[k] & 0x00040004u) + (ml[k] & 0x00040004u);  // codes 8/12/16
            cds[k >> 1] |= ((c2 & 0xFFu) | ((c2 >> 8) & 0xFF00u)) << (16 * (k & 1));
          }
        }
        cmk[jj] += (mm[0] + mm[1]) + (mm[2] + mm[3]);
        clk[jj] += (ml[0] + ml[1]) + (ml[2] + ml[3]);
        if (EXPORT && vt) *reinterpret_cast<uint2*>(vt) = make_uint2(cds[0], cds[1]);
      }
    }
    if (!S::PAGEACC) pv6_fold<G, HC, NT>(ad, cmk, clk, p0, c.scr, acc, adj);
  }
}

template <int G, bool EXPORT>
__global__ void __launch_bounds__(32 * Pv6Shape<G>::WARPS, Pv6Shape<G>::MINB)
    pv6_kernel(akv_store_t s, akv_cfg_t cfg, akv_step_t st, int cap, int npg_max,
               const __grid_constant__ CUtensorMap tmv, const __grid_constant__ CUtensorMap tmp,
               const __grid_constant__ CUtensorMap tms, const __grid_constant__ CUtensorMap tmn) {
  using S = Pv6Shape<G>;
  constexpr int R = S::R, HC = S::HC, MAXS = S::MAXS, RING = S::RING, NT = G > 4 ? 2 : 1;
  constexpr int MW = S::META / 4;  // meta words per page slot
  extern __shared__ __align__(1024) uint8_t pv6_raw[];
  uint8_t* sm = pv6_raw + ((1024u - (smem_u32(pv6_raw) & 1023u)) & 1023u);  // 1 KB aligned, still a shared pointer
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int g = lane >> 2, t = lane & 3;  // mma fragment coordinates
  uint8_t* ring = sm + warp * RING;
  uint8_t* misc = sm + S::WARPS * RING + warp * S::MISC;
  float* pblk = reinterpret_cast<float*>(misc + S::OFF_PB);       // [MAXS][G][R]
  uint32_t* metab = reinterpret_cast<uint32_t*>(misc + S::OFF_META);  // [NMETA] x (sel [G][8] | need [G][2][8])
  uint32_t* g1s = reinterpret_cast<uint32_t*>(misc + S::OFF_G1);  // [G][64]
  uint64_t* sbar = reinterpret_cast<uint64_t*>(misc + S::OFF_BAR);  // [MAXS] stage barriers
  uint64_t* mbar = sbar + MAXS;                                     // [NMETA] page-meta barriers
  if (lane == 0) {
    for (int i = 0; i < MAXS + S::NMETA; ++i) mbar_init(&sbar[i], 1);
    mbar_fence_init();
  }
  __syncwarp();
  pdl_trigger();
  pdl_wait();
  const int capw = cap >> 5;
  const long long total = (long long)s.n_units * npg_max;
  const long long nwarps = (long long)gridDim.x * S::WARPS, gw = (long long)blockIdx.x * S::WARPS + warp;
  const long long i0 = total * gw / nwarps, i1 = total * (gw + 1) / nwarps;

  PvCursor ic, cc;
  ic.item = i0;
  ic.pass = 0;
  ic.u = (int)(i0 / npg_max);
  ic.pg = (int)(i0 % npg_max);
  ic.up.u = -1;
  ic.up.n = 0;
  ic.npage = 0;
  bool iv = pv_cursor_seek<R>(ic, i1, s, npg_max, 1);
  cc = ic;
  bool cv = iv;

  // page-meta ring state: which page (item index) each slot holds, issue parity per slot,
  // slots with an issued-but-unwaited copy
  long long mitem[S::NMETA];
#pragma unroll
  for (int i = 0; i < S::NMETA; ++i) mitem[i] = -1;
  uint32_t mpar = 0u, mpend = 0u;
  auto meta_wait = [&](int slot) {
    if ((mpend >> slot) & 1u) {
      mbar_wait(&mbar[slot], ((mpar >> slot) & 1u) ^ 1u);
      mpend &= ~(1u << slot);
    }
  };
  auto meta_issue = [&](int u, int pg, int slot) {
    meta_wait(slot);  // a slot is re-armed only after its previous phase completed
    if (elect_one()) {
      uint32_t* dst = metab + slot * MW;
      mbar_arrive_expect_tx(&mbar[slot], 96 * G);
      tma_load_2d(dst, &tms, pg * 8, u * G, &mbar[slot]);                             // sel words of the G heads
      tma_load_2d(dst + S::SEL_B / 4, &tmn, pg * 8, 2 * u * G, &mbar[slot]);          // need-mid / need-low words
    }
    mpar ^= 1u << slot;
    mpend |= 1u << slot;
  };
  auto set_mitem = [&](int slot, long long v) {
#pragma unroll
    for (int i = 0; i < S::NMETA; ++i)
      if (i == slot) mitem[i] = v;
  };
  auto get_mitem = [&](int slot) {
    long long v = -1;
#pragma unroll
    for (int i = 0; i < S::NMETA; ++i)
      if (i == slot) v = mitem[i];
    return v;
  };

  int ioff = 0, coff = 0, used = 0;  // ring offsets of the issue / consume cursors, bytes in use
  int kiss = 0, ks = 0;              // stages issued / consumed
  int entered = 0;                   // last page (npage) whose meta the issuer has waited for
  // issue the next stage if the ring has room (warp-uniform)
  auto try_issue = [&]() -> bool {
    if (!iv || kiss - ks >= MAXS) return false;
    const int mslot = ic.npage & (S::NMETA - 1);
    if (ic.sub == 0 && entered != ic.npage) {
      // new page: its meta slot was used by page npage - 3; the consumer must be past it
      if (ic.npage - cc.npage >= 2) return false;
      const long long it = (long long)ic.u * npg_max + ic.pg;
      if (get_mitem(mslot) != it) {  // not prefetched (first page, or a skipped unit)
        meta_issue(ic.u, ic.pg, mslot);
        set_mitem(mslot, it);
      }
      meta_wait(mslot);
      entered = ic.npage;
      // prefetch the next page's meta (the page this warp visits next, if in its range)
      long long nx;
      int nu, npg;
      if ((ic.pg + 1) * P < ic.up.n) {
        nu = ic.u;
        npg = ic.pg + 1;
      } else {
        nu = ic.u + 1;
        npg = 0;
      }
      nx = (long long)nu * npg_max + npg;
      if (nx < i1 && nu < s.n_units) {
        const int ns = (ic.npage + 1) & (S::NMETA - 1);
        meta_issue(nu, npg, ns);
        set_mitem(ns, nx);
      }
    }
    const uint32_t* mt = metab + mslot * MW;
    const int sub = ic.sub, r0 = sub * R;
    const int nvs = min(R, ic.rows - r0);
    const uint32_t vmask = nvs >= 32 ? 0xFFFFFFFFu : ((1u << nvs) - 1u);
    uint32_t wm = 0u, wl = 0u;
#pragma unroll
    for (int j = 0; j < G; ++j) {
      wm |= mt[S::SEL_B / 4 + (2 * j) * 8 + sub];
      wl |= mt[S::SEL_B / 4 + (2 * j + 1) * 8 + sub];
    }
    wm &= vmask;
    wl &= vmask;
    const int nm = __popc(wm), nl = __popc(wl);
    const int size = pv6_stage_bytes(nm, nl);
    const int off = ioff + size > RING ? 0 : ioff;
    const int need = size + (off == ioff ? 0 : RING - ioff);
    if (used > 0 && used + need > RING) return false;  // an empty ring takes any stage (<= RING)
    const int slot = kiss % MAXS;
    uint8_t* dst = ring + off;
    const uint8_t* vb = s.v_pool + ic.pid * PAGE;
    if (elect_one()) {
      mbar_arrive_expect_tx(&sbar[slot], S::HEAD + 64 * (nm + nl) + S::PB);
      tma_load_2d(dst, &tmv, 0, (int)(ic.pid * 512 + r0), &sbar[slot]);
      tma_load_2d(pblk + slot * G * R, &tmp, ic.pg * P + r0, ic.u * G, &sbar[slot]);  // p of the G heads
    }
    if (wm) pv6_copy_runs(wm, dst + S::HEAD, vb + MID + r0 * (D / 2), &sbar[slot]);
    if (wl) pv6_copy_runs(wl, dst + S::HEAD + 64 * nm, vb + LOW + r0 * (D / 2), &sbar[slot]);
    used += need;
    ioff = off + size;
    ++kiss;
    iv = pv_cursor_next<R>(ic, i1, s, npg_max, 1);
    return true;
  };

  float acc[NT][8][4];
  int adj[G][3], base[G];
  float2 pad[S::HC][4];  // rule-path partials of the page (PAGEACC)
  uint32_t pcm[S::HC], pcl[S::HC];
  bool pany = false;
  long long vbytes = 0;
  int g1_unit = -1;
  for (; cv; ++ks) {
    __syncwarp();
    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
    while (try_issue()) {
    }
    const int slot = ks % MAXS;
    mbar_wait(&sbar[slot], (uint32_t)(ks / MAXS) & 1u);
    const uint32_t* mt = metab + (cc.npage & (S::NMETA - 1)) * MW;
    const int sub = cc.sub, r0 = sub * R;
    const int nvs = min(R, cc.rows - r0);
    const uint32_t vmask = nvs >= 32 ? 0xFFFFFFFFu : ((1u << nvs) - 1u);
    uint32_t selw[G], nmw[G], nlw[G], um = 0u, ul = 0u;
#pragma unroll
    for (int j = 0; j < G; ++j) {
      selw[j] = mt[j * 8 + sub];
      nmw[j] = mt[S::SEL_B / 4 + (2 * j) * 8 + sub];
      nlw[j] = mt[S::SEL_B / 4 + (2 * j + 1) * 8 + sub];
      um |= nmw[j];
      ul |= nlw[j];
    }
    um &= vmask;
    ul &= vmask;
    const int nm = __popc(um), nl = __popc(ul);
    const int size = pv6_stage_bytes(nm, nl);
    const int off = coff + size > RING ? 0 : coff;
    const int need = size + (off == coff ? 0 : RING - coff);
    uint8_t* hd = ring + off;
    float* pb = pblk + slot * G * R;
    if (sub == 0) {
#pragma unroll
      for (int nt = 0; nt < NT; ++nt)
#pragma unroll
        for (int ti = 0; ti < 8; ++ti) acc[nt][ti][0] = acc[nt][ti][1] = acc[nt][ti][2] = acc[nt][ti][3] = 0.f;
#pragma unroll
      for (int j = 0; j < G; ++j) {
        adj[j][0] = adj[j][1] = adj[j][2] = 0;
        base[j] = 0;
      }
#pragma unroll
      for (int jj = 0; jj < S::HC; ++jj) {
        pcm[jj] = pcl[jj] = 0u;
#pragma unroll
        for (int k = 0; k < 4; ++k) pad[jj][k] = make_float2(0.f, 0.f);
      }
      pany = false;
      vbytes = 0;
    }
    vbytes += (long long)nvs * D + (long long)(nm + nl) * (D / 2);
#pragma unroll
    for (int j = 0; j < G; ++j) base[j] += nvs - __popc(selw[j] & vmask);

    // rows through the CUDA-core rule: the plan rows, or every row when the whole stage is in
    // the plan or the V masks are exported; the tensor cores take the rest at T8
    // (DENSE: a full stage with most rows in the plan goes through the rule whole)
    const bool dense = S::USE_DENSE && cfg.strategy != 1 && vmask == 0xFFFFFFFFu && (EXPORT || __popc(um) >= S::DENSE_MIN);
    const uint32_t rm = (EXPORT || dense || um == vmask) ? vmask : um;
    if (rm) {
      if (cfg.strategy != 1 && g1_unit != cc.u) {
        // per-unit thresholds G1_c + 8 = 26 + target_c - margin (unknown: -16384), channel pairs
        __syncwarp();
        for (int idx = lane; idx < G * 64; idx += 32) {
          const int j = idx >> 6, pr = idx & 63;
          const int2 tg = *reinterpret_cast<const int2*>(st.targets + ((size_t)cc.u * G + j) * D + 2 * pr);
          const int a = tg.x == AKV_TARGET_UNKNOWN ? -16384 : min(max(18 + tg.x - cfg.margin_bits, -16000), 1000) + 8;
          const int b = tg.y == AKV_TARGET_UNKNOWN ? -16384 : min(max(18 + tg.y - cfg.margin_bits, -16000), 1000) + 8;
          g1s[idx] = ((uint32_t)a & 0xFFFFu) | ((uint32_t)b << 16);
        }
        __syncwarp();
        g1_unit = cc.u;
      }
      Pv6Rule<G> rc;
      rc.hd = hd;
      rc.pb = pb;
      rc.neb = reinterpret_cast<uint32_t*>(misc + S::OFF_NE);
      rc.g1s = g1s;
      rc.scr = reinterpret_cast<float*>(misc + S::OFF_SCR);
      rc.vt = EXPORT && st.v_tiers ? st.v_tiers + ((size_t)cc.u * G * cap + (size_t)cc.pg * P + r0) * D : nullptr;
      rc.vt_head = (size_t)cap * D;
      rc.rm = rm;
      rc.um = um;
      rc.ul = ul;
      rc.nm = nm;
#pragma unroll
      for (int j = 0; j < G; ++j) {
        rc.selw[j] = selw[j];
        rc.nmw[j] = nmw[j];
        rc.nlw[j] = nlw[j];
      }
      if (cfg.strategy == 1) pv6_rule_rows<G, EXPORT, true, false>(rc, acc, adj, pad, pcm, pcl);
      else if (S::USE_DENSE && dense) pv6_rule_rows<G, EXPORT, false, S::USE_DENSE>(rc, acc, adj, pad, pcm, pcl);
      else pv6_rule_rows<G, EXPORT, false, false>(rc, acc, adj, pad, pcm, pcl);
      pany = true;
    }
    if (!EXPORT && rm != vmask) {
      // T8 rows on the tensor cores (pv5): p = 0 for selected rows (D6), rows past the length
      // and the rows the rule path took
      // lane = row: fp16 hi / lo halves of p * 2^14 packed per row, 0 for dead rows
      const bool dead = !((vmask >> lane) & 1u) || ((rm >> lane) & 1u);
      uint32_t* pbh = reinterpret_cast<uint32_t*>(misc + S::OFF_NE);
      __syncwarp();
#pragma unroll
      for (int j = 0; j < G; ++j) {
        const float x = (dead || ((selw[j] >> lane) & 1u)) ? 0.f : pb[j * R + lane] * 16384.f;
        const __half hh = __float2half_rn(x);
        const __half hl = __float2half_rn(x - __half2float(hh));
        pbh[j * R + lane] = (uint32_t)__half_as_ushort(hh) | ((uint32_t)__half_as_ushort(hl) << 16);
      }
      __syncwarp();
#pragma unroll
      for (int kk = 0; kk < 2; ++kk) {
        uint32_t bf[NT][2];
#pragma unroll
        for (int nt = 0; nt < NT; ++nt) {
          const int n = 8 * nt + g, j = n >> 1;
          if (j < G) {
            const uint2 x01 = *reinterpret_cast<const uint2*>(pbh + j * R + 16 * kk + 2 * t);
            const uint2 x89 = *reinterpret_cast<const uint2*>(pbh + j * R + 16 * kk + 2 * t + 8);
            const uint32_t sel = (n & 1) ? 0x7632u : 0x5410u;  // lo halves : hi halves
            bf[nt][0] = prmt(x01.x, x01.y, sel);
            bf[nt][1] = prmt(x89.x, x89.y, sel);
          } else {
            bf[nt][0] = bf[nt][1] = 0u;
          }
        }
        const int tok = 16 * kk + (lane & 7) + ((lane >> 3) & 1) * 8;
#pragma unroll
        for (int tp = 0; tp < 4; ++tp) {
          const int chunk = 2 * tp + (lane >> 4);
          uint32_t r[4];
          ldsm_x4_trans(r, hd + tok * D + ((chunk ^ (tok & 7)) << 4));
          const uint32_t c80 = 0x80808080u;
#pragma unroll
          for (int h2 = 0; h2 < 2; ++h2) {
            const uint32_t a0 = prmt(r[2 * h2], c80, 0x2404), a1 = prmt(r[2 * h2], c80, 0x3414);
            const uint32_t a2 = prmt(r[2 * h2 + 1], c80, 0x2404), a3 = prmt(r[2 * h2 + 1], c80, 0x3414);
#pragma unroll
            for (int nt = 0; nt < NT; ++nt) mma_16816(acc[nt][2 * tp + h2], a0, a1, a2, a3, bf[nt][0], bf[nt][1]);
          }
        }
      }
    }
    used -= need;
    coff = off + size;

    if (cc.sub + 1 == cc.nsub) {
      if (S::PAGEACC && __any_sync(0xFFFFFFFFu, pany))
        pv6_fold<G, S::HC, NT>(pad, pcm, pcl, 0, reinterpret_cast<float*>(misc + S::OFF_SCR), acc, adj);
      if (lane == 0)
        atomicAdd(reinterpret_cast<unsigned long long*>(st.unit_bytes + (size_t)cc.u * 4 + 1),
                  (unsigned long long)vbytes);
      // lane (g, t): head 4nt + t, channels 16ti + 2g (d0 + d1) and 16ti + 2g + 1 (d2 + d3)
#pragma unroll
      for (int nt = 0; nt < NT; ++nt) {
        const int j = 4 * nt + t;
        if (j < G) {
          const size_t h = (size_t)cc.u * G + j;
          float* dst = st.o_partial + (h * (cap / P) + cc.pg) * D;
#pragma unroll
          for (int ti = 0; ti < 8; ++ti) {
            const int c = 16 * ti + 2 * g;
            const float o0 = (acc[nt][ti][0] + acc[nt][ti][1]) * (1.f / 16384.f);
            const float o1 = (acc[nt][ti][2] + acc[nt][ti][3]) * (1.f / 16384.f);
            *reinterpret_cast<float2*>(dst + c) = make_float2(o0, o1);
          }
        }
      }
#pragma unroll
      for (int j = 0; j < G; ++j) {
        const int a = warp_sum_i(adj[j][0]), b1 = warp_sum_i(adj[j][1]), c2 = warp_sum_i(adj[j][2]);
        if (lane == 0) {
          unsigned long long* ct = reinterpret_cast<unsigned long long*>(st.counters + ((size_t)cc.u * G + j) * 8 + 3);
          const long long t8 = a + (long long)base[j] * D;
          if (t8) atomicAdd(ct + 0, (unsigned long long)t8);
          if (b1) atomicAdd(ct + 1, (unsigned long long)b1);
          if (c2) atomicAdd(ct + 2, (unsigned long long)c2);
        }
      }
    }
    cv = pv_cursor_next<R>(cc, i1, s, npg_max, 1);
  }
  // a prefetched page meta this warp never visited (a unit past its length) must land
  // before the CTA exits
#pragma unroll
  for (int i = 0; i < S::NMETA; ++i) meta_wait(i);
}

template <int G, bool EXPORT>
static bool launch_pv6_t(const akv_store_t& s, const akv_cfg_t& cfg, const akv_step_t& st, int max_len,
                         cudaStream_t stream) {
  using S = Pv6Shape<G>;
  const int cap = s.max_pages * P;
  const unsigned long long heads = (unsigned long long)s.n_units * G;
  CUtensorMap tm, tp, ts, tn;
  if (!v_head_tmap(s, &tm)) return false;
  // p [U*G][cap] (box 32 rows x G heads), sel words [U*G][cap/32] (box 8 x G), need words
  // [U*G*2][cap/32] (box 8 x 2G): the G heads of a unit are consecutive rows
  if (!tmap_2d(st.probs, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 4, cap, heads, 32, G, CU_TENSOR_MAP_SWIZZLE_NONE, &tp)) return false;
  if (!tmap_2d(st.sel_bits, CU_TENSOR_MAP_DATA_TYPE_UINT32, 4, cap / 32, heads, 8, G, CU_TENSOR_MAP_SWIZZLE_NONE, &ts)) return false;
  if (!tmap_2d(st.need_bits, CU_TENSOR_MAP_DATA_TYPE_UINT32, 4, cap / 32, 2 * heads, 8, 2 * G, CU_TENSOR_MAP_SWIZZLE_NONE, &tn)) return false;
  const int resident = resident_ctas<pv6_kernel<G, EXPORT>>(32 * S::WARPS, S::SMEM);
  const int npg = (max_len + P - 1) / P;
  const long long items = (long long)s.n_units * npg;
  const int grid = balanced_grid(items, resident, S::WARPS, G <= 2);  // G = 4: fewer warps cost more (c3)
  launch_pdl(PDL_PV, pv6_kernel<G, EXPORT>, dim3(grid), dim3(32 * S::WARPS), (size_t)S::SMEM, stream, s, cfg, st, cap, npg, tm,
             tp, ts, tn);
  return true;
}

}  // namespace akv
