// qk9: scores_aligned for GQA groups (G = 4, 8) on the 5th-generation
// tensor cores: tcgen05.mma (kind::f16, fp32 accumulator in TMEM), operands in shared
// memory, K pages streamed by TMA bulk copies.  Included by akv_qk.cu.
//
// The G q-heads of a unit share every K tile, so a page is a GEMM
//   s[256 tokens][G] = K~[256][K-rows] x Bq[K-rows][G]
// whose K dimension is the unit's list of (channel, tier variant) rows: a channel whose G
// heads read it at tiers {v} contributes one row per distinct v, its words truncated to v
// (midpoint fill, HB:160-179) in A, and q_j(c) in B for the heads with tier_j(c) = v (0
// elsewhere):  s_j = sum_c q_jc K~_{tier_j(c)}(c) = sum_rows A[t][row] B[row][j].  Products
// of fp16 words are exact in the fp32 accumulator (D9).
//
// One CTA per SM, persistent over a balanced contiguous range of (unit, page) items:
//   warp 0 (producer): per unit, Rule 1 (k_rule1: tiers, bookkeeping) and the unit's row
//     list + B operand (double-buffered by unit parity); per page, TMA bulk copies of the
//     page's head plane (32 KB, fixed channel positions) and of the mid / low nibble rows
//     the union tiers need (compacted, 16 B cp.async per lane tracked by the stage mbarrier)
//     into a variable-size stage ring (up to 6 pages in flight);
//   warps 2-9 (builders): rebuild the rows' fp16 words from the staged planes into A
//     chunks of 64 rows x 256 tokens (MN-major, 128 B swizzle: the
//     16 B stores of a warp fall on distinct banks), 2-chunk ring; afterwards the
//     epilogue of the previous page: tcgen05.ld of the accumulator (warp w reads TMEM
//     lanes 32 (w % 4) .. of M-tile (w - 2) / 4), 1/sqrt(d), scores, per-32-token
//     (max, sum exp) chunk statistics;
//   warp 1 (MMA): one thread issues M=128 N=16 K=16 MMAs per (M-tile, 16 rows) into a
//     double-buffered TMEM accumulator (2 pages x 2 M-tiles x 16 columns) and commits
//     them to the chunk-free / accumulator-full mbarriers.
// Per unit the K bytes are the same as the CUDA-core kernels' (head rows of the non-SKIP
// channels, nibble rows of the union T12 / T16 channels); there is no per-element
// decision here (Rule 1 is per channel), so K tier masks stay bit-exact.
// Opt-in (AKV_QK_KERNEL=qk9): parity-green but slower than qk5 at c3 (the per-row fp16
// rebuild into shared memory bounds it; profiles/r02_history.md r2-7).
#include <cstdio>

namespace akv {

template <int G>
struct Qk9Shape {
  static constexpr int KC = 64;                      // rows per A chunk (8 per builder warp)
  static constexpr int RPW = KC / 8;                 // rows per builder warp per chunk
  // A chunk: 256 tokens x KC rows, fp16, MN-major with the 128 B swizzle: 1 KB atoms of
  // 8 rows x 64 tokens, atom (token / 64, row / 8) at (row / 8) * 4 KB + (token / 64) * 1 KB
  static constexpr int ACH = KC * P * 2;
  static constexpr int NA = 2;                       // A chunk ring
  static constexpr int MAXK = 3 * D;                 // rows per unit (<= 3 tier variants / channel)
  static constexpr int BB = (MAXK / 8) * 256;        // B: [rows][16 heads] fp16, K-major
  static constexpr int META = 128;
  static constexpr int NIBL = 2 * D;                 // nibble row list: mid channels, then low channels (u8)
  static constexpr int UNIT = BB + MAXK * 4 + META + NIBL;  // B | row list | meta | nibble rows
  static constexpr int NSLOT = 6;                    // K pages in flight at most
  static constexpr int NBAR = 2 * NSLOT + 4 + 2 * NA + 4;
  static constexpr int SMEM_MAX = 232448;            // 227 KB opt-in
  static constexpr int FIXED = NA * ACH + 2 * UNIT + NSLOT * 4 + NBAR * 8 + 16 + 1024;  // + 1 KB alignment slack
  static constexpr int RING = (SMEM_MAX - FIXED) & ~1023;  // variable-size K page stages (head | mid | low)
  static constexpr int OFF_A = RING;
  static constexpr int OFF_U = OFF_A + NA * ACH;
  static constexpr int OFF_SOFF = OFF_U + 2 * UNIT;
  static constexpr int OFF_BAR = OFF_SOFF + NSLOT * 4;
  static constexpr int SMEM = OFF_BAR + NBAR * 8 + 16 + 1024;
  static constexpr int BUILDERS = 8;
  static constexpr int THREADS = 32 * (2 + BUILDERS);
  static constexpr int TMEM_COLS = 64;               // 2 pages x 2 M-tiles x 16 columns
  static_assert(RING >= 2 * 65536, "two full pages must fit the stage ring");
};

// unit meta words
enum { Q9_NK = 0, Q9_NMID, Q9_NLOW, Q9_HBYTES, Q9_MHEAD = 4, Q9_MMID = 8, Q9_MLOW = 12 };

__device__ __forceinline__ void mbar_arrive1(uint64_t* bar) {
  asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem_u32(bar)) : "memory");
}
__device__ __forceinline__ void tc_fence_before() { asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory"); }
__device__ __forceinline__ void tc_fence_after() { asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory"); }
__device__ __forceinline__ void fence_async_smem() { asm volatile("fence.proxy.async.shared::cta;" ::: "memory"); }

#ifdef QK9_PROF
#define Q9_WAIT(bar, par, acc)                  \
  do {                                          \
    const long long t0_ = clock64();            \
    mbar_wait(bar, par);                        \
    acc += clock64() - t0_;                     \
  } while (0)
#else
#define Q9_WAIT(bar, par, acc) mbar_wait(bar, par)
#endif

// UMMA shared-memory descriptor, no swizzle: start, leading / stride byte offsets (16 B
// units), version 1 (sm_100).
__device__ __forceinline__ uint64_t umma_desc(uint32_t addr, uint32_t lbo, uint32_t sbo) {
  return (uint64_t)((addr >> 4) & 0x3FFFu) | ((uint64_t)((lbo >> 4) & 0x3FFFu) << 16) |
         ((uint64_t)((sbo >> 4) & 0x3FFFu) << 32) | ((uint64_t)1 << 46);
}
// the same with the 128 B swizzle (layout type 2; 1 KB aligned atoms, base offset 0)
__device__ __forceinline__ uint64_t umma_desc_sw128(uint32_t addr, uint32_t lbo, uint32_t sbo) {
  return umma_desc(addr, lbo, sbo) | ((uint64_t)2 << 61);
}

__device__ __forceinline__ void umma_f16(uint32_t d_tmem, uint64_t a, uint64_t b, uint32_t idesc, uint32_t acc) {
  asm volatile(
      "{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\t"
      "tcgen05.mma.cta_group::1.kind::f16 [%0], %1, %2, %3, p;\n\t}" ::"r"(d_tmem),
      "l"(a), "l"(b), "r"(idesc), "r"(acc)
      : "memory");
}
__device__ __forceinline__ void umma_commit(uint64_t* bar) {
  asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(smem_u32(bar))
               : "memory");
}

// Copy the rows of the set bits of mask (32 rows of rowbytes from src0), one bulk copy per
// maximal run, issued by the lane at the run start; compact: destination row = rank.
__device__ __forceinline__ void q9_copy_runs(uint32_t m, uint8_t* dst0, const uint8_t* src0, uint32_t rowbytes,
                                             bool compact, uint64_t* bar) {
  const int lane = threadIdx.x & 31;
  const uint32_t sh = m >> lane;
  const bool start = (sh & 1u) && (lane == 0 || !((m >> (lane - 1)) & 1u));
  if (start) {
    const uint32_t x = ~sh;
    const int len = x ? __ffs(x) - 1 : 32 - lane;
    const uint32_t drow = compact ? (uint32_t)__popc(m & ((1u << lane) - 1u)) : (uint32_t)lane;
    bulk_g2s(dst0 + rowbytes * drow, src0 + rowbytes * lane, rowbytes * len, bar);
  }
}

// Producer warp: Rule 1 for unit u and its row list, B operand and copy masks.
template <int G, bool TRUNC>
__device__ __forceinline__ void q9_unit_setup(uint8_t* ub, const akv_store_t& s, const akv_cfg_t& cfg,
                                              const akv_step_t& st, int u, int n, bool book) {
  using S = Qk9Shape<G>;
  const int lane = threadIdx.x & 31;
  uint16_t* B = reinterpret_cast<uint16_t*>(ub);
  uint32_t* krow = reinterpret_cast<uint32_t*>(ub + S::BB);
  uint32_t* meta = krow + S::MAXK;
  uint32_t qw[G][4];
  int code[G][4], ucode[4];
  k_rule1<G, TRUNC>(s, cfg, st, u, n, book, qw, code, ucode);
  const uint32_t lt = (1u << lane) - 1u;
  uint32_t mhead[4], mmid[4], mlow[4], has[3][4];
  int nmid = 0, nlow = 0, nh = 0;
#pragma unroll
  for (int k = 0; k < 4; ++k) {
    mhead[k] = __ballot_sync(0xFFFFFFFFu, ucode[k] != 0);
    mmid[k] = __ballot_sync(0xFFFFFFFFu, ucode[k] >= 12);
    mlow[k] = __ballot_sync(0xFFFFFFFFu, ucode[k] == 16);
#pragma unroll
    for (int v = 0; v < 3; ++v) {
      bool any = false;
#pragma unroll
      for (int j = 0; j < G; ++j) any |= code[j][k] == 8 + 4 * v;
      has[v][k] = __ballot_sync(0xFFFFFFFFu, any);
    }
  }
  int mslot[4], lslot[4];
#pragma unroll
  for (int k = 0; k < 4; ++k) {
    mslot[k] = nmid + __popc(mmid[k] & lt);
    lslot[k] = nlow + __popc(mlow[k] & lt);
    nmid += __popc(mmid[k]);
    nlow += __popc(mlow[k]);
    nh += __popc(mhead[k]);
  }
  // rows: the T8 variants (channel order), then the T12 ones, then the T16 ones
  int pos = 0;
#pragma unroll
  for (int v = 0; v < 3; ++v)
#pragma unroll
    for (int k = 0; k < 4; ++k) {
      if ((has[v][k] >> lane) & 1u) {
        const int r = pos + __popc(has[v][k] & lt);
        const int c = lane + 32 * k;
        krow[r] = (uint32_t)c | ((uint32_t)(v + 1) << 8) | ((uint32_t)mslot[k] << 16) | ((uint32_t)lslot[k] << 24);
        uint16_t* br = B + (r >> 3) * 128 + (r & 7);  // (r/8) 256 B + (j/8) 128 B + (j%8) 16 B + (r%8) 2 B
#pragma unroll
        for (int j = 0; j < G; ++j)
          br[(j >> 3) * 64 + (j & 7) * 8] = code[j][k] == 8 + 4 * v ? (uint16_t)(qw[j][k] & 0xFFFFu) : (uint16_t)0;
      }
      pos += __popc(has[v][k]);
    }
  // pad to a multiple of 16 rows (at least 16: an all-SKIP unit still writes its zero
  // scores): channel 0 at T8 (finite words) with q = 0
  const int nk = max(16, (pos + 15) & ~15);
  for (int r = pos + lane; r < nk; r += 32) {
    krow[r] = 1u << 8;
    uint16_t* br = B + (r >> 3) * 128 + (r & 7);
#pragma unroll
    for (int j = 0; j < G; ++j) br[(j >> 3) * 64 + (j & 7) * 8] = 0;
  }
  uint8_t* nib = reinterpret_cast<uint8_t*>(meta) + S::META;
#pragma unroll
  for (int k = 0; k < 4; ++k) {
    if ((mmid[k] >> lane) & 1u) nib[mslot[k]] = (uint8_t)(lane + 32 * k);
    if ((mlow[k] >> lane) & 1u) nib[nmid + lslot[k]] = (uint8_t)(lane + 32 * k);
  }
  if (lane == 0) {
    meta[Q9_NK] = nk;
    meta[Q9_NMID] = nmid;
    meta[Q9_NLOW] = nlow;
    meta[Q9_HBYTES] = 256 * nh;
  }
  if (lane < 4) {
    meta[Q9_MHEAD + lane] = lane == 0 ? mhead[0] : lane == 1 ? mhead[1] : lane == 2 ? mhead[2] : mhead[3];
    meta[Q9_MMID + lane] = lane == 0 ? mmid[0] : lane == 1 ? mmid[1] : lane == 2 ? mmid[2] : mmid[3];
    meta[Q9_MLOW + lane] = lane == 0 ? mlow[0] : lane == 1 ? mlow[1] : lane == 2 ? mlow[2] : mlow[3];
  }
}

template <int G, bool TRUNC>
__global__ void __launch_bounds__(Qk9Shape<G>::THREADS, 1)
    qk9_kernel(akv_store_t s, akv_cfg_t cfg, akv_step_t st, int cap, float isd, int npg_max) {
  using S = Qk9Shape<G>;
  extern __shared__ __align__(1024) uint8_t q9_raw[];
  uint8_t* q9 = q9_raw + ((1024u - (smem_u32(q9_raw) & 1023u)) & 1023u);  // 1 KB aligned (swizzle atoms)
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  uint64_t* full = reinterpret_cast<uint64_t*>(q9 + S::OFF_BAR);
  uint64_t* empty = full + S::NSLOT;
  uint32_t* soff = reinterpret_cast<uint32_t*>(q9 + S::OFF_SOFF);  // stage offset of page slot
  uint64_t* ufull = empty + S::NSLOT;
  uint64_t* uempty = ufull + 2;
  uint64_t* afull = uempty + 2;
  uint64_t* aempty = afull + S::NA;
  uint64_t* dfull = aempty + S::NA;
  uint64_t* dempty = dfull + 2;
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(dempty + 2);
  uint8_t* abuf = q9 + S::OFF_A;
  uint8_t* ubuf = q9 + S::OFF_U;
  constexpr int NB = S::BUILDERS;

  if (threadIdx.x == 0) {
    for (int i = 0; i < S::NSLOT; ++i) {
      mbar_init(&full[i], 33);  // the TMA expect_tx arrive + the producer lanes' cp.async arrives
      mbar_init(&empty[i], NB);
    }
    for (int i = 0; i < 2; ++i) {
      mbar_init(&ufull[i], 1);
      mbar_init(&uempty[i], NB);
      mbar_init(&dfull[i], 1);
      mbar_init(&dempty[i], NB);
    }
    for (int i = 0; i < S::NA; ++i) {
      mbar_init(&afull[i], NB);
      mbar_init(&aempty[i], 1);
    }
    mbar_fence_init();
  }
  if (warp == 1) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(smem_u32(tmem_slot)),
                 "n"(S::TMEM_COLS)
                 : "memory");
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;" ::: "memory");
  }
  // both B buffers zero: the rows of heads >= G stay zero
  for (int i = threadIdx.x; i < S::BB / 16; i += S::THREADS) {
    reinterpret_cast<uint4*>(ubuf)[i] = make_uint4(0u, 0u, 0u, 0u);
    reinterpret_cast<uint4*>(ubuf + S::UNIT)[i] = make_uint4(0u, 0u, 0u, 0u);
  }
  fence_async_smem();
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = *tmem_slot;
  long long w_a = 0, w_b = 0, w_c = 0, w_d = 0, w_e = 0, w_f = 0;
#ifdef QK9_PROF
  const long long t_start = clock64();
#endif
  pdl_trigger();
  pdl_wait();

  // balanced contiguous range of (unit, page) items; every role walks the same items
  const long long total = (long long)s.n_units * npg_max;
  const long long i0 = total * blockIdx.x / gridDim.x, i1 = total * (blockIdx.x + 1) / gridDim.x;
  const int cap_chunks = s.max_pages * (P / 32);
  struct Cur {
    long long i;
    int u, pg;
    UnitPages up;
  };
  auto seek = [&](Cur& c) {
    while (c.i < i1) {
      if (c.u != c.up.u) unit_pages_fetch(c.up, s, c.u);
      if (c.pg * P < c.up.n) return;
      c.i += npg_max - c.pg;
      c.pg = 0;
      ++c.u;
    }
  };
  auto advance = [&](Cur& c) {
    ++c.i;
    if (++c.pg == npg_max) {
      c.pg = 0;
      ++c.u;
    }
    seek(c);
  };
  Cur c;
  c.i = i0;
  c.u = (int)(i0 / npg_max);
  c.pg = (int)(i0 % npg_max);
  c.up.u = -1;
  c.up.n = 0;
  seek(c);

  if (warp == 0) {
    // ---------------- producer ----------------
    // variable-size stages in a byte ring, freed in order (oldest first)
    int cur = -1, nu = 0, kp = 0, freed = 0, used = 0, head = 0;
    int fsz[S::NSLOT];
#pragma unroll
    for (int i = 0; i < S::NSLOT; ++i) fsz[i] = 0;
    uint8_t* ub = ubuf;
    while (c.i < i1) {
      if (c.u != cur) {
        ub = ubuf + (nu & 1) * S::UNIT;
        if (nu >= 2) Q9_WAIT(&uempty[nu & 1], ((nu >> 1) - 1) & 1, w_a);
        q9_unit_setup<G, TRUNC>(ub, s, cfg, st, c.u, c.up.n, c.pg == 0);
        fence_async_smem();  // B (generic stores) before the tensor core reads it
        __syncwarp();
        if (lane == 0) mbar_arrive1(&ufull[nu & 1]);
        ++nu;
        cur = c.u;
      }
      const uint32_t* meta = reinterpret_cast<const uint32_t*>(ub + S::BB + S::MAXK * 4);
      const uint32_t nmid = meta[Q9_NMID], nlow = meta[Q9_NLOW], hb = meta[Q9_HBYTES];
      const int size = (int)((256u * D + 128u * (nmid + nlow) + 127u) & ~127u);
      const int off = head + size > S::RING ? 0 : head;
      const int need = size + (off == head ? 0 : S::RING - head);
      const int slot = kp % S::NSLOT;
      while (used + need > S::RING || kp - freed >= S::NSLOT) {
        const int fs = freed % S::NSLOT;
        Q9_WAIT(&empty[fs], (freed / S::NSLOT) & 1, w_b);
#pragma unroll
        for (int i = 0; i < S::NSLOT; ++i)
          if (i == fs) used -= fsz[i];
        ++freed;
      }
#pragma unroll
      for (int i = 0; i < S::NSLOT; ++i)
        if (i == slot) fsz[i] = need;
      used += need;
      head = off + size;
      uint8_t* dst = q9 + off;
      const uint8_t* src = s.k_pool + unit_page(c.up, s, c.pg) * PAGE;
      if (lane == 0) {
        soff[slot] = (uint32_t)off;
        mbar_arrive_expect_tx(&full[slot], hb);
      }
      __syncwarp();
      // head rows: one bulk copy (all channels), else one per run of non-SKIP channels
      if (hb == 256u * D) {
        if (lane == 0) bulk_g2s(dst, src, 256 * D, &full[slot]);
      } else {
#pragma unroll 1
        for (int k = 0; k < 4; ++k) q9_copy_runs(meta[Q9_MHEAD + k], dst + 32 * k * 256, src + 32 * k * 256, 256, false, &full[slot]);
      }
      // nibble rows (compacted): 16 B cp.async per lane (per-lane addresses: no bulk-copy
      // waterfalls), tracked by the stage barrier through cp.async.mbarrier.arrive
      const uint8_t* nib = reinterpret_cast<const uint8_t*>(meta) + S::META;
      const int nrow = (int)(nmid + nlow);
      for (int idx = lane; idx < 8 * nrow; idx += 32) {
        const int row = idx >> 3, part = idx & 7;
        const int ch = nib[row];
        const uint8_t* sp = src + (row < (int)nmid ? MID : LOW) + ch * 128 + part * 16;
        cp_async16(dst + 256 * D + row * 128 + part * 16, sp);
      }
      asm volatile("cp.async.mbarrier.arrive.noinc.shared::cta.b64 [%0];" ::"r"(smem_u32(&full[slot])) : "memory");
      ++kp;
      advance(c);
    }
  } else if (warp == 1) {
    // ---------------- MMA issuer ----------------
    // The whole warp walks the items (warp-uniform descriptors live in uniform registers);
    // one elected lane issues the MMAs and the commits.
    {
      const uint32_t idesc = (1u << 4) | (1u << 15) | ((16u >> 3) << 17) | ((128u >> 4) << 24);  // f32 D, f16 A/B, A MN-major
      int cur = -1, nu = 0, ka = 0, lp = 0;
      const uint8_t* ub = ubuf;
      while (c.i < i1) {
        if (c.u != cur) {
          ub = ubuf + (nu & 1) * S::UNIT;
          ++nu;
          cur = c.u;
        }
        const int d = lp & 1;
        if (lp >= 2) Q9_WAIT(&dempty[d], ((lp >> 1) - 1) & 1, w_a);
        int nk = 16, a = 0;
        do {
          const int slot = ka % S::NA;
          Q9_WAIT(&afull[slot], (ka / S::NA) & 1, w_b);
          tc_fence_after();
          if (a == 0) nk = (int)reinterpret_cast<const uint32_t*>(ub + S::BB + S::MAXK * 4)[Q9_NK];
          const int kbs = min(nk - S::KC * a, S::KC) >> 4;
          const uint32_t abase = smem_u32(abuf + slot * S::ACH), bbase = smem_u32(ub) + a * (S::KC / 8) * 256;
#ifdef QK9_PROF
          const long long tm0_ = clock64();
#endif
          if (elect_one()) {
#ifndef QK9_NOMMA
#pragma unroll
            for (int mt = 0; mt < 2; ++mt)
#pragma unroll
              for (int kb = 0; kb < S::KC / 16; ++kb)
                if (kb < kbs)
                  umma_f16(tmem + d * 32 + mt * 16, umma_desc_sw128(abase + mt * 2048 + kb * 8192, 1024, 4096),
                           umma_desc(bbase + kb * 512, 256, 128), idesc, (a | kb) != 0);
#endif
            umma_commit(&aempty[slot]);
          }
          __syncwarp();
#ifdef QK9_PROF
          w_e += clock64() - tm0_;
#endif
          ++ka;
          ++a;
        } while (S::KC * a < nk);
        if (elect_one()) umma_commit(&dfull[d]);
        __syncwarp();
        ++lp;
        advance(c);
      }
    }
  } else {
    // ---------------- builders / epilogue ----------------
    const int bw = warp - 2;
    uint32_t tkm = 0xFFFFFFFFu, tf = 0u;
    if (TRUNC) {
      const int kb = cfg.trunc_bits - 6;
      const uint32_t km = (0xFFFFu << (10 - kb)) & 0xFFFFu;
      const uint32_t fill = kb < 10 ? (1u << (9 - kb)) : 0u;
      tkm = km | (km << 16);
      tf = fill | (fill << 16);
    }
    struct Prev {
      int lp, u, pg, n, ub;
    };
    Prev pv{-1, 0, 0, 0, 0};
    // epilogue of page p: warp (M-tile mt, TMEM lanes 32 q ..): token t = 256 pg + 128 mt + 32 q + lane
    auto epilogue = [&](const Prev& p, bool release_unit) {
      const int d = p.lp & 1, q = warp & 3, mt = bw >> 2;
      Q9_WAIT(&dfull[d], (p.lp >> 1) & 1, w_c);
      tc_fence_after();
      uint32_t r[16];
      asm volatile(
          "tcgen05.ld.sync.aligned.32x32b.x16.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15}, [%16];"
          : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]), "=r"(r[7]), "=r"(r[8]),
            "=r"(r[9]), "=r"(r[10]), "=r"(r[11]), "=r"(r[12]), "=r"(r[13]), "=r"(r[14]), "=r"(r[15])
          : "r"(tmem + ((uint32_t)(32 * q) << 16) + d * 32 + mt * 16));
      asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
      tc_fence_before();
      __syncwarp();
      if (lane == 0) mbar_arrive1(&dempty[d]);  // the accumulator is in registers
      const int tok0 = p.pg * P + 128 * mt + 32 * q, tok = tok0 + lane;
      const bool valid = tok < p.n;
      if (tok0 < p.n) {
        // the G heads' chunk statistics with interleaved butterflies (independent chains)
        float sv[G], m[G], l[G];
#pragma unroll
        for (int j = 0; j < G; ++j) {
          sv[j] = __uint_as_float(r[j]) * isd;
          if (valid) st.scores[((size_t)p.u * G + j) * cap + tok] = sv[j];
          m[j] = valid ? sv[j] : -INFINITY;
        }
#pragma unroll
        for (int o = 16; o > 0; o >>= 1)
#pragma unroll
          for (int j = 0; j < G; ++j) m[j] = fmaxf(m[j], __shfl_xor_sync(0xFFFFFFFFu, m[j], o));
#pragma unroll
        for (int j = 0; j < G; ++j) {
          l[j] = 0.f;
          if (valid) asm("ex2.approx.ftz.f32 %0, %1;" : "=f"(l[j]) : "f"((sv[j] - m[j]) * 1.4426950408889634f));
        }
#pragma unroll
        for (int o = 16; o > 0; o >>= 1)
#pragma unroll
          for (int j = 0; j < G; ++j) l[j] += __shfl_xor_sync(0xFFFFFFFFu, l[j], o);
        if (lane < G) {
          float mj = m[0], lj = l[0];
#pragma unroll
          for (int j = 1; j < G; ++j)
            if (lane == j) {
              mj = m[j];
              lj = l[j];
            }
          float* ps = st.page_stats + (((size_t)p.u * G + lane) * cap_chunks + (tok0 >> 5)) * 2;
          ps[0] = mj;
          ps[1] = lj;
        }
      }
      if (release_unit && lane == 0) mbar_arrive1(&uempty[p.ub]);
    };
    int cur = -1, nu = 0, kp = 0, ka = 0, ubi = 0;
    const uint8_t* ub = ubuf;
    while (c.i < i1) {
      if (c.u != cur) {
        ubi = nu & 1;
        ub = ubuf + ubi * S::UNIT;
        mbar_wait(&ufull[ubi], (nu >> 1) & 1);
        ++nu;
        cur = c.u;
      }
      const uint32_t* krow = reinterpret_cast<const uint32_t*>(ub + S::BB);
      const uint32_t* meta = krow + S::MAXK;
      const int nk = (int)meta[Q9_NK], nmid = (int)meta[Q9_NMID];
      const int slot = kp % S::NSLOT;
      Q9_WAIT(&full[slot], (kp / S::NSLOT) & 1, w_a);
      const uint8_t* sg = q9 + soff[slot];
      const uint8_t* sm_mid = sg + 256 * D;
      const uint8_t* sm_low = sm_mid + 128 * nmid;
#ifdef QK9_PROF
      const long long tb0_ = clock64();
#endif
      // rows of chunk a (this warp's RPW rows): entries and every stage load; issued one
      // chunk ahead of the words so the shared-memory latency overlaps the previous build
      struct Rows {
        uint32_t e[S::RPW], mw[S::RPW], lw[S::RPW];
        uint2 hv[S::RPW];
      };
      auto load_rows = [&](Rows& R, int a) {
#pragma unroll
        for (int i = 0; i < S::RPW; ++i) {
          const int r = S::KC * a + S::RPW * bw + i;
          R.e[i] = r < nk ? krow[r] : 0u;
        }
#pragma unroll
        for (int i = 0; i < S::RPW; ++i) {
          const uint32_t e = R.e[i];
          const int v = (e >> 8) & 3;
          R.hv[i] = *reinterpret_cast<const uint2*>(sg + ((e & 0x7Fu) << 8) + 8 * lane);
          R.mw[i] = v >= 2 ? *reinterpret_cast<const uint32_t*>(sm_mid + (((e >> 16) & 0xFFu) << 7) + 4 * lane) : 0u;
          R.lw[i] = v == 3 ? *reinterpret_cast<const uint32_t*>(sm_low + ((e >> 24) << 7) + 4 * lane) : 0u;
        }
      };
      Rows cur_r, nxt_r;
      load_rows(cur_r, 0);
      for (int a = 0; S::KC * a < nk; ++a) {
        const bool more = S::KC * (a + 1) < nk;
        if (more) load_rows(nxt_r, a + 1);
        const int as = ka % S::NA;
        if (ka >= S::NA) Q9_WAIT(&aempty[as], ((ka / S::NA) - 1) & 1, w_b);
        // lane = tokens 8 lane .. + 7: atom column lane / 8, 16 B chunk lane % 8 (swizzled by the row)
        uint8_t* ach = abuf + as * S::ACH + (lane >> 3) * 1024;
        // the list is sorted T8, T12, T16 (then T8 padding): most 8-row groups are one class
        uint32_t notT8 = 0u;
#pragma unroll
        for (int i = 0; i < S::RPW; ++i) notT8 |= ((cur_r.e[i] >> 8) & 3u) ^ 1u;
        if (notT8 == 0u && !TRUNC) {
          const uint32_t c80 = 0x80808080u;
#pragma unroll
          for (int i = 0; i < S::RPW; ++i) {
            const int rl = S::RPW * bw + i;
            *reinterpret_cast<uint4*>(ach + (rl >> 3) * 4096 + (rl & 7) * 128 + (((lane & 7) ^ (rl & 7)) << 4)) =
                make_uint4(prmt(cur_r.hv[i].x, c80, 0x1404), prmt(cur_r.hv[i].x, c80, 0x3424),
                           prmt(cur_r.hv[i].y, c80, 0x1404), prmt(cur_r.hv[i].y, c80, 0x3424));
          }
        } else {
#pragma unroll
          for (int i = 0; i < S::RPW; ++i) {
            // branch-free: the word at full precision (absent nibbles are 0), then the row's tier
            // mask and midpoint fill: T8 keeps 8 bits (fill 0x80), T12 12 (fill 0x8), T16 all.
            // Rows past the list build channel 0 at "T0" and are never read by the MMA.
            const uint32_t sh = (3u - ((cur_r.e[i] >> 8) & 3u)) << 2;
            const uint32_t m16 = (0xFFFFu << sh) & 0xFFFFu, f16 = (1u << sh) >> 1;
            uint32_t mk = m16 * 0x00010001u, fl = f16 * 0x00010001u;
            if (TRUNC) {
              mk &= tkm;
              fl = tf;  // TRUNC rows are all T16: only the truncation applies
            }
            uint32_t w[4];
            assemble8(cur_r.hv[i].x, cur_r.hv[i].y, cur_r.mw[i], cur_r.lw[i], w);
#pragma unroll
            for (int k = 0; k < 4; ++k) w[k] = (w[k] & mk) | fl;
            const int rl = S::RPW * bw + i;
            *reinterpret_cast<uint4*>(ach + (rl >> 3) * 4096 + (rl & 7) * 128 + (((lane & 7) ^ (rl & 7)) << 4)) =
                make_uint4(w[0], w[1], w[2], w[3]);
          }
        }
#ifdef QK9_PROF
        const long long tf0_ = clock64();
#endif
#ifndef QK9_NOFENCE
        fence_async_smem();
#endif
        __syncwarp();
#ifdef QK9_PROF
        w_d += clock64() - tf0_;
#endif
        if (lane == 0) mbar_arrive1(&afull[as]);
        ++ka;
        if (more) cur_r = nxt_r;
      }
      __syncwarp();
      if (lane == 0) mbar_arrive1(&empty[slot]);
#ifdef QK9_PROF
      const long long tb1_ = clock64();
      w_e += tb1_ - tb0_;
#endif
      if (pv.lp >= 0) epilogue(pv, pv.u != c.u);
#ifdef QK9_PROF
      w_f += clock64() - tb1_;
#endif
      pv = Prev{kp, c.u, c.pg, c.up.n, ubi};
      ++kp;
      advance(c);
    }
    if (pv.lp >= 0) epilogue(pv, true);
  }
#ifdef QK9_PROF
  if ((blockIdx.x == 0 || blockIdx.x == 77) && lane == 0)
    printf("qk9 cta %d warp %d total %lld waits a %lld b %lld c %lld d %lld build %lld epi %lld\n", blockIdx.x, warp,
           clock64() - t_start, w_a, w_b, w_c, w_d, w_e, w_f);
#endif
  (void)w_a; (void)w_b; (void)w_c; (void)w_d; (void)w_e; (void)w_f;
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  if (warp == 1)
    asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem), "n"(S::TMEM_COLS) : "memory");
}

template <int G, bool TRUNC>
static void launch_qk9_t(const akv_store_t& s, const akv_cfg_t& cfg, const akv_step_t& st, int max_len,
                         cudaStream_t stream) {
  using S = Qk9Shape<G>;
  const int resident = resident_ctas<qk9_kernel<G, TRUNC>>(S::THREADS, S::SMEM);
  const int cap = s.max_pages * P;
  const int npg = (max_len + P - 1) / P;
  const long long items = (long long)s.n_units * npg;
  const int grid = (int)std::min<long long>(resident, std::max<long long>(items, 1));
  const float isd = (float)(1.0 / 11.313708498984761);  // 1/sqrt(128)
  launch_pdl(PDL_QK, qk9_kernel<G, TRUNC>, dim3(grid), dim3(S::THREADS), (size_t)S::SMEM, stream, s, cfg, st, cap, isd, npg);
}

}  // namespace akv
