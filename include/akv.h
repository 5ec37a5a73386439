/*
 * libakv — B200 (sm_100a) precision-aligned decode attention over a paged
 * bit-plane KV cache.  Plain C ABI: device pointers, sizes, POD structs and a
 * cudaStream_t passed as void*.  No torch types, no allocation, no global
 * state beyond cached device attributes; the caller owns every buffer.
 *
 * The reference exposes this path only as Python names (there is no FFI in
 * /root/reference).  Each entry point below cites the reference interface it
 * replaces:
 *   akv_append            <- KVStore.append_token
 *   akv_append_ws         <- KVStore.append (bulk / prefill) SPEC.md:233-241
 *   akv_read_elements     <- KVStore.read_element / read_channel SPEC.md:242-259
 *                            (+ split_chunks HB:154-157, ColMax/RowMax SPEC.md:219-226,278-279)
 *   akv_qk                <- attention_decode.scores_aligned SPEC.md:315-323
 *                            (k_channel_tiers/rule1_target SPEC.md:157-183,
 *                             required_mantissa_bits :139-147, read_channel :251-259)
 *   akv_softmax_select    <- attention_decode.softmax + estimate_output SPEC.md:324-341
 *                            (+ rule2_targets SPEC.md:166-174)
 *   akv_pv                <- attention_decode.output_aligned SPEC.md:342-350
 *   akv_combine           <- (split-K reduction; AttentionResult.o SPEC.md:309-312)
 *   akv_decode_step       <- the whole call stack SURVEY §3(2)
 *   akv_export_planes     <- PlaneTensor plane0/1/2 bytes
 *   akv_error_histogram   <- analysis.relative_error_histogram SPEC.md:410-418
 *
 * Errors: every call returns AKV_OK or a negative code.  Data-dependent
 * errors (non-finite append, degenerate q) are written to caller-provided
 * int64 status words that the host turns into ValueError /
 * DegenerateInputError (see AKV_STATUS_*).
 */
#ifndef AKV_H_
#define AKV_H_

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define AKV_VERSION 100 /* 1.0.0 */

#define AKV_HEAD_DIM 128      /* d; the only head_dim compiled in this round */
#define AKV_PAGE_TOKENS 256   /* tokens per page */
#define AKV_PAGE_BYTES 65536  /* head d*P + mid d*P/2 + low d*P/2 */
#define AKV_PAGE_MID_OFF 32768
#define AKV_PAGE_LOW_OFF 49152
#define AKV_MAX_GROUP 8       /* q heads per kv head */
#define AKV_MAX_KSEL 64

enum {
  AKV_OK = 0,
  AKV_EINVAL = -1,
  AKV_EUNSUPPORTED = -2,
  AKV_ECUDA = -3,
};

/* status word layout (int64):  bits 60..62 = code, rest = position */
#define AKV_STATUS_NONFINITE 1LL  /* [59]=V?, [40..47]=channel, [0..31]=token offset in the append */
#define AKV_STATUS_DEGENERATE 2LL /* degenerate dot product (no q_c!=0 with colmax_c!=0) */
#define AKV_STATUS_BAD_Q 3LL      /* non-finite q; [40..47]=channel */
#define AKV_STATUS_CAPACITY 4LL   /* append beyond the page table capacity */
#define AKV_STATUS_POSITION 5LL   /* akv_append_at position beyond the unit's length */

#define AKV_TARGET_UNKNOWN ((int32_t)0x80000000) /* rule2 target for o_est_r == 0 */

/* Paged bit-plane store.  A page holds AKV_PAGE_TOKENS tokens of one
 * (batch, kv-head) unit:
 *   K page: head [d][P] u8 (channel-major), mid/low [d][P/2] u8
 *   V page: head [P][d] u8 (token-major),  mid/low [P][d/2] u8
 * Nibbles are packed per 8-group (tokens for K, channels for V): byte i of the
 * group's 32-bit mid word = mid(i)<<4 | mid(i+4); of the low word =
 * low(i) | low(i+4)<<4 (i = 0..3).  akv_export_planes produces SPEC row-major
 * planes from this layout.                                                 */
typedef struct {
  int32_t n_units;      /* B * Hkv */
  int32_t head_dim;     /* must be AKV_HEAD_DIM */
  int32_t max_pages;    /* page_table row length; capacity = max_pages * P */
  int32_t pool_pages;   /* pages in k_pool / v_pool (0: n_units * max_pages); bounds the TMA tensor maps */
  uint8_t* k_pool;      /* [num_pool_pages][AKV_PAGE_BYTES] */
  uint8_t* v_pool;      /* [num_pool_pages][AKV_PAGE_BYTES] */
  const int32_t* page_table; /* [n_units][max_pages] pool page ids */
  int32_t* lengths;     /* [n_units] tokens stored (device) */
  uint32_t* colmax;     /* [n_units][d] |K| running max, fp16 pattern (sign clear) */
  uint16_t* rowmax;     /* [n_units][max_pages*P] max |V| per token, fp16 pattern */
} akv_store_t;

typedef struct {
  int32_t group;        /* q heads per kv head, 1..AKV_MAX_GROUP */
  int32_t margin_bits;  /* AlignConfig.margin_bits in [-2,4] */
  int32_t zero_skip;    /* AlignConfig.zero_skip */
  int32_t force_tier;   /* 0 = aligned; 8/12/16 = forced tier, estimation off (D8) */
  int32_t k_sel;        /* estimation cap (default 32); 0 = softmax only, no estimate */
  int32_t m;            /* estimation threshold exponent (default 5) */
  int32_t strategy;     /* 0 = element, 1 = row */
  int32_t trunc_bits;   /* 0 = off; 8..16 = baseline_truncated(bits), estimation off */
} akv_cfg_t;

/* Per-step buffers.  Rows are indexed by h = unit*group + j. */
typedef struct {
  const uint16_t* q;    /* [U*g][d] fp16 bits (in) */
  float* scores;        /* [U*g][cap] raw scores s_t (QK out) */
  float* probs;         /* [U*g][cap] softmax p_t (may alias scores) */
  float* page_stats;    /* [U*g][max_pages*P/32][2] per 32-token chunk (max, sum exp) */
  float* o_est;         /* [U*g][d] */
  int32_t* targets;     /* [U*g][d] rule2 targets (AKV_TARGET_UNKNOWN) */
  uint32_t* sel_bits;   /* [U*g][cap/32] selection bitmap */
  int32_t* sel_idx;     /* [U*g][AKV_MAX_KSEL] selected tokens, ascending */
  int32_t* head_meta;   /* [U*g][4] sel_count, min_target, any_unknown, n */
  float* head_metaf;    /* [U*g][4] M, L, pmax, thr */
  float* o_partial;     /* [U*g][max_pages][d] per-page partial outputs */
  float* o;             /* [U*g][d] attention output (out) */
  int64_t* counters;    /* [U*g][8] k8,k12,k16, v8,v12,v16, 0, 0 (elements) */
  int64_t* unit_bytes;  /* [U][4] physical plane bytes: K, V, 0, 0 */
  int64_t* status;      /* [U*g] */
  uint8_t* k_tiers;     /* [U*g][d] read-bit codes 0/8/12/16 (out) */
  uint8_t* v_tiers;     /* [U*g][cap][d] or NULL: per-element V codes (debug/parity) */
  uint32_t* work;       /* [8] reserved scratch (kept zero); the kernels use static work splits */
  uint32_t* need_bits;  /* [U*g][2][cap/32] V rows needing the mid / low nibble row (superset rule) */
} akv_step_t;

int akv_version(void);

/* Bytes of one contiguous workspace that akv_step_carve() splits into every
 * akv_step_t buffer except q, o and v_tiers.  Zero it once before its first
 * use (every per-step buffer is fully rewritten by the kernels each step). */
int64_t akv_workspace_bytes(int32_t n_units, int32_t group, int32_t max_pages);
int akv_step_carve(akv_step_t* step, void* workspace, int32_t n_units, int32_t group, int32_t max_pages);

/* Append n_new tokens per unit: k,v [U][n_new][d] fp16 bits.  status [U].
 * Non-finite input or a full page table rejects that unit's whole append
 * (length unchanged).  Status words are sticky: the kernels write only error
 * codes, keep the first one, and a multi-token append refuses a unit whose
 * word is already non-zero; the caller zeroes status before an append whose
 * outcome it reads (KVStore.append does), so errors survive graph replays. */
int akv_append(const akv_store_t* store, const uint16_t* k, const uint16_t* v, int32_t n_new,
               int64_t* status, void* stream);

/* Truncate every unit to pos tokens (pos <= its length, else AKV_STATUS_POSITION and the
 * unit is unchanged) and append one token there (length = pos + 1): a rollback of
 * speculative tokens, or a fixed-context replay (benchmarks, DecodeGraph(rewind_to)) in one
 * launch.  ColMax keeps the running max over every token ever appended (SPEC.md:219-222 is
 * a running max; withdrawing a truncated token's contribution is not possible), so K tiers
 * stay sound.  Same validation and sticky status words as akv_append.  Extension: the
 * reference has no truncation. */
int akv_append_at(const akv_store_t* store, const uint16_t* k, const uint16_t* v, int32_t pos, int64_t* status,
                  void* stream);

/* Bulk append (prefill writer) with a caller workspace of
 * akv_append_workspace_bytes(n_units, n_new) bytes (no zeroing needed): one CTA per
 * (unit, page span) stages the span's K rows in shared memory and writes the
 * channel-major K planes / token-major V planes with 16 B stores, validation fused
 * in; a per-unit commit rejects the whole append (same status words and stickiness
 * as akv_append) or folds the ColMax partials and bumps the length.  k, v 16 B
 * aligned.  n_new == 1 runs akv_append.  Replaces KVStore.append (bulk form,
 * SPEC.md:233-241). */
int64_t akv_append_workspace_bytes(int32_t n_units, int32_t n_new);
int akv_append_ws(const akv_store_t* store, const uint16_t* k, const uint16_t* v, int32_t n_new, int64_t* status,
                  void* workspace, int64_t workspace_bytes, void* stream);

/* Metered reads: n requests (unit, token, channel, tier code 0/8/12/16) of plane set
 * which (0 = K, 1 = V); out[i] = the word rebuilt at the tier with the midpoint fill
 * (SKIP -> 0); counters[3] (int64, device) += elements read at T8 / T12 / T16.  Only the
 * planes a tier needs are touched.  Out-of-range requests give 0 and are not counted.
 * Replaces KVStore.read_element / read_channel. */
int akv_read_elements(const akv_store_t* store, int32_t which, const int32_t* unit, const int32_t* tok,
                      const int32_t* chan, const int32_t* tier, int64_t n, uint16_t* out, int64_t* counters,
                      void* stream);

/* max_len: host-side upper bound on lengths[] (sizes the grid). */
int akv_qk(const akv_store_t* store, const akv_cfg_t* cfg, const akv_step_t* step, int32_t max_len,
           void* stream);
int akv_softmax_select(const akv_store_t* store, const akv_cfg_t* cfg, const akv_step_t* step,
                       int32_t max_len, void* stream);
int akv_pv(const akv_store_t* store, const akv_cfg_t* cfg, const akv_step_t* step, int32_t max_len,
           void* stream);
int akv_combine(const akv_store_t* store, const akv_cfg_t* cfg, const akv_step_t* step, int32_t max_len,
                void* stream);
/* qk -> softmax_select -> pv -> combine on one stream. */
int akv_decode_step(const akv_store_t* store, const akv_cfg_t* cfg, const akv_step_t* step,
                    int32_t max_len, void* stream);

/* SPEC row-major planes for every unit: plane0 [U][cap][d], plane1/2
 * [U][cap][d/2] (byte j = nib[2j] | nib[2j+1]<<4).  which: 0 = K, 1 = V. */
int akv_export_planes(const akv_store_t* store, int32_t which, uint8_t* plane0, uint8_t* plane1,
                      uint8_t* plane2, void* stream);

/* relative_error_histogram over n device (test, ref) fp32
 * pairs into counts[6] (int64, device; zeroed by the call): buckets {0},
 * (0,2^-10), [2^-10,2^-9), [2^-9,2^-8), [2^-8,2^-7), [2^-7,inf).  fp16_round:
 * round both to the fp16 grid first (A-hist, HB:187-190). */
int akv_error_histogram(const float* test, const float* ref, int64_t n, int32_t fp16_round, int64_t* counts,
                        void* stream);

#ifdef __cplusplus
}
#endif
#endif /* AKV_H_ */
