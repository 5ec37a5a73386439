// extern "C" entry points of libakv (declared in include/akv.h).
#include "akv_common.cuh"

namespace akv {
void launch_qk(const akv_store_t&, const akv_cfg_t&, const akv_step_t&, int, cudaStream_t);
void launch_select(const akv_store_t&, const akv_cfg_t&, const akv_step_t&, int, cudaStream_t);
void launch_pv(const akv_store_t&, const akv_cfg_t&, const akv_step_t&, int, cudaStream_t);
void launch_combine(const akv_store_t&, const akv_cfg_t&, const akv_step_t&, cudaStream_t);

// SPEC row-major planes from the paged layout.
__global__ void export_planes_kernel(akv_store_t s, int which, uint8_t* p0, uint8_t* p1, uint8_t* p2) {
  const int u = blockIdx.y;
  const int cap = s.max_pages * P;
  const int n = s.lengths[u];
  const uint8_t* pool = which ? s.v_pool : s.k_pool;
  for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < n * (D / 2); i += gridDim.x * blockDim.x) {
    const int t = i / (D / 2), c = 2 * (i % (D / 2));
    const uint8_t* pp = page_ptr(pool, s.page_table, s.max_pages, u, t / P);
    const int tt = t % P;
    uint32_t hd[2], md[2], lo[2];
#pragma unroll
    for (int e = 0; e < 2; ++e) {
      const int ch = c + e;
      if (which == 0) {  // K: channel-major, nibble groups over tokens
        hd[e] = pp[ch * P + tt];
        const int byte = ch * (P / 2) + (tt >> 3) * 4 + (tt & 3);
        const bool first = (tt & 7) < 4;
        md[e] = first ? pp[MID + byte] >> 4 : pp[MID + byte] & 0xF;
        lo[e] = first ? pp[LOW + byte] & 0xF : pp[LOW + byte] >> 4;
      } else {  // V: token-major, nibble groups over channels
        hd[e] = pp[tt * D + ch];
        const int byte = tt * (D / 2) + (ch >> 3) * 4 + (ch & 3);
        const bool first = (ch & 7) < 4;
        md[e] = first ? pp[MID + byte] >> 4 : pp[MID + byte] & 0xF;
        lo[e] = first ? pp[LOW + byte] & 0xF : pp[LOW + byte] >> 4;
      }
    }
    const size_t row = (size_t)u * cap + t;
    p0[row * D + c] = (uint8_t)hd[0];
    p0[row * D + c + 1] = (uint8_t)hd[1];
    p1[row * (D / 2) + c / 2] = (uint8_t)(md[0] | (md[1] << 4));
    p2[row * (D / 2) + c / 2] = (uint8_t)(lo[0] | (lo[1] << 4));
  }
}

static int check(const akv_store_t* s, const akv_cfg_t* c, const akv_step_t* st) {
  if (!s || !c || !st) return AKV_EINVAL;
  if (s->head_dim != D) return AKV_EUNSUPPORTED;
  if (!(c->group == 1 || c->group == 2 || c->group == 4 || c->group == 8)) return AKV_EUNSUPPORTED;
  if (c->margin_bits < -2 || c->margin_bits > 4) return AKV_EINVAL;
  if (!(c->force_tier == 0 || c->force_tier == 8 || c->force_tier == 12 || c->force_tier == 16)) return AKV_EINVAL;
  if (c->trunc_bits && (c->trunc_bits < 8 || c->trunc_bits > 16)) return AKV_EINVAL;
  if (c->k_sel < 0 || c->k_sel > AKV_MAX_KSEL || c->m < 0 || c->m > 126) return AKV_EINVAL;
  if (c->strategy != 0 && c->strategy != 1) return AKV_EINVAL;
  return AKV_OK;
}

static int last_error() { return cudaGetLastError() == cudaSuccess ? AKV_OK : AKV_ECUDA; }

}  // namespace akv

using namespace akv;

extern "C" int akv_version(void) { return AKV_VERSION; }

static inline int64_t align256(int64_t x) { return (x + 255) & ~(int64_t)255; }

static int64_t carve(akv_step_t* st, uint8_t* ws, int32_t U, int32_t G, int32_t max_pages) {
  const int64_t H = (int64_t)U * G, cap = (int64_t)max_pages * P;
  int64_t off = 0;
  auto take = [&](int64_t bytes) {
    uint8_t* p = ws ? ws + off : nullptr;
    off += align256(bytes);
    return p;
  };
  uint8_t* scores = take(H * cap * 4);
  uint8_t* page_stats = take(H * max_pages * (P / 32) * 2 * 4);
  uint8_t* o_est = take(H * D * 4);
  uint8_t* targets = take(H * D * 4);
  uint8_t* sel_bits = take(H * (cap / 32) * 4);
  uint8_t* sel_idx = take(H * AKV_MAX_KSEL * 4);
  uint8_t* head_meta = take(H * 4 * 4);
  uint8_t* head_metaf = take(H * 4 * 4);
  uint8_t* o_partial = take(H * max_pages * D * 4);
  uint8_t* counters = take(H * 8 * 8);
  uint8_t* unit_bytes = take((int64_t)U * 4 * 8);
  uint8_t* status = take(H * 8);
  uint8_t* k_tiers = take(H * D);
  uint8_t* work = take(8 * 4);
  uint8_t* need_bits = take(H * 2 * (cap / 32) * 4);
  if (st) {
    st->scores = reinterpret_cast<float*>(scores);
    st->probs = reinterpret_cast<float*>(scores);
    st->page_stats = reinterpret_cast<float*>(page_stats);
    st->o_est = reinterpret_cast<float*>(o_est);
    st->targets = reinterpret_cast<int32_t*>(targets);
    st->sel_bits = reinterpret_cast<uint32_t*>(sel_bits);
    st->sel_idx = reinterpret_cast<int32_t*>(sel_idx);
    st->head_meta = reinterpret_cast<int32_t*>(head_meta);
    st->head_metaf = reinterpret_cast<float*>(head_metaf);
    st->o_partial = reinterpret_cast<float*>(o_partial);
    st->counters = reinterpret_cast<int64_t*>(counters);
    st->unit_bytes = reinterpret_cast<int64_t*>(unit_bytes);
    st->status = reinterpret_cast<int64_t*>(status);
    st->k_tiers = k_tiers;
    st->work = reinterpret_cast<uint32_t*>(work);
    st->need_bits = reinterpret_cast<uint32_t*>(need_bits);
  }
  return off;
}

extern "C" int64_t akv_workspace_bytes(int32_t n_units, int32_t group, int32_t max_pages) {
  if (n_units < 0 || group < 1 || max_pages < 0) return AKV_EINVAL;
  return carve(nullptr, nullptr, n_units, group, max_pages);
}

extern "C" int akv_step_carve(akv_step_t* step, void* workspace, int32_t n_units, int32_t group, int32_t max_pages) {
  if (!step || !workspace) return AKV_EINVAL;
  if ((reinterpret_cast<uintptr_t>(workspace) & 255) != 0) return AKV_EINVAL;
  carve(step, static_cast<uint8_t*>(workspace), n_units, group, max_pages);
  return AKV_OK;
}

extern "C" int akv_qk(const akv_store_t* s, const akv_cfg_t* c, const akv_step_t* st, int32_t max_len,
                      void* stream) {
  int e = check(s, c, st);
  if (e) return e;
  if (max_len <= 0 || s->n_units == 0) return AKV_OK;
  launch_qk(*s, *c, *st, max_len, (cudaStream_t)stream);
  return last_error();
}

extern "C" int akv_softmax_select(const akv_store_t* s, const akv_cfg_t* c, const akv_step_t* st, int32_t max_len,
                                  void* stream) {
  int e = check(s, c, st);
  if (e) return e;
  if (max_len <= 0 || s->n_units == 0) return AKV_OK;
  launch_select(*s, *c, *st, max_len, (cudaStream_t)stream);
  return last_error();
}

extern "C" int akv_pv(const akv_store_t* s, const akv_cfg_t* c, const akv_step_t* st, int32_t max_len,
                      void* stream) {
  int e = check(s, c, st);
  if (e) return e;
  if (max_len <= 0 || s->n_units == 0) return AKV_OK;
  launch_pv(*s, *c, *st, max_len, (cudaStream_t)stream);
  return last_error();
}

extern "C" int akv_combine(const akv_store_t* s, const akv_cfg_t* c, const akv_step_t* st, int32_t max_len,
                           void* stream) {
  int e = check(s, c, st);
  if (e) return e;
  if (max_len <= 0 || s->n_units == 0) return AKV_OK;
  launch_combine(*s, *c, *st, (cudaStream_t)stream);
  return last_error();
}

extern "C" int akv_decode_step(const akv_store_t* s, const akv_cfg_t* c, const akv_step_t* st, int32_t max_len,
                               void* stream) {
  int e = check(s, c, st);
  if (e) return e;
  if (max_len <= 0 || s->n_units == 0) return AKV_OK;
  cudaStream_t cs = (cudaStream_t)stream;
  launch_qk(*s, *c, *st, max_len, cs);
  launch_select(*s, *c, *st, max_len, cs);
  launch_pv(*s, *c, *st, max_len, cs);
  launch_combine(*s, *c, *st, cs);
  return last_error();
}

extern "C" int akv_export_planes(const akv_store_t* s, int32_t which, uint8_t* p0, uint8_t* p1, uint8_t* p2,
                                 void* stream) {
  if (!s || !p0 || !p1 || !p2 || (which != 0 && which != 1)) return AKV_EINVAL;
  if (s->head_dim != D) return AKV_EUNSUPPORTED;
  if (s->n_units == 0) return AKV_OK;
  dim3 grid(64, s->n_units);
  export_planes_kernel<<<grid, 256, 0, (cudaStream_t)stream>>>(*s, which, p0, p1, p2);
  return last_error();
}
