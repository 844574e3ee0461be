// plan.cpp — automatic configuration (NEXT-3): the paper's memory model (§3.5,
// App. B, PAPER.md:318-337 / 498-552) and its Eq. (1) tier / pipeline choice
// (PAPER.md:339-357), plus the App. A block-size pick.
// Host-only, pure functions; readings Q23-Q27 in DESIGN.md.
//
// Arithmetic: bytes as doubles.  Every term is an integer times a precision that is
// a dyadic rational (2, 17/32, ...), so with magnitudes < 2^48 all sums and products
// below are exact — the result does not depend on evaluation order.
#include <algorithm>
#include <cmath>

#include "host.h"

namespace {

bool spec_ok(const pipo_mem_spec* sp) {
  return sp && sp->n_layers >= 1 && sp->d_model >= 1 && sp->vocab >= 1 && sp->n_heads >= 1 && sp->n_kv_heads >= 1 &&
         sp->n_kv_heads <= sp->n_heads && sp->n_heads % sp->n_kv_heads == 0 && sp->ffn_hidden >= 1 &&
         (sp->mlp_mats == 2 || sp->mlp_mats == 3) && sp->p_weight > 0 && sp->p_act > 0 &&
         std::isfinite(sp->p_weight) && std::isfinite(sp->p_act);
}

}  // namespace

extern "C" {

int64_t pipo_ffn_hidden_dim(int64_t d, int64_t m, double gamma) {
  // d_h = m * ceil(gamma * floor(8d/3) / m)
  if (d < 1 || m < 1 || !(gamma > 0)) return -1;
  return m * (int64_t)std::ceil(gamma * (double)((8 * d) / 3) / (double)m);
}

pipo_status pipo_memory_model(const pipo_mem_spec* sp, int64_t b, int64_t s, int32_t stage, int32_t preload,
                              pipo_mem_report* out) {
  if (!spec_ok(sp) || !out || b < 1 || s < 0 || (stage != PIPO_STAGE_PREFILL && stage != PIPO_STAGE_DECODE))
    return pipo::set_last_error(PIPO_E_INVALID_ARG, "bad memory-model arguments");
  const double pw = sp->p_weight, pa = sp->p_act;
  const double d = (double)sp->d_model, V = (double)sp->vocab, h = (double)sp->n_heads, dh = (double)sp->ffn_hidden;
  const double l = (double)sp->n_layers, B = (double)b, S = (double)s, mm = (double)sp->mlp_mats;
  // d h_kv / h (the K or V width under GQA), exact whenever h | d h_kv (head_dim integral)
  const double dkv = (double)(sp->d_model * sp->n_kv_heads) / h;
  pipo_mem_report o{};
  // §3.5: W_embed = p d V; W_mha = p d (2d + 2d h_kv/h + 1) (App. B form, Q23); W_mlp = p d (3 d_h + 1)
  o.w_embed = pw * d * V;
  o.w_mha = pw * d * (2 * d + 2 * dkv + 1);
  o.w_mlp = pw * d * (mm * dh + 1);
  o.w_total = 2 * o.w_embed + l * (o.w_mha + o.w_mlp);
  // C = 2 p b s l d h_kv / h
  o.c_total = 2 * pa * B * S * l * dkv;
  const double kv1 = 2 * pa * B * S * dkv;   // C / l
  if (stage == PIPO_STAGE_PREFILL) {
    o.m_mha = pa * B * S * (5 * d + h * S) + o.w_mha + (preload ? o.w_mlp : 0.0) + kv1;
    o.m_mlp = pa * B * S * (mm * dh + 2 * d) + o.w_mlp + (preload ? o.w_mha : 0.0);
    o.m_embed = pa * B * S * (d + V) + (preload ? std::max(o.w_mha, o.w_embed) : 0.0) + o.w_embed;
  } else if (preload) {
    // App. B decoding with preloading, expanded forms (Q24): 4 p b s d h_kv/h = 2 C / l
    o.m_mha = pa * B * (5 * d + h) + o.w_mha + o.w_mlp + 2 * kv1;
    o.m_mlp = pa * B * (mm * dh + 2 * d) + o.w_mlp + o.w_mha + 2 * kv1;
    o.m_embed = pa * B * (d + V) + std::max(o.w_mha, o.w_embed) + o.w_embed;
  } else {
    o.m_mha = pa * B * (5 * d + h * S) + o.w_mha + kv1;
    o.m_mlp = pa * B * (mm * dh + 2 * d) + o.w_mlp;
    o.m_embed = pa * B * (d + V) + o.w_embed;
  }
  o.m_peak = std::max(o.m_mha, std::max(o.m_mlp, o.m_embed));
  *out = o;
  return PIPO_OK;
}

int64_t pipo_choose_block_size(const int64_t* sizes, const double* h2d_bps, const double* disk_bps, int32_t n) {
  // smallest probed size whose min-over-edges throughput is within 5 % of the best (Q26)
  if (!sizes || !h2d_bps || n < 1) return -1;
  double best = 0;
  for (int i = 0; i < n; ++i) best = std::max(best, disk_bps ? std::min(h2d_bps[i], disk_bps[i]) : h2d_bps[i]);
  int64_t pick = -1;
  for (int i = 0; i < n; ++i) {
    const double e = disk_bps ? std::min(h2d_bps[i], disk_bps[i]) : h2d_bps[i];
    if (e >= 0.95 * best && (pick < 0 || sizes[i] < pick)) pick = sizes[i];
  }
  return pick;
}

pipo_status pipo_choose_plan(const pipo_mem_spec* sp, int64_t b, int64_t s, const pipo_hw_spec* hw,
                             const int64_t* block_sizes, const double* h2d_bps, const double* disk_bps,
                             int32_t n_sizes, pipo_plan* out) {
  if (!spec_ok(sp) || !hw || !out || b < 1 || s < 1 || !(hw->m_gpu > 0) || !(hw->m_cpu > 0) || !(hw->b_gpu > 0) ||
      !(hw->b_ssd > 0))
    return pipo::set_last_error(PIPO_E_INVALID_ARG, "bad plan arguments");
  pipo_mem_report pre{}, pre_nopl{};
  pipo_status st = pipo_memory_model(sp, b, s, PIPO_STAGE_PREFILL, 1, &pre);
  if (st != PIPO_OK) return st;
  st = pipo_memory_model(sp, b, s, PIPO_STAGE_PREFILL, 0, &pre_nopl);
  if (st != PIPO_OK) return st;
  pipo_plan p{};
  const double W = pre.w_total, C = pre.c_total, M = pre.m_peak;
  // Eq. (1): weight tier, as an else-chain
  if (W + M < hw->m_gpu) p.weight_tier = PIPO_TIER_DEVICE;
  else if (W + C < hw->m_cpu && hw->b_ssd < hw->b_gpu) p.weight_tier = PIPO_TIER_HOST;
  else p.weight_tier = PIPO_TIER_DISK;
  // Eq. (1): pipeline; memory-efficient must still fit its own (no-preload) peak (Q25)
  if (M < hw->m_gpu) p.ring_layers = 2;
  else if (pre_nopl.m_peak < hw->m_gpu) p.ring_layers = 1;
  else return pipo::set_last_error(PIPO_E_INFEASIBLE, "even the memory-efficient pipeline exceeds M_GPU");
  // §3.5 / PAPER.md:360: the INT4 compute kernel below batch 16
  p.use_quant_kernel = (sp->p_weight < 2.0 && b < 16) ? 1 : 0;
  p.gemv_max_m = 15;
  p.block_bytes = (n_sizes > 0 && block_sizes && h2d_bps) ? pipo_choose_block_size(block_sizes, h2d_bps, disk_bps, n_sizes)
                                                         : 0;
  p.w_total = W;
  p.c_total = C;
  p.m_peak = M;
  p.m_peak_no_preload = pre_nopl.m_peak;
  *out = p;
  return PIPO_OK;
}

}  // extern "C"
