// Host-side validation and tile schedule for parse_verify_attn.
//
// the packed sequence (N shared rows + K appended
// suffix copies of S rows) is cut into 128-row Q tiles; each tile lists only
// the 128-key KV tiles its rows can see — draft tiles [0, ceil(max b/128))
// and the tile(s) holding its own suffix copy.  KV tiles that are fully
// masked for every row of a tile are never emitted (north_star: "fully masked
// draft tiles beyond b_k are skipped rather than computed").
#include <algorithm>
#include <cmath>
#include <cstring>

#include "internal.h"

namespace parse {

static inline int cdiv(long long a, long long b) { return int((a + b - 1) / b); }

parse_status_t make_problem(const parse_attn_desc_t* d, Problem* p, std::string* err) {
  if (!d) { *err = "desc is NULL"; return PARSE_ERR_INVALID; }
  if (d->batch < 1 || d->num_q_heads < 1 || d->num_kv_heads < 1) {
    *err = "batch, num_q_heads, num_kv_heads must be >= 1"; return PARSE_ERR_INVALID;
  }
  if (d->num_q_heads % d->num_kv_heads) {
    *err = "num_q_heads must be a multiple of num_kv_heads"; return PARSE_ERR_INVALID;
  }
  if (d->draft_len < 1 || d->num_suffixes < 1 || d->suffix_len < 1) {
    *err = "draft_len, num_suffixes, suffix_len must be >= 1"; return PARSE_ERR_INVALID;
  }
  if (d->head_dim != 64 && d->head_dim != 128) {
    *err = "head_dim must be 64 or 128"; return PARSE_ERR_UNSUPPORTED;
  }
  long long L = (long long)d->draft_len + (long long)d->num_suffixes * d->suffix_len;
  if (L > (1ll << 30)) { *err = "packed length too large"; return PARSE_ERR_INVALID; }
  if (!d->boundaries) { *err = "boundaries is NULL"; return PARSE_ERR_INVALID; }
  if (d->boundary_batch_stride < 0) { *err = "boundary_batch_stride < 0"; return PARSE_ERR_INVALID; }
  const int64_t* strides[4] = {d->q_strides, d->k_strides, d->v_strides, d->o_strides};
  const char* names[4] = {"q", "k", "v", "o"};
  for (int t = 0; t < 4; ++t)
    for (int i = 0; i < 3; ++i) {
      int64_t s = strides[t][i];
      if (s <= 0 || (s % 8) != 0 || s >= (1ll << 36)) {
        *err = std::string(names[t]) + "_strides must be positive multiples of 8 elements";
        return PARSE_ERR_INVALID;
      }
    }
  p->B = d->batch; p->Hq = d->num_q_heads; p->Hkv = d->num_kv_heads; p->D = d->head_dim;
  p->N = d->draft_len; p->K = d->num_suffixes; p->S = d->suffix_len; p->L = int(L);
  p->bnd.resize(size_t(p->B) * p->K);
  for (int b = 0; b < p->B; ++b)
    for (int k = 0; k < p->K; ++k) {
      int32_t v = d->boundaries[b * d->boundary_batch_stride + k];
      if (v < 0 || v > p->N) {
        *err = "boundary b[" + std::to_string(b) + "][" + std::to_string(k) + "]=" +
               std::to_string(v) + " outside [0, draft_len]";
        return PARSE_ERR_INVALID;
      }
      p->bnd[size_t(b) * p->K + k] = v;
    }
  p->tree = d->tree_parent != nullptr;
  p->anc.clear();
  if (p->tree) {
    if (p->S > kMaxTreeS) { *err = "tree masks need suffix_len <= 64"; return PARSE_ERR_UNSUPPORTED; }
    p->anc.resize(p->S);
    for (int s = 0; s < p->S; ++s) {
      int par = d->tree_parent[s];
      if (!(par == -1 || (par >= 0 && par < s))) {
        *err = "tree_parent[" + std::to_string(s) + "] must be -1 or in [0, s)";
        return PARSE_ERR_INVALID;
      }
      p->anc[s] = (uint64_t(1) << s) | (par >= 0 ? p->anc[par] : 0);
    }
  }
  p->scale = d->softmax_scale > 0.f ? d->softmax_scale : 1.0f / std::sqrt(float(p->D));
  return PARSE_OK;
}

int suffix_heads_per_tile(const Problem& p) {
  const int r = p.Hq / p.Hkv;
  if (p.S > kTile || (kTile % p.S) != 0) return 0;
  const int hpt = kTile / p.S;
  if (hpt > r || (r % hpt) != 0) return 0;
  return hpt;
}

namespace {

struct TileSpec { int t0, t_end, self_lo, n_draft, n_self; };

// Token-major tile of rows [t0, t_end) for request b (rows may straddle the
// shared/suffix border and several suffix copies).
TileSpec token_tile(const Problem& p, int b, int t0, int t_end) {
  TileSpec ts{t0, t_end, 0, 0, 0};
  int max_lim = 0;
  if (t0 < p.N) max_lim = std::min(t_end, p.N);            // draft rows: lim = t + 1
  if (t_end > p.N) {                                       // suffix rows
    int k_lo = (std::max(t0, p.N) - p.N) / p.S;
    int k_hi = (t_end - 1 - p.N) / p.S;
    for (int k = k_lo; k <= k_hi; ++k) max_lim = std::max(max_lim, p.bnd[size_t(b) * p.K + k]);
    ts.self_lo = p.N + k_lo * p.S;
    ts.n_self = cdiv(t_end - ts.self_lo, kTile);
  }
  ts.n_draft = cdiv(max_lim, kTile);
  return ts;
}

template <class F>
void for_each_item(const Problem& p, F&& emit) {
  const int r = p.Hq / p.Hkv;
  const int hpt_s = suffix_heads_per_tile(p);
  const int tok_end = hpt_s ? p.N : p.L;
  for (int t0 = 0; t0 < tok_end; t0 += kTile) {
    const int t_end = std::min(t0 + kTile, tok_end);
    for (int b = 0; b < p.B; ++b) {
      TileSpec ts = token_tile(p, b, t0, t_end);
      for (int g = 0; g < p.Hkv; ++g)
        for (int hh = 0; hh < r; hh += 2) {
          const int nq = (hh + 1 < r) ? 2 : 1;
          emit(WorkItem{b, g * r + hh, ts.t0, ts.t_end, ts.self_lo, ts.n_draft, ts.n_self,
                        1 | ((nq == 2) << 8)});
        }
    }
  }
  if (hpt_s) {
    const int ntile = r / hpt_s;
    for (int b = 0; b < p.B; ++b) {
      if (ntile >= 2) {
        // two head-packs of one copy per item (identical visibility)
        for (int k = 0; k < p.K; ++k) {
          const int t0 = p.N + k * p.S;
          const int n_draft = cdiv(p.bnd[size_t(b) * p.K + k], kTile);
          for (int g = 0; g < p.Hkv; ++g)
            for (int ti = 0; ti < ntile; ti += 2) {
              const int nq = (ti + 1 < ntile) ? 2 : 1;
              emit(WorkItem{b, g * r + ti * hpt_s, t0, t0 + p.S, t0, n_draft, 1, hpt_s | ((nq == 2) << 8)});
            }
        }
      } else {
        // one head-pack covers the group: pair copies k and k+1 (tile 1 = next
        // copy, same heads).  The KV range is the union; each row keeps its
        // own boundary through the mask, and one self tile holds both copies
        // when 2S <= 128.
        const bool can_pair = 2 * p.S <= kTile;
        for (int k = 0; k < p.K; k += can_pair ? 2 : 1) {
          const int nq = (can_pair && k + 1 < p.K) ? 2 : 1;
          const int t0 = p.N + k * p.S;
          int lim = p.bnd[size_t(b) * p.K + k];
          if (nq == 2) lim = std::max(lim, p.bnd[size_t(b) * p.K + k + 1]);
          const int n_draft = cdiv(lim, kTile);
          for (int g = 0; g < p.Hkv; ++g)
            emit(WorkItem{b, g * r, t0, t0 + nq * p.S, t0, n_draft, 1,
                          hpt_s | ((nq == 2) << 8) | ((nq == 2) << 9)});
        }
      }
    }
  }
}

}  // namespace

size_t count_schedule(const Problem& p) {
  size_t n = 0;
  for_each_item(p, [&](const WorkItem&) { ++n; });
  return n;
}

// Group-major order: all items of one (request, KV-head group) are adjacent,
// largest first within the group.  The kernel hands items out dynamically in
// this order, so the ~148 items in flight at any time read the same group's
// K/V (4 MB at N=8192) from L2, and the tail of the launch is made of the
// last group's smallest items (imbalance <= one small item per CTA).
void build_schedule(const Problem& p, std::vector<WorkItem>* items) {
  items->clear();
  items->reserve(count_schedule(p));
  for_each_item(p, [&](const WorkItem& w) { items->push_back(w); });
  const int r = p.Hq / p.Hkv;
  auto cost = [](const WorkItem& w) { return (w.n_draft + w.n_self) * ((w.flags >> 8) & 1 ? 2 : 1); };
  std::stable_sort(items->begin(), items->end(), [&](const WorkItem& a, const WorkItem& b) {
    const int ga = a.b * p.Hkv + a.h0 / r, gb = b.b * p.Hkv + b.h0 / r;
    if (ga != gb) return ga < gb;
    return cost(a) > cost(b);
  });
}

WorkspaceLayout workspace_layout(const Problem& p, bool need_items) {
  auto al = [](size_t x) { return (x + 255) & ~size_t(255); };
  WorkspaceLayout w{};
  w.counter_off = 0;
  w.bnd_off = 256;
  w.anc_off = al(w.bnd_off + sizeof(int32_t) * size_t(p.B) * p.K);
  w.items_off = al(w.anc_off + sizeof(uint64_t) * size_t(p.tree ? p.S : 0));
  w.n_items = need_items ? count_schedule(p) : 0;
  w.total = al(w.items_off + sizeof(WorkItem) * w.n_items);
  return w;
}

}  // namespace parse
