// Host-side validation and tile schedule for parse_verify_attn.
//
// the packed sequence (N shared rows + K appended
// suffix copies of S rows) is cut into 128-row Q tiles; each tile lists only
// the 128-key KV tiles its rows can see — draft tiles [0, ceil(max b/128))
// and the tile(s) holding its own suffix copy.  KV tiles that are fully
// masked for every row of a tile are never emitted (north_star: "fully masked
// draft tiles beyond b_k are skipped rather than computed").
#include <array>
#include <map>
#include <algorithm>
#include <cmath>
#include <cstring>

#include "internal.h"

namespace parse {

static inline int cdiv(long long a, long long b) { return int((a + b - 1) / b); }
static inline int align_down(int x, int a) { return x - x % a; }

static parse_status_t finish_problem(const int16_t* tree_parent, float softmax_scale, Problem* p,
                                     std::string* err) {
  p->tree = tree_parent != nullptr;
  p->anc.clear();
  if (p->tree) {
    if (p->S > kMaxTreeS) { *err = "tree masks need suffix_len <= 64"; return PARSE_ERR_UNSUPPORTED; }
    p->anc.resize(p->S);
    for (int s = 0; s < p->S; ++s) {
      int par = tree_parent[s];
      if (!(par == -1 || (par >= 0 && par < s))) {
        *err = "tree_parent[" + std::to_string(s) + "] must be -1 or in [0, s)";
        return PARSE_ERR_INVALID;
      }
      p->anc[s] = (uint64_t(1) << s) | (par >= 0 ? p->anc[par] : 0);
    }
  }
  p->scale = softmax_scale > 0.f ? softmax_scale : 1.0f / std::sqrt(float(p->D));
  return PARSE_OK;
}

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
  p->varlen = false;
  p->Nb.assign(p->B, p->N);
  p->Kb.assign(p->B, p->K);
  p->bnd_off.resize(p->B);
  for (int b = 0; b < p->B; ++b) p->bnd_off[b] = b * p->K;
  p->q_row0.assign(p->B, 0);
  p->kv_row0.assign(p->B, 0);
  if ((long long)p->B * p->K > (1ll << 30)) { *err = "batch * num_suffixes too large"; return PARSE_ERR_INVALID; }
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
  return finish_problem(d->tree_parent, d->softmax_scale, p, err);
}

parse_status_t make_problem_varlen(const parse_varlen_desc_t* d, Problem* p, std::string* err) {
  if (!d) { *err = "desc is NULL"; return PARSE_ERR_INVALID; }
  if (d->batch < 1 || d->num_q_heads < 1 || d->num_kv_heads < 1) {
    *err = "batch, num_q_heads, num_kv_heads must be >= 1"; return PARSE_ERR_INVALID;
  }
  if (d->num_q_heads % d->num_kv_heads) {
    *err = "num_q_heads must be a multiple of num_kv_heads"; return PARSE_ERR_INVALID;
  }
  if (d->suffix_len < 1) { *err = "suffix_len must be >= 1"; return PARSE_ERR_INVALID; }
  if (d->head_dim != 64 && d->head_dim != 128) { *err = "head_dim must be 64 or 128"; return PARSE_ERR_UNSUPPORTED; }
  if (!d->draft_lens || !d->num_suffixes || !d->row_offsets) {
    *err = "draft_lens, num_suffixes, row_offsets must be non-NULL"; return PARSE_ERR_INVALID;
  }
  if (d->total_rows < 1 || d->total_rows >= (1ll << 31)) { *err = "total_rows must be in [1, 2^31)"; return PARSE_ERR_INVALID; }
  const bool paged = d->page_size != 0;
  if (paged) {
    if (d->page_size < 16 || (d->page_size & (d->page_size - 1)) || d->page_size > (1 << 20)) {
      *err = "page_size must be a power of two in [16, 2^20]"; return PARSE_ERR_INVALID;
    }
    if (d->num_pages < 1 || !d->block_table || d->block_table_stride < 1) {
      *err = "paged K/V needs num_pages >= 1, block_table and block_table_stride >= 1"; return PARSE_ERR_INVALID;
    }
  } else if (d->kv_row_offsets && (d->kv_total_rows < 1 || d->kv_total_rows >= (1ll << 31))) {
    *err = "kv_total_rows must be in [1, 2^31)"; return PARSE_ERR_INVALID;
  }
  auto bad_stride = [](int64_t s) { return s <= 0 || (s % 8) != 0 || s >= (1ll << 36); };
  for (int i = 0; i < 2; ++i)
    if (bad_stride(d->q_strides[i]) || bad_stride(d->o_strides[i])) {
      *err = "q_strides / o_strides must be positive multiples of 8 elements"; return PARSE_ERR_INVALID;
    }
  for (int i = 0; i < (paged ? 3 : 2); ++i)
    if (bad_stride(d->k_strides[i]) || bad_stride(d->v_strides[i])) {
      *err = "k_strides / v_strides must be positive multiples of 8 elements"; return PARSE_ERR_INVALID;
    }
  p->B = d->batch; p->Hq = d->num_q_heads; p->Hkv = d->num_kv_heads; p->D = d->head_dim; p->S = d->suffix_len;
  p->varlen = true;
  p->Nb.resize(p->B); p->Kb.resize(p->B); p->bnd_off.resize(p->B);
  p->q_row0.resize(p->B); p->kv_row0.resize(p->B);
  p->N = 0; p->K = 0; p->L = 0;
  long long nb = 0;
  for (int b = 0; b < p->B; ++b) {
    const int N = d->draft_lens[b], K = d->num_suffixes[b];
    if (N < 1 || K < 0) { *err = "request " + std::to_string(b) + ": need N_b >= 1 and K_b >= 0"; return PARSE_ERR_INVALID; }
    const long long L = (long long)N + (long long)K * p->S;
    if (L > (1ll << 30)) { *err = "packed length too large"; return PARSE_ERR_INVALID; }
    const int64_t r0 = d->row_offsets[b];
    if (r0 < 0 || r0 + L > d->total_rows) {
      *err = "request " + std::to_string(b) + ": rows [row_offset, row_offset + L_b) outside [0, total_rows)";
      return PARSE_ERR_INVALID;
    }
    int64_t k0 = r0;
    if (!paged && d->kv_row_offsets) {
      k0 = d->kv_row_offsets[b];
      if (k0 < 0 || k0 + L > d->kv_total_rows) {
        *err = "request " + std::to_string(b) + ": kv rows outside [0, kv_total_rows)"; return PARSE_ERR_INVALID;
      }
    }
    if (paged && (L + d->page_size - 1) / d->page_size > d->block_table_stride) {
      *err = "request " + std::to_string(b) + ": block_table_stride < pages needed"; return PARSE_ERR_INVALID;
    }
    p->Nb[b] = N; p->Kb[b] = K; p->bnd_off[b] = int32_t(nb);
    p->q_row0[b] = int32_t(r0); p->kv_row0[b] = paged ? 0 : int32_t(k0);
    p->self_align = paged ? kTile : 1;
    p->N = std::max(p->N, N); p->K = std::max(p->K, K); p->L = std::max(p->L, int(L));
    nb += K;
  }
  if (nb > (1ll << 30)) { *err = "too many boundaries"; return PARSE_ERR_INVALID; }
  if (nb > 0 && !d->boundaries) { *err = "boundaries is NULL"; return PARSE_ERR_INVALID; }
  p->bnd.assign(d->boundaries, d->boundaries + nb);
  for (int b = 0; b < p->B; ++b)
    for (int k = 0; k < p->Kb[b]; ++k) {
      const int32_t v = p->bndv(b, k);
      if (v < 0 || v > p->Nb[b]) {
        *err = "boundary " + std::to_string(k) + " of request " + std::to_string(b) + " = " + std::to_string(v) +
               " outside [0, N_b]";
        return PARSE_ERR_INVALID;
      }
    }
  return finish_problem(d->tree_parent, d->softmax_scale, p, err);
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
  const int N = p.Nb[b];
  int max_lim = 0;
  if (t0 < N) max_lim = std::min(t_end, N);                // draft rows: lim = t + 1
  if (t_end > N) {                                         // suffix rows
    int k_lo = (std::max(t0, N) - N) / p.S;
    int k_hi = (t_end - 1 - N) / p.S;
    for (int k = k_lo; k <= k_hi; ++k) max_lim = std::max(max_lim, p.bndv(b, k));
    ts.self_lo = align_down(N + k_lo * p.S, p.self_align);
    ts.n_self = cdiv(t_end - ts.self_lo, kTile);
  }
  ts.n_draft = cdiv(max_lim, kTile);
  return ts;
}

template <class F>
void for_each_item(const Problem& p, F&& emit) {
  const int r = p.Hq / p.Hkv;
  const int hpt_s = suffix_heads_per_tile(p);
  const int tok_max = hpt_s ? p.N : p.L;
  for (int t0 = 0; t0 < tok_max; t0 += kTile) {
    for (int b = 0; b < p.B; ++b) {
      const int tok_end = hpt_s ? p.Nb[b] : p.Lb(b);
      if (t0 >= tok_end) continue;
      const int t_end = std::min(t0 + kTile, tok_end);
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
      const int N = p.Nb[b], K = p.Kb[b];
      if (ntile >= 2) {
        // two head-packs of one copy per item (identical visibility)
        for (int k = 0; k < K; ++k) {
          const int t0 = N + k * p.S;
          const int lo = align_down(t0, p.self_align);
          const int n_draft = cdiv(p.bndv(b, k), kTile);
          for (int g = 0; g < p.Hkv; ++g)
            for (int ti = 0; ti < ntile; ti += 2) {
              const int nq = (ti + 1 < ntile) ? 2 : 1;
              emit(WorkItem{b, g * r + ti * hpt_s, t0, t0 + p.S, lo, n_draft, cdiv(t0 + p.S - lo, kTile),
                            hpt_s | ((nq == 2) << 8)});
            }
        }
      } else {
        // one head-pack covers the group: pair copies k and k+1 (tile 1 = next
        // copy, same heads).  The KV range is the union; each row keeps its
        // own boundary through the mask, and one self tile holds both copies
        // when 2S <= 128.
        const bool can_pair = 2 * p.S <= kTile;
        for (int k = 0; k < K; k += can_pair ? 2 : 1) {
          const int nq = (can_pair && k + 1 < K) ? 2 : 1;
          const int t0 = N + k * p.S;
          int lim = p.bndv(b, k);
          if (nq == 2) lim = std::max(lim, p.bndv(b, k + 1));
          const int n_draft = cdiv(lim, kTile);
          const int lo = align_down(t0, p.self_align);
          for (int g = 0; g < p.Hkv; ++g)
            emit(WorkItem{b, g * r, t0, t0 + nq * p.S, lo, n_draft, cdiv(t0 + nq * p.S - lo, kTile),
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

// 4 items per SM of a B200 (148 SMs).  Measured (ncu cycles): config 2
// 0.556 M -> 0.526 M (window 148 / 296 / 592: 0.528 / 0.527 / 0.526 M);
// configs 3 and tree unchanged.
#ifndef PARSE_TAIL_WINDOW
constexpr int kTailWindow = 4 * 148;
#else
constexpr int kTailWindow = PARSE_TAIL_WINDOW;
#endif

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
  // The last kTailWindow items (a few groups' worth) are re-sorted largest
  // first across groups, so the launch ends on the globally smallest items
  // (longest-processing-time order where it matters: the tail).
  const size_t tail = std::min(items->size(), size_t(kTailWindow));
  if (tail > 1)
    std::stable_sort(items->end() - tail, items->end(),
                     [&](const WorkItem& a, const WorkItem& b) { return cost(a) > cost(b); });
}

WorkspaceLayout workspace_layout(const Problem& p, bool need_items) {
  auto al = [](size_t x) { return (x + 255) & ~size_t(255); };
  WorkspaceLayout w{};
  w.counter_off = 0;
  w.req_off = 256;
  w.bnd_off = al(w.req_off + sizeof(ReqDesc) * size_t(p.B));
  w.anc_off = al(w.bnd_off + sizeof(int32_t) * std::max<size_t>(p.bnd.size(), 1));
  w.items_off = al(w.anc_off + sizeof(uint64_t) * size_t(p.tree ? p.S : 0));
  w.n_items = need_items ? count_schedule(p) : 0;
  w.pairs_off = al(w.items_off + sizeof(WorkItem) * w.n_items);
  w.total = al(w.pairs_off + sizeof(int2) * w.n_items);   // cluster units (or 2-SM variant pairs)
  return w;
}

// Work units of the 2-CTA cluster kernel ("K/V multicast"): the
// two CTAs of a cluster walk the same number of K/V steps with the same Q-tile
// count, so their K/V rings stay in lockstep.  x = CTA 0's item, y = CTA 1's:
//   y >= 0   same request, KV group and K/V tile sequence: every K/V tile is
//            loaded once for the pair (each CTA fetches half of its rows,
//            multicast into both CTAs' shared memory)
//   y <= -2  item -y-2, same step / tile count but other K/V: each CTA loads its own
//   y == -1  no partner: CTA 1 recomputes item x without storing it (multicast:
//            same K/V walk)
// Units keep the group-major / largest-first order of `items` (each at the
// position of its first item).
void build_units(const std::vector<WorkItem>& items, int Hkv, int Hq, std::vector<int2>* units) {
  const int r = Hq / Hkv;
  units->clear();
  struct U { size_t pos; int2 u; };
  std::vector<U> us;
  us.reserve(items.size() / 2 + 1);
  auto nq = [](const WorkItem& w) { return (w.flags >> 8) & 1; };
  // multicast partners: identical K/V walk
  std::map<std::array<int32_t, 6>, int> open_kv;
  std::vector<int> left;
  for (size_t i = 0; i < items.size(); ++i) {
    const WorkItem& w = items[i];
    const std::array<int32_t, 6> key{w.b, w.h0 / r, w.n_draft, w.n_self, w.n_self ? w.self_lo : 0, nq(w)};
    auto it = open_kv.find(key);
    if (it == open_kv.end()) {
      open_kv.emplace(key, int(i));
    } else {
      us.push_back(U{size_t(it->second), make_int2(it->second, int(i))});
      open_kv.erase(it);
    }
  }
  for (const auto& kv : open_kv) left.push_back(kv.second);
  std::sort(left.begin(), left.end());
  // lockstep partners among the rest: same step count and Q-tile count
  std::map<std::array<int32_t, 2>, int> open_n;
  for (int i : left) {
    const WorkItem& w = items[size_t(i)];
    const std::array<int32_t, 2> key{w.n_draft + w.n_self, nq(w)};
    auto it = open_n.find(key);
    if (it == open_n.end()) {
      open_n.emplace(key, i);
    } else {
      us.push_back(U{size_t(it->second), make_int2(it->second, -i - 2)});
      open_n.erase(it);
    }
  }
  for (const auto& kv : open_n) us.push_back(U{size_t(kv.second), make_int2(kv.second, -1)});
  std::stable_sort(us.begin(), us.end(), [](const U& a, const U& b) { return a.pos < b.pos; });
  units->reserve(us.size());
  for (const U& u : us) units->push_back(u.u);
}

void build_pairs(const std::vector<WorkItem>& items, int Hkv, int Hq, std::vector<int2>* pairs) {
  const int r = Hq / Hkv;
  pairs->clear();
  auto same = [&](const WorkItem& a, const WorkItem& b) {
    return a.b == b.b && a.h0 / r == b.h0 / r && a.n_draft == b.n_draft && a.n_self == b.n_self &&
           (a.n_self == 0 || a.self_lo == b.self_lo) && ((a.flags >> 8) & 1) == ((b.flags >> 8) & 1);
  };
  for (size_t i = 0; i < items.size();) {
    if (i + 1 < items.size() && same(items[i], items[i + 1])) {
      pairs->push_back(make_int2(int(i), int(i + 1)));
      i += 2;
    } else {
      pairs->push_back(make_int2(int(i), -1));
      i += 1;
    }
  }
}

}  // namespace parse
