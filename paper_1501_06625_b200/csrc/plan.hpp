// plan.hpp -- host-side compile_plan for the CUDA tracker.
//
// Turns the structural homotopy (g, f, gamma, k) into flat int32/double tables
// the kernels walk:
//  * monomial table: distinct supports of g and f, ordered by
//    size DESCENDING so the longest reverse-mode chains start first; the
//    value and partials of monomial q live in the monomial workspace at
//    mono_out[q] + p*32 (p = 0 value, p = 1+k partial k): a warp's 32
//    consecutive monomials write 32 consecutive entries per step (coalesced,
//    the "aligned" layout of PAPER.md:434-442).
//  * slot tasks: one per output entry (row i, col j), j == n is the value
//    slot.  Each task carries the contribution lists of g and f in term order
//    and the canonical-sum widths; equations identical in g and f are summed
//    once ("shared").
//  * contributions: (coefficient index, workspace index); workspace index -1
//    marks a constant term whose contribution is the coefficient itself.
#pragma once

#include <algorithm>
#include <cstdlib>
#include <cstdint>
#include <cstring>
#include <map>
#include <stdexcept>
#include <string>
#include <vector>

#include "../../include/pathtrack_b200.h"

namespace ptplan {

constexpr int kWarpChunk = 32;

inline int pow2ceil(int x) {
  int p = 1;
  while (p < x) p <<= 1;
  return p;
}
// Canonical widths; the oracle uses the same rules.
inline int width_eval(int K) { return std::min(256, std::max(32, pow2ceil((K + 15) / 16))); }
inline int width_mgs(int N) { return std::min(256, std::max(32, pow2ceil((N + 1) / 2))); }
// warps per MGS group: enough for one element per thread up to N = 256 (the
// canonical width only fixes the partials, not who computes the products)
inline int mgs_group_warps(int N) {
  const int P = width_mgs(N);
  if (N > 256) return 8;
  return std::max(P / 32, std::min(8, pow2ceil((N + 31) / 32)));
}

struct SlotTask {
  int32_t row, col;
  int32_t g_beg, g_cnt;
  int32_t f_beg, f_cnt;  // f_cnt == -1: shared with g
  int32_t gw;            // group width in warps = max canonical width / 32; 0 = lane task
  int32_t pad;
};

// Tasks whose sums have at most lane_k contributions on each side run one per
// lane: lane_canon32 (device.cuh) evaluates the width-32 canonical tree of any
// K <= 512 sequentially in one lane -- same shape, same bits.  Two partitions
// of the same tasks: the single-path engines are latency bound and keep only
// short sums on lanes; the batch kernel (one path per CTA, many CTAs) is
// throughput bound and runs everything up to 128 contributions on lanes, so
// no lane idles through a warp tree of a short sum.
inline int lane_k(int L) { return L == 4 ? 4 : 8; }
inline int lane_k_batch(int L) {
  const char* e = std::getenv("PT_LANE_K_BATCH");  // tuning knob
  if (e) return std::atoi(e);
  return L == 4 ? 4 : 128;
}

// Batch lane tasks are dealt to warps in bundles of 32 (one task per lane).
// A bundle's contributions are stored as lane-interleaved streams: entry
// (pos, lane) at pos*32 + lane holds that lane's contribution number
// pos - s (workspace index + the coefficient itself), so a warp loading
// contribution r of all its lanes issues one coalesced 128-byte index load
// and 2L coalesced coefficient loads.  Tasks are ordered column-major before
// bundling: for systems whose equations share a support (the random dense
// batch system) the 32 lanes of a bundle then read the SAME workspace entry
// at every step (a broadcast) -- no gathers anywhere.  Summation order is
// unchanged (each lane runs the canonical width-32 tree of its own slot).
struct Bundle {
  int32_t task_beg, ntasks;  // lane l < ntasks runs btasks[task_beg + l]
  int32_t sg, kg;            // g stream: rows sg .. sg+kg-1 (kg = max g_cnt over the lanes)
  int32_t sf, kf;            // f stream (kf = 0 when every lane is shared)
  int32_t dc;                // D << 8 | c: the lanes sum the subtree c of D (D = 1: the whole slot)
  int32_t split;             // D > 1: scratch row base of the split group (g: base + c, f: base + D + c)
};
constexpr int64_t kStreamCapBytes = 4LL << 30;  // contribution streams larger than this: no bundles

struct HostPlan {
  int n = 0, N = 0, L = 1;
  // monomials (device order)
  std::vector<int32_t> mono_size, mono_vbeg, mono_out, mono_flags, mono_var, mono_exp;
  int64_t ws_len = 0;  // complex entries in the monomial workspace
  // slots
  std::vector<SlotTask> tasks;
  int32_t class_beg[6] = {0, 0, 0, 0, 0, 0};  // lane tasks, then gw = 8,4,2,1
  std::vector<SlotTask> tasks_b;                // batch partition (lane_k_batch)
  int32_t class_beg_b[6] = {0, 0, 0, 0, 0, 0};
  std::vector<int32_t> ctr_coef, ctr_ws;
  // batch lane-task bundles (empty: the batch runs its lane tasks unbundled)
  std::vector<Bundle> bundles;            // largest first (claimed by the warps through a shared counter)
  std::vector<int32_t> splits;            // split groups: task_beg, ntasks, D, scratch row base
  int32_t scratch_units = 0;              // 32-lane complex rows of split scratch
  std::vector<SlotTask> btasks;           // lane tasks in bundle order
  std::vector<int32_t> s_ws;              // [s_len][32] workspace index (-1: constant term)
  std::vector<double> s_coef;             // [2L][s_len * 32] coefficient limbs ([2][..] when s_hi)
  int32_t s_hi = 0;                       // every streamed coefficient has +0.0 lower limbs: only
                                          // the leading limb of re / im is stored (half the bytes)
  int64_t s_len = 0;
  // coefficients of all terms of g then f, complex SoA [2][L][n_coef]
  std::vector<double> coef;
  int64_t n_coef = 0;
  int max_mono = 0;
};

inline void check(bool ok, const char* what) {
  if (!ok) throw std::invalid_argument(what);
}

inline void validate(const pt_system_desc* s) {
  check(s && s->eq_ptr && s->term_ptr && s->coef, "null system descriptor");
  check(s->n_vars >= 1 && s->n_eqs >= 1 && s->n_terms >= 0, "bad system dimensions");
  check(s->eq_ptr[0] == 0 && s->eq_ptr[s->n_eqs] == s->n_terms, "eq_ptr does not cover the terms");
  for (int i = 0; i < s->n_eqs; ++i) check(s->eq_ptr[i] <= s->eq_ptr[i + 1], "eq_ptr not monotone");
  check(s->term_ptr[0] == 0, "term_ptr[0] != 0");
  for (int t = 0; t < s->n_terms; ++t) {
    check(s->term_ptr[t] <= s->term_ptr[t + 1], "term_ptr not monotone");
    for (int q = s->term_ptr[t]; q < s->term_ptr[t + 1]; ++q) {
      check(s->var[q] >= 0 && s->var[q] < s->n_vars, "variable index out of range");
      check(s->exp[q] >= 1, "exponent < 1");
      if (q > s->term_ptr[t]) check(s->var[q] > s->var[q - 1], "support variables not strictly increasing");
    }
  }
}

// Bundles of the batch partition (see Bundle): every slot whose canonical
// widths are <= 128 on both sides becomes a lane task; a slot with many
// contributions is split over D lanes (subtrees c = 0..D-1 of its tree,
// D = pow2ceil(K / 128) within [P / 32, 8]) so no lane runs much more than
// 128 contributions.  Tasks of one D are ordered column-major and dealt 32
// per bundle; the remaining tasks stay in tasks_b's warp-group classes.
inline void build_bundles(HostPlan& P) {
  const char* e = std::getenv("PT_BUNDLES");  // tuning knob: 0 disables the streams
  if (e && e[0] == '0') return;
  const int L = P.L;
  auto width = [](int K) { return K > 0 ? width_eval(K) : 32; };
  std::map<int, std::vector<SlotTask>> byD;
  std::vector<SlotTask> rest;
  for (const SlotTask& t : P.tasks_b) {
    const int pmax = std::max(width(t.g_cnt), width(t.f_cnt));
    if (pmax > 128) {
      rest.push_back(t);
      continue;
    }
    const int kmax = std::max(t.g_cnt, t.f_cnt);
    int D = pow2ceil((kmax + 127) / 128);
    D = std::max(D, pmax / 32);
    D = std::min(D, 8);
    byD[D].push_back(t);
  }
  if (byD.empty()) return;
  std::vector<SlotTask> lt;
  std::vector<Bundle> bs;
  std::vector<int32_t> splits;
  int64_t len = 0;
  int32_t units = 0;
  for (auto& kv : byD) {
    const int D = kv.first;
    std::vector<SlotTask>& ts = kv.second;
    std::stable_sort(ts.begin(), ts.end(), [](const SlotTask& a, const SlotTask& b) {
      return a.col != b.col ? a.col < b.col : a.row < b.row;
    });
    for (size_t b0 = 0; b0 < ts.size(); b0 += 32) {
      Bundle B{};
      B.task_beg = (int32_t)lt.size();
      B.ntasks = (int32_t)std::min<size_t>(32, ts.size() - b0);
      for (int l = 0; l < B.ntasks; ++l) {
        const SlotTask& t = ts[b0 + l];
        lt.push_back(t);
        B.kg = std::max(B.kg, t.g_cnt);
        B.kf = std::max(B.kf, t.f_cnt);
      }
      B.sg = (int32_t)len;
      len += B.kg;
      B.sf = (int32_t)len;
      len += B.kf;
      B.split = -1;
      if (D == 1) {
        B.dc = 1 << 8;
        bs.push_back(B);
      } else {
        splits.insert(splits.end(), {B.task_beg, B.ntasks, D, units});
        B.split = units;
        units += 2 * D;
        for (int c = 0; c < D; ++c) {
          B.dc = (D << 8) | c;
          bs.push_back(B);
        }
      }
    }
  }
  if (len * 32 * (4 + 16 * (int64_t)L) > kStreamCapBytes) return;  // the all-limb size bounds the hi-only one
  P.s_len = std::max<int64_t>(len, 1);
  const int64_t S = P.s_len * 32;
  // coefficients built from binary64 values (random / integer systems): the
  // lower limbs are exactly +0.0 (bit pattern 0), so the device rebuilds them
  // from the leading limb alone -- the same operands, half the stream
  const char* he = std::getenv("PT_STREAM_HI");  // tuning knob: 0 keeps every limb
  bool hi = L > 1 && !(he && he[0] == '0');
  for (int64_t t = 0; hi && t < P.n_coef; ++t)
    for (int q = 0; q < 2 * L && hi; ++q) {
      if (q % L == 0) continue;
      const double v = P.coef[(size_t)q * P.n_coef + t];
      uint64_t bits;
      std::memcpy(&bits, &v, 8);
      hi = bits == 0;
    }
  P.s_hi = hi ? 1 : 0;
  const int planes = hi ? 2 : 2 * L;
  P.s_ws.assign((size_t)S, 0);
  P.s_coef.assign((size_t)planes * S, 0.0);
  auto fill = [&](int64_t row, int lane, int32_t beg, int32_t cnt) {
    for (int32_t r = 0; r < cnt; ++r) {
      const int64_t at = (row + r) * 32 + lane;
      const int32_t ci = P.ctr_coef[beg + r];
      P.s_ws[at] = P.ctr_ws[beg + r];
      for (int q = 0; q < planes; ++q) {
        const int src = hi ? q * L : q;  // leading limb of re (q = 0) / im (q = 1)
        P.s_coef[(size_t)q * S + at] = P.coef[(size_t)src * P.n_coef + ci];
      }
    }
  };
  for (const Bundle& B : bs) {
    if ((B.dc & 255) != 0) continue;  // the sub-bundles of a split group share its streams
    for (int l = 0; l < B.ntasks; ++l) {
      const SlotTask& t = lt[B.task_beg + l];
      fill(B.sg, l, t.g_beg, t.g_cnt);
      if (t.f_cnt > 0) fill(B.sf, l, t.f_beg, t.f_cnt);
    }
  }
  // largest first: the warps of a batch CTA claim bundles in this order from a
  // shared counter (greedy list scheduling, any warp count)
  std::stable_sort(bs.begin(), bs.end(), [](const Bundle& x, const Bundle& y) {
    return (x.kg + x.kf) / (x.dc >> 8) > (y.kg + y.kf) / (y.dc >> 8);
  });
  P.bundles = std::move(bs);
  P.splits = std::move(splits);
  P.scratch_units = units;
  P.btasks = std::move(lt);
  // the batch's group classes keep only the slots that were not bundled
  const int classes[5] = {0, 8, 4, 2, 1};
  std::vector<SlotTask> out;
  for (int c = 0; c < 5; ++c) {
    P.class_beg_b[c] = (int32_t)out.size();
    for (const auto& tk : rest)
      if (tk.gw == classes[c]) out.push_back(tk);
  }
  P.class_beg_b[5] = (int32_t)out.size();
  P.tasks_b = std::move(out);
}

inline HostPlan compile(const pt_system_desc* g, const pt_system_desc* f, int L) {
  validate(g);
  validate(f);
  check(g->n_vars == f->n_vars && g->n_eqs == f->n_eqs, "start and target dimensions differ");
  check(g->n_eqs >= g->n_vars, "need N >= n equations");
  HostPlan P;
  P.n = g->n_vars;
  P.N = g->n_eqs;
  P.L = L;
  const int n = P.n, N = P.N;
  const pt_system_desc* sys[2] = {g, f};

  // --- distinct supports in first-appearance order ------------------------
  using Key = std::vector<int32_t>;  // var0, exp0, var1, exp1, ...
  std::map<Key, int> index;
  std::vector<Key> keys;
  std::vector<int> term_mono[2];
  for (int s = 0; s < 2; ++s) {
    const pt_system_desc* d = sys[s];
    term_mono[s].resize(d->n_terms);
    for (int t = 0; t < d->n_terms; ++t) {
      Key k;
      for (int q = d->term_ptr[t]; q < d->term_ptr[t + 1]; ++q) {
        k.push_back(d->var[q]);
        k.push_back(d->exp[q]);
      }
      if (k.empty()) {
        term_mono[s][t] = -1;
        continue;
      }
      auto it = index.find(k);
      if (it == index.end()) {
        it = index.emplace(k, (int)keys.size()).first;
        keys.push_back(k);
      }
      term_mono[s][t] = it->second;
    }
  }
  const int M = (int)keys.size();
  // device order: size descending, ties by first appearance
  std::vector<int> order(M);
  for (int q = 0; q < M; ++q) order[q] = q;
  std::stable_sort(order.begin(), order.end(),
                   [&](int a, int b) { return keys[a].size() > keys[b].size(); });
  std::vector<int> dev_of(M);
  for (int q = 0; q < M; ++q) dev_of[order[q]] = q;
  P.mono_size.resize(M);
  P.mono_vbeg.resize(M);
  P.mono_out.resize(M);
  P.mono_flags.resize(M);
  // chunked workspace layout: chunk c = monomials [32c, 32c+32) uses
  // 32 * (max size in chunk + 1) entries
  int64_t ws = 0;
  for (int c0 = 0; c0 < M; c0 += kWarpChunk) {
    int maxsz = 0;
    for (int q = c0; q < std::min(M, c0 + kWarpChunk); ++q) maxsz = std::max(maxsz, (int)keys[order[q]].size() / 2);
    for (int q = c0; q < std::min(M, c0 + kWarpChunk); ++q) P.mono_out[q] = (int32_t)(ws + (q - c0));
    ws += (int64_t)kWarpChunk * (maxsz + 1);
  }
  check(ws < (int64_t)1 << 31, "monomial workspace exceeds 2^31 entries");
  P.ws_len = std::max<int64_t>(ws, 1);
  for (int q = 0; q < M; ++q) {
    const Key& k = keys[order[q]];
    const int m = (int)k.size() / 2;
    P.mono_size[q] = m;
    P.mono_vbeg[q] = (int32_t)P.mono_var.size();
    int flags = 0;
    for (int p = 0; p < m; ++p) {
      P.mono_var.push_back(k[2 * p]);
      P.mono_exp.push_back(k[2 * p + 1]);
      if (k[2 * p + 1] >= 2) flags |= 1;
    }
    P.mono_flags[q] = flags;
    P.max_mono = std::max(P.max_mono, m);
  }
  if (P.mono_var.empty()) {
    P.mono_var.push_back(0);
    P.mono_exp.push_back(1);
  }

  // --- coefficients: g terms then f terms ---------------------------------
  P.n_coef = (int64_t)g->n_terms + f->n_terms;
  const int64_t NC = std::max<int64_t>(P.n_coef, 1);
  P.coef.assign((size_t)2 * L * NC, 0.0);
  for (int s = 0; s < 2; ++s) {
    const pt_system_desc* d = sys[s];
    const int64_t base = s == 0 ? 0 : g->n_terms;
    for (int t = 0; t < d->n_terms; ++t)
      for (int q = 0; q < 2 * L; ++q) P.coef[(size_t)q * NC + base + t] = d->coef[(size_t)q * d->n_terms + t];
  }
  P.n_coef = NC;

  // --- shared equations ----------------------------------------------------
  std::vector<char> shared(N, 0);
  for (int i = 0; i < N; ++i) {
    const int gb = g->eq_ptr[i], ge = g->eq_ptr[i + 1], fb = f->eq_ptr[i], fe = f->eq_ptr[i + 1];
    bool same = (ge - gb) == (fe - fb);
    for (int q = 0; same && q < ge - gb; ++q) {
      same = term_mono[0][gb + q] == term_mono[1][fb + q];
      for (int l = 0; same && l < 2 * L; ++l) {
        const double a = g->coef[(size_t)l * g->n_terms + gb + q];
        const double b = f->coef[(size_t)l * f->n_terms + fb + q];
        same = std::memcmp(&a, &b, 8) == 0;
      }
    }
    shared[i] = same;
  }

  // --- slot contribution lists --------------------------------------------
  // per system, per equation: value list + per-variable lists, in term order
  struct Lists {
    std::vector<int32_t> coef, wsi;
  };
  std::vector<SlotTask> tasks;
  tasks.reserve((size_t)N * (n + 1));
  std::vector<std::vector<Lists>> L2(2, std::vector<Lists>(n + 1));
  for (int i = 0; i < N; ++i) {
    const int ns = shared[i] ? 1 : 2;
    for (int s = 0; s < ns; ++s) {
      for (auto& l : L2[s]) {
        l.coef.clear();
        l.wsi.clear();
      }
      const pt_system_desc* d = sys[s];
      const int64_t cbase = s == 0 ? 0 : g->n_terms;
      for (int t = d->eq_ptr[i]; t < d->eq_ptr[i + 1]; ++t) {
        const int mo = term_mono[s][t];
        const int32_t ci = (int32_t)(cbase + t);
        if (mo < 0) {
          L2[s][n].coef.push_back(ci);
          L2[s][n].wsi.push_back(-1);
          continue;
        }
        const int q = dev_of[mo];
        L2[s][n].coef.push_back(ci);
        L2[s][n].wsi.push_back(P.mono_out[q]);
        for (int p = d->term_ptr[t]; p < d->term_ptr[t + 1]; ++p) {
          const int k = p - d->term_ptr[t];
          L2[s][d->var[p]].coef.push_back(ci);
          L2[s][d->var[p]].wsi.push_back(P.mono_out[q] + kWarpChunk * (1 + k));
        }
      }
    }
    for (int j = 0; j <= n; ++j) {
      SlotTask tk{};
      tk.row = i;
      tk.col = j;
      tk.g_beg = (int32_t)P.ctr_coef.size();
      tk.g_cnt = (int32_t)L2[0][j].coef.size();
      P.ctr_coef.insert(P.ctr_coef.end(), L2[0][j].coef.begin(), L2[0][j].coef.end());
      P.ctr_ws.insert(P.ctr_ws.end(), L2[0][j].wsi.begin(), L2[0][j].wsi.end());
      int w = tk.g_cnt > 0 ? width_eval(tk.g_cnt) : 32;
      if (shared[i]) {
        tk.f_beg = tk.g_beg;
        tk.f_cnt = -1;
      } else {
        tk.f_beg = (int32_t)P.ctr_coef.size();
        tk.f_cnt = (int32_t)L2[1][j].coef.size();
        P.ctr_coef.insert(P.ctr_coef.end(), L2[1][j].coef.begin(), L2[1][j].coef.end());
        P.ctr_ws.insert(P.ctr_ws.end(), L2[1][j].wsi.begin(), L2[1][j].wsi.end());
        if (tk.f_cnt > 0) w = std::max(w, width_eval(tk.f_cnt));
      }
      check(P.ctr_coef.size() < ((size_t)1 << 31), "too many contributions");
      tk.gw = w / 32;  // group width in warps when not a lane task
      tasks.push_back(tk);
    }
  }
  // group tasks by class (lane tasks, then 8, 4, 2, 1 warps); stable within a class
  const int classes[5] = {0, 8, 4, 2, 1};
  auto partition = [&](int lk, std::vector<SlotTask>& out, int32_t* cb) {
    for (int c = 0; c < 5; ++c) {
      cb[c] = (int32_t)out.size();
      for (const auto& tk : tasks) {
        const bool lane = tk.g_cnt <= lk && (tk.f_cnt < 0 || tk.f_cnt <= lk);
        if ((lane ? 0 : tk.gw) == classes[c]) {
          out.push_back(tk);
          out.back().gw = lane ? 0 : tk.gw;
        }
      }
    }
    cb[5] = (int32_t)out.size();
  };
  partition(lane_k(L), P.tasks, P.class_beg);
  partition(lane_k_batch(L), P.tasks_b, P.class_beg_b);
  build_bundles(P);
  if (P.ctr_coef.empty()) {
    P.ctr_coef.push_back(0);
    P.ctr_ws.push_back(-1);
  }
  return P;
}

}  // namespace ptplan
