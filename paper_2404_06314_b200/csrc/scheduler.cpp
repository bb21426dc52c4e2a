// Circuit -> device program lowering (see program.h for the execution model).
//
// The reference applies gates strictly one after another, one full state
// sweep each (_kernels.py:137-141, 257-281). Here gates are grouped so that a
// tile/register-resident chunk of the state receives many gates per memory
// round trip. Gates are only reordered when they commute, using the Pauli
// structure of the gate set: on a shared qubit, two gates commute iff both act
// diagonally there (RZ, CZ, CNOT control: "Z"), or both act like X (RX, X,
// CNOT target), or both like Y (RY). H commutes with nothing. Reordering
// commuting gates is exact in real arithmetic; in floating point it moves
// results by ~1e-16 (SURVEY §8c noise floor).
#include "scheduler.h"

#include <algorithm>
#include <functional>
#include <cstdio>

namespace vqc {
namespace {

enum Act { A_Z = 0, A_X = 1, A_Y = 2, A_G = 3 };

struct GateInfo {
  int nq = 1;
  int q[2] = {0, 0};
  int act[2] = {0, 0};
  uint32_t mix = 0;  // qubits that must be local (tile) / a register slot (segment)
  bool rot = false;
  bool cnot = false;
  bool need_grad = false;
  std::vector<int> preds;
};

struct Group {
  uint32_t mask = 0;
  std::vector<int> gates;
};

int popc(uint32_t x) { return __builtin_popcount(x); }

std::string analyze(const std::vector<GateIn>& gates, int n, int64_t total_params,
                    const std::vector<int64_t>& wrt_col, std::vector<GateInfo>* out) {
  const int G = (int)gates.size();
  out->assign(G, GateInfo());
  struct QubitBlocks {
    int cur_type = -1;
    std::vector<int> cur, prev;
  };
  std::vector<QubitBlocks> blocks(n);
  char buf[256];
  for (int g = 0; g < G; ++g) {
    const GateIn& gi = gates[g];
    GateInfo& inf = (*out)[g];
    auto qcheck = [&](int q) -> bool { return q >= 0 && q < n; };
    switch (gi.kind) {
      case G_RX: case G_RY: case G_RZ: case G_H: case G_X:
        if (!qcheck(gi.q0)) { snprintf(buf, sizeof buf, "gate %d: qubit %d out of range", g, gi.q0); return buf; }
        inf.nq = 1; inf.q[0] = gi.q0;
        inf.act[0] = gi.kind == G_RX || gi.kind == G_X ? A_X
                   : gi.kind == G_RY ? A_Y : gi.kind == G_RZ ? A_Z : A_G;
        inf.mix = gi.kind == G_RZ ? 0u : (1u << gi.q0);
        inf.rot = gi.kind <= G_RZ;
        break;
      case G_CNOT: case G_CZ:
        if (!qcheck(gi.q0) || !qcheck(gi.q1)) {
          snprintf(buf, sizeof buf, "gate %d: qubit out of range", g); return buf;
        }
        if (gi.q0 == gi.q1) { snprintf(buf, sizeof buf, "gate %d: duplicate qubit indices", g); return buf; }
        inf.nq = 2; inf.q[0] = gi.q0; inf.q[1] = gi.q1;
        inf.act[0] = A_Z; inf.act[1] = gi.kind == G_CNOT ? A_X : A_Z;
        inf.mix = gi.kind == G_CNOT ? (1u << gi.q1) : 0u;
        inf.cnot = gi.kind == G_CNOT;
        break;
      default:
        snprintf(buf, sizeof buf, "gate %d: unknown gate kind %d", g, gi.kind); return buf;
    }
    if (inf.rot) {
      if ((int)gi.fidx.size() > kMaxFactors) {
        snprintf(buf, sizeof buf, "gate %d: %d angle factors (this path supports <= %d)", g,
                 (int)gi.fidx.size(), kMaxFactors);
        return buf;
      }
      for (int32_t f : gi.fidx) {
        if (f < 0 || f >= total_params) { snprintf(buf, sizeof buf, "gate %d: factor index %d out of range", g, f); return buf; }
        if (wrt_col[f] >= 0) inf.need_grad = true;
      }
    }
    // Per qubit, consecutive gates of one commuting type form a block. A gate
    // joining the current block depends on every member of the previous
    // block (a different type); a gate of a new type closes the current
    // block and depends on all of it. H (A_G) always starts its own block.
    for (int i = 0; i < inf.nq; ++i) {
      QubitBlocks& qb = blocks[inf.q[i]];
      const int t = inf.act[i];
      if (t == qb.cur_type && t != A_G) {
        qb.cur.push_back(g);
      } else {
        qb.prev.swap(qb.cur);
        qb.cur.assign(1, g);
        qb.cur_type = t;
      }
      inf.preds.insert(inf.preds.end(), qb.prev.begin(), qb.prev.end());
    }
    std::sort(inf.preds.begin(), inf.preds.end());
    inf.preds.erase(std::unique(inf.preds.begin(), inf.preds.end()), inf.preds.end());
  }
  return "";
}

// Greedy partition of `todo` (a topological order) into groups whose mixing
// qubits fit `cap` local qubits (always including `forced`). status: 0 pending,
// 1 done; gates outside `todo` must be marked done.
// fold_cnots (register segments): keep each group of the form
// [CNOTs][body][CNOTs] so both CNOT runs fold into the segment's shared-memory
// address maps instead of costing register permutations.
// free_folds: boundary CNOTs fold into the address maps whatever their
// target (a tile-local qubit), so they take no register slot.
std::vector<Group> greedy_groups(const std::vector<int>& todo, const std::vector<GateInfo>& info,
                                 int cap, uint32_t forced, std::vector<uint8_t>& status,
                                 bool fold_cnots = false, int variants = 1, bool free_folds = false) {
  std::vector<Group> groups;
  std::vector<int> remaining = todo;
  // One scan of `remaining`: variant v refuses the first v requests for new
  // local qubits, so later (often better-packed) qubit sets get a chance.
  // status 2 = taken by this scan, 3 = blocked; both reset by the caller.
  auto scan = [&](int v, Group& grp) {
    grp = Group();
    grp.mask = forced;
    int phase = 0;  // 0 leading CNOTs, 1 body, 2 trailing CNOTs
    int refused = 0;
    for (int g : remaining) {
      bool ok = true;
      for (int p : info[g].preds)
        if (status[p] != 1 && status[p] != 2) { ok = false; break; }
      if (ok && fold_cnots && phase == 2 && !info[g].cnot) ok = false;
      if (ok) {
        // in a folded group every CNOT is leading or trailing (body CNOTs end the body)
        const bool free_cnot = free_folds && fold_cnots && info[g].cnot;
        const uint32_t m = grp.mask | (free_cnot ? 0u : info[g].mix);
        if (m != grp.mask && refused < v) {
          ++refused;
          ok = false;
        } else if (popc(m) <= cap) {
          grp.mask = m;
          status[g] = 2;
          grp.gates.push_back(g);
          if (!info[g].cnot) phase = 1;
          else if (phase == 1) phase = 2;
        } else {
          ok = false;
        }
      }
      if (!ok) status[g] = 3;
    }
  };
  auto score = [&](const Group& grp) {
    int sc = 0;
    for (int g : grp.gates) sc += info[g].rot ? 4 : 1;
    return sc;
  };
  while (!remaining.empty()) {
    Group best;
    int best_v = 0, best_score = -1;
    for (int v = 0; v < variants; ++v) {
      Group grp;
      scan(v, grp);
      const int sc = grp.gates.empty() ? -1 : score(grp);
      if (sc > best_score) {
        best_score = sc;
        best_v = v;
        best = grp;
      }
      for (int g : remaining) status[g] = 0;
    }
    if (best.gates.empty()) return {};  // cannot happen when cap >= popc(forced) + 1
    Group grp;
    scan(best_v, grp);
    std::vector<int> next;
    for (int g : remaining) {
      if (status[g] == 2) status[g] = 1;
      else { status[g] = 0; next.push_back(g); }
    }
    groups.push_back(std::move(grp));
    remaining.swap(next);
  }
  return groups;
}

// Thread-group synchronisation (JIT HBM plans). A segment boundary is a
// shared-memory transpose; the threads that exchange data are those that agree
// on every tile position which is a thread bit on both sides. If the top t
// thread-index bits of two consecutive segments sit on the same tile positions
// (same order) and the folded CNOT maps leave those positions alone, a group
// of blockDim >> t threads stores exactly the cells it loads next: the
// boundary needs a barrier over that group only (a warp: __syncwarp), and
// groups drift apart so shared-memory phases of one overlap arithmetic of
// another. Dynamic programme over the segments of a pass: states are ordered
// choices of the top T positions, cost per boundary = other warps waited for.
void assign_thread_groups(std::vector<SegDesc>& segs, const PassDesc& pd, int k) {
  const int m = (int)segs.size();
  const int nthr = segs[0].nthr;
  const int T = std::min(3, std::max(0, nthr - 5));  // thread bits above the lane bits that are planned
  auto ident = [&](const uint32_t* row, int p) { return row[p] == (1u << pd.local_q[p]); };
  auto finish = [&](SegDesc& sd, const std::vector<int>& top) {
    // lane bits: the first three cover distinct residues mod 3 (bank groups
    // under the mod-3 fold swizzle), then the rest ascending; top bits last
    std::vector<int> rest;
    for (int i = 0; i < sd.nthr; ++i)
      if (std::find(top.begin(), top.end(), (int)sd.thr_l[i]) == top.end()) rest.push_back(sd.thr_l[i]);
    std::sort(rest.begin(), rest.end());
    // (positions 0-2, the tile's contiguous 128 bytes in HBM, have distinct
    // residues and sort first: as the lowest lane bits they also make the
    // first / last segment's direct HBM accesses coalesce)
    std::vector<int> order;
    for (int r = 0; r < 3; ++r)
      for (size_t i = 0; i < rest.size(); ++i)
        if (rest[i] >= 0 && rest[i] % 3 == r) { order.push_back(rest[i]); rest[i] = -1; break; }
    for (int p : rest)
      if (p >= 0) order.push_back(p);
    for (int i = (int)top.size() - 1; i >= 0; --i) order.push_back(top[i]);  // top[0] = highest bit
    for (size_t i = 0; i < order.size(); ++i) {
      sd.thr_l[i] = (int8_t)order[i];
      sd.thr_g[i] = pd.local_q[order[i]];
      sd.tsw[i] = (uint16_t)swz_index(1u << order[i]);
    }
  };
  if (T == 0) {
    for (SegDesc& sd : segs) sd.sync_ld = sd.sync_st = sd.sync_self = 0;
    return;
  }
  // candidate states per segment: ordered T-tuples of its thread positions (top bit first)
  std::vector<std::vector<std::vector<int>>> states(m);
  for (int i = 0; i < m; ++i) {
    std::vector<int> pos;
    for (int t = 0; t < segs[i].nthr; ++t) pos.push_back(segs[i].thr_l[t]);
    std::sort(pos.begin(), pos.end());
    std::vector<int> cur;
    std::function<void()> rec = [&]() {
      if ((int)cur.size() == T) {
        // keep one residue of each class among the lane bits when possible
        int have = 0, all = 0;
        for (int p : pos) {
          all |= 1 << (p % 3);
          if (std::find(cur.begin(), cur.end(), p) == cur.end()) have |= 1 << (p % 3);
        }
        // the segments that open / close a sweep exchange registers with HBM
        // directly: keep positions 0-2 among their lane bits (coalescing)
        bool low_top = false;
        if (i == 0 || i + 1 == m)
          for (int p : cur) low_top = low_top || p < 3;
        if (have == all && !low_top) states[i].push_back(cur);
        return;
      }
      for (int p : pos)
        if (std::find(cur.begin(), cur.end(), p) == cur.end()) {
          cur.push_back(p);
          rec();
          cur.pop_back();
        }
    };
    rec();
    if (states[i].empty()) {  // no residue-complete choice: take any
      cur.assign(pos.end() - T, pos.end());
      states[i].push_back(cur);
    }
  }
  // level of boundary i -> i + 1 for states a, b: common top prefix on identity rows
  auto level = [&](int i, const std::vector<int>& a, const std::vector<int>& b) {
    int t = 0;
    while (t < T && a[t] == b[t] && ident(segs[i].st_row, a[t]) && ident(segs[i + 1].ld_row, a[t])) ++t;
    return t;
  };
  auto cost_of = [&](int t) { return (1 << (T - t)) - 1; };
  std::vector<std::vector<int>> best(m), from(m);
  best[0].assign(states[0].size(), 0);
  from[0].assign(states[0].size(), -1);
  for (int i = 1; i < m; ++i) {
    best[i].assign(states[i].size(), 1 << 30);
    from[i].assign(states[i].size(), 0);
    for (size_t b = 0; b < states[i].size(); ++b)
      for (size_t a = 0; a < states[i - 1].size(); ++a) {
        const int c = best[i - 1][a] + cost_of(level(i - 1, states[i - 1][a], states[i][b]));
        if (c < best[i][b]) { best[i][b] = c; from[i][b] = (int)a; }
      }
  }
  int cur = (int)(std::min_element(best[m - 1].begin(), best[m - 1].end()) - best[m - 1].begin());
  std::vector<int> pick(m);
  for (int i = m - 1; i >= 0; --i) {
    pick[i] = cur;
    cur = from[i][cur];
  }
  for (int i = 0; i < m; ++i) {
    const std::vector<int>& top = states[i][pick[i]];
    finish(segs[i], top);
    segs[i].sync_ld = i > 0 ? (int8_t)level(i - 1, states[i - 1][pick[i - 1]], top) : 0;
    segs[i].sync_st = i + 1 < m ? (int8_t)level(i, top, states[i + 1][pick[i + 1]]) : 0;
    int t = 0;
    while (t < T && ident(segs[i].ld_row, top[t]) && ident(segs[i].st_row, top[t])) ++t;
    segs[i].sync_self = (int8_t)t;
  }
}

uint32_t enc(uint32_t code, uint32_t a, uint32_t b, uint32_t ipl, bool adj) {
  return code | (a << 5) | (b << 11) | (ipl << 17) | (adj ? (1u << 31) : 0u);
}

}  // namespace

int absorb_trailing_gates(std::vector<GateIn>* gates, int n, std::vector<uint32_t>* zmask,
                          std::vector<double>* zcoeff) {
  int count = 0;
  auto ok_q = [&](int q) { return q >= 0 && q < n; };
  while (!gates->empty()) {
    const GateIn& g = gates->back();
    if (g.kind == G_CNOT || g.kind == G_CZ) {
      if (!ok_q(g.q0) || !ok_q(g.q1) || g.q0 == g.q1) break;
      if (g.kind == G_CNOT)
        for (uint32_t& s : *zmask) s ^= ((s >> g.q1) & 1u) << g.q0;  // CNOT Z_t CNOT = Z_c Z_t
    } else if (g.kind == G_X) {
      if (!ok_q(g.q0)) break;
      for (size_t t = 0; t < zmask->size(); ++t)
        if (((*zmask)[t] >> g.q0) & 1u) (*zcoeff)[t] = -(*zcoeff)[t];  // X Z X = -Z
    } else {
      break;
    }
    gates->pop_back();
    ++count;
  }
  return count;
}

std::string build_program(const std::vector<GateIn>& gates, int n, int64_t total_params,
                          const std::vector<int64_t>& wrt_col, const ScheduleOptions& opt,
                          HostProgram* P) {
  if (n < 1 || n > kMaxQubits) return "num_qubits must be in [1, 24]";
  std::vector<GateInfo> info;
  std::string err = analyze(gates, n, total_params, wrt_col, &info);
  if (!err.empty()) return err;
  const int G = (int)gates.size();

  *P = HostProgram();
  P->n = n;
  P->hbm = n > opt.smem_max_qubits;
  P->group_sync = opt.group_sync && P->hbm;
  P->k = P->hbm ? std::min(opt.tile_qubits, n) : n;
  P->R = std::min(opt.reg_slots, P->k);
  if (P->hbm && P->k < opt.forced_low + 1) return "tile too small";
  const int k = P->k, R = P->R;
  const uint32_t all_mask = n == 32 ? 0xffffffffu : ((1u << n) - 1u);

  // ---- level 1: passes (tiles of k local qubits) ----
  std::vector<uint8_t> status(G, 0);
  std::vector<int> todo(G);
  for (int g = 0; g < G; ++g) todo[g] = g;
  std::vector<Group> passes;
  if (P->hbm) {
    const uint32_t forced = (1u << opt.forced_low) - 1u;
    passes = greedy_groups(todo, info, k, forced, status, false, opt.variants);
    if (G > 0 && passes.empty()) return "pass scheduling failed";
  } else {
    Group all;
    all.mask = all_mask;
    all.gates = todo;
    passes.push_back(all);
    for (int g = 0; g < G; ++g) status[g] = 1;
  }
  if (passes.empty()) {  // no gates: one empty pass still observes the state
    Group g0;
    g0.mask = P->hbm ? ((1u << k) - 1u) : all_mask;
    passes.push_back(g0);
  }

  std::vector<int> rot_id(G, -1), gslot(G, -1);
  int next_rot = 0, next_g = 0;
  uint32_t touched = 0;  // qubits some scheduled operation has acted on so far

  // ---- level 2: register segments inside a tile ----
  // Two policies, priced per pass: segments shaped [CNOTs][body][CNOTs]
  // (every CNOT folds into address maps, but more segments), or free
  // placement (interior CNOTs become register permutations). A segment
  // boundary costs a shared-memory round trip of the tile; an interior
  // CNOT a few dozen register moves/selects per thread.
  auto interior_cnots = [&](const std::vector<Group>& gs) {
    int cost = 0;
    for (const Group& gr : gs) {
      size_t a = 0, b = gr.gates.size();
      while (a < b && info[gr.gates[a]].cnot) ++a;
      while (b > a && info[gr.gates[b - 1]].cnot) --b;
      for (size_t i = a; i < b; ++i) cost += info[gr.gates[i]].cnot ? 1 : 0;
    }
    return cost;
  };
  auto make_segments = [&](const std::vector<int>& pgates) {
    std::vector<uint8_t> st2(G, 1);
    for (int g : pgates) st2[g] = 0;
    std::vector<Group> folded = greedy_groups(pgates, info, R, 0u, st2, true, opt.variants, opt.fold_thread_targets);
    for (int g : pgates) st2[g] = 0;
    std::vector<Group> free_ = greedy_groups(pgates, info, R, 0u, st2, false, opt.variants);
    const int seg_cost = opt.segment_cost, cnot_cost = 1;
    const int c_fold = (int)folded.size() * seg_cost + interior_cnots(folded) * cnot_cost;
    const int c_free = (int)free_.size() * seg_cost + interior_cnots(free_) * cnot_cost;
    return (c_free < c_fold) ? std::move(free_) : std::move(folded);
  };
  // Pass splitting (whole-state tiles): a JIT pass kernel is one straight-line
  // function, and compile time grows with its segments (cfg3's 32 + 32
  // segments: ~20 s of NVRTC on one core). Passes of more than
  // max_pass_segments segments are cut into equal passes over the same local
  // qubits, whose units compile in parallel; each cut costs a state round
  // trip (measured: cuts down to 6 / 4 segments cost cfg3 25 % / 40 %, so the
  // default only bounds the compile time of deep circuits).
  if (opt.max_pass_segments > 0) {
    std::vector<Group> cut;
    for (Group& pg : passes) {
      const std::vector<Group> sg = make_segments(pg.gates);
      if ((int)sg.size() <= opt.max_pass_segments) {
        cut.push_back(pg);
        continue;
      }
      const int parts = ((int)sg.size() + opt.max_pass_segments - 1) / opt.max_pass_segments;
      const int per = ((int)sg.size() + parts - 1) / parts;
      for (size_t i = 0; i < sg.size(); i += (size_t)per) {
        Group sub;
        sub.mask = pg.mask;
        for (size_t j = i; j < sg.size() && j < i + (size_t)per; ++j)
          sub.gates.insert(sub.gates.end(), sg[j].gates.begin(), sg[j].gates.end());
        cut.push_back(std::move(sub));
      }
    }
    passes.swap(cut);
  }

  for (size_t pi = 0; pi < passes.size(); ++pi) {
    Group& pg = passes[pi];
    // pad the local set to exactly k qubits (lowest unused first)
    for (int q = 0; q < n && popc(pg.mask) < k; ++q) pg.mask |= 1u << q;
    PassDesc pd{};
    pd.k = k;
    pd.local_mask = pg.mask;
    int pos_of[kMaxQubits];
    for (int q = 0, p = 0; q < n; ++q) {
      pos_of[q] = -1;
      if (pg.mask >> q & 1u) { pd.local_q[p] = (int8_t)q; pos_of[q] = p++; }
    }
    pd.rot_begin = next_rot;
    pd.blk_begin = (int)P->blocks.size();
    pd.av_begin = P->n_av;

    std::vector<Group> segs = make_segments(pg.gates);
    if (!pg.gates.empty() && segs.empty()) return "segment scheduling failed";

    struct Item {
      int type;               // 0 single gate, 1 block (1q run on a slot), 2 CZ run, 3 block set
      std::vector<int> gates;
      int id = -1;            // block id / diag-run id / packed set ids
      std::vector<Item> sub;  // blocks of a set
      // first operation on its qubit in the whole schedule: the adjoint sweep
      // needs its inner products but not its un-apply (nothing later in the
      // reverse sweep acts on that qubit, and operators on the other qubits
      // commute with it, so leaving U on both psi and phi changes no later
      // inner product)
      bool dead = false;
    };
    pd.seg_begin = (int)P->segs.size();
    std::vector<SegDesc> fwd_descs;
    std::vector<std::vector<Item>> fwd_items;
    for (Group& sgp : segs) {
      // pad register set to exactly R local qubits
      for (int q = 0; q < n && popc(sgp.mask) < R; ++q)
        if ((pg.mask >> q & 1u) && !(sgp.mask >> q & 1u)) sgp.mask |= 1u << q;
      SegDesc sd{};
      int slot_of[kMaxQubits];
      for (int q = 0; q < kMaxQubits; ++q) slot_of[q] = -1;
      int ns = 0;
      for (int q = 0; q < n; ++q)
        if (sgp.mask >> q & 1u) {
          sd.reg_g[ns] = (int8_t)q;
          sd.reg_l[ns] = (int8_t)pos_of[q];
          slot_of[q] = ns++;
        }
      sd.nreg = (int8_t)ns;
      // thread bits: remaining local positions; the first three cover distinct
      // residues mod 3 so each quarter-warp's 16-byte smem accesses hit 8
      // distinct bank groups under the mod-3 fold swizzle (kernels.cuh swz()).
      std::vector<int> rest;
      for (int p = 0; p < k; ++p)
        if (!(sgp.mask >> pd.local_q[p] & 1u)) rest.push_back(p);
      std::vector<int> order;
      for (int r = 0; r < 3; ++r)
        for (size_t i = 0; i < rest.size(); ++i)
          if (rest[i] >= 0 && rest[i] % 3 == r) { order.push_back(rest[i]); rest[i] = -1; break; }
      for (int p : rest)
        if (p >= 0) order.push_back(p);
      sd.nthr = (int8_t)order.size();
      for (size_t i = 0; i < order.size(); ++i) {
        sd.thr_l[i] = (int8_t)order[i];
        sd.thr_g[i] = pd.local_q[order[i]];
        sd.tsw[i] = (uint16_t)swz_index(1u << order[i]);
      }
      for (int s2 = 0; s2 < ns; ++s2) sd.ps[s2] = (uint16_t)swz_index(1u << sd.reg_l[s2]);
      auto operand = [&](int q) -> uint32_t {
        return slot_of[q] >= 0 ? (kSlotFlag | (uint32_t)slot_of[q]) : (uint32_t)q;
      };

      // group the segment's gates into items: runs of 1q gates on one register
      // qubit become a fused block (placed at its first member; later members
      // only cross gates on other qubits), consecutive CZs become one run
      std::vector<Item> items;
      int open_blk[kMaxQubits];
      for (int q = 0; q < kMaxQubits; ++q) open_blk[q] = -1;
      int open_run = -1;
      for (int g : sgp.gates) {
        const GateIn& gi = gates[g];
        const bool one_q = gi.kind == G_RX || gi.kind == G_RY || gi.kind == G_RZ || gi.kind == G_H ||
                           gi.kind == G_X;
        if (one_q && slot_of[gi.q0] >= 0) {
          if (open_blk[gi.q0] >= 0) {
            items[open_blk[gi.q0]].gates.push_back(g);
          } else {
            open_run = -1;
            items.push_back({1, {g}});
            open_blk[gi.q0] = (int)items.size() - 1;
          }
          continue;
        }
        if (gi.kind == G_CZ) {
          open_blk[gi.q0] = open_blk[gi.q1] = -1;
          if (open_run >= 0) {
            items[open_run].gates.push_back(g);
          } else {
            items.push_back({2, {g}});
            open_run = (int)items.size() - 1;
          }
          continue;
        }
        open_run = -1;
        if (gi.kind == G_CNOT) open_blk[gi.q0] = open_blk[gi.q1] = -1;
        items.push_back({0, {g}});
      }
      // items in execution order: flag 1q items that open their qubit
      if (opt.skip_dead_unapply)
        for (Item& it : items) {
          uint32_t qs = 0;
          bool one_q = true;
          for (int g : it.gates) {
            qs |= 1u << gates[g].q0;
            if (gates[g].kind == G_CNOT || gates[g].kind == G_CZ) {
              qs |= 1u << gates[g].q1;
              one_q = false;
            }
          }
          it.dead = one_q && (qs & touched) == 0u;
          touched |= qs;
        }
      // leading / trailing CNOT runs fold into the load / store address maps
      auto is_cnot = [&](const Item& it) { return it.type == 0 && gates[it.gates[0]].kind == G_CNOT; };
      size_t lead = 0;
      while (lead < items.size() && is_cnot(items[lead])) ++lead;
      size_t trail = items.size();
      while (trail > lead && is_cnot(items[trail - 1])) --trail;
      for (size_t i = 0; i < items.size(); ++i) {
        const bool folded_cnot = (i < lead || i >= trail) && opt.fold_thread_targets;
        for (int g : items[i].gates)
          if (!folded_cnot && (info[g].mix & sgp.mask) != info[g].mix)
            return "internal: mixing qubit not in registers";
          else if (folded_cnot && !(pg.mask >> gates[g].q1 & 1u))
            return "internal: folded CNOT target not in the tile";
      }
      // affine map of a CNOT sequence, restricted to register bits: register
      // output bit t = XOR of register inputs col-masks + const qubits kmask
      auto fold = [&](const std::vector<int>& cnots, uint8_t* col, uint32_t* kmask, uint32_t* lrow) {
        uint32_t row[kMaxQubits];  // row[q]: global-bit mask feeding output bit q
        for (int q = 0; q < n; ++q) row[q] = 1u << q;
        for (int g : cnots) row[gates[g].q1] ^= row[gates[g].q0];
        for (int p = 0; p < kMaxTile; ++p) lrow[p] = p < k ? row[(int)pd.local_q[p]] : 0u;
        uint32_t regmask = 0;
        for (int s2 = 0; s2 < ns; ++s2) regmask |= 1u << sd.reg_g[s2];
        for (int s2 = 0; s2 < kMaxR; ++s2) { col[s2] = 0; kmask[s2] = 0; }
        for (int t = 0; t < ns; ++t) {
          const uint32_t r = row[(int)sd.reg_g[t]];
          kmask[t] = r & ~regmask;
          for (int s2 = 0; s2 < ns; ++s2)
            if (r >> sd.reg_g[s2] & 1u) col[s2] |= (uint8_t)(1u << t);
        }
      };
      std::vector<int> lead_g, trail_g;
      for (size_t i = 0; i < lead; ++i) lead_g.push_back(items[i].gates[0]);
      for (size_t i = trail; i < items.size(); ++i) trail_g.push_back(items[i].gates[0]);
      {
        // loads see C_lead^{-1} (the lead CNOTs in reverse order); stores C_trail
        std::vector<int> inv(lead_g.rbegin(), lead_g.rend());
        fold(inv, sd.ld_col, sd.ld_k, sd.ld_row);
        fold(trail_g, sd.st_col, sd.st_k, sd.st_row);
        // register columns: the swizzled address of register bit s under the
        // map = XOR of swz(e_p) over output positions p whose row reads it
        for (int s2 = 0; s2 < kMaxR; ++s2) {
          uint32_t lcv = 0, scv = 0;
          if (s2 < ns)
            for (int p = 0; p < k; ++p) {
              if (sd.ld_row[p] >> sd.reg_g[s2] & 1u) lcv ^= swz_index(1u << p);
              if (sd.st_row[p] >> sd.reg_g[s2] & 1u) scv ^= swz_index(1u << p);
            }
          sd.ldc[s2] = (uint16_t)lcv;
          sd.stc[s2] = (uint16_t)scv;
        }
        // general maps: some thread-bit output reads other bits
        sd.gen = 0;
        for (int p = 0; p < k; ++p)
          if (!(sgp.mask >> pd.local_q[p] & 1u) &&
              (sd.ld_row[p] != (1u << pd.local_q[p]) || sd.st_row[p] != (1u << pd.local_q[p])))
            sd.gen = 1;
        if (sd.gen && !opt.fold_thread_targets) return "internal: general CNOT fold in an interpreter plan";
      }
      std::vector<Item> body(items.begin() + lead, items.begin() + trail);
      // consecutive fused blocks (distinct slots, commuting) dispatch as one set
      std::vector<Item> grouped;
      for (size_t i = 0; i < body.size();) {
        if (body[i].type == 1) {
          size_t j = i;
          while (j < body.size() && body[j].type == 1) ++j;
          if (j - i >= 2) {
            Item set{3, {}};
            set.sub.assign(body.begin() + i, body.begin() + j);
            grouped.push_back(std::move(set));
            i = j;
            continue;
          }
        }
        grouped.push_back(body[i]);
        ++i;
      }

      auto new_block = [&](const Item& it) {
        for (int g : it.gates)
          if (gates[g].kind <= G_RZ) {
            rot_id[g] = next_rot++;
            if (info[g].need_grad) gslot[g] = next_g++;
          }
        BlockDesc bd{};
        bd.mem_begin = (int)P->members.size();
        for (int g : it.gates) {
          MemberDesc md{};
          md.kind = gates[g].kind;
          md.rot = rot_id[g];
          md.avec = (gates[g].kind <= G_RZ && info[g].need_grad) ? P->n_av++ : -1;
          P->members.push_back(md);
        }
        bd.mem_end = (int)P->members.size();
        P->blocks.push_back(bd);
        return (int)P->blocks.size() - 1;
      };

      sd.op_begin = (int)P->ops.size();
      for (Item& it : grouped) {
        Op op{};
        if (it.type == 3) {
          const int set_id = (int)(P->setids.size() / kMaxR);
          P->setids.resize(P->setids.size() + kMaxR, (int16_t)-1);
          for (Item& sub : it.sub) {
            sub.id = new_block(sub);
            const int rel = sub.id - pd.blk_begin;
            if (rel > 32767) return "too many fused blocks in one pass";
            const int slot = slot_of[gates[sub.gates[0]].q0];
            P->setids[(size_t)set_id * kMaxR + slot] = (int16_t)rel;
          }
          it.id = set_id;
          const uint32_t ids = (uint32_t)set_id;
          uint32_t smask = 0;  // slots of the set (operand b): compile-time dispatch in the kernels
          for (const Item& sub : it.sub) smask |= 1u << slot_of[gates[sub.gates[0]].q0];
          op.w0 = enc(OP_U2SET, 0, smask, 0, false);
          op.param = ids;
          P->ops.push_back(op);
          continue;
        }
        const int g0 = it.gates[0];
        const GateIn& gi0 = gates[g0];
        if (it.type == 1 && it.gates.size() > 1) {
          it.id = new_block(it);
          op.w0 = enc(OP_U2, operand(gi0.q0), 0, 0, false);
          op.param = (uint32_t)it.id;
        } else if (it.type == 2 && it.gates.size() > 1) {
          it.id = (int)P->diag.size();
          DiagRun dr{};
          for (int g : it.gates) {
            const int qa = gates[g].q0, qb = gates[g].q1;
            const int sa = slot_of[qa], sb = slot_of[qb];
            if (sa >= 0 && sb >= 0) {
              for (int r = 0; r < (1 << R); ++r)
                if ((r >> sa & 1) && (r >> sb & 1)) dr.qreg ^= 1u << r;
            } else if (sa >= 0) {
              dr.part[sa] ^= 1u << qb;
            } else if (sb >= 0) {
              dr.part[sb] ^= 1u << qa;
            } else {
              dr.upper[std::min(qa, qb)] ^= 1u << std::max(qa, qb);
            }
          }
          P->diag.push_back(dr);
          op.w0 = enc(OP_CZRUN, 0, 0, 0, false);
          op.param = (uint32_t)it.id;
        } else if (gi0.kind <= G_RZ) {
          rot_id[g0] = next_rot++;
          if (info[g0].need_grad) gslot[g0] = next_g++;
          op.w0 = enc(gi0.kind, operand(gi0.q0), 0, 0, false);
          op.param = (uint32_t)rot_id[g0];
        } else if (gi0.kind == G_H || gi0.kind == G_X) {
          op.w0 = enc(gi0.kind, operand(gi0.q0), 0, 0, false);
        } else {
          op.w0 = enc(gi0.kind, operand(gi0.q0), operand(gi0.q1), 0, false);
        }
        P->ops.push_back(op);
      }
      sd.op_end = (int)P->ops.size();
      P->segs.push_back(sd);
      fwd_descs.push_back(sd);
      fwd_items.push_back(std::move(grouped));
    }
    pd.seg_end = (int)P->segs.size();
    if (P->group_sync && !fwd_descs.empty()) {
      assign_thread_groups(fwd_descs, pd, k);
      for (size_t i = 0; i < fwd_descs.size(); ++i) {
        SegDesc& dst = P->segs[(size_t)pd.seg_begin + i];
        const SegDesc& src = fwd_descs[i];
        for (int t = 0; t < kMaxQubits; ++t) {
          dst.thr_l[t] = src.thr_l[t];
          dst.thr_g[t] = src.thr_g[t];
          dst.tsw[t] = src.tsw[t];
        }
        dst.sync_ld = src.sync_ld;
        dst.sync_st = src.sync_st;
        dst.sync_self = src.sync_self;
      }
    }
    pd.rot_end = next_rot;
    pd.blk_end = (int)P->blocks.size();
    pd.av_end = P->n_av;
    P->max_rot_per_pass = std::max(P->max_rot_per_pass, pd.rot_end - pd.rot_begin);
    P->max_blk_per_pass = std::max(P->max_blk_per_pass, pd.blk_end - pd.blk_begin);
    P->max_av_per_pass = std::max(P->max_av_per_pass, pd.av_end - pd.av_begin);

    // adjoint segments: forward segments reversed (load/store maps swapped),
    // items reversed; gradient inner products before each un-apply
    pd.bseg_begin = (int)P->segs.size();
    for (int si = (int)fwd_descs.size() - 1; si >= 0; --si) {
      SegDesc sd = fwd_descs[si];
      for (int s2 = 0; s2 < kMaxR; ++s2) {
        std::swap(sd.ld_col[s2], sd.st_col[s2]);
        std::swap(sd.ld_k[s2], sd.st_k[s2]);
        std::swap(sd.ldc[s2], sd.stc[s2]);
      }
      for (int p2 = 0; p2 < kMaxTile; ++p2) std::swap(sd.ld_row[p2], sd.st_row[p2]);
      std::swap(sd.sync_ld, sd.sync_st);  // the adjoint sweep meets the boundaries in reverse
      int slot_of[kMaxQubits];
      for (int q = 0; q < kMaxQubits; ++q) slot_of[q] = -1;
      for (int s2 = 0; s2 < sd.nreg; ++s2) slot_of[(int)sd.reg_g[s2]] = s2;
      auto operand = [&](int q) -> uint32_t {
        return slot_of[q] >= 0 ? (kSlotFlag | (uint32_t)slot_of[q]) : (uint32_t)q;
      };
      sd.op_begin = (int)P->ops.size();
      sd.ip_begin = (int)P->ipouts.size();
      int nred = 0, nout = 0;
      auto block_outputs = [&](const Item& it, int red0) {
        const BlockDesc& bd = P->blocks[it.id];
        for (int mi = bd.mem_begin; mi < bd.mem_end; ++mi) {
          const MemberDesc& md = P->members[mi];
          if (md.avec < 0) continue;
          P->ipouts.push_back({gslot[it.gates[mi - bd.mem_begin]], red0, md.avec});
          ++nout;
        }
      };
      auto block_has_grad = [&](const Item& it) {
        for (int g : it.gates)
          if (gates[g].kind <= G_RZ && info[g].need_grad) return true;
        return false;
      };
      const std::vector<Item>& items = fwd_items[si];
      // split adjoint: the partner's state is read from shared memory, which
      // is current only until this segment modifies the registers
      bool dirty = false;
      auto publish_if_dirty = [&]() {
        if (!dirty) return;
        Op pub{};
        pub.w0 = enc(OP_PUBLISH, 0, 0, 0, false);
        P->ops.push_back(pub);
        dirty = false;
      };
      for (int ii = (int)items.size() - 1; ii >= 0; --ii) {
        const Item& it = items[ii];
        Op op{};
        dirty = dirty || ii < (int)items.size() - 1;
        if (it.type == 3) {
          uint32_t gmask = 0;
          for (const Item& sub : it.sub)
            if (block_has_grad(sub)) gmask |= 1u << slot_of[gates[sub.gates[0]].q0];
          if (gmask) {
            publish_if_dirty();
            Op ip{};
            ip.w0 = enc(OP_IP3SET, 0, gmask, (uint32_t)nred, false);
            ip.param = (uint32_t)it.id;
            P->ops.push_back(ip);
            // reduction slots: 3 per flagged register slot, in slot order
            for (const Item& sub : it.sub) {
              const int slot = slot_of[gates[sub.gates[0]].q0];
              if (!(gmask >> slot & 1u)) continue;
              block_outputs(sub, nred + 3 * __builtin_popcount(gmask & ((1u << slot) - 1u)));
            }
            nred += 3 * __builtin_popcount(gmask);
          }
          uint32_t smask = 0, live = 0;
          for (const Item& sub : it.sub) {
            smask |= 1u << slot_of[gates[sub.gates[0]].q0];
            if (!sub.dead) live |= 1u << slot_of[gates[sub.gates[0]].q0];
          }
          if (live == 0u) continue;  // every block of the set opens its qubit: nothing to un-apply
          int set_id = it.id;
          if (live != smask) {  // un-apply the live blocks only: its own id row
            set_id = (int)(P->setids.size() / kMaxR);
            P->setids.resize(P->setids.size() + kMaxR, (int16_t)-1);
            for (int sl = 0; sl < kMaxR; ++sl)
              if (live >> sl & 1u) P->setids[(size_t)set_id * kMaxR + sl] = P->setids[(size_t)it.id * kMaxR + sl];
          }
          op.w0 = enc(OP_U2SET, 0, live, 0, true);
          op.param = (uint32_t)set_id;
          P->ops.push_back(op);
          continue;
        }
        const int g0 = it.gates[0];
        const GateIn& gi0 = gates[g0];
        const bool one_q_item = it.type == 1 || (it.type == 0 && gi0.kind != G_CNOT && gi0.kind != G_CZ);
        if (it.type == 1 && it.gates.size() > 1) {
          if (block_has_grad(it)) {
            publish_if_dirty();
            Op ip{};
            ip.w0 = enc(OP_IP3, operand(gi0.q0), 0, (uint32_t)nred, false);
            ip.param = (uint32_t)it.id;
            P->ops.push_back(ip);
            block_outputs(it, nred);
            nred += 3;
          }
          op.w0 = enc(OP_U2, operand(gi0.q0), 0, 0, true);
          op.param = (uint32_t)it.id;
        } else if (it.type == 2 && it.gates.size() > 1) {
          op.w0 = enc(OP_CZRUN, 0, 0, 0, false);
          op.param = (uint32_t)it.id;
        } else if (gi0.kind <= G_RZ) {
          if (info[g0].need_grad) {
            publish_if_dirty();
            Op ip{};
            ip.w0 = enc(OP_IPX + gi0.kind, operand(gi0.q0), 0, (uint32_t)nred, false);
            ip.param = (uint32_t)gslot[g0];
            P->ops.push_back(ip);
            P->ipouts.push_back({gslot[g0], nred, -1});
            ++nred;
            ++nout;
          }
          op.w0 = enc(gi0.kind, operand(gi0.q0), 0, 0, true);
          op.param = (uint32_t)rot_id[g0];
        } else if (gi0.kind == G_H || gi0.kind == G_X) {
          op.w0 = enc(gi0.kind, operand(gi0.q0), 0, 0, false);
        } else {
          op.w0 = enc(gi0.kind, operand(gi0.q0), operand(gi0.q1), 0, false);
        }
        if (it.dead && one_q_item) continue;  // inner products only (Item::dead)
        P->ops.push_back(op);
      }
      if (nred > 1023) return "too many gradient rotations in one segment";
      sd.op_end = (int)P->ops.size();
      sd.ip_count = nout;
      sd.red_count = nred;
      P->max_red_per_seg = std::max(P->max_red_per_seg, nred);
      P->max_ipout_per_seg = std::max(P->max_ipout_per_seg, nout);
      P->segs.push_back(sd);
    }
    pd.bseg_end = (int)P->segs.size();
    {
      int pass_red = 0;
      for (int s2 = pd.bseg_begin; s2 < pd.bseg_end; ++s2) pass_red += P->segs[s2].red_count;
      P->max_red_per_pass = std::max(P->max_red_per_pass, pass_red);
    }
    P->passes.push_back(pd);
  }
  P->n_rot = next_rot;
  P->NG = next_g;
  P->n_blk = (int)P->blocks.size();
  P->n_fwd_ops = 0;
  P->n_bwd_ops = 0;
  for (const PassDesc& pd : P->passes) {
    for (int s = pd.seg_begin; s < pd.seg_end; ++s) P->n_fwd_ops += P->segs[s].op_end - P->segs[s].op_begin;
    for (int s = pd.bseg_begin; s < pd.bseg_end; ++s) P->n_bwd_ops += P->segs[s].op_end - P->segs[s].op_begin;
  }

  // rotation angle descriptors, indexed by rotation id
  P->rots.assign(P->n_rot, RotDesc{});
  for (int g = 0; g < G; ++g)
    if (rot_id[g] >= 0) {
      RotDesc& rd = P->rots[rot_id[g]];
      rd.coeff = gates[g].coeff;
      rd.nf = (int32_t)gates[g].fidx.size();
      for (int i = 0; i < rd.nf; ++i) rd.fidx[i] = gates[g].fidx[i];
    }

  // chain rule table (_kernels.py:269-278), reference accumulation order:
  // gates from last to first, factors in expression order
  int64_t max_col = -1;
  for (int64_t c : wrt_col) max_col = std::max(max_col, c);
  P->n_cols = (int)(max_col + 1);
  std::vector<std::vector<ChainEntry>> per_col(P->n_cols);
  for (int g = G - 1; g >= 0; --g) {
    if (gslot[g] < 0) continue;
    const std::vector<int32_t>& fx = gates[g].fidx;
    for (size_t t = 0; t < fx.size(); ++t) {
      const int64_t col = wrt_col[fx[t]];
      if (col < 0) continue;
      ChainEntry ce{};
      ce.gslot = gslot[g];
      ce.coeff = gates[g].coeff;
      ce.nother = 0;
      for (size_t u = 0; u < fx.size(); ++u)
        if (u != t) ce.other[ce.nother++] = fx[u];
      per_col[col].push_back(ce);
    }
  }
  P->col_offs.assign(P->n_cols + 1, 0);
  for (int c = 0; c < P->n_cols; ++c) {
    P->col_offs[c + 1] = P->col_offs[c] + (int32_t)per_col[c].size();
    P->chain.insert(P->chain.end(), per_col[c].begin(), per_col[c].end());
  }
  return "";
}

}  // namespace vqc
