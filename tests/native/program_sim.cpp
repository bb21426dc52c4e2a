// TEST INFRASTRUCTURE: semantic CPU interpreter of the device program that
// scheduler.cpp emits (program.h), used to check the scheduler on CPU.
//
// It executes passes / segments / ops exactly in the order the kernels do,
// resolving register slots to qubits through the segment descriptors, on a
// full complex128 state — so a wrong reordering, operand encoding, IP
// placement, gradient-slot map or chain-rule table shows up as a mismatch
// against the oracle. It also asserts the structural invariants the kernels
// rely on (tile sizes, slot/thread-bit partitions, mixing operands in
// registers). It does not model the kernels' tiling arithmetic (swizzle,
// pdep); the GPU parity tests cover that.
#include <stdexcept>
#include <array>
#include <cmath>
#include <cstdio>
#include <algorithm>
#include <complex>
#include <cstring>
#include <string>
#include <vector>

#include "../../paper_2404_06314_b200/csrc/blockmath.h"
#include "../../paper_2404_06314_b200/csrc/scheduler.h"

using namespace vqc;
using cd = std::complex<double>;

namespace {

struct Sim {
  int n;
  std::vector<cd> psi, phi;
  bool dual = false;

  void rot(std::vector<cd>& s, int kind, int q, double c, double sn) {
    const size_t step = (size_t)1 << q;
    for (size_t j = 0; j < s.size(); ++j) {
      if (j & step) continue;
      cd a0 = s[j], a1 = s[j | step];
      if (kind == G_RX) {
        s[j] = c * a0 - cd(0, sn) * a1;
        s[j | step] = -cd(0, sn) * a0 + c * a1;
      } else if (kind == G_RY) {
        s[j] = c * a0 - sn * a1;
        s[j | step] = sn * a0 + c * a1;
      } else {
        s[j] = cd(c, -sn) * a0;
        s[j | step] = cd(c, sn) * a1;
      }
    }
  }
  void fixed(std::vector<cd>& s, int kind, int a, int b) {
    const size_t ma = (size_t)1 << a, mb = (size_t)1 << b;
    for (size_t j = 0; j < s.size(); ++j) {
      if (kind == G_H && !(j & ma)) {
        cd x = s[j], y = s[j | ma];
        const double inv = 1.0 / std::sqrt(2.0);
        s[j] = (x + y) * inv;
        s[j | ma] = (x - y) * inv;
      } else if (kind == G_X && !(j & ma)) {
        std::swap(s[j], s[j | ma]);
      } else if (kind == G_CNOT && (j & ma) && !(j & mb)) {
        std::swap(s[j], s[j | mb]);
      } else if (kind == G_CZ && (j & ma) && (j & mb)) {
        s[j] = -s[j];
      }
    }
  }
  double ip(int axis, int q) {
    const size_t m = (size_t)1 << q;
    cd acc = 0;
    for (size_t j = 0; j < psi.size(); ++j) {
      cd pj;
      if (axis == 0) pj = psi[j ^ m];
      else if (axis == 1) pj = (j & m) ? cd(0, 1) * psi[j ^ m] : cd(0, -1) * psi[j ^ m];
      else pj = (j & m) ? -psi[j] : psi[j];
      acc += std::conj(phi[j]) * pj;
    }
    return acc.imag();
  }
};

std::string check_program(const HostProgram& P, const ScheduleOptions& opt) {
  for (size_t pi = 0; pi < P.passes.size(); ++pi) {
    const PassDesc& pd = P.passes[pi];
    if (__builtin_popcount(pd.local_mask) != P.k) return "pass local set size != k";
    if (P.hbm && (pd.local_mask & ((1u << opt.forced_low) - 1u)) != ((1u << opt.forced_low) - 1u))
      return "pass misses forced low qubits";
    for (int p = 0; p < P.k; ++p)
      if (!((pd.local_mask >> pd.local_q[p]) & 1u) || (p > 0 && pd.local_q[p] <= pd.local_q[p - 1]))
        return "local_q not the ascending local set";
    auto check_seg = [&](const SegDesc& sd) -> std::string {
      if (sd.nreg != P.R || sd.nthr != P.k - P.R) return "segment slot/thread counts";
      uint32_t seen = 0;
      for (int s = 0; s < sd.nreg; ++s) {
        if (pd.local_q[(int)sd.reg_l[s]] != sd.reg_g[s]) return "reg_l/reg_g mismatch";
        seen |= 1u << sd.reg_g[s];
      }
      for (int i = 0; i < sd.nthr; ++i) {
        if (pd.local_q[(int)sd.thr_l[i]] != sd.thr_g[i]) return "thr_l/thr_g mismatch";
        if (seen >> sd.thr_g[i] & 1u) return "thread bit overlaps a slot";
        seen |= 1u << sd.thr_g[i];
      }
      if (seen != pd.local_mask) return "slots + thread bits != local set";
      // the JIT kernels' shared-memory addresses (jit.cpp emit_segment: thread
      // base from the rows' thread bits, tile translation from their tile
      // bits, register columns ldc / stc) must equal swz(local part of the
      // row map) for every thread, register index and tile
      {
        const uint32_t nmask = (P.n >= 32) ? 0xffffffffu : ((1u << P.n) - 1u);
        const uint32_t thr_mask = pd.local_mask & ~[&] { uint32_t r = 0; for (int q = 0; q < sd.nreg; ++q) r |= 1u << sd.reg_g[q]; return r; }();
        const uint32_t tile_mask = ~pd.local_mask & nmask;
        auto kernel_addr = [&](const uint32_t* row, const uint16_t* cols, uint32_t j, uint32_t i, uint32_t tb) {
          uint32_t a = 0;
          for (int q = 0; q < P.k && q < kMaxTile; ++q) {
            if (__builtin_popcount(j & row[q] & thr_mask) & 1) a ^= swz_index(1u << q);
            if (__builtin_popcount(tb & row[q] & tile_mask) & 1) a ^= swz_index(1u << q);
          }
          for (int s2 = 0; s2 < sd.nreg; ++s2)
            if (i >> s2 & 1u) a ^= cols[s2];
          return a;
        };
        auto want_addr = [&](const uint32_t* row, uint32_t x) {
          uint32_t v = 0;
          for (int q = 0; q < P.k && q < kMaxTile; ++q) v |= (uint32_t)(__builtin_popcount(x & row[q]) & 1) << q;
          return swz_index(v);
        };
        const uint32_t tiles[3] = {0u, tile_mask, tile_mask & 0x5555u};
        for (uint32_t g = 0; g < (1u << sd.nthr); ++g)
          for (uint32_t i = 0; i < (1u << sd.nreg); ++i)
            for (uint32_t tb : tiles) {
              uint32_t j = 0, r = 0;
              for (int b = 0; b < sd.nthr; ++b) j |= ((g >> b) & 1u) << sd.thr_g[b];
              for (int b = 0; b < sd.nreg; ++b) r |= ((i >> b) & 1u) << sd.reg_g[b];
              const uint32_t x = j | r | tb;
              if (kernel_addr(sd.ld_row, sd.ldc, j, i, tb) != want_addr(sd.ld_row, x)) return "JIT load address != row map";
              if (kernel_addr(sd.st_row, sd.stc, j, i, tb) != want_addr(sd.st_row, x)) return "JIT store address != row map";
            }
      }
      for (int o = sd.op_begin; o < sd.op_end; ++o) {
        const Op& op = P.ops[o];
        const uint32_t code = op_code(op.w0), a = op_a(op.w0), b = op_b(op.w0);
        auto in_regs = [&](uint32_t x) { return (x & kSlotFlag) && (int)(x & 7u) < sd.nreg; };
        auto ok_const = [&](uint32_t x) {
          if (x & kSlotFlag) return (int)(x & 7u) < sd.nreg;
          if ((int)x >= P.n) return false;
          for (int s = 0; s < sd.nreg; ++s)
            if ((uint32_t)sd.reg_g[s] == x) return false;  // register qubits must use slots
          return true;
        };
        switch (code) {
          case OP_CZRUN:
            if ((int)op.param >= (int)P.diag.size()) return "bad diag run id";
            break;
          case OP_PUBLISH:
            break;
          case OP_U2SET: case OP_IP3SET:
            for (int sl = 0; sl < sd.nreg; ++sl) {
              const int id = P.setids[op.param * kMaxR + sl];
              if (id >= pd.blk_end - pd.blk_begin) return "set block id out of range";
            }
            if (code == OP_IP3SET && (b & ~((1u << sd.nreg) - 1u))) return "IP3SET mask beyond slots";
            if (code == OP_U2SET) {
              uint32_t m = 0;
              for (int sl = 0; sl < kMaxR; ++sl)
                if (P.setids[op.param * kMaxR + sl] >= 0) m |= 1u << sl;
              if (m != b) return "U2SET slot mask (operand b) disagrees with its block ids";
            }
            break;
          case OP_U2: case OP_IP3:
            if ((int)op.param < pd.blk_begin || (int)op.param >= pd.blk_end) return "block id outside pass range";
            if (!in_regs(a)) return "block operand not a register slot";
            break;
          case OP_RX: case OP_RY: case OP_H: case OP_X: case OP_IPX: case OP_IPY:
            if (!in_regs(a)) return "mixing operand not a register slot";
            break;
          case OP_RZ: case OP_IPZ:
            if (!ok_const(a)) return "bad RZ operand";
            break;
          case OP_CNOT:
            if (!in_regs(b)) return "CNOT target not in registers";
            if (!ok_const(a)) return "bad CNOT control";
            break;
          case OP_CZ:
            if (!ok_const(a) || !ok_const(b)) return "bad CZ operand";
            break;
          default:
            return "unknown opcode";
        }
      }
      return "";
    };
    // Thread-group barriers (scheduler.cpp assign_thread_groups): a boundary
    // with sync level t is synchronised over the groups of threads sharing
    // the top t thread-index bits only, so every such group must store
    // exactly the shared-memory cells it loads in the next segment (and load
    // / store the same cells inside a segment whose stores leave the loading
    // threads' cells, level sync_self).
    if (opt.group_sync) {
      const uint32_t nmask = (P.n >= 32) ? 0xffffffffu : ((1u << P.n) - 1u);
      const uint32_t tile_mask = ~pd.local_mask & nmask;
      auto cells = [&](const SegDesc& sd, const uint32_t* row, int t, uint32_t grp, uint32_t tb) {
        std::vector<uint32_t> out;
        const int low = sd.nthr - t;
        for (uint32_t g = 0; g < (1u << sd.nthr); ++g) {
          if (t > 0 && (g >> low) != grp) continue;
          for (uint32_t i = 0; i < (1u << sd.nreg); ++i) {
            uint32_t x = tb;
            for (int b = 0; b < sd.nthr; ++b) x |= ((g >> b) & 1u) << sd.thr_g[b];
            for (int b = 0; b < sd.nreg; ++b) x |= ((i >> b) & 1u) << sd.reg_g[b];
            uint32_t v = 0;
            for (int q = 0; q < P.k && q < kMaxTile; ++q) v |= (uint32_t)(__builtin_popcount(x & row[q]) & 1) << q;
            out.push_back(swz_index(v));
          }
        }
        std::sort(out.begin(), out.end());
        return out;
      };
      const uint32_t tiles[3] = {0u, tile_mask, tile_mask & 0x5555u};
      auto check_sweep = [&](int sb, int se) -> std::string {
        for (int s = sb; s < se; ++s) {
          const SegDesc& a = P.segs[s];
          if (s == sb && a.sync_ld != 0) return "first segment of a sweep must load behind a CTA barrier";
          if (s + 1 == se && a.sync_st != 0) return "last segment of a sweep must store before a CTA barrier";
          for (uint32_t tb : tiles) {
            if (a.gen && a.sync_self > 0)
              for (uint32_t grp = 0; grp < (1u << a.sync_self); ++grp)
                if (cells(a, a.ld_row, a.sync_self, grp, tb) != cells(a, a.st_row, a.sync_self, grp, tb))
                  return "thread group loads and stores different cells (sync_self)";
            if (s + 1 < se) {
              const SegDesc& b = P.segs[s + 1];
              if (a.sync_st != b.sync_ld) return "sync_st / sync_ld of a boundary disagree";
              for (uint32_t grp = 0; grp < (1u << a.sync_st); ++grp)
                if (cells(a, a.st_row, a.sync_st, grp, tb) != cells(b, b.ld_row, b.sync_ld, grp, tb))
                  return "thread group stores cells another group loads next";
            }
          }
        }
        return "";
      };
      std::string e = check_sweep(pd.seg_begin, pd.seg_end);
      if (e.empty()) e = check_sweep(pd.bseg_begin, pd.bseg_end);
      if (!e.empty()) return e;
    }
    for (int s = pd.seg_begin; s < pd.seg_end; ++s) {
      std::string e = check_seg(P.segs[s]);
      if (!e.empty()) return e;
    }
    for (int s = pd.bseg_begin; s < pd.bseg_end; ++s) {
      std::string e = check_seg(P.segs[s]);
      if (!e.empty()) return e;
    }
  }
  return "";
}

}  // namespace

static int sim_exec(const HostProgram& P, int n, int M, const int64_t* term_offs, const std::vector<uint32_t>& zm,
                    const std::vector<double>& zc, const double* flat, const double* upstream, double* expect_out,
                    double* grad_out, int64_t* stats);

extern "C" {

// One row: flat (total_params) with the encoding slice already set.
// upstream (M) != NULL -> VJP (grad_out: n_cols); else Jacobian (M x n_cols).
// stats: [passes, segments, rotations, grad_slots].
int sim_run(int n, int64_t G, const int64_t* kinds, const int64_t* q0, const int64_t* q1,
            const double* coeff, const int64_t* f_offs, const int64_t* f_idx, int64_t total_params,
            const int64_t* wrt_col, int tile_qubits, int smem_max_qubits, int reg_slots, int M, const int64_t* term_offs,
            const double* t_coeff, const int64_t* t_smask, const double* flat, const double* upstream,
            double* expect_out, double* grad_out, int64_t* stats, char* err, int errcap) {
  std::vector<GateIn> gates((size_t)G);
  for (int64_t g = 0; g < G; ++g) {
    gates[g].kind = (int)kinds[g];
    gates[g].q0 = (int)q0[g];
    gates[g].q1 = (int)q1[g];
    gates[g].coeff = coeff[g];
    if (kinds[g] <= 2)
      for (int64_t t = f_offs[g]; t < f_offs[g + 1]; ++t) gates[g].fidx.push_back((int32_t)f_idx[t]);
  }
  std::vector<int64_t> wc(wrt_col, wrt_col + total_params);
  ScheduleOptions opt;
  opt.tile_qubits = tile_qubits;
  opt.smem_max_qubits = smem_max_qubits;
  opt.reg_slots = reg_slots;
  // boundary CNOTs folded onto thread-bit targets, as JIT HBM plans do
  // (VQC_FOLD_THREAD_TARGETS=0 turns it off, like the engine)
  {
    const char* ft = getenv("VQC_FOLD_THREAD_TARGETS");
    opt.fold_thread_targets = n > smem_max_qubits && !(ft && ft[0] == '0');
    const char* ps = getenv("VQC_PASS_SEGMENTS");  // pass splitting (whole-state tiles), as the engine
    if (ps && n <= 12 && n > smem_max_qubits) opt.max_pass_segments = atoi(ps);
    const char* gs = getenv("VQC_GROUP_SYNC");  // thread-group barriers, as JIT HBM plans
    opt.group_sync = n > smem_max_qubits && !(gs && gs[0] == '0');
  }
  // as vqc_plan_create: trailing CNOT / CZ / X gates fold into the (Z-string)
  // observables, which the expectation step below then uses
  const int64_t T = M > 0 ? term_offs[M] : 0;
  std::vector<uint32_t> zm(T);
  std::vector<double> zc(t_coeff, t_coeff + T);
  for (int64_t t = 0; t < T; ++t) zm[t] = (uint32_t)t_smask[t];
  absorb_trailing_gates(&gates, n, &zm, &zc);
  HostProgram P;
  std::string e = build_program(gates, n, total_params, wc, opt, &P);
  if (e.empty()) e = check_program(P, opt);
  if (!e.empty()) {
    snprintf(err, (size_t)errcap, "%s", e.c_str());
    return -1;
  }
  try {
    return sim_exec(P, n, M, term_offs, zm, zc, flat, upstream, expect_out, grad_out, stats);
  } catch (const std::exception& ex) {
    snprintf(err, (size_t)errcap, "%s", ex.what());
    return -2;
  }
}

}  // extern "C"

static int sim_exec(const HostProgram& P, int n, int M, const int64_t* term_offs, const std::vector<uint32_t>& zm,
                    const std::vector<double>& zc, const double* flat, const double* upstream, double* expect_out,
                    double* grad_out, int64_t* stats) {
  int nseg = 0;
  for (const PassDesc& pd : P.passes) nseg += pd.seg_end - pd.seg_begin;
  stats[0] = (int64_t)P.passes.size();
  stats[1] = nseg;
  stats[2] = P.n_rot;
  stats[3] = P.NG;

  std::vector<double> c(P.n_rot), s(P.n_rot);
  for (int r = 0; r < P.n_rot; ++r) {
    double a = P.rots[r].coeff;
    for (int t = 0; t < P.rots[r].nf; ++t) a *= flat[P.rots[r].fidx[t]];
    c[r] = std::cos(0.5 * a);
    s[r] = std::sin(0.5 * a);
  }
  Sim S;
  S.n = n;
  const size_t N = (size_t)1 << n;
  S.psi.assign(N, 0);
  S.psi[0] = 1;
  auto qubit_of = [](const SegDesc& sd, uint32_t x) -> int {
    return (x & kSlotFlag) ? sd.reg_g[x & 7u] : (int)x;
  };
  // per-sample block tables (same math as the kernels' build_tables)
  struct CS { double x, y; };
  std::vector<M2> U(P.blocks.size());
  std::vector<std::array<double, 3>> avec((size_t)P.n_av);
  for (size_t bi = 0; bi < P.blocks.size(); ++bi) {
    const BlockDesc& bd = P.blocks[bi];
    U[bi] = block_unitary(P.members.data() + bd.mem_begin, bd.mem_end - bd.mem_begin,
                          [&](int r) { return CS{c[r], s[r]}; },
                          [&](int slot, const double* v) { avec[slot] = {v[0], v[1], v[2]}; });
  }
  int cur_blk_base = 0;
  // folded CNOT runs: every tile-local output bit p of an index is
  // parity(index & row[p]) (SegDesc ld_row / st_row), the general form the
  // JIT kernels compute their smem addresses from; for interpreter plans
  // (gen = 0) the rows must agree with the register-only (col, k) form
  const PassDesc* cur_pd = nullptr;
  auto remap_rows = [&](const uint32_t* row, uint32_t x) {
    uint32_t out = x & ~cur_pd->local_mask;
    for (int p = 0; p < P.k; ++p)
      out |= (uint32_t)(__builtin_popcount(x & row[p]) & 1) << cur_pd->local_q[p];
    return out;
  };
  auto remap = [&](const SegDesc& sd, const uint8_t* col, const uint32_t* km, uint32_t x) {
    uint32_t regmask = 0;
    for (int q = 0; q < sd.nreg; ++q) regmask |= 1u << sd.reg_g[q];
    const uint32_t J0 = x & ~regmask;
    uint32_t i = 0;
    for (int q = 0; q < sd.nreg; ++q) i |= ((x >> sd.reg_g[q]) & 1u) << q;
    uint32_t y = 0;
    for (int q = 0; q < sd.nreg; ++q)
      if (i >> q & 1u) y ^= col[q];
    for (int t = 0; t < sd.nreg; ++t)
      if (__builtin_popcount(J0 & km[t]) & 1) y ^= 1u << t;
    uint32_t out = J0;
    for (int q = 0; q < sd.nreg; ++q) out |= ((y >> q) & 1u) << sd.reg_g[q];
    return out;
  };
  auto map_ld = [&](const SegDesc& sd, uint32_t x) {
    const uint32_t r = remap_rows(sd.ld_row, x);
    if (!sd.gen && r != remap(sd, sd.ld_col, sd.ld_k, x)) {
      char m[256];
      snprintf(m, sizeof m, "ld rows disagree: x=%x rows=%x colk=%x nreg=%d reg0=%d row0=%x k0=%x col0=%x", x, r,
               remap(sd, sd.ld_col, sd.ld_k, x), sd.nreg, sd.reg_g[0], sd.ld_row[0], sd.ld_k[0], sd.ld_col[0]);
      throw std::runtime_error(m);
    }
    return r;
  };
  auto map_st = [&](const SegDesc& sd, uint32_t x) {
    const uint32_t r = remap_rows(sd.st_row, x);
    if (!sd.gen && r != remap(sd, sd.st_col, sd.st_k, x)) throw std::runtime_error("st rows disagree");
    return r;
  };
  // load: reg content at x = state[map_ld(x)]; store: state'[map_st(x)] = reg content at x
  auto do_load = [&](std::vector<cd>& st, const SegDesc& sd) {
    std::vector<cd> o(st.size());
    for (size_t x = 0; x < st.size(); ++x) o[x] = st[map_ld(sd, (uint32_t)x)];
    st.swap(o);
  };
  auto do_store = [&](std::vector<cd>& st, const SegDesc& sd) {
    std::vector<cd> o(st.size());
    for (size_t x = 0; x < st.size(); ++x) o[map_st(sd, (uint32_t)x)] = st[x];
    st.swap(o);
  };
  auto apply = [&](std::vector<cd>& st, const SegDesc& sd, const Op& op) {
    const uint32_t code = op_code(op.w0);
    const int qa = qubit_of(sd, op_a(op.w0)), qb = qubit_of(sd, op_b(op.w0));
    if (code <= OP_RZ) {
      const double sn = op_adj(op.w0) ? -s[op.param] : s[op.param];
      S.rot(st, (int)code, qa, c[op.param], sn);
    } else if (code == OP_U2) {
      M2 u = U[op.param];
      if (op_adj(op.w0)) u = mdag(u);
      const size_t m = (size_t)1 << qa;
      for (size_t j = 0; j < st.size(); ++j) {
        if (j & m) continue;
        const cd x = st[j], y = st[j | m];
        st[j] = cd(u.a.re, u.a.im) * x + cd(u.b.re, u.b.im) * y;
        st[j | m] = cd(u.c.re, u.c.im) * x + cd(u.d.re, u.d.im) * y;
      }
    } else if (code == OP_U2SET) {
      for (int sl = 0; sl < sd.nreg; ++sl) {
        const int id = P.setids[op.param * kMaxR + sl];
        if (id < 0) continue;
        M2 u = U[cur_blk_base + id];
        if (op_adj(op.w0)) u = mdag(u);
        const size_t m = (size_t)1 << sd.reg_g[sl];
        for (size_t j = 0; j < st.size(); ++j) {
          if (j & m) continue;
          const cd x = st[j], y = st[j | m];
          st[j] = cd(u.a.re, u.a.im) * x + cd(u.b.re, u.b.im) * y;
          st[j | m] = cd(u.c.re, u.c.im) * x + cd(u.d.re, u.d.im) * y;
        }
      }
    } else if (code == OP_CZRUN) {
      const DiagRun& dr = P.diag[op.param];
      uint32_t regmask = 0;
      for (int q = 0; q < sd.nreg; ++q) regmask |= 1u << sd.reg_g[q];
      for (size_t j = 0; j < st.size(); ++j) {
        const uint32_t J0 = (uint32_t)j & ~regmask;
        uint32_t r = 0;
        for (int q = 0; q < sd.nreg; ++q) r |= ((uint32_t)(j >> sd.reg_g[q]) & 1u) << q;
        uint32_t qc = 0, mm = 0;
        for (int cb = 0; cb < n; ++cb)
          if (J0 >> cb & 1u) qc ^= (uint32_t)__builtin_popcount(J0 & dr.upper[cb]);
        for (int q = 0; q < sd.nreg; ++q) mm |= ((uint32_t)__builtin_popcount(J0 & dr.part[q]) & 1u) << q;
        if ((qc ^ (dr.qreg >> r) ^ (uint32_t)__builtin_popcount(r & mm)) & 1u) st[j] = -st[j];
      }
    } else {
      S.fixed(st, (int)code, qa, qb);
    }
  };
  for (const PassDesc& pd : P.passes) {
    cur_blk_base = pd.blk_begin;
    cur_pd = &pd;
    for (int sg = pd.seg_begin; sg < pd.seg_end; ++sg) {
      const SegDesc& sd = P.segs[sg];
      do_load(S.psi, sd);
      for (int o = sd.op_begin; o < sd.op_end; ++o) apply(S.psi, sd, P.ops[o]);
      do_store(S.psi, sd);
    }
  }
  auto zw = [&](size_t j, int lo, int hi) {
    double w = 0;
    for (int t = lo; t < hi; ++t) w += (__builtin_popcountll(j & (size_t)zm[t]) & 1) ? -zc[t] : zc[t];
    return w;
  };
  for (int m = 0; m < M; ++m) {
    double acc = 0;
    for (size_t j = 0; j < N; ++j) acc += zw(j, (int)term_offs[m], (int)term_offs[m + 1]) * std::norm(S.psi[j]);
    expect_out[m] = acc;
  }
  const int K = upstream ? 1 : M;
  const std::vector<cd> psi_fin = S.psi;
  std::vector<double> ipv((size_t)P.NG);
  for (int kb = 0; kb < K; ++kb) {
    S.psi = psi_fin;
    S.phi.assign(N, 0);
    for (size_t j = 0; j < N; ++j) {
      double w = 0;
      if (upstream) {
        for (int m = 0; m < M; ++m) w += upstream[m] * zw(j, (int)term_offs[m], (int)term_offs[m + 1]);
      } else {
        w = zw(j, (int)term_offs[kb], (int)term_offs[kb + 1]);
      }
      S.phi[j] = w * S.psi[j];
    }
    std::fill(ipv.begin(), ipv.end(), 0.0);
    for (int pi = (int)P.passes.size() - 1; pi >= 0; --pi) {
      const PassDesc& pd = P.passes[pi];
      cur_blk_base = pd.blk_begin;
      cur_pd = &pd;
      for (int sg = pd.bseg_begin; sg < pd.bseg_end; ++sg) {
        const SegDesc& sd = P.segs[sg];
        do_load(S.psi, sd);
        do_load(S.phi, sd);
        std::vector<double> red((size_t)std::max(1, sd.red_count), 0.0);
        for (int o = sd.op_begin; o < sd.op_end; ++o) {
          const Op& op = P.ops[o];
          const uint32_t code = op_code(op.w0);
          const int q = qubit_of(sd, op_a(op.w0));
          if (code == OP_PUBLISH) {
            continue;
          } else if (code == OP_IPX || code == OP_IPY || code == OP_IPZ) {
            red[op_ip(op.w0)] = S.ip((int)(code - OP_IPX), q);
          } else if (code == OP_IP3) {
            for (int ax = 0; ax < 3; ++ax) red[op_ip(op.w0) + ax] = S.ip(ax, q);
          } else if (code == OP_IP3SET) {
            int r0 = (int)op_ip(op.w0);
            for (int sl = 0; sl < sd.nreg; ++sl) {
              if (!(op_b(op.w0) >> sl & 1u)) continue;
              for (int ax = 0; ax < 3; ++ax) red[r0 + ax] = S.ip(ax, sd.reg_g[sl]);
              r0 += 3;
            }
          } else {
            apply(S.psi, sd, op);
            apply(S.phi, sd, op);
          }
        }
        do_store(S.psi, sd);
        do_store(S.phi, sd);
        for (int oi = 0; oi < sd.ip_count; ++oi) {
          const IpOut& io = P.ipouts[sd.ip_begin + oi];
          if (io.red < 0 || io.red >= sd.red_count) throw std::runtime_error("IpOut reduction slot out of range");
          ipv[io.gslot] = io.avec < 0 ? red[io.red]
                                      : avec[io.avec][0] * red[io.red] + avec[io.avec][1] * red[io.red + 1] +
                                            avec[io.avec][2] * red[io.red + 2];
        }
      }
    }
    for (int col = 0; col < P.n_cols; ++col) {
      double acc = 0;
      for (int e2 = P.col_offs[col]; e2 < P.col_offs[col + 1]; ++e2) {
        const ChainEntry& ce = P.chain[e2];
        double partial = ce.coeff;
        for (int u = 0; u < ce.nother; ++u) partial *= flat[ce.other[u]];
        acc += ipv[ce.gslot] * partial;
      }
      grad_out[(size_t)kb * P.n_cols + col] = acc;
    }
  }
  return 0;
}

extern "C" {
// Debug: print the lowered program (op codes per segment) to stdout.
int sim_dump(int n, int64_t G, const int64_t* kinds, const int64_t* q0, const int64_t* q1,
             const double* coeff, const int64_t* f_offs, const int64_t* f_idx, int64_t total_params,
             const int64_t* wrt_col, int tile_qubits, int smem_max_qubits, int reg_slots) {
  std::vector<GateIn> gates((size_t)G);
  for (int64_t g = 0; g < G; ++g) {
    gates[g].kind = (int)kinds[g];
    gates[g].q0 = (int)q0[g];
    gates[g].q1 = (int)q1[g];
    gates[g].coeff = coeff[g];
    if (kinds[g] <= 2)
      for (int64_t t = f_offs[g]; t < f_offs[g + 1]; ++t) gates[g].fidx.push_back((int32_t)f_idx[t]);
  }
  std::vector<int64_t> wc(wrt_col, wrt_col + total_params);
  ScheduleOptions opt;
  opt.tile_qubits = tile_qubits;
  opt.smem_max_qubits = smem_max_qubits;
  opt.reg_slots = reg_slots;
  {
    const char* ft = getenv("VQC_FOLD_THREAD_TARGETS");
    opt.fold_thread_targets = n > smem_max_qubits && !(ft && ft[0] == '0');
    const char* gs = getenv("VQC_GROUP_SYNC");  // thread-group barriers, as JIT HBM plans
    opt.group_sync = n > smem_max_qubits && !(gs && gs[0] == '0');
  }
  HostProgram P;
  std::string e = build_program(gates, n, total_params, wc, opt, &P);
  if (!e.empty()) { printf("error: %s\n", e.c_str()); return -1; }
  static const char* names[] = {"RX","RY","RZ","CNOT","H","X","CZ","IPX","IPY","IPZ","U2","IP3","CZRUN","U2SET","IP3SET","PUB"};
  for (size_t pi = 0; pi < P.passes.size(); ++pi) {
    const PassDesc& pd = P.passes[pi];
    printf("pass %zu local=%x\n", pi, pd.local_mask);
    for (int sg = pd.seg_begin; sg < pd.seg_end; ++sg) {
      const SegDesc& sd = P.segs[sg];
      printf("  fseg regs=");
      for (int s = 0; s < sd.nreg; ++s) printf("%d,", sd.reg_g[s]);
      printf(" ops:");
      for (int o = sd.op_begin; o < sd.op_end; ++o) {
        const Op& op = P.ops[o];
        printf(" %s", names[op_code(op.w0)]);
        if (op_code(op.w0) == OP_U2SET) {
          printf("[");
          for (int s2 = 0; s2 < kMaxR; ++s2) {
            const int id = P.setids[op.param * kMaxR + s2];
            if (id >= 0) {
              const BlockDesc& bd = P.blocks[pd.blk_begin + id];
              printf("q%d:%d ", sd.reg_g[s2], bd.mem_end - bd.mem_begin);
            }
          }
          printf("]");
        } else if (op_code(op.w0) == OP_U2) {
          const BlockDesc& bd = P.blocks[op.param];
          printf("[q%d:%d]", (op_a(op.w0) & kSlotFlag) ? sd.reg_g[op_a(op.w0) & 7] : -1, bd.mem_end - bd.mem_begin);
        }
      }
      printf("  ldmap=%s stmap=%s\n", (sd.ld_col[0] == 1 && sd.ld_col[1] == 2 && !sd.ld_k[0] && !sd.ld_k[1] && !sd.ld_k[2] && !sd.ld_k[3]) ? "id" : "cnot",
             (sd.st_col[0] == 1 && sd.st_col[1] == 2 && !sd.st_k[0] && !sd.st_k[1] && !sd.st_k[2] && !sd.st_k[3]) ? "id" : "cnot");
    }
    for (int sg = pd.bseg_begin; sg < pd.bseg_end; ++sg) {
      const SegDesc& sd = P.segs[sg];
      printf("  bseg ops:");
      for (int o = sd.op_begin; o < sd.op_end; ++o) printf(" %s", names[op_code(P.ops[o].w0)]);
      printf("  (ipouts %d red %d)\n", sd.ip_count, sd.red_count);
    }
  }
  return 0;
}
}
