// Host-side lowering of the reference's flat gate list (CompiledCircuit,
// circuit.py:168-216) into the pass/segment device program of program.h.
#pragma once
#include <stdint.h>

#include <string>
#include <vector>

#include "program.h"

namespace vqc {

struct GateIn {
  int kind = 0;
  int q0 = 0, q1 = 0;
  double coeff = 1.0;
  std::vector<int32_t> fidx;  // flat parameter indices (product factors)
};

struct ScheduleOptions {
  int tile_qubits = 11;      // k for HBM passes
  int reg_slots = 4;         // R
  int forced_low = 3;        // qubits 0..forced_low-1 always local in HBM passes
  int smem_max_qubits = kSmemMaxQubits;  // n above this streams tiles through HBM
  int segment_cost = 4;      // price of a segment boundary in interior-CNOT units
  int variants = 1;          // greedy restarts per group (refuse the first v new-qubit requests)
  bool fold_thread_targets = false;  // boundary CNOTs may target thread bits (JIT HBM plans)
  int max_pass_segments = 0;  // cut passes of more segments into several over the same local qubits (0: never)
  bool skip_dead_unapply = true;  // adjoint sweep: no un-apply for the first 1q operation on a qubit
  bool group_sync = false;   // plan thread-index bits for thread-group barriers (JIT HBM plans)
};

struct HostProgram {
  int n = 0, k = 0, R = 0;
  bool hbm = false;
  int n_rot = 0;   // rotations (angle table entries)
  int NG = 0;      // grad slots (rotations with a requested factor)
  int n_blk = 0, n_av = 0;
  int max_red_per_seg = 0;    // reduction slots
  int max_red_per_pass = 0;   // reduction slots of a pass's adjoint segments together
  bool group_sync = false;    // thread-index bits planned for thread-group barriers (ScheduleOptions)
  int jit_kernels = 3;        // HBM pass kernels to build: bit 0 forward, bit 1 adjoint (a plan with a
                              // separate forward schedule needs one kind from each program)
  // Z-string observables as compile-time constants of the JIT pass kernels
  // (term masks, coefficients, term_offs): the expectation / seed loops of the
  // observing pass unroll and their sign bits fold (empty: generic loops)
  std::vector<uint32_t> obs_mask;
  std::vector<double> obs_coeff;
  std::vector<int32_t> obs_offs;  // M + 1
  bool direct_io = false;     // JIT HBM passes: first / last segment of a sweep exchange registers with HBM directly
  bool warp_red = false;      // JIT HBM adjoint: per-warp reductions, gradients written at the end of the pass
  int max_ipout_per_seg = 0;
  int max_rot_per_pass = 0, max_blk_per_pass = 0, max_av_per_pass = 0;
  std::vector<PassDesc> passes;
  std::vector<SegDesc> segs;
  std::vector<Op> ops;
  std::vector<IpOut> ipouts;
  std::vector<RotDesc> rots;
  std::vector<BlockDesc> blocks;
  std::vector<MemberDesc> members;
  std::vector<DiagRun> diag;
  std::vector<int16_t> setids;  // kMaxR per block set
  int n_cols = 0;
  std::vector<int32_t> col_offs;  // n_cols + 1
  std::vector<ChainEntry> chain;
  // stats
  int n_fwd_ops = 0, n_bwd_ops = 0;
  int absorbed = 0;  // trailing gates folded into the observables (absorb_trailing_gates)
  bool adj_dual = false;  // HBM adjoint passes: both states per thread (JIT only) instead of thread pairs
  int precision = 0;      // 0 = complex128 states, 1 = complex64 (JIT kernels compiled with VQC_C64)
  bool checks = false;    // JIT units with device bounds checks (VQC_CHECKS)
  int pingpong = 0;       // HBM pass kernels: two tiles per CTA; 1 = arithmetic phases alternate,
                          // 2 = shared-memory phases alternate (VQC_PINGPONG, default off)
};

// Fold the circuit's trailing parameter-free gates that map Z strings to Z
// strings into the observables: <psi|G^dagger O G|psi> with O a weighted Z
// string stays a Z string (CNOT: Z_t -> Z_c Z_t; CZ: commutes; X: Z -> -Z).
// Pops them from `gates` (last gate first) and rewrites each term's sign mask
// / coefficient. Stops at the first gate that is not such a gate or has
// invalid qubits (left for build_program to report). Returns the count.
int absorb_trailing_gates(std::vector<GateIn>* gates, int n_qubits, std::vector<uint32_t>* zmask,
                          std::vector<double>* zcoeff);

// Returns "" on success, else an error message. wrt_col: flat index -> column or -1.
std::string build_program(const std::vector<GateIn>& gates, int n_qubits, int64_t total_params,
                          const std::vector<int64_t>& wrt_col, const ScheduleOptions& opt,
                          HostProgram* out);

}  // namespace vqc
