// 2x2 algebra for fused single-qubit blocks, shared by the kernels (per-sample
// prologue) and the CPU program checker.
//
// A block is a run of 1q gates M_0..M_{m-1} on one qubit (forward order);
// U = M_{m-1} ... M_0. In the adjoint sweep the reference evaluates, for each
// member rotation j, Im<phi_j|P_j|psi_j> at the state right after gate j
// (_kernels.py:258-268). With V_j = M_{m-1}...M_{j+1} and both states taken
// after the whole block, that is Im<phi|V_j P_j V_j^dagger|psi>; the
// conjugated generator is a real combination a_x X + a_y Y + a_z Z, so every
// member's inner product follows from the three Pauli inner products of the
// block: IP_j = a_j . (Im<phi|X|psi>, Im<phi|Y|psi>, Im<phi|Z|psi>).
#pragma once
#include "program.h"

namespace vqc {

struct C2 {
  double re, im;
};
struct M2 {
  C2 a, b, c, d;  // [[a, b], [c, d]]
};

VQC_HD inline C2 cmul(C2 x, C2 y) { return {x.re * y.re - x.im * y.im, x.re * y.im + x.im * y.re}; }
VQC_HD inline C2 cadd(C2 x, C2 y) { return {x.re + y.re, x.im + y.im}; }
VQC_HD inline C2 cconj(C2 x) { return {x.re, -x.im}; }

VQC_HD inline M2 mmul(const M2& x, const M2& y) {
  return {cadd(cmul(x.a, y.a), cmul(x.b, y.c)), cadd(cmul(x.a, y.b), cmul(x.b, y.d)),
          cadd(cmul(x.c, y.a), cmul(x.d, y.c)), cadd(cmul(x.c, y.b), cmul(x.d, y.d))};
}
VQC_HD inline M2 mdag(const M2& x) { return {cconj(x.a), cconj(x.c), cconj(x.b), cconj(x.d)}; }
VQC_HD inline M2 midentity() { return {{1, 0}, {0, 0}, {0, 0}, {1, 0}}; }

// gate matrices, U(theta) = exp(-i theta P / 2), (c, s) = (cos, sin)(theta/2)
// (_kernels.py:32-88)
VQC_HD inline M2 gate_m2(int kind, double c, double s) {
  switch (kind) {
    case G_RX: return {{c, 0}, {0, -s}, {0, -s}, {c, 0}};
    case G_RY: return {{c, 0}, {-s, 0}, {s, 0}, {c, 0}};
    case G_RZ: return {{c, -s}, {0, 0}, {0, 0}, {c, s}};
    case G_H: {
      const double inv = 0.70710678118654746;  // 1.0 / np.sqrt(2.0)
      return {{inv, 0}, {inv, 0}, {inv, 0}, {-inv, 0}};
    }
    default: return {{0, 0}, {1, 0}, {1, 0}, {0, 0}};  // X
  }
}

VQC_HD inline M2 pauli_m2(int axis) {
  switch (axis) {
    case 0: return {{0, 0}, {1, 0}, {1, 0}, {0, 0}};
    case 1: return {{0, 0}, {0, -1}, {0, 1}, {0, 0}};
    default: return {{1, 0}, {0, 0}, {0, 0}, {-1, 0}};
  }
}

// real Pauli coordinates of A = V P V^dagger (A Hermitian, traceless):
// A = ax X + ay Y + az Z  =>  ax = Re A01, ay = Im A10, az = (A00 - A11)/2
VQC_HD inline void pauli_vector(const M2& V, int axis, double out[3]) {
  const M2 A = mmul(mmul(V, pauli_m2(axis)), mdag(V));
  out[0] = A.b.re;
  out[1] = A.c.im;
  out[2] = 0.5 * (A.a.re - A.d.re);
}

// Walk members backwards: emits a_j for gradient members and returns U.
// cs(rot) -> (c, s); avec(slot, a[3]) receives the vectors.
template <class CS, class AV>
VQC_HD inline M2 block_unitary(const MemberDesc* mem, int m, CS&& cs, AV&& avec) {
  M2 V = midentity();
  for (int j = m - 1; j >= 0; --j) {
    const MemberDesc md = mem[j];
    double c = 1.0, s = 0.0;
    if (md.kind <= G_RZ) {
      const auto t = cs(md.rot);
      c = t.x;
      s = t.y;
      if (md.avec >= 0) {
        double a[3];
        pauli_vector(V, md.kind, a);
        avec(md.avec, a);
      }
    }
    V = mmul(V, gate_m2(md.kind, c, s));
  }
  return V;
}

}  // namespace vqc
