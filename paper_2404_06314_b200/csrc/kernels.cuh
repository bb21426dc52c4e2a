// sm_100a kernels for batched statevector forward + adjoint sweeps (complex128).
//
// Reference algorithm: vqckit/_kernels.py (apply_* 32-116, run_program
// 137-141, seed_bras 209-217, adjoint_reverse_pass 241-281). The reference
// sweeps the whole state once per gate; here a CTA keeps a tile (or the whole
// state) in shared memory, each thread holds 2^R amplitudes in registers and a
// program of ops (program.h) is applied per register segment. FP64 FMA is the
// bounding pipe: one rotation costs 4 DFMA per amplitude, one shared-memory
// round trip 32 B per amplitude (0.25 clk/amp/SM at 128 B/clk) — segments
// amortise the round trip over every gate on their R qubits.
#pragma once
#include <cuda_runtime.h>
#include <stdint.h>

#include <type_traits>

#include "program.h"

namespace vqc {

struct DevProgram {
  const Op* ops;
  const SegDesc* segs;
  const int32_t* seg_ip;
  const PassDesc* passes;
  const RotDesc* rots;
  const int32_t* term_offs;  // M + 1
  const uint32_t* t_smask;   // T
  const double* t_coeff;     // T (coeff * Re(phase); Z strings only)
  int n, k, R, NG, n_rot, M, n_pass;
  int64_t enc_off, enc_size;
};

enum PassFlags : uint32_t {
  F_INIT = 1u, F_LOAD_PSI = 2u, F_LOAD_FIN = 4u, F_LOAD_PHI = 8u, F_FWD = 16u,
  F_STORE_FIN = 32u, F_OBSERVE = 64u, F_SEED = 128u, F_BWD = 256u, F_STORE_PSI = 512u,
  F_STORE_PHI = 1024u,
};

struct RunArgs {
  const double* inputs;    // (B_total, enc_size), row b at inputs + b * enc_size
  const double* weights;   // flat parameter vector
  const double* upstream;  // (B_total, M) or nullptr
  int64_t b0;              // first global row handled by this launch
  int64_t nb;              // rows handled by this launch
  int K;                   // bras per row in the ip output (1 = VJP, M = Jacobian)
  int bra;                 // Jacobian bra for this launch (-1: VJP seed / all in-kernel)
  double* expect;          // (nb, M, n_tiles) rows relative to b0
  double* ip;              // (nb, K, NG, n_tiles) rows relative to b0
  double2* psi;            // HBM mode: (nb, 2^n) state buffers, row relative to b0
  double2* phi;
  double2* psi_fin;        // HBM Jacobian / smem Jacobian scratch
  int pass;
  uint32_t flags;
  int S;                   // samples per CTA (smem mode)
  int red_slots;           // reduction slots per buffer
  int jacobian;            // smem mode: loop over all M bras in-kernel
};

// ---------------------------------------------------------------------------
// shared-memory swizzle: 16-byte element l lives at l ^ fold3(l >> 3), i.e.
// bank group (p mod 8) = XOR of l's bits grouped by (bit position mod 3).
// Linear over GF(2), so swz(a ^ b) = swz(a) ^ swz(b).
__device__ __forceinline__ uint32_t swz(uint32_t l) {
  const uint32_t x = l >> 3;
  const uint32_t f = x ^ (x >> 3) ^ (x >> 6) ^ (x >> 9) ^ (x >> 12) ^ (x >> 15) ^ (x >> 18);
  return l ^ (f & 7u);
}

__host__ __device__ constexpr int ctz_const(int i) { return (i & 1) ? 0 : 1 + ctz_const(i >> 1); }

__device__ __forceinline__ double neg_if(double x, bool c) {
  const int hi = __double2hiint(x) ^ (c ? (int)0x80000000 : 0);
  return __hiloint2double(hi, __double2loint(x));
}

__device__ __forceinline__ double flat_val(const DevProgram& D, const RunArgs& A, int64_t b, int idx) {
  const int64_t e = (int64_t)idx - D.enc_off;
  return (e >= 0 && e < D.enc_size) ? A.inputs[b * D.enc_size + e] : A.weights[idx];
}

// (cos(angle/2), sin(angle/2)); angle = coeff * prod factors (_kernels.py:128-134)
__device__ __forceinline__ double2 rot_cs(const DevProgram& D, const RunArgs& A, int64_t b, int r) {
  const RotDesc rd = D.rots[r];
  double a = rd.coeff;
  for (int t = 0; t < rd.nf; ++t) a *= flat_val(D, A, b, rd.fidx[t]);
  double s, c;
  sincos(0.5 * a, &s, &c);
  return make_double2(c, s);
}

// ---------------------------------------------------------------------------
// register-level gate kernels; slot S is a compile-time register index bit
template <int R, typename F>
__device__ __forceinline__ void with_slot(uint32_t s, F&& f) {
  switch (s) {
    case 0: f(std::integral_constant<int, 0>{}); break;
    case 1: if constexpr (R > 1) f(std::integral_constant<int, 1>{}); break;
    case 2: if constexpr (R > 2) f(std::integral_constant<int, 2>{}); break;
    default: if constexpr (R > 3) f(std::integral_constant<int, 3>{}); break;
  }
}

// RX: a0' = c a0 - i s a1 ; a1' = -i s a0 + c a1   (_kernels.py:32-42)
template <int R, int S>
__device__ __forceinline__ void g_rx(double2 (&a)[1 << R], double c, double s) {
#pragma unroll
  for (int i = 0; i < (1 << R); ++i)
    if (!((i >> S) & 1)) {
      const int j = i | (1 << S);
      const double2 x = a[i], y = a[j];
      a[i] = make_double2(c * x.x + s * y.y, c * x.y - s * y.x);
      a[j] = make_double2(s * x.y + c * y.x, c * y.y - s * x.x);
    }
}

// RY: a0' = c a0 - s a1 ; a1' = s a0 + c a1   (_kernels.py:45-55)
template <int R, int S>
__device__ __forceinline__ void g_ry(double2 (&a)[1 << R], double c, double s) {
#pragma unroll
  for (int i = 0; i < (1 << R); ++i)
    if (!((i >> S) & 1)) {
      const int j = i | (1 << S);
      const double2 x = a[i], y = a[j];
      a[i] = make_double2(c * x.x - s * y.x, c * x.y - s * y.y);
      a[j] = make_double2(s * x.x + c * y.x, s * x.y + c * y.y);
    }
}

// H (_kernels.py:69-78)
template <int R, int S>
__device__ __forceinline__ void g_h(double2 (&a)[1 << R]) {
  const double inv = 0.70710678118654746;  // 1.0 / np.sqrt(2.0) as float64
#pragma unroll
  for (int i = 0; i < (1 << R); ++i)
    if (!((i >> S) & 1)) {
      const int j = i | (1 << S);
      const double2 x = a[i], y = a[j];
      a[i] = make_double2((x.x + y.x) * inv, (x.y + y.y) * inv);
      a[j] = make_double2((x.x - y.x) * inv, (x.y - y.y) * inv);
    }
}

// X: swap pairs (_kernels.py:81-88) — pure register renaming
template <int R, int S>
__device__ __forceinline__ void g_x(double2 (&a)[1 << R]) {
#pragma unroll
  for (int i = 0; i < (1 << R); ++i)
    if (!((i >> S) & 1)) {
      const int j = i | (1 << S);
      const double2 t = a[i];
      a[i] = a[j];
      a[j] = t;
    }
}

// CNOT with both qubits in registers (_kernels.py:91-100)
template <int R, int C, int T>
__device__ __forceinline__ void g_cnot_rr(double2 (&a)[1 << R]) {
  if constexpr (C != T) {
#pragma unroll
    for (int i = 0; i < (1 << R); ++i)
      if (((i >> C) & 1) && !((i >> T) & 1)) {
        const int j = i | (1 << T);
        const double2 t = a[i];
        a[i] = a[j];
        a[j] = t;
      }
  }
}

// CNOT with a per-thread constant control bit
template <int R, int T>
__device__ __forceinline__ void g_cnot_cr(double2 (&a)[1 << R], bool ctrl) {
#pragma unroll
  for (int i = 0; i < (1 << R); ++i)
    if (!((i >> T) & 1)) {
      const int j = i | (1 << T);
      const double2 x = a[i], y = a[j];
      a[i] = ctrl ? y : x;
      a[j] = ctrl ? x : y;
    }
}

// diagonal RZ phase: bit 0 -> e^{-i s}, bit 1 -> e^{+i s} (_kernels.py:58-66)
template <int R>
__device__ __forceinline__ void g_rz(double2 (&a)[1 << R], double c, double s, uint32_t slot_mask,
                                     bool cbit) {
#pragma unroll
  for (int i = 0; i < (1 << R); ++i) {
    const bool one = slot_mask ? ((i & slot_mask) != 0) : cbit;
    const double t = one ? s : -s;
    const double2 x = a[i];
    a[i] = make_double2(c * x.x - t * x.y, c * x.y + t * x.x);
  }
}

// CZ: negate where both bits are 1 (sign-bit flips, no FP64 work)
template <int R>
__device__ __forceinline__ void g_cz(double2 (&a)[1 << R], uint32_t mask, bool cond) {
#pragma unroll
  for (int i = 0; i < (1 << R); ++i) {
    const bool neg = cond && ((i & mask) == mask);
    a[i] = make_double2(neg_if(a[i].x, neg), neg_if(a[i].y, neg));
  }
}

// Im<phi|P|psi> partial sums over this thread's registers (_kernels.py:266-268)
template <int R, int S>
__device__ __forceinline__ double ip_x(const double2 (&p)[1 << R], const double2 (&f)[1 << R]) {
  double acc = 0.0;
#pragma unroll
  for (int i = 0; i < (1 << R); ++i)
    if (!((i >> S) & 1)) {
      const int j = i | (1 << S);
      acc += f[i].x * p[j].y - f[i].y * p[j].x;
      acc += f[j].x * p[i].y - f[j].y * p[i].x;
    }
  return acc;
}
template <int R, int S>
__device__ __forceinline__ double ip_y(const double2 (&p)[1 << R], const double2 (&f)[1 << R]) {
  double acc = 0.0;
#pragma unroll
  for (int i = 0; i < (1 << R); ++i)
    if (!((i >> S) & 1)) {
      const int j = i | (1 << S);
      acc -= f[i].x * p[j].x + f[i].y * p[j].y;
      acc += f[j].x * p[i].x + f[j].y * p[i].y;
    }
  return acc;
}
template <int R>
__device__ __forceinline__ double ip_z(const double2 (&p)[1 << R], const double2 (&f)[1 << R],
                                       uint32_t slot_mask, bool cbit) {
  double acc = 0.0;
#pragma unroll
  for (int i = 0; i < (1 << R); ++i) {
    const bool one = slot_mask ? ((i & slot_mask) != 0) : cbit;
    const double v = f[i].x * p[i].y - f[i].y * p[i].x;
    acc += one ? -v : v;
  }
  return acc;
}

// ---------------------------------------------------------------------------
// per-sample group reduction (TPS threads per sample, power of two)
struct Group {
  int tid, gi, sl, TPS, S, W;  // W = partials per sample (warps per sample, >= 1)
  __device__ __forceinline__ double reduce(double v) const {
    const int width = TPS < 32 ? TPS : 32;
    for (int off = width >> 1; off > 0; off >>= 1) v += __shfl_xor_sync(0xffffffffu, v, off);
    return v;
  }
  __device__ __forceinline__ bool leader() const { return (gi & 31) == 0; }
  __device__ __forceinline__ int red_index(int slot) const { return (slot * S + sl) * W + (gi >> 5); }
};

template <int R, bool DUAL>
__device__ __forceinline__ void exec_op(const Op op, double2 (&a)[1 << R], double2 (&f)[1 << R],
                                        uint32_t J0, const double2* s_cs, int rot_base,
                                        double* s_redbuf, const Group& grp) {
  const uint32_t w0 = op.w0;
  const uint32_t A = op_a(w0), Bq = op_b(w0);
  switch (op_code(w0)) {
    case OP_RX: {
      const double2 cs = s_cs[(int)op.param - rot_base];
      const double sn = op_adj(w0) ? -cs.y : cs.y;
      with_slot<R>(A & 7u, [&](auto SL) {
        g_rx<R, SL.value>(a, cs.x, sn);
        if constexpr (DUAL) g_rx<R, SL.value>(f, cs.x, sn);
      });
    } break;
    case OP_RY: {
      const double2 cs = s_cs[(int)op.param - rot_base];
      const double sn = op_adj(w0) ? -cs.y : cs.y;
      with_slot<R>(A & 7u, [&](auto SL) {
        g_ry<R, SL.value>(a, cs.x, sn);
        if constexpr (DUAL) g_ry<R, SL.value>(f, cs.x, sn);
      });
    } break;
    case OP_RZ: {
      const double2 cs = s_cs[(int)op.param - rot_base];
      const double sn = op_adj(w0) ? -cs.y : cs.y;
      const uint32_t m = (A & kSlotFlag) ? (1u << (A & 7u)) : 0u;
      const bool cb = (A & kSlotFlag) ? false : ((J0 >> A) & 1u);
      g_rz<R>(a, cs.x, sn, m, cb);
      if constexpr (DUAL) g_rz<R>(f, cs.x, sn, m, cb);
    } break;
    case OP_CNOT: {
      if (A & kSlotFlag) {
        with_slot<R>(A & 7u, [&](auto C) {
          with_slot<R>(Bq & 7u, [&](auto T) {
            g_cnot_rr<R, C.value, T.value>(a);
            if constexpr (DUAL) g_cnot_rr<R, C.value, T.value>(f);
          });
        });
      } else {
        const bool cb = (J0 >> A) & 1u;
        with_slot<R>(Bq & 7u, [&](auto T) {
          g_cnot_cr<R, T.value>(a, cb);
          if constexpr (DUAL) g_cnot_cr<R, T.value>(f, cb);
        });
      }
    } break;
    case OP_H:
      with_slot<R>(A & 7u, [&](auto SL) {
        g_h<R, SL.value>(a);
        if constexpr (DUAL) g_h<R, SL.value>(f);
      });
      break;
    case OP_X:
      with_slot<R>(A & 7u, [&](auto SL) {
        g_x<R, SL.value>(a);
        if constexpr (DUAL) g_x<R, SL.value>(f);
      });
      break;
    case OP_CZ: {
      uint32_t m = 0;
      bool cond = true;
      if (A & kSlotFlag) m |= 1u << (A & 7u); else cond = cond && ((J0 >> A) & 1u);
      if (Bq & kSlotFlag) m |= 1u << (Bq & 7u); else cond = cond && ((J0 >> Bq) & 1u);
      g_cz<R>(a, m, cond);
      if constexpr (DUAL) g_cz<R>(f, m, cond);
    } break;
    default:
      if constexpr (DUAL) {
        double v = 0.0;
        const uint32_t code = op_code(w0);
        if (code == OP_IPX) {
          with_slot<R>(A & 7u, [&](auto SL) { v = ip_x<R, SL.value>(a, f); });
        } else if (code == OP_IPY) {
          with_slot<R>(A & 7u, [&](auto SL) { v = ip_y<R, SL.value>(a, f); });
        } else {
          const uint32_t m = (A & kSlotFlag) ? (1u << (A & 7u)) : 0u;
          const bool cb = (A & kSlotFlag) ? false : ((J0 >> A) & 1u);
          v = ip_z<R>(a, f, m, cb);
        }
        v = grp.reduce(v);
        if (grp.leader()) s_redbuf[grp.red_index((int)op_ip(w0))] = v;
      }
      break;
  }
}

// Run segments [sb, se) on the tile(s) in shared memory. s_psi / s_phi point at
// this thread's sample block. IP results go to ip_out (relative row bl).
template <int R, bool DUAL>
__device__ void run_segments(const DevProgram& D, const RunArgs& A, int sb, int se, double2* s_psi,
                             double2* s_phi, const double2* s_cs, int rot_base, double* s_red,
                             int& red_buf, const Group& grp, uint32_t tile_base, int64_t bl0,
                             int64_t nb, int bra, int tile, int n_tiles) {
  constexpr int N = 1 << R;
  const int red_stride = A.red_slots * grp.S * grp.W;
  for (int sg = sb; sg < se; ++sg) {
    const SegDesc* sd = D.segs + sg;
    const int nthr = sd->nthr;
    uint32_t L0 = 0, J0 = tile_base;
    for (int i = 0; i < nthr; ++i)
      if ((grp.gi >> i) & 1) {
        L0 |= 1u << sd->thr_l[i];
        J0 |= 1u << sd->thr_g[i];
      }
    uint32_t ps[R];
#pragma unroll
    for (int s = 0; s < R; ++s) ps[s] = swz(1u << sd->reg_l[s]);
    uint32_t addr[N];
    addr[0] = swz(L0);
#pragma unroll
    for (int i = 1; i < N; ++i) addr[i] = addr[i & (i - 1)] ^ ps[ctz_const(i)];
    double2 a[N], f[N];
#pragma unroll
    for (int i = 0; i < N; ++i) {
      a[i] = s_psi[addr[i]];
      if constexpr (DUAL) f[i] = s_phi[addr[i]];
    }
    double* redbuf = s_red + red_buf * red_stride;
    const int ob = sd->op_begin, oe = sd->op_end;
    for (int o = ob; o < oe; ++o) exec_op<R, DUAL>(D.ops[o], a, f, J0, s_cs, rot_base, redbuf, grp);
#pragma unroll
    for (int i = 0; i < N; ++i) {
      s_psi[addr[i]] = a[i];
      if constexpr (DUAL) s_phi[addr[i]] = f[i];
    }
    __syncthreads();
    if constexpr (DUAL) {
      const int nip = sd->ip_count;
      if (nip > 0) {
        const int total = nip * grp.S;
        for (int idx = threadIdx.x; idx < total; idx += blockDim.x) {
          const int ipl = idx / grp.S, s_ = idx - ipl * grp.S;
          double v = 0.0;
          for (int w = 0; w < grp.W; ++w) v += redbuf[(ipl * grp.S + s_) * grp.W + w];
          const int64_t bl = bl0 + s_;
          if (bl < nb) {
            const int g = D.seg_ip[sd->ip_begin + ipl];
            A.ip[(((bl * A.K) + bra) * D.NG + g) * n_tiles + tile] = v;
          }
        }
        red_buf ^= 1;
      }
    }
  }
}

// global index of tile-local element l (pdep of l into the pass's local qubits)
__device__ __forceinline__ uint32_t local_to_global(const PassDesc& pd, uint32_t l, int k) {
  uint32_t j = 0;
  for (int p = 0; p < k; ++p) j |= ((l >> p) & 1u) << pd.local_q[p];
  return j;
}

// Z-string signs and weights for global index j over terms [lo, hi)
__device__ __forceinline__ double zweight(const DevProgram& D, uint32_t j, int lo, int hi) {
  double w = 0.0;
  for (int t = lo; t < hi; ++t) {
    const double c = D.t_coeff[t];
    w += (__popc(j & D.t_smask[t]) & 1) ? -c : c;
  }
  return w;
}

}  // namespace vqc
