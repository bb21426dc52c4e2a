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
#ifndef __CUDACC_RTC__
#include <cuda_runtime.h>
#include <stdint.h>
#endif

#include "blockmath.h"
#include "program.h"

namespace vqc {

// compile-time integer (std::integral_constant without <type_traits>, which
// NVRTC cannot include)
template <int V>
struct IC {
  static constexpr int value = V;
};

// State element type. complex128 by default; a plan created with precision
// 1 (complex64) is JIT-compiled with VQC_C64 defined: states, registers and
// gate arithmetic are single precision, while angles, fused-block matrices,
// inner-product reductions, expectations and gradients stay float64 (the
// north star's optional complex64 mode, 1e-5 against the reference).
#ifdef VQC_C64
typedef float real_t;
typedef float2 cplx_t;
__device__ __forceinline__ cplx_t mk_c(real_t a, real_t b) { return make_float2(a, b); }
#else
typedef double real_t;
typedef double2 cplx_t;
__device__ __forceinline__ cplx_t mk_c(real_t a, real_t b) { return make_double2(a, b); }
#endif

// CTA view. Plain kernels treat the CTA as one thread group. HBM pass
// kernels built with VQC_PINGPONG run two half-CTA groups on two tiles and
// order their segment phases with named barriers (seg_begin ends in
// phase_a(), seg_end starts with phase_b()):
//   VQC_PINGPONG == 1: the register phases (gate arithmetic) alternate
//     between the groups;
//   VQC_PINGPONG == 2: the shared-memory phases (register store, reduction,
//     next register load) alternate, arithmetic may overlap.
// vtid / vdim / vsync are the group's thread index, size and barrier.
#ifdef VQC_PINGPONG
__device__ __forceinline__ unsigned cta_group() { return threadIdx.x >= (blockDim.x >> 1) ? 1u : 0u; }
__device__ __forceinline__ unsigned vdim() { return blockDim.x >> 1; }
__device__ __forceinline__ unsigned vtid() { return threadIdx.x - cta_group() * (blockDim.x >> 1); }
__device__ __forceinline__ void vsync() {
  asm volatile("bar.sync %0, %1;" ::"r"(1u + cta_group()), "r"(blockDim.x >> 1) : "memory");
}
// barrier 3 + g: group g waits there for the other group's hand-over
__device__ __forceinline__ void turn_wait() {
  asm volatile("bar.sync %0, %1;" ::"r"(3u + cta_group()), "r"(blockDim.x) : "memory");
}
__device__ __forceinline__ void turn_pass() {
  asm volatile("bar.arrive %0, %1;" ::"r"(4u - cta_group()), "r"(blockDim.x) : "memory");
}
#if VQC_PINGPONG == 1
__device__ __forceinline__ void phase_a() { turn_wait(); }
__device__ __forceinline__ void phase_b() { turn_pass(); }
// group 0 takes the first turn; it also consumes group 1's last hand-over
__device__ __forceinline__ void turn_init() {
  if (cta_group() == 1u) turn_pass();
}
__device__ __forceinline__ void turn_fini() {
  if (cta_group() == 0u) turn_wait();
}
#else
__device__ __forceinline__ void phase_a() { turn_pass(); }
__device__ __forceinline__ void phase_b() { turn_wait(); }
// group 1 starts after group 0's first register load; group 0 hands over
// once more at the end for group 1's last shared-memory phase
__device__ __forceinline__ void turn_init() {
  if (cta_group() == 1u) turn_wait();
}
__device__ __forceinline__ void turn_fini() {
  if (cta_group() == 0u) turn_pass();
}
#endif
constexpr int kCtaGroups = 2;
#else
__device__ __forceinline__ unsigned cta_group() { return 0u; }
__device__ __forceinline__ unsigned vdim() { return blockDim.x; }
__device__ __forceinline__ unsigned vtid() { return threadIdx.x; }
__device__ __forceinline__ void vsync() { __syncthreads(); }
__device__ __forceinline__ void phase_a() {}
__device__ __forceinline__ void phase_b() {}
__device__ __forceinline__ void turn_init() {}
__device__ __forceinline__ void turn_fini() {}
constexpr int kCtaGroups = 1;
#endif

struct DevProgram {
  const Op* ops;
  const SegDesc* segs;
  const PassDesc* passes;
  const RotDesc* rots;
  const IpOut* ipouts;
  const BlockDesc* blocks;
  const MemberDesc* members;
  const DiagRun* diag;
  const int16_t* setids;
  const ThrEntry* thr_tab;
  const int32_t* term_offs;  // M + 1
  const uint32_t* t_smask;   // T sign masks (Y/Z letters)
  const uint32_t* t_xmask;   // T flip masks (X/Y letters; nonzero only when has_xy)
  const int32_t* t_phase;    // T powers of i
  const double* t_coeff;     // T
  const int32_t* t_obs;      // T observable index of each term
  int has_xy;                // any X/Y string (on-chip states only)
  int n, k, R, NG, n_rot, M, n_pass;
  int n_blk, n_av, max_rot_pass, max_blk_pass, max_av_pass;
  int T;  // observable terms
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
  cplx_t* psi;             // HBM mode: (nb, 2^n) state buffers, row relative to b0
  cplx_t* phi;
  cplx_t* psi_fin;        // HBM Jacobian / smem Jacobian scratch
  int pass;
  uint32_t flags;
  int S;                   // samples per CTA (smem mode)
  int red_slots;           // reduction slots per buffer
  int jacobian;            // smem mode: loop over all M bras in-kernel
  unsigned long long* dbg; // VQC_DEBUG_TIMING: per-phase clock64 totals (thread 0 of each CTA)
  unsigned int* check;     // VQC_CHECKS: bounds-check failure bits (VQC_DEVICE_CHECKS kernels)
  const double* tables;    // HBM mode: per-sample tables from k_tables (rows relative to b0)
  int64_t table_stride;    // doubles per sample
};

// Device bounds checks (plans created with VQC_CHECKS=1 compile their JIT
// units with VQC_DEVICE_CHECKS): every shared-memory tile address of the
// register loads / stores and the observe step, and every global state index
// of the tile loads / stores, is range-checked; a failure ORs a bit into
// A.check and the host call fails. (compute-sanitizer is closed on this
// pool; these checks plus the bitwise run / chunking invariance tests stand
// in for memcheck / racecheck.)
enum { CHK_SEG_LOAD = 1u, CHK_SEG_STORE = 2u, CHK_TILE_GLOBAL = 4u, CHK_TILE_SMEM = 8u, CHK_OBSERVE = 16u,
       CHK_IP_OUT = 32u };
#ifdef VQC_DEVICE_CHECKS
#define VQC_CHECK(A, cond, bit) \
  do {                          \
    if (!(cond)) atomicOr((A).check, (unsigned)(bit)); \
  } while (0)
#else
#define VQC_CHECK(A, cond, bit) \
  do {                          \
  } while (0)
#endif

// phase timing (debug only): dbg[slot] += clock64 delta, slots fixed below
enum { DBG_PROLOGUE = 0, DBG_FWD = 1, DBG_OBSERVE = 2, DBG_BWD = 3, DBG_STORE = 4, DBG_SEG_LOAD = 5,
       DBG_SEG_OPS = 6, DBG_SEG_STORE = 7, DBG_SEG_FINAL = 8, DBG_CTAS = 9, DBG_N = 10 };
__device__ __forceinline__ void dbg_add(const RunArgs& A, int slot, long long& t) {
  if (A.dbg != nullptr && vtid() == 0) {
    const long long now = clock64();
    atomicAdd(A.dbg + slot, (unsigned long long)(now - t));
    t = now;
  }
}

// ---------------------------------------------------------------------------
// shared-memory swizzle: 16-byte element l lives at l ^ fold3(l >> 3), i.e.
// bank group (p mod 8) = XOR of l's bits grouped by (bit position mod 3).
// Linear over GF(2), so swz(a ^ b) = swz(a) ^ swz(b).
__device__ __forceinline__ uint32_t swz(uint32_t l) { return swz_index(l); }

__host__ __device__ constexpr int ctz_const(int i) { return (i & 1) ? 0 : 1 + ctz_const(i >> 1); }
__host__ __device__ constexpr int popc_const(int i) { return i == 0 ? 0 : (i & 1) + popc_const(i >> 1); }

__device__ __forceinline__ double neg_if(double x, bool c) {
  const int hi = __double2hiint(x) ^ (c ? (int)0x80000000 : 0);
  return __hiloint2double(hi, __double2loint(x));
}
__device__ __forceinline__ float neg_if(float x, bool c) {
  return __int_as_float(__float_as_int(x) ^ (c ? (int)0x80000000 : 0));
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
    case 0: f(IC<0>{}); break;
    case 1: if constexpr (R > 1) f(IC<1>{}); break;
    case 2: if constexpr (R > 2) f(IC<2>{}); break;
    case 3: if constexpr (R > 3) f(IC<3>{}); break;
    default: if constexpr (R > 4) f(IC<4>{}); break;
  }
}

// RX: a0' = c a0 - i s a1 ; a1' = -i s a0 + c a1   (_kernels.py:32-42)
template <int R, int S>
__device__ __forceinline__ void g_rx(cplx_t (&a)[1 << R], real_t c, real_t s) {
#pragma unroll
  for (int i = 0; i < (1 << R); ++i)
    if (!((i >> S) & 1)) {
      const int j = i | (1 << S);
      const cplx_t x = a[i], y = a[j];
      a[i] = mk_c(c * x.x + s * y.y, c * x.y - s * y.x);
      a[j] = mk_c(s * x.y + c * y.x, c * y.y - s * x.x);
    }
}

// RY: a0' = c a0 - s a1 ; a1' = s a0 + c a1   (_kernels.py:45-55)
template <int R, int S>
__device__ __forceinline__ void g_ry(cplx_t (&a)[1 << R], real_t c, real_t s) {
#pragma unroll
  for (int i = 0; i < (1 << R); ++i)
    if (!((i >> S) & 1)) {
      const int j = i | (1 << S);
      const cplx_t x = a[i], y = a[j];
      a[i] = mk_c(c * x.x - s * y.x, c * x.y - s * y.y);
      a[j] = mk_c(s * x.x + c * y.x, s * x.y + c * y.y);
    }
}

// H (_kernels.py:69-78)
template <int R, int S>
__device__ __forceinline__ void g_h(cplx_t (&a)[1 << R]) {
  const real_t inv = (real_t)0.70710678118654746;  // 1.0 / np.sqrt(2.0) as float64
#pragma unroll
  for (int i = 0; i < (1 << R); ++i)
    if (!((i >> S) & 1)) {
      const int j = i | (1 << S);
      const cplx_t x = a[i], y = a[j];
      a[i] = mk_c((x.x + y.x) * inv, (x.y + y.y) * inv);
      a[j] = mk_c((x.x - y.x) * inv, (x.y - y.y) * inv);
    }
}

// X: swap pairs (_kernels.py:81-88) — pure register renaming
template <int R, int S>
__device__ __forceinline__ void g_x(cplx_t (&a)[1 << R]) {
#pragma unroll
  for (int i = 0; i < (1 << R); ++i)
    if (!((i >> S) & 1)) {
      const int j = i | (1 << S);
      const cplx_t t = a[i];
      a[i] = a[j];
      a[j] = t;
    }
}

// CNOT with both qubits in registers (_kernels.py:91-100)
template <int R, int C, int T>
__device__ __forceinline__ void g_cnot_rr(cplx_t (&a)[1 << R]) {
  if constexpr (C != T) {
#pragma unroll
    for (int i = 0; i < (1 << R); ++i)
      if (((i >> C) & 1) && !((i >> T) & 1)) {
        const int j = i | (1 << T);
        const cplx_t t = a[i];
        a[i] = a[j];
        a[j] = t;
      }
  }
}

// CNOT with a per-thread constant control bit
template <int R, int T>
__device__ __forceinline__ void g_cnot_cr(cplx_t (&a)[1 << R], bool ctrl) {
#pragma unroll
  for (int i = 0; i < (1 << R); ++i)
    if (!((i >> T) & 1)) {
      const int j = i | (1 << T);
      const cplx_t x = a[i], y = a[j];
      a[i] = ctrl ? y : x;
      a[j] = ctrl ? x : y;
    }
}

// diagonal RZ phase: bit 0 -> e^{-i s}, bit 1 -> e^{+i s} (_kernels.py:58-66)
template <int R>
__device__ __forceinline__ void g_rz(cplx_t (&a)[1 << R], real_t c, real_t s, uint32_t slot_mask,
                                     bool cbit) {
#pragma unroll
  for (int i = 0; i < (1 << R); ++i) {
    const bool one = slot_mask ? ((i & slot_mask) != 0) : cbit;
    const real_t t = one ? s : -s;
    const cplx_t x = a[i];
    a[i] = mk_c(c * x.x - t * x.y, c * x.y + t * x.x);
  }
}

// CZ: negate where both bits are 1 (sign-bit flips, no FP64 work)
template <int R>
__device__ __forceinline__ void g_cz(cplx_t (&a)[1 << R], uint32_t mask, bool cond) {
#pragma unroll
  for (int i = 0; i < (1 << R); ++i) {
    const bool neg = cond && ((i & mask) == mask);
    a[i] = mk_c(neg_if(a[i].x, neg), neg_if(a[i].y, neg));
  }
}

// ---------------------------------------------------------------------------
// Im<phi|P|psi> partial sums (_kernels.py:266-268). P(i), F(i) return element
// i of psi / phi (registers, or the partner thread's copy in shared memory).
// PART = -1 sums every pair; PART = 0/1 sums the half of the pairs whose
// balance bit (the lowest register bit other than S) equals PART, so the two
// threads of a split (psi, phi) pair share the work.
template <int R, int S, int PART>
__device__ __forceinline__ constexpr bool take_pair(int i) {
  if constexpr (PART < 0 || R < 2) {
    return PART <= 0;
  } else {
    constexpr int BB = S == 0 ? 1 : 0;
    return ((i >> BB) & 1) == PART;
  }
}

template <int R, int S, int PART, class P, class F>
__device__ __forceinline__ double ip_x(P&& p, F&& f) {
  real_t acc = 0;
#pragma unroll
  for (int i = 0; i < (1 << R); ++i)
    if (!((i >> S) & 1) && take_pair<R, S, PART>(i)) {
      const int j = i | (1 << S);
      const cplx_t f0 = f(i), f1 = f(j), p0 = p(i), p1 = p(j);
      acc += f0.x * p1.y - f0.y * p1.x;
      acc += f1.x * p0.y - f1.y * p0.x;
    }
  return (double)acc;
}
template <int R, int S, int PART, class P, class F>
__device__ __forceinline__ double ip_y(P&& p, F&& f) {
  real_t acc = 0;
#pragma unroll
  for (int i = 0; i < (1 << R); ++i)
    if (!((i >> S) & 1) && take_pair<R, S, PART>(i)) {
      const int j = i | (1 << S);
      const cplx_t f0 = f(i), f1 = f(j), p0 = p(i), p1 = p(j);
      acc -= f0.x * p1.x + f0.y * p1.y;
      acc += f1.x * p0.x + f1.y * p0.y;
    }
  return (double)acc;
}
// Z on a register slot (mask = 1 << slot) or a per-thread constant bit (mask 0)
template <int R, int PART, class P, class F>
__device__ __forceinline__ double ip_z(P&& p, F&& f, uint32_t slot_mask, bool cbit) {
  real_t acc = 0;
#pragma unroll
  for (int i = 0; i < (1 << R); ++i) {
    if (PART >= 0 && R >= 1 && (i & 1) != PART) continue;
    const bool one = slot_mask ? ((i & slot_mask) != 0) : cbit;
    const cplx_t fi = f(i), pi = p(i);
    const real_t v = fi.x * pi.y - fi.y * pi.x;
    acc += one ? -v : v;
  }
  return (double)acc;
}
// All three Pauli inner products of slot S in one sweep, as explicit FMA
// chains (12 DFMA per pair) split over two accumulator sets (alternate pairs)
// so the dependent chains are half as long.
template <int R, int S, int PART, class P, class F>
__device__ __forceinline__ void ip_xyz(P&& p, F&& f, double& ix, double& iy, double& iz) {
  real_t ax[2] = {0, 0}, ay[2] = {0, 0}, az[2] = {0, 0};
  int k = 0;
#pragma unroll
  for (int i = 0; i < (1 << R); ++i)
    if (!((i >> S) & 1) && take_pair<R, S, PART>(i)) {
      const int j = i | (1 << S);
      const int c = k & 1;
      ++k;
      const cplx_t f0 = f(i), f1 = f(j), p0 = p(i), p1 = p(j);
      ax[c] = fma(f0.x, p1.y, ax[c]);
      ax[c] = fma(-f0.y, p1.x, ax[c]);
      ax[c] = fma(f1.x, p0.y, ax[c]);
      ax[c] = fma(-f1.y, p0.x, ax[c]);
      ay[c] = fma(-f0.x, p1.x, ay[c]);
      ay[c] = fma(-f0.y, p1.y, ay[c]);
      ay[c] = fma(f1.x, p0.x, ay[c]);
      ay[c] = fma(f1.y, p0.y, ay[c]);
      az[c] = fma(f0.x, p0.y, az[c]);
      az[c] = fma(-f0.y, p0.x, az[c]);
      az[c] = fma(-f1.x, p1.y, az[c]);
      az[c] = fma(f1.y, p1.x, az[c]);
    }
  ix += (double)(ax[0] + ax[1]);   // per-thread partials widen to float64
  iy += (double)(ay[0] + ay[1]);
  iz += (double)(az[0] + az[1]);
}

// ---------------------------------------------------------------------------
// Threads of one sample. Forward / dual: TPS threads, one register group each.
// Split adjoint: 2*TPS threads, role 0 holds psi and role 1 phi of group gi.
struct Group {
  int tid, gi, sl, TPS, S, W;  // W = partials per sample (warps per sample, >= 1)
  int role = 0, TT = 0;        // TT = threads per sample
  __device__ __forceinline__ double reduce(double v) const {
    const int width = TT < 32 ? TT : 32;
    const unsigned mask = vdim() >= 32 ? 0xffffffffu : ((1u << vdim()) - 1u);
    for (int off = width >> 1; off > 0; off >>= 1) v += __shfl_xor_sync(mask, v, off);
    return v;
  }
  __device__ __forceinline__ int lane_in_sample() const { return role * TPS + gi; }
  __device__ __forceinline__ bool leader() const { return (lane_in_sample() & 31) == 0; }
  __device__ __forceinline__ int red_index(int slot) const {
    return (slot * S + sl) * W + (lane_in_sample() >> 5);
  }
};

// general 2x2 on slot S: a0' = u00 a0 + u01 a1 ; a1' = u10 a0 + u11 a1
template <int R, int S>
__device__ __forceinline__ void g_u2(cplx_t (&a)[1 << R], const cplx_t u00, const cplx_t u01,
                                     const cplx_t u10, const cplx_t u11) {
#pragma unroll
  for (int i = 0; i < (1 << R); ++i)
    if (!((i >> S) & 1)) {
      const int j = i | (1 << S);
      const cplx_t x = a[i], y = a[j];
      a[i] = mk_c(u00.x * x.x - u00.y * x.y + u01.x * y.x - u01.y * y.y,
                          u00.x * x.y + u00.y * x.x + u01.x * y.y + u01.y * y.x);
      a[j] = mk_c(u10.x * x.x - u10.y * x.y + u11.x * y.x - u11.y * y.y,
                          u10.x * x.y + u10.y * x.x + u11.x * y.y + u11.y * y.x);
    }
}

// fused CZ run (program.h DiagRun): per-register sign from a quadratic form
template <int R>
__device__ __forceinline__ void g_czrun(cplx_t (&a)[1 << R], uint32_t qreg, uint32_t m, uint32_t qc) {
#pragma unroll
  for (int i = 0; i < (1 << R); ++i) {
    const bool neg = ((qc ^ (qreg >> i) ^ (uint32_t)__popc((uint32_t)i & m)) & 1u) != 0u;
    a[i] = mk_c(neg_if(a[i].x, neg), neg_if(a[i].y, neg));
  }
}

// this thread's partial inner product for reduction slot `slot` (reduced over
// the sample's threads at the end of the segment, in a fixed order)
__device__ __forceinline__ void put_partial(double* redbuf, int slot, double v) {
  redbuf[slot * vdim() + vtid()] = v;
}
// lagged JIT reductions: lanes 2i, 2i+1 add their partials first and one half
// row (blockDim/2 entries) per slot is written, so two segments' partial
// buffers fit in the space of one (jred_phase1)
template <bool PAIR>
__device__ __forceinline__ void put_part(double* redbuf, int slot, double v) {
  if constexpr (PAIR) {
    v += __shfl_xor_sync(0xffffffffu, v, 1);
    if (!(vtid() & 1u)) redbuf[slot * (vdim() >> 1) + (vtid() >> 1)] = v;
  } else {
    put_partial(redbuf, slot, v);
  }
}

// compile-time slot from an unrolled loop index (no branch after unrolling)
template <int R, typename F>
__device__ __forceinline__ void with_const_slot(int s, F&& f) {
  if (s == 0) f(IC<0>{});
  if constexpr (R > 1) if (s == 1) f(IC<1>{});
  if constexpr (R > 2) if (s == 2) f(IC<2>{});
  if constexpr (R > 3) if (s == 3) f(IC<3>{});
  if constexpr (R > 4) if (s == 4) f(IC<4>{});
}

// per-sample parameter tables in shared memory
struct SampleTables {
  const double2* cs;  // (cos, sin) of theta/2 per rotation (relative to rot_base)
  const double2* u;   // 4 entries per fused block (relative to blk_base)
  int rot_base, blk_base;
};

enum { MODE_FWD = 0, MODE_DUAL = 1, MODE_SPLIT = 2 };

// Register-tile context of the current segment: the state registers live in
// a[] (and f[] in dual mode); in split mode the partner's copy of element i
// is in shared memory at addr(i) (the segment's load map).
template <int R>
struct SegCtx {
  uint32_t J0;
  uint32_t lp0;
  uint32_t lc[R];
  cplx_t* own;
  const cplx_t* partner;
  __device__ __forceinline__ uint32_t addr(int i) const {
    uint32_t ad = lp0;
#pragma unroll
    for (int s = 0; s < R; ++s)
      if ((i >> s) & 1) ad ^= lc[s];
    return ad;
  }
};

// Run one inner-product op: dual reads both register sets; split computes
// half of the pairs from its own registers and the partner's shared copy.
template <int R, int MODE, class K>
__device__ __forceinline__ void ip_dispatch(const SegCtx<R>& C, const cplx_t (&a)[1 << R],
                                            const cplx_t (&f)[1 << R], int role, K&& kernel) {
  auto ra = [&](int i) { return a[i]; };
  if constexpr (MODE == MODE_DUAL) {
    auto rf = [&](int i) { return f[i]; };
    kernel(IC<-1>{}, ra, rf);
  } else {
    // recompute partner addresses here (pinned by the empty asm) instead of
    // letting the compiler keep 2^R loop-invariant addresses live
    uint32_t base = C.lp0;
    asm volatile("" : "+r"(base));
    auto sm = [&](int i) {
      uint32_t ad = base;
#pragma unroll
      for (int s = 0; s < R; ++s)
        if ((i >> s) & 1) ad ^= C.lc[s];
      return C.partner[ad];
    };
    if (role == 0) kernel(IC<0>{}, ra, sm);
    else kernel(IC<1>{}, sm, ra);
  }
}

// ---------------------------------------------------------------------------
// Ops with compile-time operands. The interpreter (exec_op) dispatches to
// these through with_slot; the per-plan JIT (jit.cpp) emits direct calls, so
// both paths run the same arithmetic in the same order.
template <int R>
using Regs = cplx_t[1 << R];

template <int R, int MODE, int KIND, int S, bool ADJ>
__device__ __forceinline__ void jop_rot(Regs<R>& a, Regs<R>& f, const SampleTables& T, int r) {
  const double2 cs = T.cs[r];
  const real_t c = (real_t)cs.x, sn = (real_t)(ADJ ? -cs.y : cs.y);
  if constexpr (KIND == G_RX) {
    g_rx<R, S>(a, c, sn);
    if constexpr (MODE == MODE_DUAL) g_rx<R, S>(f, c, sn);
  } else {
    g_ry<R, S>(a, c, sn);
    if constexpr (MODE == MODE_DUAL) g_ry<R, S>(f, c, sn);
  }
}

// RZ on register slot mask m (power of two), or on a thread/tile bit cb (m = 0)
template <int R, int MODE, bool ADJ>
__device__ __forceinline__ void jop_rz(Regs<R>& a, Regs<R>& f, const SampleTables& T, int r, uint32_t m, bool cb) {
  const double2 cs = T.cs[r];
  const real_t c = (real_t)cs.x, sn = (real_t)(ADJ ? -cs.y : cs.y);
  g_rz<R>(a, c, sn, m, cb);
  if constexpr (MODE == MODE_DUAL) g_rz<R>(f, c, sn, m, cb);
}

// fused block (relative id blk) on slot S; ADJ applies U^dagger
template <int R, int MODE, int S, bool ADJ>
__device__ __forceinline__ void jop_u2(Regs<R>& a, Regs<R>& f, const SampleTables& T, int blk) {
  const double2* u = T.u + 4 * blk;
  cplx_t u00 = mk_c((real_t)u[0].x, (real_t)u[0].y), u01 = mk_c((real_t)u[1].x, (real_t)u[1].y),
         u10 = mk_c((real_t)u[2].x, (real_t)u[2].y), u11 = mk_c((real_t)u[3].x, (real_t)u[3].y);
  if constexpr (ADJ) {
    const cplx_t t = u01;
    u00.y = -u00.y;
    u11.y = -u11.y;
    u01 = mk_c(u10.x, -u10.y);
    u10 = mk_c(t.x, -t.y);
  }
  g_u2<R, S>(a, u00, u01, u10, u11);
  if constexpr (MODE == MODE_DUAL) g_u2<R, S>(f, u00, u01, u10, u11);
}

template <int R, int MODE, int C, int T>
__device__ __forceinline__ void jop_cnot_rr(Regs<R>& a, Regs<R>& f) {
  g_cnot_rr<R, C, T>(a);
  if constexpr (MODE == MODE_DUAL) g_cnot_rr<R, C, T>(f);
}
template <int R, int MODE, int T>
__device__ __forceinline__ void jop_cnot_cr(Regs<R>& a, Regs<R>& f, bool cb) {
  g_cnot_cr<R, T>(a, cb);
  if constexpr (MODE == MODE_DUAL) g_cnot_cr<R, T>(f, cb);
}
template <int R, int MODE, int S>
__device__ __forceinline__ void jop_h(Regs<R>& a, Regs<R>& f) {
  g_h<R, S>(a);
  if constexpr (MODE == MODE_DUAL) g_h<R, S>(f);
}
template <int R, int MODE, int S>
__device__ __forceinline__ void jop_x(Regs<R>& a, Regs<R>& f) {
  g_x<R, S>(a);
  if constexpr (MODE == MODE_DUAL) g_x<R, S>(f);
}
template <int R, int MODE>
__device__ __forceinline__ void jop_cz(Regs<R>& a, Regs<R>& f, uint32_t m, bool cond) {
  g_cz<R>(a, m, cond);
  if constexpr (MODE == MODE_DUAL) g_cz<R>(f, m, cond);
}
template <int R, int MODE>
__device__ __forceinline__ void jop_czrun(Regs<R>& a, Regs<R>& f, const DiagRun* dr, uint32_t J0) {
  uint32_t qc = 0, m = 0;
  for (uint32_t rest = J0; rest != 0; rest &= rest - 1) qc ^= (uint32_t)__popc(J0 & dr->upper[__ffs(rest) - 1]);
#pragma unroll
  for (int s = 0; s < R; ++s) m |= ((uint32_t)__popc(J0 & dr->part[s]) & 1u) << s;
  const uint32_t qreg = dr->qreg;
  g_czrun<R>(a, qreg, m, qc);
  if constexpr (MODE == MODE_DUAL) g_czrun<R>(f, qreg, m, qc);
}

// fused CZ run with the quadratic form already evaluated (JIT: the run's
// masks are compile-time constants, no descriptor loads)
template <int R, int MODE>
__device__ __forceinline__ void jop_czsign(Regs<R>& a, Regs<R>& f, uint32_t qreg, uint32_t m, uint32_t qc) {
  g_czrun<R>(a, qreg, m, qc);
  if constexpr (MODE == MODE_DUAL) g_czrun<R>(f, qreg, m, qc);
}

// inner products: partial sums into reduction slots (adjoint modes only)
template <int R, int MODE, int S, bool PAIR = false>
__device__ __forceinline__ void jop_ip3(const SegCtx<R>& C, const Regs<R>& a, const Regs<R>& f, int role,
                                        double* s_red, int r0) {
  if constexpr (MODE != MODE_FWD) {
    double ix = 0.0, iy = 0.0, iz = 0.0;
    ip_dispatch<R, MODE>(C, a, f, role, [&](auto PART, auto&& p, auto&& q) {
      ip_xyz<R, S, PART.value>(p, q, ix, iy, iz);
    });
    put_part<PAIR>(s_red, r0, ix);
    put_part<PAIR>(s_red, r0 + 1, iy);
    put_part<PAIR>(s_red, r0 + 2, iz);
  }
}
// KIND: 0 = X, 1 = Y on slot S
template <int R, int MODE, int KIND, int S, bool PAIR = false>
__device__ __forceinline__ void jop_ipxy(const SegCtx<R>& C, const Regs<R>& a, const Regs<R>& f, int role,
                                         double* s_red, int r) {
  if constexpr (MODE != MODE_FWD) {
    double v = 0.0;
    ip_dispatch<R, MODE>(C, a, f, role, [&](auto PART, auto&& p, auto&& q) {
      if constexpr (KIND == 0) v = ip_x<R, S, PART.value>(p, q);
      else v = ip_y<R, S, PART.value>(p, q);
    });
    put_part<PAIR>(s_red, r, v);
  }
}
template <int R, int MODE, bool PAIR = false>
__device__ __forceinline__ void jop_ipz(const SegCtx<R>& C, const Regs<R>& a, const Regs<R>& f, int role,
                                        double* s_red, int r, uint32_t m, bool cb) {
  if constexpr (MODE != MODE_FWD) {
    double v = 0.0;
    ip_dispatch<R, MODE>(C, a, f, role, [&](auto PART, auto&& p, auto&& q) {
      v = ip_z<R, PART.value>(p, q, m, cb);
    });
    put_part<PAIR>(s_red, r, v);
  }
}

// Fused blocks on the register slots of compile-time MASK (one op of the
// program): straight-line code, so the block results only need to reach the
// loop-carried registers once per set instead of once per block.
template <int R, int MODE, bool ADJ, int MASK>
__device__ __forceinline__ void jop_u2set(Regs<R>& a, Regs<R>& f, const SampleTables& T, const int16_t* ids) {
  if constexpr ((MASK & 1) != 0) jop_u2<R, MODE, 0, ADJ>(a, f, T, ids[0]);
  if constexpr (R > 1 && (MASK & 2) != 0) jop_u2<R, MODE, 1, ADJ>(a, f, T, ids[1]);
  if constexpr (R > 2 && (MASK & 4) != 0) jop_u2<R, MODE, 2, ADJ>(a, f, T, ids[2]);
  if constexpr (R > 3 && (MASK & 8) != 0) jop_u2<R, MODE, 3, ADJ>(a, f, T, ids[3]);
  if constexpr (R > 4 && (MASK & 16) != 0) jop_u2<R, MODE, 4, ADJ>(a, f, T, ids[4]);
}

// Im<phi|X,Y,Z|psi> on every slot of MASK; reduction slots r0, r0 + 3, ... in
// slot order. The split-role branch is taken once for the whole set.
template <int R, int PART, int MASK, bool PAIR, class P, class F>
__device__ __forceinline__ void ip3set_part(P&& p, F&& q, double* s_red, int r0) {
  auto one = [&](auto SL, int r) {
    if constexpr (SL.value < R && ((MASK >> SL.value) & 1) != 0) {
      double ix = 0.0, iy = 0.0, iz = 0.0;
      ip_xyz<R, SL.value, PART>(p, q, ix, iy, iz);
      put_part<PAIR>(s_red, r, ix);
      put_part<PAIR>(s_red, r + 1, iy);
      put_part<PAIR>(s_red, r + 2, iz);
    }
  };
  one(IC<0>{}, r0);
  one(IC<1>{}, r0 + 3 * popc_const(MASK & 1));
  one(IC<2>{}, r0 + 3 * popc_const(MASK & 3));
  one(IC<3>{}, r0 + 3 * popc_const(MASK & 7));
  one(IC<4>{}, r0 + 3 * popc_const(MASK & 15));
}
template <int R, int MODE, int MASK, bool PAIR = false>
__device__ __forceinline__ void jop_ip3set(const SegCtx<R>& C, const Regs<R>& a, const Regs<R>& f, int role,
                                           double* s_red, int r0) {
  if constexpr (MODE != MODE_FWD) {
    ip_dispatch<R, MODE>(C, a, f, role, [&](auto PART, auto&& p, auto&& q) {
      ip3set_part<R, PART.value, MASK, PAIR>(p, q, s_red, r0);
    });
  }
}

// run-time mask -> compile-time MASK for the common wide sets (R = 4, three
// or four slots); other masks take the per-slot path. Kept narrow: every
// specialisation is ~1-2k FP64 instructions per kernel instantiation.
template <int R, class F, class G>
__device__ __forceinline__ void with_wide_mask(uint32_t mask, F&& f, G&& generic) {
  if constexpr (R == 4) {
    switch (mask) {
      case 15: f(IC<15>{}); return;
      case 7: f(IC<7>{}); return;
      case 11: f(IC<11>{}); return;
      case 13: f(IC<13>{}); return;
      case 14: f(IC<14>{}); return;
      default: break;
    }
  }
  generic();
}

// interpreter: one op of the device program, operands decoded at run time
template <int R, int MODE>
__device__ __forceinline__ void exec_op(const DevProgram& D, const Op op, Regs<R>& a, Regs<R>& f,
                                        const SegCtx<R>& C, int role, const SampleTables& T, double* s_redbuf) {
  const uint32_t w0 = op.w0;
  const uint32_t A = op_a(w0), Bq = op_b(w0);
  const uint32_t J0 = C.J0;
  const bool adj = op_adj(w0);
  switch (op_code(w0)) {
    case OP_RX:
    case OP_RY: {
      const int r = (int)op.param - T.rot_base;
      const bool rx = op_code(w0) == OP_RX;
      with_slot<R>(A & 7u, [&](auto SL) {
        if (rx) {
          if (adj) jop_rot<R, MODE, G_RX, SL.value, true>(a, f, T, r);
          else jop_rot<R, MODE, G_RX, SL.value, false>(a, f, T, r);
        } else {
          if (adj) jop_rot<R, MODE, G_RY, SL.value, true>(a, f, T, r);
          else jop_rot<R, MODE, G_RY, SL.value, false>(a, f, T, r);
        }
      });
    } break;
    case OP_RZ: {
      const uint32_t m = (A & kSlotFlag) ? (1u << (A & 7u)) : 0u;
      const bool cb = (A & kSlotFlag) ? false : ((J0 >> A) & 1u);
      const int r = (int)op.param - T.rot_base;
      if (adj) jop_rz<R, MODE, true>(a, f, T, r, m, cb);
      else jop_rz<R, MODE, false>(a, f, T, r, m, cb);
    } break;
    case OP_U2: {
      const int blk = (int)op.param - T.blk_base;
      with_slot<R>(A & 7u, [&](auto SL) {
        if (adj) jop_u2<R, MODE, SL.value, true>(a, f, T, blk);
        else jop_u2<R, MODE, SL.value, false>(a, f, T, blk);
      });
    } break;
    case OP_U2SET: {
      // forward segments apply blocks, adjoint segments un-apply them
      constexpr bool ADJ = MODE != MODE_FWD;
      const int16_t* ids = D.setids + op.param * kMaxR;
      with_wide_mask<R>(
          Bq, [&](auto MK) { jop_u2set<R, MODE, ADJ, MK.value>(a, f, T, ids); },
          [&]() {
#pragma unroll
            for (int sl = 0; sl < R; ++sl) {
              const int id = ids[sl];
              if (id < 0) continue;
              with_const_slot<R>(sl, [&](auto SL) {
                if (adj) jop_u2<R, MODE, SL.value, true>(a, f, T, id);
                else jop_u2<R, MODE, SL.value, false>(a, f, T, id);
              });
            }
          });
    } break;
    case OP_CNOT: {
      if (A & kSlotFlag) {
        with_slot<R>(A & 7u, [&](auto Cc) {
          with_slot<R>(Bq & 7u, [&](auto Tt) { jop_cnot_rr<R, MODE, Cc.value, Tt.value>(a, f); });
        });
      } else {
        const bool cb = (J0 >> A) & 1u;
        with_slot<R>(Bq & 7u, [&](auto Tt) { jop_cnot_cr<R, MODE, Tt.value>(a, f, cb); });
      }
    } break;
    case OP_H:
      with_slot<R>(A & 7u, [&](auto SL) { jop_h<R, MODE, SL.value>(a, f); });
      break;
    case OP_X:
      with_slot<R>(A & 7u, [&](auto SL) { jop_x<R, MODE, SL.value>(a, f); });
      break;
    case OP_CZ: {
      uint32_t m = 0;
      bool cond = true;
      if (A & kSlotFlag) m |= 1u << (A & 7u); else cond = cond && ((J0 >> A) & 1u);
      if (Bq & kSlotFlag) m |= 1u << (Bq & 7u); else cond = cond && ((J0 >> Bq) & 1u);
      jop_cz<R, MODE>(a, f, m, cond);
    } break;
    case OP_CZRUN:
      jop_czrun<R, MODE>(a, f, D.diag + op.param, J0);
      break;
    case OP_PUBLISH:
      break;  // handled by the segment loop (needs the CTA barrier)
    case OP_IP3:
      with_slot<R>(A & 7u, [&](auto SL) { jop_ip3<R, MODE, SL.value>(C, a, f, role, s_redbuf, (int)op_ip(w0)); });
      break;
    case OP_IP3SET:
      if constexpr (MODE != MODE_FWD) {
        with_wide_mask<R>(
            Bq, [&](auto MK) { jop_ip3set<R, MODE, MK.value>(C, a, f, role, s_redbuf, (int)op_ip(w0)); },
            [&]() {
              int r0 = (int)op_ip(w0);
#pragma unroll
              for (int sl = 0; sl < R; ++sl) {
                if (!((Bq >> sl) & 1u)) continue;
                with_const_slot<R>(sl, [&](auto SL) { jop_ip3<R, MODE, SL.value>(C, a, f, role, s_redbuf, r0); });
                r0 += 3;
              }
            });
      }
      break;
    case OP_IPX:
      with_slot<R>(A & 7u, [&](auto SL) { jop_ipxy<R, MODE, 0, SL.value>(C, a, f, role, s_redbuf, (int)op_ip(w0)); });
      break;
    case OP_IPY:
      with_slot<R>(A & 7u, [&](auto SL) { jop_ipxy<R, MODE, 1, SL.value>(C, a, f, role, s_redbuf, (int)op_ip(w0)); });
      break;
    default: {  // OP_IPZ
      const uint32_t m = (A & kSlotFlag) ? (1u << (A & 7u)) : 0u;
      const bool cb = (A & kSlotFlag) ? false : ((J0 >> A) & 1u);
      jop_ipz<R, MODE>(C, a, f, role, s_redbuf, (int)op_ip(w0), m, cb);
    } break;
  }
}

// ---------------------------------------------------------------------------
// Segment frame shared by the interpreter and the JIT: everything a segment
// needs besides its ops (the caller's run_segments arguments).
struct SegEnv {
  const DevProgram& D;
  const RunArgs& A;
  cplx_t* s_psi;
  cplx_t* s_phi;
  const double* s_av_all;
  int av_stride, av_base;
  double* s_red;
  double* s_fin;
  const Group& grp;
  bool active;
  uint32_t tile_base;
  int64_t bl0;
  int bra, tile, n_tiles;
  cplx_t* own;
  const cplx_t* partner;
  // direct tile I/O of the first / last segment of a sweep (JIT HBM passes)
  uint32_t io = 0;
  cplx_t* g_psi = nullptr;  // this row's states in HBM
  cplx_t* g_phi = nullptr;
};

// SegEnv::io. The first segment of a pass's sweep can take its registers
// straight from HBM (IO_LD) or set them to |0...0> (IO_INIT) and the last one
// can store them straight back (IO_ST) or drop them (IO_NOST: nothing reads
// the states after the adjoint sweep's last pass): the tile then crosses
// shared memory only between segments, half the shared-memory traffic of a
// three-segment pass, and warps start as soon as their own elements arrive.
enum { IO_LD = 1u, IO_INIT = 2u, IO_ST = 4u, IO_NOST = 8u };

template <int MODE>
__device__ __forceinline__ SegEnv make_env(const DevProgram& D, const RunArgs& A, cplx_t* s_psi, cplx_t* s_phi,
                                           const double* s_av_all, int av_stride, int av_base, double* s_red,
                                           double* s_fin, const Group& grp, bool active, uint32_t tile_base,
                                           int64_t bl0, int bra, int tile, int n_tiles) {
  cplx_t* own = (MODE == MODE_SPLIT && grp.role) ? s_phi : s_psi;
  const cplx_t* partner = (MODE == MODE_SPLIT && grp.role) ? s_psi : s_phi;
  return SegEnv{D, A, s_psi, s_phi, s_av_all, av_stride, av_base, s_red, s_fin, grp, active, tile_base,
                bl0, bra, tile, n_tiles, own, partner};
}

// Segment descriptor access: RtSeg reads the device table at run time (the
// interpreter); the JIT emits a struct with the same static members as
// compile-time constants, so unused folds and address maps disappear.
struct RtSeg {
  // JIT descriptors compute the thread maps from gi (thr_j0 / thr_lp0 / thr_sp0)
  __host__ __device__ static constexpr bool thr_const() { return false; }
  __device__ static uint32_t thr_j0(uint32_t) { return 0u; }
  __device__ static uint32_t thr_lp0(uint32_t) { return 0u; }
  __device__ static uint32_t thr_sp0(uint32_t) { return 0u; }
  const SegDesc* sd;
  __device__ __forceinline__ int nthr() const { return sd->nthr; }
  __device__ __forceinline__ int thr_off() const { return sd->thr_off; }
  __device__ __forceinline__ uint32_t ld_k(int t) const { return sd->ld_k[t]; }
  __device__ __forceinline__ uint32_t st_k(int t) const { return sd->st_k[t]; }
  __device__ __forceinline__ uint32_t ps(int t) const { return sd->ps[t]; }
  __device__ __forceinline__ uint32_t ldc(int t) const { return sd->ldc[t]; }
  __device__ __forceinline__ uint32_t stc(int t) const { return sd->stc[t]; }
  __device__ __forceinline__ int ip_count() const { return sd->ip_count; }
  __device__ __forceinline__ int red_count() const { return sd->red_count; }
  __device__ __forceinline__ int ip_begin() const { return sd->ip_begin; }
  // stores leave the loading threads' cells (CNOT folds onto thread bits):
  // every thread must finish its loads before any thread stores
  __device__ __forceinline__ bool st_sync() const { return sd->gen != 0; }
  // translation of the load / store base by the tile's (non-local) bits:
  // folded CNOTs controlled by tile bits (register targets only here, gen = 0)
  __device__ __forceinline__ uint32_t tile_ld(uint32_t tb) const {
    uint32_t t0 = 0u;
#pragma unroll
    for (int t = 0; t < kMaxR; ++t)
      if (__popc(tb & sd->ld_k[t]) & 1) t0 ^= sd->ps[t];
    return t0;
  }
  __device__ __forceinline__ uint32_t tile_st(uint32_t tb) const {
    uint32_t t0 = 0u;
#pragma unroll
    for (int t = 0; t < kMaxR; ++t)
      if (__popc(tb & sd->st_k[t]) & 1) t0 ^= sd->ps[t];
    return t0;
  }
};

// segment start: address maps and the register load (shared-memory transpose)
template <int R, int MODE, class SD>
__device__ __forceinline__ void seg_begin(const SegEnv& E, const SD& sd, SegCtx<R>& C, Regs<R>& a, Regs<R>& f) {
  constexpr int N = 1 << R;
  const int nthr = sd.nthr();
  C.own = E.own;
  C.partner = E.partner;
  if constexpr (SD::thr_const()) {
    const uint32_t gi = (uint32_t)E.grp.gi & ((1u << nthr) - 1u);
    C.J0 = E.tile_base | SD::thr_j0(gi);
    C.lp0 = SD::thr_lp0(gi);
  } else {
    const ThrEntry* te = E.D.thr_tab + sd.thr_off() + (E.grp.gi & ((1 << nthr) - 1));
    const uint2 e01 = *reinterpret_cast<const uint2*>(te);
    C.J0 = E.tile_base | e01.x;
    C.lp0 = e01.y;
  }
  // folded CNOT runs controlled by tile (non-local) bits
  if (E.tile_base != 0) C.lp0 ^= sd.tile_ld(E.tile_base);
#pragma unroll
  for (int t = 0; t < R; ++t) C.lc[t] = sd.ldc(t);
  if (E.active) {
#pragma unroll
    for (int i = 0; i < N; ++i) {
      const uint32_t ad = C.addr(i);
      VQC_CHECK(E.A, ad < (1u << E.D.k), CHK_SEG_LOAD);
      a[i] = E.own[ad];
      if constexpr (MODE == MODE_DUAL) f[i] = E.s_phi[ad];
    }
  }
  phase_a();  // ping-pong hand-over point (see cta_group)
}

// split adjoint: write this thread's registers back for the partner's inner products
template <int R, int MODE>
__device__ __forceinline__ void seg_publish(const SegEnv& E, const SegCtx<R>& C, const Regs<R>& a) {
  if constexpr (MODE == MODE_SPLIT) {
    vsync();
    if (E.active) {
      uint32_t base = C.lp0;
      asm volatile("" : "+r"(base));
#pragma unroll
      for (int i = 0; i < (1 << R); ++i) {
        uint32_t ad = base;
#pragma unroll
        for (int s = 0; s < R; ++s)
          if ((i >> s) & 1) ad ^= C.lc[s];
        E.own[ad] = a[i];
      }
    }
    vsync();
  }
}

// timing ablations (wrong results; VQC_JIT_OPTS=-DVQC_ABL_WSYNC / -DVQC_ABL_NORED)
#ifdef VQC_ABL_ALL
#define VQC_ABL_WSYNC 1
#define VQC_ABL_NORED 1
#endif
#ifdef VQC_ABL_WSYNC
#define VQC_ABL_SYNC() __syncwarp()
#else
#define VQC_ABL_SYNC() vsync()
#endif

// segment end: register store (through the folded store map), barrier, and the
// segment's gradient outputs
template <int R, int MODE, bool REDUCE = true, class SD>
__device__ __forceinline__ void seg_end(const SegEnv& E, const SD& sd, const Regs<R>& a, const Regs<R>& f) {
  constexpr int N = 1 << R;
  const Group& grp = E.grp;
  const RunArgs& A = E.A;
  phase_b();  // ping-pong hand-over point
  if ((MODE == MODE_SPLIT && sd.ip_count() > 0) || sd.st_sync()) VQC_ABL_SYNC();  // partners / other cells done reading
  asm volatile("" ::: "memory");  // keep the store map's loads and math after the op loop
  if (E.active) {
    uint32_t sp0, sc[R];
    if constexpr (SD::thr_const()) {
      sp0 = SD::thr_sp0((uint32_t)grp.gi & ((1u << sd.nthr()) - 1u));
    } else {
      const ThrEntry* te = E.D.thr_tab + sd.thr_off() + (grp.gi & ((1 << sd.nthr()) - 1));
      sp0 = te->sp0;
    }
    if (E.tile_base != 0) sp0 ^= sd.tile_st(E.tile_base);
    asm volatile("" : "+r"(sp0));
#pragma unroll
    for (int t = 0; t < R; ++t) sc[t] = sd.stc(t);
#pragma unroll
    for (int i = 0; i < N; ++i) {
      uint32_t ad = sp0;
#pragma unroll
      for (int s = 0; s < R; ++s)
        if ((i >> s) & 1) ad ^= sc[s];
      VQC_CHECK(A, ad < (1u << E.D.k), CHK_SEG_STORE);
      E.own[ad] = a[i];
      if constexpr (MODE == MODE_DUAL) E.s_phi[ad] = f[i];
    }
  }
  VQC_ABL_SYNC();
#ifdef VQC_ABL_NORED
  return;
#endif
  if constexpr (MODE != MODE_FWD && REDUCE) {
    const int nout = sd.ip_count();
    if (nout > 0) {
      // phase 1: one warp per (reduction slot, sample) sums the sample's
      // per-thread partials in a fixed order; phase 2: one thread per
      // (output, sample) applies the block gradient vector. Blocks narrower
      // than a warp (tiny n) reduce serially on thread 0.
      const int nred = sd.red_count();
      const bool narrow = vdim() < 32;
      const int lane = narrow ? 0 : (vtid() & 31);
      const int warp = narrow ? (vtid() == 0 ? 0 : 1 << 30) : (vtid() >> 5);
      const int nwarp = narrow ? 1 : (vdim() >> 5);
      for (int task = warp; task < nred * grp.S; task += nwarp) {
        const int slot = task / grp.S, s_ = task - slot * grp.S;
        const double* base = E.s_red + slot * (int)vdim() + s_ * grp.TT;
        double v = 0.0;
        if (narrow) {
          for (int t = 0; t < grp.TT; ++t) v += base[t];
        } else {
          for (int t = lane; t < grp.TT; t += 32) v += base[t];
          for (int off = 16; off > 0; off >>= 1) v += __shfl_xor_sync(0xffffffffu, v, off);
        }
        if (lane == 0) E.s_fin[slot * grp.S + s_] = v;
      }
      vsync();
      for (int task = vtid(); task < nout * grp.S; task += vdim()) {
        const int oi = task / grp.S, s_ = task - oi * grp.S;
        const IpOut io = E.D.ipouts[sd.ip_begin() + oi];
        const double* r = E.s_fin + s_;
        double v;
        if (io.avec < 0) {
          v = r[io.red * grp.S];
        } else {
          const double* av = E.s_av_all + (size_t)s_ * E.av_stride + 4 * (io.avec - E.av_base);
          v = av[0] * r[io.red * grp.S] + av[1] * r[(io.red + 1) * grp.S] + av[2] * r[(io.red + 2) * grp.S];
        }
        const int64_t bl = E.bl0 + s_;
        VQC_CHECK(A, io.gslot >= 0 && io.gslot < E.D.NG && E.tile < E.n_tiles, CHK_IP_OUT);
        if (bl < A.nb) A.ip[(((bl * A.K) + E.bra) * E.D.NG + io.gslot) * E.n_tiles + E.tile] = v;
      }
    }
  }
}

// ---------------------------------------------------------------------------
// Thread-group barriers and per-warp reductions (JIT HBM pass kernels; the
// scheduler's assign_thread_groups plans the thread-index bits).
//
// group_sync_t<T, NTHR>: barrier over the 2^NTHR >> T threads that share the top T
// thread-index bits (T = 0: the CTA; a warp or less: __syncwarp). Named
// barriers 2^T - 1 + group index (levels 1..3 use ids 1..14).
template <int T, int NTHR>
__device__ __forceinline__ void group_sync_t() {
  // T: compile-time level (the JIT's segment descriptors). Immediate barrier
  // ids, and only those of this level: a register id makes ptxas reserve all
  // 16 named barriers, which caps the resident CTAs per SM at 4.
  if constexpr (T <= 0) {
    vsync();
  } else {
    constexpr unsigned g = (1u << NTHR) >> T;  // NTHR thread-index bits: the tile's threads
    if constexpr (g <= 32u) {
      __syncwarp();
    } else if constexpr ((1 << T) > 4) {
      // eight groups (512-thread tiles, one CTA per SM anyway): a register id
      const unsigned id = (1u << T) - 1u + vtid() / g;
      asm volatile("bar.sync %0, %1;" ::"r"(id), "n"(g) : "memory");
    } else {
      const unsigned grp = vtid() / g;
#define VQC_BAR_CASE(I)                                                       \
  if constexpr ((I) < (1 << T)) {                                             \
    if (grp == (I)) asm volatile("bar.sync %0, %1;" ::"n"((1 << T) - 1 + (I)), "r"(g) : "memory"); \
  }
      VQC_BAR_CASE(0) VQC_BAR_CASE(1) VQC_BAR_CASE(2) VQC_BAR_CASE(3) VQC_BAR_CASE(4) VQC_BAR_CASE(5) VQC_BAR_CASE(6)
      VQC_BAR_CASE(7)
#undef VQC_BAR_CASE
    }
  }
}

// segment end with a group barrier: register store through the folded store
// map, then the barrier the next segment's loads need (sd.sync_st top bits
// shared). Gradient partials are reduced per warp (wr_split / wr_join), so no
// reduction phases follow.
template <int R, int MODE, class SD>
__device__ __forceinline__ void seg_end_g(const SegEnv& E, const SD& sd, const Regs<R>& a, const Regs<R>& f) {
  constexpr int N = 1 << R;
  const Group& grp = E.grp;
  if (sd.st_sync()) group_sync_t<SD::sync_self(), SD::nthr()>();  // the group's loads are done before its cells are overwritten
  asm volatile("" ::: "memory");
  uint32_t sp0, sc[R];
  sp0 = SD::thr_sp0((uint32_t)grp.gi & ((1u << sd.nthr()) - 1u));
  if (E.tile_base != 0) sp0 ^= sd.tile_st(E.tile_base);
  asm volatile("" : "+r"(sp0));
#pragma unroll
  for (int t = 0; t < R; ++t) sc[t] = sd.stc(t);
#pragma unroll
  for (int i = 0; i < N; ++i) {
    uint32_t ad = sp0;
#pragma unroll
    for (int s = 0; s < R; ++s)
      if ((i >> s) & 1) ad ^= sc[s];
    VQC_CHECK(E.A, ad < (1u << E.D.k), CHK_SEG_STORE);
    E.own[ad] = a[i];
    if constexpr (MODE == MODE_DUAL) E.s_phi[ad] = f[i];
  }
  group_sync_t<SD::sync_st(), SD::nthr()>();
}

__device__ __forceinline__ void cp_async_wait_all_();

// First segment of a sweep: registers from HBM (IO_LD), the initial state
// (IO_INIT) or shared memory. The global index of register element i is the
// folded load map applied to (thread bits | register bits | tile bits),
// deposited on the pass's local qubits: GF(2)-linear like the shared-memory
// address, so base ^ XOR of per-register-bit columns (SD::thr_gl, tile_gl,
// gcol_l). The per-sample tables (cp.async in pass_body) are awaited here,
// after the loads are in flight; that CTA barrier also orders these loads
// before any thread's direct stores to the same cells at the end of the pass.
template <int R, int MODE, class SD>
__device__ __forceinline__ void seg_begin_io(const SegEnv& E, const SD& sd, SegCtx<R>& C, Regs<R>& a, Regs<R>& f) {
  constexpr int N = 1 << R;
  if (!(E.io & (IO_LD | IO_INIT))) {
    seg_begin<R, MODE>(E, sd, C, a, f);
    return;
  }
  const uint32_t gi = (uint32_t)E.grp.gi & ((1u << sd.nthr()) - 1u);
  C.own = E.own;
  C.partner = E.partner;
  C.J0 = E.tile_base | SD::thr_j0(gi);
  C.lp0 = 0;
#pragma unroll
  for (int t = 0; t < R; ++t) C.lc[t] = 0;
  if (E.io & IO_INIT) {
#pragma unroll
    for (int i = 0; i < N; ++i) {
      a[i] = mk_c((C.J0 == 0u && i == 0) ? 1 : 0, 0);
      if constexpr (MODE == MODE_DUAL) f[i] = mk_c(0, 0);
    }
  } else {
    uint32_t gb = E.tile_base | SD::thr_gl(gi);
    if (E.tile_base != 0) gb ^= SD::tile_gl(E.tile_base);
#pragma unroll
    for (int i = 0; i < N; ++i) {
      uint32_t idx = gb;
#pragma unroll
      for (int s2 = 0; s2 < R; ++s2)
        if ((i >> s2) & 1) idx ^= SD::gcol_l(s2);
      VQC_CHECK(E.A, idx < (1u << E.D.n), CHK_TILE_GLOBAL);
      a[i] = E.g_psi[idx];  // through L1: 16-byte pieces of one sector merge there
      if constexpr (MODE == MODE_DUAL) f[i] = E.g_phi[idx];
    }
  }
  cp_async_wait_all_();
  vsync();
}

// Last segment of a sweep: registers straight to HBM (IO_ST), nowhere
// (IO_NOST) or to shared memory behind a CTA barrier.
template <int R, int MODE, class SD>
__device__ __forceinline__ void seg_end_io(const SegEnv& E, const SD& sd, const Regs<R>& a, const Regs<R>& f) {
  constexpr int N = 1 << R;
  if (E.io & IO_NOST) return;
  if (!(E.io & IO_ST)) {
    seg_end_g<R, MODE>(E, sd, a, f);
    return;
  }
  const uint32_t gi = (uint32_t)E.grp.gi & ((1u << sd.nthr()) - 1u);
  uint32_t gb = E.tile_base | SD::thr_gs(gi);
  if (E.tile_base != 0) gb ^= SD::tile_gs(E.tile_base);
#pragma unroll
  for (int i = 0; i < N; ++i) {
    uint32_t idx = gb;
#pragma unroll
    for (int s2 = 0; s2 < R; ++s2)
      if ((i >> s2) & 1) idx ^= SD::gcol_s(s2);
    VQC_CHECK(E.A, idx < (1u << E.D.n), CHK_TILE_GLOBAL);
    __stcg(E.g_psi + idx, a[i]);
    if constexpr (MODE == MODE_DUAL) __stcg(E.g_phi + idx, f[i]);
  }
}

// Deterministic warp reduction of N per-thread partials by recursive halving:
// at lane bit B the lanes with the bit clear keep the lower half of the
// values and send the upper half to their partner (and vice versa), so after
// the five steps each value's total sits in the lanes of one group; values
// beyond nv (padding of odd halves) are zero and the lane whose lower bits
// are clear writes dst[index]: 2 * (N/2 + N/4 + ...) shuffles instead of 5
// per value.
// It runs in stages the JIT weaves between a segment's gate blocks, so each
// round's shuffle latency hides behind FP64 work instead of stalling the warp
// five times: wr_split sends this round's halves (base / nv track which value
// indices the lane still holds), wr_join adds what arrived.
template <int N, int BIT>
__device__ __forceinline__ void wr_split(const double (&v)[N], unsigned lane, double (&keep)[(N + 1) / 2],
                                         double (&recv)[(N + 1) / 2], int& base, int& nv) {
  const bool up = ((lane >> BIT) & 1u) != 0u;
  if constexpr (N == 1) {
    keep[0] = v[0];
    recv[0] = __shfl_xor_sync(0xffffffffu, v[0], 1 << BIT);
    if (up) nv = 0;  // both lanes of the pair hold the same total; the lower one goes on
  } else {
    constexpr int H = (N + 1) / 2;
#pragma unroll
    for (int i = 0; i < H; ++i) {
      const double lo = v[i], hi = (i + H < N) ? v[i + H] : 0.0;
      const double send = up ? lo : hi;
      keep[i] = up ? hi : lo;
      recv[i] = __shfl_xor_sync(0xffffffffu, send, 1 << BIT);
    }
    const int nlo = nv < H ? nv : H;
    base += up ? H : 0;
    nv = up ? nv - nlo : nlo;
  }
}
template <int H>
__device__ __forceinline__ void wr_join(const double (&keep)[H], const double (&recv)[H], double (&w)[H]) {
#pragma unroll
  for (int i = 0; i < H; ++i) w[i] = keep[i] + recv[i];
}

// inner products into per-thread partials (both states in registers)
template <int R, int S>
__device__ __forceinline__ void jop_ip3w(const Regs<R>& a, const Regs<R>& f, double& ix, double& iy, double& iz) {
  ix = iy = iz = 0.0;
  auto ra = [&](int i) { return a[i]; };
  auto rf = [&](int i) { return f[i]; };
  ip_xyz<R, S, -1>(ra, rf, ix, iy, iz);
}
// Im<phi|X,Y,Z|psi> on every slot of MASK at once (a set of fused blocks):
// the Z products Im(conj(phi_i) psi_i) are the same for every slot, which
// only signs them differently, so they are formed once (2 FP64 ops per
// element) and each slot's Z sum costs adds instead of its own 4 products
// per pair. pr: 3 values per slot of MASK in slot order.
template <int R, int MASK>
__device__ __forceinline__ void jop_ip3w_set(const Regs<R>& a, const Regs<R>& f, double* pr) {
  constexpr int N = 1 << R;
  real_t d[N];
#pragma unroll
  for (int i = 0; i < N; ++i) d[i] = fma(f[i].x, a[i].y, -(f[i].y * a[i].x));
  int k = 0;
#pragma unroll
  for (int s = 0; s < R; ++s) {
    if (!((MASK >> s) & 1)) continue;
    real_t ax[2] = {0, 0}, ay[2] = {0, 0}, z0 = 0, z1 = 0;
    int c = 0;
#pragma unroll
    for (int i = 0; i < N; ++i) {
      if ((i >> s) & 1) {
        z1 += d[i];
        continue;
      }
      z0 += d[i];
      const int j = i | (1 << s);
      const cplx_t f0 = f[i], f1 = f[j], p0 = a[i], p1 = a[j];
      ax[c] = fma(f0.x, p1.y, ax[c]);
      ax[c] = fma(-f0.y, p1.x, ax[c]);
      ax[c] = fma(f1.x, p0.y, ax[c]);
      ax[c] = fma(-f1.y, p0.x, ax[c]);
      ay[c] = fma(-f0.x, p1.x, ay[c]);
      ay[c] = fma(-f0.y, p1.y, ay[c]);
      ay[c] = fma(f1.x, p0.x, ay[c]);
      ay[c] = fma(f1.y, p0.y, ay[c]);
      c ^= 1;
    }
    pr[3 * k] = (double)(ax[0] + ax[1]);
    pr[3 * k + 1] = (double)(ay[0] + ay[1]);
    pr[3 * k + 2] = (double)(z0 - z1);
    ++k;
  }
}

template <int R, int KIND, int S>
__device__ __forceinline__ double jop_ipxyw(const Regs<R>& a, const Regs<R>& f) {
  auto ra = [&](int i) { return a[i]; };
  auto rf = [&](int i) { return f[i]; };
  if constexpr (KIND == 0) return ip_x<R, S, -1>(ra, rf);
  else return ip_y<R, S, -1>(ra, rf);
}
template <int R>
__device__ __forceinline__ double jop_ipzw(const Regs<R>& a, const Regs<R>& f, uint32_t m, bool cb) {
  auto ra = [&](int i) { return a[i]; };
  auto rf = [&](int i) { return f[i]; };
  return ip_z<R, -1>(ra, rf, m, cb);
}

// End of a pass's adjoint segments: sum each reduction slot over the warps in
// warp order and write the pass's gradient outputs. tab rows: (gradient slot,
// pass-relative reduction slot, pass-relative block gradient vector or -1).
// The caller's last group barrier (the CTA) ordered the partial table.
__device__ __forceinline__ void wred_outputs(const SegEnv& E, const int (*tab)[3], int count, int wstride) {
  const RunArgs& A = E.A;
  const int nw = (int)(vdim() >> 5);
  for (int oi = (int)vtid(); oi < count; oi += (int)vdim()) {
    const int gslot = tab[oi][0], red = tab[oi][1], avec = tab[oi][2];
    const int nr = avec < 0 ? 1 : 3;
    double r[3] = {0.0, 0.0, 0.0};
    for (int w = 0; w < nw; ++w)
      for (int j = 0; j < nr; ++j) r[j] += E.s_red[w * wstride + red + j];
    double v = r[0];
    if (avec >= 0) {
      const double* av = E.s_av_all + 4 * avec;
      v = av[0] * r[0] + av[1] * r[1] + av[2] * r[2];
    }
    VQC_CHECK(A, gslot >= 0 && gslot < E.D.NG && E.tile < E.n_tiles, CHK_IP_OUT);
    if (E.bl0 < A.nb) A.ip[(((E.bl0 * A.K) + E.bra) * E.D.NG + gslot) * E.n_tiles + E.tile] = v;
  }
}

// Lagged segment reductions (JIT, one sample per CTA): after segment s's
// post-store barrier run phase 2 of the previous inner-product segment (its
// outputs from s_fin) and phase 1 of segment s (one warp per slot over the
// pair-reduced partial rows, into the other s_fin buffer). Partial rows and
// s_fin alternate between segments and the next post-store barrier orders
// every reuse, so the reduction needs no barrier of its own.
__device__ __forceinline__ void jred_phase1(const SegEnv& E, int slot0, int nred, int fin0) {
  const int lane = vtid() & 31, warp = vtid() >> 5, nwarp = vdim() >> 5;
  const int W = (int)(vdim() >> 1);
  for (int s = warp; s < nred; s += nwarp) {
    const double* base = E.s_red + (slot0 + s) * W;
    double v = 0.0;
    for (int t = lane; t < W; t += 32) v += base[t];
#pragma unroll
    for (int off = 16; off > 0; off >>= 1) v += __shfl_xor_sync(0xffffffffu, v, off);
    if (lane == 0) E.s_fin[fin0 + s] = v;
  }
}
template <class SD>
__device__ __forceinline__ void jred_phase2(const SegEnv& E, const SD& sd, int fin0) {
  const RunArgs& A = E.A;
  for (int oi = vtid(); oi < sd.ip_count(); oi += vdim()) {
    const IpOut io = E.D.ipouts[sd.ip_begin() + oi];
    const double* r = E.s_fin + fin0;
    double v;
    if (io.avec < 0) {
      v = r[io.red];
    } else {
      const double* av = E.s_av_all + 4 * (io.avec - E.av_base);
      v = av[0] * r[io.red] + av[1] * r[io.red + 1] + av[2] * r[io.red + 2];
    }
    const int64_t bl = E.bl0;
    if (bl < A.nb) A.ip[(((bl * A.K) + E.bra) * E.D.NG + io.gslot) * E.n_tiles + E.tile] = v;
  }
}

// Interpreter: run segments [sb, se) on the tile(s) in shared memory.
// MODE_FWD: psi only; MODE_DUAL: each thread holds psi and phi of its register
// group; MODE_SPLIT: role-0 threads hold psi, role-1 threads phi. Gradient
// outputs go to A.ip (rows relative to A.b0, times n_tiles). Threads with
// active == false only take part in the barriers.
struct RtPassMap;  // pass index maps (defined with the tile walk below)
struct RtTerms;  // observable terms read at run time (skeleton.cuh)
struct InterpSegs {
  using PM = RtPassMap;
  using Terms = RtTerms;
  // tiles always staged through shared memory
  static constexpr bool kDioF = false, kDioB = false, kDioFL = false, kDioFS = false, kDioBL = false, kDioBS = false;
  template <int R, int MODE>
  __device__ __forceinline__ static void run(const SegEnv& E, const SampleTables& T, int sb, int se) {
    const DevProgram& D = E.D;
    long long tdbg = E.A.dbg ? clock64() : 0;
    for (int sg = sb; sg < se; ++sg) {
      const SegDesc* sdp = D.segs + sg;
      const RtSeg sd{sdp};
      SegCtx<R> C;
      Regs<R> a, f;
      seg_begin<R, MODE>(E, sd, C, a, f);
      dbg_add(E.A, DBG_SEG_LOAD, tdbg);
      const int ob = sdp->op_begin, oe = sdp->op_end;
      Op nxt = ob < oe ? D.ops[ob] : Op{0u, 0u};
      for (int o = ob; o < oe; ++o) {
        const Op op = nxt;
        if (o + 1 < oe) nxt = D.ops[o + 1];
        if (MODE == MODE_SPLIT && op_code(op.w0) == OP_PUBLISH) {
          seg_publish<R, MODE>(E, C, a);
          continue;
        }
        if (E.active) exec_op<R, MODE>(D, op, a, f, C, E.grp.role, T, E.s_red);
      }
      dbg_add(E.A, DBG_SEG_OPS, tdbg);
      seg_end<R, MODE>(E, sd, a, f);
      dbg_add(E.A, DBG_SEG_FINAL, tdbg);
    }
  }
};

// Per-sample tables for one pass: (cos, sin) of every rotation, then each
// fused block's unitary and gradient vectors (blockmath.h). Ends synchronised.
__device__ __forceinline__ void build_tables(const DevProgram& D, const RunArgs& A, const PassDesc* pd,
                                             int64_t b, bool valid, double2* cs, double2* u, double* av,
                                             int lane, int width) {
  const int nrot = pd->rot_end - pd->rot_begin;
  for (int r = lane; r < nrot; r += width)
    cs[r] = valid ? rot_cs(D, A, b, pd->rot_begin + r) : make_double2(1.0, 0.0);
  vsync();
  const int nblk = pd->blk_end - pd->blk_begin;
  for (int k = lane; k < nblk; k += width) {
    const BlockDesc bd = D.blocks[pd->blk_begin + k];
    const M2 U = block_unitary(
        D.members + bd.mem_begin, bd.mem_end - bd.mem_begin,
        [&](int rot) { return cs[rot - pd->rot_begin]; },
        [&](int slot, const double* v) {
          double* o = av + 4 * (slot - pd->av_begin);
          o[0] = v[0];
          o[1] = v[1];
          o[2] = v[2];
          o[3] = 0.0;
        });
    double2* o = u + 4 * k;
    o[0] = make_double2(U.a.re, U.a.im);
    o[1] = make_double2(U.b.re, U.b.im);
    o[2] = make_double2(U.c.re, U.c.im);
    o[3] = make_double2(U.d.re, U.d.im);
  }
  vsync();
}

// Global indices of the tile elements a thread visits in a strided loop
// l = lane + i * stride (stride a power of two): dep() is GF(2)-linear, so
// j(i) = base ^ XOR_{b in i} hi[b]; visiting i in Gray-code order costs one
// XOR per element.
struct TileWalk {
  uint32_t base;           // global index of this thread's first element
  uint32_t hi[kMaxR];      // global index bit of element-index bit b
  uint32_t sbase;          // swizzled tile address of the first element
  uint32_t shi[kMaxR];     // swizzled address bit of element-index bit b
  int count;  // elements per thread: 2^k / stride = 2^R <= 16
};

// pdep: the bits of l deposited into the set bits of m (ascending); the
// pass's local qubits are local_mask's set bits in ascending order
__device__ __forceinline__ uint32_t pdep32(uint32_t l, uint32_t m) {
  uint32_t j = 0;
  for (uint32_t bb = 1; m != 0; bb <<= 1) {
    const uint32_t low = m & (0u - m);
    if (l & bb) j |= low;
    m ^= low;
  }
  return j;
}

// Pass index maps: tile-local position p -> global qubit bit (the pass's
// local qubits in ascending order) and tile id -> the non-local global bits.
// RtPassMap reads the pass descriptor; the JIT emits a map with the positions
// as constants (kConst), so the tile walk's index math folds to shifts.
struct RtPassMap {
  static constexpr bool kConst = false;
  static constexpr int k = 0;
  __device__ __forceinline__ static uint32_t lane_dep(const PassDesc* pd, uint32_t l) {
    uint32_t j = 0;
    while (l) {
      j |= 1u << pd->local_q[__ffs(l) - 1];
      l &= l - 1;
    }
    return j;
  }
  __device__ __forceinline__ static uint32_t local_bit(const PassDesc* pd, int p) { return 1u << pd->local_q[p]; }
  __device__ __forceinline__ static uint32_t tile_dep(const PassDesc* pd, int n, uint32_t t) {
    return pdep32(t, ~pd->local_mask & ((1u << n) - 1u));
  }
};

template <class PM = RtPassMap>
__device__ __forceinline__ TileWalk tile_walk(const PassDesc* pd, uint32_t tile_base, int k, int lane,
                                              int stride) {
  TileWalk w;
  const int Nt = 1 << k;
  w.count = Nt / stride;
  w.base = tile_base | (pd ? PM::lane_dep(pd, (uint32_t)lane) : (uint32_t)lane);
  w.sbase = swz((uint32_t)lane);
  const int s0 = __ffs(stride) - 1;  // stride is a power of two: hi[b] is one local bit
#pragma unroll
  for (int b = 0; b < kMaxR; ++b) {
    const int p = s0 + b;
    w.hi[b] = p < k ? (pd ? PM::local_bit(pd, p) : (1u << p)) : 0u;
    w.shi[b] = p < k ? swz(1u << p) : 0u;
  }
  return w;
}

// calls f(sw, j) for every element of this thread: sw its swizzled tile
// address, j its global index (both GF(2)-linear in the element index).
// E = elements per thread (compile time): unrolled in Gray-code order, so each
// element costs one XOR per index (the walk used to be a rolled loop with a
// per-element bit scan, ~20 integer instructions per element).
template <int G, int E, class F>
__device__ __forceinline__ void for_tile_step(const TileWalk& w, uint32_t j, uint32_t sw, F&& f) {
  if constexpr (G < E) {
    constexpr int b = ctz_const(G);  // Gray code: element G differs from element G - 1 in bit b
    j ^= w.hi[b];
    sw ^= w.shi[b];
    f(sw, j);
    for_tile_step<G + 1, E>(w, j, sw, f);
  }
}
template <int E, class F>
__device__ __forceinline__ void for_tile(const TileWalk& w, F&& f) {
  f(w.sbase, w.base);
  for_tile_step<1, E>(w, w.base, w.sbase, f);
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
