/*
 * TEST INFRASTRUCTURE — NOT PRODUCT CODE.
 *
 * CPU oracle: a plain-C restatement of the reference's statevector hot path
 * (vqckit, /root/reference/pkg/src/vqckit). It is the parity checker for the
 * sm_100a kernels and the CPU baseline arm of bench.py. Only tests/,
 * __graft_entry__.smoke() and bench.py's cpu_baseline / --impl reference legs
 * may load it. The product path (paper_2404_06314_b200) never links it.
 *
 * Parity pinned against: golden vectors produced by importing the reference
 * itself (tests/golden/make_golden.py) plus the reference's own known-answer
 * tests (tests/test_oracle_golden.py).
 *
 * States are complex128 stored as interleaved (re, im) doubles, little-endian
 * basis order: qubit q is bit q of the amplitude index
 * (statevector.py:1-11).
 */
#include <math.h>
#include <stdint.h>
#include <stdlib.h>
#include <string.h>

/* gate codes: _kernels.py:16-22; CZ (6) is new — the reference lacks it and
 * its golden vectors spell CZ(c,t) as H(t) CNOT(c,t) H(t). */
enum { ORC_RX = 0, ORC_RY = 1, ORC_RZ = 2, ORC_CNOT = 3, ORC_H = 4, ORC_X = 5, ORC_CZ = 6 };
/* generator axes: _kernels.py:24-27 */
enum { ORC_AX_X = 0, ORC_AX_Y = 1, ORC_AX_Z = 2 };

typedef struct { double re, im; } cplx;

/* _kernels.py:32-42 */
static void apply_rx(cplx* st, int64_t dim, int q, double theta) {
  const double c = cos(0.5 * theta), s = sin(0.5 * theta);
  const int64_t step = (int64_t)1 << q;
  for (int64_t base = 0; base < dim; base += step << 1)
    for (int64_t off = base; off < base + step; ++off) {
      cplx a0 = st[off], a1 = st[off + step];
      st[off].re = c * a0.re + s * a1.im;
      st[off].im = c * a0.im - s * a1.re;
      st[off + step].re = s * a0.im + c * a1.re;
      st[off + step].im = -s * a0.re + c * a1.im;
    }
}

/* _kernels.py:45-55 */
static void apply_ry(cplx* st, int64_t dim, int q, double theta) {
  const double c = cos(0.5 * theta), s = sin(0.5 * theta);
  const int64_t step = (int64_t)1 << q;
  for (int64_t base = 0; base < dim; base += step << 1)
    for (int64_t off = base; off < base + step; ++off) {
      cplx a0 = st[off], a1 = st[off + step];
      st[off].re = c * a0.re - s * a1.re;
      st[off].im = c * a0.im - s * a1.im;
      st[off + step].re = s * a0.re + c * a1.re;
      st[off + step].im = s * a0.im + c * a1.im;
    }
}

/* _kernels.py:58-66: ph0 = exp(-i theta/2), ph1 = exp(+i theta/2) */
static void apply_rz(cplx* st, int64_t dim, int q, double theta) {
  const double c = cos(0.5 * theta), s = sin(0.5 * theta);
  const int64_t step = (int64_t)1 << q;
  for (int64_t base = 0; base < dim; base += step << 1)
    for (int64_t off = base; off < base + step; ++off) {
      cplx a0 = st[off], a1 = st[off + step];
      st[off].re = c * a0.re + s * a0.im;
      st[off].im = c * a0.im - s * a0.re;
      st[off + step].re = c * a1.re - s * a1.im;
      st[off + step].im = c * a1.im + s * a1.re;
    }
}

/* _kernels.py:69-78 */
static void apply_h(cplx* st, int64_t dim, int q) {
  const double inv = 1.0 / sqrt(2.0);
  const int64_t step = (int64_t)1 << q;
  for (int64_t base = 0; base < dim; base += step << 1)
    for (int64_t off = base; off < base + step; ++off) {
      cplx a0 = st[off], a1 = st[off + step];
      st[off].re = (a0.re + a1.re) * inv;
      st[off].im = (a0.im + a1.im) * inv;
      st[off + step].re = (a0.re - a1.re) * inv;
      st[off + step].im = (a0.im - a1.im) * inv;
    }
}

/* _kernels.py:81-88 */
static void apply_x(cplx* st, int64_t dim, int q) {
  const int64_t step = (int64_t)1 << q;
  for (int64_t base = 0; base < dim; base += step << 1)
    for (int64_t off = base; off < base + step; ++off) {
      cplx a0 = st[off];
      st[off] = st[off + step];
      st[off + step] = a0;
    }
}

/* _kernels.py:91-100 (full scan, swap when control=1 and target=0) */
static void apply_cnot(cplx* st, int64_t dim, int control, int target) {
  const int64_t cbit = (int64_t)1 << control, tbit = (int64_t)1 << target;
  for (int64_t j = 0; j < dim; ++j)
    if ((j & cbit) != 0 && (j & tbit) == 0) {
      int64_t k = j | tbit;
      cplx a = st[j];
      st[j] = st[k];
      st[k] = a;
    }
}

/* new gate: diag(1,1,1,-1) on (c,t) — equals H(t) CNOT(c,t) H(t) */
static void apply_cz(cplx* st, int64_t dim, int a, int b) {
  const int64_t m = ((int64_t)1 << a) | ((int64_t)1 << b);
  for (int64_t j = 0; j < dim; ++j)
    if ((j & m) == m) { st[j].re = -st[j].re; st[j].im = -st[j].im; }
}

/* _kernels.py:103-116 */
static void apply_coded(cplx* st, int64_t dim, int64_t kind, int64_t q0, int64_t q1, double angle) {
  switch (kind) {
    case ORC_RX: apply_rx(st, dim, (int)q0, angle); break;
    case ORC_RY: apply_ry(st, dim, (int)q0, angle); break;
    case ORC_RZ: apply_rz(st, dim, (int)q0, angle); break;
    case ORC_CNOT: apply_cnot(st, dim, (int)q0, (int)q1); break;
    case ORC_H: apply_h(st, dim, (int)q0); break;
    case ORC_CZ: apply_cz(st, dim, (int)q0, (int)q1); break;
    default: apply_x(st, dim, (int)q0); break;
  }
}

/* _kernels.py:119-125: rotations invert by negating the angle */
static void apply_coded_adjoint(cplx* st, int64_t dim, int64_t kind, int64_t q0, int64_t q1, double angle) {
  apply_coded(st, dim, kind, q0, q1, kind <= ORC_RZ ? -angle : angle);
}

/* _kernels.py:128-134 */
void orc_compute_angles(const double* coeff, const int64_t* f_offs, const int64_t* f_idx,
                        const double* flat, int64_t n_gates, double* out) {
  for (int64_t g = 0; g < n_gates; ++g) {
    double a = coeff[g];
    for (int64_t t = f_offs[g]; t < f_offs[g + 1]; ++t) a *= flat[f_idx[t]];
    out[g] = a;
  }
}

/* _kernels.py:137-141 */
void orc_run_program(double* state, int n_qubits, const int64_t* kinds, const int64_t* q0,
                     const int64_t* q1, const double* angles, int64_t n_gates) {
  cplx* st = (cplx*)state;
  const int64_t dim = (int64_t)1 << n_qubits;
  for (int64_t g = 0; g < n_gates; ++g) apply_coded(st, dim, kinds[g], q0[g], q1[g], angles[g]);
}

static int parity64(int64_t x) { return __builtin_parityll((unsigned long long)x); }

/* _kernels.py:166-179: dst = sum_t coeff_t * phase_t * P_t src */
static void pauli_sum_apply(cplx* dst, const cplx* src, int64_t dim, const double* coeffs,
                            const int64_t* x_masks, const int64_t* sign_masks,
                            const double* phases /* (T,2) */, int64_t lo, int64_t hi) {
  for (int64_t j = 0; j < dim; ++j) dst[j].re = dst[j].im = 0.0;
  for (int64_t t = lo; t < hi; ++t) {
    const double wr = coeffs[t] * phases[2 * t], wi = coeffs[t] * phases[2 * t + 1];
    const int64_t xm = x_masks[t], sm = sign_masks[t];
    for (int64_t j = 0; j < dim; ++j) {
      const int64_t k = j ^ xm;
      const double pr = wr * src[k].re - wi * src[k].im;
      const double pi = wr * src[k].im + wi * src[k].re;
      if (parity64(k & sm)) { dst[j].re -= pr; dst[j].im -= pi; }
      else { dst[j].re += pr; dst[j].im += pi; }
    }
  }
}

/* _kernels.py:182-198: <state|O|state> without materialising O|state> */
void orc_expval_terms(const double* state, int n_qubits, const double* coeffs,
                      const int64_t* x_masks, const int64_t* sign_masks, const double* phases,
                      int64_t lo, int64_t hi, double* out_re_im) {
  const cplx* st = (const cplx*)state;
  const int64_t dim = (int64_t)1 << n_qubits;
  double ar = 0.0, ai = 0.0;
  for (int64_t t = lo; t < hi; ++t) {
    const double wr = coeffs[t] * phases[2 * t], wi = coeffs[t] * phases[2 * t + 1];
    const int64_t xm = x_masks[t], sm = sign_masks[t];
    double tr = 0.0, ti = 0.0;
    for (int64_t j = 0; j < dim; ++j) {
      const int64_t k = j ^ xm;
      /* conj(st[j]) * st[k] */
      const double pr = st[j].re * st[k].re + st[j].im * st[k].im;
      const double pi = st[j].re * st[k].im - st[j].im * st[k].re;
      if (parity64(k & sm)) { tr -= pr; ti -= pi; } else { tr += pr; ti += pi; }
    }
    ar += wr * tr - wi * ti;
    ai += wr * ti + wi * tr;
  }
  out_re_im[0] = ar;
  out_re_im[1] = ai;
}

/* _kernels.py:201-206 */
static void vdot(const cplx* a, const cplx* b, int64_t dim, double* re, double* im) {
  double ar = 0.0, ai = 0.0;
  for (int64_t j = 0; j < dim; ++j) {
    ar += a[j].re * b[j].re + a[j].im * b[j].im;
    ai += a[j].re * b[j].im - a[j].im * b[j].re;
  }
  *re = ar;
  *im = ai;
}

/* _kernels.py:220-238: dst = P_axis(q) src */
static void single_pauli_apply(cplx* dst, const cplx* src, int64_t dim, int64_t axis, int q) {
  const int64_t step = (int64_t)1 << q;
  for (int64_t base = 0; base < dim; base += step << 1)
    for (int64_t off = base; off < base + step; ++off) {
      const cplx a0 = src[off], a1 = src[off + step];
      if (axis == ORC_AX_X) { dst[off] = a1; dst[off + step] = a0; }
      else if (axis == ORC_AX_Y) {
        dst[off].re = a1.im; dst[off].im = -a1.re;          /* -i * a1 */
        dst[off + step].re = -a0.im; dst[off + step].im = a0.re;  /* i * a0 */
      } else {
        dst[off] = a0;
        dst[off + step].re = -a1.re; dst[off + step].im = -a1.im;
      }
    }
}

/* _kernels.py:241-281: one reverse pass over the gate list */
static void adjoint_reverse_pass(cplx* psi, cplx* phis, int64_t n_obs, int64_t dim,
                                 const int64_t* kinds, const int64_t* q0, const int64_t* q1,
                                 const double* angles, const int64_t* gen_axis, const double* coeff,
                                 const int64_t* f_offs, const int64_t* f_idx, const double* flat,
                                 const int64_t* wrt_col, int64_t n_cols, int64_t n_gates,
                                 cplx* tmp, double* ims, double* grad_out /* (M, n_cols) */) {
  for (int64_t g = n_gates - 1; g >= 0; --g) {
    const int64_t ax = gen_axis[g];
    if (ax >= 0) {
      int needed = 0;
      for (int64_t t = f_offs[g]; t < f_offs[g + 1]; ++t)
        if (wrt_col[f_idx[t]] >= 0) { needed = 1; break; }
      if (needed) {
        single_pauli_apply(tmp, psi, dim, ax, (int)q0[g]);
        for (int64_t i = 0; i < n_obs; ++i) {
          double re, im;
          vdot(phis + i * dim, tmp, dim, &re, &im);
          ims[i] = im;
        }
        for (int64_t t = f_offs[g]; t < f_offs[g + 1]; ++t) {
          const int64_t col = wrt_col[f_idx[t]];
          if (col < 0) continue;
          double partial = coeff[g];
          for (int64_t u = f_offs[g]; u < f_offs[g + 1]; ++u)
            if (u != t) partial *= flat[f_idx[u]];
          for (int64_t i = 0; i < n_obs; ++i) grad_out[i * n_cols + col] += ims[i] * partial;
        }
      }
    }
    apply_coded_adjoint(psi, dim, kinds[g], q0[g], q1[g], angles[g]);
    for (int64_t i = 0; i < n_obs; ++i)
      apply_coded_adjoint(phis + i * dim, dim, kinds[g], q0[g], q1[g], angles[g]);
  }
}

typedef struct {
  int64_t n_qubits, n_gates;
  const int64_t *kinds, *q0, *q1, *gen_axis;
  const double* coeff;
  const int64_t *f_offs, *f_idx;
  int64_t total_params;
  /* observable pack (observables.py:132-167) */
  int64_t n_obs;
  const int64_t* term_offs;
  const double* t_coeffs;
  const int64_t *t_xmask, *t_smask;
  const double* t_phases; /* (T, 2) re/im */
} OrcProblem;

/* gradients.py:104-118 (adjoint_flat) with the reverse pass gated on n_cols>0;
 * workspace: (n_obs + 2) * dim complex + n_obs doubles */
static void adjoint_flat(const OrcProblem* p, const double* flat, const int64_t* wrt_col,
                         int64_t n_cols, double* expect_out, double* grad_out, cplx* work,
                         double* angles, double* ims) {
  const int64_t dim = (int64_t)1 << p->n_qubits;
  cplx* psi = work;
  cplx* tmp = work + dim;
  cplx* phis = work + 2 * dim;
  orc_compute_angles(p->coeff, p->f_offs, p->f_idx, flat, p->n_gates, angles);
  memset(psi, 0, sizeof(cplx) * dim);
  psi[0].re = 1.0;
  orc_run_program((double*)psi, (int)p->n_qubits, p->kinds, p->q0, p->q1, angles, p->n_gates);
  /* seed_bras: _kernels.py:209-217 */
  for (int64_t i = 0; i < p->n_obs; ++i) {
    pauli_sum_apply(phis + i * dim, psi, dim, p->t_coeffs, p->t_xmask, p->t_smask, p->t_phases,
                    p->term_offs[i], p->term_offs[i + 1]);
    double re, im;
    vdot(psi, phis + i * dim, dim, &re, &im);
    expect_out[i] = re;
  }
  if (n_cols > 0 && p->n_gates > 0)
    adjoint_reverse_pass(psi, phis, p->n_obs, dim, p->kinds, p->q0, p->q1, angles, p->gen_axis,
                         p->coeff, p->f_offs, p->f_idx, flat, wrt_col, n_cols, p->n_gates, tmp,
                         ims, grad_out);
}

/* gradients.py:84-99 (pack_expectations); returns nonzero if |Im| > 1e-10 */
static int pack_expectations(const OrcProblem* p, const cplx* psi, double* out) {
  for (int64_t i = 0; i < p->n_obs; ++i) {
    double v[2];
    orc_expval_terms((const double*)psi, (int)p->n_qubits, p->t_coeffs, p->t_xmask, p->t_smask,
                     p->t_phases, p->term_offs[i], p->term_offs[i + 1], v);
    if (fabs(v[1]) > 1e-10) return 1;
    out[i] = v[0];
  }
  return 0;
}

/* batch.py:54-72 (split_workload): contiguous ranges, the first B - T*floor(B/T)
 * ranges one larger. */
static void split_range(int64_t B, int T, int t, int64_t* lo, int64_t* hi) {
  const int64_t base = B / T, extra = B - (int64_t)T * base;
  const int64_t start = t * base + (t < extra ? t : extra);
  *lo = start;
  *hi = start + base + (t < extra ? 1 : 0);
}

/*
 * batch.py:147-217 (BatchEngine.run_batch, method="adjoint"): one row per
 * encoding input; the encoding slice of base_flat is overwritten per row.
 * grad_out is (B, M, n_cols) zero-initialised by this call; forward-only when
 * n_cols == 0. Rows are split over `threads` OpenMP threads exactly like the
 * reference's thread pool, so results are bit-identical for every thread
 * count. Returns -1 - row on a hermiticity failure in the forward-only path.
 */
int orc_run_batch(const OrcProblem* p, const double* base_flat, int64_t enc_off, int64_t enc_size,
                  const double* inputs, int64_t B, const int64_t* wrt_col, int64_t n_cols,
                  int threads, double* expect_out, double* grad_out) {
  if (B == 0 || p->n_obs == 0) return 0;
  if (threads < 1) threads = 1;
  if (threads > B) threads = (int)B;
  const int64_t dim = (int64_t)1 << p->n_qubits;
  int failed_row = -1;
  memset(grad_out, 0, sizeof(double) * (size_t)(B * p->n_obs * n_cols));
#pragma omp parallel num_threads(threads)
  {
#ifdef _OPENMP
    extern int omp_get_thread_num(void);
    const int t = omp_get_thread_num();
#else
    const int t = 0;
#endif
    int64_t lo, hi;
    split_range(B, threads, t, &lo, &hi);
    cplx* work = (cplx*)malloc(sizeof(cplx) * (size_t)dim * (size_t)(p->n_obs + 2));
    double* flat = (double*)malloc(sizeof(double) * (size_t)(p->total_params + 1));
    double* angles = (double*)malloc(sizeof(double) * (size_t)(p->n_gates + 1));
    double* ims = (double*)malloc(sizeof(double) * (size_t)(p->n_obs + 1));
    memcpy(flat, base_flat, sizeof(double) * (size_t)p->total_params);
    for (int64_t b = lo; b < hi; ++b) {
      memcpy(flat + enc_off, inputs + b * enc_size, sizeof(double) * (size_t)enc_size);
      if (n_cols == 0) {
        orc_compute_angles(p->coeff, p->f_offs, p->f_idx, flat, p->n_gates, angles);
        memset(work, 0, sizeof(cplx) * (size_t)dim);
        work[0].re = 1.0;
        orc_run_program((double*)work, (int)p->n_qubits, p->kinds, p->q0, p->q1, angles, p->n_gates);
        if (pack_expectations(p, work, expect_out + b * p->n_obs)) {
#pragma omp critical
          { if (failed_row < 0 || b < failed_row) failed_row = (int)b; }
        }
      } else {
        adjoint_flat(p, flat, wrt_col, n_cols, expect_out + b * p->n_obs,
                     grad_out + b * p->n_obs * n_cols, work, angles, ims);
      }
    }
    free(work); free(flat); free(angles); free(ims);
  }
  return failed_row >= 0 ? -1 - failed_row : 0;
}

/* one forward evolution from |0..0> (circuit.py:229-238) */
void orc_evolve(const OrcProblem* p, const double* flat, double* state_out) {
  const int64_t dim = (int64_t)1 << p->n_qubits;
  double* angles = (double*)malloc(sizeof(double) * (size_t)(p->n_gates + 1));
  orc_compute_angles(p->coeff, p->f_offs, p->f_idx, flat, p->n_gates, angles);
  memset(state_out, 0, sizeof(cplx) * (size_t)dim);
  state_out[0] = 1.0;
  orc_run_program(state_out, (int)p->n_qubits, p->kinds, p->q0, p->q1, angles, p->n_gates);
  free(angles);
}

/* gate-level entry points used by the known-answer tests (statevector.py:404-420) */
void orc_apply_gate(double* state, int n_qubits, int64_t kind, int64_t q0, int64_t q1, double angle,
                    int adjoint) {
  const int64_t dim = (int64_t)1 << n_qubits;
  if (adjoint) apply_coded_adjoint((cplx*)state, dim, kind, q0, q1, angle);
  else apply_coded((cplx*)state, dim, kind, q0, q1, angle);
}
