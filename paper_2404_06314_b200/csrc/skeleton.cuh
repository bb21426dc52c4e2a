// Kernel skeletons shared by the prebuilt interpreter kernels (engine.cu) and
// the per-plan JIT kernels (jit.cpp): staging, expectations / adjoint seed,
// tile load / store. The segment work is a policy (SEGS::run<R, MODE>):
// InterpSegs decodes the device program at run time, a JIT policy is
// straight-line code with every operand a compile-time constant.
#pragma once
#include "kernels.cuh"

namespace vqc {

// Observable terms staged in shared memory (Z strings only on this path).
struct TermSm {
  uint32_t mask;   // sign mask (Y/Z letters)
  int32_t obs;     // observable index
  uint32_t xmask;  // flip mask (X/Y letters); 0 for Z strings
  int32_t phase;   // i^phase = i^{#Y}
  double coeff;
};

__device__ __forceinline__ void stage_terms(const DevProgram& D, TermSm* s_terms) {
  for (int t = vtid(); t < D.T; t += vdim()) {
    TermSm ts;
    ts.mask = D.t_smask[t];
    ts.xmask = D.t_xmask[t];
    ts.phase = D.t_phase[t];
    ts.coeff = D.t_coeff[t];
    ts.obs = D.t_obs[t];
    s_terms[t] = ts;
  }
}

// In-place Walsh-Hadamard transform of a thread's E values (natural order):
// W[h] = sum_i (-1)^{popc(i & h)} v[i]. A Z string's sign over a thread's
// elements is (-1)^{p0 ^ popc(i & h)} with h the same for every thread of the
// tile, so its sum over them is +-W[h], and the adjoint seed's weights are the
// transform of the per-h sums of the term coefficients.
template <int E>
__device__ __forceinline__ void wht(double (&v)[E]) {
#pragma unroll
  for (int len = 1; len < E; len <<= 1) {
#pragma unroll
    for (int i = 0; i < E; ++i)
      if (!(i & len)) {
        const double a = v[i], b = v[i | len];
        v[i] = a + b;
        v[i | len] = a - b;
      }
  }
}
// v[h] with a run-time (tile-uniform) h: a uniform branch, no local memory
template <int E>
__device__ __forceinline__ double pick(const double (&v)[E], uint32_t h) {
  double r = v[0];
#pragma unroll
  for (int i = 1; i < E; ++i)
    if (h == (uint32_t)i) r = v[i];
  return r;
}
template <int E>
__device__ __forceinline__ void add_at(double (&v)[E], uint32_t h, double x) {
#pragma unroll
  for (int i = 0; i < E; ++i)
    if (h == (uint32_t)i) v[i] += x;
}

// Observable terms known at compile time (JIT pass kernels emit a struct with
// the same members and kConst = true); RtTerms: read from shared memory.
struct RtTerms {
  static constexpr bool kConst = false;
  static constexpr int T = 0, M = 0;
  __device__ static constexpr uint32_t mask(int) { return 0u; }
  __device__ static constexpr double coeff(int) { return 0.0; }
  __device__ static constexpr int off(int) { return 0; }
};

// Expectations (observables.py / _kernels.py:182-198, Z strings) and the
// adjoint seed phi = w(j) psi with w = sum_m u_m O_m(j) (VJP) or O_bra(j)
// (_kernels.py:209-217). Each thread owns `count` tile elements; a term's
// sign over them is parity(base & s) ^ parity(i & h), h bit b =
// parity(hi[b] & s), so no per-element index arithmetic is needed.
// E: elements per thread (compile time; equals the tile walk's count)
template <bool DUAL, int E, class PM = RtPassMap, class TMS = RtTerms>
__device__ __forceinline__ void observe(const DevProgram& D, const RunArgs& A, const PassDesc* pd, cplx_t* s_psi,
                                        cplx_t* s_phi, const double* s_u_row, const TermSm* s_terms,
                                        const Group& grp, double* s_red, double* s_fin, uint32_t tile_base, int k,
                                        int64_t bl0, bool do_expect, int seed_mode, int bra, int tile,
                                        int n_tiles) {
  const int lane = grp.lane_in_sample();
  const TileWalk tw = tile_walk<PM>(pd, tile_base, k, lane, grp.TT);
  const int count = tw.count;
  constexpr int EB = ctz_const(E);  // element-index bits of a thread
  auto term_bits = [&](uint32_t mask, uint32_t& p0, uint32_t& h) {
    p0 = (uint32_t)__popc(tw.base & mask) & 1u;
    h = 0;
#pragma unroll
    for (int b = 0; b < EB; ++b) h |= ((uint32_t)__popc(tw.hi[b] & mask) & 1u) << b;
  };
  if (do_expect) {
    double p2[E];
#pragma unroll
    for (int i = 0; i < E; ++i) {
      p2[i] = 0.0;
      if (i < count) {
        VQC_CHECK(A, swz((uint32_t)lane + (uint32_t)i * (uint32_t)grp.TT) < (1u << k), CHK_OBSERVE);
        const cplx_t x = s_psi[swz((uint32_t)lane + (uint32_t)i * (uint32_t)grp.TT)];
        const double xr = x.x, xi = x.y;   // |psi_j|^2 in float64 for either state type
        p2[i] = xr * xr + xi * xi;
      }
    }
    double wh[E];
#pragma unroll
    for (int i = 0; i < E; ++i) wh[i] = p2[i];
    wht<E>(wh);
    if constexpr (TMS::kConst) {
      // constant masks: h and the pick fold, one accumulator and store per observable
#pragma unroll
      for (int m = 0; m < TMS::M; ++m) {
        double acc = 0.0;
#pragma unroll
        for (int t = TMS::off(m); t < TMS::off(m + 1); ++t) {
          uint32_t p0, h;
          term_bits(TMS::mask(t), p0, h);
          const double v = pick<E>(wh, h);
          acc += TMS::coeff(t) * (p0 ? -v : v);
        }
        s_red[m * (int)vdim() + vtid()] = acc;
      }
    } else {
    for (int m = 0; m < D.M; ++m) s_red[m * (int)vdim() + vtid()] = 0.0;
    for (int t = 0; t < D.T; ++t) {
      const TermSm ts = s_terms[t];
      if (ts.xmask != 0u) continue;
      uint32_t p0, h;
      term_bits(ts.mask, p0, h);
      const double v = pick<E>(wh, h);
      s_red[ts.obs * (int)vdim() + vtid()] += ts.coeff * (p0 ? -v : v);
    }
    }
    if (D.has_xy) {
      // X/Y strings (on-chip states only): Re sum_j conj(psi_j) i^k (-1)^{popc((j^x)&s)} psi_{j^x}
      for (int t = 0; t < D.T; ++t) {
        const TermSm ts = s_terms[t];
        if (ts.xmask == 0u) continue;
        double v = 0.0;
        for (int i = 0; i < count; ++i) {
          const uint32_t l = (uint32_t)lane + (uint32_t)i * (uint32_t)grp.TT;
          const uint32_t kx = l ^ ts.xmask;
          const cplx_t ca = s_psi[swz(l)], cb = s_psi[swz(kx)];
          const double ax = ca.x, ay = ca.y, bx = cb.x, by = cb.y;
          // conj(a) * bq
          double re = ax * bx + ay * by, im = ax * by - ay * bx;
          const int ph = ts.phase & 3;  // multiply by i^ph, keep the real part
          double r = ph == 0 ? re : ph == 1 ? -im : ph == 2 ? -re : im;
          v += (__popc(kx & ts.mask) & 1) ? -r : r;
        }
        s_red[ts.obs * (int)vdim() + vtid()] += ts.coeff * v;
      }
    }
    vsync();
    const int warp = vtid() >> 5, lane32 = vtid() & 31, nwarp = (vdim() + 31) >> 5;
    const bool narrow = vdim() < 32;
    for (int task = warp; task < D.M * grp.S; task += nwarp) {
      const int m = task / grp.S, s_ = task - m * grp.S;
      const double* base = s_red + m * (int)vdim() + s_ * grp.TT;
      double v = 0.0;
      if (narrow) {
        if (lane32 == 0)
          for (int t = 0; t < grp.TT; ++t) v += base[t];
      } else {
        for (int t = lane32; t < grp.TT; t += 32) v += base[t];
        for (int off = 16; off > 0; off >>= 1) v += __shfl_xor_sync(0xffffffffu, v, off);
      }
      const int64_t bl = bl0 + s_;
      if (lane32 == 0 && bl < A.nb) A.expect[(bl * D.M + m) * n_tiles + tile] = v;
    }
    vsync();
  }
  if constexpr (DUAL) {
    if (seed_mode != 0) {
      double w[E];
#pragma unroll
      for (int i = 0; i < E; ++i) w[i] = 0.0;
      if constexpr (TMS::kConst) {
#pragma unroll
        for (int m = 0; m < TMS::M; ++m) {
          const double um = seed_mode == 1 ? s_u_row[m] : (m == bra ? 1.0 : 0.0);
#pragma unroll
          for (int t = TMS::off(m); t < TMS::off(m + 1); ++t) {
            uint32_t p0, h;
            term_bits(TMS::mask(t), p0, h);
            const double e = um * TMS::coeff(t);
            add_at<E>(w, h, p0 ? -e : e);
          }
        }
      } else {
      for (int t = 0; t < D.T; ++t) {
        const TermSm ts = s_terms[t];
        if (ts.xmask != 0u) continue;
        const double e = seed_mode == 1 ? s_u_row[ts.obs] * ts.coeff : (ts.obs == bra ? ts.coeff : 0.0);
        if (e == 0.0) continue;
        uint32_t p0, h;
        term_bits(ts.mask, p0, h);
        add_at<E>(w, h, p0 ? -e : e);
      }
      }
      wht<E>(w);  // w[i] = sum_h (-1)^{popc(i & h)} (per-h sums)
#pragma unroll
      for (int i = 0; i < E; ++i) {
        if (i >= count) break;
        const uint32_t l = (uint32_t)lane + (uint32_t)i * (uint32_t)grp.TT;
        const uint32_t p = swz(l);
        const cplx_t x = s_psi[p];
        double2 phi = make_double2(w[i] * (double)x.x, w[i] * (double)x.y);
        if (D.has_xy) {
          // pauli_sum_apply (_kernels.py:166-179) for the X/Y strings
          for (int t = 0; t < D.T; ++t) {
            const TermSm ts = s_terms[t];
            if (ts.xmask == 0u) continue;
            const double e = seed_mode == 1 ? s_u_row[ts.obs] * ts.coeff : (ts.obs == bra ? ts.coeff : 0.0);
            if (e == 0.0) continue;
            const uint32_t kx = l ^ ts.xmask;
            const double2 bq = make_double2((double)s_psi[swz(kx)].x, (double)s_psi[swz(kx)].y);
            const int ph = ts.phase & 3;
            double2 v = ph == 0 ? bq : ph == 1 ? make_double2(-bq.y, bq.x)
                      : ph == 2 ? make_double2(-bq.x, -bq.y) : make_double2(bq.y, -bq.x);
            const double sg = (__popc(kx & ts.mask) & 1) ? -e : e;
            phi.x += sg * v.x;
            phi.y += sg * v.y;
          }
        }
        s_phi[p] = mk_c((real_t)phi.x, (real_t)phi.y);
      }
    }
  }
}

// Shared-memory carve-up (kernels and host sizing must agree).
struct SmemLayout {
  size_t psi, phi, cs, u, av, red, fin, up, terms, total;  // byte offsets
  // esz: bytes per state element (16 complex128, 8 complex64)
  __host__ __device__ SmemLayout(int S, int n_amp, bool dual, int nrot, int nblk, int nav, int red_slots,
                                 int threads, int M, int n_terms, int esz) {
    size_t o = 0;
    psi = o; o += (size_t)S * n_amp * esz;
    phi = o; o += dual ? (size_t)S * n_amp * esz : 0;
    cs = o; o += (size_t)S * nrot * 16;
    u = o; o += (size_t)S * nblk * 64;
    av = o; o += (size_t)S * nav * 32;
    red = o; o += (size_t)red_slots * threads * 8;
    fin = o; o += (size_t)2 * red_slots * S * 8;  // two buffers (lagged JIT reductions)
    up = o; o += (size_t)S * M * 8;
    terms = o; o += (size_t)n_terms * sizeof(TermSm);
    total = (o + 16 + 127) & ~(size_t)127;  // 128-byte aligned: ping-pong groups sit back to back
  }
};

// kernel modes: forward only / adjoint with both states per thread (small n) /
// adjoint split over (psi, phi) thread pairs
enum { KM_FWD = 0, KM_DUAL = 1, KM_SPLIT = 2 };

template <int R, int KM>
__device__ __forceinline__ Group make_group(int threads_per_role, int samples) {
  Group g;
  g.tid = vtid();
  g.TPS = threads_per_role;
  g.TT = KM == KM_SPLIT ? 2 * threads_per_role : threads_per_role;
  g.S = samples;
  const int lane = vtid() % g.TT;
  g.sl = vtid() / g.TT;
  g.role = lane / g.TPS;
  g.gi = lane % g.TPS;
  g.W = g.TT >= 32 ? g.TT >> 5 : 1;
  return g;
}

// Whole state on chip: one CTA owns S samples of n <= 12 qubits and runs
// forward, expectations, seed and the adjoint sweep without touching HBM.
__host__ __device__ constexpr int smem_max_threads(int R, int KM) {
  return R >= 5 ? 256 : (KM == KM_SPLIT ? 512 : (R >= 4 ? 256 : 512));
}
__host__ __device__ constexpr int pass_max_threads(int R) { return R >= 5 ? 256 : 512; }

template <int R, int KM, class SEGS>
__device__ __forceinline__ void smem_body(const DevProgram& D, const RunArgs& A) {
  constexpr int OBS_E = KM == KM_SPLIT ? (1 << (R - 1)) : (1 << R);
  extern __shared__ __align__(16) unsigned char smem_raw[];
  constexpr bool ADJ = KM != KM_FWD;
  constexpr int BM = KM == KM_SPLIT ? MODE_SPLIT : MODE_DUAL;
  const int n = D.n, N = 1 << n;
  const Group grp = make_group<R, KM>(1 << (n - R), A.S);
  const int lane = grp.lane_in_sample();
  const int64_t bl0 = (int64_t)blockIdx.x * A.S;
  const int64_t bl = bl0 + grp.sl;
  const bool valid = bl < A.nb;
  const int64_t b = A.b0 + (valid ? bl : 0);
  const PassDesc* pd = D.passes;
  const int nrot = D.n_rot, nblk = D.n_blk, nav = D.n_av;
  const SmemLayout L(A.S, N, ADJ, nrot, nblk, nav, A.red_slots, (int)blockDim.x, D.M, D.T, (int)sizeof(cplx_t));
  cplx_t* s_psi = reinterpret_cast<cplx_t*>(smem_raw + L.psi) + (size_t)grp.sl * N;
  cplx_t* s_phi = reinterpret_cast<cplx_t*>(smem_raw + L.phi) + (size_t)grp.sl * N;
  double2* s_cs = reinterpret_cast<double2*>(smem_raw + L.cs) + (size_t)grp.sl * nrot;
  double2* s_u = reinterpret_cast<double2*>(smem_raw + L.u) + (size_t)grp.sl * nblk * 4;
  double* s_av_all = reinterpret_cast<double*>(smem_raw + L.av);
  double* s_red = reinterpret_cast<double*>(smem_raw + L.red);
  double* s_fin = reinterpret_cast<double*>(smem_raw + L.fin);
  double* s_up = reinterpret_cast<double*>(smem_raw + L.up);
  TermSm* s_terms = reinterpret_cast<TermSm*>(smem_raw + L.terms);
  stage_terms(D, s_terms);

  for (int l = lane; l < N; l += grp.TT) s_psi[swz((uint32_t)l)] = mk_c(l == 0 ? 1 : 0, 0);
  if (ADJ && A.upstream != nullptr)
    for (int m = lane; m < D.M; m += grp.TT) s_up[grp.sl * D.M + m] = valid ? A.upstream[b * D.M + m] : 0.0;
  if (A.tables != nullptr) {
    // per-sample tables precomputed by k_tables: [cs | u | av] of this sample
    const double* t = A.tables + (size_t)(valid ? bl : 0) * A.table_stride;
    double* dcs = reinterpret_cast<double*>(s_cs);
    double* du = reinterpret_cast<double*>(s_u);
    double* dav = s_av_all + (size_t)grp.sl * nav * 4;
    for (int i = lane; i < 2 * nrot; i += grp.TT) dcs[i] = t[i];
    for (int i = lane; i < 8 * nblk; i += grp.TT) du[i] = t[2 * nrot + i];
    for (int i = lane; i < 4 * nav; i += grp.TT) dav[i] = t[2 * nrot + 8 * nblk + i];
    __syncthreads();
  } else {
    build_tables(D, A, pd, b, valid, s_cs, s_u, s_av_all + (size_t)grp.sl * nav * 4, lane, grp.TT);
  }
  const SampleTables T{s_cs, s_u, 0, 0};

  SEGS::template run<R, MODE_FWD>(make_env<MODE_FWD>(D, A, s_psi, s_psi, s_av_all, nav * 4, 0, s_red, s_fin,
                            grp, grp.role == 0, 0u, bl0, 0, 0, 1), T, pd->seg_begin, pd->seg_end);
  if constexpr (!ADJ) {
    observe<false, OBS_E>(D, A, nullptr, s_psi, s_psi, nullptr, s_terms, grp, s_red, s_fin, 0u, n, bl0, true, 0, 0, 0, 1);
  } else {
    if (!A.jacobian) {
      observe<true, OBS_E>(D, A, nullptr, s_psi, s_phi, s_up + grp.sl * D.M, s_terms, grp, s_red, s_fin, 0u, n, bl0,
                    A.expect != nullptr, 1, 0, 0, 1);
      __syncthreads();
      SEGS::template run<R, BM>(make_env<BM>(D, A, s_psi, s_phi, s_av_all, nav * 4, 0, s_red, s_fin,
                          grp, true, 0u, bl0, 0, 0, 1), T, pd->bseg_begin, pd->bseg_end);
    } else {
      observe<true, OBS_E>(D, A, nullptr, s_psi, s_phi, nullptr, s_terms, grp, s_red, s_fin, 0u, n, bl0,
                    A.expect != nullptr, 0, 0, 0, 1);
      cplx_t* fin = A.psi_fin + (size_t)bl * N;
      if (D.M > 1 && valid)
        for (int l = lane; l < N; l += grp.TT) fin[l] = s_psi[swz((uint32_t)l)];
      for (int m = 0; m < D.M; ++m) {
        if (m > 0) {
          __syncthreads();
          if (valid)
            for (int l = lane; l < N; l += grp.TT) s_psi[swz((uint32_t)l)] = fin[l];
        }
        observe<true, OBS_E>(D, A, nullptr, s_psi, s_phi, nullptr, s_terms, grp, s_red, s_fin, 0u, n, bl0, false, 2, m,
                      0, 1);
        __syncthreads();
        SEGS::template run<R, BM>(make_env<BM>(D, A, s_psi, s_phi, s_av_all, nav * 4, 0,
                            s_red, s_fin, grp, true, 0u, bl0, m, 0, 1), T, pd->bseg_begin, pd->bseg_end);
      }
    }
  }
}

__device__ __forceinline__ void cp_async16(void* smem_dst, const void* gmem_src) {
  const uint32_t d = (uint32_t)__cvta_generic_to_shared(smem_dst);
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16;\n" ::"r"(d), "l"(gmem_src) : "memory");
}
__device__ __forceinline__ void cp_async_wait_all() { asm volatile("cp.async.wait_all;\n" ::: "memory"); }
__device__ __forceinline__ void cp_async_wait_all_() { cp_async_wait_all(); }  // declared in kernels.cuh (seg_begin_io)
// one state element (16 B complex128 through L2 only; 8 B complex64)
__device__ __forceinline__ void cp_async_elem(cplx_t* smem_dst, const cplx_t* gmem_src) {
#ifdef VQC_C64
  const uint32_t d = (uint32_t)__cvta_generic_to_shared(smem_dst);
  asm volatile("cp.async.ca.shared.global [%0], [%1], 8;\n" ::"r"(d), "l"(gmem_src) : "memory");
#else
  cp_async16(smem_dst, gmem_src);
#endif
}

// One pass over HBM-resident states: CTA (tile, row) stages 2^k amplitudes.
template <int R, int KM, class SEGS>
__device__ __forceinline__ void pass_body(const DevProgram& D, const RunArgs& A) {
  constexpr int OBS_E = KM == KM_SPLIT ? (1 << (R - 1)) : (1 << R);
  constexpr int BMP = KM == KM_SPLIT ? MODE_SPLIT : MODE_DUAL;  // adjoint segments
  extern __shared__ __align__(16) unsigned char smem_raw[];
  constexpr bool ADJ = KM != KM_FWD;
  using PM = typename SEGS::PM;
  const PassDesc* pd = D.passes + A.pass;
  const int k = PM::kConst ? PM::k : pd->k, Nt = 1 << k;
  // threads per tile (the walk stride): compile time for JIT pass maps
  const int wstride = PM::kConst ? ((KM == KM_SPLIT ? 2 : 1) << (PM::k - R)) : (int)vdim();
  const uint32_t flags = A.flags;
  const Group grp = make_group<R, KM>(1 << (k - R), 1);
  // ping-pong kernels: CTA x holds tiles kCtaGroups * x + group
  const int tile = (int)(blockIdx.x * kCtaGroups + cta_group()), n_tiles = (int)gridDim.x * kCtaGroups;
  const int64_t bl = blockIdx.y;
  const int64_t b = A.b0 + bl;
  const size_t N = (size_t)1 << D.n;
  const uint32_t tile_base = PM::tile_dep(pd, D.n, (uint32_t)tile);
  const SmemLayout L(1, Nt, ADJ, D.max_rot_pass, D.max_blk_pass, D.max_av_pass, A.red_slots, (int)vdim(),
                     D.M, D.T, (int)sizeof(cplx_t));
  unsigned char* const smem_grp = smem_raw + (size_t)cta_group() * L.total;  // this group's carve-up
  cplx_t* s_psi = reinterpret_cast<cplx_t*>(smem_grp + L.psi);
  cplx_t* s_phi = reinterpret_cast<cplx_t*>(smem_grp + L.phi);
  double2* s_cs = reinterpret_cast<double2*>(smem_grp + L.cs);
  double2* s_u = reinterpret_cast<double2*>(smem_grp + L.u);
  double* s_av = reinterpret_cast<double*>(smem_grp + L.av);
  double* s_red = reinterpret_cast<double*>(smem_grp + L.red);
  double* s_fin = reinterpret_cast<double*>(smem_grp + L.fin);
  double* s_up = reinterpret_cast<double*>(smem_grp + L.up);
  TermSm* s_terms = reinterpret_cast<TermSm*>(smem_grp + L.terms);
  if (flags & (F_OBSERVE | F_SEED)) stage_terms(D, s_terms);

  long long tdbg = A.dbg ? clock64() : 0;
  if (A.dbg && vtid() == 0) atomicAdd(A.dbg + DBG_CTAS, 1ull);
  turn_init();
  if (ADJ && (flags & F_SEED) && A.bra < 0)
    for (int m = vtid(); m < D.M; m += vdim()) s_up[m] = A.upstream[b * D.M + m];
  // direct tile I/O (kernels.cuh IO_*): which sweep's first / last segment
  // exchanges its registers with HBM instead of the shared-memory tile
  uint32_t io_f = 0, io_b = 0;
  // (per sweep end: the JIT allows it where a warp's accesses coalesce)
  if ((flags & F_FWD) && pd->seg_end > pd->seg_begin) {
    if constexpr (SEGS::kDioF)
      if (flags & F_INIT) io_f |= IO_INIT;
    if constexpr (SEGS::kDioFL)
      if (!(flags & F_INIT) && (flags & F_LOAD_PSI) && !(flags & F_LOAD_FIN)) io_f |= IO_LD;
    if constexpr (SEGS::kDioFS)
      if ((flags & F_STORE_PSI) && !(flags & (F_STORE_FIN | F_OBSERVE | F_SEED | F_BWD))) io_f |= IO_ST;
  }
  if constexpr (ADJ) {
    if ((flags & F_BWD) && pd->bseg_end > pd->bseg_begin) {
      if constexpr (SEGS::kDioBL)
        if (!(flags & (F_FWD | F_OBSERVE | F_SEED | F_INIT | F_LOAD_FIN)) && (flags & F_LOAD_PSI) && (flags & F_LOAD_PHI))
          io_b |= IO_LD;
      if constexpr (SEGS::kDioBS)
        if ((flags & F_STORE_PSI) && (flags & F_STORE_PHI)) io_b |= IO_ST;
      if constexpr (SEGS::kDioB)
        if (!(flags & (F_STORE_PSI | F_STORE_PHI))) io_b |= IO_NOST;
    }
  }
  const bool direct_first = ((io_f | io_b) & (IO_LD | IO_INIT)) != 0u;
  if (direct_first) {
    // the first segment fills its registers itself
  } else if (flags & F_INIT) {
    for (int l = vtid(); l < Nt; l += vdim())
      s_psi[swz((uint32_t)l)] = mk_c((tile_base == 0 && l == 0) ? 1 : 0, 0);
  } else {
    // asynchronous 16-byte copies straight into the swizzled tile; they land
    // while the per-sample tables are built
    const cplx_t* src = ((flags & F_LOAD_FIN) ? A.psi_fin : A.psi) + (size_t)bl * N;
    const cplx_t* srcf = A.phi + (size_t)bl * N;
    const bool lphi = ADJ && (flags & F_LOAD_PHI);
    const TileWalk tw = tile_walk<PM>(pd, tile_base, k, vtid(), wstride);
    for_tile<OBS_E>(tw, [&](uint32_t sw, uint32_t j) {
      VQC_CHECK(A, j < (uint32_t)N, CHK_TILE_GLOBAL);
      VQC_CHECK(A, sw < (uint32_t)Nt, CHK_TILE_SMEM);
      cp_async_elem(s_psi + sw, src + j);
      if (lphi) cp_async_elem(s_phi + sw, srcf + j);
    });
  }
  if (A.tables != nullptr) {
    // per-sample tables precomputed by k_tables: copy this pass's slices
    const double* t = A.tables + (size_t)bl * A.table_stride;
    const int nrot = pd->rot_end - pd->rot_begin, nblk = pd->blk_end - pd->blk_begin,
              nav = pd->av_end - pd->av_begin;
    const double* tcs = t + 2 * pd->rot_begin;
    const double* tu = t + 2 * (size_t)D.n_rot + 8 * (size_t)pd->blk_begin;
    const double* tav = t + 2 * (size_t)D.n_rot + 8 * (size_t)D.n_blk + 4 * (size_t)pd->av_begin;
    for (int i = vtid(); i < nrot; i += vdim()) cp_async16(s_cs + i, tcs + 2 * i);
    for (int i = vtid(); i < 4 * nblk; i += vdim()) cp_async16(s_u + i, tu + 2 * i);
    for (int i = vtid(); i < 2 * nav; i += vdim()) cp_async16(s_av + 2 * i, tav + 2 * i);
  } else {
    build_tables(D, A, pd, b, true, s_cs, s_u, s_av, vtid(), vdim());
  }
  if (!direct_first) {  // else awaited by the first segment, behind its own loads (seg_begin_io)
    cp_async_wait_all();
    vsync();
  }
  dbg_add(A, DBG_PROLOGUE, tdbg);
  const SampleTables T{s_cs, s_u, pd->rot_begin, pd->blk_begin};
  if (flags & F_FWD) {
    SegEnv env = make_env<MODE_FWD>(D, A, s_psi, s_psi, s_av, 0, pd->av_begin, s_red, s_fin,
                                    grp, grp.role == 0, tile_base, bl, 0, tile, n_tiles);
    env.io = io_f;
    env.g_psi = A.psi + (size_t)bl * N;
    SEGS::template run<R, MODE_FWD>(env, T, pd->seg_begin, pd->seg_end);
  }
  dbg_add(A, DBG_FWD, tdbg);
  if (flags & F_STORE_FIN) {
    uint32_t tb = tile_base;
    asm volatile("" : "+r"(tb));
    const TileWalk tw = tile_walk<PM>(pd, tb, k, vtid(), wstride);
    cplx_t* dst = A.psi_fin + (size_t)bl * N;
    for_tile<OBS_E>(tw, [&](uint32_t sw, uint32_t j) { dst[j] = s_psi[sw]; });
  }
  if (flags & (F_OBSERVE | F_SEED)) {
    observe<ADJ, OBS_E, PM, typename SEGS::Terms>(D, A, pd, s_psi, s_phi, s_up, s_terms, grp, s_red, s_fin, tile_base, k, bl, (flags & F_OBSERVE) != 0,
                 (flags & F_SEED) ? (A.bra < 0 ? 1 : 2) : 0, A.bra, tile, n_tiles);
    vsync();
  }
  dbg_add(A, DBG_OBSERVE, tdbg);
  if constexpr (ADJ) {
    if (flags & F_BWD) {
      SegEnv env = make_env<BMP>(D, A, s_psi, s_phi, s_av, 0, pd->av_begin,
                                 s_red, s_fin, grp, true, tile_base, bl, A.bra < 0 ? 0 : A.bra, tile, n_tiles);
      env.io = io_b;
      env.g_psi = A.psi + (size_t)bl * N;
      env.g_phi = A.phi + (size_t)bl * N;
      SEGS::template run<R, BMP>(env, T, pd->bseg_begin, pd->bseg_end);
    }
  }
  dbg_add(A, DBG_BWD, tdbg);
  const bool sphi = ADJ && (flags & F_STORE_PHI);
  if (((flags & F_STORE_PSI) || sphi) && !((io_f | io_b) & IO_ST)) {
    asm volatile("" ::: "memory");
    uint32_t tb = tile_base;
    asm volatile("" : "+r"(tb));  // rebuild the tile walk here rather than keep it live
    const TileWalk tw = tile_walk<PM>(pd, tb, k, vtid(), wstride);
    const bool spsi = (flags & F_STORE_PSI) != 0;
    cplx_t* dst = A.psi + (size_t)bl * N;
    cplx_t* dstf = A.phi + (size_t)bl * N;
    for_tile<OBS_E>(tw, [&](uint32_t sw, uint32_t j) {
      VQC_CHECK(A, j < (uint32_t)N && sw < (uint32_t)Nt, CHK_TILE_GLOBAL);
      if (spsi) dst[j] = s_psi[sw];
      if (sphi) dstf[j] = s_phi[sw];
    });
  }
  dbg_add(A, DBG_STORE, tdbg);
  turn_fini();
}

}  // namespace vqc
