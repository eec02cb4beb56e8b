// stencil.cuh -- variable-coefficient operator, included
// at the end of bspde_b200.cu (shares the CG state machine and reductions).
//
// The reference's on-the-fly operator (operator.py:217-229 over
// stencil_block, assembly.py:460-472) builds, per node l, the (2p+1)^3
// stencil
//
//   P[a, l] = sum_terms s_term sum_b f_term[l + b] Tz[az, bz] Ty[ay, by] Tx[ax, bx]
//
// from per-axis trilinear tables (kernels.py:158-173, positional edge rows
// assembly.py:83-108) and the parameter fields (diffusion for the three
// stiffness terms, absorption for the mass term), then applies
// t_l = sum_a P[a, l] c[l + a].  Here the stencil is assembled once into HBM
// (structure of arrays: P[a * N + l], coalesced in l) by stencil_assemble_kernel
// and applied by a streaming gather (stencil_apply_kernel) -- the B200
// counterpart of the reference's "sparse" strategy, sized for up to ~300^3
// per GPU (2.7 KB per DoF at p = 3).  Jacobi-PCG runs the reference
// recurrence with three kernels per iteration (p formation, apply + <p,Ap>,
// x/r update + dots) and the same device-side scalar state as the
// constant-coefficient solver.

namespace {

// per-thread accumulation of the stencil PCG's dot products: double-double
// (BSPDE_ST_DD=1, correctly rounded with the dd tree) or plain FMAs
#ifndef BSPDE_ST_DD
#define BSPDE_ST_DD 1
#endif
#if BSPDE_ST_DD
#define ST_ACC(h, l, a, b) dd_add(h, l, __dmul_rn(a, b))
#else
#define ST_ACC(h, l, a, b) (h = fma(a, b, h))
#endif

constexpr int ST_NT = 256;

struct StencilDev {
  int nb, np, A, B, mw;     // A = 2nb+1 trial offsets, B = 2mw+1 parameter offsets
  int nz, ny, nx;           // coefficient extents (dense arrays)
  int pz, py, px;           // parameter-field extents
  int ext, ext_p;
  int ew[3];
  long long N;              // nz*ny*nx
  double s_stiff[3], s_mass;
  const double* tab;        // [axis][d][class][A][B] (class stride 2*EWMAX+1)
  int ncls;                 // class stride
  // box faces: P += w (v v^T)_axis (x) (h M)_others
  int nfaces;
  int face_axis[6], face_side[6];
  double face_weight[6];
  double fv[MAXP + 1];          // low-face values (ew entries)
  double gram[11 * 11];         // unit mass Gram class table (2ew+1) x (2nb+1)
  double step[3];
  int degen[3];             // unit axes of 1-D / 2-D problems (no extension)
  int ex[3], exp_[3];       // per-axis ext / ext_p (0 on unit axes)
  // compact mode (mask domains): only the active rows are stored and
  // iterated, P[a * nact + k] for active row k = dense index rows[k]
  // (ascending); vectors stay dense, inactive entries are never touched
  const int64_t* rows;
  long long nact;
};

// rows iterated by the row-wise kernels (all nodes, or the active rows)
__device__ __forceinline__ long long st_nrows(const StencilDev& S) {
  return S.rows ? S.nact : S.N;
}
__device__ __forceinline__ long long st_row(const StencilDev& S, long long k) {
  return S.rows ? S.rows[k] : k;
}

__device__ __forceinline__ double st_face_value(const StencilDev& S, int i, int n, int side) {
  const int ew = (S.ncls - 1) / 2;  // == edge_width(n_b) for face tables
  if (side == 0) return i >= 0 && i < ew ? S.fv[i] : 0.0;
  const int m = n - 1 - i;
  return m >= 0 && m < ew ? S.fv[m] : 0.0;
}

__device__ __forceinline__ int st_cls(int i, int n, int ew) {
  return i < ew ? i : (i >= n - ew ? 2 * ew - (n - 1 - i) : ew);
}

__device__ __forceinline__ const double* st_tab(const StencilDev& S, const double* tab, int axis,
                                                int d, int cls) {
  return tab + ((((long long)axis * 2 + d) * S.ncls + cls) * S.A) * S.B;
}

// one thread per (entry a, node l): consecutive threads = consecutive l
__global__ void __launch_bounds__(ST_NT) stencil_assemble_kernel(const StencilDev S,
                                                                 const double* __restrict__ dfield,
                                                                 const double* __restrict__ mfield,
                                                                 double* __restrict__ P) {
  extern __shared__ double s_tab[];
  const int ntab = 3 * 2 * S.ncls * S.A * S.B;
  for (int i = threadIdx.x; i < ntab; i += blockDim.x) s_tab[i] = S.tab[i];
  __syncthreads();
  const long long A3 = (long long)S.A * S.A * S.A;
  const long long nr = st_nrows(S);
  const long long total = A3 * nr;
  for (long long t = blockIdx.x * (long long)blockDim.x + threadIdx.x; t < total;
       t += (long long)gridDim.x * blockDim.x) {
    const long long kr = t % nr;
    const long long l = st_row(S, kr);
    const int a = (int)(t / nr);
    const int ax = a % S.A, ay = (a / S.A) % S.A, az = a / (S.A * S.A);
    const int lx = (int)(l % S.nx), ly = (int)((l / S.nx) % S.ny), lz = (int)(l / ((long long)S.nx * S.ny));
    const int cz = st_cls(lz, S.nz, S.ew[0]), cy = st_cls(ly, S.ny, S.ew[1]),
              cx = st_cls(lx, S.nx, S.ew[2]);
    const double* tz0 = st_tab(S, s_tab, 0, 0, cz) + az * S.B;
    const double* tz1 = st_tab(S, s_tab, 0, 1, cz) + az * S.B;
    const double* ty0 = st_tab(S, s_tab, 1, 0, cy) + ay * S.B;
    const double* ty1 = st_tab(S, s_tab, 1, 1, cy) + ay * S.B;
    const double* tx0 = st_tab(S, s_tab, 2, 0, cx) + ax * S.B;
    const double* tx1 = st_tab(S, s_tab, 2, 1, cx) + ax * S.B;
    // parameter window of node l: field index (l - ext) + ext_p + (b - mw)
    const int fz0 = lz - S.ex[0] + S.exp_[0] - S.mw, fy0 = ly - S.ex[1] + S.exp_[1] - S.mw,
              fx0 = lx - S.ex[2] + S.exp_[2] - S.mw;
    double acc = 0.0;
    for (int bz = 0; bz < S.B; ++bz) {
      const int fz = fz0 + bz;
      if (fz < 0 || fz >= S.pz) continue;
      for (int by = 0; by < S.B; ++by) {
        const int fy = fy0 + by;
        if (fy < 0 || fy >= S.py) continue;
        const double zy00 = tz0[bz] * ty0[by];
        const double k_z = S.s_stiff[0] * tz1[bz] * ty0[by];
        const double k_y = S.s_stiff[1] * tz0[bz] * ty1[by];
        const double k_x = S.s_stiff[2] * zy00;
        const double m_zy = S.s_mass * zy00;
        const long long row = ((long long)fz * S.py + fy) * S.px;
        for (int bx = 0; bx < S.B; ++bx) {
          const int fx = fx0 + bx;
          if (fx < 0 || fx >= S.px) continue;
          const double dv = dfield[row + fx], mv = mfield[row + fx];
          const double kd = (k_z + k_y) * tx0[bx] + k_x * tx1[bx];
          acc = fma(dv, kd, fma(mv, m_zy * tx0[bx], acc));
        }
      }
    }
    for (int f = 0; f < S.nfaces; ++f) {
      double prod = S.face_weight[f];
      const int li[3] = {lz, ly, lx}, ai[3] = {az - S.nb, ay - S.nb, ax - S.nb};
      const int ni[3] = {S.nz, S.ny, S.nx}, ci[3] = {cz, cy, cx};
#pragma unroll
      for (int ax3 = 0; ax3 < 3; ++ax3) {
        if (ax3 == S.face_axis[f]) {
          prod *= st_face_value(S, li[ax3], ni[ax3], S.face_side[f]) *
                  st_face_value(S, li[ax3] + ai[ax3], ni[ax3], S.face_side[f]);
        } else {
          const int j = li[ax3] + ai[ax3];
          if (S.degen[ax3])
            prod *= ai[ax3] == 0 ? 1.0 : 0.0;
          else
            prod *= (j >= 0 && j < ni[ax3]) ? S.step[ax3] * S.gram[ci[ax3] * S.A + ai[ax3] + S.nb]
                                            : 0.0;
        }
      }
      acc += prod;
    }
    P[(long long)a * nr + kr] = acc;
  }
}

// t_l = sum_a P[a, l] c[l + a] with three epilogues:
//   0 apply:  out = t
//   1 resid:  out = r = b - t;  sums {<b,b>, <r,D^-1 r>, <r,r>}   (kind 0)
//   2 cg:     out = Ap;         sums {<p,Ap>}                    (kind 1)
// Each thread computes XB consecutive x outputs: one c row segment of
// XB + 2p values serves XB * (2p+1) taps (the gather is load-instruction
// bound), and the P loads of neighbouring threads stay coalesced.
constexpr int XB = 4;

template <int MODE, int NB>
__global__ void __launch_bounds__(ST_NT) stencil_apply_kernel(const StencilDev S,
                                                              const double* __restrict__ P,
                                                              const double* __restrict__ c,
                                                              double* __restrict__ out,
                                                              const double* __restrict__ aux,
                                                              double* partials, unsigned* counter,
                                                              CgState* st, int precond,
                                                              const uint8_t* __restrict__ live = nullptr) {
  __shared__ double s_red[(ST_NT / 32) * 8];
  __shared__ unsigned s_last;
  if (MODE == 2 && !ld_vol(&st->active)) return;
  constexpr int A = 2 * NB + 1, hb = NB;
  constexpr int center = (hb * A + hb) * A + hb;
  const int nxb = (S.nx + XB - 1) / XB;
  const long long groups = (long long)S.nz * S.ny * nxb;
  double s0 = 0.0, s1 = 0.0, s2 = 0.0, s0l = 0.0, s1l = 0.0, s2l = 0.0;  // double-double
  for (long long gi = blockIdx.x * (long long)blockDim.x + threadIdx.x; gi < groups;
       gi += (long long)gridDim.x * blockDim.x) {
    const int xb = (int)(gi % nxb);
    const long long zy = gi / nxb;
    const int ly = (int)(zy % S.ny), lz = (int)(zy / S.ny);
    const int lx0 = xb * XB;
    const long long l0 = (zy * S.nx) + lx0;
    const int nv = min(XB, S.nx - lx0);
    if (MODE != 1 && live && !live[gi]) {
      // every stencil entry of these rows is zero (inactive mask nodes): the
      // gather would produce +0 exactly, and add nothing to <c, out>
#pragma unroll
      for (int v = 0; v < XB; ++v)
        if (v < nv) out[l0 + v] = 0.0;
      continue;
    }
    double t[XB];
#pragma unroll
    for (int v = 0; v < XB; ++v) t[v] = 0.0;
    int a = 0;
    for (int az = -hb; az <= hb; ++az) {
      const int z = lz + az;
      const bool zok = z >= 0 && z < S.nz;
      for (int ay = -hb; ay <= hb; ++ay, a += A) {
        const int y = ly + ay;
        if (!(zok && y >= 0 && y < S.ny)) continue;
        const double* crow = c + ((long long)z * S.ny + y) * S.nx;
        double seg[XB + 2 * NB];
#pragma unroll
        for (int k = 0; k < XB + 2 * NB; ++k) {
          const int x = lx0 - hb + k;
          seg[k] = (x >= 0 && x < S.nx) ? crow[x] : 0.0;
        }
#pragma unroll
        for (int ax = 0; ax < A; ++ax) {
          const double* pa = P + (long long)(a + ax) * S.N + l0;
#pragma unroll
          for (int v = 0; v < XB; ++v)
            if (v < nv) t[v] = fma(pa[v], seg[v + ax], t[v]);
        }
      }
    }
#pragma unroll
    for (int v = 0; v < XB; ++v) {
      if (v >= nv) break;
      const long long l = l0 + v;
      if (MODE == 0) {
        out[l] = t[v];
      } else if (MODE == 1) {
        const double bb = aux[l];
        const double r = bb - t[v];
        out[l] = r;
        const double dg = P[(long long)center * S.N + l];
        const double inv = (precond && dg != 0.0) ? 1.0 / dg : 1.0;
        ST_ACC(s0, s0l, bb, bb);
        ST_ACC(s1, s1l, r, __dmul_rn(inv, r));
        ST_ACC(s2, s2l, r, r);
      } else {
        out[l] = t[v];
        ST_ACC(s0, s0l, c[l], t[v]);
      }
    }
  }
  if (MODE == 1) {
    double vh[3] = {s0, s1, s2}, vl[3] = {s0l, s1l, s2l};
    reduce_and_finalize<3, ST_NT / 32>(vh, vl, s_red, &s_last, partials, counter, st, 1, 0);
  } else if (MODE == 2) {
    double vh[1] = {s0}, vl[1] = {s0l};
    reduce_and_finalize<1, ST_NT / 32>(vh, vl, s_red, &s_last, partials, counter, st, 1, 1);
  }
}

// p = D^-1 r + beta p (reference rounding order, solver.py:96-100)
__global__ void __launch_bounds__(ST_NT) stencil_pform_kernel(const StencilDev S, const double* P,
                                                              const double* __restrict__ r,
                                                              double* __restrict__ p,
                                                              CgState* st, int precond) {
  if (!ld_vol(&st->active)) return;
  const double beta = ld_vol(&st->beta);
  const int A = S.A, hb = S.nb;
  const int center = (hb * A + hb) * A + hb;
  // two grid-stride elements per trip (loads of both issued together; the
  // per-element arithmetic is unchanged)
  const long long stride = (long long)gridDim.x * blockDim.x;
  const long long nr = st_nrows(S);
  const double* diag = P + (long long)center * nr;
  for (long long k = blockIdx.x * (long long)blockDim.x + threadIdx.x; k < nr; k += 2 * stride) {
    const long long k2 = k + stride;
    const bool two = k2 < nr;
    const long long l = st_row(S, k), l2 = two ? st_row(S, k2) : 0;
    const double dg = diag[k], rv = r[l], pv = p[l];
    const double dg2 = two ? diag[k2] : 1.0, rv2 = two ? r[l2] : 0.0, pv2 = two ? p[l2] : 0.0;
    const double inv = (precond && dg != 0.0) ? 1.0 / dg : 1.0;
    p[l] = pdir(rv, inv, pv, beta);
    if (two) {
      const double inv2 = (precond && dg2 != 0.0) ? 1.0 / dg2 : 1.0;
      p[l2] = pdir(rv2, inv2, pv2, beta);
    }
  }
}

// x += alpha p; r -= alpha Ap; sums {<r, D^-1 r>, <r, r>}  (kind 2)
__global__ void __launch_bounds__(ST_NT) stencil_update_kernel(const StencilDev S, const double* P,
                                                               double* __restrict__ x,
                                                               double* __restrict__ r,
                                                               const double* __restrict__ p,
                                                               const double* __restrict__ ap,
                                                               double* partials, unsigned* counter,
                                                               CgState* st, int precond) {
  __shared__ double s_red[(ST_NT / 32) * 8];
  __shared__ unsigned s_last;
  if (!ld_vol(&st->active)) return;
  const double alpha = ld_vol(&st->alpha);
  const int A = S.A, hb = S.nb;
  const int center = (hb * A + hb) * A + hb;
  double rz = 0.0, rr = 0.0, rzl = 0.0, rrl = 0.0;  // double-double
  // two grid-stride elements per trip, accumulated in the same order as a
  // one-element loop (bitwise the same sums)
  const long long stride = (long long)gridDim.x * blockDim.x;
  const long long nr = st_nrows(S);
  const double* diag = P + (long long)center * nr;
  for (long long k = blockIdx.x * (long long)blockDim.x + threadIdx.x; k < nr; k += 2 * stride) {
    const long long k2 = k + stride;
    const bool two = k2 < nr;
    const long long l = st_row(S, k), l2 = two ? st_row(S, k2) : 0;
    const double xv = x[l], pv = p[l], rv = r[l], av = ap[l], dg = diag[k];
    double xv2 = 0.0, pv2 = 0.0, rv2 = 0.0, av2 = 0.0, dg2 = 1.0;
    if (two) {
      xv2 = x[l2];
      pv2 = p[l2];
      rv2 = r[l2];
      av2 = ap[l2];
      dg2 = diag[k2];
    }
    x[l] = __dadd_rn(xv, __dmul_rn(alpha, pv));
    const double rn = __dsub_rn(rv, __dmul_rn(alpha, av));
    r[l] = rn;
    const double inv = (precond && dg != 0.0) ? 1.0 / dg : 1.0;
    ST_ACC(rz, rzl, rn, __dmul_rn(inv, rn));
    ST_ACC(rr, rrl, rn, rn);
    if (two) {
      x[l2] = __dadd_rn(xv2, __dmul_rn(alpha, pv2));
      const double rn2 = __dsub_rn(rv2, __dmul_rn(alpha, av2));
      r[l2] = rn2;
      const double inv2 = (precond && dg2 != 0.0) ? 1.0 / dg2 : 1.0;
      ST_ACC(rz, rzl, rn2, __dmul_rn(inv2, rn2));
      ST_ACC(rr, rrl, rn2, rn2);
    }
  }
  double vh[2] = {rz, rr}, vl[2] = {rzl, rrl};
  reduce_and_finalize<2, ST_NT / 32>(vh, vl, s_red, &s_last, partials, counter, st, 1, 2);
}

__global__ void stencil_diag_kernel(const StencilDev S, const double* P, double* out) {
  const int A = S.A, hb = S.nb;
  const int center = (hb * A + hb) * A + hb;
  const long long nr = st_nrows(S);
  for (long long k = blockIdx.x * (long long)blockDim.x + threadIdx.x; k < nr;
       k += (long long)gridDim.x * blockDim.x)
    out[st_row(S, k)] = P[(long long)center * nr + k];
}

// Compact mode apply: one thread per active row, t = sum_a P[a, k] c[l + a]
// (ascending a, as the dense kernels), epilogues as stencil_apply_kernel.
template <int MODE, int NB>
__global__ void __launch_bounds__(ST_NT) stencil_capply_kernel(
    const StencilDev S, const double* __restrict__ P, const double* __restrict__ c,
    double* __restrict__ out, const double* __restrict__ aux, double* partials,
    unsigned* counter, CgState* st, int precond) {
  __shared__ double s_red[(ST_NT / 32) * 8];
  __shared__ unsigned s_last;
  if (MODE == 2 && !ld_vol(&st->active)) return;
  constexpr int A = 2 * NB + 1, hb = NB;
  constexpr int center = (hb * A + hb) * A + hb;
  const long long nr = S.nact;
  double s0 = 0.0, s1 = 0.0, s2 = 0.0, s0l = 0.0, s1l = 0.0, s2l = 0.0;
  for (long long k = blockIdx.x * (long long)blockDim.x + threadIdx.x; k < nr;
       k += (long long)gridDim.x * blockDim.x) {
    const long long l = S.rows[k];
    const int lx = (int)(l % S.nx), ly = (int)((l / S.nx) % S.ny),
              lz = (int)(l / ((long long)S.nx * S.ny));
    double t = 0.0;
    int a = 0;
#pragma unroll
    for (int az = -hb; az <= hb; ++az) {
      const int z = lz + az;
#pragma unroll
      for (int ay = -hb; ay <= hb; ++ay) {
        const int y = ly + ay;
        const bool ok = z >= 0 && z < S.nz && y >= 0 && y < S.ny;
        const double* crow = c + ((long long)z * S.ny + y) * S.nx;
#pragma unroll
        for (int ax = -hb; ax <= hb; ++ax, ++a) {
          const int x = lx + ax;
          if (ok && x >= 0 && x < S.nx) t = fma(P[(long long)a * nr + k], crow[x], t);
        }
      }
    }
    if (MODE == 0) {
      out[l] = t;
    } else if (MODE == 1) {
      const double bb = aux[l];
      const double r = bb - t;
      out[l] = r;
      const double dg = P[(long long)center * nr + k];
      const double inv = (precond && dg != 0.0) ? 1.0 / dg : 1.0;
      ST_ACC(s0, s0l, bb, bb);
      ST_ACC(s1, s1l, r, __dmul_rn(inv, r));
      ST_ACC(s2, s2l, r, r);
    } else {
      out[l] = t;
      ST_ACC(s0, s0l, c[l], t);
    }
  }
  if (MODE == 1) {
    double vh[3] = {s0, s1, s2}, vl[3] = {s0l, s1l, s2l};
    reduce_and_finalize<3, ST_NT / 32>(vh, vl, s_red, &s_last, partials, counter, st, 1, 0);
  } else if (MODE == 2) {
    double vh[1] = {s0}, vl[1] = {s0l};
    reduce_and_finalize<1, ST_NT / 32>(vh, vl, s_red, &s_last, partials, counter, st, 1, 1);
  }
}

}  // namespace

struct bspde_stencil {
  bspde_stencil_desc d;
  StencilDev S;
  int device = 0;
  int num_sms = 148;
  double* d_tab = nullptr;
  size_t tab_bytes = 0;
  void* host_state = nullptr;
  cudaStream_t work = nullptr;
  cudaEvent_t ev_in = nullptr, ev_out = nullptr;
  int64_t launches = 0;
  uint8_t* d_live = nullptr;  // per apply group: any nonzero stencil entry (PCG skip list)
  size_t live_bytes = 0;
  std::vector<double> host_tab;  // [axis][d][class][A*B] (copy of the desc's tables)
  // on-the-fly operator (otf.cuh): the parameter fields and the Jacobi diagonal
  const double* otf_d = nullptr;
  const double* otf_m = nullptr;
  double* otf_diag = nullptr;
};

namespace {

int st_check(bspde_stencil* s) {
  if (!s) return fail(BSPDE_ERR_ARG, "null stencil plan");
  cudaError_t e = cudaSetDevice(s->device);
  if (e != cudaSuccess) return fail(BSPDE_ERR_CUDA, std::string("cudaSetDevice: ") + cudaGetErrorString(e));
  return BSPDE_OK;
}

unsigned st_grid(const bspde_stencil* s, long long n) {
  // (the apply kernel covers XB outputs per thread; over-provisioned grids
  // just stride less)
  const long long want = (n + ST_NT - 1) / ST_NT;
  return (unsigned)std::max<long long>(1, std::min<long long>(want, std::min(MAXGRID, s->num_sms * 8)));
}

// Same operator, outputs mapped along y: a thread owns XB consecutive y
// outputs at one x, consecutive lanes take consecutive x.  Every P load of a
// warp is then one contiguous 256-byte access (the x-mapped kernel's lanes
// sit 4 doubles apart), and each output still sums its stencil entries in
// ascending a = (az, ay, ax), so t is bitwise the x-mapped result.
template <int MODE, int NB>
__global__ void __launch_bounds__(ST_NT) stencil_apply_y_kernel(const StencilDev S,
                                                                const double* __restrict__ P,
                                                                const double* __restrict__ c,
                                                                double* __restrict__ out,
                                                                const double* __restrict__ aux,
                                                                double* partials, unsigned* counter,
                                                                CgState* st, int precond,
                                                                const uint8_t* __restrict__ live = nullptr) {
  __shared__ double s_red[(ST_NT / 32) * 8];
  __shared__ unsigned s_last;
  if (MODE == 2 && !ld_vol(&st->active)) return;
  constexpr int A = 2 * NB + 1, hb = NB, NR = XB + 2 * NB;
  constexpr int center = (hb * A + hb) * A + hb;
  const int nyb = (S.ny + XB - 1) / XB;
  const long long groups = (long long)S.nz * nyb * S.nx;
  const long long sy = S.nx;
  double s0 = 0.0, s1 = 0.0, s2 = 0.0, s0l = 0.0, s1l = 0.0, s2l = 0.0;  // double-double
  for (long long gi = blockIdx.x * (long long)blockDim.x + threadIdx.x; gi < groups;
       gi += (long long)gridDim.x * blockDim.x) {
    const int lx = (int)(gi % S.nx);
    const long long r = gi / S.nx;
    const int yb = (int)(r % nyb), lz = (int)(r / nyb);
    const int ly0 = yb * XB;
    const long long l0 = ((long long)lz * S.ny + ly0) * S.nx + lx;
    const int nv = min(XB, S.ny - ly0);
    if (MODE != 1 && live && !live[gi]) {  // all-zero rows: +0 exactly (see stencil_live_kernel)
#pragma unroll
      for (int v = 0; v < XB; ++v)
        if (v < nv) out[l0 + v * sy] = 0.0;
      continue;
    }
    double t[XB];
#pragma unroll
    for (int v = 0; v < XB; ++v) t[v] = 0.0;
#pragma unroll 1
    for (int az = -hb; az <= hb; ++az) {
      const int z = lz + az;
      if (z < 0 || z >= S.nz) continue;
      const long long abase = (long long)(az + hb) * A * A;
#pragma unroll
      for (int yr = 0; yr < NR; ++yr) {  // c row y' = ly0 - hb + yr
        const int y = ly0 - hb + yr;
        if (y < 0 || y >= S.ny) continue;
        const double* crow = c + ((long long)z * S.ny + y) * S.nx;
        double seg[A];
#pragma unroll
        for (int ax = 0; ax < A; ++ax) {
          const int x = lx - hb + ax;
          seg[ax] = (x >= 0 && x < S.nx) ? crow[x] : 0.0;
        }
#pragma unroll
        for (int v = 0; v < XB; ++v) {
          const int ay = yr - v;  // + hb offset: row index of the stencil
          if (ay < 0 || ay >= A) continue;
          if (v >= nv) continue;
          const double* pa = P + (abase + (long long)ay * A) * S.N + l0 + v * sy;
#pragma unroll
          for (int ax = 0; ax < A; ++ax) t[v] = fma(pa[(long long)ax * S.N], seg[ax], t[v]);
        }
      }
    }
#pragma unroll
    for (int v = 0; v < XB; ++v) {
      if (v >= nv) break;
      const long long l = l0 + v * sy;
      if (MODE == 0) {
        out[l] = t[v];
      } else if (MODE == 1) {
        const double bb = aux[l];
        const double rr = bb - t[v];
        out[l] = rr;
        const double dg = P[(long long)center * S.N + l];
        const double inv = (precond && dg != 0.0) ? 1.0 / dg : 1.0;
        ST_ACC(s0, s0l, bb, bb);
        ST_ACC(s1, s1l, rr, __dmul_rn(inv, rr));
        ST_ACC(s2, s2l, rr, rr);
      } else {
        out[l] = t[v];
        ST_ACC(s0, s0l, c[l], t[v]);
      }
    }
  }
  if (MODE == 1) {
    double vh[3] = {s0, s1, s2}, vl[3] = {s0l, s1l, s2l};
    reduce_and_finalize<3, ST_NT / 32>(vh, vl, s_red, &s_last, partials, counter, st, 1, 0);
  } else if (MODE == 2) {
    double vh[1] = {s0}, vl[1] = {s0l};
    reduce_and_finalize<1, ST_NT / 32>(vh, vl, s_red, &s_last, partials, counter, st, 1, 1);
  }
}

// live[g] = 1 iff output group g (XB consecutive x of one (z, y) row, the
// x-mapped apply's unit) has a nonzero stencil entry.  Mask systems keep
// their inactive nodes as all-zero rows (79% of the leg's 864k rows); the
// CG apply skips those groups' 27..125 stencil loads.
// YMAP: the y-mapped apply's groups (XB consecutive y at one x).
template <int NB, bool YMAP>
__global__ void __launch_bounds__(ST_NT) stencil_live_kernel(const StencilDev S,
                                                             const double* __restrict__ P,
                                                             uint8_t* __restrict__ live) {
  constexpr int A = 2 * NB + 1, A3 = A * A * A;
  const int nxb = (S.nx + XB - 1) / XB, nyb = (S.ny + XB - 1) / XB;
  const long long groups = YMAP ? (long long)S.nz * nyb * S.nx : (long long)S.nz * S.ny * nxb;
  for (long long gi = blockIdx.x * (long long)blockDim.x + threadIdx.x; gi < groups;
       gi += (long long)gridDim.x * blockDim.x) {
    long long l0, step;
    int nv;
    if (YMAP) {
      const int lx = (int)(gi % S.nx);
      const long long r = gi / S.nx;
      const int yb = (int)(r % nyb), lz = (int)(r / nyb);
      l0 = ((long long)lz * S.ny + yb * XB) * S.nx + lx;
      nv = min(XB, S.ny - yb * XB);
      step = S.nx;
    } else {
      const int xb = (int)(gi % nxb);
      l0 = (gi / nxb) * S.nx + xb * XB;
      nv = min(XB, S.nx - xb * XB);
      step = 1;
    }
    bool nz = false;
    for (int e = 0; e < A3 && !nz; ++e) {
      const double* pe = P + (long long)e * S.N + l0;
#pragma unroll
      for (int v = 0; v < XB; ++v)
        if (v < nv && pe[v * step] != 0.0) nz = true;
    }
    live[gi] = nz ? 1 : 0;
  }
}

inline bool st_ymap() {
  static const int v = [] {
    const char* e = getenv("BSPDE_ST_XMAP");
    return (e && e[0] == '1') ? 0 : 1;
  }();
  return v != 0;
}

template <int MODE>
void st_apply(const bspde_stencil* s, unsigned grid, cudaStream_t st, const double* P,
              const double* c, double* out, const double* aux, double* partials,
              unsigned* counter, CgState* state, int precond, const uint8_t* live = nullptr) {
  if (s->S.rows) {  // compact (active rows only)
    const unsigned cg = st_grid(s, s->S.nact);
    switch (s->S.nb) {
      case 1: stencil_capply_kernel<MODE, 1><<<cg, ST_NT, 0, st>>>(s->S, P, c, out, aux, partials, counter, state, precond); break;
      case 2: stencil_capply_kernel<MODE, 2><<<cg, ST_NT, 0, st>>>(s->S, P, c, out, aux, partials, counter, state, precond); break;
      case 3: stencil_capply_kernel<MODE, 3><<<cg, ST_NT, 0, st>>>(s->S, P, c, out, aux, partials, counter, state, precond); break;
      case 4: stencil_capply_kernel<MODE, 4><<<cg, ST_NT, 0, st>>>(s->S, P, c, out, aux, partials, counter, state, precond); break;
      default: stencil_capply_kernel<MODE, 5><<<cg, ST_NT, 0, st>>>(s->S, P, c, out, aux, partials, counter, state, precond); break;
    }
    return;
  }
  // y mapping for p >= 3 (measured +5-30% apply, +25% PCG at p = 3); at
  // p = 1, 2 the compiler batches every load of the short stencil into
  // registers (128-255) and the x mapping is faster
  if (st_ymap() && s->S.nb >= 3) {
    switch (s->S.nb) {
      case 3: stencil_apply_y_kernel<MODE, 3><<<grid, ST_NT, 0, st>>>(s->S, P, c, out, aux, partials, counter, state, precond, live); break;
      case 4: stencil_apply_y_kernel<MODE, 4><<<grid, ST_NT, 0, st>>>(s->S, P, c, out, aux, partials, counter, state, precond, live); break;
      default: stencil_apply_y_kernel<MODE, 5><<<grid, ST_NT, 0, st>>>(s->S, P, c, out, aux, partials, counter, state, precond, live); break;
    }
    return;
  }
  switch (s->S.nb) {
    case 1: stencil_apply_kernel<MODE, 1><<<grid, ST_NT, 0, st>>>(s->S, P, c, out, aux, partials, counter, state, precond, live); break;
    case 2: stencil_apply_kernel<MODE, 2><<<grid, ST_NT, 0, st>>>(s->S, P, c, out, aux, partials, counter, state, precond, live); break;
    case 3: stencil_apply_kernel<MODE, 3><<<grid, ST_NT, 0, st>>>(s->S, P, c, out, aux, partials, counter, state, precond, live); break;
    case 4: stencil_apply_kernel<MODE, 4><<<grid, ST_NT, 0, st>>>(s->S, P, c, out, aux, partials, counter, state, precond, live); break;
    default: stencil_apply_kernel<MODE, 5><<<grid, ST_NT, 0, st>>>(s->S, P, c, out, aux, partials, counter, state, precond, live); break;
  }
}

// live flags in the group order of the apply kernel st_apply launches
int st_live(bspde_stencil* s, const double* P, cudaStream_t st, uint8_t** live) {
  *live = nullptr;
  if (getenv("BSPDE_ST_NOSKIP")) return BSPDE_OK;
  const bool ymap = st_ymap() && s->S.nb >= 3;
  const long long groups =
      ymap ? (long long)s->S.nz * ((s->S.ny + XB - 1) / XB) * s->S.nx
           : (long long)s->S.nz * s->S.ny * ((s->S.nx + XB - 1) / XB);
  if ((size_t)groups > s->live_bytes) {
    if (s->d_live) CUDA_TRY(cudaFree(s->d_live));
    s->d_live = nullptr;
    s->live_bytes = 0;
    CUDA_TRY(cudaMalloc(&s->d_live, (size_t)groups));
    s->live_bytes = (size_t)groups;
  }
  const unsigned grid = st_grid(s, groups);
  switch (s->S.nb * 2 + (ymap ? 1 : 0)) {
    case 2: stencil_live_kernel<1, false><<<grid, ST_NT, 0, st>>>(s->S, P, s->d_live); break;
    case 4: stencil_live_kernel<2, false><<<grid, ST_NT, 0, st>>>(s->S, P, s->d_live); break;
    case 6: stencil_live_kernel<3, false><<<grid, ST_NT, 0, st>>>(s->S, P, s->d_live); break;
    case 7: stencil_live_kernel<3, true><<<grid, ST_NT, 0, st>>>(s->S, P, s->d_live); break;
    case 8: stencil_live_kernel<4, false><<<grid, ST_NT, 0, st>>>(s->S, P, s->d_live); break;
    case 9: stencil_live_kernel<4, true><<<grid, ST_NT, 0, st>>>(s->S, P, s->d_live); break;
    case 10: stencil_live_kernel<5, false><<<grid, ST_NT, 0, st>>>(s->S, P, s->d_live); break;
    default: stencil_live_kernel<5, true><<<grid, ST_NT, 0, st>>>(s->S, P, s->d_live); break;
  }
  s->launches++;
  CUDA_TRY(cudaGetLastError());
  *live = s->d_live;
  return BSPDE_OK;
}

template <int MODE>
int otf_launch(const bspde_stencil* s, cudaStream_t st, const double* c, double* out,
               const double* aux, double* partials, unsigned* counter, CgState* state,
               int precond);  // otf.cuh

int st_read(bspde_stencil* s, void* scratch, bspde_cg_report* rep, int32_t* active, cudaStream_t st) {
  CgState* hs = reinterpret_cast<CgState*>(s->host_state);
  CUDA_TRY(cudaMemcpyAsync(hs, scratch_state(scratch), sizeof(CgState), cudaMemcpyDeviceToHost, st));
  CUDA_TRY(cudaStreamSynchronize(st));
  if (rep) {
    rep->iterations = hs->it;
    rep->status = hs->status;
    rep->residual = hs->res;
    rep->residual0 = hs->res0;
    rep->rhs_norm = hs->rhs_norm;
    rep->relative_residual = hs->res / hs->scale;
    rep->last_pAp = hs->pAp;
  }
  if (active) *active = hs->active;
  return BSPDE_OK;
}

// Jacobi-PCG over the stencil (or, otf = true, the on-the-fly operator of
// otf.cuh, whose Jacobi diagonal P's centre slice points at): the reference
// recurrence with three kernels per iteration
int st_pcg(bspde_stencil* s, const double* P, const double* b, double* x, double* r, double* p,
           double* ap, void* scratch, double* history, const bspde_cg_config* cfg,
           bspde_cg_report* report, int32_t precond, void* stream, bool otf) {
  if (!P || !b || !x || !r || !p || !ap || !scratch || !cfg)
    return fail(BSPDE_ERR_ARG, "null argument");
  if (!(cfg->tol > 0.0)) return fail(BSPDE_ERR_ARG, "tol must be positive");
  if (cfg->max_iter < 1) return fail(BSPDE_ERR_ARG, "max_iter must be >= 1");
  if (cfg->record_history && !history) return fail(BSPDE_ERR_ARG, "history buffer required");
  cudaStream_t caller = (cudaStream_t)stream, st = s->work;
  CUDA_TRY(cudaEventRecord(s->ev_in, caller));
  CUDA_TRY(cudaStreamWaitEvent(st, s->ev_in, 0));
  // scalar state (same layout and state machine as bspde_cg_setup)
  CgState* hs = reinterpret_cast<CgState*>(s->host_state);
  CUDA_TRY(cudaStreamSynchronize(st));
  std::memset(hs, 0, sizeof(CgState));
  hs->tol = cfg->tol;
  hs->max_iter = cfg->max_iter;
  hs->record_history = cfg->record_history ? 1 : 0;
  hs->has_x0 = cfg->has_x0 ? 1 : 0;
  hs->ring = kPRing;  // finalize_state's x-ring bookkeeping (unused by the stencil CG)
  hs->history = history;
  hs->scale = 1.0;
  CUDA_TRY(cudaMemcpyAsync(scratch_state(scratch), hs, sizeof(CgState), cudaMemcpyHostToDevice, st));
  CUDA_TRY(cudaMemsetAsync(scratch_counter(scratch), 0, 64, st));
  const size_t bytes = (size_t)s->S.N * sizeof(double);
  if (!cfg->has_x0) CUDA_TRY(cudaMemsetAsync(x, 0, bytes, st));
  CUDA_TRY(cudaMemsetAsync(p, 0, bytes, st));
  if (s->S.rows) {  // compact: the inactive entries of r and Ap are never written
    CUDA_TRY(cudaMemsetAsync(r, 0, bytes, st));
    CUDA_TRY(cudaMemsetAsync(ap, 0, bytes, st));
  }
  const unsigned grid = st_grid(s, s->S.N);
  double* partials = scratch_partials(scratch);
  unsigned* counter = scratch_counter(scratch);
  CgState* state = scratch_state(scratch);
  const unsigned agrid = st_grid(s, s->S.N / XB + 1);
  uint8_t* live = nullptr;
  if (!otf)
    if (!s->S.rows)
      if (int lrc = st_live(s, P, st, &live)) return lrc;
  if (otf) {
    if (int orc = otf_launch<1>(s, st, x, r, b, partials, counter, state, precond)) return orc;
  } else {
    st_apply<1>(s, agrid, st, P, x, r, b, partials, counter, state, precond);
  }
  s->launches++;
  CUDA_TRY(cudaGetLastError());
  int32_t active = 0;
  int rc = st_read(s, scratch, report, &active, st);
  const int K = cfg->poll_every > 0 ? cfg->poll_every : 8;
  while (rc == BSPDE_OK && active) {
    for (int k = 0; k < K; ++k) {
      stencil_pform_kernel<<<grid, ST_NT, 0, st>>>(s->S, P, r, p, state, precond);
      if (otf) {
        if (int orc = otf_launch<2>(s, st, p, ap, nullptr, partials, counter, state, precond))
          return orc;
      } else {
        st_apply<2>(s, agrid, st, P, p, ap, nullptr, partials, counter, state, precond, live);
      }
      stencil_update_kernel<<<grid, ST_NT, 0, st>>>(s->S, P, x, r, p, ap, partials, counter,
                                                    state, precond);
      s->launches += 3;
    }
    CUDA_TRY(cudaGetLastError());
    rc = st_read(s, scratch, report, &active, st);
  }
  cudaEventRecord(s->ev_out, st);
  cudaStreamWaitEvent(caller, s->ev_out, 0);
  return rc;
}


}  // namespace

extern "C" {

int bspde_stencil_create(const bspde_stencil_desc* desc, bspde_stencil** out) {
  if (!desc || !out) return fail(BSPDE_ERR_ARG, "null argument");
  const auto& d = *desc;
  if (d.degree < 1 || d.degree > MAXP || d.param_degree < 0 || d.param_degree > MAXP)
    return fail(BSPDE_ERR_ARG, "degrees must be n_b in 1..5, n_p in 0..5");
  if (d.nz < 1 || d.ny < 1 || d.nx < 1 || d.pz < 1 || d.py < 1 || d.px < 1)
    return fail(BSPDE_ERR_ARG, "empty extents");
  const int EW = edge_width_of(d.degree);
  for (int a = 0; a < 3; ++a) {
    if (d.ew[a] < 0 || d.ew[a] > EW) return fail(BSPDE_ERR_ARG, "edge width out of range");
    for (int k = 0; k < 2; ++k)
      if (!d.tables[a][k]) return fail(BSPDE_ERR_ARG, "missing trilinear tables");
  }
  if (d.device < 0) return fail(BSPDE_ERR_ARG, "bad device ordinal");
  CUDA_TRY(cudaSetDevice(d.device));
  auto* s = new bspde_stencil();
  s->d = d;
  s->device = d.device;
  cudaDeviceGetAttribute(&s->num_sms, cudaDevAttrMultiProcessorCount, d.device);
  StencilDev& S = s->S;
  S.nb = d.degree;
  S.np = d.param_degree;
  S.mw = (d.degree + d.param_degree + 1) / 2;
  S.A = 2 * S.nb + 1;
  S.B = 2 * S.mw + 1;
  S.nz = d.nz;
  S.ny = d.ny;
  S.nx = d.nx;
  S.pz = d.pz;
  S.py = d.py;
  S.px = d.px;
  S.ext = d.ext;
  S.ext_p = d.ext_p;
  for (int a = 0; a < 3; ++a) {
    S.ew[a] = d.ew[a];
    S.s_stiff[a] = d.scale_stiff[a];
  }
  S.s_mass = d.scale_mass;
  S.N = (long long)d.nz * d.ny * d.nx;
  S.ncls = 2 * EW + 1;
  if (d.nfaces < 0 || d.nfaces > 6) {
    delete s;
    return fail(BSPDE_ERR_ARG, "nfaces must be 0..6");
  }
  S.nfaces = d.nfaces;
  for (int f = 0; f < 6; ++f) {
    S.face_axis[f] = f < d.nfaces ? d.face_axis[f] : 0;
    S.face_side[f] = f < d.nfaces ? d.face_side[f] : 0;
    S.face_weight[f] = f < d.nfaces ? d.face_weight[f] : 0.0;
    if (f < d.nfaces && (S.face_axis[f] < 0 || S.face_axis[f] > 2 || S.face_side[f] < 0 ||
                         S.face_side[f] > 1)) {
      delete s;
      return fail(BSPDE_ERR_ARG, "bad face axis / side");
    }
  }
  S.rows = nullptr;
  S.nact = 0;
  for (int k = 0; k < MAXP + 1; ++k) S.fv[k] = 0.0;
  for (int k = 0; k < 121; ++k) S.gram[k] = 0.0;
  if (d.nfaces > 0) {
    if (!d.face_values || !d.mass_gram) {
      delete s;
      return fail(BSPDE_ERR_ARG, "face terms need face_values and mass_gram");
    }
    for (int k = 0; k < EW; ++k) S.fv[k] = d.face_values[k];
    for (int k = 0; k < (2 * EW + 1) * S.A; ++k) S.gram[k] = d.mass_gram[k];
  }
  for (int a = 0; a < 3; ++a) {
    S.step[a] = d.step[a];
    S.degen[a] = d.degenerate[a] ? 1 : 0;
    S.ex[a] = S.degen[a] ? 0 : d.ext;
    S.exp_[a] = S.degen[a] ? 0 : d.ext_p;
    if (S.degen[a] && ((a == 0 ? d.nz : a == 1 ? d.ny : d.nx) != 1 ||
                       (a == 0 ? d.pz : a == 1 ? d.py : d.px) != 1)) {
      delete s;
      return fail(BSPDE_ERR_ARG, "a degenerate axis must have extent 1");
    }
  }
  const size_t per = (size_t)S.A * S.B;
  std::vector<double> tab((size_t)3 * 2 * S.ncls * per, 0.0);
  for (int a = 0; a < 3; ++a)
    for (int k = 0; k < 2; ++k)
      for (int c = 0; c < 2 * d.ew[a] + 1; ++c)
        for (size_t e = 0; e < per; ++e)
          tab[(((size_t)a * 2 + k) * S.ncls + c) * per + e] = d.tables[a][k][c * per + e];
  s->tab_bytes = tab.size() * sizeof(double);
  cudaError_t e1 = cudaMalloc(&s->d_tab, s->tab_bytes);
  cudaError_t e2 = cudaMallocHost(&s->host_state, sizeof(CgState));
  cudaError_t e3 = cudaStreamCreateWithFlags(&s->work, cudaStreamNonBlocking);
  cudaError_t e4 = cudaEventCreateWithFlags(&s->ev_in, cudaEventDisableTiming);
  cudaError_t e5 = cudaEventCreateWithFlags(&s->ev_out, cudaEventDisableTiming);
  if (e1 != cudaSuccess || e2 != cudaSuccess || e3 != cudaSuccess || e4 != cudaSuccess ||
      e5 != cudaSuccess) {
    bspde_stencil_destroy(s);
    return fail(BSPDE_ERR_CUDA, "stencil plan allocation failed");
  }
  cudaError_t e6 = cudaMemcpy(s->d_tab, tab.data(), s->tab_bytes, cudaMemcpyHostToDevice);
  if (e6 != cudaSuccess) {
    bspde_stencil_destroy(s);
    return fail(BSPDE_ERR_CUDA, std::string("table upload: ") + cudaGetErrorString(e6));
  }
  S.tab = s->d_tab;
  s->host_tab = tab;
  *out = s;
  return BSPDE_OK;
}

int bspde_stencil_destroy(bspde_stencil* s) {
  if (!s) return BSPDE_OK;
  cudaSetDevice(s->device);
  if (s->d_tab) cudaFree(s->d_tab);
  if (s->d_live) cudaFree(s->d_live);
  if (s->host_state) cudaFreeHost(s->host_state);
  if (s->work) cudaStreamDestroy(s->work);
  if (s->ev_in) cudaEventDestroy(s->ev_in);
  if (s->ev_out) cudaEventDestroy(s->ev_out);
  delete s;
  return BSPDE_OK;
}

int64_t bspde_stencil_entries(const bspde_stencil* s) {
  if (!s) return -1;
  return (int64_t)s->S.A * s->S.A * s->S.A * (s->S.rows ? s->S.nact : s->S.N);
}

int bspde_stencil_set_rows(bspde_stencil* s, const int64_t* rows, int64_t nact) {
  if (int rc = st_check(s)) return rc;
  if ((rows == nullptr) != (nact == 0) || nact < 0 || nact > s->S.N)
    return fail(BSPDE_ERR_ARG, "rows / nact: device array of 1..N ascending active rows");
  s->S.rows = rows;
  s->S.nact = nact;
  return BSPDE_OK;
}

int64_t bspde_stencil_launch_count(const bspde_stencil* s) { return s ? s->launches : -1; }

int bspde_stencil_assemble(bspde_stencil* s, const double* dfield, const double* mfield,
                           double* P, void* stream) {
  if (int rc = st_check(s)) return rc;
  if (!dfield || !mfield || !P) return fail(BSPDE_ERR_ARG, "null argument");
  const long long total = (long long)s->S.A * s->S.A * s->S.A * s->S.N;
  const unsigned grid = (unsigned)std::min<long long>((total + ST_NT - 1) / ST_NT, 1 << 20);
  const size_t smem = s->tab_bytes;
  if (smem > 48 * 1024)
    CUDA_TRY(cudaFuncSetAttribute(reinterpret_cast<const void*>(&stencil_assemble_kernel),
                                  cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
  stencil_assemble_kernel<<<grid, ST_NT, smem, (cudaStream_t)stream>>>(s->S, dfield, mfield, P);
  s->launches++;
  CUDA_TRY(cudaGetLastError());
  return BSPDE_OK;
}

int bspde_stencil_apply(bspde_stencil* s, const double* P, const double* c, double* out,
                        void* stream) {
  if (int rc = st_check(s)) return rc;
  if (!P || !c || !out) return fail(BSPDE_ERR_ARG, "null argument");
  st_apply<0>(s, st_grid(s, s->S.N / XB + 1), (cudaStream_t)stream, P, c, out, nullptr, nullptr,
              nullptr, nullptr, 0);
  s->launches++;
  CUDA_TRY(cudaGetLastError());
  return BSPDE_OK;
}

int bspde_stencil_diagonal(bspde_stencil* s, const double* P, double* out, void* stream) {
  if (int rc = st_check(s)) return rc;
  if (!P || !out) return fail(BSPDE_ERR_ARG, "null argument");
  stencil_diag_kernel<<<st_grid(s, s->S.N), ST_NT, 0, (cudaStream_t)stream>>>(s->S, P, out);
  s->launches++;
  CUDA_TRY(cudaGetLastError());
  return BSPDE_OK;
}

int bspde_stencil_pcg(bspde_stencil* s, const double* P, const double* b, double* x, double* r,
                      double* p, double* ap, void* scratch, double* history,
                      const bspde_cg_config* cfg, bspde_cg_report* report, int32_t precond,
                      void* stream) {
  if (int rc = st_check(s)) return rc;
  return st_pcg(s, P, b, x, r, p, ap, scratch, history, cfg, report, precond, stream, false);
}

}  // extern "C"

// ---------------------------------------------------------------------------
// Mask (voxel) domains.  The reference assembles the
// rows of boundary nodes cell by cell on the host and scatters them
// (assembly.py:538-737); here one thread owns one (boundary row, offset)
// entry and gathers it from the occupied cells of the row's support, so the
// rows are written exactly once, without atomics, straight into P.

namespace {

constexpr int MASK_MAXJ = 6;  // cell_node_offsets of degree 5: 6 offsets

__device__ __forceinline__ bool mask_occ(const bspde_mask_desc& M, int z, int y, int x) {
  if (z < 0 || y < 0 || x < 0 || z >= M.cells[0] || y >= M.cells[1] || x >= M.cells[2])
    return false;  // cells beyond the grid count as unoccupied
  return M.occupancy[((long long)z * M.cells[1] + y) * M.cells[2] + x] != 0;
}

// face (axis, side) of cell c borders an unoccupied cell (exposed_faces,
// assembly.py:640-654)
__device__ __forceinline__ bool mask_exposed(const bspde_mask_desc& M, const int (&c)[3],
                                             int axis, int side) {
  if (!mask_occ(M, c[0], c[1], c[2])) return false;
  int n[3] = {c[0], c[1], c[2]};
  n[axis] += side ? 1 : -1;
  return !mask_occ(M, n[0], n[1], n[2]);
}

__global__ void __launch_bounds__(ST_NT) mask_zero_kernel(const StencilDev S,
                                                          const uint8_t* __restrict__ cls,
                                                          double* __restrict__ P) {
  const long long total = (long long)S.A * S.A * S.A * S.N;
  for (long long t = blockIdx.x * (long long)blockDim.x + threadIdx.x; t < total;
       t += (long long)gridDim.x * blockDim.x)
    if (cls[t % S.N] == 0) P[t] = 0.0;
}

__global__ void __launch_bounds__(ST_NT) mask_rows_kernel(const StencilDev S,
                                                          const bspde_mask_desc M,
                                                          const double* __restrict__ dfield,
                                                          const double* __restrict__ mfield,
                                                          double* __restrict__ P) {
  const long long A3 = (long long)S.A * S.A * S.A;
  const long long total = A3 * M.nbrows;
  const int nj = M.nj, nbp = M.nbp;
  const long long tstride = (long long)nj * nj * nbp;
  for (long long t = blockIdx.x * (long long)blockDim.x + threadIdx.x; t < total;
       t += (long long)gridDim.x * blockDim.x) {
    const long long l = M.brows[t % M.nbrows];
    const int a = (int)(t / M.nbrows);
    const int off[3] = {a / (S.A * S.A) - S.nb, (a / S.A) % S.A - S.nb, a % S.A - S.nb};
    const int lz = (int)(l / ((long long)S.nx * S.ny)), ly = (int)((l / S.nx) % S.ny),
              lx = (int)(l % S.nx);
    const int sp[3] = {lz - S.ex[0], ly - S.ex[1], lx - S.ex[2]};  // spline indices of the row
    // per axis: the cells of the row's support (test offset j2) whose trial
    // offset j1 = j2 + off also lies on the cell.  A unit axis has one cell
    // layer, one offset and the identity factor (value 1, derivative 0).
    const double unit[2] = {1.0, 0.0};
    int j2lo[3], j2hi[3], jl[3], nbx[3], bl[3];
#pragma unroll
    for (int d = 0; d < 3; ++d) {
      const int n = M.degenerate[d] ? 1 : nj;
      j2lo[d] = max(0, -off[d]);
      j2hi[d] = min(n, n - off[d]);
      jl[d] = M.degenerate[d] ? 0 : M.jlo;
      nbx[d] = M.degenerate[d] ? 1 : nbp;
      bl[d] = M.degenerate[d] ? 0 : M.blo;
    }
    auto tri = [&](int d, int j2, int k) -> const double* {  // k: 0 value, 1 derivative
      if (M.degenerate[d]) return unit + k;
      return M.cell_tri + ((long long)(j2 + off[d]) * nj + j2) * nbp + k * tstride;
    };
    double acc = 0.0;
    for (int jz = j2lo[0]; jz < j2hi[0]; ++jz) {
      const int cz = sp[0] - (jl[0] + jz);
      const double* tz0 = tri(0, jz, 0);
      const double* tz1 = tri(0, jz, 1);
      for (int jy = j2lo[1]; jy < j2hi[1]; ++jy) {
        const int cy = sp[1] - (jl[1] + jy);
        const double* ty0 = tri(1, jy, 0);
        const double* ty1 = tri(1, jy, 1);
        for (int jx = j2lo[2]; jx < j2hi[2]; ++jx) {
          const int cx = sp[2] - (jl[2] + jx);
          if (!mask_occ(M, cz, cy, cx)) continue;
          const double* tx0 = tri(2, jx, 0);
          const double* tx1 = tri(2, jx, 1);
          // parameter spline c + blo + b lives at field index c + blo + b + ext_p
          const int fz0 = cz + bl[0] + S.exp_[0], fy0 = cy + bl[1] + S.exp_[1],
                    fx0 = cx + bl[2] + S.exp_[2];
          double cell = 0.0;
          for (int bz = 0; bz < nbx[0]; ++bz) {
            const int fz = fz0 + bz;
            if (fz < 0 || fz >= S.pz) continue;
            for (int by = 0; by < nbx[1]; ++by) {
              const int fy = fy0 + by;
              if (fy < 0 || fy >= S.py) continue;
              const double zy00 = tz0[bz] * ty0[by];
              const double k_z = S.s_stiff[0] * tz1[bz] * ty0[by];
              const double k_y = S.s_stiff[1] * tz0[bz] * ty1[by];
              const double k_x = S.s_stiff[2] * zy00;
              const double m_zy = S.s_mass * zy00;
              const long long row = ((long long)fz * S.py + fy) * S.px;
              for (int bx = 0; bx < nbx[2]; ++bx) {
                const int fx = fx0 + bx;
                if (fx < 0 || fx >= S.px) continue;
                const double kd = (k_z + k_y) * tx0[bx] + k_x * tx1[bx];
                cell = fma(dfield[row + fx], kd, fma(mfield[row + fx], m_zy * tx0[bx], cell));
              }
            }
          }
          acc += cell;
        }
      }
    }
    if (M.has_surface) {
      // exposed faces: (v v)_normal (x) R (x) R over the tangential axes
      // (a unit axis is never a face normal and contributes the factor 1)
      const int nv = 2 * M.fc - 1;
      for (int axn = 0; axn < 3; ++axn) {
        if (M.degenerate[axn]) continue;
        const int t1 = axn == 0 ? 1 : 0, t2 = axn == 2 ? 1 : 2;
        const double tscale = S.step[t1] * S.step[t2];
        for (int side = 0; side < 2; ++side) {
          for (int k = 0; k < nv; ++k) {  // test normal offset jn = side + k - (fc-1)
            const int k1 = k + off[axn];
            if (k1 < 0 || k1 >= nv) continue;
            const double vv = M.face_vals[k] * M.face_vals[k1];
            if (vv == 0.0) continue;
            int c[3];
            c[axn] = sp[axn] - (side + k - (M.fc - 1));
            for (int ja = j2lo[t1]; ja < j2hi[t1]; ++ja) {
              c[t1] = sp[t1] - (jl[t1] + ja);
              const double ra = M.degenerate[t1] ? 1.0 : M.cell_bil[(ja + off[t1]) * nj + ja];
              for (int jb = j2lo[t2]; jb < j2hi[t2]; ++jb) {
                c[t2] = sp[t2] - (jl[t2] + jb);
                if (!mask_exposed(M, c, axn, side)) continue;
                const double rb = M.degenerate[t2] ? 1.0 : M.cell_bil[(jb + off[t2]) * nj + jb];
                acc += M.surface_weight * tscale * vv * ra * rb;
              }
            }
          }
        }
      }
    }
    // compact mode: the row's slot in the active-row list (M.brows_k)
    P[(long long)a * st_nrows(S) + (S.rows ? M.brows_k[t % M.nbrows] : l)] = acc;
  }
}

__global__ void __launch_bounds__(ST_NT) mask_surface_rhs_kernel(const StencilDev S,
                                                                 const bspde_mask_desc M,
                                                                 double scale,
                                                                 double* __restrict__ out) {
  const int nv = 2 * M.fc - 1;
  for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < M.nbrows;
       i += (long long)gridDim.x * blockDim.x) {
    const long long l = M.brows[i];
    const int sp[3] = {(int)(l / ((long long)S.nx * S.ny)) - S.ex[0],
                       (int)((l / S.nx) % S.ny) - S.ex[1], (int)(l % S.nx) - S.ex[2]};
    double acc = 0.0;
    for (int axn = 0; axn < 3; ++axn) {
      if (M.degenerate[axn]) continue;
      const int t1 = axn == 0 ? 1 : 0, t2 = axn == 2 ? 1 : 2;
      const int n1 = M.degenerate[t1] ? 1 : M.nj, n2 = M.degenerate[t2] ? 1 : M.nj;
      const int l1 = M.degenerate[t1] ? 0 : M.jlo, l2 = M.degenerate[t2] ? 0 : M.jlo;
      const double tscale = S.step[t1] * S.step[t2];
      for (int side = 0; side < 2; ++side)
        for (int k = 0; k < nv; ++k) {
          int c[3];
          c[axn] = sp[axn] - (side + k - (M.fc - 1));
          for (int ja = 0; ja < n1; ++ja) {
            c[t1] = sp[t1] - (l1 + ja);
            const double sa = M.degenerate[t1] ? 1.0 : M.cell_single[ja];
            for (int jb = 0; jb < n2; ++jb) {
              c[t2] = sp[t2] - (l2 + jb);
              if (!mask_exposed(M, c, axn, side)) continue;
              const double sb = M.degenerate[t2] ? 1.0 : M.cell_single[jb];
              acc += scale * tscale * M.face_vals[k] * sa * sb;
            }
          }
        }
    }
    out[l] += acc;
  }
}

int mask_check(const bspde_stencil* s, const bspde_mask_desc* m) {
  if (!m || !m->occupancy || !m->node_class || (m->nbrows > 0 && !m->brows) || !m->cell_tri ||
      !m->cell_bil || !m->cell_single || !m->face_vals)
    return fail(BSPDE_ERR_ARG, "mask desc: null pointer");
  if (m->nj < 1 || m->nj > MASK_MAXJ || m->nbp < 1 || m->nbp > MASK_MAXJ || m->fc < 1 ||
      m->fc > 3 || m->nbrows < 0)
    return fail(BSPDE_ERR_ARG, "mask desc: table sizes out of range");
  const int n3[3] = {s->S.nz, s->S.ny, s->S.nx};
  for (int a = 0; a < 3; ++a) {
    if ((m->degenerate[a] != 0) != (s->S.degen[a] != 0))
      return fail(BSPDE_ERR_ARG, "mask and plan disagree on unit axes");
    const int want = s->S.degen[a] ? 1 : n3[a] - 2 * s->S.ext - 1;
    if (m->cells[a] != want) return fail(BSPDE_ERR_ARG, "mask cell extents do not match the plan");
  }
  return BSPDE_OK;
}

}  // namespace

extern "C" {

int bspde_stencil_mask_patch(bspde_stencil* s, const bspde_mask_desc* m, const double* dfield,
                             const double* mfield, double* P, void* stream) {
  if (int rc = st_check(s)) return rc;
  if (int rc = mask_check(s, m)) return rc;
  if (!dfield || !mfield || !P) return fail(BSPDE_ERR_ARG, "null argument");
  const cudaStream_t st = (cudaStream_t)stream;
  const long long A3 = (long long)s->S.A * s->S.A * s->S.A;
  if (!s->S.rows) {  // dense: zero the rows of inactive nodes (compact P has none)
    mask_zero_kernel<<<st_grid(s, A3 * s->S.N), ST_NT, 0, st>>>(s->S, m->node_class, P);
    s->launches++;
  } else if (m->nbrows > 0 && !m->brows_k) {
    return fail(BSPDE_ERR_ARG, "compact mask plan: brows_k required");
  }
  if (m->nbrows > 0) {
    mask_rows_kernel<<<st_grid(s, A3 * m->nbrows), ST_NT, 0, st>>>(s->S, *m, dfield, mfield, P);
    s->launches++;
  }
  CUDA_TRY(cudaGetLastError());
  return BSPDE_OK;
}

int bspde_stencil_mask_surface_rhs(bspde_stencil* s, const bspde_mask_desc* m, double value,
                                   double* out, void* stream) {
  if (int rc = st_check(s)) return rc;
  if (int rc = mask_check(s, m)) return rc;
  if (!out) return fail(BSPDE_ERR_ARG, "null argument");
  if (m->nbrows == 0 || !m->has_surface) return BSPDE_OK;
  mask_surface_rhs_kernel<<<st_grid(s, m->nbrows), ST_NT, 0, (cudaStream_t)stream>>>(
      s->S, *m, value * m->surface_weight, out);
  s->launches++;
  CUDA_TRY(cudaGetLastError());
  return BSPDE_OK;
}

}  // extern "C"
