// otf.cuh -- matrix-free variable-coefficient operator,
// included at the end of bspde_b200.cu after stencil.cuh (shares StencilDev,
// the CG state machine, the double-double reductions and the stencil PCG's
// vector kernels).
//
// The reference's on-the-fly operator (operator.py:217-229 over
// stencil_block / term_stencil, assembly.py:280-297, :460-472) forms, block
// by block, the (2p+1)^3 stencil of every node from the parameter fields and
// per-axis trilinear tables, then contracts it with the coefficients:
//
//   (A c)[l] = sum_{a,b} [ D[l+b] (s_z Tz'Ty Tx + s_y Tz Ty' Tx + s_x Tz Ty Tx')
//                         + mu[l+b] s_m Tz Ty Tx ][a, b] c[l+a]
//
// (T = value table, T' = derivative table of the output node's class).  No
// stencil is ever stored here.  Sum factorisation, with z-streaming:
//
//   (A c)[l] = sum_bz sum_{ay,ax} ( Wz[ay,ax](fz) C0K[bz](ly+ay, lx+ax)
//                                 + Wxy[ay,ax](fz) C0M[bz](ly+ay, lx+ax) ),
//   fz = lz + dz + bz (the field plane), with
//   Wz  = s_z (Ty (x) Tx) D,   Wxy = (s_y Ty' (x) Tx + s_x Ty (x) Tx') D + s_m (Ty (x) Tx) mu
//         (2-D separable filters of ONE field plane),
//   C0K[bz] = sum_az Tz'[az,bz] c[lz+az],  C0M[bz] = sum_az Tz[az,bz] c[lz+az]
//         (z filters of the coefficient planes).
//
// A CTA owns a 32 x 8 x-y tile and streams the field planes fz along z.  Per
// field plane it stages the D / mu plane tile and one new coefficient plane
// (a ring of B + 2p planes in shared memory), forms the x-stage of W (V =
// Tx D, U = s_x Tx' D + s_m Tx mu) and the 2B C0 planes of the B output
// planes that field plane touches, then every thread builds W for its two
// output rows column by column (y-stage, registers) and scatters it into a
// ring of B partial outputs per point (like the constant-coefficient
// kernel's z ring); the output plane that received its last field plane is
// complete and is emitted with the apply / residual / CG epilogue.  About
// 2.2 k FP64 FMAs per output (vs ~6 k for forming the stencil block and 117 k
// naive), no HBM traffic beyond the fields and vectors (32 B/DoF), and no
// memory cap: 522^3 or 240 x 240 x 960 fit next to the CG vectors.
// Supported: 3-D boxes without face terms, n_b = n_p = 1..3 (other systems
// use the assembled stencil of stencil.cuh).

namespace {

#ifndef BSPDE_OTF_RPT
#define BSPDE_OTF_RPT 1
#endif
// a CTA: 32 x 8 outputs per plane; each thread RPT rows of one column
constexpr int OTF_TX = 32, OTF_TY = 8, OTF_RPT = BSPDE_OTF_RPT, OTF_NT = 32 * OTF_TY / OTF_RPT;
constexpr int OTF_MAXNB = 3;

template <int NB>
struct OtfCfg {
  static constexpr int A = 2 * NB + 1;
  static constexpr int MW = NB;  // param_reach(n_b, n_p = n_b)
  static constexpr int B = 2 * MW + 1;
  static constexpr int HY = OTF_TY + 2 * NB, HX = OTF_TX + 2 * NB;  // coefficient / C0 tile
  static constexpr int FY = OTF_TY + B - 1, FX = OTF_TX + B - 1;    // field tile
  static constexpr int CR = B + 2 * NB;                             // coefficient ring planes
  static constexpr int CPL = HY * HX;
  static constexpr int VSZ = A * FY * OTF_TX;
  static constexpr int C0SZ = B * CPL;
  static constexpr int FSZ = FY * FX;
  static constexpr int TABD = A * B;  // one class table
};

// interior (Toeplitz-position) class tables per degree: [deg-1][d][a*B + b]
// (value d=0, derivative d=1); identical for every plan of that degree
// (unit trilinear integrals), so concurrent plans never disagree.
__constant__ double c_otf_tab[OTF_MAXNB][2][49];

// table accessors: compile-time-indexed constant-bank operands (interior
// class) or a class table in shared memory (edge rows)
template <int NB>
struct TabC {
  __device__ __forceinline__ double v(int d, int a, int b) const {
    return c_otf_tab[NB - 1][d][a * OtfCfg<NB>::B + b];
  }
};
template <int NB>
struct TabS {
  const double* t0;  // value table of the class
  const double* t1;  // derivative table
  __device__ __forceinline__ double v(int d, int a, int b) const {
    return (d ? t1 : t0)[a * OtfCfg<NB>::B + b];
  }
};

__device__ __forceinline__ int otf_mod(int q, int m) {
  const int r = q % m;
  return r < 0 ? r + m : r;
}

// x-stage of one field row position: V[ax] = sum_bx Tx[ax,bx] D,
// U[ax] = s_x sum Tx'[ax,bx] D + s_m sum Tx[ax,bx] mu
template <int NB, typename T>
__device__ __forceinline__ void otf_xstage(const T& tab, const double* F, const double* MU,
                                           double sx, double sm, double* V, double* U,
                                           int stride) {
  using C = OtfCfg<NB>;
  double f[C::B], m[C::B];
#pragma unroll
  for (int b = 0; b < C::B; ++b) {
    f[b] = F[b];
    m[b] = MU[b];
  }
#pragma unroll
  for (int ax = 0; ax < C::A; ++ax) {
    double v = 0.0, k = 0.0, w = 0.0;
#pragma unroll
    for (int b = 0; b < C::B; ++b) {
      v = fma(tab.v(0, ax, b), f[b], v);
      k = fma(tab.v(1, ax, b), f[b], k);
      w = fma(tab.v(0, ax, b), m[b], w);
    }
    V[ax * stride] = v;
    U[ax * stride] = fma(sx, k, sm * w);
  }
}

// C0 of one coefficient position for the B output planes of field plane fz
template <int NB, typename T>
__device__ __forceinline__ void otf_c0(const T& tab, const double (&cr)[OtfCfg<NB>::CR], int bz,
                                       double& ck, double& cm) {
  using C = OtfCfg<NB>;
  double k = 0.0, m = 0.0;
#pragma unroll
  for (int az = 0; az < C::A; ++az) {
    // plane lz + az - NB = base + (B-1) - bz + az
    const double cv = cr[(C::B - 1) - bz + az];
    k = fma(tab.v(1, az, bz), cv, k);
    m = fma(tab.v(0, az, bz), cv, m);
  }
  ck = k;
  cm = m;
}

// W of one output point for trial offset (ay, ax) from the thread's V / U
// column (rows i .. i + B - 1)
template <int NB, typename T>
__device__ __forceinline__ void otf_w(const T& tab, const double* v, const double* u, int ay,
                                      double sz, double sy, double& wz, double& wxy) {
  using C = OtfCfg<NB>;
  double a = 0.0, k = 0.0, m = 0.0;
#pragma unroll
  for (int b = 0; b < C::B; ++b) {
    a = fma(tab.v(0, ay, b), v[b], a);
    k = fma(tab.v(1, ay, b), v[b], k);
    m = fma(tab.v(0, ay, b), u[b], m);
  }
  wz = sz * a;
  wxy = fma(sy, k, m);
}

// MODE 0: out = A c;  1: out = r = aux - A c, sums {<b,b>, <r,D^-1 r>, <r,r>};
// 2: out = A c, sums {<c, A c>}.  diag: the Jacobi diagonal (RESID).
template <int NB, int MODE>
__global__ void __launch_bounds__(OTF_NT, 1)
    otf_apply_kernel(const StencilDev S, const double* __restrict__ dfield,
                     const double* __restrict__ mfield, const double* __restrict__ c,
                     double* __restrict__ out, const double* __restrict__ aux,
                     const double* __restrict__ diag, double* partials, unsigned* counter,
                     CgState* st, int precond, int zchunk) {
  using C = OtfCfg<NB>;
  constexpr int A = C::A, B = C::B, CR = C::CR, HX = C::HX, FY = C::FY, FX = C::FX;
  constexpr int TX = OTF_TX, TY = OTF_TY, RPT = OTF_RPT;
  if (MODE == 2 && !ld_vol(&st->active)) return;
  extern __shared__ __align__(16) double otf_smem_buf[];
  double* ring = otf_smem_buf;                 // CR planes of HY x HX
  double* c0k = ring + CR * C::CPL;            // B planes of HY x HX
  double* c0m = c0k + C::C0SZ;
  double* V = c0m + C::C0SZ;                   // [ax][FY][TX]
  double* U = V + C::VSZ;
  double* Ft = U + C::VSZ;                     // FY x FX
  double* Mt = Ft + C::FSZ;
  double* tab = Mt + C::FSZ;                   // [axis][d][ncls][A][B]
  double* s_red = tab + 6 * S.ncls * C::TABD;  // 8 warps x 8 (only 4 used)
  __shared__ unsigned s_last;

  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int ntab = 6 * S.ncls * C::TABD;
  for (int i = tid; i < ntab; i += OTF_NT) tab[i] = S.tab[i];
  // item = (x-y tile, z-chunk of zchunk output planes): a chunk streams B - 1
  // extra field planes to warm up its partial-output ring
  const int tiles_x = (S.nx + TX - 1) / TX;
  const int tiles = tiles_x * ((S.ny + TY - 1) / TY);
  const int tile = blockIdx.x % tiles, chunk = blockIdx.x / tiles;
  const int x0 = (tile % tiles_x) * TX, y0 = (tile / tiles_x) * TY;
  const int lz0 = chunk * zchunk, lz1 = min(lz0 + zchunk, S.nz);
  const int dz = S.exp_[0] - S.ex[0] - C::MW, dy = S.exp_[1] - S.ex[1] - C::MW,
            dx = S.exp_[2] - S.ex[2] - C::MW;
  const int ewz = S.ew[0], ewy = S.ew[1], ewx = S.ew[2];
  const double sz = S.s_stiff[0], sy = S.s_stiff[1], sx = S.s_stiff[2], sm = S.s_mass;
  auto tabp = [&](int axis, int d, int cls) -> const double* {
    return tab + (((axis * 2 + d) * S.ncls) + cls) * C::TABD;
  };
  // this thread's output points: rows y0 + 2 warp + i, column x0 + lane
  const int r0 = OTF_RPT * warp;
  const int gx = x0 + lane;
  int cyi[RPT];
  bool rowok[RPT];
#pragma unroll
  for (int i = 0; i < RPT; ++i) {
    const int gy = y0 + r0 + i;
    rowok[i] = gy < S.ny && gx < S.nx;
    cyi[i] = gy < S.ny ? st_cls(gy, S.ny, ewy) : ewy;
  }
  const bool rows_int = cyi[0] == ewy && cyi[RPT - 1] == ewy;
  double acc[B][RPT];
#pragma unroll
  for (int k = 0; k < B; ++k)
#pragma unroll
    for (int i = 0; i < RPT; ++i) acc[k][i] = 0.0;
  double dsh[3] = {0.0, 0.0, 0.0}, dsl[3] = {0.0, 0.0, 0.0};

  auto load_cplane = [&](int q) {
    double* dst = ring + otf_mod(q, CR) * C::CPL;
    const bool zok = q >= 0 && q < S.nz;
    for (int e = tid; e < C::CPL; e += OTF_NT) {
      const int my = e / HX, mx = e - my * HX;
      const int gyy = y0 - NB + my, gxx = x0 - NB + mx;
      dst[e] = (zok && gyy >= 0 && gyy < S.ny && gxx >= 0 && gxx < S.nx)
                   ? c[((long long)q * S.ny + gyy) * S.nx + gxx]
                   : 0.0;
    }
  };
  // ring: planes [fz - dz - (B-1) - NB, fz - dz + NB] at field plane fz
  const int fz0 = lz0 + dz, fz1 = lz1 - 1 + dz + B - 1;
  for (int i = tid; i < CR * C::CPL; i += OTF_NT) ring[i] = 0.0;
  __syncthreads();
  for (int q = fz0 - dz - (B - 1) - NB; q < fz0 - dz + NB; ++q)
    if (q >= 0 && q < S.nz) load_cplane(q);

  for (int fz = fz0; fz <= fz1; ++fz) {
    // ---- stage: newest coefficient plane, field plane tiles ----
    load_cplane(fz - dz + NB);
    const bool fok = fz >= 0 && fz < S.pz;
    for (int e = tid; e < C::FSZ; e += OTF_NT) {
      const int ty = e / FX, tx = e - ty * FX;
      const int fy = y0 + dy + ty, fx = x0 + dx + tx;
      const bool ok = fok && fy >= 0 && fy < S.py && fx >= 0 && fx < S.px;
      const long long off = ((long long)fz * S.py + fy) * S.px + fx;
      Ft[e] = ok ? dfield[off] : 0.0;
      Mt[e] = ok ? mfield[off] : 0.0;
    }
    __syncthreads();
    // ---- x-stage of W (V, U) and the C0 planes ----
    for (int e = tid; e < FY * TX; e += OTF_NT) {
      const int ty = e / TX, lx = e - ty * TX;
      const int gxx = x0 + lx;
      const int cx = gxx < S.nx ? st_cls(gxx, S.nx, ewx) : ewx;
      if (cx == ewx)
        otf_xstage<NB>(TabC<NB>{}, Ft + ty * FX + lx, Mt + ty * FX + lx, sx, sm,
                       V + ty * TX + lx, U + ty * TX + lx, FY * TX);
      else
        otf_xstage<NB>(TabS<NB>{tabp(2, 0, cx), tabp(2, 1, cx)}, Ft + ty * FX + lx,
                       Mt + ty * FX + lx, sx, sm, V + ty * TX + lx, U + ty * TX + lx, FY * TX);
    }
    {
      const int base = fz - dz - (B - 1) - NB;  // oldest ring plane
      int slot[CR];
#pragma unroll
      for (int k = 0; k < CR; ++k) slot[k] = otf_mod(base + k, CR) * C::CPL;
      for (int e = tid; e < C::CPL; e += OTF_NT) {
        double cr[CR];
#pragma unroll
        for (int k = 0; k < CR; ++k) cr[k] = ring[slot[k] + e];
#pragma unroll
        for (int bz = 0; bz < B; ++bz) {
          const int lz = fz - dz - bz;
          double ck = 0.0, cm = 0.0;
          if (lz >= 0 && lz < S.nz) {
            const int cz = st_cls(lz, S.nz, ewz);
            if (cz == ewz)
              otf_c0<NB>(TabC<NB>{}, cr, bz, ck, cm);
            else
              otf_c0<NB>(TabS<NB>{tabp(0, 0, cz), tabp(0, 1, cz)}, cr, bz, ck, cm);
          }
          c0k[bz * C::CPL + e] = ck;
          c0m[bz * C::CPL + e] = cm;
        }
      }
    }
    __syncthreads();
    // ---- y-stage + scatter into the B partial outputs of each point ----
#pragma unroll 1
    for (int ax = 0; ax < A; ++ax) {
      double v[RPT + B - 1], u[RPT + B - 1];
#pragma unroll
      for (int k = 0; k < RPT + B - 1; ++k) {
        v[k] = V[(ax * FY + r0 + k) * TX + lane];
        u[k] = U[(ax * FY + r0 + k) * TX + lane];
      }
#pragma unroll
      for (int m = 0; m < RPT + A - 1; ++m) {  // C0 row r0 + m serves (i, ay = m - i)
        double gk[B], gm[B];
        const int e = (r0 + m) * HX + lane + ax;
#pragma unroll
        for (int bz = 0; bz < B; ++bz) {
          gk[bz] = c0k[bz * C::CPL + e];
          gm[bz] = c0m[bz * C::CPL + e];
        }
#pragma unroll
        for (int i = 0; i < RPT; ++i) {
          const int ay = m - i;
          if (ay < 0 || ay >= A) continue;
          double wz, wxy;
          if (rows_int)
            otf_w<NB>(TabC<NB>{}, v + i, u + i, ay, sz, sy, wz, wxy);
          else
            otf_w<NB>(TabS<NB>{tabp(1, 0, cyi[i]), tabp(1, 1, cyi[i])}, v + i, u + i, ay, sz,
                      sy, wz, wxy);
#pragma unroll
          for (int bz = 0; bz < B; ++bz) acc[bz][i] = fma(wz, gk[bz], fma(wxy, gm[bz], acc[bz][i]));
        }
      }
    }
    // ---- output plane lz = fz - dz - (B - 1) is complete ----
    const int lz = fz - dz - (B - 1);
    if (lz >= lz0 && lz < lz1) {
      double g0 = 0.0, g1 = 0.0, g2 = 0.0;
#pragma unroll
      for (int i = 0; i < RPT; ++i) {
        if (!rowok[i]) continue;
        const long long l = ((long long)lz * S.ny + (y0 + r0 + i)) * S.nx + gx;
        const double t = acc[B - 1][i];
        if (MODE == 0) {
          out[l] = t;
        } else if (MODE == 1) {
          const double bb = aux[l];
          const double r = bb - t;
          out[l] = r;
          const double dg = diag[l];
          const double inv = (precond && dg != 0.0) ? 1.0 / dg : 1.0;
          g0 = fma(bb, bb, g0);
          g1 = fma(r, __dmul_rn(inv, r), g1);
          g2 = fma(r, r, g2);
        } else {
          out[l] = t;
          const double cv = ring[otf_mod(lz, CR) * C::CPL + (r0 + i + NB) * HX + lane + NB];
          g0 = fma(cv, t, g0);
        }
      }
      if (MODE != 0) dd_add(dsh[0], dsl[0], g0);
      if (MODE == 1) {
        dd_add(dsh[1], dsl[1], g1);
        dd_add(dsh[2], dsl[2], g2);
      }
    }
#pragma unroll
    for (int k = B - 1; k > 0; --k)
#pragma unroll
      for (int i = 0; i < RPT; ++i) acc[k][i] = acc[k - 1][i];
#pragma unroll
    for (int i = 0; i < RPT; ++i) acc[0][i] = 0.0;
    __syncthreads();  // the next plane overwrites the tiles, V, U and C0
  }
  if (MODE == 1) {
    double vh[3] = {dsh[0], dsh[1], dsh[2]}, vl[3] = {dsl[0], dsl[1], dsl[2]};
    reduce_and_finalize<3, OTF_NT / 32>(vh, vl, s_red, &s_last, partials, counter, st, 1, 0);
  } else if (MODE == 2) {
    double vh[1] = {dsh[0]}, vl[1] = {dsl[0]};
    reduce_and_finalize<1, OTF_NT / 32>(vh, vl, s_red, &s_last, partials, counter, st, 1, 1);
  }
}

// Jacobi diagonal P[center, l] of the on-the-fly operator (the stencil's
// centre entry, same sum as stencil_assemble_kernel restricted to a = 0)
__global__ void __launch_bounds__(ST_NT) otf_diag_kernel(const StencilDev S,
                                                         const double* __restrict__ dfield,
                                                         const double* __restrict__ mfield,
                                                         double* __restrict__ diag) {
  const int c = S.nb;  // centre trial offset index
  for (long long l = blockIdx.x * (long long)blockDim.x + threadIdx.x; l < S.N;
       l += (long long)gridDim.x * blockDim.x) {
    const int lx = (int)(l % S.nx), ly = (int)((l / S.nx) % S.ny),
              lz = (int)(l / ((long long)S.nx * S.ny));
    const int cz = st_cls(lz, S.nz, S.ew[0]), cy = st_cls(ly, S.ny, S.ew[1]),
              cx = st_cls(lx, S.nx, S.ew[2]);
    const double* tz0 = st_tab(S, S.tab, 0, 0, cz) + c * S.B;
    const double* tz1 = st_tab(S, S.tab, 0, 1, cz) + c * S.B;
    const double* ty0 = st_tab(S, S.tab, 1, 0, cy) + c * S.B;
    const double* ty1 = st_tab(S, S.tab, 1, 1, cy) + c * S.B;
    const double* tx0 = st_tab(S, S.tab, 2, 0, cx) + c * S.B;
    const double* tx1 = st_tab(S, S.tab, 2, 1, cx) + c * S.B;
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
          const double kd = (k_z + k_y) * tx0[bx] + k_x * tx1[bx];
          acc = fma(dfield[row + fx], kd, fma(mfield[row + fx], m_zy * tx0[bx], acc));
        }
      }
    }
    diag[l] = acc;
  }
}

template <int NB>
size_t otf_smem(const StencilDev& S) {
  using C = OtfCfg<NB>;
  return 8 * ((size_t)C::CR * C::CPL + 2 * C::C0SZ + 2 * C::VSZ + 2 * C::FSZ +
              6 * (size_t)S.ncls * C::TABD + 8 * 8);
}

template <int NB, int MODE>
int otf_launch_nb(const bspde_stencil* s, cudaStream_t st, const double* c, double* out,
                  const double* aux, double* partials, unsigned* counter, CgState* state,
                  int precond) {
  const size_t smem = otf_smem<NB>(s->S);
  const void* fn = reinterpret_cast<const void*>(&otf_apply_kernel<NB, MODE>);
  static bool attr = false;
  if (!attr) {
    CUDA_TRY(cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
    attr = true;
  }
  const int tiles = ((s->S.nx + OTF_TX - 1) / OTF_TX) * ((s->S.ny + OTF_TY - 1) / OTF_TY);
  if (tiles > MAXGRID && MODE != 0) return fail(BSPDE_ERR_STATE, "OTF grid exceeds MAXGRID");
  // z-chunks: one CTA per (tile, chunk), chosen to minimise waves x (chunk +
  // B - 1 warm-up planes) -- a small x-y grid (240 x 240: 240 tiles on 148
  // SMs) would otherwise run 1.6 waves
  static int nsm = 0;
  if (!nsm) {
    int dev = 0;
    CUDA_TRY(cudaGetDevice(&dev));
    CUDA_TRY(cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, dev));
  }
  const int nz = s->S.nz;
  int zchunk = nz;
  if (const char* e = getenv("BSPDE_OTF_ZCHUNK")) zchunk = std::max(1, atoi(e));
  else {
    double best = 1e300;
    for (int nc = 1; nc <= nz; ++nc) {
      const int len = (nz + nc - 1) / nc;
      const int ncr = (nz + len - 1) / len;
      if ((long long)tiles * ncr > MAXGRID) break;
      const long long waves = ((long long)tiles * ncr + nsm - 1) / nsm;
      const double cost = (double)waves * (len + OtfCfg<NB>::B - 1);
      if (cost < best * (1.0 - 1e-9)) {
        best = cost;
        zchunk = len;
      }
    }
  }
  const int grid = tiles * ((nz + zchunk - 1) / zchunk);
  if (grid > MAXGRID && MODE != 0) return fail(BSPDE_ERR_STATE, "OTF grid exceeds MAXGRID");
  otf_apply_kernel<NB, MODE><<<grid, OTF_NT, smem, st>>>(s->S, s->otf_d, s->otf_m, c, out, aux,
                                                         s->otf_diag, partials, counter, state,
                                                         precond, zchunk);
  return BSPDE_OK;
}

template <int MODE>
int otf_launch(const bspde_stencil* s, cudaStream_t st, const double* c, double* out,
               const double* aux, double* partials, unsigned* counter, CgState* state,
               int precond) {
  switch (s->S.nb) {
    case 1: return otf_launch_nb<1, MODE>(s, st, c, out, aux, partials, counter, state, precond);
    case 2: return otf_launch_nb<2, MODE>(s, st, c, out, aux, partials, counter, state, precond);
    default: return otf_launch_nb<3, MODE>(s, st, c, out, aux, partials, counter, state, precond);
  }
}

int otf_check(bspde_stencil* s) {
  if (int rc = st_check(s)) return rc;
  if (!s->otf_d || !s->otf_m || !s->otf_diag)
    return fail(BSPDE_ERR_STATE, "on-the-fly operator not prepared (bspde_otf_prepare)");
  return BSPDE_OK;
}

}  // namespace

extern "C" {

int bspde_otf_supported(const bspde_stencil* s) {
  if (!s) return 0;
  const auto& S = s->S;
  return (S.nb >= 1 && S.nb <= OTF_MAXNB && S.np == S.nb && S.nfaces == 0 && !S.degen[0] &&
          !S.degen[1] && !S.degen[2])
             ? 1
             : 0;
}

int bspde_otf_prepare(bspde_stencil* s, const double* dfield, const double* mfield, double* diag,
                      void* stream) {
  if (int rc = st_check(s)) return rc;
  if (!bspde_otf_supported(s))
    return fail(BSPDE_ERR_ARG, "on-the-fly operator: 3-D box, no face terms, n_b = n_p <= 3");
  if (!dfield || !mfield || !diag) return fail(BSPDE_ERR_ARG, "null argument");
  // interior class tables of this degree -> constant bank (same values for
  // every plan of the degree)
  {
    const int nb = s->S.nb, A = s->S.A, B = s->S.B;
    std::vector<double> h((size_t)2 * 49, 0.0);
    for (int d = 0; d < 2; ++d)
      for (int e = 0; e < A * B; ++e)
        h[d * 49 + e] = s->host_tab[((size_t)(2 * 2 + d) * s->S.ncls + s->d.ew[2]) * A * B + e];
    CUDA_TRY(cudaMemcpyToSymbolAsync(c_otf_tab, h.data(), h.size() * sizeof(double),
                                     (size_t)(nb - 1) * 2 * 49 * sizeof(double),
                                     cudaMemcpyHostToDevice, (cudaStream_t)stream));
  }
  s->otf_d = dfield;
  s->otf_m = mfield;
  s->otf_diag = diag;
  otf_diag_kernel<<<st_grid(s, s->S.N), ST_NT, 0, (cudaStream_t)stream>>>(s->S, dfield, mfield,
                                                                          diag);
  s->launches++;
  CUDA_TRY(cudaGetLastError());
  return BSPDE_OK;
}

int bspde_otf_apply(bspde_stencil* s, const double* c, double* out, void* stream) {
  if (int rc = otf_check(s)) return rc;
  if (!c || !out) return fail(BSPDE_ERR_ARG, "null argument");
  if (int rc = otf_launch<0>(s, (cudaStream_t)stream, c, out, nullptr, nullptr, nullptr, nullptr,
                             0))
    return rc;
  s->launches++;
  CUDA_TRY(cudaGetLastError());
  return BSPDE_OK;
}

int bspde_otf_pcg(bspde_stencil* s, const double* b, double* x, double* r, double* p, double* ap,
                  void* scratch, double* history, const bspde_cg_config* cfg,
                  bspde_cg_report* report, int32_t precond, void* stream) {
  if (int rc = otf_check(s)) return rc;
  // the stencil PCG's vector kernels read the Jacobi diagonal as the centre
  // slice of P: point P at diag - centre * N
  const int A = s->S.A, hb = s->S.nb;
  const long long center = (long long)(hb * A + hb) * A + hb;
  const double* Pc = s->otf_diag - center * s->S.N;
  return st_pcg(s, Pc, b, x, r, p, ap, scratch, history, cfg, report, precond, stream,
                /*otf=*/true);
}

}  // extern "C"
