// bspde_b200.cu -- sm_100a kernels and C ABI for the tensor B-spline
// (M + dt K) apply, Jacobi-PCG and RHS assembly.  See include/bspde_b200.h
// and DESIGN.md.
//
// Kernel family `sep_kernel<P, MODE>`: a persistent 2.5-D streaming apply of
//   A = Mz(x)(My(x)(c_mass Mx + cx Kx) + cy Ky(x)Mx) + cz Kz(x)My(x)Mx
// Work item = (32x32 x-y tile, z-chunk).  Per input z-plane:
//   1. TMA (cp.async.bulk.tensor.3d) lands the haloed (32+2p)^2 plane tile in
//      shared memory (out-of-bounds x/y -> zeros; z ghost planes are zeros or
//      the neighbour slab's planes),
//   2. [CG pass A] p = D^-1 r + beta p_old is formed in place on the tile,
//   3. x-pass: u1 = Mx c, u2 = Kx c for all 32+2p rows -> shared memory,
//   4. y-pass: wm = My u1, wa = My(c_mass u1 + cx u2) + cy Ky u1 in registers,
//   5. z-pass: scatter wa, wm of this plane into a register ring of 2p+1
//      partial outputs (the z-Gram factors are symmetric, so the scatter uses
//      row z' of Mz/Kz); the output plane z'-p is complete and is emitted with
//      the mode's epilogue (plain store / mass+axpy / residual / CG dot).
// Edge rows (non-Toeplitz first/last ew rows of each axis) use per-class
// tables in shared memory on warp/plane-uniform slow paths.
//
// Reference algorithm this replaces: stencil_block + _contract_block
// (/root/reference/pkg/src/bspde/assembly.py:460-472, operator.py:77-89,
// operator.py:217-229) and the pcg loop (solver.py:51-117).

#include "../../include/bspde_b200.h"
#include "gram_taps.cuh"

#include <cuda.h>
#include <cuda_runtime.h>

#include <algorithm>
#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <map>
#include <string>
#include <tuple>
#include <type_traits>
#include <vector>

namespace {

// ---------------------------------------------------------------------------
// configuration
//
// One persistent CTA per SM.  Warp w owns output columns 32*(w&1) .. +31
// (one per lane) and output rows 4*(w>>1) .. +3 of the 64 x TY tile (the z
// ring of those 4 points lives in its registers); for the x-pass and the CG
// p-formation it owns whole haloed rows w, w+NW, w+2NW.  p <= 3: 16 warps
// (512 threads, 128 registers), 64x32 tiles.  p >= 4: the ring of 2p+p
// doubles per point needs more registers: 12 warps (384 threads, 168
// registers), 64x24 tiles.
constexpr int TX = 64;               // tile width (x)
constexpr int RPT = 4;               // output rows per thread
constexpr int MAXP = 5;
constexpr int MAXTAP = 2 * MAXP + 1;

// BSPDE_W_LOWP (tuning build): warps per CTA for p <= 3 (16: 128 registers;
// 12: 168 registers, 64 x 24 tiles)
#ifndef BSPDE_W_LOWP
#define BSPDE_W_LOWP 16
#endif
// fused heat residual: F's owned tile of the output plane is staged by TMA
// with the input plane instead of prefetched into registers (Cfg::AS)
#ifndef BSPDE_AUX_TMA
#define BSPDE_AUX_TMA 1
#endif
// Per (degree, mode): CG pass A at p = 3 carries the p ring and the x update
// and runs 12 warps with 168 registers (64 x 24 tiles; 16 warps spill at the
// 128-register cap); the other p <= 3 kernels run 16 warps (64 x 32 tiles)
#ifndef BSPDE_W_CGA3
#define BSPDE_W_CGA3 12
#endif
__host__ __device__ constexpr int warps_of(int p, int mode) {
  return p <= 3 ? ((p == 3 && (mode == 3 /* M_CGA */ || mode == 4 /* M_HRES */)) ? BSPDE_W_CGA3
                                                                                 : BSPDE_W_LOWP)
                : 12;
}
__host__ __device__ constexpr int tile_h_of(int p, int mode) { return RPT * warps_of(p, mode) / 2; }

template <int P, int MODE>
struct Geo {
  static constexpr int NW = warps_of(P, MODE);   // warps (2 x-groups)
  static constexpr int NT = 32 * NW;       // threads
  static constexpr int TY = tile_h_of(P, MODE);  // tile height (y)
};

// M_HRES: the heat step's first residual fused with its right-hand side,
// r0 = (rhs_cm (Mz(x)My(x)Mx) u + a F) - A u with the three initial sums,
// b never stored (a second z ring carries the pure mass apply)
enum Mode { M_APPLY = 0, M_MASS = 1, M_RESID = 2, M_CGA = 3, M_HRES = 4 };

__host__ __device__ constexpr int edge_width_of(int p) {
  return p == 1 ? 1 : (p <= 3 ? 3 : 5);
}

template <int P, int MODE>
struct Cfg {
  static constexpr int NW = Geo<P, MODE>::NW, NT = Geo<P, MODE>::NT, TY = Geo<P, MODE>::TY;
  static constexpr int R = 2 * P + 1;
  // TMA needs the box's inner start (x0 - PX) * 8 bytes to be 16-byte aligned:
  // the x halo is padded to an even width PX (odd p: one extra column per side)
  static constexpr int PX = P + (P & 1);
  static constexpr int DX = PX - P;  // 0 or 1: first used column of a window
  static constexpr int HX = TX + 2 * PX;
  static constexpr int HY = TY + 2 * P;
  static constexpr int EW = edge_width_of(P);
  static constexpr int NC = 2 * EW + 1;          // max classes per axis
  static constexpr int NA = (MODE == M_CGA) ? 2 : 1;   // staged arrays per plane
  static constexpr int NS = (MODE == M_CGA) ? 3 : 4;  // TMA stages (fits 227 KB for p = 1..5)
  static constexpr bool STIFF = (MODE != M_MASS);
  static constexpr bool INVD = (MODE == M_CGA || MODE == M_RESID || MODE == M_HRES);
  static constexpr int ARR = HX * HY;                        // doubles
  static constexpr int ARR_D = ((ARR * 8 + 127) / 128) * 16; // doubles, 128B-rounded
  static constexpr int XARR = HY * TX;                       // doubles per X array
  static constexpr int TAB = 6 * NC * R;                     // doubles
  static constexpr int INV = INVD ? NC * NC * NC : 0;
  static constexpr int AST = TX * TY;  // doubles per staged aux tile
  static constexpr size_t BASE_BYTES =
      (size_t)8 * (NS * NA * ARR_D + 2 * 2 * XARR + TAB + INV + NW * 8 + 2) + 8 * NS;
  static constexpr bool AS = (MODE == M_HRES) && BSPDE_AUX_TMA &&
                             BASE_BYTES + (size_t)8 * NS * AST <= 227 * 1024;
  static constexpr int AS_D = AS ? NS * AST : 0;
  static constexpr size_t smem_bytes() { return BASE_BYTES + (size_t)8 * AS_D; }
};

// Search directions live in a ring of R <= kPRing fields (R = CgState::ring,
// 2 or 4): iteration k writes p_k to field k % R and its pass A applies
// x += alpha_{k-1} p_{k-1} from field (k-1) % R; the flush at the end of a
// solve applies the last update (x_flush_kernel)
constexpr int kPRing = BSPDE_P_RING;

struct CgState {
  double sums[4];        // the dot products of the last pass (fuse = 1: rounded totals;
  double sums_lo[4];     // fuse = 0: this rank's double-double pairs sums + sums_lo)
  double rz, alpha, beta, pAp;
  double res, res0, scale, tol;
  double rhs_norm, pad_d;
  int it, max_iter, active, status;
  int record_history, has_x0, x_done, ring;  // x_done: iterations applied to x; ring: R
  double* history;
  double alpha_ring[kPRing];  // alpha_j at j % R for the pending x updates
};

struct SepParams {
  int nx, ny, nz, nz_glob, z_off, ghost;
  long long pitch_y, pitch_z;
  int ew[3];
  int tiles_x, tiles_y, nchunks, chunk_len, nitems;
  int z_begin, z_end;  // owned output planes [z_begin, z_end) this launch produces
  int main_items, tail_split, sub_len;  // items >= main_items: tail chunks split tail_split ways
  int zfast;  // 1: interior z rows use the compile-time taps (0 for a degenerate z axis)
  double tzm[MAXTAP], tzk[MAXTAP], tym[MAXTAP], tyk[MAXTAP], txm[MAXTAP], txk[MAXTAP];
  double gm[MAXTAP], gk[MAXTAP];  // unit interior Gram taps (BSPDE_PARAM_TAPS builds)
  double c_mass, cx, cy, cz;     // cz is folded into tzk; kept for edge rows
  const double* tab;             // device: [axis][kind][NC*R] (NC = class stride)
  const double* invd;            // device: NCz*NCy*NCx
  double* out;
  const double* aux;
  double aux_scale;
  double rhs_cm;       // M_HRES: mass scale of the right-hand side (vol)
  const double* cg_r;  // CG pass A: r and p_old (TMA-staged with their halos)
  const double* cg_p;
  double* cg_pout;     // CG pass A: p_k at owned points (ping-pong partner of cg_p)
  double* cg_x;        // CG pass A: x += alpha_{k-1} p_{k-1} at owned points (k >= 1)
  double* partials;
  unsigned* counter;
  CgState* state;
  int fuse;
  int accumulate;  // 1: add this launch's sums to the state's (a z-ranged piece)
};

// BSPDE_ALL_EDGE=1 (measurement build): every tile takes the edge-tile
// path, to weigh edge against interior tiles in the launch planner.
#ifndef BSPDE_ALL_EDGE
#define BSPDE_ALL_EDGE 0
#endif
// Interior taps of the fast paths: compile-time immediates (measured faster
// than __constant__ or kernel-parameter operands; profiles/r01_ncu_summary.md).
#ifndef BSPDE_PARAM_TAPS
#define BSPDE_PARAM_TAPS 0
#endif
// Interior taps: compile-time immediates, except in CG pass A, whose DFMAs
// take them as constant-bank operands (kernel parameters): the immediates are
// rematerialised through uniform registers every plane there (measured -1%
// pass A time at 930^3 with params; the other modes are better with
// immediates).  BSPDE_PARAM_TAPS=1 uses parameters everywhere (tuning).
template <int P, int MODE>
struct TapSrc {
  const SepParams& prm;
  static constexpr bool PARAM = BSPDE_PARAM_TAPS || MODE == 3 /* M_CGA */;
  __device__ __forceinline__ double M(int k) const {
    return PARAM ? prm.gm[k] : GramTaps<P>::M(k);
  }
  __device__ __forceinline__ double K(int k) const {
    return PARAM ? prm.gk[k] : GramTaps<P>::K(k);
  }
};

struct PassBParams {
  int nx, ny, nz, nz_glob, z_off, ghost;
  long long pitch_y, pitch_z;
  int ew[3];
  int rows_per_cta;
  const double* invd;
  double* x;
  double* r;
  const double* pring;    // R fields, pstride doubles apart
  long long pstride;
  const double* ap;
  double* partials;
  unsigned* counter;
  CgState* state;
  int fuse;
  // z-slab peer halos: the new r and the preceding pass A's p_k of the first /
  // last `ghost` owned planes are also stored into the lower / upper
  // neighbour's ghost planes (NVLink peer memory / CUDA IPC; the lower
  // neighbour owns nz_lo planes)
  double* peer_lo;
  double* peer_hi;
  const double* p_src;
  double* p_lo;
  double* p_hi;
  int nz_lo;
};

// ---------------------------------------------------------------------------
// PTX helpers: mbarrier + TMA

__device__ __forceinline__ uint32_t smem_u32(const void* p) {
  return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}

__device__ __forceinline__ void mbar_init(uint64_t* bar, uint32_t count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count)
               : "memory");
}

__device__ __forceinline__ void mbar_expect_tx(uint64_t* bar, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)),
               "r"(bytes)
               : "memory");
}

// try_wait with a suspend-time hint: the warp sleeps in hardware until the
// phase completes (or the hint expires) instead of re-polling, so waiting
// warps do not steal issue slots from the working role on the same SMSP.
__device__ __forceinline__ bool mbar_try_wait(uint32_t addr, uint32_t phase) {
  uint32_t ok;
  asm volatile(
      "{\n\t.reg .pred p;\n\t"
      "mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2, %3;\n\t"
      "selp.u32 %0, 1, 0, p;\n\t}"
      : "=r"(ok)
      : "r"(addr), "r"(phase), "r"(1000000u)
      : "memory");
  return ok != 0;
}

__device__ __forceinline__ void mbar_wait(uint64_t* bar, uint32_t phase) {
  const uint32_t a = smem_u32(bar);
  while (!mbar_try_wait(a, phase)) {
  }
}

__device__ __forceinline__ void tma_load_3d(void* dst, const CUtensorMap* map, int x, int y,
                                            int z, uint64_t* bar) {
  asm volatile(
      "cp.async.bulk.tensor.3d.shared::cluster.global.tile.mbarrier::complete_tx::bytes"
      " [%0], [%1, {%2, %3, %4}], [%5];" ::"r"(smem_u32(dst)),
      "l"(reinterpret_cast<uint64_t>(map)), "r"(x), "r"(y), "r"(z), "r"(smem_u32(bar))
      : "memory");
}

__device__ __forceinline__ void fence_proxy_async() {
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
}

__device__ __forceinline__ void fence_mbar_init() {
  asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
}

__device__ __forceinline__ int cls_of(int g, int n, int ew) {
  return g < ew ? g : (g >= n - ew ? 2 * ew - (n - 1 - g) : ew);
}

// The CG search direction p = z + beta*p_old with z = r*inv_diag, rounded in
// the reference's order (solver.py:96-100: z = r*inv_diag; p = z + beta*p) and
// bitwise identical in pass A and pass B.
__device__ __forceinline__ double pdir(double r, double invd, double pold, double beta) {
  return __dadd_rn(__dmul_rn(r, invd), __dmul_rn(beta, pold));
}

template <typename T>
__device__ __forceinline__ T ld_vol(const T* p) {
  return *reinterpret_cast<const volatile T*>(p);
}

// ---------------------------------------------------------------------------
// scalar state machine (device).  Mirrors solver.py:63-108 step by step.

__device__ void update_active(CgState* s) {
  if (!(s->res / s->scale > s->tol)) {
    s->status = BSPDE_CG_CONVERGED;
    s->active = 0;
  } else if (s->it >= s->max_iter) {
    s->status = BSPDE_CG_MAXITER;
    s->active = 0;
  } else {
    s->status = BSPDE_CG_RUNNING;
    s->active = 1;
  }
}

// kind 0: after r = b - A x0           (solver.py:63-83)
// kind 1: after Ap, <p,Ap>              (solver.py:88-93)
// kind 2: after x, r updates, <r,z>     (solver.py:96-108)
__device__ void finalize_state(CgState* s, int kind) {
  if (kind == 0) {
    const double bb = s->sums[0], rz = s->sums[1], rr = s->sums[2];
    s->rhs_norm = sqrt(bb);
    s->it = 0;
    s->beta = 0.0;
    s->x_done = 0;
    if (s->rhs_norm == 0.0 && !s->has_x0) {
      s->status = BSPDE_CG_ZERO_RHS;
      s->active = 0;
      s->res = 0.0;
      s->res0 = 0.0;
      s->scale = 1.0;
      s->rz = 0.0;
      if (s->record_history) s->history[0] = 0.0;
      return;
    }
    s->scale = s->rhs_norm > 0.0 ? s->rhs_norm : 1.0;
    s->rz = rz;
    s->res = sqrt(rr);
    s->res0 = s->res;
    if (s->record_history) s->history[0] = sqrt(fmax(rz, 0.0));
    update_active(s);
  } else if (kind == 1) {
    const double pAp = s->sums[0];
    // pass A of iteration it applied x += alpha_j p_j for j < it
    s->x_done = s->it;
    s->pAp = pAp;
    if (pAp <= 0.0) {
      s->status = BSPDE_CG_INDEFINITE;
      s->active = 0;
      return;
    }
    s->alpha = s->rz / pAp;
  } else {
    const double rz_new = s->sums[0], rr = s->sums[1];
    // alpha_k for the x update of the next pass A / the final flush
    s->alpha_ring[s->it % s->ring] = s->alpha;
    s->beta = rz_new / s->rz;
    s->rz = rz_new;
    s->res = sqrt(rr);
    s->it += 1;
    if (s->record_history) s->history[s->it] = sqrt(fmax(rz_new, 0.0));
    if (s->res > 1e3 * s->res0) {
      s->status = BSPDE_CG_DIVERGED;
      s->active = 0;
      return;
    }
    update_active(s);
  }
}

// kind 3: the pending x updates have been applied (after x_flush_kernel)
__global__ void finalize_kernel(CgState* s, int kind) {
  if (threadIdx.x == 0 && blockIdx.x == 0) {
    if (kind == 3) {
      s->x_done = s->it;
      return;
    }
    if (kind != 0 && !s->active) return;
    for (int i = 0; i < 4; ++i) {  // round the (single-rank) double-double pairs
      s->sums[i] = __dadd_rn(s->sums[i], s->sums_lo[i]);
      s->sums_lo[i] = 0.0;
    }
    finalize_state(s, kind);
  }
}

// Double-double ("compensated") accumulation of the CG scalars.  Every dot
// product is accumulated as an unevaluated sum hi + lo: small position-
// determined groups of terms (a thread's 4 output rows of one plane in pass
// A, a row pair in pass B) are summed with plain FMAs, and everything above
// that -- a thread's groups, the warp, the CTA and the grid -- is added with
// error-free transformations (Knuth TwoSum).  The total is then the sum of
// the group sums to ~1e-32 relative, i.e. correctly rounded except at near
// ties: the scalars, hence the CG iterates, do not depend on the tile
// geometry, the CTA count or the number of z-slabs (the reference itself
// sums with numpy/BLAS; correctly rounded dots reproduce its iteration
// counts).
__device__ __forceinline__ void dd_add(double& hi, double& lo, double x) {
  const double s = __dadd_rn(hi, x);
  const double bp = __dsub_rn(s, hi);
  const double e = __dadd_rn(__dsub_rn(hi, __dsub_rn(s, bp)), __dsub_rn(x, bp));
  hi = s;
  lo = __dadd_rn(lo, e);
}

__device__ __forceinline__ void dd_add2(double& hi, double& lo, double xhi, double xlo) {
  dd_add(hi, lo, xhi);
  lo = __dadd_rn(lo, xlo);
}

// Multi-rank scalar update: `gathered` holds every rank's 8 doubles
// (sums[4], sums_lo[4]; rank-major, the all-gather of the first 64 bytes of
// each rank's scratch).  The pairs are added in rank order in double-double
// and rounded once, so every rank computes the same scalars -- equal to the
// single-device ones (the total is the correctly rounded dot either way).
__global__ void finalize_gathered_kernel(CgState* s, const double* gathered, int world, int kind) {
  if (threadIdx.x == 0 && blockIdx.x == 0) {
    if (kind != 0 && !s->active) return;
    for (int i = 0; i < 4; ++i) {
      double h = 0.0, l = 0.0;
      for (int r = 0; r < world; ++r) dd_add2(h, l, gathered[r * 8 + i], gathered[r * 8 + 4 + i]);
      s->sums[i] = __dadd_rn(h, l);
      s->sums_lo[i] = 0.0;
    }
    finalize_state(s, kind);
  }
}

// Deterministic block reduction of NV double-double values (hi, lo), per-CTA
// partials (hi, lo pairs), then the last CTA to finish reduces the partials
// in fixed order (and optionally runs the scalar update).  s_red must hold
// NWARP*8 doubles.
template <int NV, int NWARP>
__device__ void reduce_and_finalize(double (&vh)[NV], double (&vl)[NV], double* s_red,
                                    unsigned* s_last_p, double* partials, unsigned* counter,
                                    CgState* st, int fuse, int kind, int accumulate = 0) {
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
#pragma unroll
  for (int i = 0; i < NV; ++i) {
#pragma unroll
    for (int off = 16; off > 0; off >>= 1) {
      const double oh = __shfl_xor_sync(0xffffffffu, vh[i], off);
      const double ol = __shfl_xor_sync(0xffffffffu, vl[i], off);
      dd_add2(vh[i], vl[i], oh, ol);
    }
  }
  if (lane == 0) {
#pragma unroll
    for (int i = 0; i < NV; ++i) {
      s_red[warp * 8 + 2 * i] = vh[i];
      s_red[warp * 8 + 2 * i + 1] = vl[i];
    }
  }
  __syncthreads();
  unsigned& s_last = *s_last_p;
  if (threadIdx.x == 0) {
#pragma unroll
    for (int i = 0; i < NV; ++i) {
      double h = 0.0, l = 0.0;
      for (int w = 0; w < NWARP; ++w) dd_add2(h, l, s_red[w * 8 + 2 * i], s_red[w * 8 + 2 * i + 1]);
      partials[blockIdx.x * 8 + 2 * i] = h;
      partials[blockIdx.x * 8 + 2 * i + 1] = l;
    }
    __threadfence();
    const unsigned ticket = atomicAdd(counter, 1u);
    s_last = (ticket == gridDim.x - 1) ? 1u : 0u;
  }
  __syncthreads();
  if (s_last && warp == 0) {
    __threadfence();
    double th[NV], tl[NV];
#pragma unroll
    for (int i = 0; i < NV; ++i) th[i] = tl[i] = 0.0;
    for (int b = lane; b < (int)gridDim.x; b += 32) {
#pragma unroll
      for (int i = 0; i < NV; ++i)
        dd_add2(th[i], tl[i], ld_vol(&partials[b * 8 + 2 * i]), ld_vol(&partials[b * 8 + 2 * i + 1]));
    }
#pragma unroll
    for (int i = 0; i < NV; ++i) {
#pragma unroll
      for (int off = 16; off > 0; off >>= 1) {
        const double oh = __shfl_xor_sync(0xffffffffu, th[i], off);
        const double ol = __shfl_xor_sync(0xffffffffu, tl[i], off);
        dd_add2(th[i], tl[i], oh, ol);
      }
    }
    if (lane == 0) {
#pragma unroll
      for (int i = 0; i < NV; ++i) {
        if (fuse) {
          const double tot = __dadd_rn(th[i], tl[i]);
          st->sums[i] = accumulate ? st->sums[i] + tot : tot;
        } else {  // keep the pair: the ranks' pairs are combined before rounding
          if (accumulate) dd_add2(th[i], tl[i], st->sums[i], st->sums_lo[i]);
          st->sums[i] = th[i];
          st->sums_lo[i] = tl[i];
        }
      }
      if (fuse) finalize_state(st, kind);
      *counter = 0u;
      __threadfence();
    }
  }
}

// plain per-thread sums (each value one group)
template <int NV, int NWARP>
__device__ void reduce_and_finalize(double (&v)[NV], double* s_red, unsigned* s_last_p,
                                    double* partials, unsigned* counter, CgState* st, int fuse,
                                    int kind, int accumulate = 0) {
  double lo[NV];
#pragma unroll
  for (int i = 0; i < NV; ++i) lo[i] = 0.0;
  reduce_and_finalize<NV, NWARP>(v, lo, s_red, s_last_p, partials, counter, st, fuse, kind,
                                 accumulate);
}

// ---------------------------------------------------------------------------
// the separable streaming kernel
//
// Per work item (64x32 tile, z-chunk) the plane loop is software-pipelined:
// iteration j runs the *front* of plane j+1 (TMA wait, CG p-formation, x-pass
// into X[(j+1)&1]) and the *back* of plane j (y-pass from X[j&1], z-ring
// update, epilogue of output plane j-2p), then one block barrier.  Each warp
// therefore interleaves two independent instruction streams, and the x-pass
// row imbalance is diluted by the balanced back half.

// tile kinds (compile-time variants of the plane loop): interior tiles use
// the Toeplitz taps everywhere; edge tiles check classes per row/column;
// ragged tiles (last tile row, fewer than TY valid rows) also skip the rows
// below the grid
constexpr int TILE_EDGE = 0, TILE_INTERIOR = 1, TILE_RAGGED = 2;

struct ItemGeom {
  int x0, y0, zc0, zc1;
};

// valid output rows of a tile (< TY only in a ragged last tile row)
template <int P, int MODE>
__device__ __forceinline__ int tile_rows(const SepParams& prm, const ItemGeom& g) {
  return min(Geo<P, MODE>::TY, prm.ny - g.y0);
}

// Items: (tile, z-chunk) in tile-fastest order, dealt round-robin so all
// CTAs stream neighbouring tiles at the same z in lockstep (x/y halo planes
// are then L2 hits).  The first main_items form whole waves; each remaining
// chunk (the ragged last wave) is split tail_split ways so it is spread over
// all SMs instead of extending the makespan by a full chunk.
template <int P, int MODE>
__device__ __forceinline__ ItemGeom item_geom(const SepParams& prm, int item) {
  constexpr int TY = Geo<P, MODE>::TY;
  const int tiles_xy = prm.tiles_x * prm.tiles_y;
  // branch-free: for main items jt < 0 maps to (it = item, sub = 0) via max()
  const int jt = max(item - prm.main_items, 0);
  const int it = min(item, prm.main_items + jt / prm.tail_split);
  const int sub = jt - (it - min(item, prm.main_items)) * prm.tail_split;
  const int t = it % tiles_xy;
  const int ch = it / tiles_xy;
  const int len = prm.sub_len;  // == chunk_len when tail_split == 1
  ItemGeom g;
  g.x0 = (t % prm.tiles_x) * TX;
  g.y0 = (t / prm.tiles_x) * TY;
  const int c0 = prm.z_begin + ch * prm.chunk_len;
  const int c1 = min(c0 + prm.chunk_len, prm.z_end);
  const bool tail = item >= prm.main_items;
  g.zc0 = tail ? min(c0 + sub * len, c1) : c0;   // an empty sub-chunk streams only its
  g.zc1 = tail ? min(g.zc0 + len, c1) : c1;      // 2p warm-up planes
  return g;
}

template <int P, int MODE>
__device__ __forceinline__ bool tile_interior(const SepParams& prm, const ItemGeom& g) {
  using C = Cfg<P, MODE>;
  [[maybe_unused]] constexpr int NW = C::NW, NT = C::NT, TY = C::TY;
  if (BSPDE_ALL_EDGE) return false;  // tuning: measure the edge-tile path everywhere
  return (g.x0 - C::PX >= prm.ew[2]) && (g.x0 + TX + C::PX <= prm.nx - prm.ew[2]) &&
         (g.y0 - P >= prm.ew[1]) && (g.y0 + TY + P <= prm.ny - prm.ew[1]);
}

// TMA producer cursor (thread 0 only): issues the CTA's planes in work order
template <int P, int MODE>
struct Producer {
  int item, j;
  uint32_t flat;
  const CUtensorMap* tma;  // Cfg::AS: the aux (F) map, nullptr: no aux
  __device__ __forceinline__ void issue(const SepParams& prm, const CUtensorMap* tm0,
                                        const CUtensorMap* tm1, double* s_stage,
                                        uint64_t* s_full) {
    using C = Cfg<P, MODE>;
  [[maybe_unused]] constexpr int NW = C::NW, NT = C::NT, TY = C::TY;
    if (item >= prm.nitems) return;
    const ItemGeom g = item_geom<P, MODE>(prm, item);
    const int nin = g.zc1 - g.zc0 + 2 * P;
    const int s = flat % C::NS;
    const int zb = g.zc0 - P + j + prm.ghost;
    // Cfg::AS: the aux tile of output plane zc0 - 2P + j rides with input plane j
    const bool al = C::AS && tma != nullptr && j >= 2 * P;
    mbar_expect_tx(&s_full[s], C::NA * C::HX * C::HY * 8 + (al ? C::AST * 8 : 0));
    tma_load_3d(s_stage + (s * C::NA + 0) * C::ARR_D, tm0, g.x0 - C::PX, g.y0 - P, zb, &s_full[s]);
    if (C::NA == 2)
      tma_load_3d(s_stage + (s * C::NA + 1) * C::ARR_D, tm1, g.x0 - C::PX, g.y0 - P, zb,
                  &s_full[s]);
    if (al)
      tma_load_3d(s_stage + C::NS * C::NA * C::ARR_D + s * C::AST, tma, g.x0, g.y0, zb - P,
                  &s_full[s]);
    ++flat;
    if (++j == nin) {
      j = 0;
      item += gridDim.x;
    }
  }
};

struct Smem {
  double* stage;
  double* X;
  double* tab;
  double* invd;
  uint64_t* full;
};

// front half of plane jj (flat index f): wait for its stage, form p (CG),
// x-pass of this warp's rows into X[f & 1]
template <int P, int MODE, int TK>
__device__ __forceinline__ void plane_front(const SepParams& prm, const Smem& sm,
                                            const ItemGeom& g, int jj, uint32_t f, double beta) {
  constexpr bool INTERIOR = (TK == TILE_INTERIOR), RAGGED = (TK == TILE_RAGGED);
  using C = Cfg<P, MODE>;
  [[maybe_unused]] constexpr int NW = C::NW, NT = C::NT, TY = C::TY;
  const TapSrc<P, MODE> T{prm};
  constexpr int R = C::R, HX = C::HX, HY = C::HY, NA = C::NA, NS = C::NS, NC = C::NC;
  constexpr int PX = C::PX, DX = C::DX;
  constexpr bool STIFF = C::STIFF;
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int nx = prm.nx, ny = prm.ny;
  const int ewz = prm.ew[0], ewy = prm.ew[1], ewx = prm.ew[2];
  const int zg = prm.z_off + g.zc0 - P + jj;
  const int s = f % NS;
  mbar_wait(&sm.full[s], (f / NS) & 1);
  if (!(zg >= 0 && zg < prm.nz_glob)) return;  // ghost/outside plane: no contribution
  // CG: p_k is formed over r in slot 0 (r is dead afterwards) and p_{k-1}
  // stays in slot 1 for the x update (run_item); other modes: one slot
  double* stC = sm.stage + (s * NA + 0) * C::ARR_D;
  const double* stP = sm.stage + (s * NA + (NA - 1)) * C::ARR_D;
  double* X1 = sm.X + (f & 1) * 2 * C::XARR;
  double* X2 = X1 + C::XARR;
  const int cz = cls_of(zg, prm.nz_glob, ewz);

  if (MODE == M_CGA) {
    // p = D^-1 r + beta p_old over this warp's rows of the haloed tile, in
    // place in the p_old stage.  The warp's rows (warp, warp+NW, ...) are
    // walked as one flat list of double2 pairs so all lanes stay busy.
    constexpr int PPR = HX / 2;                       // pairs per row
    constexpr int NROW = (HY + NW - 1) / NW;          // rows of warps 0.. (HY % NW) - 1
    // a ragged last tile row only needs its valid rows + 2p halo rows
    const int nrow = !RAGGED
                         ? ((warp < HY - NW * (NROW - 1)) ? NROW : NROW - 1)
                         : max(0, (tile_rows<P, MODE>(prm, g) + 2 * P - warp + NW - 1) / NW);
    const int npair = nrow * PPR;
    const int ncy = 2 * ewy + 1, ncx = 2 * ewx + 1;
    if (INTERIOR && cz == ewz) {
      const double inv0 = sm.invd[(cz * ncy + ewy) * ncx + ewx];
#pragma unroll
      for (int h = 0; h < (NROW * PPR + 31) / 32; ++h) {
        const int t = lane + 32 * h;
        if (t < npair) {
          const int m = t / PPR, q = t - m * PPR;
          const int e = (warp + NW * m) * HX + 2 * q;
          const double2 rv = *reinterpret_cast<const double2*>(stC + e);
          const double2 qv = *reinterpret_cast<const double2*>(stP + e);
          double2 pv;
          pv.x = pdir(rv.x, inv0, qv.x, beta);
          pv.y = pdir(rv.y, inv0, qv.y, beta);
          *reinterpret_cast<double2*>(stC + e) = pv;
        }
      }
    } else {
      // edge tile or edge z plane: elements inside the x/y interior band use
      // the plane's interior entry; only the boundary band looks up classes
      const double inv_c = sm.invd[(cz * ncy + ewy) * ncx + ewx];
      for (int t = lane; t < npair; t += 32) {
        const int m = t / PPR, q = t - m * PPR;
        const int row = warp + NW * m;
        const int e = row * HX + 2 * q;
        const int gyy = g.y0 - P + row;
        const int gxx = g.x0 - PX + 2 * q;
        double i0 = inv_c, i1 = inv_c;
        if (!(gyy >= ewy && gyy < ny - ewy && gxx >= ewx && gxx + 1 < nx - ewx)) {
          const bool rok = (gyy >= 0 && gyy < ny);
          const double* trow = sm.invd + (cz * ncy + (rok ? cls_of(gyy, ny, ewy) : ewy)) * ncx;
          i0 = (rok && gxx >= 0 && gxx < nx) ? trow[cls_of(gxx, nx, ewx)] : 0.0;
          i1 = (rok && gxx + 1 >= 0 && gxx + 1 < nx) ? trow[cls_of(gxx + 1, nx, ewx)] : 0.0;
        }
        const double2 rv = *reinterpret_cast<const double2*>(stC + e);
        const double2 qv = *reinterpret_cast<const double2*>(stP + e);
        double2 pv;
        pv.x = pdir(rv.x, i0, qv.x, beta);
        pv.y = pdir(rv.y, i1, qv.y, beta);
        *reinterpret_cast<double2*>(stC + e) = pv;
      }
    }
    __syncwarp();
  }
  // x-pass: X1 = u1 = Mx c, X2 = t = c_mass*u1 + cx*Kx c
#pragma unroll
  for (int m = 0; m < (HY + NW - 1) / NW; ++m) {
    const int row = warp + NW * m;
    if (row < HY && (!RAGGED || row < tile_rows<P, MODE>(prm, g) + 2 * P)) {
      const double* w = stC + row * HX + 2 * lane;
      double raw[2 * P + 2 + 2 * DX];
#pragma unroll
      for (int k = 0; k < P + 1 + DX; ++k) {
        const double2 t = *reinterpret_cast<const double2*>(w + 2 * k);
        raw[2 * k] = t.x;
        raw[2 * k + 1] = t.y;
      }
      double m0 = 0.0, m1 = 0.0, k0 = 0.0, k1 = 0.0;
      const int gx0 = g.x0 + 2 * lane;
      if (INTERIOR || ((gx0 >= ewx) && (gx0 + 1 < nx - ewx))) {
#pragma unroll
        for (int k = 0; k < P; ++k) {
          const double s0 = raw[DX + k] + raw[DX + 2 * P - k];
          const double s1 = raw[DX + 1 + k] + raw[DX + 1 + 2 * P - k];
          m0 = fma(T.M(k), s0, m0);
          m1 = fma(T.M(k), s1, m1);
          if (STIFF) {
            k0 = fma(T.K(k), s0, k0);
            k1 = fma(T.K(k), s1, k1);
          }
        }
        m0 = fma(T.M(P), raw[DX + P], m0);
        m1 = fma(T.M(P), raw[DX + P + 1], m1);
        if (STIFF) {
          k0 = fma(T.K(P), raw[DX + P], k0);
          k1 = fma(T.K(P), raw[DX + P + 1], k1);
        }
      } else {
        const int c0 = (gx0 < nx) ? cls_of(gx0, nx, ewx) : ewx;
        const int c1 = (gx0 + 1 < nx) ? cls_of(gx0 + 1, nx, ewx) : ewx;
        const double* tm0 = sm.tab + ((2 * 2 + 0) * NC + c0) * R;
        const double* tm1 = sm.tab + ((2 * 2 + 0) * NC + c1) * R;
        const double* tk0 = sm.tab + ((2 * 2 + 1) * NC + c0) * R;
        const double* tk1 = sm.tab + ((2 * 2 + 1) * NC + c1) * R;
#pragma unroll
        for (int k = 0; k < 2 * P + 1; ++k) {
          m0 = fma(tm0[k], raw[DX + k], m0);
          m1 = fma(tm1[k], raw[DX + k + 1], m1);
          if (STIFF) {
            k0 = fma(tk0[k], raw[DX + k], k0);
            k1 = fma(tk1[k], raw[DX + k + 1], k1);
          }
        }
      }
      *reinterpret_cast<double2*>(X1 + row * TX + 2 * lane) = make_double2(m0, m1);
      if (STIFF) {
        const double t0 = fma(prm.cx, k0, prm.c_mass * m0);
        const double t1 = fma(prm.cx, k1, prm.c_mass * m1);
        *reinterpret_cast<double2*>(X2 + row * TX + 2 * lane) = make_double2(t0, t1);
      }
    }
  }
}

// back half of plane j (flat index f): y-pass, z-ring shift update, epilogue
template <int P, int MODE, int TK>
__device__ __forceinline__ void plane_back(const SepParams& prm, const Smem& sm, const ItemGeom& g,
                                           int j, uint32_t f, double (&acc)[2 * P][RPT],
                                           double (&pr)[P][RPT], const double (&auxv)[RPT],
                                           double (&dsum)[6], double beta,
                                           double (&accm)[2 * P][RPT]) {
  constexpr bool INTERIOR = (TK == TILE_INTERIOR), RAGGED = (TK == TILE_RAGGED);
  using C = Cfg<P, MODE>;
  [[maybe_unused]] constexpr int NW = C::NW, NT = C::NT, TY = C::TY;
  const TapSrc<P, MODE> T{prm};
  constexpr int R = C::R, HX = C::HX, NA = C::NA, NS = C::NS, NC = C::NC, S = 2 * P;
  constexpr int PX = C::PX;
  constexpr bool STIFF = C::STIFF;
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int gcol = warp & 1, rg = warp >> 1;
  const int cxl = gcol * 32 + lane;
  const int gx = g.x0 + cxl;
  const int gy0 = g.y0 + rg * RPT;
  const int nx = prm.nx, ny = prm.ny;
  const int ewz = prm.ew[0], ewy = prm.ew[1], ewx = prm.ew[2];
  const int ncy = 2 * ewy + 1, ncx = 2 * ewx + 1;
  const int zl = g.zc0 - P + j;
  const int zg = prm.z_off + zl;
  const bool in_grid = (zg >= 0) && (zg < prm.nz_glob);
  const double* X1 = sm.X + (f & 1) * 2 * C::XARR;
  const double* X2 = X1 + C::XARR;
  double out[RPT], om[RPT];
  // ghost planes (outside the global grid) enter the z ring as zeros through
  // the same FMA path: one writer of acc keeps the ring registers coalesced
  double wm[RPT], wa[RPT];
#pragma unroll
  for (int i = 0; i < RPT; ++i) {
    wm[i] = 0.0;
    wa[i] = 0.0;
  }
  if (in_grid) {
    // ---- y-pass: wm = My u1, wa = My t + cy Ky u1 for rows gy0 .. gy0+3 ----
    const double* x1c = X1 + (rg * RPT) * TX + cxl;
    const double* x2c = X2 + (rg * RPT) * TX + cxl;
    const bool fast_y = INTERIOR || ((gy0 >= ewy) && (gy0 + RPT - 1 < ny - ewy));
    if (RAGGED && gy0 >= ny) {
      // row group below the grid (ragged last tile row): nothing to filter
    } else if (fast_y) {
#pragma unroll
      for (int rr = 0; rr < RPT + 2 * P; ++rr) {
        const double a1 = x1c[rr * TX];
        const double t = STIFF ? x2c[rr * TX] : 0.0;
        const double u1c = STIFF ? prm.cy * a1 : 0.0;
#pragma unroll
        for (int i = 0; i < RPT; ++i) {
          const int k = rr - i;
          if (k >= 0 && k <= 2 * P) {
            wm[i] = fma(T.M(k), a1, wm[i]);
            if (STIFF) {
              wa[i] = fma(T.M(k), t, wa[i]);
              wa[i] = fma(T.K(k), u1c, wa[i]);
            }
          }
        }
      }
    } else {
      int cyr[RPT];
#pragma unroll
      for (int i = 0; i < RPT; ++i) {
        const int gy = gy0 + i;
        cyr[i] = (gy < ny) ? cls_of(gy, ny, ewy) : ewy;
      }
#pragma unroll
      for (int rr = 0; rr < RPT + 2 * P; ++rr) {
        const double a1 = x1c[rr * TX];
        const double t = STIFF ? x2c[rr * TX] : 0.0;
        const double u1c = STIFF ? prm.cy * a1 : 0.0;
#pragma unroll
        for (int i = 0; i < RPT; ++i) {
          const int k = rr - i;
          if (k >= 0 && k <= 2 * P) {
            const double* ty = sm.tab + ((1 * 2 + 0) * NC + cyr[i]) * R;
            wm[i] = fma(ty[k], a1, wm[i]);
            if (STIFF) {
              wa[i] = fma(ty[k], t, wa[i]);
              wa[i] = fma(ty[NC * R + k], u1c, wa[i]);
            }
          }
        }
      }
    }
  }
  {
    // ---- z: shift-register scatter (row z' of the symmetric Mz, Kz) ----
    const int cz = in_grid ? cls_of(zg, prm.nz_glob, ewz) : ewz;
    if (cz == ewz && prm.zfast) {
#pragma unroll
      for (int i = 0; i < RPT; ++i) {
        const double a = STIFF ? wa[i] : wm[i];
        const double w2 = STIFF ? wm[i] * prm.cz : 0.0;
        double o = fma(T.M(0), a, acc[0][i]);
        if (STIFF) o = fma(T.K(0), w2, o);
        out[i] = o;
#pragma unroll
        for (int k = 0; k < S - 1; ++k) {
          double v = fma(T.M(k + 1), a, acc[k + 1][i]);
          if (STIFF) v = fma(T.K(k + 1), w2, v);
          acc[k][i] = v;
        }
        double v = T.M(S) * a;
        if (STIFF) v = fma(T.K(S), w2, v);
        acc[S - 1][i] = v;
      }
    } else {
      const double* tzm = sm.tab + ((0 * 2 + 0) * NC + cz) * R;
      const double* tzk = sm.tab + ((0 * 2 + 1) * NC + cz) * R;
#pragma unroll
      for (int i = 0; i < RPT; ++i) {
        const double a = STIFF ? wa[i] : wm[i];
        const double w2 = STIFF ? wm[i] * prm.cz : 0.0;
        double o = fma(tzm[0], a, acc[0][i]);
        if (STIFF) o = fma(tzk[0], w2, o);
        out[i] = o;
#pragma unroll
        for (int k = 0; k < S - 1; ++k) {
          double v = fma(tzm[k + 1], a, acc[k + 1][i]);
          if (STIFF) v = fma(tzk[k + 1], w2, v);
          acc[k][i] = v;
        }
        double v = tzm[S] * a;
        if (STIFF) v = fma(tzk[S], w2, v);
        acc[S - 1][i] = v;
      }
    }
    if (MODE == M_HRES) {
      // pure mass ring (Mz(x)My(x)Mx) u: the M_MASS kernel's z pass on wm
      const double* tzm = sm.tab + ((0 * 2 + 0) * NC + cz) * R;
      // two plane-uniform branches (interior taps / class table), like the
      // main ring: a per-FMA select made both operands live (LDS + SEL per
      // tap; 16% of the kernel's instructions)
      auto mass_ring = [&](auto tap) {
#pragma unroll
        for (int i = 0; i < RPT; ++i) {
          const double a = wm[i];
          om[i] = fma(tap(0), a, accm[0][i]);
#pragma unroll
          for (int k = 0; k < S - 1; ++k) accm[k][i] = fma(tap(k + 1), a, accm[k + 1][i]);
          accm[S - 1][i] = tap(S) * a;
        }
      };
      if (cz == ewz && prm.zfast)
        mass_ring([&](int k) { return T.M(k); });
      else
        mass_ring([&](int k) { return tzm[k]; });
    }
  }

  // ---- epilogue: output plane zo = zl - P (complete once j >= 2P) ----
  if (j >= 2 * P) {
    const int zo = zl - P;
    const long long obase =
        (long long)(zo + prm.ghost) * prm.pitch_z + (long long)gy0 * prm.pitch_y + gx;
    const int czo = cls_of(prm.z_off + zo, prm.nz_glob, ewz);
    double g0 = 0.0, g1 = 0.0, g2 = 0.0;  // group sums of this thread's rows (dd_add)
#pragma unroll
    for (int i = 0; i < RPT; ++i) {
      const int y = gy0 + i;
      if (INTERIOR || (y < ny && gx < nx)) {
        const long long off = obase + (long long)i * prm.pitch_y;
        const double v = out[i];
        if (MODE == M_APPLY) {
          __stcs(prm.out + off, v);
        } else if (MODE == M_CGA) {
          __stcs(prm.out + off, v);
          prm.cg_pout[off] = pr[0][i];  // p_k for pass B (ping-pong partner of p_{k-1})
          g0 = fma(pr[0][i], v, g0);
        } else if (MODE == M_MASS) {
          double o = prm.c_mass * v;
          if (prm.aux) o = fma(prm.aux_scale, auxv[i], o);
          __stcs(prm.out + off, o);
        } else {  // M_RESID (b loaded) / M_HRES (b = rhs_cm M u + a F, rounded as M_MASS)
          double bb = auxv[i];
          if (MODE == M_HRES) {
            bb = prm.rhs_cm * om[i];
            if (prm.aux) {
              const double fv =
                  C::AS ? sm.stage[NS * NA * C::ARR_D + (f % NS) * C::AST + (rg * RPT + i) * TX +
                                   cxl]
                        : auxv[i];
              bb = fma(prm.aux_scale, fv, bb);
            }
          }
          const double r = bb - v;
          __stcs(prm.out + off, r);
          const double inv =
              sm.invd[(czo * ncy + (INTERIOR ? ewy : cls_of(y, ny, ewy))) * ncx +
                      (INTERIOR ? ewx : cls_of(gx, nx, ewx))];
          g0 = fma(bb, bb, g0);
          g1 = fma(r, __dmul_rn(inv, r), g1);
          g2 = fma(r, r, g2);
        }
      }
    }
    if (MODE == M_CGA || MODE == M_RESID || MODE == M_HRES) dd_add(dsum[0], dsum[3], g0);
    if (MODE == M_RESID || MODE == M_HRES) {
      dd_add(dsum[1], dsum[4], g1);
      dd_add(dsum[2], dsum[5], g2);
    }
  }
  if (MODE == M_CGA) {
    // own p_k of plane zl (slot 0; the stage is released only after this iteration)
    const int s = f % NS;
    const double* stP = sm.stage + (s * NA + 0) * C::ARR_D;
#pragma unroll
    for (int i = 0; i < RPT; ++i) {
#pragma unroll
      for (int k = 0; k < P - 1; ++k) pr[k][i] = pr[k + 1][i];
      pr[P - 1][i] = stP[(rg * RPT + i + P) * HX + cxl + PX];
    }
  }
}

// BSPDE_CORE_ITER=0 (measurement build): interior tiles use the generic
// plane_front / plane_back for every plane
#ifndef BSPDE_CORE_ITER
#define BSPDE_CORE_ITER 1
#endif
// degrees whose pass A prefetches x a plane ahead (tuning)
#ifndef BSPDE_XPF_MAXP
#define BSPDE_XPF_MAXP 3
#endif
// core iterations in CG pass A too (measured slower: register pressure)
#ifndef BSPDE_CORE_CGA
#define BSPDE_CORE_CGA 0
#endif
template <int P, int MODE>
__host__ __device__ constexpr bool C_INVD() { return Cfg<P, MODE>::INVD; }

// the thread that issues the plane TMA loads (lane 0 of one warp): the last
// warp owns one haloed row fewer in the front half than warps 0..(HY % NW)-1
#ifndef BSPDE_PROD_WARP
#define BSPDE_PROD_WARP -1
#endif
template <int P, int MODE>
constexpr int kProdThread =
    (BSPDE_PROD_WARP < 0 ? Geo<P, MODE>::NW + BSPDE_PROD_WARP : BSPDE_PROD_WARP) * 32;

// ---------------------------------------------------------------------------
// Core iterations of an interior tile.  Iteration j (front of plane j+1 +
// back of plane j) is "core" when both planes are z-interior rows inside the
// global grid (and, for the residual, the output plane j - P too): Toeplitz
// taps on every axis, the interior inverse diagonal, no ghost planes.  The
// body below is plane_front + plane_back specialised to that case -- the same
// floating-point operations in the same order (bitwise-identical results),
// but without class lookups, tile-kind / ghost-plane branches, per-pair
// index divisions or per-plane 64-bit offset arithmetic, so the compiler sees
// one straight-line block per plane and can overlap the front's shared-memory
// latency with the back's FMAs.

// pair offsets of this thread's CG p-formation work in a staged (haloed)
// plane array (interior, full-height tiles; -1: no pair), fixed per kernel
template <int P, int MODE>
__device__ __forceinline__ void core_pform_offsets(int (&pfe)[4]) {
  using C = Cfg<P, MODE>;
  constexpr int NW = C::NW, HX = C::HX, HY = C::HY;
  constexpr int PPR = HX / 2;
  constexpr int NROW = (HY + NW - 1) / NW;
  static_assert((NROW * PPR + 31) / 32 <= 4, "p-formation needs more than 4 rounds");
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int nrow = (warp < HY - NW * (NROW - 1)) ? NROW : NROW - 1;
  const int npair = nrow * PPR;
#pragma unroll
  for (int h = 0; h < 4; ++h) {
    const int t = lane + 32 * h;
    const int m = t / PPR, q = t - m * PPR;
    pfe[h] = (t < npair) ? (warp + NW * m) * HX + 2 * q : -1;
  }
}

template <int P, int MODE>
__device__ __forceinline__ void core_iter(const SepParams& prm, const Smem& sm, int j, uint32_t f,
                                          double (&acc)[2 * P][RPT], double (&pr)[P][RPT],
                                          double (&dsum)[6], double beta, const int (&pfe)[4],
                                          double inv0, double* op, double* pp, const double* xp,
                                          long long py) {
  using C = Cfg<P, MODE>;
  constexpr int NW = C::NW, TY = C::TY, HX = C::HX, HY = C::HY, NA = C::NA, NS = C::NS;
  constexpr int PX = C::PX, DX = C::DX, S = 2 * P;
  constexpr bool STIFF = C::STIFF;
  const TapSrc<P, MODE> T{prm};
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int rg = warp >> 1;
  const int cxl = (warp & 1) * 32 + lane;
  (void)TY;

  // epilogue operand prefetch (RESID: b, MASS: f) for output plane j - 2P
  double auxv[RPT];
#pragma unroll
  for (int i = 0; i < RPT; ++i) auxv[i] = 0.0;
  if ((MODE == M_RESID || (MODE == M_MASS && prm.aux != nullptr)) && j >= 2 * P) {
#pragma unroll
    for (int i = 0; i < RPT; ++i) auxv[i] = __ldcs(xp + i * py);
  }

  // ---- front of plane j+1: stage wait, p = D^-1 r + beta p_old, x-pass ----
  {
    const uint32_t f1 = f + 1;
    const int s1 = f1 % NS;
    mbar_wait(&sm.full[s1], (f1 / NS) & 1);
    double* stC = sm.stage + (s1 * NA + 0) * C::ARR_D;
    const double* stP = sm.stage + (s1 * NA + (NA - 1)) * C::ARR_D;
    double* X1 = sm.X + (f1 & 1) * 2 * C::XARR;
    double* X2 = X1 + C::XARR;
    if (MODE == M_CGA) {
#pragma unroll
      for (int h = 0; h < 4; ++h) {
        const int e = pfe[h];
        if (e >= 0) {
          const double2 rv = *reinterpret_cast<const double2*>(stC + e);
          const double2 qv = *reinterpret_cast<const double2*>(stP + e);
          double2 pv;
          pv.x = pdir(rv.x, inv0, qv.x, beta);
          pv.y = pdir(rv.y, inv0, qv.y, beta);
          *reinterpret_cast<double2*>(stC + e) = pv;
        }
      }
      __syncwarp();
    }
#pragma unroll
    for (int m = 0; m < (HY + NW - 1) / NW; ++m) {
      const int row = warp + NW * m;
      if (row < HY) {
        const double* w = stC + row * HX + 2 * lane;
        double raw[2 * P + 2 + 2 * DX];
#pragma unroll
        for (int k = 0; k < P + 1 + DX; ++k) {
          const double2 t = *reinterpret_cast<const double2*>(w + 2 * k);
          raw[2 * k] = t.x;
          raw[2 * k + 1] = t.y;
        }
        double m0 = 0.0, m1 = 0.0, k0 = 0.0, k1 = 0.0;
#pragma unroll
        for (int k = 0; k < P; ++k) {
          const double s0 = raw[DX + k] + raw[DX + 2 * P - k];
          const double s1 = raw[DX + 1 + k] + raw[DX + 1 + 2 * P - k];
          m0 = fma(T.M(k), s0, m0);
          m1 = fma(T.M(k), s1, m1);
          if (STIFF) {
            k0 = fma(T.K(k), s0, k0);
            k1 = fma(T.K(k), s1, k1);
          }
        }
        m0 = fma(T.M(P), raw[DX + P], m0);
        m1 = fma(T.M(P), raw[DX + P + 1], m1);
        if (STIFF) {
          k0 = fma(T.K(P), raw[DX + P], k0);
          k1 = fma(T.K(P), raw[DX + P + 1], k1);
        }
        *reinterpret_cast<double2*>(X1 + row * TX + 2 * lane) = make_double2(m0, m1);
        if (STIFF) {
          const double t0 = fma(prm.cx, k0, prm.c_mass * m0);
          const double t1 = fma(prm.cx, k1, prm.c_mass * m1);
          *reinterpret_cast<double2*>(X2 + row * TX + 2 * lane) = make_double2(t0, t1);
        }
      }
    }
  }

  // ---- back of plane j: y-pass, z ring, epilogue of output plane j - 2P ----
  const double* X1 = sm.X + (f & 1) * 2 * C::XARR;
  const double* X2 = X1 + C::XARR;
  double wm[RPT], wa[RPT], out[RPT];
#pragma unroll
  for (int i = 0; i < RPT; ++i) {
    wm[i] = 0.0;
    wa[i] = 0.0;
  }
  {
    const double* x1c = X1 + (rg * RPT) * TX + cxl;
    const double* x2c = X2 + (rg * RPT) * TX + cxl;
#pragma unroll
    for (int rr = 0; rr < RPT + 2 * P; ++rr) {
      const double a1 = x1c[rr * TX];
      const double t = STIFF ? x2c[rr * TX] : 0.0;
      const double u1c = STIFF ? prm.cy * a1 : 0.0;
#pragma unroll
      for (int i = 0; i < RPT; ++i) {
        const int k = rr - i;
        if (k >= 0 && k <= 2 * P) {
          wm[i] = fma(T.M(k), a1, wm[i]);
          if (STIFF) {
            wa[i] = fma(T.M(k), t, wa[i]);
            wa[i] = fma(T.K(k), u1c, wa[i]);
          }
        }
      }
    }
  }
#pragma unroll
  for (int i = 0; i < RPT; ++i) {
    const double a = STIFF ? wa[i] : wm[i];
    const double w2 = STIFF ? wm[i] * prm.cz : 0.0;
    double o = fma(T.M(0), a, acc[0][i]);
    if (STIFF) o = fma(T.K(0), w2, o);
    out[i] = o;
#pragma unroll
    for (int k = 0; k < S - 1; ++k) {
      double v = fma(T.M(k + 1), a, acc[k + 1][i]);
      if (STIFF) v = fma(T.K(k + 1), w2, v);
      acc[k][i] = v;
    }
    double v = T.M(S) * a;
    if (STIFF) v = fma(T.K(S), w2, v);
    acc[S - 1][i] = v;
  }
  if (j >= 2 * P) {
    double g0 = 0.0, g1 = 0.0, g2 = 0.0;  // group sums of this thread's rows (dd_add)
#pragma unroll
    for (int i = 0; i < RPT; ++i) {
      const double v = out[i];
      if (MODE == M_APPLY) {
        __stcs(op + i * py, v);
      } else if (MODE == M_CGA) {
        __stcs(op + i * py, v);
        pp[i * py] = pr[0][i];
        g0 = fma(pr[0][i], v, g0);
      } else if (MODE == M_MASS) {
        double o = prm.c_mass * v;
        if (prm.aux) o = fma(prm.aux_scale, auxv[i], o);
        __stcs(op + i * py, o);
      } else {  // M_RESID
        const double bb = auxv[i];
        const double r = bb - v;
        __stcs(op + i * py, r);
        g0 = fma(bb, bb, g0);
        g1 = fma(r, __dmul_rn(inv0, r), g1);
        g2 = fma(r, r, g2);
      }
    }
    if (MODE == M_CGA || MODE == M_RESID) dd_add(dsum[0], dsum[3], g0);
    if (MODE == M_RESID) {
      dd_add(dsum[1], dsum[4], g1);
      dd_add(dsum[2], dsum[5], g2);
    }
  }
  if (MODE == M_CGA) {
    const int s = f % NS;
    const double* stP = sm.stage + (s * NA + 0) * C::ARR_D;  // p_k
#pragma unroll
    for (int i = 0; i < RPT; ++i) {
#pragma unroll
      for (int k = 0; k < P - 1; ++k) pr[k][i] = pr[k + 1][i];
      pr[P - 1][i] = stP[(rg * RPT + i + P) * HX + cxl + PX];
    }
  }
}

template <int P, int MODE, int TK>
__device__ __forceinline__ void run_item(const SepParams& prm, const CUtensorMap* tm0,
                                         const CUtensorMap* tm1, const Smem& sm,
                                         const ItemGeom& g, uint32_t& flat, double beta,
                                         double (&dsum)[6], Producer<P, MODE>& prod,
                                         double xalpha, bool xok) {
  constexpr bool INTERIOR = (TK == TILE_INTERIOR), RAGGED = (TK == TILE_RAGGED);
  constexpr int S = 2 * P;
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int gx = g.x0 + (warp & 1) * 32 + lane;
  const int gy0 = g.y0 + (warp >> 1) * RPT;
  const int nin = g.zc1 - g.zc0 + 2 * P;
  double acc[S][RPT];
  double pr[P][RPT];
  double accm[S][RPT];  // M_HRES: the pure mass ring
#pragma unroll
  for (int k = 0; k < S; ++k)
#pragma unroll
    for (int i = 0; i < RPT; ++i) acc[k][i] = accm[k][i] = 0.0;
#pragma unroll
  for (int k = 0; k < P; ++k)
#pragma unroll
    for (int i = 0; i < RPT; ++i) pr[k][i] = 0.0;

  // core iterations [jlo, jhi) of an interior tile (see core_iter)
  int jlo = 0, jhi = 0;
  int pfe[4] = {-1, -1, -1, -1};
  double inv0 = 0.0;
  double *op = nullptr, *pp = nullptr;
  const double* xp = nullptr;
  const long long py = prm.pitch_y;
  constexpr bool CORE = INTERIOR && BSPDE_CORE_ITER && MODE != M_HRES &&
                        (MODE != M_CGA || BSPDE_CORE_CGA);
  if (CORE) {
    const int ewz = prm.ew[0];
    const int zbase = prm.z_off + g.zc0 - P;  // global z of streamed plane 0
    jlo = max(0, ewz - zbase + (MODE == M_RESID ? P : 0));
    jhi = prm.zfast ? min(nin - 1, prm.nz_glob - ewz - zbase - 1) : 0;
    if (MODE == M_CGA) core_pform_offsets<P, MODE>(pfe);
    if (C_INVD<P, MODE>())
      inv0 = sm.invd[(ewz * (2 * prm.ew[1] + 1) + prm.ew[1]) * (2 * prm.ew[2] + 1) + prm.ew[2]];
    // output plane of iteration 0 is zc0 - 2P (advanced one plane per iteration)
    const long long o0 = (long long)(g.zc0 - 2 * P + prm.ghost) * prm.pitch_z +
                         (long long)gy0 * py + gx;
    op = prm.out + o0;
    if (MODE == M_CGA) pp = prm.cg_pout + o0;
    if (prm.aux) xp = prm.aux + o0;
  }

  // CG: x += alpha_{k-1} p_{k-1} at this thread's owned points of every owned
  // plane (p_{k-1} is staged with the halos anyway; x is read a plane ahead of
  // its update so the load latency hides under the plane's work)
  const bool xupd = (MODE == M_CGA) && prm.cg_x != nullptr && xok;
  const int cxl = (warp & 1) * 32 + lane, rg = warp >> 1;
  double* xrow = xupd ? prm.cg_x + (long long)(g.zc0 - P + prm.ghost) * prm.pitch_z +
                            (long long)gy0 * prm.pitch_y + gx
                      : nullptr;

  plane_front<P, MODE, TK>(prm, sm, g, 0, flat, beta);
  __syncthreads();
  for (int j = 0; j < nin; ++j) {
    // x is prefetched at the start of the plane for p <= 3; p >= 4 loads it
    // at the update (the 3p-deep rings leave no registers to hold it)
    constexpr bool XPF = P <= BSPDE_XPF_MAXP;
    double xv[RPT];
    const bool xown = xupd && j >= P && j < nin - P;  // plane zc0 - P + j is owned
    if (XPF && xown) {
#pragma unroll
      for (int i = 0; i < RPT; ++i)
        xv[i] = (INTERIOR || (gy0 + i < prm.ny && gx < prm.nx)) ? xrow[i * prm.pitch_y] : 0.0;
    }
    if (CORE && j >= jlo && j < jhi) {
      core_iter<P, MODE>(prm, sm, j, flat, acc, pr, dsum, beta, pfe, inv0, op, pp, xp, py);
    } else {
      // epilogue operand prefetch (RESID: b, MASS: f) for output plane zl - P
      double auxv[RPT];
#pragma unroll
      for (int i = 0; i < RPT; ++i) auxv[i] = 0.0;
      if ((MODE == M_RESID ||
           ((MODE == M_MASS || (MODE == M_HRES && !Cfg<P, MODE>::AS)) && prm.aux != nullptr)) &&
          j >= 2 * P) {
        const int zo = g.zc0 - 2 * P + j;
        const long long base = (long long)(zo + prm.ghost) * prm.pitch_z + gx;
#pragma unroll
        for (int i = 0; i < RPT; ++i) {
          const int y = gy0 + i;
          if (INTERIOR || (y < prm.ny && gx < prm.nx))
            auxv[i] = __ldcs(prm.aux + base + (long long)y * prm.pitch_y);
        }
      }
      if (j + 1 < nin) plane_front<P, MODE, TK>(prm, sm, g, j + 1, flat + 1, beta);
      plane_back<P, MODE, TK>(prm, sm, g, j, flat, acc, pr, auxv, dsum, beta, accm);
    }
    if (xown) {  // x + alpha p, rounded like the reference's x += alpha * p (solver.py:94)
      if (!XPF) {
#pragma unroll
        for (int i = 0; i < RPT; ++i)
          xv[i] = (INTERIOR || (gy0 + i < prm.ny && gx < prm.nx)) ? xrow[i * prm.pitch_y] : 0.0;
      }
      const double* stO = sm.stage + ((flat % Cfg<P, MODE>::NS) * Cfg<P, MODE>::NA + 1) *
                                         Cfg<P, MODE>::ARR_D;
#pragma unroll
      for (int i = 0; i < RPT; ++i) {
        if (INTERIOR || (gy0 + i < prm.ny && gx < prm.nx)) {
          const double po = stO[(rg * RPT + i + P) * Cfg<P, MODE>::HX + cxl + Cfg<P, MODE>::PX];
          xrow[i * prm.pitch_y] = __dadd_rn(xv[i], __dmul_rn(xalpha, po));
        }
      }
    }
    if (xupd) xrow += prm.pitch_z;
    if (CORE) {
      op += prm.pitch_z;
      if (MODE == M_CGA) pp += prm.pitch_z;
      if (xp) xp += prm.pitch_z;
    }
    __syncthreads();
    if (threadIdx.x == kProdThread<P, MODE>) {
      // the stage of plane j is consumed (x-pass one iteration ago, own p now)
      fence_proxy_async();
      prod.issue(prm, tm0, tm1, sm.stage, sm.full);
    }
    ++flat;
  }
}

template <int P, int MODE>
__global__ void __launch_bounds__(Geo<P, MODE>::NT, 1)
    sep_kernel(const __grid_constant__ SepParams prm, const __grid_constant__ CUtensorMap tm0,
               const __grid_constant__ CUtensorMap tm1, const __grid_constant__ CUtensorMap tm2) {
  using C = Cfg<P, MODE>;
  [[maybe_unused]] constexpr int NW = C::NW, NT = C::NT, TY = C::TY;
  constexpr int NS = C::NS;

  if (MODE == M_CGA) {
    if (!ld_vol(&prm.state->active)) return;
  }

  // no static shared memory in this kernel: the dynamic window starts at the
  // (1 KB aligned) base, so every TMA destination below is 128-byte aligned
  extern __shared__ __align__(1024) double smem[];
  Smem sm;
  sm.stage = smem;
  sm.X = sm.stage + NS * C::NA * C::ARR_D + C::AS_D;
  sm.tab = sm.X + 2 * 2 * C::XARR;
  sm.invd = sm.tab + C::TAB;
  double* s_red = sm.invd + C::INV;
  unsigned* s_last = reinterpret_cast<unsigned*>(s_red + NW * 8);
  sm.full = reinterpret_cast<uint64_t*>(s_red + NW * 8 + 2);

  const int tid = threadIdx.x;
  for (int i = tid; i < C::TAB; i += NT) sm.tab[i] = prm.tab[i];
  if (C::INVD) {
    const int n = (2 * prm.ew[0] + 1) * (2 * prm.ew[1] + 1) * (2 * prm.ew[2] + 1);
    for (int i = tid; i < n; i += NT) sm.invd[i] = prm.invd[i];
  }
  if (tid == 0) {
    for (int s = 0; s < NS; ++s) mbar_init(&sm.full[s], 1);
    fence_mbar_init();
  }
  __syncthreads();

  const double beta = (MODE == M_CGA) ? ld_vol(&prm.state->beta) : 0.0;
  // pass A of iteration k applies x += alpha_{k-1} p_{k-1} (k >= 1): alpha
  // still holds alpha_{k-1} here (every CTA reads it before the last CTA's
  // finalize overwrites it with alpha_k)
  // (skipped when a flush already applied it: x_done == it)
  const int k_it = (MODE == M_CGA) ? ld_vol(&prm.state->it) : 0;
  const double xalpha = (MODE == M_CGA) ? ld_vol(&prm.state->alpha) : 0.0;
  const bool xok = k_it >= 1 && ld_vol(&prm.state->x_done) < k_it;
  double dsum[6] = {0.0, 0.0, 0.0, 0.0, 0.0, 0.0};  // hi[3], lo[3]
  Producer<P, MODE> prod{(int)blockIdx.x, 0, 0u,
                         (C::AS && prm.aux != nullptr) ? &tm2 : nullptr};
  if (tid == kProdThread<P, MODE>) {
    for (int s = 0; s < NS; ++s) prod.issue(prm, &tm0, &tm1, sm.stage, sm.full);
  }
  uint32_t flat = 0;
  for (int item = blockIdx.x; item < prm.nitems; item += gridDim.x) {
    const ItemGeom g = item_geom<P, MODE>(prm, item);
    if (tile_interior<P, MODE>(prm, g))
      run_item<P, MODE, TILE_INTERIOR>(prm, &tm0, &tm1, sm, g, flat, beta, dsum, prod, xalpha, xok);
    else if (tile_rows<P, MODE>(prm, g) == TY)
      run_item<P, MODE, TILE_EDGE>(prm, &tm0, &tm1, sm, g, flat, beta, dsum, prod, xalpha, xok);
    else
      run_item<P, MODE, TILE_RAGGED>(prm, &tm0, &tm1, sm, g, flat, beta, dsum, prod, xalpha, xok);
  }

  if (MODE == M_CGA) {
    double vh[1] = {dsum[0]}, vl[1] = {dsum[3]};
    reduce_and_finalize<1, NW>(vh, vl, s_red, s_last, prm.partials, prm.counter, prm.state,
                               prm.fuse, 1, prm.accumulate);
  } else if (MODE == M_RESID || MODE == M_HRES) {
    double vh[3] = {dsum[0], dsum[1], dsum[2]}, vl[3] = {dsum[3], dsum[4], dsum[5]};
    reduce_and_finalize<3, NW>(vh, vl, s_red, s_last, prm.partials, prm.counter, prm.state,
                               prm.fuse, 0);
  }
}

// ---------------------------------------------------------------------------
// CG pass B: r -= alpha Ap, <r, D^-1 r>, <r, r> (solver.py:95-101)
//
// x += alpha_k p_k (solver.py:94) is applied by the NEXT pass A, which stages
// p_k with its halos anyway and is latency- rather than bandwidth-bound, in
// the reference's rounding order x = fl(x + fl(alpha_k p_k)); the update of
// the last iteration is applied by x_flush_kernel at the end of a solve.  So
// pass B streams r and Ap only: 24 B/DoF (r, Ap in; r out).

constexpr int NTB = 256;

// TMA L2 promotion of the plane boxes: 64 B (256 B over-fetches the 32-byte
// misaligned haloed rows: pass A DRAM reads 19.7 -> 17.1 GB at 930^3)
constexpr CUtensorMapL2promotion kL2Promotion = CU_TENSOR_MAP_L2_PROMOTION_L2_64B;

// plain 16-byte loads/stores of the CG vectors (streaming cache hints were
// measured much slower)
__device__ __forceinline__ double2 ld2(const double* p) {
  return *reinterpret_cast<const double2*>(p);
}
__device__ __forceinline__ void st2(double* p, double2 v) { *reinterpret_cast<double2*>(p) = v; }

__global__ void __launch_bounds__(NTB) cg_pass_b_kernel(const __grid_constant__ PassBParams prm) {
  if (!ld_vol(&prm.state->active)) return;
  __shared__ double s_red[(NTB / 32) * 8];
  __shared__ unsigned s_last;
  extern __shared__ double s_inv[];
  const int ewz = prm.ew[0], ewy = prm.ew[1], ewx = prm.ew[2];
  const int ncy = 2 * ewy + 1, ncx = 2 * ewx + 1, ncz = 2 * ewz + 1;
  for (int i = threadIdx.x; i < ncz * ncy * ncx; i += NTB) s_inv[i] = prm.invd[i];
  __syncthreads();
  const double alpha = ld_vol(&prm.state->alpha);
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int nx = prm.nx, ny = prm.ny;
  const int nrows = prm.nz * ny;
  const int r0 = blockIdx.x * prm.rows_per_cta;
  const int r1 = min(r0 + prm.rows_per_cta, nrows);
  double rz = 0.0, rr = 0.0, rzl = 0.0, rrl = 0.0;  // double-double sums
  for (int row = r0 + warp; row < r1; row += NTB / 32) {
    const int zl = row / ny, y = row - zl * ny;
    const int cz = cls_of(prm.z_off + zl, prm.nz_glob, ewz);
    const int cy = cls_of(y, ny, ewy);
    const double* trow = s_inv + (cz * ncy + cy) * ncx;
    const double inv_int = trow[ewx];
    const long long base = (long long)(zl + prm.ghost) * prm.pitch_z + (long long)y * prm.pitch_y;
    double* rrw = prm.r + base;
    const double* apr = prm.ap + base;
    const int npair = nx >> 1;  // pitch is even: double2 rows
    int q = lane;
    // two pairs per step with every load issued before any store, for
    // memory-level parallelism
    for (; q + 32 < npair; q += 64) {
      const int xa = 2 * q, xb = 2 * (q + 32);
      const double2 ra = ld2(rrw + xa), aa = ld2(apr + xa);
      const double2 rb = ld2(rrw + xb), ab = ld2(apr + xb);
      const double ia0 = (xa >= ewx && xa < nx - ewx) ? inv_int : trow[cls_of(xa, nx, ewx)];
      const double ia1 = (xa + 1 >= ewx && xa + 1 < nx - ewx) ? inv_int : trow[cls_of(xa + 1, nx, ewx)];
      const double ib0 = (xb >= ewx && xb < nx - ewx) ? inv_int : trow[cls_of(xb, nx, ewx)];
      const double ib1 = (xb + 1 >= ewx && xb + 1 < nx - ewx) ? inv_int : trow[cls_of(xb + 1, nx, ewx)];
      double2 na, nb;
      na.x = __dsub_rn(ra.x, __dmul_rn(alpha, aa.x));
      na.y = __dsub_rn(ra.y, __dmul_rn(alpha, aa.y));
      nb.x = __dsub_rn(rb.x, __dmul_rn(alpha, ab.x));
      nb.y = __dsub_rn(rb.y, __dmul_rn(alpha, ab.y));
      // group sums of pairs q, q+32 (position-determined), added in dd
      double gz = __dmul_rn(na.x, __dmul_rn(ia0, na.x)), gr = __dmul_rn(na.x, na.x);
      gz = fma(na.y, __dmul_rn(ia1, na.y), gz);
      gr = fma(na.y, na.y, gr);
      gz = fma(nb.x, __dmul_rn(ib0, nb.x), gz);
      gr = fma(nb.x, nb.x, gr);
      gz = fma(nb.y, __dmul_rn(ib1, nb.y), gz);
      gr = fma(nb.y, nb.y, gr);
      dd_add(rz, rzl, gz);
      dd_add(rr, rrl, gr);
      st2(rrw + xa, na);
      st2(rrw + xb, nb);
    }
    for (; q < npair; q += 32) {
      const int xx = 2 * q;
      const double2 rv = ld2(rrw + xx);
      const double2 av = ld2(apr + xx);
      const double i0 = (xx >= ewx && xx < nx - ewx) ? inv_int : trow[cls_of(xx, nx, ewx)];
      const double i1 =
          (xx + 1 >= ewx && xx + 1 < nx - ewx) ? inv_int : trow[cls_of(xx + 1, nx, ewx)];
      double2 rn;
      rn.x = __dsub_rn(rv.x, __dmul_rn(alpha, av.x));
      rn.y = __dsub_rn(rv.y, __dmul_rn(alpha, av.y));
      double gz = __dmul_rn(rn.x, __dmul_rn(i0, rn.x)), gr = __dmul_rn(rn.x, rn.x);
      gz = fma(rn.y, __dmul_rn(i1, rn.y), gz);
      gr = fma(rn.y, rn.y, gr);
      dd_add(rz, rzl, gz);
      dd_add(rr, rrl, gr);
      st2(rrw + xx, rn);
    }
    if ((nx & 1) && lane == 0) {
      const int xx = nx - 1;
      const double i0 = trow[cls_of(xx, nx, ewx)];
      const double rn = __dsub_rn(rrw[xx], __dmul_rn(alpha, apr[xx]));
      rrw[xx] = rn;
      dd_add(rz, rzl, __dmul_rn(rn, __dmul_rn(i0, rn)));
      dd_add(rr, rrl, __dmul_rn(rn, rn));
    }
    // z-slab peer halos: a boundary row of the new r (and of p_k) is also a
    // neighbour's ghost row
    const bool plo = prm.peer_lo != nullptr && zl < prm.ghost;
    const bool phi = prm.peer_hi != nullptr && zl >= prm.nz - prm.ghost;
    if (plo || phi) {
      __syncwarp();
      const long long olo = base + (long long)prm.nz_lo * prm.pitch_z;
      const long long ohi = base - (long long)prm.nz * prm.pitch_z;
      const double* ps = prm.p_src ? prm.p_src + base : nullptr;
      for (int xx = lane; xx < nx; xx += 32) {
        const double rv = rrw[xx];
        const double pv = ps ? ps[xx] : 0.0;
        if (plo) {
          prm.peer_lo[olo + xx] = rv;
          if (ps && prm.p_lo) prm.p_lo[olo + xx] = pv;
        }
        if (phi) {
          prm.peer_hi[ohi + xx] = rv;
          if (ps && prm.p_hi) prm.p_hi[ohi + xx] = pv;
        }
      }
      __threadfence_system();
    }
  }
  double vh[2] = {rz, rr}, vl[2] = {rzl, rrl};
  reduce_and_finalize<2, NTB / 32>(vh, vl, s_red, &s_last, prm.partials, prm.counter, prm.state,
                                   prm.fuse, 2);
}

// Applies the pending x updates of a solve (iterations x_done .. it-1, in
// order, p_j in ring field j % kPRing).  Same row partition and double2
// accesses as pass B.
__global__ void __launch_bounds__(NTB) x_flush_kernel(const __grid_constant__ PassBParams prm) {
  const int it = ld_vol(&prm.state->it), j0 = ld_vol(&prm.state->x_done);
  const int R = ld_vol(&prm.state->ring);
  if (j0 >= it) return;
  double aj[kPRing];
  const double* pj[kPRing];
#pragma unroll
  for (int t = 0; t < kPRing; ++t) {
    const int j = j0 + t;
    const bool on = j < it && t < R;  // at most R - 1 updates are pending
    aj[t] = on ? ld_vol(&prm.state->alpha_ring[j % R]) : 0.0;
    pj[t] = on ? prm.pring + (long long)(j % R) * prm.pstride : nullptr;
  }
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int nx = prm.nx, ny = prm.ny;
  const int nrows = prm.nz * ny;
  const int r0 = blockIdx.x * prm.rows_per_cta;
  const int r1 = min(r0 + prm.rows_per_cta, nrows);
  if (it - j0 == 1) {
    // one pending update (the end of every solve): loads batched 4 deep
    const double a = aj[0];
    const double* p0 = pj[0];
    for (int row = r0 + warp; row < r1; row += NTB / 32) {
      const int zl = row / ny, y = row - zl * ny;
      const long long base =
          (long long)(zl + prm.ghost) * prm.pitch_z + (long long)y * prm.pitch_y;
      double* xr = prm.x + base;
      const double* pr = p0 + base;
      const int npair = nx >> 1;
      for (int q0 = lane; q0 < npair; q0 += 4 * 32) {
        double2 xv[4], pv[4];
#pragma unroll
        for (int u = 0; u < 4; ++u) {
          const int q = q0 + 32 * u;
          if (q < npair) {
            xv[u] = *reinterpret_cast<const double2*>(xr + 2 * q);
            pv[u] = *reinterpret_cast<const double2*>(pr + 2 * q);
          }
        }
#pragma unroll
        for (int u = 0; u < 4; ++u) {
          const int q = q0 + 32 * u;
          if (q < npair)
            *reinterpret_cast<double2*>(xr + 2 * q) =
                make_double2(__dadd_rn(xv[u].x, __dmul_rn(a, pv[u].x)),
                             __dadd_rn(xv[u].y, __dmul_rn(a, pv[u].y)));
        }
      }
      if ((nx & 1) && lane == 0) xr[nx - 1] = __dadd_rn(xr[nx - 1], __dmul_rn(a, pr[nx - 1]));
    }
    return;
  }
  for (int row = r0 + warp; row < r1; row += NTB / 32) {
    const int zl = row / ny, y = row - zl * ny;
    const long long base = (long long)(zl + prm.ghost) * prm.pitch_z + (long long)y * prm.pitch_y;
    double* xr = prm.x + base;
    const int npair = nx >> 1;
    for (int q = lane; q < npair; q += 32) {
      double2 xv = *reinterpret_cast<const double2*>(xr + 2 * q);
#pragma unroll
      for (int t = 0; t < kPRing; ++t) {
        if (pj[t]) {
          const double2 pv = *reinterpret_cast<const double2*>(pj[t] + base + 2 * q);
          xv.x = __dadd_rn(xv.x, __dmul_rn(aj[t], pv.x));
          xv.y = __dadd_rn(xv.y, __dmul_rn(aj[t], pv.y));
        }
      }
      *reinterpret_cast<double2*>(xr + 2 * q) = xv;
    }
    if ((nx & 1) && lane == 0) {
      double xs = xr[nx - 1];
#pragma unroll
      for (int t = 0; t < kPRing; ++t)
        if (pj[t]) xs = __dadd_rn(xs, __dmul_rn(aj[t], pj[t][base + nx - 1]));
      xr[nx - 1] = xs;
    }
  }
}

// ---------------------------------------------------------------------------
// B-spline field transforms (setup / I/O)
//
// Direct transform (node samples -> coefficients): the reference's separable
// causal/anticausal recursive prefilter (bspline.py:168-242), one thread per
// line, every operation in the reference's rounding order (gain, truncated
// series causal init at 1e-12, closed-form anticausal init).  Lines along y
// or z are coalesced across threads; lines along x (stride 1 per thread) reuse
// each 32-byte sector from L1 over four consecutive steps.

__device__ __forceinline__ int mirror_index(int i, int n) {
  if (n == 1) return 0;
  const int period = 2 * n - 2;
  i %= period;
  return i >= n ? period - i : i;
}

struct Lines {
  double* data;
  int n;               // line length
  long long stride;    // element stride along a line
  int na, nb;          // line grid (a varies fastest across threads)
  long long sa, sb;
};

__global__ void __launch_bounds__(128) prefilter_kernel(const Lines L, const int npoles,
                                                        const double z0, const double z1,
                                                        const int h0, const int h1,
                                                        const double gain, const int mode) {
  const long long line = blockIdx.x * (long long)blockDim.x + threadIdx.x;
  if (line >= (long long)L.na * L.nb) return;
  const int ia = (int)(line % L.na), ib = (int)(line / L.na);
  double* c = L.data + ia * L.sa + ib * L.sb;
  const long long s = L.stride;
  const int n = L.n;
  for (int ip = 0; ip < npoles; ++ip) {
    const double z = ip ? z1 : z0;
    const int H = ip ? h1 : h0;
    // the first cascade reads the raw samples times the gain (c = lines * gain)
    auto rd = [&](int k) -> double { return ip == 0 ? __dmul_rn(c[k * s], gain) : c[k * s]; };
    double init = rd(0), zk = 1.0;
    if (mode == 0) {  // mirror
      for (int k = 1; k < H; ++k) {
        zk = __dmul_rn(zk, z);
        init = __dadd_rn(init, __dmul_rn(zk, rd(mirror_index(k, n))));
      }
    } else {  // replicate (1) / zero (2)
      const int kmax = min(H, n);
      for (int k = 1; k < kmax; ++k) {
        zk = __dmul_rn(zk, z);
        init = __dadd_rn(init, __dmul_rn(zk, rd(k)));
      }
      if (mode == 1 && H > n)  // geometric tail of the replicated edge sample
        init = __dadd_rn(init, __ddiv_rn(__dmul_rn(rd(n - 1), pow(z, (double)n)), __dsub_rn(1.0, z)));
    }
    const double last = rd(n - 1);  // stage input at the right edge, pre-causal
    double prev = init, prev2 = 0.0;
    c[0] = init;
    for (int k = 1; k < n; ++k) {
      prev2 = prev;
      prev = __dadd_rn(rd(k), __dmul_rn(z, prev));
      c[k * s] = prev;
    }
    double cn;
    if (mode == 0) {
      cn = __dmul_rn(__ddiv_rn(z, __dsub_rn(__dmul_rn(z, z), 1.0)),
                     __dadd_rn(prev, __dmul_rn(z, n >= 2 ? prev2 : prev)));
    } else if (mode == 1) {
      const double s_inf = __ddiv_rn(last, __dsub_rn(1.0, z));
      cn = __dmul_rn(-z, __dadd_rn(__ddiv_rn(s_inf, __dsub_rn(1.0, z)),
                                   __ddiv_rn(__dsub_rn(prev, s_inf), __dsub_rn(1.0, __dmul_rn(z, z)))));
    } else {
      cn = __ddiv_rn(__dmul_rn(z, prev), __dsub_rn(__dmul_rn(z, z), 1.0));
    }
    c[(n - 1) * s] = cn;
    double nxt = cn;
    for (int k = n - 2; k >= 0; --k) {
      nxt = __dmul_rn(z, __dsub_rn(nxt, c[k * s]));
      c[k * s] = nxt;
    }
  }
}

// whole-sample reflection of the ext pad planes of one axis (np.pad "reflect")
__global__ void reflect_pad_kernel(double* data, const int d0, const int d1, const int d2,
                                   const long long s0, const long long s1, const long long s2,
                                   const int axis, const int ext) {
  // thread grid: the two other axes x (2*ext pad positions)
  const int da = axis == 0 ? d1 : d0, db = axis == 2 ? d1 : d2;
  const long long sa = axis == 0 ? s1 : s0, sb = axis == 2 ? s1 : s2;
  const int dn = axis == 0 ? d0 : (axis == 1 ? d1 : d2);
  const long long sn = axis == 0 ? s0 : (axis == 1 ? s1 : s2);
  const long long total = (long long)da * db * 2 * ext;
  for (long long t = blockIdx.x * (long long)blockDim.x + threadIdx.x; t < total;
       t += (long long)gridDim.x * blockDim.x) {
    const int ib = (int)(t % db);
    long long r = t / db;
    const int ia = (int)(r % da);
    const int q = (int)(r / da);  // 0..2*ext-1
    double* base = data + ia * sa + ib * sb;
    int dst, src;
    if (q < ext) {  // low side: index ext-1-i <- ext+1+i
      dst = ext - 1 - q;
      src = ext + 1 + q;
    } else {        // high side: index dn-ext+i <- dn-ext-2-i
      const int i = q - ext;
      dst = dn - ext + i;
      src = dn - ext - 2 - i;
    }
    base[dst * sn] = base[src * sn];
  }
}

// out[i] = sum_t taps[t] * in[i + offset + t] along one axis (separable FIR;
// sample_solution, problem.py:330-348), accumulated in the reference's order
constexpr int MAXFIR = 11;
struct Fir {
  const double* in;
  long long is0, is1, is2;
  double* out;
  int d0, d1, d2;  // output extents
  long long os0, os1, os2;
  int axis, offset, ntaps;
  double taps[MAXFIR];
};

__global__ void __launch_bounds__(256) fir_axis_kernel(const __grid_constant__ Fir f) {
  const long long total = (long long)f.d0 * f.d1 * f.d2;
  for (long long t = blockIdx.x * (long long)blockDim.x + threadIdx.x; t < total;
       t += (long long)gridDim.x * blockDim.x) {
    const int i2 = (int)(t % f.d2);
    const long long r = t / f.d2;
    const int i1 = (int)(r % f.d1), i0 = (int)(r / f.d1);
    const long long sa = f.axis == 0 ? f.is0 : (f.axis == 1 ? f.is1 : f.is2);
    const double* src = f.in + i0 * f.is0 + i1 * f.is1 + i2 * f.is2 + (long long)f.offset * sa;
    double acc = __dmul_rn(f.taps[0], src[0]);
    for (int k = 1; k < f.ntaps; ++k) acc = __dadd_rn(acc, __dmul_rn(f.taps[k], src[k * sa]));
    f.out[i0 * f.os0 + i1 * f.os1 + i2 * f.os2] = acc;
  }
}

// x = U^-1 L^-1 x in place along lines: the banded LU (no pivoting; same
// factors for every line) of the mirror-folded Gram system of the "l2"
// prefilter (_l2_project_axis, problem.py:142-175).  lb[i*m + k-1] = L[i, i-k],
// ub[i*(m+1) + k] = U[i, i+k].
__global__ void __launch_bounds__(128) banded_solve_kernel(const Lines L,
                                                           const double* __restrict__ lb,
                                                           const double* __restrict__ ub,
                                                           const int m) {
  const long long line = blockIdx.x * (long long)blockDim.x + threadIdx.x;
  if (line >= (long long)L.na * L.nb) return;
  const int ia = (int)(line % L.na), ib = (int)(line / L.na);
  double* c = L.data + ia * L.sa + ib * L.sb;
  const long long s = L.stride;
  const int n = L.n;
  for (int i = 1; i < n; ++i) {  // forward: unit lower band
    double v = c[i * s];
    for (int k = 1; k <= m && k <= i; ++k) v = fma(-lb[(long long)i * m + k - 1], c[(i - k) * s], v);
    c[i * s] = v;
  }
  for (int i = n - 1; i >= 0; --i) {  // backward: upper band
    double v = c[i * s];
    for (int k = 1; k <= m && i + k < n; ++k) v = fma(-ub[(long long)i * (m + 1) + k], c[(i + k) * s], v);
    c[i * s] = v / ub[(long long)i * (m + 1)];
  }
}

// out[.., i, ..] = sum_t w[i, t] * in[.., idx[i, t], ..] along one axis:
// spline evaluation on a lattice of points (indirect_transform,
// bspline.py:245-310, separably per axis), per-output taps and gather
// indices with the extension policy already folded into idx
struct Resample {
  const double* in;
  long long is0, is1, is2;
  double* out;
  int d0, d1, d2;  // output extents
  long long os0, os1, os2;
  int axis, ntaps;
  const int* idx;
  const double* w;
};

__global__ void __launch_bounds__(256) resample_axis_kernel(const __grid_constant__ Resample f) {
  const long long total = (long long)f.d0 * f.d1 * f.d2;
  for (long long t = blockIdx.x * (long long)blockDim.x + threadIdx.x; t < total;
       t += (long long)gridDim.x * blockDim.x) {
    const int i2 = (int)(t % f.d2);
    const long long r = t / f.d2;
    const int i1 = (int)(r % f.d1), i0 = (int)(r / f.d1);
    const int io = f.axis == 0 ? i0 : (f.axis == 1 ? i1 : i2);
    const long long sa = f.axis == 0 ? f.is0 : (f.axis == 1 ? f.is1 : f.is2);
    const double* src = f.in + (f.axis == 0 ? 0 : i0 * f.is0) + (f.axis == 1 ? 0 : i1 * f.is1) +
                        (f.axis == 2 ? 0 : i2 * f.is2);
    const int* ix = f.idx + (long long)io * f.ntaps;
    const double* wt = f.w + (long long)io * f.ntaps;
    double acc = 0.0;
    for (int k = 0; k < f.ntaps; ++k) acc = fma(wt[k], src[ix[k] * sa], acc);
    f.out[i0 * f.os0 + i1 * f.os1 + i2 * f.os2] = acc;
  }
}

// out[q] = sum_{i,j,k} wz[q,i] wy[q,j] wx[q,k] c[iz[q,i], iy[q,j], ix[q,k]]:
// the expansion at scattered points (indirect_transform, bspline.py:253-310),
// taps / folded indices per point and axis precomputed, one thread per point
__global__ void __launch_bounds__(256) eval_points_kernel(
    const double* __restrict__ c, long long sz, long long sy, long long sx, long long npts,
    int nt, const int* __restrict__ idx, const double* __restrict__ w, double* __restrict__ out) {
  for (long long q = blockIdx.x * (long long)blockDim.x + threadIdx.x; q < npts;
       q += (long long)gridDim.x * blockDim.x) {
    const int* iz = idx + q * nt;
    const int* iy = iz + npts * nt;
    const int* ix = iy + npts * nt;
    const double* wz = w + q * nt;
    const double* wy = wz + npts * nt;
    const double* wx = wy + npts * nt;
    double acc = 0.0;
    for (int a = 0; a < nt; ++a) {
      double ya = 0.0;
      for (int b = 0; b < nt; ++b) {
        const double* row = c + iz[a] * sz + iy[b] * sy;
        double xa = 0.0;
        for (int k = 0; k < nt; ++k) xa = fma(wx[k], row[ix[k] * sx], xa);
        ya = fma(wy[b], xa, ya);
      }
      acc = fma(wz[a], ya, acc);
    }
    out[q] = acc;
  }
}

// out = diag(A) expanded from the class table
__global__ void diag_kernel(const double* __restrict__ tab, int nx, int ny, int nz, int nz_glob,
                            int z_off, int ghost, long long pitch_y, long long pitch_z, int ewz,
                            int ewy, int ewx, double* __restrict__ out) {
  const int ncy = 2 * ewy + 1, ncx = 2 * ewx + 1;
  const long long total = (long long)nz * ny * nx;
  for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < total;
       i += (long long)gridDim.x * blockDim.x) {
    const int x = (int)(i % nx);
    const long long t = i / nx;
    const int y = (int)(t % ny);
    const int zl = (int)(t / ny);
    const int cz = cls_of(z_off + zl, nz_glob, ewz);
    out[(long long)(zl + ghost) * pitch_z + (long long)y * pitch_y + x] =
        tab[(cz * ncy + cls_of(y, ny, ewy)) * ncx + cls_of(x, nx, ewx)];
  }
}

// ---------------------------------------------------------------------------
// host side

thread_local std::string g_err;

int fail(int code, const std::string& msg) {
  g_err = msg;
  return code;
}

#define CUDA_TRY(expr)                                                                   \
  do {                                                                                   \
    cudaError_t _e = (expr);                                                             \
    if (_e != cudaSuccess)                                                               \
      return fail(BSPDE_ERR_CUDA, std::string(#expr) + ": " + cudaGetErrorString(_e));   \
  } while (0)

using EncodeTiledFn = CUresult (*)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*,
                                   const cuuint64_t*, const cuuint64_t*, const cuuint32_t*,
                                   const cuuint32_t*, CUtensorMapInterleave, CUtensorMapSwizzle,
                                   CUtensorMapL2promotion, CUtensorMapFloatOOBfill);

EncodeTiledFn get_encode() {
  static EncodeTiledFn fn = nullptr;
  if (!fn) {
    void* p = nullptr;
    cudaDriverEntryPointQueryResult q;
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q) ==
            cudaSuccess &&
        q == cudaDriverEntryPointSuccess)
      fn = reinterpret_cast<EncodeTiledFn>(p);
  }
  return fn;
}

struct KernelInfo {
  const void* fn;
  size_t smem;
  int ctas_per_sm;
  int nt;  // threads per CTA
};

struct Launch {
  int grid;
  int nchunks, chunk_len, nitems;
  int main_items = 0, tail_split = 1;
};

}  // namespace

struct bspde_plan {
  bspde_plan_desc d;
  int device = 0;
  int p;
  int NC;  // class stride of the device table (edge_width_of(p)*2+1)
  int num_sms;
  long long pitch_z;
  double* d_tab = nullptr;   // [3][2][NC*R]
  double* d_invd = nullptr;  // NCz*NCy*NCx
  int64_t launches = 0;
  // CUDA graph cache for the CG loop
  struct GraphKey {
    const void *x, *r, *p, *p2, *ap, *scratch;
    int k;
    bool operator<(const GraphKey& o) const {
      return std::tie(x, r, p, p2, ap, scratch, k) <
             std::tie(o.x, o.r, o.p, o.p2, o.ap, o.scratch, o.k);
    }
  };
  std::map<GraphKey, cudaGraphExec_t> graphs;
  void* host_state = nullptr;  // pinned CgState staging
  std::vector<double> host_tab;  // [axis][kind][NC][R]
  cudaStream_t work = nullptr;    // private stream: CUDA graphs cannot be captured on
  cudaEvent_t ev_in = nullptr;    // the legacy default stream the caller may use
  cudaEvent_t ev_out = nullptr;
  // per (kernel mode, planes streamed): plan_launch is a simulation
  std::map<std::pair<int, int>, Launch> launch_cache;
  bool peers = false;         // z-slab peer halos (bspde_slab_set_peers)
  bspde_slab_peers peer{};
  const double* peer_p_src = nullptr;  // p_k of the last pass A (its pass B copies the halo)
  double* peer_p_lo = nullptr;
  double* peer_p_hi = nullptr;
};

namespace {

template <int P, int MODE>
KernelInfo kernel_info() {
  using C = Cfg<P, MODE>;
  [[maybe_unused]] constexpr int NW = C::NW, NT = C::NT, TY = C::TY;
  KernelInfo ki;
  ki.fn = reinterpret_cast<const void*>(&sep_kernel<P, MODE>);
  ki.smem = C::smem_bytes();
  ki.nt = NT;
  static int ctas = -1;
  if (ctas < 0) {
    cudaFuncSetAttribute(ki.fn, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)ki.smem);
    int n = 0;
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&n, ki.fn, ki.nt, ki.smem);
    ctas = std::max(n, 1);
  }
  ki.ctas_per_sm = ctas;
  return ki;
}

template <int MODE>
KernelInfo kernel_info_p(int p) {
  switch (p) {
    case 1: return kernel_info<1, MODE>();
    case 2: return kernel_info<2, MODE>();
    case 3: return kernel_info<3, MODE>();
    case 4: return kernel_info<4, MODE>();
    default: return kernel_info<5, MODE>();
  }
}

#ifdef BSPDE_PROBE_P
// register/spill probe build (tools: ptxas of one instantiation)
KernelInfo kernel_for(int, int) { return kernel_info<BSPDE_PROBE_P, BSPDE_PROBE_MODE>(); }
#else
KernelInfo kernel_for(int p, int mode) {
  switch (mode) {
    case M_APPLY: return kernel_info_p<M_APPLY>(p);
    case M_MASS: return kernel_info_p<M_MASS>(p);
    case M_RESID: return kernel_info_p<M_RESID>(p);
    case M_HRES: return kernel_info_p<M_HRES>(p);
    default: return kernel_info_p<M_CGA>(p);
  }
}
#endif

bool kAsOf(int p) {
  switch (p) {
    case 1: return Cfg<1, M_HRES>::AS;
    case 2: return Cfg<2, M_HRES>::AS;
    case 3: return Cfg<3, M_HRES>::AS;
    case 4: return Cfg<4, M_HRES>::AS;
    default: return Cfg<5, M_HRES>::AS;
  }
}

// Choose the z-chunking.  Items are dealt round-robin (item i -> CTA
// i % grid, see item_geom), so the kernel time is the largest per-CTA sum of
// streamed planes (chunk + 2p warm-up), with edge tiles weighted by their
// measured extra cost.  Candidates: chunk counts nc (chunk length capped so
// CTAs stay close in z and share halo planes through L2), each with and
// without splitting the ragged last wave.  The plan is simulated exactly.
constexpr double kEdgeTileWeight = 1.08;  // edge-tile plane cost / interior (B200, p=3, measured)

Launch plan_launch(const bspde_plan* pl, const KernelInfo& ki, int nz, int mode) {
  const int TY = tile_h_of(pl->p, mode);
  const int tx = (pl->d.nx + TX - 1) / TX, ty = (pl->d.ny + TY - 1) / TY;
  const int tiles = tx * ty;
  const int slots = std::max(1, pl->num_sms * ki.ctas_per_sm);
  const int p = pl->p, px = p + (p & 1);
  if (const char* fc = getenv("BSPDE_FORCE_CHUNKS")) {  // debug / tuning override
    const int nc = std::max(1, std::min(nz, atoi(fc)));
    const int len = (nz + nc - 1) / nc;
    const int ncr = (nz + len - 1) / len;
    const long long items = (long long)tiles * ncr;
    Launch f{(int)std::min<long long>(items, slots), ncr, len, (int)items};
    f.main_items = (int)items;
    return f;
  }
  std::vector<double> w(tiles);
  for (int t = 0; t < tiles; ++t) {
    const int x0 = (t % tx) * TX, y0 = (t / tx) * TY;
    const bool in = (x0 - px >= pl->d.ew[2]) && (x0 + TX + px <= pl->d.nx - pl->d.ew[2]) &&
                    (y0 - p >= pl->d.ew[1]) && (y0 + TY + p <= pl->d.ny - pl->d.ew[1]);
    w[t] = in ? 1.0 : kEdgeTileWeight;
  }
  const char* ml = getenv("BSPDE_MAX_LEN");
  const int max_len = ml ? std::max(1, atoi(ml)) : 200;
  Launch best{1, 1, nz, tiles};
  best.main_items = tiles;
  double best_cost = 1e300;
  std::vector<double> load;
  for (int nc = 1; nc <= nz; ++nc) {
    const int len = (nz + nc - 1) / nc;
    const int ncr = (nz + len - 1) / len;
    if (len > max_len && nc < nz) continue;
    const long long items = (long long)tiles * ncr;
    if (items > (1 << 22)) break;
    const long long waves = items / slots;
    const long long rem = items - waves * slots;
    const int split_opt = rem > 0 ? (int)std::max<long long>(1, slots / rem) : 1;
    for (int split : {1, split_opt}) {
      const long long main_items = split > 1 ? waves * slots : items;
      const long long nitems = main_items + (items - main_items) * split;
      const int grid = (int)std::min<long long>(nitems, slots);
      const int sub = (len + split - 1) / split;
      load.assign(grid, 0.0);
      for (long long i = 0; i < nitems; ++i) {
        long long it = i;
        int zl;
        if (i < main_items) {
          const int ch = (int)(it / tiles);
          zl = std::min(len, nz - ch * len);
        } else {
          const long long jt = i - main_items;
          it = main_items + jt / split;
          const int sb = (int)(jt % split);
          const int ch = (int)(it / tiles);
          const int c1 = std::min(ch * len + len, nz);
          const int z0 = std::min(ch * len + sb * sub, c1);
          zl = std::min(z0 + sub, c1) - z0;
        }
        load[i % grid] += (zl + 2 * p) * w[it % tiles];
      }
      const double cost = *std::max_element(load.begin(), load.end());
      if (cost < best_cost * (1.0 - 1e-9)) {
        best_cost = cost;
        best = Launch{grid, ncr, len, (int)nitems};
        best.main_items = (int)main_items;
        best.tail_split = split;
      }
      if (split_opt == 1) break;
    }
    if (len <= 4 * p) break;
  }
  return best;
}

int make_map(CUtensorMap* m, const bspde_plan* pl, const double* base, int mode,
             bool owned_box = false) {
  EncodeTiledFn enc = get_encode();
  if (!enc) return fail(BSPDE_ERR_CUDA, "cuTensorMapEncodeTiled unavailable");
  const int p = pl->p;
  cuuint64_t dims[3] = {(cuuint64_t)pl->d.nx, (cuuint64_t)pl->d.ny,
                        (cuuint64_t)(pl->d.nz + 2 * p)};
  cuuint64_t strides[2] = {(cuuint64_t)(pl->d.pitch_y * 8), (cuuint64_t)(pl->pitch_z * 8)};
  const int px = p + (p & 1);
  cuuint32_t box[3] = {(cuuint32_t)(TX + 2 * px), (cuuint32_t)(tile_h_of(p, mode) + 2 * p), 1u};
  if (owned_box) {  // the tile itself (Cfg::AS)
    box[0] = TX;
    box[1] = (cuuint32_t)tile_h_of(p, mode);
  }
  cuuint32_t es[3] = {1u, 1u, 1u};
  CUresult rc = enc(m, CU_TENSOR_MAP_DATA_TYPE_FLOAT64, 3, const_cast<double*>(base), dims,
                    strides, box, es, CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE,
                    kL2Promotion, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  if (rc != CUDA_SUCCESS) return fail(BSPDE_ERR_CUDA, "cuTensorMapEncodeTiled failed (" +
                                                          std::to_string((int)rc) + ")");
  return BSPDE_OK;
}

void fill_common(SepParams& sp, const bspde_plan* pl, int mode) {
  const auto& d = pl->d;
  const int p = pl->p, R = 2 * p + 1;
  sp.nx = d.nx;
  sp.ny = d.ny;
  sp.nz = d.nz;
  sp.z_begin = 0;
  sp.z_end = d.nz;
  sp.accumulate = 0;
  sp.nz_glob = d.nz_global;
  sp.z_off = d.z_offset;
  sp.ghost = p;
  sp.pitch_y = d.pitch_y;
  sp.pitch_z = pl->pitch_z;
  for (int a = 0; a < 3; ++a) sp.ew[a] = d.ew[a];
  sp.tiles_x = (d.nx + TX - 1) / TX;
  sp.tiles_y = (d.ny + tile_h_of(pl->p, mode) - 1) / tile_h_of(pl->p, mode);
  for (int k = 0; k < MAXTAP; ++k) {
    sp.tzm[k] = sp.tzk[k] = sp.tym[k] = sp.tyk[k] = sp.txm[k] = sp.txk[k] = 0.0;
    sp.gm[k] = sp.gk[k] = 0.0;
  }
  for (int k = 0; k < R; ++k) {
    sp.tzm[k] = d.mass_table[0][d.ew[0] * R + k];
    sp.tzk[k] = d.c_stiff[0] * d.stiff_table[0][d.ew[0] * R + k];
    sp.tym[k] = d.mass_table[1][d.ew[1] * R + k];
    sp.tyk[k] = d.c_stiff[1] * d.stiff_table[1][d.ew[1] * R + k];
    sp.txm[k] = d.mass_table[2][d.ew[2] * R + k];
    sp.txk[k] = d.stiff_table[2][d.ew[2] * R + k];
    sp.gm[k] = kHostGramM[p - 1][k];
    sp.gk[k] = kHostGramK[p - 1][k];
  }
  sp.zfast = (d.nz_global > 1 && d.ew[0] > 0) ? 1 : 0;
  sp.c_mass = d.c_mass;
  sp.cx = d.c_stiff[2];
  sp.cy = d.c_stiff[1];
  sp.cz = d.c_stiff[0];
  sp.tab = pl->d_tab;
  sp.invd = pl->d_invd;
  sp.out = nullptr;
  sp.aux = nullptr;
  sp.aux_scale = 0.0;
  sp.rhs_cm = 0.0;
  sp.cg_r = nullptr;
  sp.cg_p = nullptr;
  sp.partials = nullptr;
  sp.counter = nullptr;
  sp.state = nullptr;
  sp.fuse = 1;
}

// scratch layout: CgState | partials[8*MAXGRID] (hi, lo of up to 4 sums) | counter
constexpr int MAXGRID = 4096;
size_t scratch_size() { return sizeof(CgState) + sizeof(double) * 8 * MAXGRID + 64; }
CgState* scratch_state(void* s) { return reinterpret_cast<CgState*>(s); }
double* scratch_partials(void* s) {
  return reinterpret_cast<double*>(reinterpret_cast<char*>(s) + sizeof(CgState));
}
unsigned* scratch_counter(void* s) {
  return reinterpret_cast<unsigned*>(reinterpret_cast<char*>(s) + sizeof(CgState) +
                                     sizeof(double) * 8 * MAXGRID);
}

int launch_sep(bspde_plan* pl, int mode, const double* in0, const double* in1, double* out,
               const double* aux, double aux_scale, double c_mass_override, bool use_override,
               void* scratch, int fuse, cudaStream_t st, double* cg_pout = nullptr,
               int z_begin = 0, int z_count = -1, int accumulate = 0, double* cg_x = nullptr) {
  KernelInfo ki = kernel_for(pl->p, mode);
  if (z_count < 0) z_count = pl->d.nz - z_begin;
  const auto key = std::make_pair(mode, z_count);
  auto lit = pl->launch_cache.find(key);
  if (lit == pl->launch_cache.end()) {
    lit = pl->launch_cache.emplace(key, plan_launch(pl, ki, z_count, mode)).first;
    if (getenv("BSPDE_PLAN_DEBUG"))
      fprintf(stderr, "bspde plan: mode %d grid %d chunks %d len %d items %d main %d split %d\n", mode,
              lit->second.grid, lit->second.nchunks, lit->second.chunk_len, lit->second.nitems,
              lit->second.main_items, lit->second.tail_split);
  }
  const Launch ln = lit->second;
  SepParams sp;
  fill_common(sp, pl, mode);
  sp.nchunks = ln.nchunks;
  sp.chunk_len = ln.chunk_len;
  sp.nitems = ln.nitems;
  sp.main_items = ln.main_items;
  sp.tail_split = ln.tail_split;
  sp.sub_len = (ln.chunk_len + ln.tail_split - 1) / ln.tail_split;
  sp.out = out;
  sp.aux = aux;
  sp.aux_scale = aux_scale;
  sp.cg_r = (mode == M_CGA) ? in0 : nullptr;
  sp.cg_p = (mode == M_CGA) ? in1 : nullptr;
  sp.cg_pout = cg_pout;
  sp.cg_x = cg_x;
  if (mode == M_CGA && pl->peers) {
    // z-slab peer halos: p_out is ring field k % R of this rank; the next
    // pass B stores its boundary planes into the neighbours' field k % R
    const bspde_slab_peers& q = pl->peer;
    const long long d = cg_pout ? cg_pout - q.ring : -1;
    pl->peer_p_src = nullptr;
    if (q.ring_stride > 0 && d >= 0 && d % q.ring_stride == 0 && d / q.ring_stride < q.ring_len) {
      const long long slot = d / q.ring_stride;
      pl->peer_p_src = cg_pout;
      pl->peer_p_lo = q.lo_ring ? q.lo_ring + slot * q.lo_ring_stride : nullptr;
      pl->peer_p_hi = q.hi_ring ? q.hi_ring + slot * q.hi_ring_stride : nullptr;
    }
  }
  if (mode == M_HRES)
    sp.rhs_cm = c_mass_override;  // the RHS mass scale (A keeps the plan's c_mass)
  else if (use_override)
    sp.c_mass = c_mass_override;
  if (scratch) {
    sp.state = scratch_state(scratch);
    sp.partials = scratch_partials(scratch);
    sp.counter = scratch_counter(scratch);
  }
  sp.fuse = fuse;
  sp.z_begin = z_begin;
  sp.z_end = z_begin + z_count;
  sp.accumulate = accumulate;
  if (ln.grid > MAXGRID) return fail(BSPDE_ERR_STATE, "grid exceeds MAXGRID");
  CUtensorMap m0, m1;
  int rc = make_map(&m0, pl, in0, mode);
  if (rc) return rc;
  if (in1) {
    rc = make_map(&m1, pl, in1, mode);
    if (rc) return rc;
  } else {
    m1 = m0;
  }
  CUtensorMap m2 = m0;
  if (mode == M_HRES && aux && kAsOf(pl->p)) {
    rc = make_map(&m2, pl, aux, mode, true);
    if (rc) return rc;
  }
  void* args[4] = {&sp, &m0, &m1, &m2};
  CUDA_TRY(cudaLaunchKernel(ki.fn, dim3(ln.grid), dim3(ki.nt), args, ki.smem, st));
  pl->launches++;
  return BSPDE_OK;
}

int launch_pass_b(bspde_plan* pl, double* x, double* r, const double* pring, const double* ap,
                  void* scratch, int fuse, cudaStream_t st, bool flush = false) {
  PassBParams bp;
  const auto& d = pl->d;
  bp.nx = d.nx;
  bp.ny = d.ny;
  bp.nz = d.nz;
  bp.nz_glob = d.nz_global;
  bp.z_off = d.z_offset;
  bp.ghost = pl->p;
  bp.pitch_y = d.pitch_y;
  bp.pitch_z = pl->pitch_z;
  for (int a = 0; a < 3; ++a) bp.ew[a] = d.ew[a];
  const int nrows = d.nz * d.ny;
  int grid = std::min(std::max(1, pl->num_sms * 6), std::min(MAXGRID, (nrows + 7) / 8));
  grid = std::max(grid, 1);
  bp.rows_per_cta = (nrows + grid - 1) / grid;
  grid = (nrows + bp.rows_per_cta - 1) / bp.rows_per_cta;
  bp.invd = pl->d_invd;
  bp.x = x;
  bp.r = r;
  bp.pring = pring;
  bp.pstride = (long long)(d.nz + 2 * pl->p) * pl->pitch_z;
  bp.ap = ap;
  bp.partials = scratch_partials(scratch);
  bp.counter = scratch_counter(scratch);
  bp.state = scratch_state(scratch);
  bp.fuse = fuse;
  bp.peer_lo = bp.peer_hi = bp.p_lo = bp.p_hi = nullptr;
  bp.p_src = nullptr;
  bp.nz_lo = 0;
  if (!flush && pl->peers && r && r == pl->peer.r) {
    bp.peer_lo = pl->peer.lo_r;
    bp.peer_hi = pl->peer.hi_r;
    bp.nz_lo = pl->peer.lo_nz;
    bp.p_src = pl->peer_p_src;
    bp.p_lo = pl->peer_p_lo;
    bp.p_hi = pl->peer_p_hi;
    pl->peer_p_src = nullptr;
  }
  const int ninv = (2 * d.ew[0] + 1) * (2 * d.ew[1] + 1) * (2 * d.ew[2] + 1);
  void* args[1] = {&bp};
  if (flush) {
    CUDA_TRY(cudaLaunchKernel(reinterpret_cast<const void*>(&x_flush_kernel), dim3(grid),
                              dim3(NTB), args, 0, st));
    finalize_kernel<<<1, 32, 0, st>>>(bp.state, 3);
    pl->launches += 2;
    CUDA_TRY(cudaGetLastError());
    return BSPDE_OK;
  }
  CUDA_TRY(cudaLaunchKernel(reinterpret_cast<const void*>(&cg_pass_b_kernel), dim3(grid),
                            dim3(NTB), args, sizeof(double) * ninv, st));
  pl->launches++;
  return BSPDE_OK;
}

int check_plan(const bspde_plan* pl) {
  if (!pl) return fail(BSPDE_ERR_ARG, "null plan");
  // the statically linked runtime keeps its own current-device state
  cudaError_t e = cudaSetDevice(pl->device);
  if (e != cudaSuccess) return fail(BSPDE_ERR_CUDA, std::string("cudaSetDevice: ") + cudaGetErrorString(e));
  return BSPDE_OK;
}

}  // namespace

// forward declarations of ABI functions used by the solve helper
extern "C" {
int bspde_cg_setup(bspde_plan*, void*, double*, const bspde_cg_config*, void*);
int bspde_cg_read_report(bspde_plan*, const void*, bspde_cg_report*, int32_t*, void*);
}
namespace {

// b == nullptr: heat step, r0 = (hcm M x + ha hf) - A x by the fused M_HRES
// kernel (b is never formed)
int pcg_solve_on(bspde_plan* pl, const double* b, double* x, double* r, double* pring,
                 double* ap, void* scratch, double* history, const bspde_cg_config* cfg,
                 bspde_cg_report* report, cudaStream_t st, const double* hf = nullptr,
                 double hcm = 0.0, double ha = 0.0) {
  void* stream = (void*)st;
  const size_t bytes = (size_t)(pl->d.nz + 2 * pl->p) * pl->pitch_z * sizeof(double);
  int rc = bspde_cg_setup(pl, scratch, history, cfg, stream);
  if (rc) return rc;
  if (!cfg->has_x0) CUDA_TRY(cudaMemsetAsync(x, 0, bytes, st));
  const int R = cfg->p_ring > 0 ? cfg->p_ring : 2;
  const long long fs = (long long)(pl->d.nz + 2 * pl->p) * pl->pitch_z;
  rc = b ? launch_sep(pl, M_RESID, x, nullptr, r, b, 0.0, 0.0, false, scratch, 1, st)
         : launch_sep(pl, M_HRES, x, nullptr, r, hf, ha, hcm, true, scratch, 1, st);
  if (rc) return rc;
  int32_t active = 0;
  rc = bspde_cg_read_report(pl, scratch, report, &active, stream);
  if (rc) return rc;
  if (active) {
    // iteration 0: beta = 0, so p_0 = D^-1 r + 0 * p_in for any finite p_in --
    // r itself is staged as p_{-1} (no zeroed field, no 6.4 GB memset per
    // solve at 930^3); it writes ring field 0
    rc = launch_sep(pl, M_CGA, r, r, ap, nullptr, 0.0, 0.0, false, scratch, 1, st, pring, 0, -1,
                    0, x);
    if (rc == BSPDE_OK) rc = launch_pass_b(pl, nullptr, r, nullptr, ap, scratch, 1, st);
    if (rc) return rc;
  }
  // iteration k >= 1 reads ring field (k-1) % R and writes k % R: chunks of a
  // multiple of R iterations (k = 1 .. K, K + 1 .. 2K, ...) make every replay
  // of the captured graph start from the same field
  int K = cfg->poll_every > 0 ? cfg->poll_every : 8;
  K = ((K + R - 1) / R) * R;
  while (active) {
    bspde_plan::GraphKey key{x, r, pring, nullptr, ap, scratch, K};
    auto itg = pl->graphs.find(key);
    cudaGraphExec_t exec = nullptr;
    if (itg == pl->graphs.end()) {
      cudaGraph_t graph = nullptr;
      CUDA_TRY(cudaStreamBeginCapture(st, cudaStreamCaptureModeThreadLocal));
      int crc = BSPDE_OK;
      for (int k = 1; k <= K && crc == BSPDE_OK; ++k) {
        crc = launch_sep(pl, M_CGA, r, pring + ((k + R - 1) % R) * fs, ap, nullptr, 0.0,
                         0.0, false, scratch, 1, st, pring + (k % R) * fs, 0, -1, 0, x);
        if (crc == BSPDE_OK) crc = launch_pass_b(pl, nullptr, r, nullptr, ap, scratch, 1, st);
      }
      cudaError_t ce = cudaStreamEndCapture(st, &graph);
      if (crc) {
        if (graph) cudaGraphDestroy(graph);
        return crc;
      }
      if (ce != cudaSuccess)
        return fail(BSPDE_ERR_CUDA, std::string("capture: ") + cudaGetErrorString(ce));
      ce = cudaGraphInstantiate(&exec, graph, 0);
      cudaGraphDestroy(graph);
      if (ce != cudaSuccess)
        return fail(BSPDE_ERR_CUDA, std::string("instantiate: ") + cudaGetErrorString(ce));
      pl->graphs[key] = exec;
      pl->launches -= 2 * K;  // captured launches are counted per replay below
    } else {
      exec = itg->second;
    }
    CUDA_TRY(cudaGraphLaunch(exec, st));
    pl->launches += 2 * K;
    rc = bspde_cg_read_report(pl, scratch, report, &active, stream);
    if (rc) return rc;
  }
  return launch_pass_b(pl, x, r, pring, ap, scratch, 1, st, /*flush=*/true);
}

}  // namespace

// ===========================================================================
// C ABI

extern "C" {

const char* bspde_last_error(void) { return g_err.c_str(); }

int bspde_version(void) { return 1; }

int bspde_device_ok(int device) {
  int dev = device;
  int n = 0;
  if (cudaGetDeviceCount(&n) != cudaSuccess || device < 0 || device >= n) return 0;
  cudaDeviceProp prop;
  if (cudaGetDeviceProperties(&prop, dev) != cudaSuccess) return 0;
  return prop.major == 10 ? 1 : 0;
}

int bspde_plan_create(const bspde_plan_desc* desc, bspde_plan** out) {
  if (!desc || !out) return fail(BSPDE_ERR_ARG, "null argument");
  const auto& d = *desc;
  if (d.degree < 1 || d.degree > MAXP) return fail(BSPDE_ERR_ARG, "degree must be in 1..5");
  if (d.nx < 1 || d.ny < 1 || d.nz < 1) return fail(BSPDE_ERR_ARG, "empty extents");
  if (d.pitch_y < d.nx || (d.pitch_y & 1)) return fail(BSPDE_ERR_ARG, "pitch_y must be even and >= nx");
  const int EW = edge_width_of(d.degree);
  for (int a = 0; a < 3; ++a) {
    if (d.ew[a] < 0 || d.ew[a] > EW) return fail(BSPDE_ERR_ARG, "edge width out of range");
    if (!d.mass_table[a] || !d.stiff_table[a]) return fail(BSPDE_ERR_ARG, "missing tables");
  }
  if (!d.inv_diag_table) return fail(BSPDE_ERR_ARG, "missing inverse diagonal table");
  // the fast paths use compile-time interior taps: a non-degenerate axis'
  // interior class row must be the unit Gram taps (faces live in edge rows)
  for (int a = 0; a < 3; ++a) {
    if (d.ew[a] == 0) continue;  // degenerate (padded) axis: tables only
    const int Rr = 2 * d.degree + 1;
    for (int k = 0; k < Rr; ++k) {
      const double m = d.mass_table[a][d.ew[a] * Rr + k], kk = d.stiff_table[a][d.ew[a] * Rr + k];
      const double gm = kHostGramM[d.degree - 1][k], gk = kHostGramK[d.degree - 1][k];
      if (std::fabs(m - gm) > 1e-15 * std::fabs(gm) || std::fabs(kk - gk) > 1e-15 * std::fabs(gk) + 1e-300)
        return fail(BSPDE_ERR_ARG, "interior table rows must be the unit B-spline Gram taps "
                                   "(scale with c_mass / c_stiff; faces go in the edge rows)");
    }
  }
  if (d.z_offset < 0 || d.z_offset + d.nz > d.nz_global) return fail(BSPDE_ERR_ARG, "bad z slab");
  if (d.device < 0) return fail(BSPDE_ERR_ARG, "bad device ordinal");
  {
    cudaError_t e = cudaSetDevice(d.device);
    if (e != cudaSuccess) return fail(BSPDE_ERR_CUDA, std::string("cudaSetDevice: ") + cudaGetErrorString(e));
  }
  auto* pl = new bspde_plan();
  pl->d = d;
  pl->device = d.device;
  pl->p = d.degree;
  pl->NC = 2 * EW + 1;
  pl->pitch_z = (long long)d.ny * d.pitch_y;
  cudaDeviceGetAttribute(&pl->num_sms, cudaDevAttrMultiProcessorCount, d.device);
  const int R = 2 * d.degree + 1;
  // device tables: [axis][kind][NC][R], classes beyond 2*ew unused
  std::vector<double> tab((size_t)6 * pl->NC * R, 0.0);
  for (int a = 0; a < 3; ++a) {
    const int nca = 2 * d.ew[a] + 1;
    for (int c = 0; c < nca; ++c)
      for (int k = 0; k < R; ++k) {
        tab[((a * 2 + 0) * pl->NC + c) * R + k] = d.mass_table[a][c * R + k];
        tab[((a * 2 + 1) * pl->NC + c) * R + k] = d.stiff_table[a][c * R + k];
      }
  }
  const int ninv = (2 * d.ew[0] + 1) * (2 * d.ew[1] + 1) * (2 * d.ew[2] + 1);
  cudaError_t e1 = cudaMalloc(&pl->d_tab, tab.size() * sizeof(double));
  cudaError_t e2 = cudaMalloc(&pl->d_invd, ninv * sizeof(double));
  cudaError_t e3 = cudaMallocHost(&pl->host_state, sizeof(CgState));
  cudaError_t e4 = cudaStreamCreateWithFlags(&pl->work, cudaStreamNonBlocking);
  cudaError_t e5 = cudaEventCreateWithFlags(&pl->ev_in, cudaEventDisableTiming);
  cudaError_t e6 = cudaEventCreateWithFlags(&pl->ev_out, cudaEventDisableTiming);
  if (e1 != cudaSuccess || e2 != cudaSuccess || e3 != cudaSuccess || e4 != cudaSuccess ||
      e5 != cudaSuccess || e6 != cudaSuccess) {
    bspde_plan_destroy(pl);
    return fail(BSPDE_ERR_CUDA, "plan allocation failed");
  }
  cudaMemcpy(pl->d_tab, tab.data(), tab.size() * sizeof(double), cudaMemcpyHostToDevice);
  cudaMemcpy(pl->d_invd, d.inv_diag_table, ninv * sizeof(double), cudaMemcpyHostToDevice);
  // the plan keeps copies of the host tables it needs later
  for (int a = 0; a < 3; ++a) {
    pl->d.mass_table[a] = nullptr;
    pl->d.stiff_table[a] = nullptr;
  }
  pl->d.inv_diag_table = nullptr;
  pl->host_tab = tab;
  for (int a = 0; a < 3; ++a) {
    pl->d.mass_table[a] = pl->host_tab.data() + ((a * 2 + 0) * pl->NC) * R;
    pl->d.stiff_table[a] = pl->host_tab.data() + ((a * 2 + 1) * pl->NC) * R;
  }
  // resolve kernel attributes before any stream capture
  for (int mode = 0; mode < 5; ++mode) kernel_for(pl->p, mode);
  cudaError_t e = cudaGetLastError();
  if (e != cudaSuccess) {
    bspde_plan_destroy(pl);
    return fail(BSPDE_ERR_CUDA, std::string("plan setup: ") + cudaGetErrorString(e));
  }
  *out = pl;
  return BSPDE_OK;
}

int bspde_plan_destroy(bspde_plan* pl) {
  if (!pl) return BSPDE_OK;
  for (auto& kv : pl->graphs) cudaGraphExecDestroy(kv.second);
  if (pl->d_tab) cudaFree(pl->d_tab);
  if (pl->d_invd) cudaFree(pl->d_invd);
  if (pl->host_state) cudaFreeHost(pl->host_state);
  if (pl->work) cudaStreamDestroy(pl->work);
  if (pl->ev_in) cudaEventDestroy(pl->ev_in);
  if (pl->ev_out) cudaEventDestroy(pl->ev_out);
  delete pl;
  return BSPDE_OK;
}

int64_t bspde_scratch_bytes(const bspde_plan* pl) {
  (void)pl;
  return (int64_t)scratch_size();
}

int64_t bspde_launch_count(const bspde_plan* pl) { return pl ? pl->launches : 0; }

int bspde_apply(bspde_plan* pl, const double* c, double* out, void* stream) {
  if (int rc = check_plan(pl)) return rc;
  if (!c || !out) return fail(BSPDE_ERR_ARG, "null field");
  return launch_sep(pl, M_APPLY, c, nullptr, out, nullptr, 0.0, 0.0, false, nullptr, 1,
                    (cudaStream_t)stream);
}

int bspde_mass_apply(bspde_plan* pl, const double* c, const double* f, double cm, double a,
                     double* out, void* stream) {
  if (int rc = check_plan(pl)) return rc;
  if (!c || !out) return fail(BSPDE_ERR_ARG, "null field");
  return launch_sep(pl, M_MASS, c, nullptr, out, f, a, cm, true, nullptr, 1,
                    (cudaStream_t)stream);
}

int bspde_prefilter_lines(double* data, int32_t n, int64_t stride, int32_t na, int32_t nb,
                          int64_t sa, int64_t sb, const double* poles, int32_t npoles,
                          double gain, int32_t extension, void* stream) {
  if (!data || (npoles > 0 && !poles)) return fail(BSPDE_ERR_ARG, "null argument");
  if (n < 1 || na < 0 || nb < 0) return fail(BSPDE_ERR_ARG, "bad line geometry");
  if (npoles < 0 || npoles > 2) return fail(BSPDE_ERR_ARG, "npoles must be 0..2 (degree <= 5)");
  if (extension < 0 || extension > 2) return fail(BSPDE_ERR_ARG, "extension must be 0 (mirror), 1 (replicate) or 2 (zero)");
  if (npoles > 0 && n < 2) return fail(BSPDE_ERR_ARG, "lines of length < 2 cannot be prefiltered");
  const long long lines = (long long)na * nb;
  if (lines == 0 || npoles == 0) {
    if (lines > 0 && gain != 1.0) return fail(BSPDE_ERR_ARG, "gain without poles");
    return BSPDE_OK;
  }
  int h[2] = {0, 0};
  for (int i = 0; i < npoles; ++i) {
    if (!(std::fabs(poles[i]) < 1.0) || poles[i] == 0.0) return fail(BSPDE_ERR_ARG, "poles must be in (-1, 1) \\ {0}");
    // horizon of the truncated causal-init series at relative tolerance 1e-12
    h[i] = (int)std::ceil(std::log(1e-12) / std::log(std::fabs(poles[i]))) + 1;
  }
  Lines L{data, n, stride, na, nb, sa, sb};
  const int threads = 128;
  prefilter_kernel<<<(unsigned)((lines + threads - 1) / threads), threads, 0, (cudaStream_t)stream>>>(
      L, npoles, poles[0], npoles > 1 ? poles[1] : 0.0, h[0], h[1], gain, extension);
  CUDA_TRY(cudaGetLastError());
  return BSPDE_OK;
}

int bspde_banded_solve_lines(double* data, int32_t n, int64_t stride, int32_t na, int32_t nb,
                             int64_t sa, int64_t sb, const double* lb, const double* ub,
                             int32_t m, void* stream) {
  if (!data || !lb || !ub) return fail(BSPDE_ERR_ARG, "null argument");
  if (n < 1 || na < 0 || nb < 0 || m < 1 || m > 8) return fail(BSPDE_ERR_ARG, "bad line geometry / band");
  const long long lines = (long long)na * nb;
  if (lines == 0) return BSPDE_OK;
  Lines L{data, n, stride, na, nb, sa, sb};
  const int threads = 128;
  banded_solve_kernel<<<(unsigned)((lines + threads - 1) / threads), threads, 0, (cudaStream_t)stream>>>(
      L, lb, ub, m);
  CUDA_TRY(cudaGetLastError());
  return BSPDE_OK;
}

int bspde_reflect_pad(double* data, const int32_t* dims, const int64_t* strides, int32_t axis,
                      int32_t ext, void* stream) {
  if (!data || !dims || !strides) return fail(BSPDE_ERR_ARG, "null argument");
  if (axis < 0 || axis > 2 || ext < 0) return fail(BSPDE_ERR_ARG, "bad axis / ext");
  if (ext == 0) return BSPDE_OK;
  if (dims[axis] < 2 * ext + ext + 2) return fail(BSPDE_ERR_ARG, "axis too short to reflect");
  const long long other = (long long)dims[0] * dims[1] * dims[2] / dims[axis];
  const long long total = other * 2 * ext;
  const int threads = 256;
  const unsigned blocks = (unsigned)std::min<long long>((total + threads - 1) / threads, 1 << 20);
  reflect_pad_kernel<<<blocks, threads, 0, (cudaStream_t)stream>>>(
      data, dims[0], dims[1], dims[2], strides[0], strides[1], strides[2], axis, ext);
  CUDA_TRY(cudaGetLastError());
  return BSPDE_OK;
}

int bspde_fir_axis(const double* in, const int64_t* in_strides, double* out,
                   const int32_t* out_dims, const int64_t* out_strides, int32_t axis,
                   int32_t offset, const double* taps, int32_t ntaps, void* stream) {
  if (!in || !in_strides || !out || !out_dims || !out_strides || !taps)
    return fail(BSPDE_ERR_ARG, "null argument");
  if (axis < 0 || axis > 2 || ntaps < 1 || ntaps > MAXFIR) return fail(BSPDE_ERR_ARG, "bad axis / taps");
  Fir f;
  f.in = in;
  f.is0 = in_strides[0];
  f.is1 = in_strides[1];
  f.is2 = in_strides[2];
  f.out = out;
  f.d0 = out_dims[0];
  f.d1 = out_dims[1];
  f.d2 = out_dims[2];
  f.os0 = out_strides[0];
  f.os1 = out_strides[1];
  f.os2 = out_strides[2];
  f.axis = axis;
  f.offset = offset;
  f.ntaps = ntaps;
  for (int k = 0; k < MAXFIR; ++k) f.taps[k] = k < ntaps ? taps[k] : 0.0;
  const long long total = (long long)f.d0 * f.d1 * f.d2;
  if (total == 0) return BSPDE_OK;
  const int threads = 256;
  const unsigned blocks = (unsigned)std::min<long long>((total + threads - 1) / threads, 1 << 20);
  void* args[1] = {&f};
  CUDA_TRY(cudaLaunchKernel(reinterpret_cast<const void*>(&fir_axis_kernel), dim3(blocks),
                            dim3(threads), args, 0, (cudaStream_t)stream));
  return BSPDE_OK;
}

int bspde_resample_axis(const double* in, const int64_t* in_strides, double* out,
                        const int32_t* out_dims, const int64_t* out_strides, int32_t axis,
                        const int32_t* idx, const double* w, int32_t ntaps, void* stream) {
  if (!in || !in_strides || !out || !out_dims || !out_strides || !idx || !w)
    return fail(BSPDE_ERR_ARG, "null argument");
  if (axis < 0 || axis > 2 || ntaps < 1 || ntaps > MAXFIR) return fail(BSPDE_ERR_ARG, "bad axis / taps");
  Resample f;
  f.in = in;
  f.is0 = in_strides[0];
  f.is1 = in_strides[1];
  f.is2 = in_strides[2];
  f.out = out;
  f.d0 = out_dims[0];
  f.d1 = out_dims[1];
  f.d2 = out_dims[2];
  f.os0 = out_strides[0];
  f.os1 = out_strides[1];
  f.os2 = out_strides[2];
  f.axis = axis;
  f.ntaps = ntaps;
  f.idx = idx;
  f.w = w;
  const long long total = (long long)f.d0 * f.d1 * f.d2;
  if (total == 0) return BSPDE_OK;
  const int threads = 256;
  const unsigned blocks = (unsigned)std::min<long long>((total + threads - 1) / threads, 1 << 20);
  void* args[1] = {&f};
  CUDA_TRY(cudaLaunchKernel(reinterpret_cast<const void*>(&resample_axis_kernel), dim3(blocks),
                            dim3(threads), args, 0, (cudaStream_t)stream));
  return BSPDE_OK;
}

int bspde_eval_points(const double* c, const int64_t* strides, int64_t npts, int32_t ntaps,
                      const int32_t* idx, const double* w, double* out, void* stream) {
  if (!c || !strides || !idx || !w || !out) return fail(BSPDE_ERR_ARG, "null argument");
  if (ntaps < 1 || ntaps > MAXFIR || npts < 0) return fail(BSPDE_ERR_ARG, "bad taps / point count");
  if (npts == 0) return BSPDE_OK;
  const unsigned blocks = (unsigned)std::min<long long>((npts + 255) / 256, 1 << 20);
  eval_points_kernel<<<blocks, 256, 0, (cudaStream_t)stream>>>(c, strides[0], strides[1],
                                                              strides[2], npts, ntaps, idx, w, out);
  CUDA_TRY(cudaGetLastError());
  return BSPDE_OK;
}

int bspde_jacobi_diagonal(bspde_plan* pl, const double* diag_table, double* out, void* stream) {
  if (int rc = check_plan(pl)) return rc;
  const auto& d = pl->d;
  const int ninv = (2 * d.ew[0] + 1) * (2 * d.ew[1] + 1) * (2 * d.ew[2] + 1);
  double* dt = nullptr;
  CUDA_TRY(cudaMalloc(&dt, ninv * sizeof(double)));
  CUDA_TRY(cudaMemcpy(dt, diag_table, ninv * sizeof(double), cudaMemcpyHostToDevice));
  const long long total = (long long)d.nz * d.ny * d.nx;
  const int grid = (int)std::min<long long>((total + 255) / 256, pl->num_sms * 8);
  diag_kernel<<<std::max(grid, 1), 256, 0, (cudaStream_t)stream>>>(
      dt, d.nx, d.ny, d.nz, d.nz_global, d.z_offset, pl->p, d.pitch_y, pl->pitch_z, d.ew[0],
      d.ew[1], d.ew[2], out);
  pl->launches++;
  CUDA_TRY(cudaGetLastError());
  CUDA_TRY(cudaStreamSynchronize((cudaStream_t)stream));
  CUDA_TRY(cudaFree(dt));
  return BSPDE_OK;
}

int bspde_cg_setup(bspde_plan* pl, void* scratch, double* history, const bspde_cg_config* cfg,
                   void* stream) {
  if (int rc = check_plan(pl)) return rc;
  if (!scratch || !cfg) return fail(BSPDE_ERR_ARG, "null argument");
  if (!(cfg->tol > 0.0)) return fail(BSPDE_ERR_ARG, "tol must be positive");
  if (cfg->max_iter < 1) return fail(BSPDE_ERR_ARG, "max_iter must be >= 1");
  if (cfg->record_history && !history) return fail(BSPDE_ERR_ARG, "history buffer required");
  if (!(cfg->p_ring == 0 || cfg->p_ring == 2 || cfg->p_ring == kPRing))
    return fail(BSPDE_ERR_ARG, "p_ring must be 2 or 4 (0: default 2)");
  CgState* hs = reinterpret_cast<CgState*>(pl->host_state);
  cudaStream_t st = (cudaStream_t)stream;
  // the pinned staging buffer may still be in use by a previous async copy
  CUDA_TRY(cudaStreamSynchronize(st));
  std::memset(hs, 0, sizeof(CgState));
  hs->tol = cfg->tol;
  hs->max_iter = cfg->max_iter;
  hs->record_history = cfg->record_history ? 1 : 0;
  hs->has_x0 = cfg->has_x0 ? 1 : 0;
  hs->ring = cfg->p_ring > 0 ? cfg->p_ring : 2;
  hs->history = history;
  hs->scale = 1.0;
  CUDA_TRY(cudaMemcpyAsync(scratch_state(scratch), hs, sizeof(CgState), cudaMemcpyHostToDevice, st));
  CUDA_TRY(cudaMemsetAsync(scratch_counter(scratch), 0, 64, st));
  return BSPDE_OK;
}

int bspde_cg_residual(bspde_plan* pl, const double* b, const double* x, double* r,
                      void* scratch, int fuse, void* stream) {
  if (int rc = check_plan(pl)) return rc;
  if (!b || !x || !r || !scratch) return fail(BSPDE_ERR_ARG, "null argument");
  return launch_sep(pl, M_RESID, x, nullptr, r, b, 0.0, 0.0, false, scratch, fuse,
                    (cudaStream_t)stream);
}

int bspde_cg_pass_a(bspde_plan* pl, double* x, const double* r, const double* p_in,
                    double* p_out, double* ap, void* scratch, int fuse, void* stream) {
  if (int rc = check_plan(pl)) return rc;
  if (!x || !r || !p_in || !p_out || !ap || !scratch) return fail(BSPDE_ERR_ARG, "null argument");
  if (p_in == p_out) return fail(BSPDE_ERR_ARG, "p_in and p_out must be different buffers");
  return launch_sep(pl, M_CGA, r, p_in, ap, nullptr, 0.0, 0.0, false, scratch, fuse,
                    (cudaStream_t)stream, p_out, 0, -1, 0, x);
}

int bspde_cg_pass_a_range(bspde_plan* pl, double* x, const double* r, const double* p_in,
                          double* p_out, double* ap, void* scratch, int z_begin, int z_count,
                          int accumulate, int fuse, void* stream) {
  if (int rc = check_plan(pl)) return rc;
  if (!x || !r || !p_in || !p_out || !ap || !scratch) return fail(BSPDE_ERR_ARG, "null argument");
  if (p_in == p_out) return fail(BSPDE_ERR_ARG, "p_in and p_out must be different buffers");
  if (z_begin < 0 || z_count < 1 || z_begin + z_count > pl->d.nz)
    return fail(BSPDE_ERR_ARG, "z range outside the owned planes");
  return launch_sep(pl, M_CGA, r, p_in, ap, nullptr, 0.0, 0.0, false, scratch, fuse,
                    (cudaStream_t)stream, p_out, z_begin, z_count, accumulate ? 1 : 0, x);
}

int bspde_cg_pass_b(bspde_plan* pl, double* r, const double* ap, void* scratch, int fuse,
                    void* stream) {
  if (int rc = check_plan(pl)) return rc;
  if (!r || !ap || !scratch) return fail(BSPDE_ERR_ARG, "null argument");
  return launch_pass_b(pl, nullptr, r, nullptr, ap, scratch, fuse, (cudaStream_t)stream);
}

int bspde_cg_flush_x(bspde_plan* pl, double* x, const double* p_ring, void* scratch,
                     void* stream) {
  if (int rc = check_plan(pl)) return rc;
  if (!x || !p_ring || !scratch) return fail(BSPDE_ERR_ARG, "null argument");
  return launch_pass_b(pl, x, nullptr, p_ring, nullptr, scratch, 1, (cudaStream_t)stream,
                       /*flush=*/true);
}

int bspde_cg_finalize(bspde_plan* pl, void* scratch, int kind, void* stream) {
  if (int rc = check_plan(pl)) return rc;
  if (kind < 0 || kind > 3) return fail(BSPDE_ERR_ARG, "finalize kind must be 0..3");
  finalize_kernel<<<1, 32, 0, (cudaStream_t)stream>>>(scratch_state(scratch), kind);
  pl->launches++;
  CUDA_TRY(cudaGetLastError());
  return BSPDE_OK;
}

int bspde_slab_set_peers(bspde_plan* pl, const bspde_slab_peers* peers) {
  if (int rc = check_plan(pl)) return rc;
  pl->peer_p_src = nullptr;
  if (!peers) {
    pl->peers = false;
    pl->peer = bspde_slab_peers{};
    return BSPDE_OK;
  }
  const bspde_slab_peers& q = *peers;
  if (!q.ring || !q.r || q.ring_stride <= 0 || q.ring_len < 2 || q.ring_len > kPRing)
    return fail(BSPDE_ERR_ARG, "slab peers: bad ring / r");
  if ((q.lo_ring == nullptr) != (q.lo_r == nullptr) || (q.hi_ring == nullptr) != (q.hi_r == nullptr))
    return fail(BSPDE_ERR_ARG, "slab peers: a neighbour needs both its ring and r");
  if (q.lo_ring && (q.lo_ring_stride <= 0 || q.lo_nz < pl->p))
    return fail(BSPDE_ERR_ARG, "slab peers: bad lower neighbour");
  if (q.hi_ring && q.hi_ring_stride <= 0) return fail(BSPDE_ERR_ARG, "slab peers: bad upper neighbour");
  if (pl->d.nz < pl->p) return fail(BSPDE_ERR_ARG, "slab peers: slab thinner than the halo");
  pl->peer = q;
  pl->peers = true;
  return BSPDE_OK;
}

namespace {
using GetRangeFn = CUresult (*)(CUdeviceptr*, size_t*, CUdeviceptr);
GetRangeFn get_range_fn() {
  static GetRangeFn fn = nullptr;
  if (!fn) {
    void* p = nullptr;
    cudaDriverEntryPointQueryResult q;
    if (cudaGetDriverEntryPoint("cuMemGetAddressRange", &p, cudaEnableDefault, &q) == cudaSuccess &&
        q == cudaDriverEntryPointSuccess)
      fn = reinterpret_cast<GetRangeFn>(p);
  }
  return fn;
}
}  // namespace

int bspde_ipc_export(const void* ptr, void* handle, uint64_t* offset) {
  if (!ptr || !handle || !offset) return fail(BSPDE_ERR_ARG, "null argument");
  GetRangeFn rng = get_range_fn();
  if (!rng) return fail(BSPDE_ERR_CUDA, "cuMemGetAddressRange unavailable");
  CUdeviceptr base = 0;
  size_t size = 0;
  if (rng(&base, &size, (CUdeviceptr)ptr) != CUDA_SUCCESS)
    return fail(BSPDE_ERR_ARG, "ipc export: not a device allocation");
  cudaIpcMemHandle_t h;
  CUDA_TRY(cudaIpcGetMemHandle(&h, (void*)base));
  std::memcpy(handle, &h, sizeof(h));
  *offset = (uint64_t)((const char*)ptr - (const char*)base);
  return BSPDE_OK;
}

int bspde_ipc_import(const void* handle, uint64_t offset, void** ptr) {
  if (!handle || !ptr) return fail(BSPDE_ERR_ARG, "null argument");
  cudaIpcMemHandle_t h;
  std::memcpy(&h, handle, sizeof(h));
  void* base = nullptr;
  CUDA_TRY(cudaIpcOpenMemHandle(&base, h, cudaIpcMemLazyEnablePeerAccess));
  *ptr = (char*)base + offset;
  return BSPDE_OK;
}

int bspde_ipc_close(void* ptr) {
  if (!ptr) return BSPDE_OK;
  GetRangeFn rng = get_range_fn();
  CUdeviceptr base = (CUdeviceptr)ptr;
  size_t size = 0;
  if (rng) rng(&base, &size, (CUdeviceptr)ptr);
  CUDA_TRY(cudaIpcCloseMemHandle((void*)base));
  return BSPDE_OK;
}

int bspde_cg_finalize_gathered(bspde_plan* pl, void* scratch, const void* gathered, int world,
                               int kind, void* stream) {
  if (int rc = check_plan(pl)) return rc;
  if (kind < 0 || kind > 2) return fail(BSPDE_ERR_ARG, "finalize_gathered kind must be 0..2");
  if (world < 1 || !gathered) return fail(BSPDE_ERR_ARG, "finalize_gathered: bad world/buffer");
  finalize_gathered_kernel<<<1, 32, 0, (cudaStream_t)stream>>>(
      scratch_state(scratch), (const double*)gathered, world, kind);
  pl->launches++;
  CUDA_TRY(cudaGetLastError());
  return BSPDE_OK;
}

int bspde_cg_read_report(bspde_plan* pl, const void* scratch, bspde_cg_report* rep,
                         int32_t* active, void* stream) {
  if (int rc = check_plan(pl)) return rc;
  cudaStream_t st = (cudaStream_t)stream;
  CgState* hs = reinterpret_cast<CgState*>(pl->host_state);
  CUDA_TRY(cudaMemcpyAsync(hs, scratch_state(const_cast<void*>(scratch)), sizeof(CgState),
                           cudaMemcpyDeviceToHost, st));
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

int bspde_heat_residual(bspde_plan* pl, const double* u, const double* f, double cm, double a,
                        double* r, void* scratch, int fuse, void* stream) {
  if (int rc = check_plan(pl)) return rc;
  if (!u || !r || !scratch) return fail(BSPDE_ERR_ARG, "null argument");
  return launch_sep(pl, M_HRES, u, nullptr, r, f, f ? a : 0.0, cm, true, scratch, fuse,
                    (cudaStream_t)stream);
}

int bspde_heat_step(bspde_plan* pl, double* u, const double* f, double cm, double a, double* r,
                    double* p_ring, double* ap, void* scratch, double* history,
                    const bspde_cg_config* cfg, bspde_cg_report* report, void* stream) {
  if (int rc = check_plan(pl)) return rc;
  if (!u || !r || !p_ring || !ap || !scratch || !cfg) return fail(BSPDE_ERR_ARG, "null argument");
  if (!cfg->has_x0) return fail(BSPDE_ERR_ARG, "a heat step starts from x0 = u (has_x0 = 1)");
  cudaStream_t caller = (cudaStream_t)stream;
  cudaStream_t st = pl->work;
  CUDA_TRY(cudaEventRecord(pl->ev_in, caller));
  CUDA_TRY(cudaStreamWaitEvent(st, pl->ev_in, 0));
  int rc = pcg_solve_on(pl, nullptr, u, r, p_ring, ap, scratch, history, cfg, report, st, f, cm,
                        f ? a : 0.0);
  cudaEventRecord(pl->ev_out, st);
  cudaStreamWaitEvent(caller, pl->ev_out, 0);
  return rc;
}

int bspde_pcg_solve(bspde_plan* pl, const double* b, double* x, double* r, double* p_ring,
                    double* ap, void* scratch, double* history, const bspde_cg_config* cfg,
                    bspde_cg_report* report, void* stream) {
  if (int rc = check_plan(pl)) return rc;
  if (!b || !x || !r || !p_ring || !ap || !scratch || !cfg)
    return fail(BSPDE_ERR_ARG, "null argument");
  // everything runs on the plan's private stream, ordered after the caller's
  // stream on entry and before it on exit
  cudaStream_t caller = (cudaStream_t)stream;
  cudaStream_t st = pl->work;
  CUDA_TRY(cudaEventRecord(pl->ev_in, caller));
  CUDA_TRY(cudaStreamWaitEvent(st, pl->ev_in, 0));
  int rc = pcg_solve_on(pl, b, x, r, p_ring, ap, scratch, history, cfg, report, st);
  cudaEventRecord(pl->ev_out, st);
  cudaStreamWaitEvent(caller, pl->ev_out, 0);
  return rc;
}

}  // extern "C"

#include "stencil.cuh"
#include "otf.cuh"
