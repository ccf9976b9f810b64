// Pseudo-acoustic TTI time step (K2 in SURVEY.md §2.1) for sm_100a.
//
// Operator (paper_1807_03032_b200/operators.py:tti_equations, authored with
// the reference API): with a = (sin th cos ph, sin th sin ph, cos th),
//   g_f   = a . grad_R f                (first derivatives, order so/2)
//   Hz f  = sum_i a_i d_i(g_f)          (same order; reach so/2 = halo)
//   Hxy p = lap_so p - Hz p
//   p+ = (m/dt^2 (2p - p-) + damp/(2dt) p- + (1+2eps) Hxy p + sqrt(1+2delta) Hz r) / (m/dt^2 + damp/(2dt))
//   r+ = (m/dt^2 (2r - r-) + damp/(2dt) r- + sqrt(1+2delta) Hxy p + Hz r)        / (m/dt^2 + damp/(2dt))
// which is the solve_for rearrangement of the authored equations. The
// arithmetic order is the kernel's own (FMA, factorised symmetric pairs):
// parity with the oracle is at the fp32 rounding floor, not bitwise.
//
// Two passes per step: tti_inner writes the rotated first-derivative
// temporaries g_p, g_r (both fields in one pass) over the loop box widened
// by the outer radius; tti_outer fuses lap, the outer rotated derivatives
// of both fields and both updates.
#include <algorithm>
#include <cstring>
#include <climits>
#include <map>
#include <memory>
#include <mutex>
#include <tuple>
#include <type_traits>
#include <unordered_map>

#include "common.cuh"
#include "kernels.cuh"

namespace {

constexpr int BZ = 32, BYT = 8;

template <typename T> struct TtiArgs {
  const T *p, *r, *pm, *rm;  // current and previous slots
  T *pn, *rn;                // next slots
  const T *m, *damp, *eps, *delta, *theta, *phi;
  T *gp, *gr;                // scratch, field layout
  int lo[3], hi[3];          // loop box
  int64_t E1, E2;            // storage extents y, z (x implied)
  int H;
  T invh[3], invh2[3];
  T dt2inv, dtinv2;          // 1/dt^2, 1/(2 dt)
  T c1[5];                   // first-derivative weights, k = 1..R
  T c2[9];                   // second-derivative weights, k = 0..H
};

template <typename T> __device__ __forceinline__ void direction(T th, T ph, T &ax, T &ay, T &az) {
  T st, ct, sp, cp;
  if (sizeof(T) == 4) {
    sincosf((float)th, (float *)&st, (float *)&ct);
    sincosf((float)ph, (float *)&sp, (float *)&cp);
  } else {
    sincos((double)th, (double *)&st, (double *)&ct);
    sincos((double)ph, (double *)&sp, (double *)&cp);
  }
  ax = st * cp;
  ay = st * sp;
  az = ct;
}

// Both passes stream along x: a thread owns one (y, z) column and walks a
// chunk of x planes; x neighbours come from per-thread register queues
// (p, r in pass 1; p, g_p, g_r in pass 2), y/z neighbours are read through
// L1 (the CTA's tile plus halo of the current plane stays L1-resident).
constexpr int XCH = 48;  // x planes per CTA

template <typename T, int SO>
__global__ void __launch_bounds__(BZ *BYT) tti_inner(const TtiArgs<T> a) {
  constexpr int R = SO / 4 > 0 ? SO / 4 : 1;
  constexpr int Q = 2 * R + 1;
  const int z = a.lo[2] - R + blockIdx.x * BZ + threadIdx.x;
  const int y = a.lo[1] - R + blockIdx.y * BYT + threadIdx.y;
  const int xb = a.lo[0] - R + blockIdx.z * XCH;            // first g plane
  const int xe = min(xb + XCH, a.hi[0] + R + 1);            // one past last
  if (z > a.hi[2] + R || y > a.hi[1] + R) return;
  const int H = a.H;
  const int64_t sx = a.E1 * a.E2, sy = a.E2;
  const int64_t col = (int64_t)(y + H) * sy + (z + H);
  T qp[Q], qr[Q];  // planes x-R .. x+R
#pragma unroll
  for (int i = 0; i < Q - 1; ++i) {
    const int64_t c = (int64_t)(xb - R + i + H) * sx + col;
    qp[i + 1] = __ldg(a.p + c);
    qr[i + 1] = __ldg(a.r + c);
  }
  for (int x = xb; x < xe; ++x) {
#pragma unroll
    for (int i = 0; i < Q - 1; ++i) {
      qp[i] = qp[i + 1];
      qr[i] = qr[i + 1];
    }
    const int64_t c = (int64_t)(x + H) * sx + col;
    qp[Q - 1] = __ldg(a.p + c + R * sx);
    qr[Q - 1] = __ldg(a.r + c + R * sx);
    T ax, ay, az;
    direction<T>(__ldg(a.theta + c), __ldg(a.phi + c), ax, ay, az);
    T dpx = 0, dpy = 0, dpz = 0, drx = 0, dry = 0, drz = 0;
#pragma unroll
    for (int k = 1; k <= R; ++k) {
      const T w = a.c1[k - 1];
      dpx = fma(w, qp[R + k] - qp[R - k], dpx);
      drx = fma(w, qr[R + k] - qr[R - k], drx);
      dpy = fma(w, __ldg(a.p + c + k * sy) - __ldg(a.p + c - k * sy), dpy);
      dry = fma(w, __ldg(a.r + c + k * sy) - __ldg(a.r + c - k * sy), dry);
      dpz = fma(w, __ldg(a.p + c + k) - __ldg(a.p + c - k), dpz);
      drz = fma(w, __ldg(a.r + c + k) - __ldg(a.r + c - k), drz);
    }
    const T bx = ax * a.invh[0], by = ay * a.invh[1], bz = az * a.invh[2];
    a.gp[c] = fma(bx, dpx, fma(by, dpy, bz * dpz));
    a.gr[c] = fma(bx, drx, fma(by, dry, bz * drz));
  }
}

template <typename T, int SO>
__global__ void __launch_bounds__(BZ *BYT) tti_outer(const TtiArgs<T> a) {
  constexpr int R = SO / 4 > 0 ? SO / 4 : 1;
  constexpr int H = SO / 2;
  constexpr int QG = 2 * R + 1, QP = 2 * H + 1;
  const int z = a.lo[2] + blockIdx.x * BZ + threadIdx.x;
  const int y = a.lo[1] + blockIdx.y * BYT + threadIdx.y;
  const int xb = a.lo[0] + blockIdx.z * XCH;
  const int xe = min(xb + XCH, a.hi[0] + 1);
  if (z > a.hi[2] || y > a.hi[1]) return;
  const int64_t sx = a.E1 * a.E2, sy = a.E2;
  const int64_t col = (int64_t)(y + a.H) * sy + (z + a.H);
  T qp[QP], qg[QG], qh[QG];
#pragma unroll
  for (int i = 0; i < QP - 1; ++i) qp[i + 1] = __ldg(a.p + (int64_t)(xb - H + i + a.H) * sx + col);
#pragma unroll
  for (int i = 0; i < QG - 1; ++i) {
    const int64_t c = (int64_t)(xb - R + i + a.H) * sx + col;
    qg[i + 1] = __ldg(a.gp + c);
    qh[i + 1] = __ldg(a.gr + c);
  }
  for (int x = xb; x < xe; ++x) {
    const int64_t c = (int64_t)(x + a.H) * sx + col;
#pragma unroll
    for (int i = 0; i < QP - 1; ++i) qp[i] = qp[i + 1];
    qp[QP - 1] = __ldg(a.p + c + H * sx);
#pragma unroll
    for (int i = 0; i < QG - 1; ++i) {
      qg[i] = qg[i + 1];
      qh[i] = qh[i + 1];
    }
    qg[QG - 1] = __ldg(a.gp + c + R * sx);
    qh[QG - 1] = __ldg(a.gr + c + R * sx);
    T ax, ay, az;
    direction<T>(__ldg(a.theta + c), __ldg(a.phi + c), ax, ay, az);
    T hpx = 0, hpy = 0, hpz = 0, hrx = 0, hry = 0, hrz = 0;
#pragma unroll
    for (int k = 1; k <= R; ++k) {
      const T w = a.c1[k - 1];
      hpx = fma(w, qg[R + k] - qg[R - k], hpx);
      hrx = fma(w, qh[R + k] - qh[R - k], hrx);
      hpy = fma(w, __ldg(a.gp + c + k * sy) - __ldg(a.gp + c - k * sy), hpy);
      hry = fma(w, __ldg(a.gr + c + k * sy) - __ldg(a.gr + c - k * sy), hry);
      hpz = fma(w, __ldg(a.gp + c + k) - __ldg(a.gp + c - k), hpz);
      hrz = fma(w, __ldg(a.gr + c + k) - __ldg(a.gr + c - k), hrz);
    }
    const T bx = ax * a.invh[0], by = ay * a.invh[1], bz = az * a.invh[2];
    const T hzp = fma(bx, hpx, fma(by, hpy, bz * hpz));
    const T hzr = fma(bx, hrx, fma(by, hry, bz * hrz));
    const T p0 = qp[H];
    T lx = a.c2[0] * p0, ly = a.c2[0] * p0, lz = a.c2[0] * p0;
#pragma unroll
    for (int k = 1; k <= H; ++k) {
      const T w = a.c2[k];
      lx = fma(w, qp[H + k] + qp[H - k], lx);
      ly = fma(w, __ldg(a.p + c + k * sy) + __ldg(a.p + c - k * sy), ly);
      lz = fma(w, __ldg(a.p + c + k) + __ldg(a.p + c - k), lz);
    }
    const T lap = fma(lx, a.invh2[0], fma(ly, a.invh2[1], lz * a.invh2[2]));
    const T hxy = lap - hzp;
    const T e2 = 1 + 2 * __ldg(a.eps + c);
    const T sd = sqrt(1 + 2 * __ldg(a.delta + c));
    const T mm = __ldg(a.m + c), dd = __ldg(a.damp + c);
    const T am = mm * a.dt2inv, ad = dd * a.dtinv2;
    const T inv = 1 / (am + ad);
    const T pm = __ldg(a.pm + c), rm = __ldg(a.rm + c), r0 = __ldg(a.r + c);
    const T rhs_p = fma(e2, hxy, sd * hzr);
    const T rhs_r = fma(sd, hxy, hzr);
    a.pn[c] = (fma(am, 2 * p0 - pm, fma(ad, pm, rhs_p))) * inv;
    a.rn[c] = (fma(am, 2 * r0 - rm, fma(ad, rm, rhs_r))) * inv;
  }
}

template <typename T, int SO> void launch_pair(const TtiArgs<T> &a, cudaStream_t st) {
  constexpr int R = SO / 4 > 0 ? SO / 4 : 1;
  const int n0 = a.hi[0] - a.lo[0] + 1, n1 = a.hi[1] - a.lo[1] + 1, n2 = a.hi[2] - a.lo[2] + 1;
  dim3 b(BZ, BYT, 1);
  dim3 gi((n2 + 2 * R + BZ - 1) / BZ, (n1 + 2 * R + BYT - 1) / BYT,
          (n0 + 2 * R + XCH - 1) / XCH);
  tti_inner<T, SO><<<gi, b, 0, st>>>(a);
  dim3 go((n2 + BZ - 1) / BZ, (n1 + BYT - 1) / BYT, (n0 + XCH - 1) / XCH);
  tti_outer<T, SO><<<go, b, 0, st>>>(a);
}

}  // namespace

int tti_fused_launch(const sc_plan *pl, const sc_dense &d, const FieldDev *fields, int t,
                     cudaStream_t st);
int tti_tma_launch(const sc_plan *pl, const sc_dense &d, const FieldDev *fields, int t,
                   cudaStream_t st, int x_lo = INT_MIN, int x_hi = INT_MIN);

// host entry: fields per sc_dense.tti_fields order
// (p, r, m, damp, epsilon, delta, theta, phi); scratch g_p, g_r
template <typename T>
int tti_launch(const sc_plan *pl, const sc_dense &d, const FieldDev *fields, int t,
               cudaStream_t st) {
  const FieldDev &fp = fields[d.tti_fields[0]], &fr = fields[d.tti_fields[1]];
  TtiArgs<T> a;
  const int64_t plane = fp.ext[1] * fp.ext[2] * fp.ext[3];
  auto slot = [&](const FieldDev &f, int tt) { return sc_slot(tt, f.nslots); };
  const T *P = reinterpret_cast<const T *>(fp.data);
  const T *Rr = reinterpret_cast<const T *>(fr.data);
  a.p = P + slot(fp, t) * plane;
  a.pm = P + slot(fp, t - 1) * plane;
  a.pn = const_cast<T *>(P) + slot(fp, t + 1) * plane;
  a.r = Rr + slot(fr, t) * plane;
  a.rm = Rr + slot(fr, t - 1) * plane;
  a.rn = const_cast<T *>(Rr) + slot(fr, t + 1) * plane;
  const T **dst[6] = {&a.m, &a.damp, &a.eps, &a.delta, &a.theta, &a.phi};
  for (int i = 0; i < 6; ++i)
    *dst[i] = reinterpret_cast<const T *>(fields[d.tti_fields[2 + i]].data);
  a.gp = reinterpret_cast<T *>(d.scratch[0]);
  a.gr = reinterpret_cast<T *>(d.scratch[1]);
  for (int k = 0; k < 3; ++k) {
    a.lo[k] = pl->lo[k];
    a.hi[k] = pl->hi[k];
  }
  a.E1 = fp.ext[2];
  a.E2 = fp.ext[3];
  a.H = d.so / 2;
  const double *kc = d.fast_consts;  // invh[3], invh2[3], dt2inv, dtinv2, c1[5], c2[9]
  for (int k = 0; k < 3; ++k) {
    a.invh[k] = (T)kc[k];
    a.invh2[k] = (T)kc[3 + k];
  }
  a.dt2inv = (T)kc[6];
  a.dtinv2 = (T)kc[7];
  for (int k = 0; k < 5; ++k) a.c1[k] = (T)kc[8 + k];
  for (int k = 0; k < 9; ++k) a.c2[k] = (T)kc[13 + k];
  // the single-pass kernel is opt-in: it moves 48 B/pt instead of ~80 but
  // is still slower than the two-pass pair (profiles/r01_tti_fused.md)
  if (sizeof(T) == 4 && getenv("SC_TTI_FUSED")) {
    const int rc = tti_fused_launch(pl, d, fields, t, st);
    if (rc < 0) return -1;
    if (rc == 0) return 0;
  }
  if (sizeof(T) == 4 && !getenv("SC_TTI_PLAIN")) {
    const int rc = tti_tma_launch(pl, d, fields, t, st);
    if (rc < 0) return -1;
    if (rc == 0) return 0;
  }
  switch (d.so) {
    case 4: launch_pair<T, 4>(a, st); break;
    case 8: launch_pair<T, 8>(a, st); break;
    case 12: launch_pair<T, 12>(a, st); break;
    case 16: launch_pair<T, 16>(a, st); break;
    default:
      sc_set_error("no TTI kernel for space order %d", d.so);
      return -1;
  }
  SC_CUDA(cudaGetLastError());
  return 0;
}

template int tti_launch<float>(const sc_plan *, const sc_dense &, const FieldDev *, int, cudaStream_t);
template int tti_launch<double>(const sc_plan *, const sc_dense &, const FieldDev *, int, cudaStream_t);

// ---------------------------------------------------------------------------
// Single-pass streaming TTI kernel (f32). One CTA owns a TY x TZ tile of
// (y, z) and walks a chunk of x planes; a producer warp streams p/r planes
// (tile + so/2 halo) into a ring, theta/phi planes widened by the outer
// radius R = so/4, and the per-point aux tiles (p-, r-, m, damp, eps, delta,
// theta, phi) with TMA. Per load plane j the consumer warps
//   A) compute g_p, g_r = a.grad_R(p, r) on the plane x0 + j - 3R over the
//      tile widened by R (shared-memory g ring, 2R+1 planes), and
//   B) finish the output plane x0 + j - 4R: lap_so p (x neighbours from a
//      per-thread register queue of 2H+1 values, y/z from the p ring), the
//      outer rotated derivatives of g_p, g_r from the g ring, couplings,
//      damping and both updates, written straight to HBM.
// The rotated temporaries never leave shared memory (48 B/pt compulsory).

namespace {

constexpr int FTZ = 32, FBY = 8;  // tile: 8 rows (one per consumer warp) x 32
constexpr int FPF = 2;

template <int SO> struct FGeo {
  static constexpr int H = SO / 2, R = SO / 4;
  static constexpr int TY = FBY;
  static constexpr int WP = ((FTZ + 2 * H + 7) / 8) * 8;          // p/r plane row
  static constexpr int PR_ROWS = TY + 2 * H;
  static constexpr int PLANE = WP * PR_ROWS;
  static constexpr int PLANE_PAD = ((PLANE * 4 + 127) / 128) * 128 / 4;
  static constexpr int DPR = 2 * R + 1 + FPF;                       // p/r ring depth
  static constexpr int EOFF = R % 4;                                // theta/phi ext alignment
  static constexpr int WE = ((FTZ + 2 * R + EOFF + 7) / 8) * 8;
  static constexpr int E_ROWS = TY + 2 * R;
  static constexpr int EPLANE = ((WE * E_ROWS * 4 + 127) / 128) * 128 / 4;
  static constexpr int DTE = 1 + FPF;
  static constexpr int GW = FTZ + 2 * R;                            // g plane (dense)
  static constexpr int GPLANE = ((GW * E_ROWS * 4 + 127) / 128) * 128 / 4;
  static constexpr int DG = 2 * R + 1;
  static constexpr int AOFF = H % 4;
  static constexpr int WA = ((FTZ + AOFF + 7) / 8) * 8;
  static constexpr int ATILE = WA * TY;
  static constexpr int NAUX = 8;  // p-, r-, m, damp, eps, delta, theta, phi
  static constexpr int DA = 1 + FPF;
  static constexpr size_t SMEM = (size_t)4 * (2 * DPR * PLANE_PAD + 2 * DTE * EPLANE +
                                              2 * DG * GPLANE + DA * NAUX * ATILE) +
                                 8 * 2 * (DPR + DTE + DA);
};

struct FusedParams {
  int lo[3], n[3];
  int64_t ext[3];   // storage extents x, y, z
  float *pn, *rn;   // next slots (base of slot)
  int cur, prev;
  int xchunk;
  float invh[3], invh2[3], dt2inv, dtinv2;
  float c1[4], c2[9];
};

struct FusedMaps {
  CUtensorMap p_h, r_h, p_i, r_i, th_e, ph_e, th_i, ph_i, m, damp, eps, delta;
};

__device__ __forceinline__ void dir3(float th, float ph, float &ax, float &ay, float &az) {
  // MUFU sin/cos: |err| < 2^-21 on the angle ranges of the model
  // (theta, phi in [0, pi/2]); the fp32 parity bar is 1e-5 rel-L2
  float st, ct, sp, cp;
  __sincosf(th, &st, &ct);
  __sincosf(ph, &sp, &cp);
  ax = st * cp;
  ay = st * sp;
  az = ct;
}

template <int SO>
__global__ void __launch_bounds__(FTZ *(FBY + 1), 1)
    tti_fused(const __grid_constant__ FusedMaps M, const FusedParams P) {
  using G = FGeo<SO>;
  constexpr int H = G::H, R = G::R, TY = G::TY;
  extern __shared__ __align__(128) unsigned char smem_raw[];
  float *pring = reinterpret_cast<float *>(smem_raw);
  float *rring = pring + G::DPR * G::PLANE_PAD;
  float *tring = rring + G::DPR * G::PLANE_PAD;   // theta ext
  float *fring = tring + G::DTE * G::EPLANE;      // phi ext
  float *gp = fring + G::DTE * G::EPLANE;
  float *gr = gp + G::DG * G::GPLANE;
  float *aux = gr + G::DG * G::GPLANE;
  uint64_t *full_pr = reinterpret_cast<uint64_t *>(aux + G::DA * G::NAUX * G::ATILE);
  uint64_t *empty_pr = full_pr + G::DPR;
  uint64_t *full_te = empty_pr + G::DPR;
  uint64_t *empty_te = full_te + G::DTE;
  uint64_t *full_a = empty_te + G::DTE;
  uint64_t *empty_a = full_a + G::DA;

  const int tz = threadIdx.x, ty = threadIdx.y;
  const int z0 = P.lo[2] + blockIdx.x * FTZ;
  const int y0 = P.lo[1] + blockIdx.y * TY;
  const int xs = blockIdx.z * P.xchunk;
  const int XC = min(P.xchunk, P.n[0] - xs);
  const int x0 = P.lo[0] + xs;
  const int total = XC + 2 * H;  // load j <-> loop x = x0 + j - H
  const int Xs = (int)P.ext[0];

  if (ty == 0 && tz == 0) {
    for (int i = 0; i < G::DPR; ++i) {
      mbar_init(full_pr + i, 1);
      mbar_init(empty_pr + i, FBY);
    }
    for (int i = 0; i < G::DTE; ++i) {
      mbar_init(full_te + i, 1);
      mbar_init(empty_te + i, FBY);
    }
    for (int i = 0; i < G::DA; ++i) {
      mbar_init(full_a + i, 1);
      mbar_init(empty_a + i, FBY);
    }
    fence_barrier_init();
  }
  __syncthreads();

  if (ty == FBY) {  // ------------------------------ producer warp
    if (tz != 0) return;
    // per load plane j, in consumption order: p/r plane j, theta/phi ext
    // plane of g (j - 3R), aux plane of the output (j - 4R)
    for (int j = 0; j < total; ++j) {
      {
        const int s = j % G::DPR;
        if (j >= G::DPR) mbar_wait(empty_pr + s, ((j / G::DPR) - 1) & 1);
        mbar_expect_tx(full_pr + s, 2 * G::PLANE * 4);
        const int row = x0 + j;  // storage x of loop x0 + j - H
        tma_load_3d(pring + s * G::PLANE_PAD, &M.p_h, full_pr + s, z0, y0, P.cur * Xs + row);
        tma_load_3d(rring + s * G::PLANE_PAD, &M.r_h, full_pr + s, z0, y0, P.cur * Xs + row);
      }
      const int e = j - 2 * R;  // theta/phi ext index (g plane x0 + j - 3R)
      if (e >= 0 && e < XC + 2 * R) {
        const int s = e % G::DTE;
        if (e >= G::DTE) mbar_wait(empty_te + s, ((e / G::DTE) - 1) & 1);
        mbar_expect_tx(full_te + s, 2 * G::E_ROWS * G::WE * 4);
        const int xst = x0 + e - R + H;  // storage x of loop x0 + e - R
        const int zs = z0 + H - R - G::EOFF, ys = y0 + H - R;
        tma_load_3d(tring + s * G::EPLANE, &M.th_e, full_te + s, zs, ys, xst);
        tma_load_3d(fring + s * G::EPLANE, &M.ph_e, full_te + s, zs, ys, xst);
      }
      const int k = j - 4 * R;  // output plane x0 + k
      if (k >= 0 && k < XC) {
        const int s = k % G::DA;
        if (k >= G::DA) mbar_wait(empty_a + s, ((k / G::DA) - 1) & 1);
        mbar_expect_tx(full_a + s, G::NAUX * G::ATILE * 4);
        float *dst = aux + s * G::NAUX * G::ATILE;
        const int xst = x0 + k + H, zs = z0 + H - G::AOFF, ys = y0 + H;
        tma_load_3d(dst + 0 * G::ATILE, &M.p_i, full_a + s, zs, ys, P.prev * Xs + xst);
        tma_load_3d(dst + 1 * G::ATILE, &M.r_i, full_a + s, zs, ys, P.prev * Xs + xst);
        tma_load_3d(dst + 2 * G::ATILE, &M.m, full_a + s, zs, ys, xst);
        tma_load_3d(dst + 3 * G::ATILE, &M.damp, full_a + s, zs, ys, xst);
        tma_load_3d(dst + 4 * G::ATILE, &M.eps, full_a + s, zs, ys, xst);
        tma_load_3d(dst + 5 * G::ATILE, &M.delta, full_a + s, zs, ys, xst);
        tma_load_3d(dst + 6 * G::ATILE, &M.th_i, full_a + s, zs, ys, xst);
        tma_load_3d(dst + 7 * G::ATILE, &M.ph_i, full_a + s, zs, ys, xst);
      }
    }
    return;
  }

  // ------------------------------------------------ consumer warps
  const int lane = tz, tid = ty * FTZ + tz;
  float q[2 * H + 1];  // p along x at the thread's point (load planes j-2H..j)
#pragma unroll
  for (int i = 0; i <= 2 * H; ++i) q[i] = 0.f;
  const int y = y0 + ty, z = z0 + tz;
  const bool active = y < P.lo[1] + P.n[1] && z < P.lo[2] + P.n[2];
  const int64_t plane = P.ext[1] * P.ext[2];
  const int64_t own = (int64_t)(y + H) * P.ext[2] + (z + H);
  const int crow = (ty + H) * G::WP + tz + H;  // thread's point in a p/r plane
  const int cg = (ty + R) * G::GW + tz + R;    // thread's point in a g plane
  constexpr int NT = FTZ * FBY;
  constexpr int NE = G::E_ROWS * G::GW;        // widened tile points
  constexpr int NEP = (NE + NT - 1) / NT;      // per thread
  // the widened-tile points this thread computes g at (fixed for the run)
  int eo_p[NEP], eo_e[NEP], eo_g[NEP];
#pragma unroll
  for (int n = 0; n < NEP; ++n) {
    const int i = tid + n * NT;
    const int ey = i / G::GW, ez = i % G::GW;
    eo_p[n] = (ey + R) * G::WP + ez + R;
    eo_e[n] = ey * G::WE + ez + G::EOFF;
    eo_g[n] = i < NE ? i : -1;
  }
  float c1[R], c2[H + 1];
#pragma unroll
  for (int k = 0; k < R; ++k) c1[k] = P.c1[k];
#pragma unroll
  for (int k = 0; k <= H; ++k) c2[k] = P.c2[k];
  auto wrap = [](int v, int n) { return v >= n ? v - n : (v < 0 ? v + n : v); };

  int sj = 0, phj = 0;       // ring slot / parity of load j
  int se = 0;                // g ring slot of g index e = j - 2R (valid e >= 0)
  int ste = 0, phte = 0;     // theta/phi ext ring
  int sa = 0, pha = 0;       // aux ring
#pragma unroll 1
  for (int j = 0; j < total; ++j) {
    mbar_wait(full_pr + sj, phj);
#pragma unroll
    for (int i = 0; i < 2 * H; ++i) q[i] = q[i + 1];
    q[2 * H] = pring[sj * G::PLANE_PAD + crow];
    named_bar_sync(1, NT);  // the g slot about to be written is no longer read
    // ---- A: g on the widened tile of loop plane x0 + j - 3R ----
    const int e = j - 2 * R;
    if (e >= 0 && e < XC + 2 * R) {
      mbar_wait(full_te + ste, phte);
      const float *th = tring + ste * G::EPLANE, *ph = fring + ste * G::EPLANE;
      float *gpo = gp + se * G::GPLANE, *gro = gr + se * G::GPLANE;
      const float *pp[2 * R + 1], *rp[2 * R + 1];  // p/r planes j-2R .. j
#pragma unroll
      for (int d = 0; d <= 2 * R; ++d) {
        const int sl = wrap(sj - 2 * R + d, G::DPR);
        pp[d] = pring + sl * G::PLANE_PAD;
        rp[d] = rring + sl * G::PLANE_PAD;
      }
#pragma unroll
      for (int n = 0; n < NEP; ++n) {
        if (eo_g[n] < 0) continue;
        const int c = eo_p[n];
        float ax, ay, az;
        dir3(th[eo_e[n]], ph[eo_e[n]], ax, ay, az);
        float dpx = 0.f, dpy = 0.f, dpz = 0.f, drx = 0.f, dry = 0.f, drz = 0.f;
        const float *pc = pp[R], *rc = rp[R];
#pragma unroll
        for (int k = 1; k <= R; ++k) {
          const float w = c1[k - 1];
          dpx = fmaf(w, pp[R + k][c] - pp[R - k][c], dpx);
          drx = fmaf(w, rp[R + k][c] - rp[R - k][c], drx);
          dpy = fmaf(w, pc[c + k * G::WP] - pc[c - k * G::WP], dpy);
          dry = fmaf(w, rc[c + k * G::WP] - rc[c - k * G::WP], dry);
          dpz = fmaf(w, pc[c + k] - pc[c - k], dpz);
          drz = fmaf(w, rc[c + k] - rc[c - k], drz);
        }
        const float bx = ax * P.invh[0], by = ay * P.invh[1], bz = az * P.invh[2];
        gpo[eo_g[n]] = fmaf(bx, dpx, fmaf(by, dpy, bz * dpz));
        gro[eo_g[n]] = fmaf(bx, drx, fmaf(by, dry, bz * drz));
      }
      __syncwarp();
      if (lane == 0) mbar_arrive(empty_te + ste);
      if (++ste == G::DTE) { ste = 0; phte ^= 1; }
    }
    named_bar_sync(1, NT);  // g plane complete
    // ---- B: output plane x0 + k, k = j - 4R ----
    const int k = j - 4 * R;
    const int so_ = wrap(sj - 2 * R, G::DPR);  // p/r slot of load j - 2R
    if (k >= 0 && k < XC) {
      mbar_wait(full_a + sa, pha);
      const float *ax_ = aux + sa * G::NAUX * G::ATILE;
      const int ai = ty * G::WA + tz + G::AOFF;
      float ax, ay, az;
      dir3(ax_[6 * G::ATILE + ai], ax_[7 * G::ATILE + ai], ax, ay, az);
      // outer rotated derivatives: g indices k .. k + 2R = e - 2R .. e
      float hpx = 0.f, hpy = 0.f, hpz = 0.f, hrx = 0.f, hry = 0.f, hrz = 0.f;
      const float *gq[2 * R + 1], *rq[2 * R + 1];
#pragma unroll
      for (int d = 0; d <= 2 * R; ++d) {
        const int sl = wrap(se - 2 * R + d, G::DG);
        gq[d] = gp + sl * G::GPLANE;
        rq[d] = gr + sl * G::GPLANE;
      }
      const float *gpc = gq[R], *grc = rq[R];
#pragma unroll
      for (int kk = 1; kk <= R; ++kk) {
        const float w = c1[kk - 1];
        hpx = fmaf(w, gq[R + kk][cg] - gq[R - kk][cg], hpx);
        hrx = fmaf(w, rq[R + kk][cg] - rq[R - kk][cg], hrx);
        hpy = fmaf(w, gpc[cg + kk * G::GW] - gpc[cg - kk * G::GW], hpy);
        hry = fmaf(w, grc[cg + kk * G::GW] - grc[cg - kk * G::GW], hry);
        hpz = fmaf(w, gpc[cg + kk] - gpc[cg - kk], hpz);
        hrz = fmaf(w, grc[cg + kk] - grc[cg - kk], hrz);
      }
      const float bx = ax * P.invh[0], by = ay * P.invh[1], bz = az * P.invh[2];
      const float hzp = fmaf(bx, hpx, fmaf(by, hpy, bz * hpz));
      const float hzr = fmaf(bx, hrx, fmaf(by, hry, bz * hrz));
      // Laplacian of p at the output plane
      const float *pc = pring + so_ * G::PLANE_PAD;
      const float p0 = q[H];
      float lx = c2[0] * p0, ly = c2[0] * p0, lz = c2[0] * p0;
#pragma unroll
      for (int kk = 1; kk <= H; ++kk) {
        const float w = c2[kk];
        lx = fmaf(w, q[H + kk] + q[H - kk], lx);
        ly = fmaf(w, pc[crow + kk * G::WP] + pc[crow - kk * G::WP], ly);
        lz = fmaf(w, pc[crow + kk] + pc[crow - kk], lz);
      }
      const float lap = fmaf(lx, P.invh2[0], fmaf(ly, P.invh2[1], lz * P.invh2[2]));
      const float hxy = lap - hzp;
      const float e2 = 1.f + 2.f * ax_[4 * G::ATILE + ai];
      const float sd = sqrtf(1.f + 2.f * ax_[5 * G::ATILE + ai]);
      const float mm = ax_[2 * G::ATILE + ai], dd = ax_[3 * G::ATILE + ai];
      const float am = mm * P.dt2inv, ad = dd * P.dtinv2;
      const float inv = 1.f / (am + ad);
      const float pm = ax_[0 * G::ATILE + ai], rm = ax_[1 * G::ATILE + ai];
      const float r0 = rring[so_ * G::PLANE_PAD + crow];
      const float rhs_p = fmaf(e2, hxy, sd * hzr);
      const float rhs_r = fmaf(sd, hxy, hzr);
      if (active) {
        const int64_t o = (int64_t)(x0 + k + H) * plane + own;
        P.pn[o] = fmaf(am, 2.f * p0 - pm, fmaf(ad, pm, rhs_p)) * inv;
        P.rn[o] = fmaf(am, 2.f * r0 - rm, fmaf(ad, rm, rhs_r)) * inv;
      }
      __syncwarp();
      if (lane == 0) {
        mbar_arrive(empty_a + sa);
        mbar_arrive(empty_pr + so_);  // p/r plane j - 2R: last use
      }
      if (++sa == G::DA) { sa = 0; pha ^= 1; }
    } else if (j >= 2 * R) {
      // planes outside the output range still release their p/r slot
      __syncwarp();
      if (lane == 0) mbar_arrive(empty_pr + so_);
    }
    if (e >= 0 && ++se == G::DG) se = 0;
    if (++sj == G::DPR) { sj = 0; phj ^= 1; }
  }
}

template <int SO> const void *fused_ptr() { return reinterpret_cast<const void *>(&tti_fused<SO>); }

const void *pick_fused(int so, size_t *smem) {
  switch (so) {
    case 4: *smem = FGeo<4>::SMEM; return fused_ptr<4>();
    case 8: *smem = FGeo<8>::SMEM; return fused_ptr<8>();
    case 12: *smem = FGeo<12>::SMEM; return fused_ptr<12>();
    case 16: *smem = FGeo<16>::SMEM; return fused_ptr<16>();
  }
  return nullptr;
}

}  // namespace

// host launch of the fused kernel (f32); returns 1 when not applicable
int tti_fused_launch(const sc_plan *pl, const sc_dense &d, const FieldDev *fields, int t,
                     cudaStream_t st) {
  const int so = d.so, H = so / 2, R = so / 4;
  const FieldDev &fp = fields[d.tti_fields[0]], &fr = fields[d.tti_fields[1]];
  if ((fp.ext[3] * 4) % 16 != 0) return 1;
  size_t smem = 0;
  const void *kp = pick_fused(so, &smem);
  if (!kp || smem > 227 * 1024) return 1;
  FusedMaps M;
  FusedParams P;
  const uint64_t Z = fp.ext[3], Y = fp.ext[2], Xs = fp.ext[1];
  uint64_t strides[2] = {Z * 4, Z * Y * 4};
  uint64_t dims_t[3] = {Z, Y, Xs * 3};
  uint64_t dims_f[3] = {Z, Y, Xs};
  const uint32_t WP = ((32 + 2 * H + 7) / 8) * 8;
  const uint32_t EOFF = R % 4, WE = ((32 + 2 * R + EOFF + 7) / 8) * 8;
  const uint32_t AOFF = H % 4, WA = ((32 + AOFF + 7) / 8) * 8;
  uint32_t box_h[3] = {WP, (uint32_t)(FBY + 2 * H), 1};
  uint32_t box_e[3] = {WE, (uint32_t)(FBY + 2 * R), 1};
  uint32_t box_i[3] = {WA, (uint32_t)FBY, 1};
  auto F = [&](int i) { return fields[d.tti_fields[i]].data; };
  if (sc_encode_tmap(&M.p_h, F(0), 4, dims_t, strides, box_h) ||
      sc_encode_tmap(&M.r_h, F(1), 4, dims_t, strides, box_h) ||
      sc_encode_tmap(&M.p_i, F(0), 4, dims_t, strides, box_i) ||
      sc_encode_tmap(&M.r_i, F(1), 4, dims_t, strides, box_i) ||
      sc_encode_tmap(&M.m, F(2), 4, dims_f, strides, box_i) ||
      sc_encode_tmap(&M.damp, F(3), 4, dims_f, strides, box_i) ||
      sc_encode_tmap(&M.eps, F(4), 4, dims_f, strides, box_i) ||
      sc_encode_tmap(&M.delta, F(5), 4, dims_f, strides, box_i) ||
      sc_encode_tmap(&M.th_e, F(6), 4, dims_f, strides, box_e) ||
      sc_encode_tmap(&M.ph_e, F(7), 4, dims_f, strides, box_e) ||
      sc_encode_tmap(&M.th_i, F(6), 4, dims_f, strides, box_i) ||
      sc_encode_tmap(&M.ph_i, F(7), 4, dims_f, strides, box_i))
    return -1;
  for (int k = 0; k < 3; ++k) {
    P.lo[k] = pl->lo[k];
    P.n[k] = pl->hi[k] - pl->lo[k] + 1;
    P.ext[k] = fp.ext[1 + k];
  }
  const int64_t slot = fp.ext[1] * fp.ext[2] * fp.ext[3];
  P.pn = reinterpret_cast<float *>(fp.data) + sc_slot(t + 1, 3) * slot;
  P.rn = reinterpret_cast<float *>(fr.data) + sc_slot(t + 1, 3) * slot;
  P.cur = sc_slot(t, 3);
  P.prev = sc_slot(t - 1, 3);
  const double *kc = d.fast_consts;
  for (int k = 0; k < 3; ++k) {
    P.invh[k] = (float)kc[k];
    P.invh2[k] = (float)kc[3 + k];
  }
  P.dt2inv = (float)kc[6];
  P.dtinv2 = (float)kc[7];
  for (int k = 0; k < 4; ++k) P.c1[k] = (float)kc[8 + k];
  for (int k = 0; k < 9; ++k) P.c2[k] = (float)kc[13 + k];
  static int sms = 0;
  if (!sms) {
    int dev = 0;
    SC_CUDA(cudaGetDevice(&dev));
    SC_CUDA(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev));
  }
  SC_CUDA(cudaFuncSetAttribute(kp, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
  const int64_t tiles = sc_ceil_div(P.n[1], FBY) * sc_ceil_div(P.n[2], FTZ);
  int64_t want = sc_ceil_div((int64_t)6 * sms, tiles);
  int64_t maxch = std::max<int64_t>(1, P.n[0] / std::max(8, 8 * R));
  int64_t nch = std::max<int64_t>(1, std::min(want, maxch));
  P.xchunk = (int)sc_ceil_div(P.n[0], nch);
  nch = sc_ceil_div(P.n[0], P.xchunk);
  dim3 grid((unsigned)sc_ceil_div(P.n[2], FTZ), (unsigned)sc_ceil_div(P.n[1], FBY), (unsigned)nch);
  dim3 block(FTZ, FBY + 1, 1);
  void *args[] = {(void *)&M, (void *)&P};
  SC_CUDA(cudaLaunchKernel(kp, grid, block, args, smem, st));
  return 0;
}

// ---------------------------------------------------------------------------
// TMA-streamed two-pass TTI (default f32 path). Same arithmetic as the
// two-pass pair above; both passes use the K1 pipeline: a producer warp
// streams planes with TMA into shared-memory rings (full/empty mbarriers),
// 8 consumer warps each own 2 y rows of one z column and keep register
// queues along x.
//   pass 1 (tti_g_tma):   g_p, g_r over the loop box widened by R
//   pass 2 (tti_upd_tma): lap p, outer rotated derivatives, both updates

namespace {

constexpr int SZ = 32, SBY = 8, SRY = 2, STY = SBY * SRY, SPF = 3;
// prefetch depth of the pass-2 rings: so 16 holds two planes ahead so its
// rings fit the 227 KB shared-memory budget
__host__ __device__ constexpr int spf_u(int so) { return so >= 16 ? 2 : SPF; }
// pass 2: rows per thread and consumer warps (same STY-row tile)
constexpr int USRY = 1, UBY = STY / USRY;

template <int NF, int HALO> struct Ring {
  // NF fields, planes of (STY + 2 HALO) rows x W (32 + 2 HALO + 3 rounded
  // up to 8 floats: room for a runtime 16-byte alignment shift)
  static constexpr int W = ((SZ + 2 * HALO + 3 + 7) / 8) * 8;
  static constexpr int ROWS = STY + 2 * HALO;
  static constexpr int PLANE = W * ROWS;
  static constexpr int PAD = ((PLANE * 4 + 127) / 128) * 128 / 4;
};

template <int NA> struct AuxTile {
  static constexpr int W = ((SZ + 3 + 7) / 8) * 8;
  static constexpr int TILE = W * STY;
};

struct StreamCommon {
  int lo[3], n[3];     // box (loop coords) this kernel covers
  int64_t ext[3];      // storage extents x, y, z
  int xchunk;
  int H;
  // tail split (1D grid, pass 2): the first `nwhole` CTAs sweep all of x on
  // tiles 0 .. nwhole-1; every later tile is cut into `tailq` x chunks, so
  // the last, partly filled wave of whole sweeps becomes several short full
  // ones. tailq = 0: the (z tile, y tile, x chunk) grid.
  int nwhole, tailq, ntz;
};

struct GParams {
  StreamCommon c;
  float *gp, *gr;      // outputs (field layout)
  int cur;
  float invh[3], c1[4];
};

struct UParams {
  StreamCommon c;
  float *pn, *rn;
  int cur, prev;
  float invh[3], invh2[3], dt2inv, dtinv2, c1[4], c2[9];
};

struct GMaps { CUtensorMap p, r, th, ph; };
struct UMaps { CUtensorMap p, gp, gr, r, pm, rm, m, damp, eps, delta, th, ph; };

__device__ __forceinline__ int wrapi(int v, int n) { return v >= n ? v - n : (v < 0 ? v + n : v); }

// pass 1 ------------------------------------------------------------------
template <int SO>
__global__ void __launch_bounds__(SZ *(SBY + 1), 1) tti_g_tma(const __grid_constant__ GMaps M,
                                                                const GParams P) {
  constexpr int R = SO / 4, H = SO / 2, Q = 2 * R + 1;
  using RG = Ring<2, R>;
  using AX = AuxTile<2>;
  constexpr int DR = R + 1 + SPF, DA = 1 + SPF;
  extern __shared__ __align__(128) unsigned char smem_raw[];
  float *ring = reinterpret_cast<float *>(smem_raw);            // [DR][2][PAD]
  float *aux = ring + DR * 2 * RG::PAD;                          // [DA][2][TILE]
  uint64_t *full_r = reinterpret_cast<uint64_t *>(aux + DA * 2 * AX::TILE);
  uint64_t *empty_r = full_r + DR;
  uint64_t *full_a = empty_r + DR;
  uint64_t *empty_a = full_a + DA;

  const int tz = threadIdx.x, ty = threadIdx.y;
  const StreamCommon &C = P.c;
  const int z0 = C.lo[2] + blockIdx.x * SZ, y0 = C.lo[1] + blockIdx.y * STY;
  const int xs = blockIdx.z * C.xchunk;
  const int XC = min(C.xchunk, C.n[0] - xs);
  const int x0 = C.lo[0] + xs;  // first output (g) plane, loop coords
  const int total = XC + 2 * R; // load j <-> loop x0 + j - R
  // storage z of the box starts, shifted down to 16-byte boundaries
  const int zr = z0 + H - R, er = zr & 3;
  const int za = z0 + H, ea = za & 3;

  if (ty == 0 && tz == 0) {
    for (int i = 0; i < DR; ++i) { mbar_init(full_r + i, 1); mbar_init(empty_r + i, SBY); }
    for (int i = 0; i < DA; ++i) { mbar_init(full_a + i, 1); mbar_init(empty_a + i, SBY); }
    fence_barrier_init();
  }
  __syncthreads();
  if (ty == SBY) {
    if (tz != 0) return;
    const int Xs = (int)C.ext[0];
    for (int j = 0; j < total; ++j) {
      const int s = j % DR;
      if (j >= DR) mbar_wait(empty_r + s, ((j / DR) - 1) & 1);
      mbar_expect_tx(full_r + s, 2 * RG::PLANE * 4);
      const int xst = x0 + j - R + H;
      float *dst = ring + s * 2 * RG::PAD;
      tma_load_3d(dst, &M.p, full_r + s, zr - er, y0 + H - R, P.cur * Xs + xst);
      tma_load_3d(dst + RG::PAD, &M.r, full_r + s, zr - er, y0 + H - R, P.cur * Xs + xst);
      const int k = j - 2 * R;
      if (k >= 0) {
        const int sa = k % DA;
        if (k >= DA) mbar_wait(empty_a + sa, ((k / DA) - 1) & 1);
        mbar_expect_tx(full_a + sa, 2 * AX::TILE * 4);
        float *ad = aux + sa * 2 * AX::TILE;
        const int xk = x0 + k + H;
        tma_load_3d(ad, &M.th, full_a + sa, za - ea, y0 + H, xk);
        tma_load_3d(ad + AX::TILE, &M.ph, full_a + sa, za - ea, y0 + H, xk);
      }
    }
    return;
  }
  const int lane = tz;
  float qp[SRY][Q], qr[SRY][Q];
#pragma unroll
  for (int r = 0; r < SRY; ++r) {
#pragma unroll
    for (int q = 0; q < Q; ++q) { qp[r][q] = 0.f; qr[r][q] = 0.f; }
  }
  const int row0 = ty * SRY + R;  // ring row of the thread's first point
  const int col = tz + R + er;
  const int z = z0 + tz, yb = y0 + ty * SRY;
  const bool zok = z < C.lo[2] + C.n[2];
  const int yend = C.lo[1] + C.n[1];
  const int64_t pl = C.ext[1] * C.ext[2];
  const int64_t own = (int64_t)(yb + H) * C.ext[2] + (z + H);
  float c1[R], ih[3];
#pragma unroll
  for (int k = 0; k < R; ++k) c1[k] = P.c1[k];
#pragma unroll
  for (int k = 0; k < 3; ++k) ih[k] = P.invh[k];
  int sj = 0, ph = 0, sa = 0, pa = 0;
#pragma unroll 1
  for (int j = 0; j < total; ++j) {
    mbar_wait(full_r + sj, ph);
    const float *pp = ring + sj * 2 * RG::PAD, *rr = pp + RG::PAD;
#pragma unroll
    for (int r = 0; r < SRY; ++r) {
#pragma unroll
      for (int i = 0; i < Q - 1; ++i) { qp[r][i] = qp[r][i + 1]; qr[r][i] = qr[r][i + 1]; }
      qp[r][Q - 1] = pp[(row0 + r) * RG::W + col];
      qr[r][Q - 1] = rr[(row0 + r) * RG::W + col];
    }
    const int k = j - 2 * R;
    const int sc = wrapi(sj - R, DR);  // ring slot of the centre plane j - R
    if (k >= 0) {
      mbar_wait(full_a + sa, pa);
      const float *cp = ring + sc * 2 * RG::PAD, *cr = cp + RG::PAD;
      const float *at = aux + sa * 2 * AX::TILE;
#pragma unroll
      for (int r = 0; r < SRY; ++r) {
        const int c = (row0 + r) * RG::W + col;
        const int ai = (ty * SRY + r) * AX::W + tz + ea;
        float ax, ay, az;
        dir3(at[ai], at[AX::TILE + ai], ax, ay, az);
        float dpx = 0.f, dpy = 0.f, dpz = 0.f, drx = 0.f, dry = 0.f, drz = 0.f;
#pragma unroll
        for (int kk = 1; kk <= R; ++kk) {
          const float w = c1[kk - 1];
          dpx = fmaf(w, qp[r][R + kk] - qp[r][R - kk], dpx);
          drx = fmaf(w, qr[r][R + kk] - qr[r][R - kk], drx);
          dpy = fmaf(w, cp[c + kk * RG::W] - cp[c - kk * RG::W], dpy);
          dry = fmaf(w, cr[c + kk * RG::W] - cr[c - kk * RG::W], dry);
          dpz = fmaf(w, cp[c + kk] - cp[c - kk], dpz);
          drz = fmaf(w, cr[c + kk] - cr[c - kk], drz);
        }
        const float bx = ax * ih[0], by = ay * ih[1], bz = az * ih[2];
        if (zok && yb + r < yend) {
          const int64_t o = (int64_t)(x0 + k + H) * pl + own + (int64_t)r * C.ext[2];
          P.gp[o] = fmaf(bx, dpx, fmaf(by, dpy, bz * dpz));
          P.gr[o] = fmaf(bx, drx, fmaf(by, dry, bz * drz));
        }
      }
      __syncwarp();
      if (lane == 0) {
        mbar_arrive(empty_a + sa);
        mbar_arrive(empty_r + sc);
      }
      if (++sa == DA) { sa = 0; pa ^= 1; }
    } else if (j >= R) {
      __syncwarp();
      if (lane == 0) mbar_arrive(empty_r + sc);
    }
    if (++sj == DR) { sj = 0; ph ^= 1; }
  }
}

// pass 1, x-blocked --------------------------------------------------------
// tti_g_tma with two x planes per ring slot (depth-2 TMA boxes) and two
// output planes per consumer iteration; 8 row-pair warps, 2 CTAs per SM.
template <int SO> struct G2Geo {
  static constexpr int R = SO / 4, H = SO / 2;
  static constexpr int W = ((SZ + 2 * R + 3 + 7) / 8) * 8;
  static constexpr int WA = ((SZ + 3 + 7) / 8) * 8;
  static constexpr int PLANE = W * (STY + 2 * R), PLANEA = WA * STY;
  static constexpr int rnd(int f) { return ((f * 4 + 127) / 128) * 128 / 4; }
  static constexpr int HALF = rnd(2 * PLANE);    // one field of a p/r pair
  static constexpr int SLOTA = rnd(2 * PLANEA);  // one field of an aux pair
  static constexpr int DRS = (R + 1) / 2 + 3, DA = 2;  // two pairs of p/r lookahead
  static constexpr size_t SMEM = (size_t)4 * (DRS * 2 * HALF + DA * 2 * SLOTA) + 16 * (DRS + DA);
};

struct GMaps2 { CUtensorMap p, r, th, ph; };

template <int SO>
__global__ void __launch_bounds__(SZ *(SBY + 1), 2) tti_g2_tma(const __grid_constant__ GMaps2 M,
                                                                 const GParams P) {
  using G = G2Geo<SO>;
  constexpr int R = G::R, H = G::H, Q = 2 * R + 2, DRS = G::DRS, DA = G::DA;
  extern __shared__ __align__(128) unsigned char smem_raw[];
  float *ring = reinterpret_cast<float *>(smem_raw);  // [DRS][2][HALF]
  float *aux = ring + DRS * 2 * G::HALF;              // [DA][2][SLOTA]
  uint64_t *full_r = reinterpret_cast<uint64_t *>(aux + DA * 2 * G::SLOTA);
  uint64_t *empty_r = full_r + DRS;
  uint64_t *full_a = empty_r + DRS;
  uint64_t *empty_a = full_a + DA;

  const int tz = threadIdx.x, ty = threadIdx.y;
  const StreamCommon &C = P.c;
  const int z0 = C.lo[2] + blockIdx.x * SZ, y0 = C.lo[1] + blockIdx.y * STY;
  const int xs = blockIdx.z * C.xchunk;
  const int XC = min(C.xchunk, C.n[0] - xs);
  const int x0 = C.lo[0] + xs;   // first output (g) plane, loop coords
  const int KP = (XC + 1) / 2, JT = KP + R;  // load j <-> loop x0 + j - R
  const int zr = z0 + H - R, er = zr & 3;
  const int za = z0 + H, ea = za & 3;

  if (ty == 0 && tz == 0) {
    for (int i = 0; i < DRS; ++i) { mbar_init(full_r + i, 1); mbar_init(empty_r + i, SBY); }
    for (int i = 0; i < DA; ++i) { mbar_init(full_a + i, 1); mbar_init(empty_a + i, SBY); }
    fence_barrier_init();
  }
  __syncthreads();
  if (ty == SBY) {
    if (tz != 0) return;
    const int Xs = (int)C.ext[0];
    for (int J = 0; J < JT; ++J) {
      const int s = J % DRS;
      if (J >= DRS) mbar_wait(empty_r + s, ((J / DRS) - 1) & 1);
      mbar_expect_tx(full_r + s, 4 * G::PLANE * 4);
      const int xst = x0 + 2 * J - R + H;
      float *dst = ring + s * 2 * G::HALF;
      tma_load_3d(dst, &M.p, full_r + s, zr - er, y0 + H - R, P.cur * Xs + xst);
      tma_load_3d(dst + G::HALF, &M.r, full_r + s, zr - er, y0 + H - R, P.cur * Xs + xst);
      const int K = J - R;
      if (K >= 0) {
        const int sa = K % DA;
        if (K >= DA) mbar_wait(empty_a + sa, ((K / DA) - 1) & 1);
        mbar_expect_tx(full_a + sa, 4 * G::PLANEA * 4);
        float *ad = aux + sa * 2 * G::SLOTA;
        const int xk = x0 + 2 * K + H;
        tma_load_3d(ad, &M.th, full_a + sa, za - ea, y0 + H, xk);
        tma_load_3d(ad + G::SLOTA, &M.ph, full_a + sa, za - ea, y0 + H, xk);
      }
    }
    return;
  }
  const int lane = tz;
  float qp[SRY][Q], qr[SRY][Q];
#pragma unroll
  for (int r = 0; r < SRY; ++r)
#pragma unroll
    for (int q = 0; q < Q; ++q) { qp[r][q] = 0.f; qr[r][q] = 0.f; }
  const int c0 = (ty * SRY + R) * G::W + tz + R + er;  // ring offset of the first row
  const int a0 = ty * SRY * G::WA + tz + ea;
  const int z = z0 + tz, yb = y0 + ty * SRY;
  const bool zok = z < C.lo[2] + C.n[2];
  const int yend = C.lo[1] + C.n[1];
  const int64_t pl = C.ext[1] * C.ext[2];
  const int64_t own = (int64_t)(yb + H) * C.ext[2] + (z + H);
  int sj = 0, ph = 0, sa = 0, pa = 0;
#pragma unroll 1
  for (int J = 0; J < JT; ++J) {
    mbar_wait(full_r + sj, ph);
    {
      const float *pp = ring + sj * 2 * G::HALF + c0;
#pragma unroll
      for (int r = 0; r < SRY; ++r) {
#pragma unroll
        for (int q = 0; q < Q - 2; ++q) { qp[r][q] = qp[r][q + 2]; qr[r][q] = qr[r][q + 2]; }
        qp[r][Q - 2] = pp[r * G::W];
        qp[r][Q - 1] = pp[r * G::W + G::PLANE];
        qr[r][Q - 2] = pp[G::HALF + r * G::W];
        qr[r][Q - 1] = pp[G::HALF + r * G::W + G::PLANE];
      }
    }
    const int K = J - R;
    if (K >= 0) {
      mbar_wait(full_a + sa, pa);
      const float *at = aux + sa * 2 * G::SLOTA + a0;
#pragma unroll
      for (int e = 0; e < 2; ++e) {
        // centre load 2K + R + e: pair K + (R + e) / 2 = J - (R - (R + e) / 2)
        const float *cp = ring + wrapi(sj - (R - (R + e) / 2), DRS) * 2 * G::HALF +
                          ((R + e) & 1) * G::PLANE + c0;
#pragma unroll
        for (int r = 0; r < SRY; ++r) {
          const float *c = cp + r * G::W;
          float ax, ay, az;
          dir3(at[e * G::PLANEA + r * G::WA], at[G::SLOTA + e * G::PLANEA + r * G::WA], ax, ay, az);
          float dpx = 0.f, dpy = 0.f, dpz = 0.f, drx = 0.f, dry = 0.f, drz = 0.f;
#pragma unroll
          for (int kk = 1; kk <= R; ++kk) {
            const float w = P.c1[kk - 1];
            dpx = fmaf(w, qp[r][e + R + kk] - qp[r][e + R - kk], dpx);
            drx = fmaf(w, qr[r][e + R + kk] - qr[r][e + R - kk], drx);
            dpy = fmaf(w, c[kk * G::W] - c[-kk * G::W], dpy);
            dry = fmaf(w, c[G::HALF + kk * G::W] - c[G::HALF - kk * G::W], dry);
            dpz = fmaf(w, c[kk] - c[-kk], dpz);
            drz = fmaf(w, c[G::HALF + kk] - c[G::HALF - kk], drz);
          }
          const float bx = ax * P.invh[0], by = ay * P.invh[1], bz = az * P.invh[2];
          if (zok && yb + r < yend && 2 * K + e < XC) {
            const int64_t o = (int64_t)(x0 + 2 * K + e + H) * pl + own + (int64_t)r * C.ext[2];
            P.gp[o] = fmaf(bx, dpx, fmaf(by, dpy, bz * dpz));
            P.gr[o] = fmaf(bx, drx, fmaf(by, dry, bz * drz));
          }
        }
      }
    }
    __syncwarp();
    if (lane == 0) {
      if (K >= 0) mbar_arrive(empty_a + sa);
      const int rel = J - R + R / 2;  // pair no longer needed as a y/z centre
      if (rel >= 0) mbar_arrive(empty_r + rel % DRS);
    }
    if (K >= 0 && ++sa == DA) { sa = 0; pa ^= 1; }
    if (++sj == DRS) { sj = 0; ph ^= 1; }
  }
}

// pass 1, x-blocked with z-pairs (so 4, 8, 12; even z origin) -------------
// tti_g2_tma's rings and producer; lane l of warp w owns row 2w + (l >> 4)
// and the z pair 2 (l & 15) + {0, 1}: x/y operand pairs are aligned LDS.64
// and packed FADD2/FFMA2, z terms per lane from a window of aligned pairs.
template <int SO>
__global__ void __launch_bounds__(SZ *(SBY + 1), 2) tti_g3_tma(const __grid_constant__ GMaps2 M,
                                                                 const GParams P) {
  using G = G2Geo<SO>;
  constexpr int R = G::R, H = G::H, Q = 2 * R + 2, DRS = G::DRS, DA = G::DA;
  constexpr int RE = R + (R & 1), NGW = (RE + R + 3) / 2;
  static_assert(H % 2 == 0, "z-pair pass 1 needs an even halo");
  extern __shared__ __align__(128) unsigned char smem_raw[];
  float *ring = reinterpret_cast<float *>(smem_raw);  // [DRS][2][HALF]
  float *aux = ring + DRS * 2 * G::HALF;              // [DA][2][SLOTA]
  uint64_t *full_r = reinterpret_cast<uint64_t *>(aux + DA * 2 * G::SLOTA);
  uint64_t *empty_r = full_r + DRS;
  uint64_t *full_a = empty_r + DRS;
  uint64_t *empty_a = full_a + DA;

  const int tz = threadIdx.x, ty = threadIdx.y;
  const StreamCommon &C = P.c;
  const int z0 = C.lo[2] + blockIdx.x * SZ, y0 = C.lo[1] + blockIdx.y * STY;
  const int xs = blockIdx.z * C.xchunk;
  const int XC = min(C.xchunk, C.n[0] - xs);
  const int x0 = C.lo[0] + xs;
  const int KP = (XC + 1) / 2, JT = KP + R;
  const int zr = z0 + H - R, er = zr & 3;
  const int za = z0 + H, ea = za & 3;

  if (ty == 0 && tz == 0) {
    for (int i = 0; i < DRS; ++i) { mbar_init(full_r + i, 1); mbar_init(empty_r + i, SBY); }
    for (int i = 0; i < DA; ++i) { mbar_init(full_a + i, 1); mbar_init(empty_a + i, SBY); }
    fence_barrier_init();
  }
  __syncthreads();
  if (ty == SBY) {
    if (tz != 0) return;
    const int Xs = (int)C.ext[0];
    for (int J = 0; J < JT; ++J) {
      const int s = J % DRS;
      if (J >= DRS) mbar_wait(empty_r + s, ((J / DRS) - 1) & 1);
      mbar_expect_tx(full_r + s, 4 * G::PLANE * 4);
      const int xst = x0 + 2 * J - R + H;
      float *dst = ring + s * 2 * G::HALF;
      tma_load_3d(dst, &M.p, full_r + s, zr - er, y0 + H - R, P.cur * Xs + xst);
      tma_load_3d(dst + G::HALF, &M.r, full_r + s, zr - er, y0 + H - R, P.cur * Xs + xst);
      const int K = J - R;
      if (K >= 0) {
        const int sa = K % DA;
        if (K >= DA) mbar_wait(empty_a + sa, ((K / DA) - 1) & 1);
        mbar_expect_tx(full_a + sa, 4 * G::PLANEA * 4);
        float *ad = aux + sa * 2 * G::SLOTA;
        const int xk = x0 + 2 * K + H;
        tma_load_3d(ad, &M.th, full_a + sa, za - ea, y0 + H, xk);
        tma_load_3d(ad + G::SLOTA, &M.ph, full_a + sa, za - ea, y0 + H, xk);
      }
    }
    return;
  }
  using X2 = P2;
  auto ld2 = [](const float *q) -> uint64_t { return *reinterpret_cast<const uint64_t *>(q); };
  const int lane = tz;
  const int zc = 2 * (lane & 15), yr = 2 * ty + (lane >> 4);
  uint64_t qp[Q], qr[Q];
#pragma unroll
  for (int q = 0; q < Q; ++q) { qp[q] = 0; qr[q] = 0; }
  const int c0 = (yr + R) * G::W + zc + R + er;
  const int a0 = yr * G::WA + zc + ea;
  const int z = z0 + zc, y = y0 + yr;
  const bool yok = y < C.lo[1] + C.n[1];
  const bool ok0 = yok && z < C.lo[2] + C.n[2], ok1 = yok && z + 1 < C.lo[2] + C.n[2];
  const int64_t pl = C.ext[1] * C.ext[2];
  const int64_t own = (int64_t)(y + H) * C.ext[2] + (z + H);
  int sj = 0, ph = 0, sa = 0, pa = 0;
#pragma unroll 1
  for (int J = 0; J < JT; ++J) {
    mbar_wait(full_r + sj, ph);
    {
      const float *pp = ring + sj * 2 * G::HALF + c0;
#pragma unroll
      for (int q = 0; q < Q - 2; ++q) { qp[q] = qp[q + 2]; qr[q] = qr[q + 2]; }
      qp[Q - 2] = ld2(pp);
      qp[Q - 1] = ld2(pp + G::PLANE);
      qr[Q - 2] = ld2(pp + G::HALF);
      qr[Q - 1] = ld2(pp + G::HALF + G::PLANE);
    }
    const int K = J - R;
    if (K >= 0) {
      mbar_wait(full_a + sa, pa);
      const float *at = aux + sa * 2 * G::SLOTA + a0;
#pragma unroll
      for (int e = 0; e < 2; ++e) {
        const float *c = ring + wrapi(sj - (R - (R + e) / 2), DRS) * 2 * G::HALF +
                         ((R + e) & 1) * G::PLANE + c0;
        const uint64_t th = ld2(at + e * G::PLANEA), phv = ld2(at + G::SLOTA + e * G::PLANEA);
        float ax0, ay0, az0, ax1, ay1, az1;
        dir3(X2::lo(th), X2::lo(phv), ax0, ay0, az0);
        dir3(X2::hi(th), X2::hi(phv), ax1, ay1, az1);
        uint64_t dpx = 0, drx = 0, dpy = 0, dry = 0;
#pragma unroll
        for (int kk = 1; kk <= R; ++kk) {
          const uint64_t w = X2::pk(P.c1[kk - 1], P.c1[kk - 1]);
          dpx = X2::fma(w, X2::sub(qp[e + R + kk], qp[e + R - kk]), dpx);
          drx = X2::fma(w, X2::sub(qr[e + R + kk], qr[e + R - kk]), drx);
          dpy = X2::fma(w, X2::sub(ld2(c + kk * G::W), ld2(c - kk * G::W)), dpy);
          dry = X2::fma(w, X2::sub(ld2(c + G::HALF + kk * G::W), ld2(c + G::HALF - kk * G::W)),
                        dry);
        }
        float pw[2 * NGW], rw[2 * NGW];  // z windows: offsets -RE ..
#pragma unroll
        for (int j = 0; j < NGW; ++j) {
          const uint64_t a = ld2(c + 2 * j - RE), b = ld2(c + G::HALF + 2 * j - RE);
          pw[2 * j] = X2::lo(a); pw[2 * j + 1] = X2::hi(a);
          rw[2 * j] = X2::lo(b); rw[2 * j + 1] = X2::hi(b);
        }
        float dpz0 = 0.f, dpz1 = 0.f, drz0 = 0.f, drz1 = 0.f;
#pragma unroll
        for (int kk = 1; kk <= R; ++kk) {
          const float w = P.c1[kk - 1];
          dpz0 = fmaf(w, pw[RE + kk] - pw[RE - kk], dpz0);
          dpz1 = fmaf(w, pw[RE + 1 + kk] - pw[RE + 1 - kk], dpz1);
          drz0 = fmaf(w, rw[RE + kk] - rw[RE - kk], drz0);
          drz1 = fmaf(w, rw[RE + 1 + kk] - rw[RE + 1 - kk], drz1);
        }
        const uint64_t bx = X2::mul0(X2::pk(ax0, ax1), X2::pk(P.invh[0], P.invh[0]));
        const uint64_t by = X2::mul0(X2::pk(ay0, ay1), X2::pk(P.invh[1], P.invh[1]));
        const uint64_t bz = X2::mul0(X2::pk(az0, az1), X2::pk(P.invh[2], P.invh[2]));
        if (2 * K + e < XC) {
          const uint64_t gp = X2::fma(bx, dpx, X2::fma(by, dpy, X2::mul0(bz, X2::pk(dpz0, dpz1))));
          const uint64_t gr = X2::fma(bx, drx, X2::fma(by, dry, X2::mul0(bz, X2::pk(drz0, drz1))));
          const int64_t o = (int64_t)(x0 + 2 * K + e + H) * pl + own;
          if (ok1) {
            SC_DCHECK(o >= 0 && o + 1 < C.ext[0] * C.ext[1] * C.ext[2]);
          *reinterpret_cast<uint64_t *>(P.gp + o) = gp;
            *reinterpret_cast<uint64_t *>(P.gr + o) = gr;
          } else if (ok0) {
            SC_DCHECK(o >= 0 && o < C.ext[0] * C.ext[1] * C.ext[2]);
          P.gp[o] = X2::lo(gp);
            P.gr[o] = X2::lo(gr);
          }
        }
      }
    }
    __syncwarp();
    if (lane == 0) {
      if (K >= 0) mbar_arrive(empty_a + sa);
      const int rel = J - R + R / 2;
      if (rel >= 0) mbar_arrive(empty_r + rel % DRS);
    }
    if (K >= 0 && ++sa == DA) { sa = 0; pa ^= 1; }
    if (++sj == DRS) { sj = 0; ph ^= 1; }
  }
}

#ifndef SC_TTI_SPLIT1
#define SC_TTI_SPLIT1 1
#endif
#ifndef SC_TTI_SPLIT2
#define SC_TTI_SPLIT2 1
#endif
// which orders use it in pass 1 / pass 2 (build-time A/B: SC_TTI_SPLIT1/2 = 0
// none, 1 the measured choice, 2 every order). Config 3 grid, GPts/s, one box,
// none / pass 1 only / pass 2 only / both: so 12 65.3 / 65.6 / 66.3 / 66.5,
// so 16 58.6 / 57.0 / 59.4 / 57.8, so 8 68.3 / 68.5 / 67.8 / 67.8, so 4 flat
// (profiles/r02_tti_splitq.md)
__host__ __device__ constexpr bool tti_split1(int so) {
  return SC_TTI_SPLIT1 == 2 || (SC_TTI_SPLIT1 == 1 && so == 12);
}
__host__ __device__ constexpr bool tti_split2(int so) {
  return SC_TTI_SPLIT2 == 2 || (SC_TTI_SPLIT2 == 1 && (so == 12 || so == 16));
}

template <int N, int I = 0, class F>
__device__ __forceinline__ void static_for(F &&f) {
  if constexpr (I < N) {
    f(std::integral_constant<int, I>{});
    static_for<N, I + 1>(f);
  }
}

// pass 1, one plane per iteration, z-pairs (default for even halos) ---------
// tti_g_tma's one-plane rings (three planes of lookahead) with the z-pair
// consumer of tti_g3_tma; two CTAs per SM.
// PF planes of TMA lookahead: four at so 8/12 (so 12: 0.999 vs 1.009 ms per
// launch with three, A/B; five drops to 1.136 ms), three at so 4 (67.6 vs
// 66.8 GPts/s) and so 16 -- with the rotating queue (SC_TTI_G1ROT=1);
// SC_TTI_G1S=1 then selects three everywhere. The default shifting queue
// always runs three planes ahead.
__host__ __device__ constexpr int g1z_pf(int so) { return (so == 8 || so == 12) ? 4 : SPF; }
template <int SO, int PF> struct G1zSmem {
  static constexpr int R = SO / 4;
  static constexpr size_t B = (size_t)4 * ((R + 1 + PF) * 2 * Ring<2, R>::PAD +
                                           (1 + PF) * 2 * AuxTile<2>::TILE) +
                              16 * ((R + 1 + PF) + (1 + PF));
};

template <int SO, bool ROT, int PF>
__global__ void __launch_bounds__(SZ *(SBY + 1), 2) tti_g1z_tma(const __grid_constant__ GMaps M,
                                                                  const GParams P) {
  constexpr int R = SO / 4, H = SO / 2, Q = 2 * R + 1;
  constexpr int RE = R + (R & 1), NGW = (RE + R + 3) / 2;
  static_assert(H % 2 == 0, "z-pair pass 1 needs an even halo");
  using RG = Ring<2, R>;
  using AX = AuxTile<2>;
  constexpr int DR = R + 1 + PF, DA = 1 + PF;
  extern __shared__ __align__(128) unsigned char smem_raw[];
  float *ring = reinterpret_cast<float *>(smem_raw);            // [DR][2][PAD]
  float *aux = ring + DR * 2 * RG::PAD;                          // [DA][2][TILE]
  uint64_t *full_r = reinterpret_cast<uint64_t *>(aux + DA * 2 * AX::TILE);
  uint64_t *empty_r = full_r + DR;
  uint64_t *full_a = empty_r + DR;
  uint64_t *empty_a = full_a + DA;

  const int tz = threadIdx.x, ty = threadIdx.y;
  const StreamCommon &C = P.c;
  const int z0 = C.lo[2] + blockIdx.x * SZ, y0 = C.lo[1] + blockIdx.y * STY;
  const int xs = blockIdx.z * C.xchunk;
  const int XC = min(C.xchunk, C.n[0] - xs);
  const int x0 = C.lo[0] + xs;
  const int total = XC + 2 * R;
  const int zr = z0 + H - R, er = zr & 3;
  const int za = z0 + H, ea = za & 3;

  if (ty == 0 && tz == 0) {
    for (int i = 0; i < DR; ++i) { mbar_init(full_r + i, 1); mbar_init(empty_r + i, SBY); }
    for (int i = 0; i < DA; ++i) { mbar_init(full_a + i, 1); mbar_init(empty_a + i, SBY); }
    fence_barrier_init();
  }
  __syncthreads();
  if (ty == SBY) {
    if (tz != 0) return;
    const int Xs = (int)C.ext[0];
    for (int j = 0; j < total; ++j) {
      const int s = j % DR;
      if (j >= DR) mbar_wait(empty_r + s, ((j / DR) - 1) & 1);
      mbar_expect_tx(full_r + s, 2 * RG::PLANE * 4);
      const int xst = x0 + j - R + H;
      float *dst = ring + s * 2 * RG::PAD;
      tma_load_3d(dst, &M.p, full_r + s, zr - er, y0 + H - R, P.cur * Xs + xst);
      tma_load_3d(dst + RG::PAD, &M.r, full_r + s, zr - er, y0 + H - R, P.cur * Xs + xst);
      const int k = j - 2 * R;
      if (k >= 0) {
        const int sa = k % DA;
        if (k >= DA) mbar_wait(empty_a + sa, ((k / DA) - 1) & 1);
        mbar_expect_tx(full_a + sa, 2 * AX::TILE * 4);
        float *ad = aux + sa * 2 * AX::TILE;
        const int xk = x0 + k + H;
        tma_load_3d(ad, &M.th, full_a + sa, za - ea, y0 + H, xk);
        tma_load_3d(ad + AX::TILE, &M.ph, full_a + sa, za - ea, y0 + H, xk);
      }
    }
    return;
  }
  using X2 = P2;
  auto ld2 = [](const float *q) -> uint64_t { return *reinterpret_cast<const uint64_t *>(q); };
  const int lane = tz;
  const int zc = 2 * (lane & 15), yr = 2 * ty + (lane >> 4);
  constexpr bool SPLIT = !ROT && tti_split1(SO);
  using SQ = SplitQ<Q>;
  constexpr int QS = SPLIT ? SQ::SIZE : Q;
  uint64_t qp[QS], qr[QS];
#pragma unroll
  for (int q = 0; q < QS; ++q) { qp[q] = 0; qr[q] = 0; }
  const int c0 = (yr + R) * RG::W + zc + R + er;
  const int a0 = yr * AX::W + zc + ea;
  const int z = z0 + zc, y = y0 + yr;
  const bool yok = y < C.lo[1] + C.n[1];
  const bool ok0 = yok && z < C.lo[2] + C.n[2], ok1 = yok && z + 1 < C.lo[2] + C.n[2];
  const int64_t pl = C.ext[1] * C.ext[2];
  const int64_t own = (int64_t)(y + H) * C.ext[2] + (z + H);
  int sj = 0, ph = 0, sa = 0, pa = 0;
  // one x plane per call; O = j mod Q names the physical slot of logical
  // queue entry i as (i + O) % Q, so with ROT the Q-fold unrolled loop
  // rotates the x queue by renaming instead of shifting registers (the
  // shift was 27 of 221 SASS instructions per plane at so=12)
  auto plane = [&](const int j, auto Oc) {
    constexpr int O = ROT ? decltype(Oc)::value : 0;
    constexpr int PAR = decltype(Oc)::value & 1;  // split queue: X / Y iteration
#define QI(i) (SPLIT ? SQ::phys((i), PAR) : (((i) + O) % Q))
      mbar_wait(full_r + sj, ph);
      {
        const float *pp = ring + sj * 2 * RG::PAD + c0;
        if constexpr (SPLIT) {
          if constexpr (PAR == 1) {
  #pragma unroll
            for (int q = 0; q < SQ::NA - 1; ++q) {
              qp[q] = qp[q + 1]; qp[SQ::NA + q] = qp[SQ::NA + q + 1];
              qr[q] = qr[q + 1]; qr[SQ::NA + q] = qr[SQ::NA + q + 1];
            }
          }
        } else if constexpr (!ROT) {
  #pragma unroll
          for (int q = 0; q < Q - 1; ++q) { qp[q] = qp[q + 1]; qr[q] = qr[q + 1]; }
        }
        qp[QI(Q - 1)] = ld2(pp);
        qr[QI(Q - 1)] = ld2(pp + RG::PAD);
      }
      const int k = j - 2 * R;
      const int sc = wrapi(sj - R, DR);  // ring slot of the centre plane j - R
      if (k >= 0) {
        mbar_wait(full_a + sa, pa);
        const float *c = ring + sc * 2 * RG::PAD + c0;
        const float *at = aux + sa * 2 * AX::TILE + a0;
        const uint64_t th = ld2(at), phv = ld2(at + AX::TILE);
        float ax0, ay0, az0, ax1, ay1, az1;
        dir3(X2::lo(th), X2::lo(phv), ax0, ay0, az0);
        dir3(X2::hi(th), X2::hi(phv), ax1, ay1, az1);
        uint64_t dpx = 0, drx = 0, dpy = 0, dry = 0;
  #pragma unroll
        for (int kk = 1; kk <= R; ++kk) {
          const uint64_t w = X2::pk(P.c1[kk - 1], P.c1[kk - 1]);
          dpx = X2::fma(w, X2::sub(qp[QI(R + kk)], qp[QI(R - kk)]), dpx);
          drx = X2::fma(w, X2::sub(qr[QI(R + kk)], qr[QI(R - kk)]), drx);
          dpy = X2::fma(w, X2::sub(ld2(c + kk * RG::W), ld2(c - kk * RG::W)), dpy);
          dry = X2::fma(w, X2::sub(ld2(c + RG::PAD + kk * RG::W), ld2(c + RG::PAD - kk * RG::W)),
                        dry);
        }
        float pw[2 * NGW], rw[2 * NGW];
  #pragma unroll
        for (int jj = 0; jj < NGW; ++jj) {
          const uint64_t a = ld2(c + 2 * jj - RE), b = ld2(c + RG::PAD + 2 * jj - RE);
          pw[2 * jj] = X2::lo(a); pw[2 * jj + 1] = X2::hi(a);
          rw[2 * jj] = X2::lo(b); rw[2 * jj + 1] = X2::hi(b);
        }
        float dpz0 = 0.f, dpz1 = 0.f, drz0 = 0.f, drz1 = 0.f;
  #pragma unroll
        for (int kk = 1; kk <= R; ++kk) {
          const float w = P.c1[kk - 1];
          dpz0 = fmaf(w, pw[RE + kk] - pw[RE - kk], dpz0);
          dpz1 = fmaf(w, pw[RE + 1 + kk] - pw[RE + 1 - kk], dpz1);
          drz0 = fmaf(w, rw[RE + kk] - rw[RE - kk], drz0);
          drz1 = fmaf(w, rw[RE + 1 + kk] - rw[RE + 1 - kk], drz1);
        }
        const uint64_t bx = X2::mul0(X2::pk(ax0, ax1), X2::pk(P.invh[0], P.invh[0]));
        const uint64_t by = X2::mul0(X2::pk(ay0, ay1), X2::pk(P.invh[1], P.invh[1]));
        const uint64_t bz = X2::mul0(X2::pk(az0, az1), X2::pk(P.invh[2], P.invh[2]));
        const uint64_t gp = X2::fma(bx, dpx, X2::fma(by, dpy, X2::mul0(bz, X2::pk(dpz0, dpz1))));
        const uint64_t gr = X2::fma(bx, drx, X2::fma(by, dry, X2::mul0(bz, X2::pk(drz0, drz1))));
        const int64_t o = (int64_t)(x0 + k + H) * pl + own;
        if (ok1) {
          SC_DCHECK(o >= 0 && o + 1 < C.ext[0] * C.ext[1] * C.ext[2]);
          *reinterpret_cast<uint64_t *>(P.gp + o) = gp;
          *reinterpret_cast<uint64_t *>(P.gr + o) = gr;
        } else if (ok0) {
          SC_DCHECK(o >= 0 && o < C.ext[0] * C.ext[1] * C.ext[2]);
          P.gp[o] = X2::lo(gp);
          P.gr[o] = X2::lo(gr);
        }
        __syncwarp();
        if (lane == 0) {
          mbar_arrive(empty_a + sa);
          mbar_arrive(empty_r + sc);
        }
        if (++sa == DA) { sa = 0; pa ^= 1; }
      } else if (j >= R) {
        __syncwarp();
        if (lane == 0) mbar_arrive(empty_r + sc);
      }
      if (++sj == DR) { sj = 0; ph ^= 1; }
#undef QI
  };
  if constexpr (ROT) {
#pragma unroll 1
    for (int j0 = 0; j0 < total; j0 += Q)
      static_for<Q>([&](auto Oc) {
        if (j0 + decltype(Oc)::value < total) plane(j0 + decltype(Oc)::value, Oc);
      });
  } else if constexpr (SPLIT) {
#pragma unroll 1
    for (int j = 0; j < total; j += 2) {
      plane(j, std::integral_constant<int, 0>{});
      if (j + 1 < total) plane(j + 1, std::integral_constant<int, 1>{});
    }
  } else {
#pragma unroll 1
    for (int j = 0; j < total; ++j) plane(j, std::integral_constant<int, 0>{});
  }
}

// pass 2 ------------------------------------------------------------------
template <int SO>
__global__ void __launch_bounds__(SZ *(UBY + 1), 1) tti_upd_tma(const __grid_constant__ UMaps M,
                                                                  const UParams P) {
  constexpr int R = SO / 4, H = SO / 2, QP = 2 * H + 1, QG = 2 * R + 1;
  using RP = Ring<1, H>;
  using RG = Ring<2, R>;
  using AX = AuxTile<9>;
  constexpr int NAUX = 9;  // r, p-, r-, m, damp, eps, delta, theta, phi
  constexpr int PF = spf_u(SO);
  constexpr int DP = H + 1 + PF, DG = R + 1 + PF, DA = 1 + PF;
  extern __shared__ __align__(128) unsigned char smem_raw[];
  float *pring = reinterpret_cast<float *>(smem_raw);  // [DP][PAD]
  float *gring = pring + DP * RP::PAD;                 // [DG][2][PAD]
  float *aux = gring + DG * 2 * RG::PAD;               // [DA][9][TILE]
  uint64_t *full_p = reinterpret_cast<uint64_t *>(aux + DA * NAUX * AX::TILE);
  uint64_t *empty_p = full_p + DP;
  uint64_t *full_g = empty_p + DP;
  uint64_t *empty_g = full_g + DG;
  uint64_t *full_a = empty_g + DG;
  uint64_t *empty_a = full_a + DA;

  const int tz = threadIdx.x, ty = threadIdx.y;
  const StreamCommon &C = P.c;
  const int z0 = C.lo[2] + blockIdx.x * SZ, y0 = C.lo[1] + blockIdx.y * STY;
  const int xs = blockIdx.z * C.xchunk;
  const int XC = min(C.xchunk, C.n[0] - xs);
  const int x0 = C.lo[0] + xs;
  const int total = XC + 2 * H;  // p load j <-> loop x0 + j - H; output k = j - 2H
  const int zp = z0, ep = zp & 3;               // p box start (storage) = loop z0 - H
  const int zg = z0 + H - R, eg = zg & 3;       // g box start
  const int za = z0 + H, ea = za & 3;

  if (ty == 0 && tz == 0) {
    for (int i = 0; i < DP; ++i) { mbar_init(full_p + i, 1); mbar_init(empty_p + i, UBY); }
    for (int i = 0; i < DG; ++i) { mbar_init(full_g + i, 1); mbar_init(empty_g + i, UBY); }
    for (int i = 0; i < DA; ++i) { mbar_init(full_a + i, 1); mbar_init(empty_a + i, UBY); }
    fence_barrier_init();
  }
  __syncthreads();
  if (ty == UBY) {
    if (tz != 0) return;
    const int Xs = (int)C.ext[0];
    for (int j = 0; j < total; ++j) {
      {
        const int s = j % DP;
        if (j >= DP) mbar_wait(empty_p + s, ((j / DP) - 1) & 1);
        mbar_expect_tx(full_p + s, RP::PLANE * 4);
        tma_load_3d(pring + s * RP::PAD, &M.p, full_p + s, zp - ep, y0, P.cur * Xs + x0 + j);
      }
      const int i = j - 2 * R;  // g index i <-> loop x0 + i - R
      if (i >= 0 && i < XC + 2 * R) {
        const int s = i % DG;
        if (i >= DG) mbar_wait(empty_g + s, ((i / DG) - 1) & 1);
        mbar_expect_tx(full_g + s, 2 * RG::PLANE * 4);
        const int xst = x0 + i - R + H;
        float *dst = gring + s * 2 * RG::PAD;
        tma_load_3d(dst, &M.gp, full_g + s, zg - eg, y0 + H - R, xst);
        tma_load_3d(dst + RG::PAD, &M.gr, full_g + s, zg - eg, y0 + H - R, xst);
      }
      const int k = j - 2 * H;
      if (k >= 0) {
        const int s = k % DA;
        if (k >= DA) mbar_wait(empty_a + s, ((k / DA) - 1) & 1);
        mbar_expect_tx(full_a + s, NAUX * AX::TILE * 4);
        float *ad = aux + s * NAUX * AX::TILE;
        const int xk = x0 + k + H, zs = za - ea, ys = y0 + H;
        tma_load_3d(ad + 0 * AX::TILE, &M.r, full_a + s, zs, ys, P.cur * Xs + xk);
        tma_load_3d(ad + 1 * AX::TILE, &M.pm, full_a + s, zs, ys, P.prev * Xs + xk);
        tma_load_3d(ad + 2 * AX::TILE, &M.rm, full_a + s, zs, ys, P.prev * Xs + xk);
        tma_load_3d(ad + 3 * AX::TILE, &M.m, full_a + s, zs, ys, xk);
        tma_load_3d(ad + 4 * AX::TILE, &M.damp, full_a + s, zs, ys, xk);
        tma_load_3d(ad + 5 * AX::TILE, &M.eps, full_a + s, zs, ys, xk);
        tma_load_3d(ad + 6 * AX::TILE, &M.delta, full_a + s, zs, ys, xk);
        tma_load_3d(ad + 7 * AX::TILE, &M.th, full_a + s, zs, ys, xk);
        tma_load_3d(ad + 8 * AX::TILE, &M.ph, full_a + s, zs, ys, xk);
      }
    }
    return;
  }
  const int lane = tz;
  float qp[USRY][QP], qg[USRY][QG], qh[USRY][QG];
#pragma unroll
  for (int r = 0; r < USRY; ++r) {
#pragma unroll
    for (int q = 0; q < QP; ++q) qp[r][q] = 0.f;
#pragma unroll
    for (int q = 0; q < QG; ++q) { qg[r][q] = 0.f; qh[r][q] = 0.f; }
  }
  const int prow0 = ty * USRY + H, pcol = tz + H + ep;
  const int grow0 = ty * USRY + R, gcol = tz + R + eg;
  const int z = z0 + tz, yb = y0 + ty * USRY;
  const bool zok = z < C.lo[2] + C.n[2];
  const int yend = C.lo[1] + C.n[1];
  const int64_t pl = C.ext[1] * C.ext[2];
  const int64_t own = (int64_t)(yb + H) * C.ext[2] + (z + H);
  float c1[R], c2[H + 1], ih[3], ih2[3];
#pragma unroll
  for (int k = 0; k < R; ++k) c1[k] = P.c1[k];
#pragma unroll
  for (int k = 0; k <= H; ++k) c2[k] = P.c2[k];
#pragma unroll
  for (int k = 0; k < 3; ++k) { ih[k] = P.invh[k]; ih2[k] = P.invh2[k]; }
  int sp = 0, php = 0, sg = 0, phg = 0, sa = 0, pha = 0;
#pragma unroll 1
  for (int j = 0; j < total; ++j) {
    mbar_wait(full_p + sp, php);
    {
      const float *pp = pring + sp * RP::PAD;
#pragma unroll
      for (int r = 0; r < USRY; ++r) {
#pragma unroll
        for (int i = 0; i < QP - 1; ++i) qp[r][i] = qp[r][i + 1];
        qp[r][QP - 1] = pp[(prow0 + r) * RP::W + pcol];
      }
    }
    const int i = j - 2 * R;
    if (i >= 0 && i < XC + 2 * R) {
      mbar_wait(full_g + sg, phg);
      const float *gg = gring + sg * 2 * RG::PAD, *gh = gg + RG::PAD;
#pragma unroll
      for (int r = 0; r < USRY; ++r) {
#pragma unroll
        for (int q = 0; q < QG - 1; ++q) { qg[r][q] = qg[r][q + 1]; qh[r][q] = qh[r][q + 1]; }
        qg[r][QG - 1] = gg[(grow0 + r) * RG::W + gcol];
        qh[r][QG - 1] = gh[(grow0 + r) * RG::W + gcol];
      }
    }
    const int k = j - 2 * H;
    const int spc = wrapi(sp - H, DP);   // p ring slot of the output plane
    const int sgc = wrapi(sg - R, DG);   // g ring slot of the output plane
    if (k >= 0) {
      mbar_wait(full_a + sa, pha);
      const float *pc = pring + spc * RP::PAD;
      const float *gpc = gring + sgc * 2 * RG::PAD, *grc = gpc + RG::PAD;
      const float *ax_ = aux + sa * NAUX * AX::TILE;
#pragma unroll
      for (int r = 0; r < USRY; ++r) {
        const int ai = (ty * USRY + r) * AX::W + tz + ea;
        float ax, ay, az;
        dir3(ax_[7 * AX::TILE + ai], ax_[8 * AX::TILE + ai], ax, ay, az);
        const int cg = (grow0 + r) * RG::W + gcol;
        float hpx = 0.f, hpy = 0.f, hpz = 0.f, hrx = 0.f, hry = 0.f, hrz = 0.f;
#pragma unroll
        for (int kk = 1; kk <= R; ++kk) {
          const float w = c1[kk - 1];
          hpx = fmaf(w, qg[r][R + kk] - qg[r][R - kk], hpx);
          hrx = fmaf(w, qh[r][R + kk] - qh[r][R - kk], hrx);
          hpy = fmaf(w, gpc[cg + kk * RG::W] - gpc[cg - kk * RG::W], hpy);
          hry = fmaf(w, grc[cg + kk * RG::W] - grc[cg - kk * RG::W], hry);
          hpz = fmaf(w, gpc[cg + kk] - gpc[cg - kk], hpz);
          hrz = fmaf(w, grc[cg + kk] - grc[cg - kk], hrz);
        }
        const float bx = ax * ih[0], by = ay * ih[1], bz = az * ih[2];
        const float hzp = fmaf(bx, hpx, fmaf(by, hpy, bz * hpz));
        const float hzr = fmaf(bx, hrx, fmaf(by, hry, bz * hrz));
        const int cp = (prow0 + r) * RP::W + pcol;
        const float p0 = qp[r][H];
        float lx = c2[0] * p0, ly = c2[0] * p0, lz = c2[0] * p0;
#pragma unroll
        for (int kk = 1; kk <= H; ++kk) {
          const float w = c2[kk];
          lx = fmaf(w, qp[r][H + kk] + qp[r][H - kk], lx);
          ly = fmaf(w, pc[cp + kk * RP::W] + pc[cp - kk * RP::W], ly);
          lz = fmaf(w, pc[cp + kk] + pc[cp - kk], lz);
        }
        const float lap = fmaf(lx, ih2[0], fmaf(ly, ih2[1], lz * ih2[2]));
        const float hxy = lap - hzp;
        // hoisted coefficients (tti_hoist): 2a, E, S, I
        const float A2 = ax_[3 * AX::TILE + ai], Ec = ax_[4 * AX::TILE + ai];
        const float Sc = ax_[5 * AX::TILE + ai], Ic = ax_[6 * AX::TILE + ai];
        const float r0 = ax_[ai], pm = ax_[1 * AX::TILE + ai], rm = ax_[2 * AX::TILE + ai];
        if (zok && yb + r < yend) {
          const int64_t o = (int64_t)(x0 + k + H) * pl + own + (int64_t)r * C.ext[2];
          P.pn[o] = fmaf(A2, p0 - pm, fmaf(Ec, hxy, fmaf(Sc, hzr, pm)));
          P.rn[o] = fmaf(A2, r0 - rm, fmaf(Sc, hxy, fmaf(Ic, hzr, rm)));
        }
      }
      __syncwarp();
      if (lane == 0) {
        mbar_arrive(empty_a + sa);
        mbar_arrive(empty_p + spc);
        mbar_arrive(empty_g + sgc);
      }
      if (++sa == DA) { sa = 0; pha ^= 1; }
    } else {
      __syncwarp();
      if (lane == 0) {
        if (j >= H) mbar_arrive(empty_p + spc);            // p plane j - H
        if (i >= R && i - R < XC + 2 * R) mbar_arrive(empty_g + sgc);  // g index i - R
      }
    }
    if (++sp == DP) { sp = 0; php ^= 1; }
    if (i >= 0 && i < XC + 2 * R && ++sg == DG) { sg = 0; phg ^= 1; }
  }
}

// pass 2, x-blocked (so <= 12) ----------------------------------------------
// Same arithmetic as tti_upd_tma, but every ring slot holds TWO consecutive x
// planes (3D TMA boxes of depth 2) and each consumer iteration produces two
// output planes: half the mbarrier round trips and loop overhead per point,
// and each register-queue shift moves two planes. 16 consumer warps own one
// y row each of a 32 x 16 (z, y) tile.
template <int SO> struct U2Geo {
  static constexpr int R = SO / 4, H = SO / 2;
  static constexpr int NW = 16;                         // consumer warps = rows
  static constexpr int WP = ((SZ + 2 * H + 3 + 7) / 8) * 8;
  static constexpr int WG = ((SZ + 2 * R + 3 + 7) / 8) * 8;
  static constexpr int WA = ((SZ + 3 + 7) / 8) * 8;
  static constexpr int PLANEP = WP * (NW + 2 * H), PLANEG = WG * (NW + 2 * R), PLANEA = WA * NW;
  static constexpr int rnd(int f) { return ((f * 4 + 127) / 128) * 128 / 4; }
  static constexpr int SLOTP = rnd(2 * PLANEP);         // one p pair
  static constexpr int HALFG = rnd(2 * PLANEG);         // one field of a g pair
  static constexpr int SLOTA = rnd(2 * PLANEA);         // one field of an aux pair
  static constexpr int DPS = H / 2 + 2;                 // p pairs: H/2 + 1 live + 1 ahead
  static constexpr int DGS = (R + 1) / 2 + 2;           // g pairs: ceil(R/2) + 1 live + 1 ahead
  static constexpr int DA = 2;
  static constexpr size_t SMEM =
      (size_t)4 * (DPS * SLOTP + DGS * 2 * HALFG + DA * 9 * SLOTA) + 16 * (DPS + DGS + DA);
};

struct UMaps2 { CUtensorMap p, gp, gr, a[9]; };

// producer of the x-blocked pass-2 kernels: one lane streams p pairs, g pairs
// and the nine aux pairs into their rings
template <int SO>
__device__ __forceinline__ void upd2_produce(const UMaps2 &M, const UParams &P, float *pring,
                                             float *gring, float *aring, uint64_t *full_p,
                                             uint64_t *empty_p, uint64_t *full_g,
                                             uint64_t *empty_g, uint64_t *full_a,
                                             uint64_t *empty_a, int x0, int y0, int JT, int GP,
                                             int zp, int ep, int zg, int eg, int za, int ea) {
  using G = U2Geo<SO>;
  constexpr int R = G::R, H = G::H, DPS = G::DPS, DGS = G::DGS, DA = G::DA;
  const StreamCommon &C = P.c;
    const int Xs = (int)C.ext[0];
    for (int J = 0; J < JT; ++J) {
      {
        const int s = J % DPS;
        if (J >= DPS) mbar_wait(empty_p + s, ((J / DPS) - 1) & 1);
        mbar_expect_tx(full_p + s, 2 * G::PLANEP * 4);
        tma_load_3d(pring + s * G::SLOTP, &M.p, full_p + s, zp - ep, y0, P.cur * Xs + x0 + 2 * J);
      }
      const int I = J - R;
      if (I >= 0 && I < GP) {
        const int s = I % DGS;
        if (I >= DGS) mbar_wait(empty_g + s, ((I / DGS) - 1) & 1);
        mbar_expect_tx(full_g + s, 4 * G::PLANEG * 4);
        const int xst = x0 + 2 * I - R + H;
        float *dst = gring + s * 2 * G::HALFG;
        tma_load_3d(dst, &M.gp, full_g + s, zg - eg, y0 + H - R, xst);
        tma_load_3d(dst + G::HALFG, &M.gr, full_g + s, zg - eg, y0 + H - R, xst);
      }
      const int K = J - H;
      if (K >= 0) {
        const int s = K % DA;
        if (K >= DA) mbar_wait(empty_a + s, ((K / DA) - 1) & 1);
        mbar_expect_tx(full_a + s, 9 * 2 * G::PLANEA * 4);
        float *ad = aring + s * 9 * G::SLOTA;
        const int xk = x0 + 2 * K + H, ys = y0 + H, zs = za - ea;
        tma_load_3d(ad + 0 * G::SLOTA, &M.a[0], full_a + s, zs, ys, P.cur * Xs + xk);
        tma_load_3d(ad + 1 * G::SLOTA, &M.a[1], full_a + s, zs, ys, P.prev * Xs + xk);
        tma_load_3d(ad + 2 * G::SLOTA, &M.a[2], full_a + s, zs, ys, P.prev * Xs + xk);
#pragma unroll
        for (int f = 3; f < 9; ++f) tma_load_3d(ad + f * G::SLOTA, &M.a[f], full_a + s, zs, ys, xk);
      }
    }
}

template <int SO>
__global__ void __launch_bounds__(SZ *(U2Geo<SO>::NW + 1), 1) tti_upd2_tma(const __grid_constant__ UMaps2 M,
                                                                             const UParams P) {
  using G = U2Geo<SO>;
  constexpr int R = G::R, H = G::H, NW = G::NW, DPS = G::DPS, DGS = G::DGS, DA = G::DA;
  constexpr int QP = 2 * H + 2, QG = 2 * R + 2;
  extern __shared__ __align__(128) unsigned char smem_raw[];
  float *pring = reinterpret_cast<float *>(smem_raw);  // [DPS][SLOTP]
  float *gring = pring + DPS * G::SLOTP;               // [DGS][2][HALFG]
  float *aring = gring + DGS * 2 * G::HALFG;           // [DA][9][SLOTA]
  uint64_t *full_p = reinterpret_cast<uint64_t *>(aring + DA * 9 * G::SLOTA);
  uint64_t *empty_p = full_p + DPS;
  uint64_t *full_g = empty_p + DPS;
  uint64_t *empty_g = full_g + DGS;
  uint64_t *full_a = empty_g + DGS;
  uint64_t *empty_a = full_a + DA;

  const int tz = threadIdx.x, ty = threadIdx.y;
  const StreamCommon &C = P.c;
  const int z0 = C.lo[2] + blockIdx.x * SZ, y0 = C.lo[1] + blockIdx.y * NW;
  const int xs = blockIdx.z * C.xchunk;
  const int XC = min(C.xchunk, C.n[0] - xs);
  const int x0 = C.lo[0] + xs;
  const int KP = (XC + 1) / 2;   // output pairs
  const int JT = KP + H;         // p pairs (p load j <-> loop x0 + j - H)
  const int GP = KP + R;         // g pairs (g index i <-> loop x0 + i - R)
  const int zp = z0, ep = zp & 3;
  const int zg = z0 + H - R, eg = zg & 3;
  const int za = z0 + H, ea = za & 3;

  if (ty == 0 && tz == 0) {
    for (int i = 0; i < DPS; ++i) { mbar_init(full_p + i, 1); mbar_init(empty_p + i, NW); }
    for (int i = 0; i < DGS; ++i) { mbar_init(full_g + i, 1); mbar_init(empty_g + i, NW); }
    for (int i = 0; i < DA; ++i) { mbar_init(full_a + i, 1); mbar_init(empty_a + i, NW); }
    fence_barrier_init();
  }
  __syncthreads();
  if (ty == NW) {
    if (tz != 0) return;
    upd2_produce<SO>(M, P, pring, gring, aring, full_p, empty_p, full_g, empty_g, full_a, empty_a,
                     x0, y0, JT, GP, zp, ep, zg, eg, za, ea);
    return;
  }
  const int lane = tz;
  float qp[QP], qg[QG], qh[QG];
#pragma unroll
  for (int q = 0; q < QP; ++q) qp[q] = 0.f;
#pragma unroll
  for (int q = 0; q < QG; ++q) { qg[q] = 0.f; qh[q] = 0.f; }
  const int cp = (ty + H) * G::WP + tz + H + ep;  // p ring offset of the thread's point
  const int cg = (ty + R) * G::WG + tz + R + eg;  // g ring offset
  const int ca = ty * G::WA + tz + ea;            // aux offset
  const int z = z0 + tz, y = y0 + ty;
  const bool ok = z < C.lo[2] + C.n[2] && y < C.lo[1] + C.n[1];
  const int64_t pl = C.ext[1] * C.ext[2];
  const int64_t own = (int64_t)(y + H) * C.ext[2] + (z + H);
  int sp = 0, php = 0, sg = 0, phg = 0, sa = 0, pha = 0;
#pragma unroll 1
  for (int J = 0; J < JT; ++J) {
    mbar_wait(full_p + sp, php);
    {
      const float *pp = pring + sp * G::SLOTP + cp;
#pragma unroll
      for (int q = 0; q < QP - 2; ++q) qp[q] = qp[q + 2];
      qp[QP - 2] = pp[0];
      qp[QP - 1] = pp[G::PLANEP];
    }
    const int I = J - R;
    const bool gin = I >= 0 && I < GP;
    if (gin) {
      mbar_wait(full_g + sg, phg);
      const float *gg = gring + sg * 2 * G::HALFG + cg;
#pragma unroll
      for (int q = 0; q < QG - 2; ++q) { qg[q] = qg[q + 2]; qh[q] = qh[q + 2]; }
      qg[QG - 2] = gg[0];
      qg[QG - 1] = gg[G::PLANEG];
      qh[QG - 2] = gg[G::HALFG];
      qh[QG - 1] = gg[G::HALFG + G::PLANEG];
    }
    const int K = J - H;
    if (K >= 0) {
      mbar_wait(full_a + sa, pha);
      const float *pcen = pring + wrapi(sp - H / 2, DPS) * G::SLOTP + cp;  // p pair K + H/2
      const float *ax_ = aring + sa * 9 * G::SLOTA + ca;
#pragma unroll
      for (int e = 0; e < 2; ++e) {
        // g centre index 2K + R + e lives in pair K + (R + e) / 2, plane (R + e) & 1;
        // the newest g pair (slot sg) is K + R
        const float *gcen = gring + wrapi(sg - (R - (R + e) / 2), DGS) * 2 * G::HALFG +
                            ((R + e) & 1) * G::PLANEG + cg;
        const float *pc = pcen + e * G::PLANEP;
        const float *av = ax_ + e * G::PLANEA;
        float ax, ay, az;
        dir3(av[7 * G::SLOTA], av[8 * G::SLOTA], ax, ay, az);
        float hpx = 0.f, hpy = 0.f, hpz = 0.f, hrx = 0.f, hry = 0.f, hrz = 0.f;
#pragma unroll
        for (int kk = 1; kk <= R; ++kk) {
          const float w = P.c1[kk - 1];
          hpx = fmaf(w, qg[e + R + kk] - qg[e + R - kk], hpx);
          hrx = fmaf(w, qh[e + R + kk] - qh[e + R - kk], hrx);
          hpy = fmaf(w, gcen[kk * G::WG] - gcen[-kk * G::WG], hpy);
          hry = fmaf(w, gcen[G::HALFG + kk * G::WG] - gcen[G::HALFG - kk * G::WG], hry);
          hpz = fmaf(w, gcen[kk] - gcen[-kk], hpz);
          hrz = fmaf(w, gcen[G::HALFG + kk] - gcen[G::HALFG - kk], hrz);
        }
        const float bx = ax * P.invh[0], by = ay * P.invh[1], bz = az * P.invh[2];
        const float hzp = fmaf(bx, hpx, fmaf(by, hpy, bz * hpz));
        const float hzr = fmaf(bx, hrx, fmaf(by, hry, bz * hrz));
        const float p0 = qp[e + H];
        const float c20 = P.c2[0];
        float lx = c20 * p0, ly = c20 * p0, lz = c20 * p0;
#pragma unroll
        for (int kk = 1; kk <= H; ++kk) {
          const float w = P.c2[kk];
          lx = fmaf(w, qp[e + H + kk] + qp[e + H - kk], lx);
          ly = fmaf(w, pc[kk * G::WP] + pc[-kk * G::WP], ly);
          lz = fmaf(w, pc[kk] + pc[-kk], lz);
        }
        const float lap = fmaf(lx, P.invh2[0], fmaf(ly, P.invh2[1], lz * P.invh2[2]));
        const float hxy = lap - hzp;
        const float A2 = av[3 * G::SLOTA], Ec = av[4 * G::SLOTA];
        const float Sc = av[5 * G::SLOTA], Ic = av[6 * G::SLOTA];
        const float r0 = av[0], pm = av[1 * G::SLOTA], rm = av[2 * G::SLOTA];
        if (ok && 2 * K + e < XC) {
          const int64_t o = (int64_t)(x0 + 2 * K + e + H) * pl + own;
          P.pn[o] = fmaf(A2, p0 - pm, fmaf(Ec, hxy, fmaf(Sc, hzr, pm)));
          P.rn[o] = fmaf(A2, r0 - rm, fmaf(Sc, hxy, fmaf(Ic, hzr, rm)));
        }
      }
    }
    __syncwarp();
    if (lane == 0) {
      if (K >= 0) mbar_arrive(empty_a + sa);
      if (J >= H / 2) mbar_arrive(empty_p + wrapi(sp - H / 2, DPS));  // p pair J - H/2
      // g pair J - 2R + R/2 (its last use as a y/z centre was output pair K)
      const int gr = J - 2 * R + R / 2;
      if (gr >= 0 && gr < GP) mbar_arrive(empty_g + gr % DGS);
    }
    if (K >= 0 && ++sa == DA) { sa = 0; pha ^= 1; }
    if (++sp == DPS) { sp = 0; php ^= 1; }
    if (gin && ++sg == DGS) { sg = 0; phg ^= 1; }
  }
}

// pass 2, x-blocked with z-pairs (so 4, 8, 12; even z origin) -------------
// Same rings, producer and arithmetic as tti_upd2_tma, but 8 consumer warps:
// lane l of warp w owns row 2w + (l >> 4) and the z pair 2 (l & 15) + {0, 1},
// two x planes per iteration (four points). Every x/y operand pair is one
// aligned LDS.64 and every x/y term is one packed FADD2/FFMA2 for both z
// points; z terms are evaluated per lane from a window of aligned pairs.
// (Reading the nine per-point operands with plain 64-bit global loads
// instead of the TMA aux ring was measured slower: 3.04 vs 2.28 ms at so 12.)
template <int SO> struct U3Geo {
  static constexpr int NWC = 8;  // consumer warps (9 warps: <= 168 registers)
};

template <int SO>
__global__ void __launch_bounds__(SZ *(U3Geo<SO>::NWC + 1), 1)
    tti_upd3_tma(const __grid_constant__ UMaps2 M, const UParams P) {
  using G = U2Geo<SO>;
  constexpr int R = G::R, H = G::H, NW = G::NW, DPS = G::DPS, DGS = G::DGS, DA = G::DA;
  constexpr int NWC = U3Geo<SO>::NWC;
  constexpr int QP = 2 * H + 2, QG = 2 * R + 2;
  constexpr int RE = R + (R & 1);  // g window starts at an even z offset
  constexpr int NPW = H + 1, NGW = (RE + R + 3) / 2;  // window pairs (p, g)
  static_assert(H % 2 == 0, "z-pair pass 2 needs an even halo");
  extern __shared__ __align__(128) unsigned char smem_raw[];
  float *pring = reinterpret_cast<float *>(smem_raw);
  float *gring = pring + DPS * G::SLOTP;
  float *aring = gring + DGS * 2 * G::HALFG;
  uint64_t *full_p = reinterpret_cast<uint64_t *>(aring + DA * 9 * G::SLOTA);
  uint64_t *empty_p = full_p + DPS;
  uint64_t *full_g = empty_p + DPS;
  uint64_t *empty_g = full_g + DGS;
  uint64_t *full_a = empty_g + DGS;
  uint64_t *empty_a = full_a + DA;

  const int tz = threadIdx.x, ty = threadIdx.y;
  const StreamCommon &C = P.c;
  const int z0 = C.lo[2] + blockIdx.x * SZ, y0 = C.lo[1] + blockIdx.y * NW;
  const int xs = blockIdx.z * C.xchunk;
  const int XC = min(C.xchunk, C.n[0] - xs);
  const int x0 = C.lo[0] + xs;
  const int KP = (XC + 1) / 2, JT = KP + H, GP = KP + R;
  const int zp = z0, ep = zp & 3;
  const int zg = z0 + H - R, eg = zg & 3;
  const int za = z0 + H, ea = za & 3;

  if (ty == 0 && tz == 0) {
    for (int i = 0; i < DPS; ++i) { mbar_init(full_p + i, 1); mbar_init(empty_p + i, NWC); }
    for (int i = 0; i < DGS; ++i) { mbar_init(full_g + i, 1); mbar_init(empty_g + i, NWC); }
    for (int i = 0; i < DA; ++i) { mbar_init(full_a + i, 1); mbar_init(empty_a + i, NWC); }
    fence_barrier_init();
  }
  __syncthreads();
  if (ty == NWC) {
    if (tz != 0) return;
    upd2_produce<SO>(M, P, pring, gring, aring, full_p, empty_p, full_g, empty_g, full_a, empty_a,
                     x0, y0, JT, GP, zp, ep, zg, eg, za, ea);
    return;
  }
  using X2 = P2;
  auto ld2 = [](const float *q) -> uint64_t { return *reinterpret_cast<const uint64_t *>(q); };
  const int lane = tz;
  const int zc = 2 * (lane & 15), yr = 2 * ty + (lane >> 4);
  uint64_t qp[QP], qg[QG], qh[QG];
#pragma unroll
  for (int q = 0; q < QP; ++q) qp[q] = 0;
#pragma unroll
  for (int q = 0; q < QG; ++q) { qg[q] = 0; qh[q] = 0; }
  const int cp = (yr + H) * G::WP + zc + H + ep;
  const int cg = (yr + R) * G::WG + zc + R + eg;
  const int ca = yr * G::WA + zc + ea;
  const int z = z0 + zc, y = y0 + yr;
  const bool yok = y < C.lo[1] + C.n[1];
  const bool ok0 = yok && z < C.lo[2] + C.n[2], ok1 = yok && z + 1 < C.lo[2] + C.n[2];
  const int64_t pl = C.ext[1] * C.ext[2];
  const int64_t own = (int64_t)(y + H) * C.ext[2] + (z + H);
  int sp = 0, php = 0, sg = 0, phg = 0, sa = 0, pha = 0;
#pragma unroll 1
  for (int J = 0; J < JT; ++J) {
    mbar_wait(full_p + sp, php);
    {
      const float *pp = pring + sp * G::SLOTP + cp;
#pragma unroll
      for (int q = 0; q < QP - 2; ++q) qp[q] = qp[q + 2];
      qp[QP - 2] = ld2(pp);
      qp[QP - 1] = ld2(pp + G::PLANEP);
    }
    const int I = J - R;
    const bool gin = I >= 0 && I < GP;
    if (gin) {
      mbar_wait(full_g + sg, phg);
      const float *gg = gring + sg * 2 * G::HALFG + cg;
#pragma unroll
      for (int q = 0; q < QG - 2; ++q) { qg[q] = qg[q + 2]; qh[q] = qh[q + 2]; }
      qg[QG - 2] = ld2(gg);
      qg[QG - 1] = ld2(gg + G::PLANEG);
      qh[QG - 2] = ld2(gg + G::HALFG);
      qh[QG - 1] = ld2(gg + G::HALFG + G::PLANEG);
    }
    const int K = J - H;
    if (K >= 0) {
      mbar_wait(full_a + sa, pha);
      const float *pcen = pring + wrapi(sp - H / 2, DPS) * G::SLOTP + cp;
      const float *ax_ = aring + sa * 9 * G::SLOTA + ca;
#pragma unroll
      for (int e = 0; e < 2; ++e) {
        const float *gcen = gring + wrapi(sg - (R - (R + e) / 2), DGS) * 2 * G::HALFG +
                            ((R + e) & 1) * G::PLANEG + cg;
        const float *pc = pcen + e * G::PLANEP;
        const float *av = ax_ + e * G::PLANEA;
        // direction cosines per lane, then packed
        const uint64_t th = ld2(av + 7 * G::SLOTA), phv = ld2(av + 8 * G::SLOTA);
        float ax0, ay0, az0, ax1, ay1, az1;
        dir3(X2::lo(th), X2::lo(phv), ax0, ay0, az0);
        dir3(X2::hi(th), X2::hi(phv), ax1, ay1, az1);
        const uint64_t bx = X2::mul0(X2::pk(ax0, ax1), X2::pk(P.invh[0], P.invh[0]));
        const uint64_t by = X2::mul0(X2::pk(ay0, ay1), X2::pk(P.invh[1], P.invh[1]));
        const uint64_t bz = X2::mul0(X2::pk(az0, az1), X2::pk(P.invh[2], P.invh[2]));
        // outer rotated derivatives of g_p (hp*) and g_r (hr*)
        uint64_t hpx = 0, hrx = 0, hpy = 0, hry = 0;
#pragma unroll
        for (int kk = 1; kk <= R; ++kk) {
          const uint64_t w = X2::pk(P.c1[kk - 1], P.c1[kk - 1]);
          hpx = X2::fma(w, X2::sub(qg[e + R + kk], qg[e + R - kk]), hpx);
          hrx = X2::fma(w, X2::sub(qh[e + R + kk], qh[e + R - kk]), hrx);
          hpy = X2::fma(w, X2::sub(ld2(gcen + kk * G::WG), ld2(gcen - kk * G::WG)), hpy);
          hry = X2::fma(w, X2::sub(ld2(gcen + G::HALFG + kk * G::WG),
                                   ld2(gcen + G::HALFG - kk * G::WG)), hry);
        }
        float gw[2 * NGW], hw[2 * NGW];  // z windows of g_p, g_r: offsets -RE ..
#pragma unroll
        for (int j = 0; j < NGW; ++j) {
          const uint64_t a = ld2(gcen + 2 * j - RE), b = ld2(gcen + G::HALFG + 2 * j - RE);
          gw[2 * j] = X2::lo(a); gw[2 * j + 1] = X2::hi(a);
          hw[2 * j] = X2::lo(b); hw[2 * j + 1] = X2::hi(b);
        }
        float hpz0 = 0.f, hpz1 = 0.f, hrz0 = 0.f, hrz1 = 0.f;
#pragma unroll
        for (int kk = 1; kk <= R; ++kk) {
          const float w = P.c1[kk - 1];
          hpz0 = fmaf(w, gw[RE + kk] - gw[RE - kk], hpz0);
          hpz1 = fmaf(w, gw[RE + 1 + kk] - gw[RE + 1 - kk], hpz1);
          hrz0 = fmaf(w, hw[RE + kk] - hw[RE - kk], hrz0);
          hrz1 = fmaf(w, hw[RE + 1 + kk] - hw[RE + 1 - kk], hrz1);
        }
        const uint64_t hzp = X2::fma(bx, hpx, X2::fma(by, hpy, X2::mul0(bz, X2::pk(hpz0, hpz1))));
        const uint64_t hzr = X2::fma(bx, hrx, X2::fma(by, hry, X2::mul0(bz, X2::pk(hrz0, hrz1))));
        // Laplacian of p
        const uint64_t p0 = qp[e + H];
        uint64_t lx = X2::mul0(X2::pk(P.c2[0], P.c2[0]), p0), ly = lx;
#pragma unroll
        for (int kk = 1; kk <= H; ++kk) {
          const uint64_t w = X2::pk(P.c2[kk], P.c2[kk]);
          lx = X2::fma(w, X2::add(qp[e + H + kk], qp[e + H - kk]), lx);
          ly = X2::fma(w, X2::add(ld2(pc + kk * G::WP), ld2(pc - kk * G::WP)), ly);
        }
        float pw[2 * NPW];  // z window of p: offsets -H .. H + 1
#pragma unroll
        for (int j = 0; j < NPW; ++j) {
          const uint64_t a = (2 * j == H) ? p0 : ld2(pc + 2 * j - H);
          pw[2 * j] = X2::lo(a); pw[2 * j + 1] = X2::hi(a);
        }
        float lz0 = P.c2[0] * pw[H], lz1 = P.c2[0] * pw[H + 1];
#pragma unroll
        for (int kk = 1; kk <= H; ++kk) {
          lz0 = fmaf(P.c2[kk], pw[H + kk] + pw[H - kk], lz0);
          lz1 = fmaf(P.c2[kk], pw[H + 1 + kk] + pw[H + 1 - kk], lz1);
        }
        const uint64_t lap =
            X2::fma(lx, X2::pk(P.invh2[0], P.invh2[0]),
                    X2::fma(ly, X2::pk(P.invh2[1], P.invh2[1]),
                            X2::mul0(X2::pk(lz0, lz1), X2::pk(P.invh2[2], P.invh2[2]))));
        const uint64_t hxy = X2::sub(lap, hzp);
        if (2 * K + e < XC) {
          const uint64_t A2 = ld2(av + 3 * G::SLOTA), Ec = ld2(av + 4 * G::SLOTA);
          const uint64_t Sc = ld2(av + 5 * G::SLOTA), Ic = ld2(av + 6 * G::SLOTA);
          const uint64_t r0 = ld2(av), pm = ld2(av + 1 * G::SLOTA), rm = ld2(av + 2 * G::SLOTA);
          const uint64_t pn =
              X2::fma(A2, X2::sub(p0, pm), X2::fma(Ec, hxy, X2::fma(Sc, hzr, pm)));
          const uint64_t rn =
              X2::fma(A2, X2::sub(r0, rm), X2::fma(Sc, hxy, X2::fma(Ic, hzr, rm)));
          const int64_t o = (int64_t)(x0 + 2 * K + e + H) * pl + own;
          if (ok1) {
            SC_DCHECK(o >= 0 && o + 1 < C.ext[0] * C.ext[1] * C.ext[2]);
          *reinterpret_cast<uint64_t *>(P.pn + o) = pn;
            *reinterpret_cast<uint64_t *>(P.rn + o) = rn;
          } else if (ok0) {
            SC_DCHECK(o >= 0 && o < C.ext[0] * C.ext[1] * C.ext[2]);
          P.pn[o] = X2::lo(pn);
            P.rn[o] = X2::lo(rn);
          }
        }
      }
    }
    __syncwarp();
    if (lane == 0) {
      if (K >= 0) mbar_arrive(empty_a + sa);
      if (J >= H / 2) mbar_arrive(empty_p + wrapi(sp - H / 2, DPS));
      const int gr = J - 2 * R + R / 2;
      if (gr >= 0 && gr < GP) mbar_arrive(empty_g + gr % DGS);
    }
    if (K >= 0 && ++sa == DA) { sa = 0; pha ^= 1; }
    if (++sp == DPS) { sp = 0; php ^= 1; }
    if (gin && ++sg == DGS) { sg = 0; phg ^= 1; }
  }
}

// pass 2, one plane per iteration, z-pairs (so 16, whose x-blocked rings do
// not fit) --------------------------------------------------------------------
// tti_upd_tma's rings and producer; 8 consumer warps, lane l of warp w owns
// row 2w + (l >> 4) and the z pair 2 (l & 15) + {0, 1} (packed x/y terms,
// LDS.64 operands, z terms per lane from windows of aligned pairs).
template <int SO>
__global__ void __launch_bounds__(SZ *(SBY + 1), 1) tti_upd1z_tma(const __grid_constant__ UMaps M,
                                                                   const UParams P) {
  constexpr int R = SO / 4, H = SO / 2, QP = 2 * H + 1, QG = 2 * R + 1, NWC = SBY;
  constexpr int RE = R + (R & 1);
  constexpr int NPW = H + 1, NGW = (RE + R + 3) / 2;
  static_assert(H % 2 == 0, "z-pair pass 2 needs an even halo");
  using RP = Ring<1, H>;
  using RG = Ring<2, R>;
  using AX = AuxTile<9>;
  constexpr int NAUX = 9;
  constexpr int PF = spf_u(SO);
  constexpr int DP = H + 1 + PF, DG = R + 1 + PF, DA = 1 + PF;
  extern __shared__ __align__(128) unsigned char smem_raw[];
  float *pring = reinterpret_cast<float *>(smem_raw);
  float *gring = pring + DP * RP::PAD;
  float *aux = gring + DG * 2 * RG::PAD;
  uint64_t *full_p = reinterpret_cast<uint64_t *>(aux + DA * NAUX * AX::TILE);
  uint64_t *empty_p = full_p + DP;
  uint64_t *full_g = empty_p + DP;
  uint64_t *empty_g = full_g + DG;
  uint64_t *full_a = empty_g + DG;
  uint64_t *empty_a = full_a + DA;

  const int tz = threadIdx.x, ty = threadIdx.y;
  const StreamCommon &C = P.c;
  int bz = blockIdx.x, by = blockIdx.y, xs = blockIdx.z * C.xchunk, xlen = C.xchunk;
  if (C.tailq > 0) {
    int tile = blockIdx.x;
    xs = 0;
    xlen = C.n[0];
    if (tile >= C.nwhole) {
      const int j = tile - C.nwhole;
      tile = C.nwhole + j / C.tailq;
      xlen = (C.n[0] + C.tailq - 1) / C.tailq;
      xs = (j % C.tailq) * xlen;
    }
    by = tile / C.ntz;
    bz = tile - by * C.ntz;
  }
  const int z0 = C.lo[2] + bz * SZ, y0 = C.lo[1] + by * STY;
  const int XC = min(xlen, C.n[0] - xs);
  if (XC <= 0) return;
  const int x0 = C.lo[0] + xs;
  const int total = XC + 2 * H;
  const int zp = z0, ep = zp & 3;
  const int zg = z0 + H - R, eg = zg & 3;
  const int za = z0 + H, ea = za & 3;

  if (ty == 0 && tz == 0) {
    for (int i = 0; i < DP; ++i) { mbar_init(full_p + i, 1); mbar_init(empty_p + i, NWC); }
    for (int i = 0; i < DG; ++i) { mbar_init(full_g + i, 1); mbar_init(empty_g + i, NWC); }
    for (int i = 0; i < DA; ++i) { mbar_init(full_a + i, 1); mbar_init(empty_a + i, NWC); }
    fence_barrier_init();
  }
  __syncthreads();
  if (ty == NWC) {
    if (tz != 0) return;
    const int Xs = (int)C.ext[0];
    for (int j = 0; j < total; ++j) {
      {
        const int s = j % DP;
        if (j >= DP) mbar_wait(empty_p + s, ((j / DP) - 1) & 1);
        mbar_expect_tx(full_p + s, RP::PLANE * 4);
        tma_load_3d(pring + s * RP::PAD, &M.p, full_p + s, zp - ep, y0, P.cur * Xs + x0 + j);
      }
      const int i = j - 2 * R;
      if (i >= 0 && i < XC + 2 * R) {
        const int s = i % DG;
        if (i >= DG) mbar_wait(empty_g + s, ((i / DG) - 1) & 1);
        mbar_expect_tx(full_g + s, 2 * RG::PLANE * 4);
        const int xst = x0 + i - R + H;
        float *dst = gring + s * 2 * RG::PAD;
        tma_load_3d(dst, &M.gp, full_g + s, zg - eg, y0 + H - R, xst);
        tma_load_3d(dst + RG::PAD, &M.gr, full_g + s, zg - eg, y0 + H - R, xst);
      }
      const int k = j - 2 * H;
      if (k >= 0) {
        const int s = k % DA;
        if (k >= DA) mbar_wait(empty_a + s, ((k / DA) - 1) & 1);
        mbar_expect_tx(full_a + s, NAUX * AX::TILE * 4);
        float *ad = aux + s * NAUX * AX::TILE;
        const int xk = x0 + k + H, zs = za - ea, ys = y0 + H;
        tma_load_3d(ad + 0 * AX::TILE, &M.r, full_a + s, zs, ys, P.cur * Xs + xk);
        tma_load_3d(ad + 1 * AX::TILE, &M.pm, full_a + s, zs, ys, P.prev * Xs + xk);
        tma_load_3d(ad + 2 * AX::TILE, &M.rm, full_a + s, zs, ys, P.prev * Xs + xk);
        tma_load_3d(ad + 3 * AX::TILE, &M.m, full_a + s, zs, ys, xk);
        tma_load_3d(ad + 4 * AX::TILE, &M.damp, full_a + s, zs, ys, xk);
        tma_load_3d(ad + 5 * AX::TILE, &M.eps, full_a + s, zs, ys, xk);
        tma_load_3d(ad + 6 * AX::TILE, &M.delta, full_a + s, zs, ys, xk);
        tma_load_3d(ad + 7 * AX::TILE, &M.th, full_a + s, zs, ys, xk);
        tma_load_3d(ad + 8 * AX::TILE, &M.ph, full_a + s, zs, ys, xk);
      }
    }
    return;
  }
  using X2 = P2;
  auto ld2 = [](const float *q) -> uint64_t { return *reinterpret_cast<const uint64_t *>(q); };
  const int lane = tz;
  const int zc = 2 * (lane & 15), yr = 2 * ty + (lane >> 4);
  constexpr bool SPLIT = tti_split2(SO);
  using SP = SplitQ<QP>;
  using SG = SplitQ<QG>;
  constexpr int QPS = SPLIT ? SP::SIZE : QP, QGS = SPLIT ? SG::SIZE : QG;
  uint64_t qp[QPS], qg[QGS], qh[QGS];
#pragma unroll
  for (int q = 0; q < QPS; ++q) qp[q] = 0;
#pragma unroll
  for (int q = 0; q < QGS; ++q) { qg[q] = 0; qh[q] = 0; }
  const int cp = (yr + H) * RP::W + zc + H + ep;
  const int cg = (yr + R) * RG::W + zc + R + eg;
  const int ca = yr * AX::W + zc + ea;
  const int z = z0 + zc, y = y0 + yr;
  const bool yok = y < C.lo[1] + C.n[1];
  const bool ok0 = yok && z < C.lo[2] + C.n[2], ok1 = yok && z + 1 < C.lo[2] + C.n[2];
  const int64_t pl = C.ext[1] * C.ext[2];
  const int64_t own = (int64_t)(y + H) * C.ext[2] + (z + H);
  int sp = 0, php = 0, sg = 0, phg = 0, sa = 0, pha = 0;
  // one x plane; PAR = j & 1 names the X / Y iteration of the split queues
  // (2 R is even, so the g queues, pushed from j = 2 R on, share it)
  auto plane = [&](const int j, auto Pc) {
    constexpr int PAR = decltype(Pc)::value;
#define QPI(i) (SPLIT ? SP::phys((i), PAR) : (i))
#define QGI(i) (SPLIT ? SG::phys((i), PAR) : (i))
    mbar_wait(full_p + sp, php);
    if constexpr (SPLIT) {
      if constexpr (PAR == 1) {
#pragma unroll
        for (int q = 0; q < SP::NA - 1; ++q) {
          qp[q] = qp[q + 1];
          qp[SP::NA + q] = qp[SP::NA + q + 1];
        }
      }
    } else {
#pragma unroll
      for (int q = 0; q < QP - 1; ++q) qp[q] = qp[q + 1];
    }
    qp[QPI(QP - 1)] = ld2(pring + sp * RP::PAD + cp);
    const int i = j - 2 * R;
    if (i >= 0 && i < XC + 2 * R) {
      mbar_wait(full_g + sg, phg);
      const float *gg = gring + sg * 2 * RG::PAD + cg;
      if constexpr (SPLIT) {
        if constexpr (PAR == 1) {
#pragma unroll
          for (int q = 0; q < SG::NA - 1; ++q) {
            qg[q] = qg[q + 1]; qg[SG::NA + q] = qg[SG::NA + q + 1];
            qh[q] = qh[q + 1]; qh[SG::NA + q] = qh[SG::NA + q + 1];
          }
        }
      } else {
#pragma unroll
        for (int q = 0; q < QG - 1; ++q) { qg[q] = qg[q + 1]; qh[q] = qh[q + 1]; }
      }
      qg[QGI(QG - 1)] = ld2(gg);
      qh[QGI(QG - 1)] = ld2(gg + RG::PAD);
    }
    const int k = j - 2 * H;
    const int spc = wrapi(sp - H, DP);
    const int sgc = wrapi(sg - R, DG);
    if (k >= 0) {
      mbar_wait(full_a + sa, pha);
      const float *pc = pring + spc * RP::PAD + cp;
      const float *gcen = gring + sgc * 2 * RG::PAD + cg;
      const float *av = aux + sa * NAUX * AX::TILE + ca;
      const uint64_t th = ld2(av + 7 * AX::TILE), phv = ld2(av + 8 * AX::TILE);
      float ax0, ay0, az0, ax1, ay1, az1;
      dir3(X2::lo(th), X2::lo(phv), ax0, ay0, az0);
      dir3(X2::hi(th), X2::hi(phv), ax1, ay1, az1);
      const uint64_t bx = X2::mul0(X2::pk(ax0, ax1), X2::pk(P.invh[0], P.invh[0]));
      const uint64_t by = X2::mul0(X2::pk(ay0, ay1), X2::pk(P.invh[1], P.invh[1]));
      const uint64_t bz = X2::mul0(X2::pk(az0, az1), X2::pk(P.invh[2], P.invh[2]));
      uint64_t hpx = 0, hrx = 0, hpy = 0, hry = 0;
#pragma unroll
      for (int kk = 1; kk <= R; ++kk) {
        const uint64_t w = X2::pk(P.c1[kk - 1], P.c1[kk - 1]);
        hpx = X2::fma(w, X2::sub(qg[QGI(R + kk)], qg[QGI(R - kk)]), hpx);
        hrx = X2::fma(w, X2::sub(qh[QGI(R + kk)], qh[QGI(R - kk)]), hrx);
        hpy = X2::fma(w, X2::sub(ld2(gcen + kk * RG::W), ld2(gcen - kk * RG::W)), hpy);
        hry = X2::fma(w, X2::sub(ld2(gcen + RG::PAD + kk * RG::W),
                                 ld2(gcen + RG::PAD - kk * RG::W)), hry);
      }
      float gw[2 * NGW], hw[2 * NGW];
#pragma unroll
      for (int jj = 0; jj < NGW; ++jj) {
        const uint64_t a = ld2(gcen + 2 * jj - RE), b = ld2(gcen + RG::PAD + 2 * jj - RE);
        gw[2 * jj] = X2::lo(a); gw[2 * jj + 1] = X2::hi(a);
        hw[2 * jj] = X2::lo(b); hw[2 * jj + 1] = X2::hi(b);
      }
      float hpz0 = 0.f, hpz1 = 0.f, hrz0 = 0.f, hrz1 = 0.f;
#pragma unroll
      for (int kk = 1; kk <= R; ++kk) {
        const float w = P.c1[kk - 1];
        hpz0 = fmaf(w, gw[RE + kk] - gw[RE - kk], hpz0);
        hpz1 = fmaf(w, gw[RE + 1 + kk] - gw[RE + 1 - kk], hpz1);
        hrz0 = fmaf(w, hw[RE + kk] - hw[RE - kk], hrz0);
        hrz1 = fmaf(w, hw[RE + 1 + kk] - hw[RE + 1 - kk], hrz1);
      }
      const uint64_t hzp = X2::fma(bx, hpx, X2::fma(by, hpy, X2::mul0(bz, X2::pk(hpz0, hpz1))));
      const uint64_t hzr = X2::fma(bx, hrx, X2::fma(by, hry, X2::mul0(bz, X2::pk(hrz0, hrz1))));
      const uint64_t p0 = qp[QPI(H)];
      uint64_t lx = X2::mul0(X2::pk(P.c2[0], P.c2[0]), p0), ly = lx;
#pragma unroll
      for (int kk = 1; kk <= H; ++kk) {
        const uint64_t w = X2::pk(P.c2[kk], P.c2[kk]);
        lx = X2::fma(w, X2::add(qp[QPI(H + kk)], qp[QPI(H - kk)]), lx);
        ly = X2::fma(w, X2::add(ld2(pc + kk * RP::W), ld2(pc - kk * RP::W)), ly);
      }
      float pw[2 * NPW];
#pragma unroll
      for (int jj = 0; jj < NPW; ++jj) {
        const uint64_t a = (2 * jj == H) ? p0 : ld2(pc + 2 * jj - H);
        pw[2 * jj] = X2::lo(a); pw[2 * jj + 1] = X2::hi(a);
      }
      float lz0 = P.c2[0] * pw[H], lz1 = P.c2[0] * pw[H + 1];
#pragma unroll
      for (int kk = 1; kk <= H; ++kk) {
        lz0 = fmaf(P.c2[kk], pw[H + kk] + pw[H - kk], lz0);
        lz1 = fmaf(P.c2[kk], pw[H + 1 + kk] + pw[H + 1 - kk], lz1);
      }
      const uint64_t lap =
          X2::fma(lx, X2::pk(P.invh2[0], P.invh2[0]),
                  X2::fma(ly, X2::pk(P.invh2[1], P.invh2[1]),
                          X2::mul0(X2::pk(lz0, lz1), X2::pk(P.invh2[2], P.invh2[2]))));
      const uint64_t hxy = X2::sub(lap, hzp);
      const uint64_t A2 = ld2(av + 3 * AX::TILE), Ec = ld2(av + 4 * AX::TILE);
      const uint64_t Sc = ld2(av + 5 * AX::TILE), Ic = ld2(av + 6 * AX::TILE);
      const uint64_t r0 = ld2(av), pm = ld2(av + 1 * AX::TILE), rm = ld2(av + 2 * AX::TILE);
      const uint64_t pn = X2::fma(A2, X2::sub(p0, pm), X2::fma(Ec, hxy, X2::fma(Sc, hzr, pm)));
      const uint64_t rn = X2::fma(A2, X2::sub(r0, rm), X2::fma(Sc, hxy, X2::fma(Ic, hzr, rm)));
      const int64_t o = (int64_t)(x0 + k + H) * pl + own;
      if (ok1) {
        SC_DCHECK(o >= 0 && o + 1 < C.ext[0] * C.ext[1] * C.ext[2]);
          *reinterpret_cast<uint64_t *>(P.pn + o) = pn;
        *reinterpret_cast<uint64_t *>(P.rn + o) = rn;
      } else if (ok0) {
        SC_DCHECK(o >= 0 && o < C.ext[0] * C.ext[1] * C.ext[2]);
          P.pn[o] = X2::lo(pn);
        P.rn[o] = X2::lo(rn);
      }
      __syncwarp();
      if (lane == 0) {
        mbar_arrive(empty_a + sa);
        mbar_arrive(empty_p + spc);
        mbar_arrive(empty_g + sgc);
      }
      if (++sa == DA) { sa = 0; pha ^= 1; }
    } else {
      __syncwarp();
      if (lane == 0) {
        if (j >= H) mbar_arrive(empty_p + spc);
        if (i >= R && i - R < XC + 2 * R) mbar_arrive(empty_g + sgc);
      }
    }
    if (++sp == DP) { sp = 0; php ^= 1; }
    if (i >= 0 && i < XC + 2 * R && ++sg == DG) { sg = 0; phg ^= 1; }
#undef QPI
#undef QGI
  };
  if constexpr (SPLIT) {
#pragma unroll 1
    for (int j = 0; j < total; j += 2) {
      plane(j, std::integral_constant<int, 0>{});
      if (j + 1 < total) plane(j + 1, std::integral_constant<int, 1>{});
    }
  } else {
#pragma unroll 1
    for (int j = 0; j < total; ++j) plane(j, std::integral_constant<int, 0>{});
  }
}

// ---------------------------------------------------------------------------
// Coupled passes (so 4/8/12, z-pair geometry): both passes of a time step in
// ONE persistent launch, g_p / g_r handed from pass 1 to pass 2 through L2.
//
// One CTA per SM, 16 warps: warps 0-7 are the pass-2 consumers of
// tti_upd1z_tma, warps 8-11 the pass-1 consumers of tti_g1z_tma (two rows
// per lane), warp 12 / 13 the pass-2 / pass-1 TMA producers, warp 14 / 15
// the pass-1 publisher / pass-2 poller of the inter-CTA counters; setmaxnreg
// moves registers from the producer warpgroup to the consumers. Tiles are
// numbered along z, then y, on pass 1's (widened) tiling. In round r CTA c
// runs pass 1 on tile s = r * gridDim.x + c and pass 2 on tile s - lag
// (lag = one tile row + 1), so the four pass-1 tiles a pass-2 tile reads g
// from are swept by CTAs c - lag .. c in the same round: every CTA walks x at
// the same time, pass 1 a few planes ahead of pass 2, and the g planes (and
// theta, phi, p, r) pass 2 loads are still in L2. Ordering:
//   * pass 1 publishes, per tile, the number of g planes completely stored
//     (prog[tile], st.release.gpu by its producer thread once every
//     consumer warp has released the plane's aux slot);
//   * the pass-2 producer acquires the counters of the (up to four) tiles
//     its g box overlaps before it issues the TMA load of a g plane;
//   * pass 1 stays within `lead` iterations of its own CTA's pass 2
//     (shared-memory counter), which bounds the g footprint in L2.
// All CTAs are co-resident (grid = number of SMs, one CTA fills an SM), and
// a pass-2 tile waits only on pass-1 tiles with a smaller or equal sequence
// number, so the waits cannot cycle. Same arithmetic as the two launches:
// bitwise equal results.
struct CplParams {
  int *prog;                    // [nty1 * ntz1], zeroed before the launch
  int nty1, ntz1, nty2, ntz2;   // pass-1 / pass-2 tiles along y and z
  int rounds, lead;
  int dbg;  // experiments: 1 = pass 2 does not wait for g (wrong results), 2 = no throttle
};

template <int SO, int PF2, int PFA, int PF1> struct CplGeo {
  static constexpr int R = SO / 4, H = SO / 2;
  using RP = Ring<1, H>;
  using RG = Ring<2, R>;
  using AX = AuxTile<9>;
  static constexpr int DP = H + 1 + PF2, DG = R + 1 + PF2, DA = 1 + PFA;
  static constexpr int DR = R + 1 + PF1, DA1 = 1 + PF1;
  static constexpr int NBAR = 2 * (DP + DG + DA + DR + DA1);
  static constexpr size_t FLOATS = (size_t)DP * RP::PAD + (size_t)DG * 2 * RG::PAD +
                                   (size_t)DA * 9 * AX::TILE + (size_t)DR * 2 * RG::PAD +
                                   (size_t)DA1 * 2 * AX::TILE;
  static constexpr size_t SMEM = FLOATS * 4 + (size_t)NBAR * 8 + 32;
};

__device__ __forceinline__ int ld_acquire_gpu(const int *p) {
  int v;
  asm volatile("ld.acquire.gpu.global.s32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
  return v;
}
__device__ __forceinline__ void st_release_gpu(int *p, int v) {
  asm volatile("st.release.gpu.global.s32 [%0], %1;" ::"l"(p), "r"(v) : "memory");
}
__device__ __forceinline__ int ld_relaxed_gpu(const int *p) {
  int v;
  asm volatile("ld.relaxed.gpu.global.s32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
  return v;
}
__device__ __forceinline__ void fence_acq_rel_gpu() { asm volatile("fence.acq_rel.gpu;" ::: "memory"); }
__device__ __forceinline__ int lds_acquire_cta(const int *p) {
  int v;
  asm volatile("ld.acquire.cta.shared::cta.s32 %0, [%1];" : "=r"(v) : "r"(smem_u32(p)) : "memory");
  return v;
}
__device__ __forceinline__ void sts_release_cta(int *p, int v) {
  asm volatile("st.release.cta.shared::cta.s32 [%0], %1;" ::"r"(smem_u32(p)), "r"(v) : "memory");
}
// generic-proxy writes (other SMs' stores of g, made visible by the acquire
// above) ordered before this thread's async-proxy (TMA) reads of them
__device__ __forceinline__ void fence_proxy_async_all() {
  asm volatile("fence.proxy.async;" ::: "memory");
}

// a wait on another CTA that lasts this many clocks (seconds) is a broken
// schedule: trap instead of hanging the device
constexpr long long CPL_WATCHDOG = 8000000000ll;
constexpr int CPL_RC2 = 152, CPL_RC1 = 136, CPL_RP = 64;  // registers per role

template <int SO, int PF2, int PFA, int PF1>
__global__ void __launch_bounds__(SZ * 16, 1)
    tti_cpl_tma(const __grid_constant__ GMaps GM, const __grid_constant__ UMaps UM, const GParams PG,
                const UParams PU, const CplParams Q) {
  using Geo = CplGeo<SO, PF2, PFA, PF1>;
  constexpr int R = Geo::R, H = Geo::H, QP = 2 * H + 1, QG = 2 * R + 1;
  constexpr int RE = R + (R & 1);
  constexpr int NPW = H + 1, NGW = (RE + R + 3) / 2;
  static_assert(H % 2 == 0, "the coupled kernel needs an even halo");
  using RP = typename Geo::RP;
  using RG = typename Geo::RG;
  using AX = typename Geo::AX;
  constexpr int NAUX = 9;
  constexpr int DP = Geo::DP, DG = Geo::DG, DA = Geo::DA, DR = Geo::DR, DA1 = Geo::DA1;
  constexpr int NW2 = 8, NW1 = 4;
  extern __shared__ __align__(128) unsigned char smem_raw[];
  float *pring = reinterpret_cast<float *>(smem_raw);   // pass 2: p planes
  float *gring = pring + DP * RP::PAD;                   // pass 2: g_p, g_r planes
  float *aux = gring + DG * 2 * RG::PAD;                 // pass 2: per-point operands
  float *ring1 = aux + DA * NAUX * AX::TILE;             // pass 1: p, r planes
  float *aux1 = ring1 + DR * 2 * RG::PAD;                // pass 1: theta, phi
  uint64_t *full_p = reinterpret_cast<uint64_t *>(aux1 + DA1 * 2 * AX::TILE);
  uint64_t *empty_p = full_p + DP;
  uint64_t *full_g = empty_p + DP;
  uint64_t *empty_g = full_g + DG;
  uint64_t *full_a = empty_g + DG;
  uint64_t *empty_a = full_a + DA;
  uint64_t *full_r = empty_a + DA;
  uint64_t *empty_r = full_r + DR;
  uint64_t *full_a1 = empty_r + DR;
  uint64_t *empty_a1 = full_a1 + DA1;
  volatile int *s_prog2 = reinterpret_cast<volatile int *>(empty_a1 + DA1);
  int *s_ready = const_cast<int *>(s_prog2) + 1;  // round << 16 | g planes ready for pass 2
  int *s_done1 = s_ready + 1;                     // [NW1] g planes stored per pass-1 warp

  const int lane = threadIdx.x, w = threadIdx.y;
  if (w == 0 && lane == 0) {
    for (int i = 0; i < DP; ++i) { mbar_init(full_p + i, 1); mbar_init(empty_p + i, NW2); }
    for (int i = 0; i < DG; ++i) { mbar_init(full_g + i, 1); mbar_init(empty_g + i, NW2); }
    for (int i = 0; i < DA; ++i) { mbar_init(full_a + i, 1); mbar_init(empty_a + i, NW2); }
    for (int i = 0; i < DR; ++i) { mbar_init(full_r + i, 1); mbar_init(empty_r + i, NW1); }
    for (int i = 0; i < DA1; ++i) { mbar_init(full_a1 + i, 1); mbar_init(empty_a1 + i, NW1); }
    *s_prog2 = 0;
    *s_ready = 0;
    for (int i = 0; i < NW1; ++i) s_done1[i] = 0;
    fence_barrier_init();
  }
  __syncthreads();

  const int NC = gridDim.x, cta = blockIdx.x;
  const int NT1 = Q.nty1 * Q.ntz1, LAG = Q.ntz1 + 1;
  const StreamCommon &C1 = PG.c;
  const StreamCommon &C2 = PU.c;
  const int T = C2.n[0] + 2 * H;  // iterations per x sweep, the same in both passes (4 R = 2 H)
  using X2 = P2;
  auto ld2 = [](const float *q) -> uint64_t { return *reinterpret_cast<const uint64_t *>(q); };

  if (w >= 12) {
    // ---- producers -------------------------------------------------------
    asm volatile("setmaxnreg.dec.sync.aligned.u32 %0;\n" ::"n"(CPL_RP));
    if (lane != 0) return;
    if (w == 14) {
      // pass-1 publisher: g planes every consumer warp has stored -> prog[tile]
      const int XC1 = C1.n[0];
      int base = 0;
      for (int r = 0; r < Q.rounds; ++r) {
        const int t1 = r * NC + cta;
        if (t1 >= NT1) break;
        int *flag = Q.prog + t1;
        int pub = 0;
        while (pub < XC1) {
          int m = min(min(lds_acquire_cta(s_done1), lds_acquire_cta(s_done1 + 1)),
                      min(lds_acquire_cta(s_done1 + 2), lds_acquire_cta(s_done1 + 3))) - base;
          m = min(m, XC1);
          if (m > pub) {
            st_release_gpu(flag, m);
            pub = m;
          }
        }
        base += XC1;
      }
      return;
    }
    if (w == 15) {
      // pass-2 poller: counters of the pass-1 tiles this tile's g box overlaps
      for (int r = 0; r < Q.rounds; ++r) {
        const int t2 = r * NC + cta - LAG;
        const int iy = t2 >= 0 ? t2 / Q.ntz1 : 0, iz = t2 - iy * Q.ntz1;
        if (t2 < 0 || t2 >= NT1 || iy >= Q.nty2 || iz >= Q.ntz2) continue;
        const bool dy = iy + 1 < Q.nty1, dz = iz + 1 < Q.ntz1;
        const int *f00 = Q.prog + t2;
        const int *f01 = dz ? f00 + 1 : f00;
        const int *f10 = dy ? f00 + Q.ntz1 : f00;
        const int *f11 = dy ? (dz ? f10 + 1 : f10) : f01;
        const int need = C2.n[0] + 2 * R;
        int seen = 0;
        long long t0 = clock64();
        while (seen < need) {
          const int m = min(min(ld_relaxed_gpu(f00), ld_relaxed_gpu(f01)),
                            min(ld_relaxed_gpu(f10), ld_relaxed_gpu(f11)));
          if (m > seen) {
            fence_acq_rel_gpu();
            fence_proxy_async_all();
            seen = m;
            sts_release_cta(s_ready, (r << 16) | m);
            t0 = clock64();
          } else if (clock64() - t0 > CPL_WATCHDOG) {
            printf("tti_cpl_tma: CTA %d round %d tile %d waits for g plane %d\n", cta, r, t2, seen);
            __trap();
          }
        }
      }
      return;
    }
    if (w == 12) {
      // pass 2
      const int Xs = (int)C2.ext[0];
      int np = 0, ng = 0, na = 0;  // planes issued into the p / g / aux rings, all rounds
      for (int r = 0; r < Q.rounds; ++r) {
        const int t2 = r * NC + cta - LAG;
        const int iy = t2 >= 0 ? t2 / Q.ntz1 : 0, iz = t2 - iy * Q.ntz1;
        if (t2 < 0 || t2 >= NT1 || iy >= Q.nty2 || iz >= Q.ntz2) {
          *s_prog2 = (r + 1) * T;
          continue;
        }
        const int y0 = C2.lo[1] + iy * STY, z0 = C2.lo[2] + iz * SZ, x0 = C2.lo[0];
        const int XC = C2.n[0];
        const int zp = z0, ep = zp & 3;
        const int zg = z0 + H - R, eg = zg & 3;
        const int za = z0 + H, ea = za & 3;
        int ready = (Q.dbg & 1) ? INT_MAX : 0;  // g planes known complete
        for (int j = 0; j < T; ++j) {
          {
            const int s = np % DP;
            if (np >= DP) mbar_wait(empty_p + s, ((np / DP) - 1) & 1);
            mbar_expect_tx(full_p + s, RP::PLANE * 4);
            tma_load_3d(pring + s * RP::PAD, &UM.p, full_p + s, zp - ep, y0, PU.cur * Xs + x0 + j);
            ++np;
          }
          const int k = j - 2 * H;
          if (k >= 0) {
            const int s = na % DA;
            if (na >= DA) mbar_wait(empty_a + s, ((na / DA) - 1) & 1);
            mbar_expect_tx(full_a + s, NAUX * AX::TILE * 4);
            float *ad = aux + s * NAUX * AX::TILE;
            const int xk = x0 + k + H, zs = za - ea, ys = y0 + H;
            tma_load_3d(ad + 0 * AX::TILE, &UM.r, full_a + s, zs, ys, PU.cur * Xs + xk);
            tma_load_3d(ad + 1 * AX::TILE, &UM.pm, full_a + s, zs, ys, PU.prev * Xs + xk);
            tma_load_3d(ad + 2 * AX::TILE, &UM.rm, full_a + s, zs, ys, PU.prev * Xs + xk);
            tma_load_3d(ad + 3 * AX::TILE, &UM.m, full_a + s, zs, ys, xk);
            tma_load_3d(ad + 4 * AX::TILE, &UM.damp, full_a + s, zs, ys, xk);
            tma_load_3d(ad + 5 * AX::TILE, &UM.eps, full_a + s, zs, ys, xk);
            tma_load_3d(ad + 6 * AX::TILE, &UM.delta, full_a + s, zs, ys, xk);
            tma_load_3d(ad + 7 * AX::TILE, &UM.th, full_a + s, zs, ys, xk);
            tma_load_3d(ad + 8 * AX::TILE, &UM.ph, full_a + s, zs, ys, xk);
            ++na;
          }
          const int i = j - 2 * R;
          if (i >= 0 && i < XC + 2 * R) {
            if (ready <= i) {
              int v;
              do {
                v = lds_acquire_cta(s_ready);
              } while (v < ((r << 16) | (i + 1)));
              ready = v - (r << 16);
              fence_proxy_async_all();
            }
            const int s = ng % DG;
            if (ng >= DG) mbar_wait(empty_g + s, ((ng / DG) - 1) & 1);
            mbar_expect_tx(full_g + s, 2 * RG::PLANE * 4);
            const int xst = x0 + i - R + H;
            float *dst = gring + s * 2 * RG::PAD;
            tma_load_3d(dst, &UM.gp, full_g + s, zg - eg, y0 + H - R, xst);
            tma_load_3d(dst + RG::PAD, &UM.gr, full_g + s, zg - eg, y0 + H - R, xst);
            ++ng;
          }
          *s_prog2 = r * T + j + 1;
        }
      }
    } else {
      // pass 1
      const int Xs = (int)C1.ext[0];
      int nr = 0, na = 0;  // planes issued into the p/r and theta/phi rings, all rounds
      for (int r = 0; r < Q.rounds; ++r) {
        const int t1 = r * NC + cta;
        if (t1 >= NT1) break;
        const int jy = t1 / Q.ntz1, jz = t1 - jy * Q.ntz1;
        const int y0 = C1.lo[1] + jy * STY, z0 = C1.lo[2] + jz * SZ, x0 = C1.lo[0];
        const int XC = C1.n[0];
        const int zr = z0 + H - R, er = zr & 3;
        const int za = z0 + H, ea = za & 3;
        for (int j = 0; j < T; ++j) {
          // stay within `lead` iterations of this CTA's pass 2
          if (!(Q.dbg & 2) && r * T + j > *s_prog2 + Q.lead) {
            const long long t0 = clock64();
            while (r * T + j > *s_prog2 + Q.lead) {
              if (clock64() - t0 > CPL_WATCHDOG) {
                printf("tti_cpl_tma: CTA %d round %d pass 1 at %d waits for pass 2 (at %d)\n", cta,
                       r, j, *s_prog2 - r * T);
                __trap();
              }
            }
          }
          const int s = nr % DR;
          if (nr >= DR) mbar_wait(empty_r + s, ((nr / DR) - 1) & 1);
          mbar_expect_tx(full_r + s, 2 * RG::PLANE * 4);
          const int xst = x0 + j - R + H;
          float *dst = ring1 + s * 2 * RG::PAD;
          tma_load_3d(dst, &GM.p, full_r + s, zr - er, y0 + H - R, PG.cur * Xs + xst);
          tma_load_3d(dst + RG::PAD, &GM.r, full_r + s, zr - er, y0 + H - R, PG.cur * Xs + xst);
          ++nr;
          const int k = j - 2 * R;
          if (k >= 0) {
            const int sa = na % DA1;
            if (na >= DA1) {
              mbar_wait(empty_a1 + sa, ((na / DA1) - 1) & 1);
            }
            mbar_expect_tx(full_a1 + sa, 2 * AX::TILE * 4);
            float *ad = aux1 + sa * 2 * AX::TILE;
            const int xk = x0 + k + H;
            tma_load_3d(ad, &GM.th, full_a1 + sa, za - ea, y0 + H, xk);
            tma_load_3d(ad + AX::TILE, &GM.ph, full_a1 + sa, za - ea, y0 + H, xk);
            ++na;
          }
        }
      }
    }
    return;
  }

  if (w >= NW2) {
    // ---- pass-1 consumers: rows yr and yr + 8 of the tile, one z pair ------
    asm volatile("setmaxnreg.inc.sync.aligned.u32 %0;\n" ::"n"(CPL_RC1));
    const int wi = w - NW2;
    const int zc = 2 * (lane & 15);
    uint64_t qp[2][QG], qr[2][QG];
#pragma unroll
    for (int h = 0; h < 2; ++h)
#pragma unroll
      for (int q = 0; q < QG; ++q) { qp[h][q] = 0; qr[h][q] = 0; }
    const int64_t pl = C1.ext[1] * C1.ext[2];
    int sj = 0, ph = 0, sa = 0, pa = 0, done = 0;
    for (int r = 0; r < Q.rounds; ++r) {
      const int t1 = r * NC + cta;
      if (t1 >= NT1) break;
      const int jy = t1 / Q.ntz1, jz = t1 - jy * Q.ntz1;
      const int y0 = C1.lo[1] + jy * STY, z0 = C1.lo[2] + jz * SZ, x0 = C1.lo[0];
      const int zr = z0 + H - R, er = zr & 3;
      const int za = z0 + H, ea = za & 3;
      const int z = z0 + zc;
      const bool zok0 = z < C1.lo[2] + C1.n[2], zok1 = z + 1 < C1.lo[2] + C1.n[2];
      int c0[2], a0[2];
      bool yok[2];
      int64_t own[2];
#pragma unroll
      for (int h = 0; h < 2; ++h) {
        const int yr = 2 * wi + (lane >> 4) + 8 * h;
        c0[h] = (yr + R) * RG::W + zc + R + er;
        a0[h] = yr * AX::W + zc + ea;
        yok[h] = y0 + yr < C1.lo[1] + C1.n[1];
        own[h] = (int64_t)(y0 + yr + H) * C1.ext[2] + (z + H);
      }
#pragma unroll 1
      for (int j = 0; j < T; ++j) {
        mbar_wait(full_r + sj, ph);
#pragma unroll
        for (int h = 0; h < 2; ++h) {
          const float *pp = ring1 + sj * 2 * RG::PAD + c0[h];
#pragma unroll
          for (int q = 0; q < QG - 1; ++q) { qp[h][q] = qp[h][q + 1]; qr[h][q] = qr[h][q + 1]; }
          qp[h][QG - 1] = ld2(pp);
          qr[h][QG - 1] = ld2(pp + RG::PAD);
        }
        const int k = j - 2 * R;
        const int sc = wrapi(sj - R, DR);  // ring slot of the centre plane j - R
        if (k >= 0) {
          mbar_wait(full_a1 + sa, pa);
#pragma unroll
          for (int h = 0; h < 2; ++h) {
            if (Q.dbg & 4) break;
            const float *c = ring1 + sc * 2 * RG::PAD + c0[h];
            const float *at = aux1 + sa * 2 * AX::TILE + a0[h];
            const uint64_t th = ld2(at), phv = ld2(at + AX::TILE);
            float ax0, ay0, az0, ax1, ay1, az1;
            dir3(X2::lo(th), X2::lo(phv), ax0, ay0, az0);
            dir3(X2::hi(th), X2::hi(phv), ax1, ay1, az1);
            uint64_t dpx = 0, drx = 0, dpy = 0, dry = 0;
#pragma unroll
            for (int kk = 1; kk <= R; ++kk) {
              const uint64_t wk = X2::pk(PG.c1[kk - 1], PG.c1[kk - 1]);
              dpx = X2::fma(wk, X2::sub(qp[h][R + kk], qp[h][R - kk]), dpx);
              drx = X2::fma(wk, X2::sub(qr[h][R + kk], qr[h][R - kk]), drx);
              dpy = X2::fma(wk, X2::sub(ld2(c + kk * RG::W), ld2(c - kk * RG::W)), dpy);
              dry = X2::fma(wk, X2::sub(ld2(c + RG::PAD + kk * RG::W),
                                        ld2(c + RG::PAD - kk * RG::W)), dry);
            }
            float pw[2 * NGW], rw[2 * NGW];
#pragma unroll
            for (int jj = 0; jj < NGW; ++jj) {
              const uint64_t a = ld2(c + 2 * jj - RE), b = ld2(c + RG::PAD + 2 * jj - RE);
              pw[2 * jj] = X2::lo(a); pw[2 * jj + 1] = X2::hi(a);
              rw[2 * jj] = X2::lo(b); rw[2 * jj + 1] = X2::hi(b);
            }
            float dpz0 = 0.f, dpz1 = 0.f, drz0 = 0.f, drz1 = 0.f;
#pragma unroll
            for (int kk = 1; kk <= R; ++kk) {
              const float wk = PG.c1[kk - 1];
              dpz0 = fmaf(wk, pw[RE + kk] - pw[RE - kk], dpz0);
              dpz1 = fmaf(wk, pw[RE + 1 + kk] - pw[RE + 1 - kk], dpz1);
              drz0 = fmaf(wk, rw[RE + kk] - rw[RE - kk], drz0);
              drz1 = fmaf(wk, rw[RE + 1 + kk] - rw[RE + 1 - kk], drz1);
            }
            const uint64_t bx = X2::mul0(X2::pk(ax0, ax1), X2::pk(PG.invh[0], PG.invh[0]));
            const uint64_t by = X2::mul0(X2::pk(ay0, ay1), X2::pk(PG.invh[1], PG.invh[1]));
            const uint64_t bz = X2::mul0(X2::pk(az0, az1), X2::pk(PG.invh[2], PG.invh[2]));
            const uint64_t gp = X2::fma(bx, dpx, X2::fma(by, dpy, X2::mul0(bz, X2::pk(dpz0, dpz1))));
            const uint64_t gr = X2::fma(bx, drx, X2::fma(by, dry, X2::mul0(bz, X2::pk(drz0, drz1))));
            const int64_t o = (int64_t)(x0 + k + H) * pl + own[h];
            if (yok[h] && zok1) {
              SC_DCHECK(o >= 0 && o + 1 < C1.ext[0] * C1.ext[1] * C1.ext[2]);
              *reinterpret_cast<uint64_t *>(PG.gp + o) = gp;
              *reinterpret_cast<uint64_t *>(PG.gr + o) = gr;
            } else if (yok[h] && zok0) {
              SC_DCHECK(o >= 0 && o < C1.ext[0] * C1.ext[1] * C1.ext[2]);
              PG.gp[o] = X2::lo(gp);
              PG.gr[o] = X2::lo(gr);
            }
          }
          __syncwarp();
          if (lane == 0) {
            sts_release_cta(s_done1 + wi, ++done);
            mbar_arrive(empty_a1 + sa);
            mbar_arrive(empty_r + sc);
          }
          if (++sa == DA1) { sa = 0; pa ^= 1; }
        } else if (j >= R) {
          __syncwarp();
          if (lane == 0) mbar_arrive(empty_r + sc);
        }
        if (++sj == DR) { sj = 0; ph ^= 1; }
      }
      // the last R planes of the sweep were only queue input: release them
      __syncwarp();
      if (lane == 0) {
#pragma unroll
        for (int q = 1; q <= R; ++q) mbar_arrive(empty_r + wrapi(sj - q, DR));
      }
    }
    return;
  }

  // ---- pass-2 consumers: row 2 w + (lane >> 4), one z pair -----------------
  asm volatile("setmaxnreg.inc.sync.aligned.u32 %0;\n" ::"n"(CPL_RC2));
  {
    const int zc = 2 * (lane & 15), yr = 2 * w + (lane >> 4);
    uint64_t qp[QP], qg[QG], qh[QG];
#pragma unroll
    for (int q = 0; q < QP; ++q) qp[q] = 0;
#pragma unroll
    for (int q = 0; q < QG; ++q) { qg[q] = 0; qh[q] = 0; }
    const int64_t pl = C2.ext[1] * C2.ext[2];
    int sp = 0, php = 0, sg = 0, phg = 0, sa = 0, pha = 0;
    for (int r = 0; r < Q.rounds; ++r) {
      const int t2 = r * NC + cta - LAG;
      const int iy = t2 >= 0 ? t2 / Q.ntz1 : 0, iz = t2 - iy * Q.ntz1;
      if (t2 < 0 || t2 >= NT1 || iy >= Q.nty2 || iz >= Q.ntz2) continue;
      const int y0 = C2.lo[1] + iy * STY, z0 = C2.lo[2] + iz * SZ, x0 = C2.lo[0];
      const int XC = C2.n[0];
      const int ep = z0 & 3, eg = (z0 + H - R) & 3, ea = (z0 + H) & 3;
      const int cp = (yr + H) * RP::W + zc + H + ep;
      const int cg = (yr + R) * RG::W + zc + R + eg;
      const int ca = yr * AX::W + zc + ea;
      const int z = z0 + zc, y = y0 + yr;
      const bool yok = y < C2.lo[1] + C2.n[1];
      const bool ok0 = yok && z < C2.lo[2] + C2.n[2], ok1 = yok && z + 1 < C2.lo[2] + C2.n[2];
      const int64_t own = (int64_t)(y + H) * C2.ext[2] + (z + H);
#pragma unroll 1
      for (int j = 0; j < T; ++j) {
        mbar_wait(full_p + sp, php);
#pragma unroll
        for (int q = 0; q < QP - 1; ++q) qp[q] = qp[q + 1];
        qp[QP - 1] = ld2(pring + sp * RP::PAD + cp);
        const int i = j - 2 * R;
        const bool gin = i >= 0 && i < XC + 2 * R;
        if (gin) {
          mbar_wait(full_g + sg, phg);
          const float *gg = gring + sg * 2 * RG::PAD + cg;
#pragma unroll
          for (int q = 0; q < QG - 1; ++q) { qg[q] = qg[q + 1]; qh[q] = qh[q + 1]; }
          qg[QG - 1] = ld2(gg);
          qh[QG - 1] = ld2(gg + RG::PAD);
        }
        const int k = j - 2 * H;
        const int spc = wrapi(sp - H, DP);
        const int sgc = wrapi(sg - R, DG);
        if (k >= 0) {
          mbar_wait(full_a + sa, pha);
          if (!(Q.dbg & 8)) {
          const float *pc = pring + spc * RP::PAD + cp;
          const float *gcen = gring + sgc * 2 * RG::PAD + cg;
          const float *av = aux + sa * NAUX * AX::TILE + ca;
          const uint64_t th = ld2(av + 7 * AX::TILE), phv = ld2(av + 8 * AX::TILE);
          float ax0, ay0, az0, ax1, ay1, az1;
          dir3(X2::lo(th), X2::lo(phv), ax0, ay0, az0);
          dir3(X2::hi(th), X2::hi(phv), ax1, ay1, az1);
          const uint64_t bx = X2::mul0(X2::pk(ax0, ax1), X2::pk(PU.invh[0], PU.invh[0]));
          const uint64_t by = X2::mul0(X2::pk(ay0, ay1), X2::pk(PU.invh[1], PU.invh[1]));
          const uint64_t bz = X2::mul0(X2::pk(az0, az1), X2::pk(PU.invh[2], PU.invh[2]));
          uint64_t hpx = 0, hrx = 0, hpy = 0, hry = 0;
#pragma unroll
          for (int kk = 1; kk <= R; ++kk) {
            const uint64_t wk = X2::pk(PU.c1[kk - 1], PU.c1[kk - 1]);
            hpx = X2::fma(wk, X2::sub(qg[R + kk], qg[R - kk]), hpx);
            hrx = X2::fma(wk, X2::sub(qh[R + kk], qh[R - kk]), hrx);
            hpy = X2::fma(wk, X2::sub(ld2(gcen + kk * RG::W), ld2(gcen - kk * RG::W)), hpy);
            hry = X2::fma(wk, X2::sub(ld2(gcen + RG::PAD + kk * RG::W),
                                      ld2(gcen + RG::PAD - kk * RG::W)), hry);
          }
          float gw[2 * NGW], hw[2 * NGW];
#pragma unroll
          for (int jj = 0; jj < NGW; ++jj) {
            const uint64_t a = ld2(gcen + 2 * jj - RE), b = ld2(gcen + RG::PAD + 2 * jj - RE);
            gw[2 * jj] = X2::lo(a); gw[2 * jj + 1] = X2::hi(a);
            hw[2 * jj] = X2::lo(b); hw[2 * jj + 1] = X2::hi(b);
          }
          float hpz0 = 0.f, hpz1 = 0.f, hrz0 = 0.f, hrz1 = 0.f;
#pragma unroll
          for (int kk = 1; kk <= R; ++kk) {
            const float wk = PU.c1[kk - 1];
            hpz0 = fmaf(wk, gw[RE + kk] - gw[RE - kk], hpz0);
            hpz1 = fmaf(wk, gw[RE + 1 + kk] - gw[RE + 1 - kk], hpz1);
            hrz0 = fmaf(wk, hw[RE + kk] - hw[RE - kk], hrz0);
            hrz1 = fmaf(wk, hw[RE + 1 + kk] - hw[RE + 1 - kk], hrz1);
          }
          const uint64_t hzp = X2::fma(bx, hpx, X2::fma(by, hpy, X2::mul0(bz, X2::pk(hpz0, hpz1))));
          const uint64_t hzr = X2::fma(bx, hrx, X2::fma(by, hry, X2::mul0(bz, X2::pk(hrz0, hrz1))));
          const uint64_t p0 = qp[H];
          uint64_t lx = X2::mul0(X2::pk(PU.c2[0], PU.c2[0]), p0), ly = lx;
#pragma unroll
          for (int kk = 1; kk <= H; ++kk) {
            const uint64_t wk = X2::pk(PU.c2[kk], PU.c2[kk]);
            lx = X2::fma(wk, X2::add(qp[H + kk], qp[H - kk]), lx);
            ly = X2::fma(wk, X2::add(ld2(pc + kk * RP::W), ld2(pc - kk * RP::W)), ly);
          }
          float pw[2 * NPW];
#pragma unroll
          for (int jj = 0; jj < NPW; ++jj) {
            const uint64_t a = (2 * jj == H) ? p0 : ld2(pc + 2 * jj - H);
            pw[2 * jj] = X2::lo(a); pw[2 * jj + 1] = X2::hi(a);
          }
          float lz0 = PU.c2[0] * pw[H], lz1 = PU.c2[0] * pw[H + 1];
#pragma unroll
          for (int kk = 1; kk <= H; ++kk) {
            lz0 = fmaf(PU.c2[kk], pw[H + kk] + pw[H - kk], lz0);
            lz1 = fmaf(PU.c2[kk], pw[H + 1 + kk] + pw[H + 1 - kk], lz1);
          }
          const uint64_t lap =
              X2::fma(lx, X2::pk(PU.invh2[0], PU.invh2[0]),
                      X2::fma(ly, X2::pk(PU.invh2[1], PU.invh2[1]),
                              X2::mul0(X2::pk(lz0, lz1), X2::pk(PU.invh2[2], PU.invh2[2]))));
          const uint64_t hxy = X2::sub(lap, hzp);
          const uint64_t A2 = ld2(av + 3 * AX::TILE), Ec = ld2(av + 4 * AX::TILE);
          const uint64_t Sc = ld2(av + 5 * AX::TILE), Ic = ld2(av + 6 * AX::TILE);
          const uint64_t r0 = ld2(av), pm = ld2(av + 1 * AX::TILE), rm = ld2(av + 2 * AX::TILE);
          const uint64_t pn = X2::fma(A2, X2::sub(p0, pm), X2::fma(Ec, hxy, X2::fma(Sc, hzr, pm)));
          const uint64_t rn = X2::fma(A2, X2::sub(r0, rm), X2::fma(Sc, hxy, X2::fma(Ic, hzr, rm)));
          const int64_t o = (int64_t)(x0 + k + H) * pl + own;
          if (ok1) {
            SC_DCHECK(o >= 0 && o + 1 < C2.ext[0] * C2.ext[1] * C2.ext[2]);
            *reinterpret_cast<uint64_t *>(PU.pn + o) = pn;
            *reinterpret_cast<uint64_t *>(PU.rn + o) = rn;
          } else if (ok0) {
            SC_DCHECK(o >= 0 && o < C2.ext[0] * C2.ext[1] * C2.ext[2]);
            PU.pn[o] = X2::lo(pn);
            PU.rn[o] = X2::lo(rn);
          }
          }
          __syncwarp();
          if (lane == 0) {
            mbar_arrive(empty_a + sa);
            mbar_arrive(empty_p + spc);
            mbar_arrive(empty_g + sgc);
          }
          if (++sa == DA) { sa = 0; pha ^= 1; }
        } else {
          __syncwarp();
          if (lane == 0) {
            if (j >= H) mbar_arrive(empty_p + spc);
            if (i >= R && i - R < XC + 2 * R) mbar_arrive(empty_g + sgc);
          }
        }
        if (++sp == DP) { sp = 0; php ^= 1; }
        if (gin && ++sg == DG) { sg = 0; phg ^= 1; }
      }
      // the last H p planes and R g planes were only queue input: release them
      __syncwarp();
      if (lane == 0) {
#pragma unroll
        for (int q = 1; q <= H; ++q) mbar_arrive(empty_p + wrapi(sp - q, DP));
#pragma unroll
        for (int q = 1; q <= R; ++q) mbar_arrive(empty_g + wrapi(sg - q, DG));
      }
    }
  }
}

template <int SO> struct TSmem {
  static constexpr int R = SO / 4, H = SO / 2;
  static constexpr size_t G = (size_t)4 * ((R + 1 + SPF) * 2 * Ring<2, R>::PAD +
                                           (1 + SPF) * 2 * AuxTile<2>::TILE) +
                              16 * ((R + 1 + SPF) + (1 + SPF));
  static constexpr int PF = spf_u(SO);
  static constexpr size_t U = (size_t)4 * ((H + 1 + PF) * Ring<1, H>::PAD +
                                           (R + 1 + PF) * 2 * Ring<2, R>::PAD +
                                           (1 + PF) * 9 * AuxTile<9>::TILE) +
                              16 * ((H + 1 + PF) + (R + 1 + PF) + (1 + PF));
};

// x planes per CTA: fill whole waves of resident CTAs, keep the re-streamed
// halo small, and on long grids keep chunks short. Sweeps of more than a few
// hundred planes let neighbouring CTAs drift apart in x until their shared
// halo rows have left L2 (config 5, 1616 planes, TTI so=12: whole sweeps 60.2
// GPts/s, 808-plane chunks 60.9, 404 63.5, 202 64.8, 101 65.2; config 3's 592
// planes show no such effect, profiles/r02_xchunk.md).
constexpr int TTI_LONG_X = 640, TTI_CHUNK_CAP = 208;
int xchunks(int n0, int64_t tiles, int sms, int halo) {
  int best = 1;
  double bs = -1.0;
  for (int c = 1; c <= 32 && c <= std::max(1, n0 / std::max(8, 4 * halo)); ++c) {
    const int xc = (n0 + c - 1) / c;
    const int64_t ctas = tiles * ((n0 + xc - 1) / xc);
    const double waves = (double)ctas / sms;
    const double drift = (n0 > TTI_LONG_X && xc > TTI_CHUNK_CAP) ? 0.9 : 1.0;
    const double s = drift * waves / std::ceil(waves) * xc / (double)(xc + halo);
    if (s > bs + 1e-9) { bs = s; best = c; }
  }
  return (n0 + best - 1) / best;
}

}  // namespace

// Per-apply prologue of the TMA path: the time-invariant per-point
// coefficients of the p/r updates (hoistable, as the
// oracle's advanced mode hoists them), computed in double and rounded once:
//   I = 1/(m/dt^2 + damp/(2dt)), 2a = 2 (m/dt^2) I, E = (1+2eps) I,
//   S = sqrt(1+2delta) I
// so that p+ = p- + 2a (p - p-) + E Hxy(p) + S Hz(r) and
// r+ = r- + 2a (r - r-) + S Hxy(p) + I Hz(r) (same update, reassociated).
__global__ void tti_hoist(const float *__restrict__ m, const float *__restrict__ damp,
                          const float *__restrict__ eps, const float *__restrict__ delta,
                          float *__restrict__ a2, float *__restrict__ ec, float *__restrict__ sc,
                          float *__restrict__ ic, int64_t n, double dt2inv, double dtinv2) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n;
       i += (int64_t)gridDim.x * blockDim.x) {
    const double am = (double)m[i] * dt2inv, ad = (double)damp[i] * dtinv2;
    const double inv = 1.0 / (am + ad);
    a2[i] = (float)(2.0 * am * inv);
    ec[i] = (float)((1.0 + 2.0 * (double)eps[i]) * inv);
    sc[i] = (float)(sqrt(1.0 + 2.0 * (double)delta[i]) * inv);
    ic[i] = (float)inv;
  }
}

int tti_prologue(const sc_dense &d, const FieldDev *fields, cudaStream_t st) {
  if (d.fast_kind != SC_FAST_TTI || !d.scratch[2]) return 0;
  const FieldDev &fp = fields[d.tti_fields[0]];  // p: (slots, x, y, z)
  const int64_t n = fp.ext[1] * fp.ext[2] * fp.ext[3];
  auto F = [&](int i) { return reinterpret_cast<const float *>(fields[d.tti_fields[i]].data); };
  auto S = [&](int i) { return reinterpret_cast<float *>(d.scratch[i]); };
  tti_hoist<<<148 * 8, 256, 0, st>>>(F(2), F(3), F(4), F(5), S(2), S(3), S(4), S(5), n,
                                     d.fast_consts[6], d.fast_consts[7]);
  SC_CUDA(cudaGetLastError());
  return 0;
}

// TMA two-pass launch (f32); 1 = not applicable (caller uses the plain pair)
// Per-stage launch configuration of the TMA two-pass path (see tti_tma_launch)
struct TtiSig {
  void *p[14];
  int64_t ext[4];
  int lo[3], hi[3], so, xblock, variant;
  double k[22];
};

struct TtiCfg {
  TtiSig sig;
  GMaps gm;
  UMaps um;
  GMaps2 gm2;
  UMaps2 um2;
  GParams G;
  UParams U;
  int64_t slot = 0;
  const void *kg = nullptr, *ku = nullptr;
  dim3 grid, block, gridu, blocku;
  size_t smg = 0, smu = 0;
  void *gmaps = nullptr, *umaps = nullptr;
  // coupled single launch (tti_cpl_tma): both passes, g through L2
  bool cpl = false;
  const void *kc = nullptr;
  size_t smc = 0;
  int ncta = 0;
  CplParams Q;
  std::shared_ptr<int> prog;  // device counters, freed with the entry
};

// Launch configurations (tensor maps, kernel choice, geometry) per prepared
// TTI stage and x range, built on first use. Keyed by the stage's address in
// its Run's plan copy; tti_forget drops a Run's entries when it is released.
// Guarded: ctypes callers release the GIL.
using TtiCache = std::map<std::tuple<const sc_dense *, int, int>, TtiCfg>;
TtiCache &tti_cache() {
  static TtiCache c;
  return c;
}
std::mutex &tti_cache_mu() {
  static std::mutex m;
  return m;
}

// the experiment switches that change the kernel choice (part of the key so
// an in-process A/B never reuses a stale choice)
int tti_variant_flags() {
  const char *names[] = {"SC_TTI_U1", "SC_TTI_NOZP", "SC_TTI_X2", "SC_TTI_G1ROT", "SC_TTI_G1S",
                         "SC_TTI_COUPLED", "SC_TTI_LEAD", "SC_TTI_CPLDBG", "SC_XBLOCK", "SC_TTI_NOTAIL"};
  int v = 0;
  for (int i = 0; i < (int)(sizeof(names) / sizeof(names[0])); ++i)
    if (getenv(names[i])) v |= 1 << i;
  return v;
}

// the two passes of step t from a built configuration: only the time slots
// change from step to step
int tti_cfg_launch(TtiCfg &c, const FieldDev *fields, const sc_dense &d, int t,
                   cudaStream_t st) {
  const FieldDev &fp = fields[d.tti_fields[0]];
  c.G.cur = c.U.cur = sc_slot(t, 3);
  c.U.prev = sc_slot(t - 1, 3);
  c.U.pn = reinterpret_cast<float *>(fp.data) + sc_slot(t + 1, 3) * c.slot;
  c.U.rn = reinterpret_cast<float *>(fields[d.tti_fields[1]].data) + sc_slot(t + 1, 3) * c.slot;
  if (c.cpl) {
    SC_CUDA(cudaMemsetAsync(c.Q.prog, 0, sizeof(int) * (size_t)c.Q.nty1 * c.Q.ntz1, st));
    void *ca[] = {(void *)&c.gm, (void *)&c.um, (void *)&c.G, (void *)&c.U, (void *)&c.Q};
    SC_CUDA(cudaLaunchKernel(c.kc, dim3(c.ncta), dim3(SZ, 16, 1), ca, c.smc, st));
    return 0;
  }
  void *ga[] = {c.gmaps, (void *)&c.G};
  SC_CUDA(cudaLaunchKernel(c.kg, c.grid, c.block, ga, c.smg, st));
  void *ua[] = {c.umaps, (void *)&c.U};
  SC_CUDA(cudaLaunchKernel(c.ku, c.gridu, c.blocku, ua, c.smu, st));
  return 0;
}

bool tti_tma_ok(const sc_dense &d, const FieldDev *fields) {
  const FieldDev &fp = fields[d.tti_fields[0]];
  return (fp.ext[3] * 4) % 16 == 0 && d.so >= 4 && d.so <= 16 && d.so % 4 == 0 &&
         d.scratch[2] != nullptr && !getenv("SC_TTI_PLAIN") && !getenv("SC_TTI_FUSED");
}

// x_lo..x_hi (loop coordinates, default: the plan's box) restricts the step
// to a slab of x planes (multi-GPU boundary/interior parts, sc_step_part)
int tti_tma_launch(const sc_plan *pl, const sc_dense &d, const FieldDev *fields, int t,
                   cudaStream_t st, int x_lo, int x_hi) {
  const int so = d.so, H = so / 2, R = so / 4;
  const FieldDev &fp = fields[d.tti_fields[0]];
  if ((fp.ext[3] * 4) % 16 != 0 || so < 4 || so > 16 || so % 4 || !d.scratch[2]) return 1;
  const int xl = x_lo == INT_MIN ? pl->lo[0] : x_lo;
  const int xh = x_hi == INT_MIN ? pl->hi[0] : x_hi;
  // tensor maps, kernel choice and launch geometry depend only on the stage
  // and its buffers: built once per prepared stage, reused every step
  // (host-driven step loops issue a TTI step in microseconds)
  std::lock_guard<std::mutex> lock(tti_cache_mu());
  auto &cache = tti_cache();
  const auto key = std::make_tuple(&d, xl, xh);
  TtiSig sig;
  memset(&sig, 0, sizeof(sig));
  sig.variant = tti_variant_flags();
  for (int i = 0; i < 8; ++i) sig.p[i] = fields[d.tti_fields[i]].data;
  for (int i = 0; i < 6; ++i) sig.p[8 + i] = d.scratch[i];
  for (int k = 0; k < 4; ++k) sig.ext[k] = fp.ext[k];
  for (int k = 0; k < 3; ++k) {
    sig.lo[k] = k ? pl->lo[k] : xl;
    sig.hi[k] = k ? pl->hi[k] : xh;
  }
  sig.so = so;
  sig.xblock = d.xblock;
  for (int k = 0; k < 22; ++k) sig.k[k] = d.fast_consts[k];
  auto hit = cache.find(key);
  if (hit != cache.end() && memcmp(&hit->second.sig, &sig, sizeof(sig)) == 0)
    return tti_cfg_launch(hit->second, fields, d, t, st);
  TtiCfg &c = cache[key];
  c = TtiCfg();
  c.sig = sig;
  struct Drop {  // a failed build must not leave a half-filled entry
    TtiCache &m;
    std::tuple<const sc_dense *, int, int> key;
    bool ok = false;
    ~Drop() {
      if (!ok) m.erase(key);
    }
  } drop{cache, key};
  const uint64_t Z = fp.ext[3], Y = fp.ext[2], Xs = fp.ext[1];
  uint64_t strides[2] = {Z * 4, Z * Y * 4};
  uint64_t dt_[3] = {Z, Y, Xs * 3}, df[3] = {Z, Y, Xs};
  auto F = [&](int i) { return fields[d.tti_fields[i]].data; };
  auto Wd = [](int halo) { return (uint32_t)(((32 + 2 * halo + 3 + 7) / 8) * 8); };
  const uint32_t WA = (uint32_t)(((32 + 3 + 7) / 8) * 8);
  uint32_t bg_r[3] = {Wd(R), (uint32_t)(STY + 2 * R), 1};
  uint32_t bu_p[3] = {Wd(H), (uint32_t)(STY + 2 * H), 1};
  uint32_t b_a[3] = {WA, (uint32_t)STY, 1};
  GMaps &gm = c.gm;
  UMaps &um = c.um;
  if (sc_encode_tmap(&gm.p, F(0), 4, dt_, strides, bg_r) ||
      sc_encode_tmap(&gm.r, F(1), 4, dt_, strides, bg_r) ||
      sc_encode_tmap(&gm.th, F(6), 4, df, strides, b_a) ||
      sc_encode_tmap(&gm.ph, F(7), 4, df, strides, b_a) ||
      sc_encode_tmap(&um.p, F(0), 4, dt_, strides, bu_p) ||
      sc_encode_tmap(&um.gp, d.scratch[0], 4, df, strides, bg_r) ||
      sc_encode_tmap(&um.gr, d.scratch[1], 4, df, strides, bg_r) ||
      sc_encode_tmap(&um.r, F(1), 4, dt_, strides, b_a) ||
      sc_encode_tmap(&um.pm, F(0), 4, dt_, strides, b_a) ||
      sc_encode_tmap(&um.rm, F(1), 4, dt_, strides, b_a) ||
      sc_encode_tmap(&um.m, d.scratch[2], 4, df, strides, b_a) ||
      sc_encode_tmap(&um.damp, d.scratch[3], 4, df, strides, b_a) ||
      sc_encode_tmap(&um.eps, d.scratch[4], 4, df, strides, b_a) ||
      sc_encode_tmap(&um.delta, d.scratch[5], 4, df, strides, b_a) ||
      sc_encode_tmap(&um.th, F(6), 4, df, strides, b_a) ||
      sc_encode_tmap(&um.ph, F(7), 4, df, strides, b_a))
    return -1;
  static int sms = 0;
  if (!sms) {
    int dev = 0;
    SC_CUDA(cudaGetDevice(&dev));
    SC_CUDA(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev));
  }
  const double *kc = d.fast_consts;
  GParams &G = c.G;
  UParams &U = c.U;
  for (int k = 0; k < 3; ++k) {
    G.c.ext[k] = U.c.ext[k] = fp.ext[1 + k];
    // pass 1 covers the loop box widened by R, pass 2 the loop box
    const int lo = k ? pl->lo[k] : xl, hi = k ? pl->hi[k] : xh;
    G.c.lo[k] = lo - R;
    G.c.n[k] = hi - lo + 1 + 2 * R;
    U.c.lo[k] = lo;
    U.c.n[k] = hi - lo + 1;
    G.invh[k] = U.invh[k] = (float)kc[k];
    U.invh2[k] = (float)kc[3 + k];
  }
  G.c.H = U.c.H = H;
  U.dt2inv = (float)kc[6];
  U.dtinv2 = (float)kc[7];
  for (int k = 0; k < 4; ++k) G.c1[k] = U.c1[k] = (float)kc[8 + k];
  for (int k = 0; k < 9; ++k) U.c2[k] = (float)kc[13 + k];
  const int64_t slot = fp.ext[1] * fp.ext[2] * fp.ext[3];
  G.gp = reinterpret_cast<float *>(d.scratch[0]);
  G.gr = reinterpret_cast<float *>(d.scratch[1]);
  c.slot = slot;
  const void *kg = nullptr, *ku = nullptr;
  size_t smg = 0, smu = 0;
  const bool xb = so <= 12 && !getenv("SC_TTI_U1");  // x-blocked pass 2
  // z-pair pass 2: even z origin and row length keep every operand pair and
  // output pair 8-byte aligned
  const bool zp3 = xb && (so / 2) % 2 == 0 && pl->lo[2] % 2 == 0 && Z % 2 == 0 &&
                   !getenv("SC_TTI_NOZP");
  UMaps2 &um2 = c.um2;
  if (xb) {
    uint32_t b2p[3] = {Wd(H), (uint32_t)(16 + 2 * H), 2};
    uint32_t b2g[3] = {Wd(R), (uint32_t)(16 + 2 * R), 2};
    uint32_t b2a[3] = {WA, 16u, 2};
    if (sc_encode_tmap(&um2.p, F(0), 4, dt_, strides, b2p) ||
        sc_encode_tmap(&um2.gp, d.scratch[0], 4, df, strides, b2g) ||
        sc_encode_tmap(&um2.gr, d.scratch[1], 4, df, strides, b2g) ||
        sc_encode_tmap(&um2.a[0], F(1), 4, dt_, strides, b2a) ||
        sc_encode_tmap(&um2.a[1], F(0), 4, dt_, strides, b2a) ||
        sc_encode_tmap(&um2.a[2], F(1), 4, dt_, strides, b2a))
      return -1;
    for (int f = 3; f < 9; ++f)
      if (sc_encode_tmap(&um2.a[f], f < 7 ? d.scratch[f - 1] : F(f - 1), 4, df, strides, b2a))
        return -1;
  }
  switch (so) {
#define SC_T(S)                                                        \
  case S:                                                              \
    kg = reinterpret_cast<const void *>(&tti_g_tma<S>);                \
    ku = reinterpret_cast<const void *>(&tti_upd_tma<S>);              \
    smg = TSmem<S>::G;                                                 \
    smu = TSmem<S>::U;                                                 \
    break;
    SC_T(4) SC_T(8) SC_T(12) SC_T(16)
#undef SC_T
  }
  // pass 1 is x-blocked for every order (so 16 included: 113 KB, two CTAs
  // per SM); z-pairs when the z origin and row length are even
  const bool xg = !getenv("SC_TTI_U1");
  const bool gz = xg && (so / 2) % 2 == 0 && pl->lo[2] % 2 == 0 && Z % 2 == 0 &&
                  !getenv("SC_TTI_NOZP");
  GMaps2 &gm2 = c.gm2;
  if (xg) {
    uint32_t b2r[3] = {Wd(R), (uint32_t)(STY + 2 * R), 2};
    uint32_t b2t[3] = {WA, (uint32_t)STY, 2};
    if (sc_encode_tmap(&gm2.p, F(0), 4, dt_, strides, b2r) ||
        sc_encode_tmap(&gm2.r, F(1), 4, dt_, strides, b2r) ||
        sc_encode_tmap(&gm2.th, F(6), 4, df, strides, b2t) ||
        sc_encode_tmap(&gm2.ph, F(7), 4, df, strides, b2t))
      return -1;
    switch (so) {
#define SC_G2(S)                                                       \
  case S:                                                              \
    kg = gz ? reinterpret_cast<const void *>(&tti_g3_tma<S>)           \
            : reinterpret_cast<const void *>(&tti_g2_tma<S>);          \
    smg = G2Geo<S>::SMEM;                                              \
    break;
      SC_G2(4) SC_G2(8) SC_G2(12) SC_G2(16)
#undef SC_G2
    }
  }
  if (xb) {
    switch (so) {
#define SC_T2(S)                                                       \
  case S:                                                              \
    ku = zp3 ? reinterpret_cast<const void *>(&tti_upd3_tma<S>)        \
             : reinterpret_cast<const void *>(&tti_upd2_tma<S>);       \
    smu = U2Geo<S>::SMEM;                                              \
    break;
      SC_T2(4) SC_T2(8) SC_T2(12)
#undef SC_T2
    }
  }
  // pass 1 likewise: one-plane z-pair rings (SC_TTI_X2=1: x-blocked tti_g3_tma)
  const bool g1z = gz && !getenv("SC_TTI_X2");
  // default: shifting queue, three planes ahead. The rotating queue
  // (SC_TTI_G1ROT=1, + SC_TTI_G1S=1 for three planes) is 1-2 % faster on
  // config 3 but 8 % slower on the config-5 slab path (56.8 vs 61.6 GPts/s)
  const bool g1q = getenv("SC_TTI_G1ROT") == nullptr;
  const bool g1s = getenv("SC_TTI_G1S") != nullptr;
  if (g1z) {
    switch (so) {
#define SC_G1Z(S)                                                                       \
  if (g1q) {                                                                            \
    kg = reinterpret_cast<const void *>(&tti_g1z_tma<S, false, SPF>);                   \
    smg = G1zSmem<S, SPF>::B;                                                           \
  } else if (g1s) {                                                                     \
    kg = reinterpret_cast<const void *>(&tti_g1z_tma<S, true, SPF>);                    \
    smg = G1zSmem<S, SPF>::B;                                                           \
  } else {                                                                              \
    kg = reinterpret_cast<const void *>(&tti_g1z_tma<S, true, g1z_pf(S)>);              \
    smg = G1zSmem<S, g1z_pf(S)>::B;                                                     \
  }                                                                                     \
  break;
      case 4: SC_G1Z(4)
      case 8: SC_G1Z(8)
      case 12: SC_G1Z(12)
      default: SC_G1Z(16)
#undef SC_G1Z
    }
  }
  // so 16: one-plane pass 2 on z-pairs when the z origin and rows allow
  // The one-plane z-pair pass 2 is the default for every even halo: its
  // single-plane rings run further ahead than the two-plane slots of
  // tti_upd3_tma (so 8: 61.7 vs 59.0 GPts/s, so 12: 55.1 vs 54.9, A/B);
  // SC_TTI_X2=1 selects tti_upd3_tma
  const bool u1z = (!xb || !getenv("SC_TTI_X2")) && (so / 2) % 2 == 0 &&
                   pl->lo[2] % 2 == 0 && Z % 2 == 0 && !getenv("SC_TTI_NOZP");
  if (u1z) {
    switch (so) {
      case 4: ku = reinterpret_cast<const void *>(&tti_upd1z_tma<4>); smu = TSmem<4>::U; break;
      case 8: ku = reinterpret_cast<const void *>(&tti_upd1z_tma<8>); smu = TSmem<8>::U; break;
      case 12: ku = reinterpret_cast<const void *>(&tti_upd1z_tma<12>); smu = TSmem<12>::U; break;
      default: ku = reinterpret_cast<const void *>(&tti_upd1z_tma<16>); smu = TSmem<16>::U; break;
    }
  }
  const bool ub = xb && !u1z;  // x-blocked pass 2 (um2 maps, 2-plane pairs)
  if (smg > 227 * 1024 || smu > 227 * 1024) return 1;
  SC_CUDA(cudaFuncSetAttribute(kg, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smg));
  SC_CUDA(cudaFuncSetAttribute(ku, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smu));
  int occg = 1, occu = 1;
  SC_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occg, kg, SZ * (SBY + 1), smg));
  if (getenv("SC_TTI_DEBUG")) fprintf(stderr, "tti pass 1: %zu B smem, %d CTAs/SM\n", smg, occg);
  const int nwu = u1z ? SBY : zp3 ? 8 : xb ? 16 : UBY;
  SC_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occu, ku, SZ * (nwu + 1), smu));
  dim3 block(SZ, SBY + 1, 1);
  if (gz && (R & 1)) {
    // z-pair pass 1 starts its (widened) box on an even z: one extra column
    // of g below lo - R (inside the halo, never read by pass 2)
    G.c.lo[2] -= 1;
    G.c.n[2] += 1;
  }
  {
    const int64_t tiles = sc_ceil_div(G.c.n[1], STY) * sc_ceil_div(G.c.n[2], SZ);
    G.c.xchunk = d.xblock > 0 ? std::min(d.xblock, std::max(G.c.n[0], 1))
                              : xchunks(G.c.n[0], tiles, sms * std::max(occg, 1), R);
    if (getenv("SC_XBLOCK")) G.c.xchunk = std::max(1, std::min(atoi(getenv("SC_XBLOCK")), G.c.n[0]));
    if (xg && !g1z) G.c.xchunk += G.c.xchunk & 1;  // whole output pairs per chunk
    dim3 grid((unsigned)sc_ceil_div(G.c.n[2], SZ), (unsigned)sc_ceil_div(G.c.n[1], STY),
              (unsigned)sc_ceil_div(G.c.n[0], G.c.xchunk));
    c.kg = kg;
    c.grid = grid;
    c.block = block;
    c.smg = smg;
    c.gmaps = xg && !g1z ? (void *)&gm2 : (void *)&gm;
  }
  {
    const int64_t tiles = sc_ceil_div(U.c.n[1], STY) * sc_ceil_div(U.c.n[2], SZ);
    U.c.xchunk = d.xblock > 0 ? std::min(d.xblock, std::max(U.c.n[0], 1))
                              : xchunks(U.c.n[0], tiles, sms * std::max(occu, 1), H);
    if (getenv("SC_XBLOCK")) U.c.xchunk = std::max(1, std::min(atoi(getenv("SC_XBLOCK")), U.c.n[0]));
    if (ub) U.c.xchunk += U.c.xchunk & 1;  // whole output pairs per chunk
    dim3 gridu((unsigned)sc_ceil_div(U.c.n[2], SZ), (unsigned)sc_ceil_div(U.c.n[1], STY),
               (unsigned)sc_ceil_div(U.c.n[0], U.c.xchunk));
    // Whole sweeps leave a partly filled last wave (config 3: 703 tiles on
    // 148 one-CTA SMs = 4.75 waves), equal x chunks pay the 2H-plane prologue
    // on every tile. Tail split: whole sweeps on the tiles of the full waves,
    // the tiles of the last wave cut into q x chunks each, q minimising
    // (waves of the tail) x (chunk + prologue). Config 3: 592 whole sweeps +
    // 111 tiles x 4 chunks, 62.2 vs 61.4 GPts/s with four equal chunks (A/B
    // twice on one box); SC_TTI_NOTAIL=1 keeps the equal chunks.
    U.c.tailq = 0;
    const int64_t slots = (int64_t)sms * std::max(occu, 1);
    if (u1z && d.xblock <= 0 && !getenv("SC_XBLOCK") && !getenv("SC_TTI_NOTAIL") &&
        U.c.n[0] <= TTI_LONG_X && tiles > slots && tiles % slots != 0) {
      const int64_t nwhole = tiles / slots * slots, tail = tiles - nwhole;
      int bestq = 1;
      double bestt = 1.0;
      for (int q = 2; q <= 8 && U.c.n[0] / q >= 4 * H; ++q) {
        const double len = (double)sc_ceil_div(U.c.n[0], q) + 2 * H;
        const double t = (double)sc_ceil_div(tail * q, slots) * len / (U.c.n[0] + 2 * H);
        if (t < bestt - 1e-9) {
          bestt = t;
          bestq = q;
        }
      }
      if (bestq > 1) {
        U.c.xchunk = U.c.n[0];
        U.c.nwhole = (int)nwhole;
        U.c.tailq = bestq;
        U.c.ntz = (int)sc_ceil_div(U.c.n[2], SZ);
        gridu = dim3((unsigned)(nwhole + tail * bestq), 1, 1);
        if (getenv("SC_TTI_DEBUG"))
          fprintf(stderr, "tti pass 2: %lld whole sweeps + %lld tiles x %d chunks\n",
                  (long long)nwhole, (long long)tail, bestq);
      }
    }
    c.ku = ku;
    c.gridu = gridu;
    c.blocku = dim3(SZ, nwu + 1, 1);
    c.smu = smu;
    c.umaps = ub ? (void *)&um2 : (void *)&um;
  }
  // SC_TTI_COUPLED=1: both passes in one persistent launch (so 4/8/12 on the
  // default z-pair kernels), g from pass 1 to pass 2 through L2. Bitwise equal
  // to the two launches but 2.5x slower (profiles/r02_tti_coupled.md), so the
  // two launches stay the default.
  if (g1z && g1q && u1z && so <= 12 && getenv("SC_TTI_COUPLED")) {
    const void *kc = nullptr;
    size_t smc = 0;
    switch (so) {
      case 4: kc = reinterpret_cast<const void *>(&tti_cpl_tma<4, 3, 3, 3>); smc = CplGeo<4, 3, 3, 3>::SMEM; break;
      case 8: kc = reinterpret_cast<const void *>(&tti_cpl_tma<8, 3, 3, 3>); smc = CplGeo<8, 3, 3, 3>::SMEM; break;
      default: kc = reinterpret_cast<const void *>(&tti_cpl_tma<12, 2, 2, 1>); smc = CplGeo<12, 2, 2, 1>::SMEM; break;
    }
    int occ = 0;
    if (smc <= 227 * 1024) {
      SC_CUDA(cudaFuncSetAttribute(kc, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smc));
      SC_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, kc, SZ * 16, smc));
    }
    if (occ >= 1) {
      CplParams &Q = c.Q;
      Q.nty1 = (int)sc_ceil_div(G.c.n[1], STY);
      Q.ntz1 = (int)sc_ceil_div(G.c.n[2], SZ);
      Q.nty2 = (int)sc_ceil_div(U.c.n[1], STY);
      Q.ntz2 = (int)sc_ceil_div(U.c.n[2], SZ);
      const int nt1 = Q.nty1 * Q.ntz1;
      c.ncta = std::min(sms, nt1 + Q.ntz1 + 1);
      Q.rounds = (int)sc_ceil_div(nt1 + Q.ntz1 + 1, c.ncta);
      const char *ld = getenv("SC_TTI_LEAD");
      Q.lead = ld ? std::max(8, atoi(ld)) : 12;
      Q.dbg = getenv("SC_TTI_CPLDBG") ? atoi(getenv("SC_TTI_CPLDBG")) : 0;
      int *prog = nullptr;
      {
        // a prepared run builds this inside a thread-local stream capture
        cudaStreamCaptureMode mode = cudaStreamCaptureModeRelaxed;
        SC_CUDA(cudaThreadExchangeStreamCaptureMode(&mode));
        const cudaError_t e = cudaMalloc((void **)&prog, sizeof(int) * (size_t)nt1);
        cudaThreadExchangeStreamCaptureMode(&mode);
        SC_CUDA(e);
      }
      c.prog = std::shared_ptr<int>(prog, [](int *q) { cudaFree(q); });
      Q.prog = prog;
      c.kc = kc;
      c.smc = smc;
      c.cpl = true;
      if (getenv("SC_TTI_DEBUG"))
        fprintf(stderr, "tti coupled: %zu B smem, %d CTAs, %d x %d pass-1 tiles, %d rounds, lead %d\n",
                smc, c.ncta, Q.nty1, Q.ntz1, Q.rounds, Q.lead);
    }
  }
  drop.ok = true;
  return tti_cfg_launch(c, fields, d, t, st);
}

// drop the cached launch configurations of a released run's TTI stages
void tti_forget(const sc_dense *first, int n) {
  std::lock_guard<std::mutex> lock(tti_cache_mu());
  auto &cache = tti_cache();
  for (auto it = cache.begin(); it != cache.end();) {
    const sc_dense *d = std::get<0>(it->first);
    if (d >= first && d < first + n)
      it = cache.erase(it);
    else
      ++it;
  }
}
