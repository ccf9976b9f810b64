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

template <typename T, int SO>
__global__ void __launch_bounds__(BZ *BYT) tti_inner(const TtiArgs<T> a) {
  constexpr int R = SO / 4 > 0 ? SO / 4 : 1;
  const int z = a.lo[2] - R + blockIdx.x * BZ + threadIdx.x;
  const int y = a.lo[1] - R + blockIdx.y * BYT + threadIdx.y;
  const int x = a.lo[0] - R + blockIdx.z;
  if (z > a.hi[2] + R || y > a.hi[1] + R) return;
  const int H = a.H;
  const int64_t sx = a.E1 * a.E2, sy = a.E2;
  const int64_t c = (int64_t)(x + H) * sx + (int64_t)(y + H) * sy + (z + H);
  T ax, ay, az;
  direction<T>(__ldg(a.theta + c), __ldg(a.phi + c), ax, ay, az);
  T dpx = 0, dpy = 0, dpz = 0, drx = 0, dry = 0, drz = 0;
#pragma unroll
  for (int k = 1; k <= R; ++k) {
    const T w = a.c1[k - 1];
    dpx = fma(w, __ldg(a.p + c + k * sx) - __ldg(a.p + c - k * sx), dpx);
    dpy = fma(w, __ldg(a.p + c + k * sy) - __ldg(a.p + c - k * sy), dpy);
    dpz = fma(w, __ldg(a.p + c + k) - __ldg(a.p + c - k), dpz);
    drx = fma(w, __ldg(a.r + c + k * sx) - __ldg(a.r + c - k * sx), drx);
    dry = fma(w, __ldg(a.r + c + k * sy) - __ldg(a.r + c - k * sy), dry);
    drz = fma(w, __ldg(a.r + c + k) - __ldg(a.r + c - k), drz);
  }
  const T bx = ax * a.invh[0], by = ay * a.invh[1], bz = az * a.invh[2];
  a.gp[c] = fma(bx, dpx, fma(by, dpy, bz * dpz));
  a.gr[c] = fma(bx, drx, fma(by, dry, bz * drz));
}

template <typename T, int SO>
__global__ void __launch_bounds__(BZ *BYT) tti_outer(const TtiArgs<T> a) {
  constexpr int R = SO / 4 > 0 ? SO / 4 : 1;
  constexpr int H = SO / 2;
  const int z = a.lo[2] + blockIdx.x * BZ + threadIdx.x;
  const int y = a.lo[1] + blockIdx.y * BYT + threadIdx.y;
  const int x = a.lo[0] + blockIdx.z;
  if (z > a.hi[2] || y > a.hi[1]) return;
  const int64_t sx = a.E1 * a.E2, sy = a.E2;
  const int64_t c = (int64_t)(x + a.H) * sx + (int64_t)(y + a.H) * sy + (z + a.H);
  T ax, ay, az;
  direction<T>(__ldg(a.theta + c), __ldg(a.phi + c), ax, ay, az);
  // outer rotated derivatives of g_p, g_r
  T hpx = 0, hpy = 0, hpz = 0, hrx = 0, hry = 0, hrz = 0;
#pragma unroll
  for (int k = 1; k <= R; ++k) {
    const T w = a.c1[k - 1];
    hpx = fma(w, __ldg(a.gp + c + k * sx) - __ldg(a.gp + c - k * sx), hpx);
    hpy = fma(w, __ldg(a.gp + c + k * sy) - __ldg(a.gp + c - k * sy), hpy);
    hpz = fma(w, __ldg(a.gp + c + k) - __ldg(a.gp + c - k), hpz);
    hrx = fma(w, __ldg(a.gr + c + k * sx) - __ldg(a.gr + c - k * sx), hrx);
    hry = fma(w, __ldg(a.gr + c + k * sy) - __ldg(a.gr + c - k * sy), hry);
    hrz = fma(w, __ldg(a.gr + c + k) - __ldg(a.gr + c - k), hrz);
  }
  const T bx = ax * a.invh[0], by = ay * a.invh[1], bz = az * a.invh[2];
  const T hzp = fma(bx, hpx, fma(by, hpy, bz * hpz));
  const T hzr = fma(bx, hrx, fma(by, hry, bz * hrz));
  // Laplacian of p
  const T p0 = __ldg(a.p + c);
  T lx = a.c2[0] * p0, ly = a.c2[0] * p0, lz = a.c2[0] * p0;
#pragma unroll
  for (int k = 1; k <= H; ++k) {
    const T w = a.c2[k];
    lx = fma(w, __ldg(a.p + c + k * sx) + __ldg(a.p + c - k * sx), lx);
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

template <typename T, int SO> void launch_pair(const TtiArgs<T> &a, cudaStream_t st) {
  constexpr int R = SO / 4 > 0 ? SO / 4 : 1;
  const int n0 = a.hi[0] - a.lo[0] + 1, n1 = a.hi[1] - a.lo[1] + 1, n2 = a.hi[2] - a.lo[2] + 1;
  dim3 b(BZ, BYT, 1);
  dim3 gi((n2 + 2 * R + BZ - 1) / BZ, (n1 + 2 * R + BYT - 1) / BYT, n0 + 2 * R);
  tti_inner<T, SO><<<gi, b, 0, st>>>(a);
  dim3 go((n2 + BZ - 1) / BZ, (n1 + BYT - 1) / BYT, n0);
  tti_outer<T, SO><<<go, b, 0, st>>>(a);
}

}  // namespace

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
