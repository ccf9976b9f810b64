// C ABI entry points, the generic exact dense-program kernel and the sparse
// (injection / interpolation) kernels. See include/stencil_b200.h for the
// reference interfaces each entry point replaces.
#include <stdarg.h>
#include <string.h>

#include <algorithm>
#include <vector>

#include "common.cuh"
#include "kernels.cuh"

static thread_local char g_err[1024] = "";

void sc_set_error(const char *fmt, ...) {
  va_list ap;
  va_start(ap, fmt);
  vsnprintf(g_err, sizeof(g_err), fmt, ap);
  va_end(ap);
}

extern "C" const char *sc_last_error(void) { return g_err; }
extern "C" int sc_version(void) { return 100; }
extern "C" int64_t sc_plan_size(void) { return (int64_t)sizeof(sc_plan); }

extern "C" int sc_device_count(int *count) {
  SC_CUDA(cudaGetDeviceCount(count));
  return 0;
}

extern "C" int sc_set_device(int device) {
  SC_CUDA(cudaSetDevice(device));
  return 0;
}

// ---------------------------------------------------------------------------
// Generic dense program: one thread per grid point evaluates the straight-line
// program compiled from the oracle's optimized tree (backend/program.py).

__device__ __forceinline__ int64_t field_index(const FieldDev &f, int slot, const int *i,
                                               int ndim) {
  int64_t li = 0;
  int a = 0;
  if (f.has_time) {
    li = slot;
    a = 1;
  }
  for (int d = 0; d < ndim; ++d) li = li * f.ext[a + d] + i[d];
  return li;
}

__device__ __forceinline__ int time_slot(const FieldDev &f, int t) {
  if (!f.has_time) return 0;
  return f.nslots > 0 ? sc_slot(t, f.nslots) : t;
}

template <typename T>
__global__ void __launch_bounds__(256) dense_generic_kernel(DenseArgs<T> a, int t) {
  int64_t n = (int64_t)a.n[0] * a.n[1] * a.n[2];
  int64_t gid = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (gid >= n) return;
  int p[3];
  p[2] = (int)(gid % a.n[2]);
  p[1] = (int)((gid / a.n[2]) % a.n[1]);
  p[0] = (int)(gid / ((int64_t)a.n[2] * a.n[1]));
  int loop[3];
  for (int d = 0; d < 3; ++d) loop[d] = a.lo[d] + p[d];
  T r[SC_GEN_MAXREG];
  for (int k = 0; k < a.nops; ++k) {
    const int4 o = a.ops[k];
    switch (o.x) {
      case SC_LOAD: {
        const LoadDev ld = a.loads[o.z];
        const FieldDev &f = a.fields[ld.field];
        int ii[3];
        for (int d = 0; d < a.ndim; ++d) ii[d] = loop[d] + ld.off[d];
        r[o.y] = reinterpret_cast<const T *>(f.data)[field_index(
            f, time_slot(f, load_time(t, ld.tshift, ld.tdiv)), ii, a.ndim)];
        break;
      }
      case SC_MULK: r[o.y] = X<T>::mul(r[o.z], (T)a.consts[o.w]); break;
      case SC_ADDK: r[o.y] = o.z < 0 ? (T)a.consts[o.w] : X<T>::add(r[o.z], (T)a.consts[o.w]); break;
      case SC_MUL: r[o.y] = X<T>::mul(r[o.z], r[o.w]); break;
      case SC_ADD: r[o.y] = X<T>::add(r[o.z], r[o.w]); break;
      case SC_RCP: r[o.y] = X<T>::rcp(r[o.z]); break;
    }
  }
  const FieldDev &f = a.fields[a.target.field];
  int ii[3];
  for (int d = 0; d < a.ndim; ++d) ii[d] = loop[d] + a.target.off[d];
  reinterpret_cast<T *>(f.data)[field_index(
      f, time_slot(f, load_time(t, a.target.tshift, a.target.tdiv)), ii, a.ndim)] = r[a.out_reg];
}

// ---------------------------------------------------------------------------
// Sparse: per point, corners in the oracle's order; each corner value is the
// ordered product of its factors (reference expr.py:461-465 fold from 1.0).

template <typename T>
__device__ __forceinline__ T corner_value(const SparseArgs<T> &s, int c, int p, int t,
                                          const T *field, const FieldDev &f, int64_t fidx) {
  T v = (T)s.lead[c];
  bool first = true;
  for (int k = 0; k < s.nfac[c]; ++k) {
    T x;
    switch (s.fac_kind[c][k]) {
      case SC_FAC_SPARSE:
        x = s.sparse[(int64_t)(t + s.sparse_tshift) * s.npoint + p];
        break;
      case SC_FAC_TABLE:
        x = s.tables[s.fac_arg[c][k]][p];
        break;
      case SC_FAC_CONST:
        x = (T)s.fac_const[c][k];
        break;
      default:
        x = field[fidx];
        break;
    }
    // the leading Python-float product is rounded once when it meets the
    // first dtype value; 1.0 * x is exact
    v = first ? X<T>::mul(v, x) : X<T>::mul(v, x);
    first = false;
  }
  return v;
}

template <typename T>
__device__ __forceinline__ int64_t corner_index(const SparseArgs<T> &s, const FieldDev &f, int c,
                                                int p, int slot) {
  int ii[3];
  for (int d = 0; d < s.ndim; ++d) ii[d] = s.base[(int64_t)d * s.npoint + p] + s.delta[c][d];
  return field_index(f, slot, ii, s.ndim);
}

template <typename T>
__global__ void __launch_bounds__(256) sparse_inject_kernel(SparseArgs<T> s, FieldDev f, int t,
                                                            int serial) {
  T *field = reinterpret_cast<T *>(f.data);
  int slot = time_slot(f, t + s.field_tshift);
  if (serial) {
    // colliding corners: replicate the oracle's p-outer, corner-inner order
    if (blockIdx.x != 0 || threadIdx.x != 0) return;
    for (int p = 0; p < s.npoint; ++p)
      for (int c = 0; c < s.ncorner; ++c) {
        int64_t idx = corner_index(s, f, c, p, slot);
        T v = corner_value(s, c, p, t, field, f, idx);
        field[idx] = X<T>::add(field[idx], v);
      }
    return;
  }
  // no two (point, corner) targets collide: one thread per increment
  const int64_t g = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (g >= (int64_t)s.npoint * s.ncorner) return;
  const int p = (int)(g / s.ncorner), c = (int)(g % s.ncorner);
  int64_t idx = corner_index(s, f, c, p, slot);
  T v = corner_value(s, c, p, t, field, f, idx);
  field[idx] = X<T>::add(field[idx], v);
}

// Interpolation: 8 lanes per receiver gather one corner product each; the
// products are then summed by the group leader in the oracle's corner order
// (sum() from 0, left to right: reference expr.py:459-460), so the
// warp-shuffle only moves values, it never reassociates the sum.
template <typename T>
__global__ void __launch_bounds__(256) sparse_interp_kernel(SparseArgs<T> s, FieldDev f, int t) {
  const int lanes = s.ncorner;  // 2, 4 or 8 (power of two)
  int gtid = blockIdx.x * blockDim.x + threadIdx.x;
  int p = gtid / lanes;
  int c = gtid % lanes;
  const T *field = reinterpret_cast<const T *>(f.data);
  int slot = time_slot(f, t + s.field_tshift);
  T term = 0;
  if (p < s.npoint) {
    int64_t idx = corner_index(s, f, c, p, slot);
    term = corner_value(s, c, p, t, field, f, idx);
  }
  // gather the group's terms to its first lane
  const unsigned full = 0xffffffffu;
  int lane = threadIdx.x & 31;
  int leader = lane - c;
  T acc = (T)0;
  for (int k = 0; k < lanes; ++k) {
    T v = __shfl_sync(full, term, leader + k);
    acc = X<T>::add(acc, v);
  }
  if (c == 0 && p < s.npoint)
    s.sparse[(int64_t)(t + s.sparse_tshift) * s.npoint + p] = acc;
}

// Interpolation with hoisted time-invariant prefixes. In the oracle's fold
// order a corner value is ((lead * f0) * f1) ... ; every factor before the
// field sample is time-invariant (weights, constants), so that prefix is
// evaluated once per prepared run (sparse_pre_kernel, same operations in the
// same order) and a time step only multiplies it by the sample, applies the
// time-invariant suffix factors and sums the corners from 0 in order. One
// thread per receiver; the corner-0 storage offset is precomputed as well.
__host__ __device__ inline int64_t field_elems(const FieldDev &f) {
  int64_t n = 1;
  for (int k = 0; k < f.ndim; ++k) n *= f.ext[k];
  return n;
}

template <typename T> struct InterpFastArgs {
  int npoint, ncorner;
  const T *pre;          // [ncorner][npoint]
  const int64_t *lin;    // [npoint] spatial offset of corner 0
  int64_t dl[SC_MAX_CORNERS];  // spatial offset of corner c from corner 0
  int64_t slot_stride;   // elements per time slot
  int npost[SC_MAX_CORNERS];
  int post_kind[SC_MAX_CORNERS][SC_MAX_FACTORS];  // SC_FAC_TABLE / SC_FAC_CONST
  const T *post_tab[SC_MAX_CORNERS][SC_MAX_FACTORS];
  T post_const[SC_MAX_CORNERS][SC_MAX_FACTORS];
  const T *field;
  FieldDev f;
  int field_tshift;
  T *sparse;
  int sparse_tshift;
};

template <typename T>
__global__ void __launch_bounds__(256) sparse_pre_kernel(SparseArgs<T> s, FieldDev f, T *pre,
                                                         int64_t *lin, int npre0, int npre1,
                                                         int npre2, int npre3, int npre4,
                                                         int npre5, int npre6, int npre7) {
  const int p = blockIdx.x * blockDim.x + threadIdx.x;
  if (p >= s.npoint) return;
  const int npre[8] = {npre0, npre1, npre2, npre3, npre4, npre5, npre6, npre7};
  int ii[3] = {0, 0, 0};
  for (int d = 0; d < s.ndim; ++d) ii[d] = s.base[(int64_t)d * s.npoint + p];
  // spatial offset of corner 0 (slot 0)
  int64_t li = 0;
  const int a = f.has_time ? 1 : 0;
  for (int d = 0; d < s.ndim; ++d) li = li * f.ext[a + d] + ii[d];
  lin[p] = li;
  for (int c = 0; c < s.ncorner; ++c) {
    T v = (T)s.lead[c];
    for (int k = 0; k < npre[c]; ++k) {
      const T x = s.fac_kind[c][k] == SC_FAC_TABLE ? s.tables[s.fac_arg[c][k]][p]
                                                   : (T)s.fac_const[c][k];
      v = X<T>::mul(v, x);
    }
    pre[(int64_t)c * s.npoint + p] = v;
  }
}

// Injection without colliding targets: one thread per (point, corner);
// prefix * datum, then the time-invariant suffix, then one exact increment.
template <typename T>
__global__ void __launch_bounds__(128) sparse_inject_fast(InterpFastArgs<T> a, int t, int p_lo,
                                                          int p_hi) {
  const int64_t g = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (g >= (int64_t)(p_hi - p_lo) * a.ncorner) return;
  const int p = p_lo + (int)(g / a.ncorner), c = (int)(g % a.ncorner);
  const int slot = time_slot(a.f, t + a.field_tshift);
  T *fp = const_cast<T *>(a.field) + (int64_t)slot * a.slot_stride + a.lin[p] + a.dl[c];
  SC_DCHECK(fp - a.field >= 0 && fp - a.field < field_elems(a.f));
  SC_DCHECK(t + a.sparse_tshift >= 0);
  const T d = a.sparse[(int64_t)(t + a.sparse_tshift) * a.npoint + p];
  const T old = *fp;
  T x = X<T>::mul(a.pre[(int64_t)c * a.npoint + p], d);
  for (int k = 0; k < a.npost[c]; ++k)
    x = X<T>::mul(x, a.post_kind[c][k] == SC_FAC_TABLE ? a.post_tab[c][k][p] : a.post_const[c][k]);
  *fp = X<T>::add(old, x);
}

// Injection with colliding targets, exact and parallel: the increments
// (point p, corner c) are grouped by target, each group keeping the oracle's
// (p-outer, corner-inner) order (reference iet.py:234-245: the ATOMIC loop
// runs points in order). One thread per distinct target folds its group's
// values into the target in that order, so every target sees the same
// sequence of rounded additions as the serial loop; different targets
// commute. order[] = increment ids g = p * ncorner + c sorted stably by
// target, gstart[] = group boundaries.
template <typename T>
__global__ void __launch_bounds__(128) sparse_inject_grouped(InterpFastArgs<T> a, int t,
                                                             const int *order, const int *gstart,
                                                             int ngroups) {
  const int gi = blockIdx.x * blockDim.x + threadIdx.x;
  if (gi >= ngroups) return;
  const int slot = time_slot(a.f, t + a.field_tshift);
  const int j0 = gstart[gi], j1 = gstart[gi + 1];
  int g = order[j0];
  int p = g / a.ncorner, c = g % a.ncorner;
  T *fp = const_cast<T *>(a.field) + (int64_t)slot * a.slot_stride + a.lin[p] + a.dl[c];
  SC_DCHECK(fp - a.field >= 0 && fp - a.field < field_elems(a.f));
  T acc = *fp;
  for (int j = j0; j < j1; ++j) {
    g = order[j];
    p = g / a.ncorner;
    c = g % a.ncorner;
    const T d = a.sparse[(int64_t)(t + a.sparse_tshift) * a.npoint + p];
    T x = X<T>::mul(a.pre[(int64_t)c * a.npoint + p], d);
    for (int k = 0; k < a.npost[c]; ++k)
      x = X<T>::mul(x, a.post_kind[c][k] == SC_FAC_TABLE ? a.post_tab[c][k][p] : a.post_const[c][k]);
    acc = X<T>::add(acc, x);
  }
  *fp = acc;
}

// Tolerance mode (SC_INJECT_ATOMIC=1): one thread per increment with a
// hardware atomic add -- the order of colliding additions is unspecified, so
// results match the oracle within rounding, not bit for bit.
template <typename T>
__global__ void __launch_bounds__(128) sparse_inject_atomic(InterpFastArgs<T> a, int t) {
  const int64_t g = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (g >= (int64_t)a.npoint * a.ncorner) return;
  const int p = (int)(g / a.ncorner), c = (int)(g % a.ncorner);
  const int slot = time_slot(a.f, t + a.field_tshift);
  T *fp = const_cast<T *>(a.field) + (int64_t)slot * a.slot_stride + a.lin[p] + a.dl[c];
  SC_DCHECK(fp - a.field >= 0 && fp - a.field < field_elems(a.f));
  const T d = a.sparse[(int64_t)(t + a.sparse_tshift) * a.npoint + p];
  T x = X<T>::mul(a.pre[(int64_t)c * a.npoint + p], d);
  for (int k = 0; k < a.npost[c]; ++k)
    x = X<T>::mul(x, a.post_kind[c][k] == SC_FAC_TABLE ? a.post_tab[c][k][p] : a.post_const[c][k]);
  atomicAdd(fp, x);
}

template <typename T, int NC>
__global__ void __launch_bounds__(256) sparse_interp_fast(InterpFastArgs<T> a, int t, int p_lo,
                                                          int p_hi) {
  const int p = p_lo + blockIdx.x * blockDim.x + threadIdx.x;
  if (p >= p_hi) return;
  const int slot = time_slot(a.f, t + a.field_tshift);
  const T *fp = a.field + (int64_t)slot * a.slot_stride + a.lin[p];
  T v[NC];
#pragma unroll
  for (int c = 0; c < NC; ++c) {
    SC_DCHECK(fp + a.dl[c] - a.field >= 0 && fp + a.dl[c] - a.field < field_elems(a.f));
    v[c] = fp[a.dl[c]];
  }
  SC_DCHECK(t + a.sparse_tshift >= 0);
  T acc = (T)0;
#pragma unroll
  for (int c = 0; c < NC; ++c) {
    T x = X<T>::mul(a.pre[(int64_t)c * a.npoint + p], v[c]);
    for (int k = 0; k < a.npost[c]; ++k)
      x = X<T>::mul(x, a.post_kind[c][k] == SC_FAC_TABLE ? a.post_tab[c][k][p]
                                                         : a.post_const[c][k]);
    acc = X<T>::add(acc, x);
  }
  a.sparse[(int64_t)(t + a.sparse_tshift) * a.npoint + p] = acc;
}

// ---------------------------------------------------------------------------
// Host side of sc_run

template <typename T>
static void fill_fields(const sc_plan *pl, FieldDev *out) {
  for (int i = 0; i < pl->nfields; ++i) {
    const sc_field &f = pl->fields[i];
    out[i].data = f.data;
    for (int k = 0; k < 4; ++k) out[i].ext[k] = f.ext[k];
    out[i].ndim = f.ndim;
    out[i].nslots = f.nslots;
    out[i].has_time = f.has_time;
  }
}

struct DeviceProgram {
  int4 *ops = nullptr;
  LoadDev *loads = nullptr;
  double *consts = nullptr;
};

static int upload_program(const sc_dense &d, DeviceProgram &dp, cudaStream_t st) {
  if (d.nregs > SC_GEN_MAXREG) {
    sc_set_error("dense program needs %d registers (max %d)", d.nregs, SC_GEN_MAXREG);
    return -1;
  }
  std::vector<int4> ops(d.nops > 0 ? d.nops : 1);
  for (int i = 0; i < d.nops; ++i)
    ops[i] = make_int4(d.ops[i].op, d.ops[i].dst, d.ops[i].a, d.ops[i].b);
  std::vector<LoadDev> loads(d.nloads > 0 ? d.nloads : 1);
  for (int i = 0; i < d.nloads; ++i) {
    loads[i].field = d.loads[i].field;
    loads[i].tshift = d.loads[i].tshift;
    loads[i].tdiv = d.loads[i].tdiv;
    for (int k = 0; k < 3; ++k) loads[i].off[k] = d.loads[i].off[k];
  }
  SC_CUDA(cudaMallocAsync((void **)&dp.ops, sizeof(int4) * ops.size(), st));
  SC_CUDA(cudaMallocAsync((void **)&dp.loads, sizeof(LoadDev) * loads.size(), st));
  SC_CUDA(cudaMallocAsync((void **)&dp.consts, sizeof(double) * (d.nconsts > 0 ? d.nconsts : 1), st));
  SC_CUDA(cudaMemcpyAsync(dp.ops, ops.data(), sizeof(int4) * ops.size(), cudaMemcpyHostToDevice, st));
  SC_CUDA(cudaMemcpyAsync(dp.loads, loads.data(), sizeof(LoadDev) * loads.size(),
                          cudaMemcpyHostToDevice, st));
  if (d.nconsts > 0)
    SC_CUDA(cudaMemcpyAsync(dp.consts, d.consts, sizeof(double) * d.nconsts,
                            cudaMemcpyHostToDevice, st));
  return 0;
}

template <typename T>
static void fill_sparse(const sc_sparse &sp, SparseArgs<T> &s) {
  memset(&s, 0, sizeof(s));
  s.npoint = sp.npoint;
  s.ncorner = sp.ncorner;
  s.ndim = sp.ndim;
  s.base = sp.base;
  memcpy(s.delta, sp.delta, sizeof(s.delta));
  memcpy(s.nfac, sp.nfac, sizeof(s.nfac));
  memcpy(s.fac_kind, sp.fac_kind, sizeof(s.fac_kind));
  memcpy(s.fac_arg, sp.fac_arg, sizeof(s.fac_arg));
  memcpy(s.fac_const, sp.fac_const, sizeof(s.fac_const));
  memcpy(s.lead, sp.lead, sizeof(s.lead));
  for (int k = 0; k < SC_MAX_TABLES; ++k) s.tables[k] = reinterpret_cast<const T *>(sp.tables[k]);
  s.field_tshift = sp.field_tshift;
  s.sparse = reinterpret_cast<T *>(sp.sparse);
  s.sparse_tshift = sp.sparse_tshift;
}

// A prepared run: device programs, fused-kernel state (tensor maps, operand
// check) and, for the canonical acoustic step order, the whole t loop
// captured as one CUDA graph. Prepared once, launched any number of times
// (Operator.apply launches once; bench.py re-launches the same run).
struct RunBase {
  int dtype = 0;
  virtual ~RunBase() {}
  virtual int launch(sc_plan *pl) = 0;
  virtual int step(int t, cudaStream_t st) = 0;
  virtual int revalidate(cudaStream_t st) = 0;
  virtual int early_download(int t_split, const void *dev, void *host, size_t bytes) = 0;
  virtual int multi_run(MultiComm *c, const sc_exchange &x, cudaStream_t st) = 0;
  virtual int multi_exchange_step(MultiComm *c, const sc_exchange &x, int t,
                                  cudaStream_t st) = 0;
  virtual int step_part(int t, cudaStream_t st, int x_lo, int x_hi, int p_lo, int p_hi,
                        int what) = 0;
};

template <typename T> struct Run : RunBase {
  sc_plan plan;  // copy (host program pointers are used during prepare only)
  FieldDev fields[SC_MAX_FIELDS];
  std::vector<DeviceProgram> progs;
  std::vector<DenseArgs<T>> dargs;
  std::vector<FastAcoustic> fast;
  std::vector<int> use_fast;
  std::vector<JitDense> jit;
  std::vector<int> use_jit;
  std::vector<SparseArgs<T>> sargs;
  std::vector<InterpFastArgs<T>> ifa;
  std::vector<int> use_ifast;
  // colliding injections: increment order grouped by target (device), or
  // the atomic tolerance mode
  struct Groups {
    int *order = nullptr, *gstart = nullptr;
    int ngroups = 0;
    bool atomic = false;
  };
  std::vector<Groups> groups;
  std::vector<void *> dev_allocs;
  bool overlap = false;
  cudaGraphExec_t exec = nullptr;
  int launches_per_run = 0;
  // sc_early_download: the loop as two graphs [t_m, t_split) and
  // [t_split, t_M]; between them a device->host copy (rows of an
  // interpolated function that are already final) starts on its own stream
  // and runs under the second graph
  cudaGraphExec_t exec_a = nullptr, exec_b = nullptr;
  int t_split = INT_MIN;
  const void *early_dev = nullptr;
  void *early_host = nullptr;
  size_t early_bytes = 0;
  cudaStream_t early_stream = nullptr;
  cudaEvent_t early_event = nullptr;

  // sc_multi_run: the slab t loop with its ghost exchange, captured once per
  // (communicator, exchange description)
  cudaGraphExec_t mexec = nullptr;
  MultiComm *mcomm = nullptr;
  sc_exchange mx;
  cudaStream_t mside = nullptr;

  ~Run() {
    tti_forget(plan.dense, SC_MAX_DENSE);
    if (exec) cudaGraphExecDestroy(exec);
    if (exec_a) cudaGraphExecDestroy(exec_a);
    if (exec_b) cudaGraphExecDestroy(exec_b);
    if (early_stream) cudaStreamDestroy(early_stream);
    if (early_event) cudaEventDestroy(early_event);
    if (mexec) cudaGraphExecDestroy(mexec);
    if (mside) cudaStreamDestroy(mside);
    for (auto &dp : progs) {
      if (dp.ops) cudaFree(dp.ops);
      if (dp.loads) cudaFree(dp.loads);
      if (dp.consts) cudaFree(dp.consts);
    }
    for (auto &fa : fast) fast_acoustic_release(fa);
    for (void *q : dev_allocs) cudaFree(q);
  }

  // 0 = hoisted-prefix sparse stage prepared, 1 = not applicable. The one
  // time-varying factor of a corner is the field sample (interpolation) or
  // the sparse datum (injection without colliding targets).
  int interp_fast_prepare(int si, cudaStream_t st) {
    const sc_sparse &sp = plan.sparse[si];
    if (sp.npoint <= 0) return 1;
    const int tv = sp.kind == 1 ? SC_FAC_FIELD : SC_FAC_SPARSE;
    const int other = sp.kind == 1 ? SC_FAC_SPARSE : SC_FAC_FIELD;
    const int nc = sp.ncorner;
    if (nc != 1 && nc != 2 && nc != 4 && nc != 8) return 1;
    if (sp.kind == 0 && sp.serial && (int64_t)sp.npoint * nc >= INT_MAX) return 1;
    InterpFastArgs<T> &a = ifa[si];
    memset(&a, 0, sizeof(a));
    int npre[8] = {0, 0, 0, 0, 0, 0, 0, 0};
    for (int c = 0; c < nc; ++c) {
      int k0 = -1;
      for (int k = 0; k < sp.nfac[c]; ++k) {
        const int kind = sp.fac_kind[c][k];
        if (kind == other) return 1;
        if (kind == tv) {
          if (k0 >= 0) return 1;
          k0 = k;
        }
      }
      if (k0 < 0) return 1;
      npre[c] = k0;
      a.npost[c] = sp.nfac[c] - k0 - 1;
      for (int k = k0 + 1; k < sp.nfac[c]; ++k) {
        const int j = k - k0 - 1;
        a.post_kind[c][j] = sp.fac_kind[c][k];
        a.post_tab[c][j] = reinterpret_cast<const T *>(sp.tables[sp.fac_arg[c][k]]);
        a.post_const[c][j] = (T)sp.fac_const[c][k];
      }
    }
    const FieldDev &f = fields[sp.field];
    const int off = f.has_time ? 1 : 0;
    int64_t stride[3] = {1, 1, 1};
    for (int d = sp.ndim - 1; d >= 0; --d)
      stride[d] = d == sp.ndim - 1 ? 1 : stride[d + 1] * f.ext[off + d + 1];
    a.slot_stride = 1;
    for (int d = 0; d < sp.ndim; ++d) a.slot_stride *= f.ext[off + d];
    if (!f.has_time) a.slot_stride = 0;
    for (int c = 0; c < nc; ++c) {
      a.dl[c] = 0;
      for (int d = 0; d < sp.ndim; ++d) a.dl[c] += (int64_t)sp.delta[c][d] * stride[d];
    }
    T *pre = nullptr;
    int64_t *lin = nullptr;
    SC_CUDA(cudaMalloc((void **)&pre, sizeof(T) * (size_t)nc * sp.npoint));
    dev_allocs.push_back(pre);
    SC_CUDA(cudaMalloc((void **)&lin, sizeof(int64_t) * (size_t)sp.npoint));
    dev_allocs.push_back(lin);
    sparse_pre_kernel<T><<<(unsigned)sc_ceil_div(sp.npoint, 256), 256, 0, st>>>(
        sargs[si], f, pre, lin, npre[0], npre[1], npre[2], npre[3], npre[4], npre[5], npre[6],
        npre[7]);
    SC_CUDA(cudaGetLastError());
    a.npoint = sp.npoint;
    a.ncorner = nc;
    a.pre = pre;
    a.lin = lin;
    a.field = reinterpret_cast<const T *>(f.data);
    a.f = f;
    a.field_tshift = sp.field_tshift;
    a.sparse = reinterpret_cast<T *>(sp.sparse);
    a.sparse_tshift = sp.sparse_tshift;
    if (sp.kind == 0 && sp.serial) return group_targets(si, st);
    return 0;
  }

  // colliding injection targets: stable sort of the increments by target
  // (once per prepared run, on the host: npoint * ncorner keys)
  int group_targets(int si, cudaStream_t st) {
    InterpFastArgs<T> &a = ifa[si];
    Groups &G = groups[si];
    if (getenv("SC_INJECT_ATOMIC")) {
      G.atomic = true;
      return 0;
    }
    const int n = a.npoint * a.ncorner;
    std::vector<int64_t> lin(a.npoint);
    SC_CUDA(cudaMemcpyAsync(lin.data(), a.lin, sizeof(int64_t) * a.npoint,
                            cudaMemcpyDeviceToHost, st));
    SC_CUDA(cudaStreamSynchronize(st));
    std::vector<int> order(n);
    for (int g = 0; g < n; ++g) order[g] = g;
    auto key = [&](int g) { return lin[g / a.ncorner] + a.dl[g % a.ncorner]; };
    std::stable_sort(order.begin(), order.end(), [&](int x, int y) { return key(x) < key(y); });
    std::vector<int> gstart;
    for (int j = 0; j < n; ++j)
      if (j == 0 || key(order[j]) != key(order[j - 1])) gstart.push_back(j);
    G.ngroups = (int)gstart.size();
    gstart.push_back(n);
    int *dorder = nullptr, *dstart = nullptr;
    SC_CUDA(cudaMalloc((void **)&dorder, sizeof(int) * n));
    dev_allocs.push_back(dorder);
    SC_CUDA(cudaMalloc((void **)&dstart, sizeof(int) * gstart.size()));
    dev_allocs.push_back(dstart);
    SC_CUDA(cudaMemcpyAsync(dorder, order.data(), sizeof(int) * n, cudaMemcpyHostToDevice, st));
    SC_CUDA(cudaMemcpyAsync(dstart, gstart.data(), sizeof(int) * gstart.size(),
                            cudaMemcpyHostToDevice, st));
    SC_CUDA(cudaStreamSynchronize(st));
    G.order = dorder;
    G.gstart = dstart;
    return 0;
  }

  // points [p_lo, p_hi) of a hoisted-prefix sparse stage (all by default)
  void interp_fast_launch(int si, int t, cudaStream_t s_, int p_lo = 0, int p_hi = -1) {
    const InterpFastArgs<T> &a = ifa[si];
    if (p_hi < 0) p_hi = a.npoint;
    if (p_hi <= p_lo) return;
    if (plan.sparse[si].kind == 0 && plan.sparse[si].serial) {
      const Groups &G = groups[si];
      if (G.atomic) {
        const int64_t n = (int64_t)a.npoint * a.ncorner;
        sparse_inject_atomic<T><<<(unsigned)sc_ceil_div(n, 128), 128, 0, s_>>>(a, t);
      } else {
        sparse_inject_grouped<T><<<(unsigned)sc_ceil_div(G.ngroups, 128), 128, 0, s_>>>(
            a, t, G.order, G.gstart, G.ngroups);
      }
      return;
    }
    if (plan.sparse[si].kind == 0) {
      const int64_t n = (int64_t)(p_hi - p_lo) * a.ncorner;
      sparse_inject_fast<T><<<(unsigned)sc_ceil_div(n, 128), 128, 0, s_>>>(a, t, p_lo, p_hi);
      return;
    }
    const unsigned g = (unsigned)sc_ceil_div(p_hi - p_lo, 256);
    switch (a.ncorner) {
      case 1: sparse_interp_fast<T, 1><<<g, 256, 0, s_>>>(a, t, p_lo, p_hi); break;
      case 2: sparse_interp_fast<T, 2><<<g, 256, 0, s_>>>(a, t, p_lo, p_hi); break;
      case 4: sparse_interp_fast<T, 4><<<g, 256, 0, s_>>>(a, t, p_lo, p_hi); break;
      default: sparse_interp_fast<T, 8><<<g, 256, 0, s_>>>(a, t, p_lo, p_hi); break;
    }
  }

  int stage(int k, int t, cudaStream_t s_) {
    const sc_plan *pl = &plan;
    int code = pl->stages[k];
    // guarded (sub-sampled) statements run only at t % tguard == 0
    if (code < 100 && pl->dense[code].tguard > 1 && t % pl->dense[code].tguard != 0) return 0;
    if (code < 100 && pl->dense[code].fast_kind == SC_FAST_TTI) {
      if (tti_launch<T>(pl, pl->dense[code], fields, t, s_) != 0) return -1;
    } else if (code < 100) {
      if (use_fast[code]) {
        if (fast_acoustic_launch<T>(fast[code], t, s_) != 0) return -1;
      } else if (use_jit[code]) {
        if (jit_dense_launch(jit[code], fields, (int)sizeof(T), t, s_) != 0) return -1;
      } else {
        DenseArgs<T> &a = dargs[code];
        int64_t n = (int64_t)a.n[0] * a.n[1] * a.n[2];
        if (n > 0) dense_generic_kernel<T><<<(unsigned)sc_ceil_div(n, 256), 256, 0, s_>>>(a, t);
      }
    } else {
      int si = code - 100;
      const sc_sparse &sp = pl->sparse[si];
      const FieldDev &f = fields[sp.field];
      if (sp.npoint > 0) {
        int64_t thr = (int64_t)sp.npoint * sp.ncorner;
        if (use_ifast[si]) {
          interp_fast_launch(si, t, s_);
        } else if (sp.kind == 0) {
          unsigned grid = sp.serial ? 1u : (unsigned)sc_ceil_div(thr, 256);
          sparse_inject_kernel<T><<<grid, 256, 0, s_>>>(sargs[si], f, t, sp.serial);
        } else {
          sparse_interp_kernel<T><<<(unsigned)sc_ceil_div(thr, 256), 256, 0, s_>>>(sargs[si], f, t);
        }
      }
    }
    SC_CUDA(cudaGetLastError());
    return 0;
  }

  int prepare(const sc_plan *pl) {
    plan = *pl;
    cudaStream_t st = reinterpret_cast<cudaStream_t>(pl->stream);
    memset(fields, 0, sizeof(fields));
    fill_fields<T>(pl, fields);
    progs.resize(pl->ndense);
    dargs.resize(pl->ndense);
    fast.resize(pl->ndense);
    use_fast.assign(pl->ndense, 0);
    jit.resize(pl->ndense);
    use_jit.assign(pl->ndense, 0);
    // generated kernels for the programs no family kernel takes (opt out
    // with SC_NO_JIT=1: the interpreter kernel, same results)
    const bool want_jit = !getenv("SC_NO_JIT");
    for (int i = 0; i < pl->ndense; ++i) {
      const sc_dense &d = pl->dense[i];
      if (d.fast_kind == SC_FAST_TTI) {
        if (pl->ndim != 3 || !d.scratch[0] || !d.scratch[1] || !d.fast_consts) {
          sc_set_error("malformed TTI stage");
          return -1;
        }
        use_fast[i] = 1;
        continue;
      }
      if (d.fast_kind != SC_FAST_NONE) {
        const int rc = fast_acoustic_prepare<T>(pl, d, fast[i]);
        if (rc < 0) return -1;
        if (rc == 0) {
          use_fast[i] = 1;
          continue;
        }
      }
      if (want_jit) {
        const int rc = jit_dense_build(pl, d, jit[i]);
        if (rc < 0) return -1;
        if (rc == 0) use_jit[i] = 1;
      }
      if (upload_program(d, progs[i], st) != 0) return -1;
      DenseArgs<T> &a = dargs[i];
      memset(&a, 0, sizeof(a));
      memcpy(a.fields, fields, sizeof(fields));
      a.ops = progs[i].ops;
      a.loads = progs[i].loads;
      a.consts = progs[i].consts;
      a.nops = d.nops;
      a.out_reg = d.out_reg;
      a.ndim = pl->ndim;
      a.target.field = d.target.field;
      a.target.tshift = d.target.tshift;
      a.target.tdiv = d.target.tdiv;
      for (int k = 0; k < 3; ++k) {
        a.target.off[k] = d.target.off[k];
        a.lo[k] = k < pl->ndim ? pl->lo[k] : 0;
        a.n[k] = k < pl->ndim ? pl->hi[k] - pl->lo[k] + 1 : 1;
      }
    }
    sargs.resize(pl->nsparse);
    for (int i = 0; i < pl->nsparse; ++i) fill_sparse<T>(pl->sparse[i], sargs[i]);
    ifa.resize(pl->nsparse);
    groups.assign(pl->nsparse, Groups());
    use_ifast.assign(pl->nsparse, 0);
    if (!getenv("SC_NO_FAST_INTERP"))
      for (int i = 0; i < pl->nsparse; ++i) {
        const int rc = interp_fast_prepare(i, st);
        if (rc < 0) return -1;
        use_ifast[i] = rc == 0;
      }
    SC_CUDA(cudaStreamSynchronize(st));
    for (int i = 0; i < pl->ndense; ++i) plan.dense[i].fast_kind = use_fast[i] ? pl->dense[i].fast_kind : 0;

    // Overlap: in the canonical per-step order [stencil u[t+1], inject into
    // u[t+1], interpolate from u[t]] the interpolation of step t only reads
    // u[t]; it runs on a side stream concurrently with the stencil of step
    // t and must finish before the stencil of step t+2 overwrites slot t%3.
    const int ns = pl->nstages;
    overlap = !getenv("SC_NO_OVERLAP") && ns == 3 && pl->stages[0] < 100 && pl->stages[1] >= 100 && pl->stages[2] >= 100;
    if (overlap) {
      const sc_dense &d = pl->dense[pl->stages[0]];
      const sc_sparse &a = pl->sparse[pl->stages[1] - 100];
      const sc_sparse &b = pl->sparse[pl->stages[2] - 100];
      const sc_field &uf = pl->fields[d.target.field];
      overlap = d.target.tshift == 1 && a.kind == 0 && a.field == d.target.field &&
                a.field_tshift == 1 && b.kind == 1 && b.field == d.target.field &&
                b.field_tshift == 0 && uf.nslots == 3;
    }
    launches_per_run = 0;
    for (int t = pl->t_m; t <= pl->t_M; ++t)
      for (int k = 0; k < ns; ++k) {
        const int c = pl->stages[k];
        const bool skip = c < 100 && pl->dense[c].tguard > 1 && t % pl->dense[c].tguard;
        // a TTI step is two kernels (g pass and update pass)
        launches_per_run += skip ? 0 : (c < 100 && pl->dense[c].fast_kind == SC_FAST_TTI ? 2 : 1);
      }
    // a plan prepared with profile=1 is launched stage by stage (profiling,
    // host-driven step loops): no graph
    if (pl->t_M >= pl->t_m && !pl->profile) return capture_range(plan.t_m, plan.t_M, &exec);
    return 0;
  }

  int capture_range(int t0, int t1, cudaGraphExec_t *out) {
    return overlap ? capture(t0, t1, out) : capture_sequential(t0, t1, out);
  }

  int capture_sequential(int t0, int t1, cudaGraphExec_t *out) {
    cudaStream_t cap;
    SC_CUDA(cudaStreamCreateWithFlags(&cap, cudaStreamNonBlocking));
    SC_CUDA(cudaStreamBeginCapture(cap, cudaStreamCaptureModeThreadLocal));
    for (int t = t0; t <= t1; ++t)
      for (int k = 0; k < plan.nstages; ++k)
        if (stage(k, t, cap)) {
          cudaGraph_t g;
          cudaStreamEndCapture(cap, &g);
          return -1;
        }
    cudaGraph_t graph;
    SC_CUDA(cudaStreamEndCapture(cap, &graph));
    SC_CUDA(cudaGraphInstantiate(out, graph, 0));
    cudaGraphDestroy(graph);
    cudaStreamDestroy(cap);
    return 0;
  }

  // The t loop (both streams) captured once: per-node launch cost is paid at
  // instantiation, not per time step.
  int capture(int t0, int t1, cudaGraphExec_t *out) {
    cudaStream_t cap, side;
    SC_CUDA(cudaStreamCreateWithFlags(&cap, cudaStreamNonBlocking));
    SC_CUDA(cudaStreamCreateWithFlags(&side, cudaStreamNonBlocking));
    const int NE = 4;
    cudaEvent_t evS[NE], evI[NE], fork;
    for (int i = 0; i < NE; ++i) {
      SC_CUDA(cudaEventCreateWithFlags(&evS[i], cudaEventDisableTiming));
      SC_CUDA(cudaEventCreateWithFlags(&evI[i], cudaEventDisableTiming));
    }
    SC_CUDA(cudaEventCreateWithFlags(&fork, cudaEventDisableTiming));
    SC_CUDA(cudaStreamBeginCapture(cap, cudaStreamCaptureModeThreadLocal));
    SC_CUDA(cudaEventRecord(fork, cap));
    for (int t = t0; t <= t1; ++t) {
      const int rel = t - t0;
      if (rel >= 2) SC_CUDA(cudaStreamWaitEvent(cap, evI[(rel - 2) % NE], 0));
      if (stage(0, t, cap) || stage(1, t, cap)) return -1;
      SC_CUDA(cudaEventRecord(evS[rel % NE], cap));
      SC_CUDA(cudaStreamWaitEvent(side, rel == 0 ? fork : evS[(rel - 1) % NE], 0));
      if (stage(2, t, side)) return -1;
      SC_CUDA(cudaEventRecord(evI[rel % NE], side));
    }
    SC_CUDA(cudaStreamWaitEvent(cap, evI[(t1 - t0) % NE], 0));
    cudaGraph_t graph;
    SC_CUDA(cudaStreamEndCapture(cap, &graph));
    SC_CUDA(cudaGraphInstantiate(out, graph, 0));
    cudaGraphDestroy(graph);
    for (int i = 0; i < NE; ++i) {
      cudaEventDestroy(evS[i]);
      cudaEventDestroy(evI[i]);
    }
    cudaEventDestroy(fork);
    cudaStreamDestroy(side);
    cudaStreamDestroy(cap);
    return 0;
  }

  // one time step, asynchronous on `st` (host-driven loops, e.g. the
  // multi-GPU slab runner exchanging ghost planes between steps)
  int prologue(cudaStream_t st) {
    for (int i = 0; i < plan.ndense; ++i)
      if (plan.dense[i].fast_kind == SC_FAST_TTI && tti_prologue(plan.dense[i], fields, st)) return -1;
    return 0;
  }

  // data-dependent preconditions of the fused stages on the current buffer
  // contents (a prepared run reused on re-uploaded inputs): 0 ok, 1 stale
  // bytes == 0 switches the early copy off (the single graph runs again)
  int early_download(int ts, const void *dev, void *host, size_t bytes) override {
    early_dev = dev;
    early_host = host;
    early_bytes = bytes;
    if (!bytes) return 0;
    if (ts <= plan.t_m || ts > plan.t_M) {
      early_bytes = 0;
      return 1;  // an empty part: nothing to overlap
    }
    if (!early_stream) {
      SC_CUDA(cudaStreamCreateWithFlags(&early_stream, cudaStreamNonBlocking));
      SC_CUDA(cudaEventCreateWithFlags(&early_event, cudaEventDisableTiming));
    }
    // stage-by-stage launches (profiled runs) start the copy from their
    // loop; a graph launch captures the two part graphs when it first needs
    // them (split_graphs)
    if (ts != t_split) {
      if (exec_a) cudaGraphExecDestroy(exec_a);
      if (exec_b) cudaGraphExecDestroy(exec_b);
      exec_a = exec_b = nullptr;
    }
    t_split = ts;
    return 0;
  }

  int split_graphs() {
    if (exec_a && exec_b) return 0;
    if (capture_range(plan.t_m, t_split - 1, &exec_a) ||
        capture_range(t_split, plan.t_M, &exec_b)) {
      early_bytes = 0;
      return -1;
    }
    return 0;
  }

  int revalidate(cudaStream_t st) override {
    for (int i = 0; i < plan.ndense; ++i) {
      if (!use_fast[i] || plan.dense[i].fast_kind == SC_FAST_TTI) continue;
      const int rc = fast_acoustic_check<T>(fast[i], st);
      if (rc != 0) return rc;
    }
    return 0;
  }

  bool t_ok(int t) {
    if (t >= plan.t_m && t <= plan.t_M) return true;
    // the sparse stages index rows (t + shift) of arrays sized for
    // [t_m, t_M]: a step outside would read/write past them
    sc_set_error("time step %d outside the prepared range [%d, %d]", t, plan.t_m, plan.t_M);
    return false;
  }

  int multi_exchange_step(MultiComm *c, const sc_exchange &x, int t, cudaStream_t st) override {
    if (!t_ok(t)) return -1;
    return multi_exchange(c, x, fields, (int)sizeof(T), t, st);
  }

  // one slab time step on `cap` (+ `side` for the overlapped exchange)
  int multi_step(MultiComm *c, const sc_exchange &x, int t, cudaStream_t cap,
                 cudaStream_t side, cudaEvent_t evB, cudaEvent_t evX) {
    const int big = 1 << 30;
    if (!x.overlap) {
      if (step(t, cap)) return -1;
      return multi_exchange(c, x, fields, (int)sizeof(T), t, cap);
    }
    for (int k = 0; k < x.nearly; ++k)
      if (step_part(t, cap, x.early[k][0], x.early[k][1], 0, 0, 1)) return -1;
    if (x.n_early_points > 0 && step_part(t, cap, 0, -1, 0, x.n_early_points, 2)) return -1;
    SC_CUDA(cudaEventRecord(evB, cap));
    SC_CUDA(cudaStreamWaitEvent(side, evB, 0));
    if (multi_exchange(c, x, fields, (int)sizeof(T), t, side)) return -1;
    SC_CUDA(cudaEventRecord(evX, side));
    if (x.interior[1] >= x.interior[0] &&
        step_part(t, cap, x.interior[0], x.interior[1], 0, 0, 1))
      return -1;
    if (step_part(t, cap, 0, -1, x.n_early_points, big, 2)) return -1;
    if (step_part(t, cap, 0, -1, 0, big, 4)) return -1;
    SC_CUDA(cudaStreamWaitEvent(cap, evX, 0));
    return 0;
  }

  int multi_run(MultiComm *c, const sc_exchange &x, cudaStream_t st) override {
    if (x.overlap && step_part(plan.t_m, st, 0, -1, 0, 0, 0)) return -1;  // capability
    const bool same = mexec && mcomm == c && memcmp(&mx, &x, sizeof(x)) == 0;
    if (!same) {
      if (mexec) cudaGraphExecDestroy(mexec);
      mexec = nullptr;
      mcomm = c;
      mx = x;
      if (!mside) SC_CUDA(cudaStreamCreateWithFlags(&mside, cudaStreamNonBlocking));
      const bool graph = !getenv("SC_MULTI_NOGRAPH");
      if (graph) {
        cudaStream_t cap;
        SC_CUDA(cudaStreamCreateWithFlags(&cap, cudaStreamNonBlocking));
        const int NE = 2;
        cudaEvent_t evB[NE], evX[NE];
        for (int i = 0; i < NE; ++i) {
          SC_CUDA(cudaEventCreateWithFlags(&evB[i], cudaEventDisableTiming));
          SC_CUDA(cudaEventCreateWithFlags(&evX[i], cudaEventDisableTiming));
        }
        SC_CUDA(cudaStreamBeginCapture(cap, cudaStreamCaptureModeThreadLocal));
        int rc = 0;
        for (int t = plan.t_m; t <= plan.t_M && !rc; ++t)
          rc = multi_step(c, x, t, cap, mside, evB[t & 1], evX[t & 1]);
        cudaGraph_t g = nullptr;
        const cudaError_t e = cudaStreamEndCapture(cap, &g);
        for (int i = 0; i < NE; ++i) {
          cudaEventDestroy(evB[i]);
          cudaEventDestroy(evX[i]);
        }
        cudaStreamDestroy(cap);
        if (rc) {
          if (g) cudaGraphDestroy(g);
          return -1;
        }
        if (e != cudaSuccess) {
          sc_set_error("capture of the slab loop failed: %s", cudaGetErrorString(e));
          return -1;
        }
        SC_CUDA(cudaGraphInstantiate(&mexec, g, 0));
        cudaGraphDestroy(g);
      }
    }
    if (mexec) {
      SC_CUDA(cudaGraphLaunch(mexec, st));
      return 0;
    }
    // eager fallback (SC_MULTI_NOGRAPH=1): same schedule, launched per step
    cudaEvent_t evB, evX;
    SC_CUDA(cudaEventCreateWithFlags(&evB, cudaEventDisableTiming));
    SC_CUDA(cudaEventCreateWithFlags(&evX, cudaEventDisableTiming));
    int rc = 0;
    for (int t = plan.t_m; t <= plan.t_M && !rc; ++t) rc = multi_step(c, x, t, st, mside, evB, evX);
    cudaEventDestroy(evB);
    cudaEventDestroy(evX);
    return rc;
  }

  int step(int t, cudaStream_t st) override {
    if (!t_ok(t)) return -1;
    if (t == plan.t_m && prologue(st)) return -1;
    for (int k = 0; k < plan.nstages; ++k)
      if (stage(k, t, st)) return -1;
    return 0;
  }

  // Part of time step t (multi-GPU overlap, backend/slab.py): what & 1 runs
  // the dense stages over loop x planes [x_lo, x_hi] (fused acoustic kernel
  // only), what & 2 the injections and what & 4 the interpolations over
  // points [p_lo, p_hi) (hoisted-prefix sparse kernels only). Stage order
  // within the parts is the plan's.
  int step_part(int t, cudaStream_t st, int x_lo, int x_hi, int p_lo, int p_hi,
                int what) override {
    if (what == 0) {  // capability probe: every stage can run in parts
      for (int k = 0; k < plan.nstages; ++k) {
        const int code = plan.stages[k];
        const bool tti = code < 100 && plan.dense[code].fast_kind == SC_FAST_TTI;
        // colliding injections (grouped by target) run whole, never in parts
        const bool ok = tti   ? sizeof(T) == 4 && tti_tma_ok(plan.dense[code], fields)
                        : code < 100 ? use_fast[code] != 0
                                     : use_ifast[code - 100] != 0 &&
                                           !(plan.sparse[code - 100].kind == 0 &&
                                             plan.sparse[code - 100].serial);
        if (!ok) {
          sc_set_error("stage %d cannot run in parts", k);
          return -1;
        }
      }
      return 0;
    }
    if (!t_ok(t)) return -1;
    for (int k = 0; k < plan.nstages; ++k) {
      const int code = plan.stages[k];
      if (code < 100) {
        if (!(what & 1)) continue;
        if (plan.dense[code].fast_kind == SC_FAST_TTI) {
          // the TTI pair over the x slab (coefficients hoisted at t_m)
          if (sizeof(T) != 4 || !tti_tma_ok(plan.dense[code], fields)) {
            sc_set_error("partial TTI steps need the f32 TMA passes");
            return -1;
          }
          if (t == plan.t_m && tti_prologue(plan.dense[code], fields, st)) return -1;
          if (x_hi >= x_lo &&
              tti_tma_launch(&plan, plan.dense[code], fields, t, st, x_lo, x_hi) != 0)
            return -1;
          continue;
        }
        if (!use_fast[code]) {
          sc_set_error("partial steps need the fused acoustic kernel");
          return -1;
        }
        if (plan.dense[code].tguard > 1 && t % plan.dense[code].tguard) continue;
        if (x_hi < x_lo) continue;
        FastAcoustic fa = fast[code];
        if (x_lo < fa.lo[0] || x_hi >= fa.lo[0] + fa.n[0]) {
          sc_set_error("partial x range [%d, %d] outside the loop box", x_lo, x_hi);
          return -1;
        }
        fa.lo[0] = x_lo;
        fa.n[0] = x_hi - x_lo + 1;
        fa.grid.z = (unsigned)sc_ceil_div(fa.n[0], fa.xchunk);
        if (fast_acoustic_launch<T>(fa, t, st) != 0) return -1;
      } else {
        const int si = code - 100;
        const int bit = plan.sparse[si].kind == 0 ? 2 : 4;
        if (!(what & bit)) continue;
        if (!use_ifast[si] || (plan.sparse[si].kind == 0 && plan.sparse[si].serial)) {
          sc_set_error("partial steps need the hoisted-prefix sparse kernels");
          return -1;
        }
        const int hi = std::min(p_hi, ifa[si].npoint);
        interp_fast_launch(si, t, st, std::max(p_lo, 0), hi);
      }
      SC_CUDA(cudaGetLastError());
    }
    return 0;
  }

  int launch(sc_plan *pl) override {
    cudaStream_t st = reinterpret_cast<cudaStream_t>(pl->stream);
    const int ns = plan.nstages;
    const int nsteps = plan.t_M - plan.t_m + 1;
    const bool timing = nsteps > 0 && pl->profile;
    for (int k = 0; k < ns; ++k) pl->stage_ms[k] = 0.f;
    for (int i = 0; i < plan.ndense; ++i) {
      pl->dense[i].fast_kind = plan.dense[i].fast_kind;
      pl->dense[i].exec_kind = plan.dense[i].fast_kind == SC_FAST_TTI ? 3
                               : use_fast[i]                           ? 2
                               : use_jit[i]                            ? 1
                                                                       : 0;
    }
    pl->launches = launches_per_run;
    cudaEvent_t whole[2];
    SC_CUDA(cudaEventCreate(&whole[0]));
    SC_CUDA(cudaEventCreate(&whole[1]));
    std::vector<cudaEvent_t> ev;
    if (timing) {
      ev.resize(2 * ns * (size_t)nsteps);
      for (auto &e : ev) SC_CUDA(cudaEventCreate(&e));
    }
    SC_CUDA(cudaEventRecord(whole[0], st));
    if (prologue(st)) return -1;
    const bool graphs = exec && !timing;
    const bool early = early_bytes && t_split > plan.t_m && t_split <= plan.t_M;
    if (graphs && early && split_graphs()) return -1;
    auto start_copy = [&]() -> int {
      SC_CUDA(cudaEventRecord(early_event, st));
      SC_CUDA(cudaStreamWaitEvent(early_stream, early_event, 0));
      SC_CUDA(cudaMemcpyAsync(early_host, early_dev, early_bytes, cudaMemcpyDeviceToHost,
                              early_stream));
      return 0;
    };
    if (graphs && early) {
      SC_CUDA(cudaGraphLaunch(exec_a, st));
      if (start_copy()) return -1;
      SC_CUDA(cudaGraphLaunch(exec_b, st));
    } else if (graphs) {
      SC_CUDA(cudaGraphLaunch(exec, st));
    } else {
      for (int t = plan.t_m; t <= plan.t_M; ++t)
        for (int k = 0; k < ns; ++k) {
          if (early && t == t_split && k == 0 && start_copy()) return -1;
          size_t eidx = 2 * ((size_t)(t - plan.t_m) * ns + k);
          if (timing) SC_CUDA(cudaEventRecord(ev[eidx], st));
          if (stage(k, t, st)) return -1;
          if (timing) SC_CUDA(cudaEventRecord(ev[eidx + 1], st));
        }
    }
    SC_CUDA(cudaEventRecord(whole[1], st));
    SC_CUDA(cudaStreamSynchronize(st));
    if (early) SC_CUDA(cudaStreamSynchronize(early_stream));
    SC_CUDA(cudaEventElapsedTime(&pl->total_ms, whole[0], whole[1]));
    cudaEventDestroy(whole[0]);
    cudaEventDestroy(whole[1]);
    if (timing) {
      for (int t = 0; t < nsteps; ++t)
        for (int k = 0; k < ns; ++k) {
          float ms = 0.f;
          size_t eidx = 2 * ((size_t)t * ns + k);
          SC_CUDA(cudaEventElapsedTime(&ms, ev[eidx], ev[eidx + 1]));
          pl->stage_ms[k] += ms;
        }
      for (auto &e : ev) cudaEventDestroy(e);
    }
    return 0;
  }
};

static int check_plan(const sc_plan *plan) {
  if (!plan) {
    sc_set_error("null plan");
    return -1;
  }
  if (plan->ndim < 1 || plan->ndim > 3) {
    sc_set_error("bad ndim %d", plan->ndim);
    return -1;
  }
  if (plan->dtype != SC_F32 && plan->dtype != SC_F64) {
    sc_set_error("bad dtype %d", plan->dtype);
    return -1;
  }
  return 0;
}

extern "C" int sc_prepare(sc_plan *plan, void **handle) {
  if (check_plan(plan) || !handle) return -1;
  RunBase *r = nullptr;
  int rc;
  if (plan->dtype == SC_F32) {
    auto *x = new Run<float>();
    rc = x->prepare(plan);
    r = x;
  } else {
    auto *x = new Run<double>();
    rc = x->prepare(plan);
    r = x;
  }
  if (rc != 0) {
    delete r;
    *handle = nullptr;
    return -1;
  }
  *handle = r;
  return 0;
}

extern "C" int sc_launch(void *handle, sc_plan *plan) {
  if (!handle || !plan) {
    sc_set_error("null run handle");
    return -1;
  }
  return reinterpret_cast<RunBase *>(handle)->launch(plan);
}

extern "C" int sc_multi_run(void *handle, void *comm, const sc_exchange *x, void *stream) {
  if (!handle || !x) {
    sc_set_error("null run handle or exchange");
    return -1;
  }
  return reinterpret_cast<RunBase *>(handle)->multi_run(reinterpret_cast<MultiComm *>(comm), *x,
                                                        reinterpret_cast<cudaStream_t>(stream));
}

extern "C" int sc_multi_exchange(void *handle, void *comm, const sc_exchange *x, int t,
                                 void *stream) {
  if (!handle || !x) {
    sc_set_error("null run handle or exchange");
    return -1;
  }
  return reinterpret_cast<RunBase *>(handle)->multi_exchange_step(
      reinterpret_cast<MultiComm *>(comm), *x, t, reinterpret_cast<cudaStream_t>(stream));
}

extern "C" int sc_revalidate(void *handle, void *stream) {
  if (!handle) {
    sc_set_error("null run handle");
    return -1;
  }
  return reinterpret_cast<RunBase *>(handle)->revalidate(reinterpret_cast<cudaStream_t>(stream));
}

extern "C" int sc_early_download(void *handle, int t_split, const void *dev, void *host,
                                 int64_t bytes) {
  if (!handle || bytes < 0) {
    sc_set_error("null run handle");
    return -1;
  }
  return reinterpret_cast<RunBase *>(handle)->early_download(t_split, dev, host, (size_t)bytes);
}

extern "C" int sc_step(void *handle, int t, void *stream) {
  if (!handle) {
    sc_set_error("null run handle");
    return -1;
  }
  return reinterpret_cast<RunBase *>(handle)->step(t, reinterpret_cast<cudaStream_t>(stream));
}

extern "C" int sc_step_part(void *handle, int t, void *stream, int x_lo, int x_hi, int p_lo,
                            int p_hi, int what) {
  if (!handle) {
    sc_set_error("null run handle");
    return -1;
  }
  return reinterpret_cast<RunBase *>(handle)->step_part(
      t, reinterpret_cast<cudaStream_t>(stream), x_lo, x_hi, p_lo, p_hi, what);
}

// ---------------------------------------------------------------------------
// FP32 peak microbenchmark (SURVEY.md §8d asks for a measured P32 next to the
// nominal one): independent packed FMA chains (FFMA2, 4 flops per lane per
// instruction) on every SM, timed with CUDA events.
__global__ void __launch_bounds__(256) fp32_peak_kernel(float *out, int iters, float a, float b) {
  uint64_t acc[8];
#pragma unroll
  for (int j = 0; j < 8; ++j) acc[j] = P2::pk(threadIdx.x * 1e-7f + j, j * 1e-7f);
  const uint64_t A = P2::pk(a, a), B = P2::pk(b, b);
#pragma unroll 1
  for (int i = 0; i < iters; ++i) {
#pragma unroll
    for (int k = 0; k < 16; ++k)
#pragma unroll
      for (int j = 0; j < 8; ++j) acc[j] = P2::fma(acc[j], A, B);
  }
  float s = 0.f;
#pragma unroll
  for (int j = 0; j < 8; ++j) s += P2::lo(acc[j]) + P2::hi(acc[j]);
  if (s == 1234.5f) out[0] = s;  // keep the chains alive
}

extern "C" int sc_measure_fp32(double *tflops) {
  int dev = 0, sms = 0;
  SC_CUDA(cudaGetDevice(&dev));
  SC_CUDA(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev));
  float *out = nullptr;
  SC_CUDA(cudaMalloc(&out, sizeof(float)));
  const int blocks = sms * 8, iters = 4096;
  cudaEvent_t e0, e1;
  SC_CUDA(cudaEventCreate(&e0));
  SC_CUDA(cudaEventCreate(&e1));
  fp32_peak_kernel<<<blocks, 256>>>(out, 64, 0.999f, 1e-6f);  // warm-up
  SC_CUDA(cudaEventRecord(e0));
  fp32_peak_kernel<<<blocks, 256>>>(out, iters, 0.999f, 1e-6f);
  SC_CUDA(cudaEventRecord(e1));
  SC_CUDA(cudaEventSynchronize(e1));
  float ms = 0.f;
  SC_CUDA(cudaEventElapsedTime(&ms, e0, e1));
  const double flops = (double)blocks * 256 * iters * 16 * 8 * 4;  // 2 lanes x 2 flops
  *tflops = flops / (ms * 1e-3) / 1e12;
  cudaEventDestroy(e0);
  cudaEventDestroy(e1);
  cudaFree(out);
  return 0;
}

// one warp per (x, y) row of 32-bit words: whole rows outside the box in x or
// y, the two z ends of the rows inside it
__global__ void upload_shell_kernel(uint32_t *__restrict__ dst, const uint32_t *__restrict__ src,
                                    int64_t nx, int64_t ny, int64_t nzw, int lo0, int hi0, int lo1,
                                    int hi1, int64_t zlo, int64_t zhi) {
  const int lane = threadIdx.x & 31;
  const int64_t wpb = blockDim.x >> 5;
  for (int64_t row = blockIdx.x * wpb + (threadIdx.x >> 5); row < nx * ny;
       row += (int64_t)gridDim.x * wpb) {
    const int64_t x = row / ny, y = row - x * ny;
    const uint32_t *s = src + row * nzw;
    uint32_t *d = dst + row * nzw;
    const bool inside = x >= lo0 && x <= hi0 && y >= lo1 && y <= hi1;
    if (!inside) {
      for (int64_t z = lane; z < nzw; z += 32) d[z] = s[z];
    } else {
      for (int64_t z = lane; z < zlo; z += 32) d[z] = s[z];
      for (int64_t z = zhi + lane; z < nzw; z += 32) d[z] = s[z];
    }
  }
}

extern "C" int sc_upload_shell(void *dst, const void *src, const int64_t ext[3],
                               const int32_t lo[3], const int32_t hi[3], int elem_bytes,
                               void *stream) {
  if (elem_bytes % 4 != 0 || !dst || !src) {
    sc_set_error("sc_upload_shell: bad arguments");
    return -1;
  }
  cudaPointerAttributes at;
  if (cudaPointerGetAttributes(&at, src) != cudaSuccess || at.type != cudaMemoryTypeHost ||
      !at.devicePointer) {
    cudaGetLastError();
    return 1;
  }
  const int64_t w = elem_bytes / 4;
  const int64_t rows = ext[0] * ext[1];
  if (rows <= 0 || ext[2] <= 0) return 0;
  const int blocks = (int)std::min<int64_t>((rows + 7) / 8, 148 * 16);
  upload_shell_kernel<<<blocks, 256, 0, reinterpret_cast<cudaStream_t>(stream)>>>(
      reinterpret_cast<uint32_t *>(dst), reinterpret_cast<const uint32_t *>(at.devicePointer),
      ext[0], ext[1], ext[2] * w, lo[0], hi[0], lo[1], hi[1], (int64_t)lo[2] * w,
      ((int64_t)hi[2] + 1) * w);
  SC_CUDA(cudaGetLastError());
  return 0;
}

extern "C" int sc_release(void *handle) {
  delete reinterpret_cast<RunBase *>(handle);
  return 0;
}

extern "C" int sc_run(sc_plan *plan) {
  void *h = nullptr;
  if (sc_prepare(plan, &h) != 0) return -1;
  int rc = sc_launch(h, plan);
  sc_release(h);
  return rc;
}
