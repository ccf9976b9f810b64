// Device-side argument structs shared by the kernels and sc_run.
#pragma once

#include <vector>

#include "common.cuh"

#define SC_GEN_MAXREG 48

struct FieldDev {
  void *data;
  int64_t ext[4];
  int ndim, nslots, has_time, pad;
};

struct LoadDev {
  int field, tshift;
  int off[3];
  int tdiv;  // >1: sub-sampled time index t / tdiv
};

__host__ __device__ inline int load_time(int t, int tshift, int tdiv) {
  return (tdiv > 1 ? t / tdiv : t) + tshift;
}

template <typename T> struct DenseArgs {
  FieldDev fields[SC_MAX_FIELDS];
  const int4 *ops;
  const LoadDev *loads;
  const double *consts;
  int nops, out_reg, ndim;
  LoadDev target;
  int lo[3], n[3];
};

template <typename T> struct SparseArgs {
  int npoint, ncorner, ndim;
  const int32_t *base;
  int delta[SC_MAX_CORNERS][3];
  int nfac[SC_MAX_CORNERS];
  int fac_kind[SC_MAX_CORNERS][SC_MAX_FACTORS];
  int fac_arg[SC_MAX_CORNERS][SC_MAX_FACTORS];
  double fac_const[SC_MAX_CORNERS][SC_MAX_FACTORS];
  double lead[SC_MAX_CORNERS];
  const T *tables[SC_MAX_TABLES];
  int field_tshift;
  T *sparse;
  int sparse_tshift;
};

// ---------------------------------------------------------------------------
// Fused acoustic kernel (acoustic.cu)

struct FastAcoustic {
  int dtype, so, basic, has_damp;
  int lo[3], n[3];           // loop box
  int64_t ext[3];            // spatial storage extents (x, y, z)
  int nslots;
  void *u, *m, *damp;
  int xchunk;
  int var;                   // consumer variant (acoustic.cu)
  dim3 grid, block;
  size_t smem;
  double k[64];              // role constants (see backend/fastpath.py)
  alignas(64) CUtensorMap tm_uh, tm_ui, tm_m, tm_d;
};

template <typename T> int fast_acoustic_prepare(const sc_plan *pl, const sc_dense &d, FastAcoustic &fa);
template <typename T> int fast_acoustic_launch(const FastAcoustic &fa, int t, cudaStream_t st);
template <typename T> int fast_acoustic_check(const FastAcoustic &fa, cudaStream_t st);
void fast_acoustic_release(FastAcoustic &fa);

// Fused TTI step (tti.cu)
template <typename T>
int tti_launch(const sc_plan *pl, const sc_dense &d, const FieldDev *fields, int t, cudaStream_t st);
// generated dense kernels (jit.cu)
struct JitPtr {
  int field, tshift, tdiv;
};
struct JitDense {
  cudaKernel_t kern = nullptr;
  std::vector<JitPtr> ptrs;
  int target_ptr = 0;
  dim3 grid, block;
};
// 0 = built, 1 = not applicable (empty box), -1 = error (sc_last_error)
int jit_dense_build(const sc_plan *pl, const sc_dense &d, JitDense &out);
int jit_dense_launch(const JitDense &j, const FieldDev *fields, int dtype_bytes, int t,
                     cudaStream_t st);

// TMA two-pass TTI over loop x planes [x_lo, x_hi] (f32); 1 = not applicable
int tti_tma_launch(const sc_plan *pl, const sc_dense &d, const FieldDev *fields, int t,
                   cudaStream_t st, int x_lo, int x_hi);
bool tti_tma_ok(const sc_dense &d, const FieldDev *fields);
// forget the cached TTI launch configurations of stages first[0..n)
void tti_forget(const sc_dense *first, int n);

// per-apply prologue of the f32 TMA path (hoisted coefficients)
int tti_prologue(const sc_dense &d, const FieldDev *fields, cudaStream_t st);

// Multi-GPU data plane (multi.cu): NCCL loaded at run time
struct MultiComm;
// grouped send/recv of the ghost planes of slot (t + 1) of every exchanged
// field on `st`; comm may be null when there are no peers
int multi_exchange(MultiComm *c, const sc_exchange &x, const FieldDev *fields, int elem_bytes,
                   int t, cudaStream_t st);
