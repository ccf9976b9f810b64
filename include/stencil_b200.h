/*
 * stencil_b200.h -- C ABI of the B200 backend for the time-stepping loop
 * behind the reference's Operator.apply.
 *
 * Reference interface this replaces (paths under /root/reference/pkg/src/stencilc):
 *   - backend/operator.py:235-244  Operator.apply(steps, buffers, workers, **params)
 *       -> sc_run(): one call runs the whole t loop (t_m..t_M) on the GPU.
 *   - backend/interpreter.py:430-449  run(iet, buffers, env, workers)
 *       -> sc_run() executes the optimized clusters (dense stencil sweeps,
 *          sparse injection / interpolation) in the oracle's per-step order.
 *   - backend/interpreter.py:279-427  vec_exec / vec_eval (dense sweep)
 *       -> sc_dense: a straight-line operation program (sc_op) evaluated per
 *          grid point, or the fused sm_100a acoustic kernel when the program
 *          matches the canonical acoustic sequence (fast_kind != 0).
 *   - backend/interpreter.py:224-240  point() over p_src / p_rec loops
 *       -> sc_sparse: corner-ordered factor programs (inject / interpolate).
 *   - backend/codegen.py:23-35,242-270  emitted `int kernel(struct dataobj*..,
 *       const float dt, ..., const int t_M, const int t_m, ...)` returning 0
 *       -> same convention: plain pointers/extents in, 0 = success.
 *   - backend/interpreter.py:35-41  BackendError -> nonzero status +
 *       sc_last_error() text (CUDA errors carry cudaGetErrorString).
 *
 * Memory: every pointer in sc_field.data / sc_sparse.* is a DEVICE pointer
 * owned by the caller (torch tensors on the Python side); the library never
 * frees caller memory. Program arrays (ops/loads/consts) are HOST pointers
 * copied into device memory by the library.
 */
#ifndef STENCIL_B200_H
#define STENCIL_B200_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define SC_MAX_FIELDS 16
#define SC_MAX_DENSE 4
#define SC_MAX_SPARSE 16
#define SC_MAX_CORNERS 8
#define SC_MAX_FACTORS 8
#define SC_MAX_TABLES 16
#define SC_MAX_STAGES 24

enum sc_dtype { SC_F32 = 0, SC_F64 = 1 };

/* dense program opcodes (paper_1807_03032_b200/backend/program.py) */
enum sc_opcode { SC_LOAD = 0, SC_MULK = 1, SC_ADDK = 2, SC_MUL = 3,
                 SC_ADD = 4, SC_RCP = 5 };

/* sparse factor kinds */
enum sc_factor { SC_FAC_SPARSE = 0, SC_FAC_TABLE = 1, SC_FAC_CONST = 2,
                 SC_FAC_FIELD = 3 };

enum sc_fast { SC_FAST_NONE = 0, SC_FAST_ACOUSTIC_FACT = 1,
               SC_FAST_ACOUSTIC_BASIC = 2, SC_FAST_TTI = 3 };

typedef struct {
  void *data;       /* device pointer, C order                              */
  int64_t ext[4];   /* storage extents, outermost first                     */
  int32_t ndim;     /* number of storage axes (time axis included)          */
  int32_t nslots;   /* >0: axis 0 is a modulo time axis with nslots slots   */
  int32_t has_time; /* axis 0 is a time axis (modulo or saved)              */
  int32_t pad;
} sc_field;

typedef struct { int32_t op, dst, a, b; } sc_op;

typedef struct {
  int32_t field;    /* index into sc_plan.fields                           */
  int32_t tshift;   /* time offset k of an access at t+k                   */
  int32_t off[3];   /* storage index minus loop index, per space dim       */
  int32_t tdiv;     /* >1: sub-sampled time axis, slot (t / tdiv) + tshift
                       (snapshot functions, reference lowering.py:246-271) */
} sc_load;

typedef struct {
  int32_t nops, nloads, nconsts, out_reg, nregs;
  const sc_op *ops;         /* host */
  const sc_load *loads;     /* host */
  const double *consts;     /* host, already rounded to the dtype          */
  sc_load target;           /* written access                              */
  int32_t fast_kind;        /* enum sc_fast                                */
  int32_t so;               /* space order (fast kernels)                  */
  int32_t has_damp;         /* fast acoustic: damping term present         */
  int32_t u_field, m_field, damp_field;  /* fast acoustic operands         */
  int32_t nfast_consts;
  const double *fast_consts;  /* host: role constants of the fused kernel   */
  int32_t tti_fields[8];      /* TTI: p, r, m, damp, epsilon, delta, theta, phi */
  int32_t exec_kind;          /* out (sc_launch): 0 interpreter kernel,
                                 1 generated (NVRTC) kernel, 2 fused
                                 acoustic, 3 TTI                          */
  int32_t tguard;             /* >1: run only at steps t % tguard == 0
                                 (reference iet.py:134-150 Conditional)    */
  int32_t xblock;             /* >0: x planes per CTA chunk of the fused
                                 kernels (Operator(block={"x": ...}), the
                                 autotuner's knob); 0 = SM-count heuristic */
  void *scratch[6];           /* TTI: device g_p, g_r temporaries (field layout);
                                 f32: [2..5] per-point coefficients hoisted
                                 once per apply (2a, E, S, I: see tti.cu)  */
  int32_t iblock, jblock;     /* >0: thread-block extent of the generated
                                 kernels along the innermost / next space
                                 axis (Operator(block={"z": .., "y": ..}),
                                 reference loop blocking iet.py:377-423);
                                 0 = 32 x 8                               */
} sc_dense;

typedef struct {
  int32_t kind;             /* 0 = inject (increment), 1 = interpolate     */
  int32_t npoint, ncorner, ndim;
  const int32_t *base;      /* device int32 [ndim][npoint], corner-0 index */
  int32_t delta[SC_MAX_CORNERS][3];
  int32_t nfac[SC_MAX_CORNERS];
  int32_t fac_kind[SC_MAX_CORNERS][SC_MAX_FACTORS];
  int32_t fac_arg[SC_MAX_CORNERS][SC_MAX_FACTORS];
  double fac_const[SC_MAX_CORNERS][SC_MAX_FACTORS];
  double lead[SC_MAX_CORNERS];        /* folded leading Python-float product */
  const void *tables[SC_MAX_TABLES];  /* device per-point arrays (dtype)     */
  int32_t field;            /* dense field written (inject) / read (interp) */
  int32_t field_tshift;
  void *sparse;             /* device [nt][npoint] sparse time function    */
  int64_t sparse_nt;
  int32_t sparse_tshift;
  int32_t serial;           /* 1: targets collide -> exact serial order    */
} sc_sparse;

typedef struct {
  int32_t dtype;            /* enum sc_dtype                               */
  int32_t ndim;             /* grid dimensions (1..3)                      */
  int32_t lo[3], hi[3];     /* loop box x_m..x_M, y_m..y_M, z_m..z_M       */
  int32_t t_m, t_M;
  int32_t nfields;
  sc_field fields[SC_MAX_FIELDS];
  int32_t ndense;
  sc_dense dense[SC_MAX_DENSE];
  int32_t nsparse;
  sc_sparse sparse[SC_MAX_SPARSE];
  int32_t nstages;          /* per-step execution order                    */
  int32_t stages[SC_MAX_STAGES];  /* d: dense[d]; 100+s: sparse[s]         */
  void *stream;             /* cudaStream_t (0 = library stream)           */
  float stage_ms[SC_MAX_STAGES];  /* out: CUDA-event time per stage        */
  int32_t launches;         /* out: kernels launched                       */
  int32_t profile;          /* in: 1 = time every stage launch (events)    */
  float total_ms;           /* out: CUDA-event time of the whole t loop    */
  int32_t pad3;
} sc_plan;

/* library / device */
int sc_version(void);
const char *sc_last_error(void);
int sc_device_count(int *count);
int sc_set_device(int device);

/* run t_m..t_M once; returns 0 on success (= sc_prepare + sc_launch +
 * sc_release) */
int sc_run(sc_plan *plan);

/* prepare a run (device programs, fused-kernel state, CUDA graph of the t
 * loop) once and launch it repeatedly; plan outputs (stage_ms, total_ms,
 * launches) are written by sc_launch */
int sc_prepare(sc_plan *plan, void **handle);
int sc_launch(void *handle, sc_plan *plan);
int sc_release(void *handle);

/* re-check a prepared run's data-dependent preconditions (the fused acoustic
 * kernel's reciprocal operand range) on the current device buffers, ordered
 * on `stream` after re-uploaded inputs: 0 = the run may be relaunched,
 * 1 = prepare afresh, -1 = error. Lets Operator.apply reuse a prepared run
 * (plan, programs, CUDA graph) across applies of the same problem; the
 * reference re-interprets its cached artifact every apply
 * (pkg/src/stencilc/backend/operator.py:235-244). */
int sc_revalidate(void *handle, void *stream);

/* sc_launch may start a device->host copy while the loop still runs: the
 * run is cut into two graphs, steps [t_m, t_split) and [t_split, t_M], and
 * `bytes` bytes from `dev` to the page-locked `host` are copied on a private
 * stream as soon as the first graph is done (the rows of an interpolated
 * function that later steps no longer touch). sc_launch returns after both
 * the loop and the copy. bytes = 0 switches it off. Returns 0 = armed,
 * 1 = not applicable (profiled plan, empty part), -1 = error. The reference
 * has no transfers (its buffers are the host arrays, operator.py:235-244). */
int sc_early_download(void *handle, int t_split, const void *dev, void *host,
                      int64_t bytes);

/* launch the stages of ONE time step t asynchronously on `stream` (host-driven
 * loops: multi-GPU ghost-plane exchange between steps) */
int sc_step(void *handle, int t, void *stream);

/* part of time step t on `stream` (multi-GPU overlap: boundary planes first,
 * interior while the ghost planes travel). what: 1 = dense stages over loop x
 * planes [x_lo, x_hi] (fused acoustic kernel), 2 = injections, 4 =
 * interpolations over sparse points [p_lo, p_hi); what = 0 only checks that
 * every stage can run in parts. No reference counterpart:
 * the reference has no decomposition. */
int sc_step_part(void *handle, int t, void *stream, int x_lo, int x_hi,
                 int p_lo, int p_hi, int what);

/* ---- multi-GPU data plane (x-slab decomposition) --------
 * One process per GPU. Rank 0 creates an NCCL unique id (128 bytes) and
 * broadcasts it; every rank creates its communicator with sc_multi_init. A
 * run prepared over the rank's x-slab (plus `halo` ghost planes per side)
 * then executes its whole t loop with sc_multi_run: per step the boundary
 * planes (and the sources touching them) first, the ghost-plane exchange of
 * the time slot just written (ncclSend/ncclRecv of `halo` planes to the x-1 /
 * x+1 neighbours, grouped, on a communication stream) overlapped with the
 * interior planes, the next step ordered after the exchange -- the t loop
 * captured as one CUDA graph per (run, exchange). NCCL is loaded at run time
 * (dlopen of libnccl.so.2, the process's own copy if torch already loaded
 * one). No reference counterpart: the reference has no decomposition
 * (SURVEY.md §2.1). */
typedef struct {
  int32_t nfields;          /* written time functions to exchange            */
  int32_t field[4];         /* their sc_plan.fields indices                  */
  int32_t lo_peer, hi_peer; /* ranks of the x-1 / x+1 neighbours, -1: none   */
  int32_t halo;             /* ghost planes per side                         */
  int32_t slab;             /* owned x planes (the window is slab + 2 halo)  */
  int32_t overlap;          /* 1: boundary / exchange / interior split       */
  int32_t nearly;           /* early (boundary) x ranges, local loop coords  */
  int32_t early[2][2];
  int32_t interior[2];      /* interior x range (hi < lo: none)              */
  int32_t n_early_points;   /* sources [0, n) touch the boundary planes      */
  int32_t pad;
} sc_exchange;

int sc_multi_unique_id(void *id128);
int sc_multi_init(const void *id128, int rank, int world, void **comm);
int sc_multi_finalize(void *comm);
/* the run's t loop with the exchange (comm may be NULL when both peers are
 * -1: the split schedule alone) */
int sc_multi_run(void *handle, void *comm, const sc_exchange *x, void *stream);
/* one ghost-plane exchange of the slot written at step t (tests, host-driven
 * loops) */
int sc_multi_exchange(void *handle, void *comm, const sc_exchange *x, int t,
                      void *stream);

/* upload only the part of one [x][y][z] array that lies OUTSIDE the box
 * lo..hi (inclusive, storage coordinates): `dst` is the device array, `src`
 * the caller's page-locked host array of the same extents. Operator.apply
 * uses it for a time slot whose box the first time step overwrites before
 * anything reads it (u[t_m + 1] of a leapfrog update): the halo shell still
 * has to arrive, the interior does not. The kernel reads the host array in
 * place (unified addressing). Returns 0 = queued on `stream`, 1 = `src` is
 * not page-locked host memory (caller copies the whole array), -1 = error.
 * The reference uploads nothing: its buffers are the host arrays
 * (pkg/src/stencilc/backend/operator.py:235-244). */
int sc_upload_shell(void *dst, const void *src, const int64_t ext[3],
                    const int32_t lo[3], const int32_t hi[3], int elem_bytes,
                    void *stream);

/* measured dense FP32 throughput of this GPU (TFLOP/s, packed FMA chains on
 * every SM): the FP32 roofline denominator of bench.py */
int sc_measure_fp32(double *tflops);

/* size of sc_plan, for binding checks */
int64_t sc_plan_size(void);

#ifdef __cplusplus
}
#endif
#endif
