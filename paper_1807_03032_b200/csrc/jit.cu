// Generated dense kernels (DSE-driven kernel
// generation for equations no hand-written family kernel covers).
//
// The straight-line program the host compiles from the oracle's optimized
// tree (backend/program.py: LOAD / MULK / ADDK / MUL / ADD / RCP over
// registers, constants already rounded to the dtype) is emitted as CUDA C
// with every extent, loop bound, stencil offset and constant folded in,
// compiled at prepare time with NVRTC for sm_100a (-fmad=false, IEEE
// round-to-nearest intrinsics: the same operations in the same order as the
// interpreter kernel dense_generic_kernel, hence bit-identical results), and
// launched through the runtime's library API so the launches are captured in
// the per-apply CUDA graph like every other stage. One thread per grid point,
// innermost storage axis on threadIdx.x (coalesced), neighbour reuse through
// L1/L2.
#include <nvrtc.h>
#include <stdio.h>

#include <algorithm>
#include <map>
#include <mutex>
#include <string>
#include <vector>

#include "common.cuh"
#include "kernels.cuh"

namespace {

std::string lit(double v, bool f32) {
  char b[64];
  if (f32) {
    snprintf(b, sizeof b, "__int_as_float(0x%08x)", [&] {
      float x = (float)v;
      uint32_t u;
      memcpy(&u, &x, 4);
      return u;
    }());
  } else {
    uint64_t u;
    memcpy(&u, &v, 8);
    snprintf(b, sizeof b, "__longlong_as_double(0x%016llxLL)", (unsigned long long)u);
  }
  return b;
}

struct Ptr {
  int field, tshift, tdiv;
  bool operator<(const Ptr &o) const {
    return field != o.field ? field < o.field
                            : (tshift != o.tshift ? tshift < o.tshift : tdiv < o.tdiv);
  }
};

// process-wide cache: source text -> loaded kernel (operators re-prepared
// every apply reuse their compiled kernels)
std::mutex g_mu;
std::map<std::string, std::pair<cudaLibrary_t, cudaKernel_t>> g_cache;

}  // namespace

int jit_dense_build(const sc_plan *pl, const sc_dense &d, JitDense &out) {
  const bool f32 = pl->dtype == SC_F32;
  const char *T = f32 ? "float" : "double";
  const char *MUL = f32 ? "__fmul_rn" : "__dmul_rn";
  const char *ADD = f32 ? "__fadd_rn" : "__dadd_rn";
  const char *RCP = f32 ? "__frcp_rn" : "__drcp_rn";
  const int nd = pl->ndim;
  int n[3] = {1, 1, 1}, lo[3] = {0, 0, 0};
  for (int k = 0; k < nd; ++k) {
    lo[k] = pl->lo[k];
    n[k] = pl->hi[k] - pl->lo[k] + 1;
    if (n[k] <= 0) return 1;
  }
  // distinct (field, time shift, t-divisor) operands -> kernel pointer args
  std::map<Ptr, int> pid;
  std::vector<Ptr> ptrs;
  auto ptr_of = [&](const sc_load &l) {
    Ptr p{l.field, l.tshift, l.tdiv > 1 ? l.tdiv : 1};
    auto it = pid.find(p);
    if (it != pid.end()) return it->second;
    pid[p] = (int)ptrs.size();
    ptrs.push_back(p);
    return (int)ptrs.size() - 1;
  };
  const int tp = ptr_of(d.target);
  std::vector<int> lp(d.nloads);
  for (int i = 0; i < d.nloads; ++i) lp[i] = ptr_of(d.loads[i]);

  // index expression of an access: storage strides of the field (row-major
  // over the space axes; the time slot is folded into the pointer)
  auto index = [&](const sc_load &l) {
    const sc_field &f = pl->fields[l.field];
    const int a = f.has_time ? 1 : 0;
    std::string s;
    int64_t stride = 1;
    for (int k = nd - 1; k >= 0; --k) {
      char b[96];
      snprintf(b, sizeof b, "%s(i%d + %d) * %lldLL", s.empty() ? "" : " + ", k, l.off[k],
               (long long)stride);
      s += b;
      stride *= f.ext[a + k];
    }
    return s;
  };
  // thread block: innermost axis BX wide, next axis BY (block={...} of the
  // operator, the reference's loop blocking; default 32 x 8)
  const int BX = d.iblock > 0 ? std::min(d.iblock, 1024) : 32;
  const int BY = nd >= 2 ? (d.jblock > 0 ? std::max(1, std::min(d.jblock, 1024 / BX)) : 8) : 1;
  std::string src;
  src += "typedef ";
  src += T;
  src += " T;\nextern \"C\" __global__ void __launch_bounds__(" + std::to_string(BX * BY) +
         ") sc_jit(T *__restrict__ out";
  for (size_t i = 0; i < ptrs.size(); ++i) src += ", const T *__restrict__ p" + std::to_string(i);
  src += ") {\n";
  char b[512];
  // innermost axis on x (32 wide), next on y (8), outermost on z
  const int in = nd - 1;
  snprintf(b, sizeof b,
           "  const int i%d = %d + (int)(blockIdx.x * %d + threadIdx.x);\n"
           "  if (i%d >= %d) return;\n",
           in, lo[in], BX, in, lo[in] + n[in]);
  src += b;
  if (nd >= 2) {
    snprintf(b, sizeof b,
             "  const int i%d = %d + (int)(blockIdx.y * %d + threadIdx.y);\n"
             "  if (i%d >= %d) return;\n",
             nd - 2, lo[nd - 2], BY, nd - 2, lo[nd - 2] + n[nd - 2]);
    src += b;
  }
  if (nd == 3) {
    snprintf(b, sizeof b, "  const int i0 = %d + (int)blockIdx.z;\n", lo[0]);
    src += b;
  }
  snprintf(b, sizeof b, "  T r[%d];\n", d.nregs > 0 ? d.nregs : 1);
  src += b;
  for (int k = 0; k < d.nops; ++k) {
    const sc_op &o = d.ops[k];
    switch (o.op) {
      case SC_LOAD:
        snprintf(b, sizeof b, "  r[%d] = __ldg(p%d + %s);\n", o.dst, lp[o.a],
                 index(d.loads[o.a]).c_str());
        break;
      case SC_MULK:
        snprintf(b, sizeof b, "  r[%d] = %s(r[%d], %s);\n", o.dst, MUL, o.a,
                 lit(d.consts[o.b], f32).c_str());
        break;
      case SC_ADDK:
        if (o.a < 0)
          snprintf(b, sizeof b, "  r[%d] = %s;\n", o.dst, lit(d.consts[o.b], f32).c_str());
        else
          snprintf(b, sizeof b, "  r[%d] = %s(r[%d], %s);\n", o.dst, ADD, o.a,
                   lit(d.consts[o.b], f32).c_str());
        break;
      case SC_MUL: snprintf(b, sizeof b, "  r[%d] = %s(r[%d], r[%d]);\n", o.dst, MUL, o.a, o.b); break;
      case SC_ADD: snprintf(b, sizeof b, "  r[%d] = %s(r[%d], r[%d]);\n", o.dst, ADD, o.a, o.b); break;
      case SC_RCP: snprintf(b, sizeof b, "  r[%d] = %s(r[%d]);\n", o.dst, RCP, o.a); break;
      default: sc_set_error("jit: bad op %d", o.op); return -1;
    }
    src += b;
  }
  snprintf(b, sizeof b, "  out[%s] = r[%d];\n}\n", index(d.target).c_str(), d.out_reg);
  src += b;
  (void)tp;

  out.ptrs.clear();
  for (auto &p : ptrs) out.ptrs.push_back({p.field, p.tshift, p.tdiv});
  out.target_ptr = tp;
  out.block = dim3(BX, BY, 1);
  out.grid = dim3((unsigned)sc_ceil_div(n[in], BX), nd >= 2 ? (unsigned)sc_ceil_div(n[nd - 2], BY) : 1u,
                  nd == 3 ? (unsigned)n[0] : 1u);

  std::lock_guard<std::mutex> lk(g_mu);
  auto hit = g_cache.find(src);
  if (hit != g_cache.end()) {
    out.kern = hit->second.second;
    return 0;
  }
  nvrtcProgram prog;
  if (nvrtcCreateProgram(&prog, src.c_str(), "sc_jit.cu", 0, nullptr, nullptr) != NVRTC_SUCCESS) {
    sc_set_error("nvrtcCreateProgram failed");
    return -1;
  }
  const char *opts[] = {"--gpu-architecture=sm_100a", "-fmad=false", "-std=c++17",
                        "-default-device"};
  const nvrtcResult rc = nvrtcCompileProgram(prog, 4, opts);
  if (rc != NVRTC_SUCCESS) {
    size_t ln = 0;
    nvrtcGetProgramLogSize(prog, &ln);
    std::string log(ln, '\0');
    nvrtcGetProgramLog(prog, &log[0]);
    sc_set_error("nvrtc: %s: %.600s", nvrtcGetErrorString(rc), log.c_str());
    nvrtcDestroyProgram(&prog);
    return -1;
  }
  size_t cn = 0;
  nvrtcGetCUBINSize(prog, &cn);
  std::vector<char> cubin(cn);
  nvrtcGetCUBIN(prog, cubin.data());
  nvrtcDestroyProgram(&prog);
  cudaLibrary_t lib;
  SC_CUDA(cudaLibraryLoadData(&lib, cubin.data(), nullptr, nullptr, 0, nullptr, nullptr, 0));
  SC_CUDA(cudaLibraryGetKernel(&out.kern, lib, "sc_jit"));
  g_cache[src] = {lib, out.kern};
  return 0;
}

int jit_dense_launch(const JitDense &j, const FieldDev *fields, int dtype_bytes, int t,
                     cudaStream_t st) {
  std::vector<void *> vals(j.ptrs.size());
  for (size_t i = 0; i < j.ptrs.size(); ++i) {
    const JitPtr &p = j.ptrs[i];
    const FieldDev &f = fields[p.field];
    int64_t slot = 0, per = 1;
    if (f.has_time) {
      const int tt = load_time(t, p.tshift, p.tdiv);
      slot = f.nslots > 0 ? sc_slot(tt, f.nslots) : tt;
      for (int k = 1; k < f.ndim; ++k) per *= f.ext[k];
    }
    vals[i] = static_cast<char *>(f.data) + slot * per * dtype_bytes;
  }
  std::vector<void *> args;
  args.push_back(&vals[j.target_ptr]);
  for (size_t i = 0; i < vals.size(); ++i) args.push_back(&vals[i]);
  SC_CUDA(cudaLaunchKernel(reinterpret_cast<const void *>(j.kern), j.grid, j.block, args.data(), 0,
                           st));
  return 0;
}
