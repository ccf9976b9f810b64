// Multi-GPU data plane of the x-slab decomposition: NCCL
// communicator setup and the per-step ghost-plane exchange, called from the
// prepared run's t loop (api.cu, Run::multi_run) so the whole loop --
// boundary planes, exchange on a communication stream, interior planes --
// is one CUDA graph per rank.
//
// NCCL is resolved at run time (dlopen "libnccl.so.2"): when torch already
// loaded its NCCL the process's copy is reused, and the library itself has
// no link-time NCCL dependency (it loads on machines without NCCL).
#include <dlfcn.h>
#include <nccl.h>
#include <string.h>

#include <mutex>

#include "common.cuh"
#include "kernels.cuh"

namespace {

struct NcclApi {
  void *lib = nullptr;
  ncclResult_t (*getUniqueId)(ncclUniqueId *) = nullptr;
  ncclResult_t (*commInitRank)(ncclComm_t *, int, ncclUniqueId, int) = nullptr;
  ncclResult_t (*commDestroy)(ncclComm_t) = nullptr;
  ncclResult_t (*send)(const void *, size_t, ncclDataType_t, int, ncclComm_t,
                       cudaStream_t) = nullptr;
  ncclResult_t (*recv)(void *, size_t, ncclDataType_t, int, ncclComm_t, cudaStream_t) = nullptr;
  ncclResult_t (*groupStart)() = nullptr;
  ncclResult_t (*groupEnd)() = nullptr;
  const char *(*errorString)(ncclResult_t) = nullptr;
};

NcclApi *nccl() {
  static NcclApi api;
  static std::once_flag once;
  std::call_once(once, [] {
    const char *names[] = {"libnccl.so.2", "libnccl.so"};
    for (const char *n : names) {
      api.lib = dlopen(n, RTLD_NOW | RTLD_GLOBAL);
      if (api.lib) break;
    }
    if (!api.lib) return;
#define SC_SYM(field, name) api.field = reinterpret_cast<decltype(api.field)>(dlsym(api.lib, name))
    SC_SYM(getUniqueId, "ncclGetUniqueId");
    SC_SYM(commInitRank, "ncclCommInitRank");
    SC_SYM(commDestroy, "ncclCommDestroy");
    SC_SYM(send, "ncclSend");
    SC_SYM(recv, "ncclRecv");
    SC_SYM(groupStart, "ncclGroupStart");
    SC_SYM(groupEnd, "ncclGroupEnd");
    SC_SYM(errorString, "ncclGetErrorString");
#undef SC_SYM
  });
  if (!api.lib || !api.getUniqueId || !api.commInitRank || !api.send || !api.recv ||
      !api.groupStart || !api.groupEnd || !api.commDestroy) {
    sc_set_error("NCCL not available (dlopen libnccl.so.2 failed or symbols missing)");
    return nullptr;
  }
  return &api;
}

#define SC_NCCL(api, call)                                                           \
  do {                                                                               \
    ncclResult_t r_ = (call);                                                        \
    if (r_ != ncclSuccess) {                                                         \
      sc_set_error("%s failed: %s", #call,                                          \
                   (api)->errorString ? (api)->errorString(r_) : "nccl error");      \
      return -1;                                                                     \
    }                                                                                \
  } while (0)

}  // namespace

struct MultiComm {
  ncclComm_t comm = nullptr;
  int rank = 0, world = 1;
};

extern "C" int sc_multi_unique_id(void *id128) {
  NcclApi *a = nccl();
  if (!a || !id128) return -1;
  ncclUniqueId id;
  SC_NCCL(a, a->getUniqueId(&id));
  memcpy(id128, &id, sizeof(id));
  return 0;
}

extern "C" int sc_multi_init(const void *id128, int rank, int world, void **comm) {
  NcclApi *a = nccl();
  if (!a || !id128 || !comm) return -1;
  if (world < 1 || rank < 0 || rank >= world) {
    sc_set_error("bad rank %d / world %d", rank, world);
    return -1;
  }
  ncclUniqueId id;
  memcpy(&id, id128, sizeof(id));
  auto *c = new MultiComm();
  c->rank = rank;
  c->world = world;
  ncclResult_t r = a->commInitRank(&c->comm, world, id, rank);
  if (r != ncclSuccess) {
    sc_set_error("ncclCommInitRank failed: %s", a->errorString ? a->errorString(r) : "");
    delete c;
    return -1;
  }
  *comm = c;
  return 0;
}

extern "C" int sc_multi_finalize(void *comm) {
  auto *c = reinterpret_cast<MultiComm *>(comm);
  if (!c) return 0;
  NcclApi *a = nccl();
  if (a && c->comm) a->commDestroy(c->comm);
  delete c;
  return 0;
}

// Ghost planes of slot (t+1) of every exchanged field. Local storage x of a
// rank's window: [0, H) lower ghosts, [H, H+n) owned, [H+n, 2H+n) upper
// ghosts. The lower neighbour needs the first H owned planes, the upper one
// the last H; every recv is matched by the neighbour's send in the same
// field order (NCCL pairs point-to-point operations per peer in issue order).
int multi_exchange(MultiComm *c, const sc_exchange &x, const FieldDev *fields, int elem_bytes,
                   int t, cudaStream_t st) {
  if (x.lo_peer < 0 && x.hi_peer < 0) return 0;
  NcclApi *a = nccl();
  if (!a) return -1;
  if (!c) {
    sc_set_error("exchange with peers needs a communicator");
    return -1;
  }
  const ncclDataType_t dt = elem_bytes == 4 ? ncclFloat32 : ncclFloat64;
  const int H = x.halo, n = x.slab;
  SC_NCCL(a, a->groupStart());
  for (int i = 0; i < x.nfields; ++i) {
    const FieldDev &f = fields[x.field[i]];
    const int64_t plane = f.ext[2] * f.ext[3];
    if (f.ext[1] != n + 2 * H) {
      a->groupEnd();
      sc_set_error("field %d window has %lld x planes, expected %d", x.field[i],
                   (long long)f.ext[1], n + 2 * H);
      return -1;
    }
    char *slot = reinterpret_cast<char *>(f.data) +
                 (int64_t)sc_slot(t + 1, f.nslots) * f.ext[1] * plane * elem_bytes;
    const size_t cnt = (size_t)H * plane;
    auto at = [&](int xs) { return slot + (int64_t)xs * plane * elem_bytes; };
    if (x.lo_peer >= 0) {
      SC_NCCL(a, a->send(at(H), cnt, dt, x.lo_peer, c->comm, st));
      SC_NCCL(a, a->recv(at(0), cnt, dt, x.lo_peer, c->comm, st));
    }
    if (x.hi_peer >= 0) {
      SC_NCCL(a, a->send(at(n), cnt, dt, x.hi_peer, c->comm, st));
      SC_NCCL(a, a->recv(at(n + H), cnt, dt, x.hi_peer, c->comm, st));
    }
  }
  SC_NCCL(a, a->groupEnd());
  return 0;
}
