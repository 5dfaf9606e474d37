// comm.cpp — NCCL communicator behind the C-ABI (ifx_comm_*), for hosts that drive the
// Ulysses exchange without torch.distributed.
//
// SURVEY §8(b) asks the boundary for `ifx_comm_init(ncclUniqueId, rank, world)`: the
// reference's `WorkerGroup` + `all_to_all(group, per_worker_send)` (parallel.py:63-111) as
// a real communicator over NVLink / NVSwitch. The Python package keeps using
// torch.distributed (plumbing); a C / C++ host (or another language over FFI) gets the same
// collective here: a unique id made on rank 0 and shipped to the others out of band,
// communicator init, the variable-size byte all-to-all of the Ulysses re-shard
// (UlyssesComm.a2a_var), and an all-gather (e.g. of the CUDA IPC handles a peer mesh needs,
// ifx_ipc_handle / ifx_ipc_open).
//
// NCCL is opened with dlopen on first use, so the library still loads on a machine without
// it (every ifx_comm_* call then fails with IFX_ENCCL); in a process that already loaded
// NCCL (e.g. through torch) the loaded copy is reused.
#include <dlfcn.h>
#include <nccl.h>

#include <cstdint>
#include <cstring>
#include <mutex>
#include <string>

#include "../../include/ifx_abi.h"
#include "common_host.h"

namespace ifx {
namespace {

struct Nccl {
  void* so = nullptr;
  std::string why;
  ncclResult_t (*get_unique_id)(ncclUniqueId*) = nullptr;
  ncclResult_t (*comm_init_rank)(ncclComm_t*, int, ncclUniqueId, int) = nullptr;
  ncclResult_t (*comm_destroy)(ncclComm_t) = nullptr;
  ncclResult_t (*group_start)() = nullptr;
  ncclResult_t (*group_end)() = nullptr;
  ncclResult_t (*send)(const void*, size_t, ncclDataType_t, int, ncclComm_t, cudaStream_t) = nullptr;
  ncclResult_t (*recv)(void*, size_t, ncclDataType_t, int, ncclComm_t, cudaStream_t) = nullptr;
  ncclResult_t (*all_gather)(const void*, void*, size_t, ncclDataType_t, ncclComm_t, cudaStream_t) = nullptr;
  const char* (*error_string)(ncclResult_t) = nullptr;
};

const Nccl& nccl() {
  static Nccl n;
  static std::once_flag once;
  std::call_once(once, [] {
    for (const char* name : {"libnccl.so.2", "libnccl.so"}) {
      n.so = dlopen(name, RTLD_NOW | RTLD_LOCAL);
      if (n.so) break;
    }
    if (!n.so) {
      const char* e = dlerror();
      n.why = std::string("NCCL not found: ") + (e ? e : "dlopen failed");
      return;
    }
    auto sym = [&](const char* s) {
      void* p = dlsym(n.so, s);
      if (!p && n.why.empty()) n.why = std::string("NCCL symbol missing: ") + s;
      return p;
    };
    n.get_unique_id = reinterpret_cast<decltype(n.get_unique_id)>(sym("ncclGetUniqueId"));
    n.comm_init_rank = reinterpret_cast<decltype(n.comm_init_rank)>(sym("ncclCommInitRank"));
    n.comm_destroy = reinterpret_cast<decltype(n.comm_destroy)>(sym("ncclCommDestroy"));
    n.group_start = reinterpret_cast<decltype(n.group_start)>(sym("ncclGroupStart"));
    n.group_end = reinterpret_cast<decltype(n.group_end)>(sym("ncclGroupEnd"));
    n.send = reinterpret_cast<decltype(n.send)>(sym("ncclSend"));
    n.recv = reinterpret_cast<decltype(n.recv)>(sym("ncclRecv"));
    n.all_gather = reinterpret_cast<decltype(n.all_gather)>(sym("ncclAllGather"));
    n.error_string = reinterpret_cast<decltype(n.error_string)>(sym("ncclGetErrorString"));
  });
  return n;
}

int nccl_fail(const char* what, ncclResult_t r) {
  const Nccl& n = nccl();
  return fail(IFX_ENCCL, std::string(what) + ": " +
                             (n.error_string ? n.error_string(r) : "NCCL error " + std::to_string(r)));
}

}  // namespace
}  // namespace ifx

struct ifx_comm {
  ncclComm_t comm;
  int world, rank;
};

extern "C" {

int ifx_comm_unique_id(void* id_out) {
  if (id_out == nullptr) return ifx::fail(IFX_EDIM, "comm_unique_id: null pointer");
  const ifx::Nccl& n = ifx::nccl();
  if (!n.why.empty()) return ifx::fail(IFX_ENCCL, n.why);
  ncclUniqueId id;
  if (ncclResult_t r = n.get_unique_id(&id)) return ifx::nccl_fail("ncclGetUniqueId", r);
  std::memcpy(id_out, &id, sizeof(id));
  return IFX_OK;
}

int ifx_comm_init(const void* id, int world, int rank, ifx_comm** out) {
  if (id == nullptr || out == nullptr) return ifx::fail(IFX_EDIM, "comm_init: null pointer");
  *out = nullptr;
  if (world < 1 || rank < 0 || rank >= world)
    return ifx::fail(IFX_EDIM, "comm_init: rank must be in [0, world)");
  const ifx::Nccl& n = ifx::nccl();
  if (!n.why.empty()) return ifx::fail(IFX_ENCCL, n.why);
  ncclUniqueId uid;
  std::memcpy(&uid, id, sizeof(uid));
  ncclComm_t c = nullptr;
  if (ncclResult_t r = n.comm_init_rank(&c, world, uid, rank)) return ifx::nccl_fail("ncclCommInitRank", r);
  *out = new ifx_comm{c, world, rank};
  return IFX_OK;
}

int ifx_comm_destroy(ifx_comm* c) {
  if (c == nullptr) return IFX_OK;
  const ifx::Nccl& n = ifx::nccl();
  ncclResult_t r = n.comm_destroy(c->comm);
  delete c;
  return r ? ifx::nccl_fail("ncclCommDestroy", r) : IFX_OK;
}

int ifx_comm_all_to_all(ifx_comm* c, const void* send, const int64_t* send_off,
                        const int64_t* send_bytes, void* recv, const int64_t* recv_off,
                        const int64_t* recv_bytes, void* stream) {
  if (c == nullptr || send_off == nullptr || send_bytes == nullptr || recv_off == nullptr ||
      recv_bytes == nullptr)
    return ifx::fail(IFX_EDIM, "comm_all_to_all: null pointer");
  for (int p = 0; p < c->world; ++p) {
    if (send_off[p] < 0 || send_bytes[p] < 0 || recv_off[p] < 0 || recv_bytes[p] < 0)
      return ifx::fail(IFX_EDIM, "comm_all_to_all: negative offset or size");
    if ((send_bytes[p] > 0 && send == nullptr) || (recv_bytes[p] > 0 && recv == nullptr))
      return ifx::fail(IFX_EDIM, "comm_all_to_all: null buffer");
  }
  const ifx::Nccl& n = ifx::nccl();
  cudaStream_t st = static_cast<cudaStream_t>(stream);
  if (ncclResult_t r = n.group_start()) return ifx::nccl_fail("ncclGroupStart", r);
  ncclResult_t err = ncclSuccess;
  for (int p = 0; p < c->world && err == ncclSuccess; ++p) {
    if (send_bytes[p] > 0)
      err = n.send(static_cast<const uint8_t*>(send) + send_off[p], (size_t)send_bytes[p], ncclUint8,
                   p, c->comm, st);
    if (err == ncclSuccess && recv_bytes[p] > 0)
      err = n.recv(static_cast<uint8_t*>(recv) + recv_off[p], (size_t)recv_bytes[p], ncclUint8, p,
                   c->comm, st);
  }
  ncclResult_t end = n.group_end();
  if (err) return ifx::nccl_fail("ncclSend/ncclRecv", err);
  return end ? ifx::nccl_fail("ncclGroupEnd", end) : IFX_OK;
}

int ifx_comm_all_gather(ifx_comm* c, const void* send, int64_t bytes, void* recv, void* stream) {
  if (c == nullptr || (bytes > 0 && (send == nullptr || recv == nullptr)))
    return ifx::fail(IFX_EDIM, "comm_all_gather: null pointer");
  if (bytes < 0) return ifx::fail(IFX_EDIM, "comm_all_gather: negative size");
  if (bytes == 0) return IFX_OK;
  const ifx::Nccl& n = ifx::nccl();
  if (ncclResult_t r = n.all_gather(send, recv, (size_t)bytes, ncclUint8, c->comm,
                                    static_cast<cudaStream_t>(stream)))
    return ifx::nccl_fail("ncclAllGather", r);
  return IFX_OK;
}

int ifx_comm_size(const ifx_comm* c, int* world, int* rank) {
  if (c == nullptr) return ifx::fail(IFX_EDIM, "comm_size: null communicator");
  if (world) *world = c->world;
  if (rank) *rank = c->rank;
  return IFX_OK;
}

}  // extern "C"
