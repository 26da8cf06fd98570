// Ghost-exchange transport over NCCL point-to-point (fr_nccl_init /
// fr_exchange).  Replaces the reference's pickled IPC messages
// (driver.py:150-201, worker.py:170-228) with one grouped ncclSend/ncclRecv
// round per exchange, enqueued on the caller's stream (graph-capturable, no
// host synchronisation).
//
// NCCL is resolved with dlopen at fr_nccl_init time rather than linked: a
// process that already runs PyTorch has its own libnccl.so.2 loaded, and the
// same soname then resolves to that copy instead of dragging a second NCCL
// build into the process.  Only the stable C types of nccl.h are used.
#include <dlfcn.h>
#include <nccl.h>
#include <cstdio>
#include <cstring>

#include "flowrec_b200.h"

#include <cstdarg>

namespace fr {
int fail_msg(const char* msg);  // capi.cu: sets fr_last_error()
}  // namespace fr

namespace {
int fail(const char* fmt, ...) __attribute__((format(printf, 1, 2)));
int fail(const char* fmt, ...) {
  char buf[512];
  va_list ap;
  va_start(ap, fmt);
  vsnprintf(buf, sizeof(buf), fmt, ap);
  va_end(ap);
  return fr::fail_msg(buf);
}
}  // namespace

struct fr_comm {
  ncclComm_t comm;
  int nranks, rank;
};

namespace {

struct NcclApi {
  bool ok = false;
  ncclResult_t (*get_unique_id)(ncclUniqueId*) = nullptr;
  ncclResult_t (*comm_init_rank)(ncclComm_t*, int, ncclUniqueId, int) = nullptr;
  ncclResult_t (*comm_destroy)(ncclComm_t) = nullptr;
  ncclResult_t (*group_start)() = nullptr;
  ncclResult_t (*group_end)() = nullptr;
  ncclResult_t (*send)(const void*, size_t, ncclDataType_t, int, ncclComm_t, cudaStream_t) = nullptr;
  ncclResult_t (*recv)(void*, size_t, ncclDataType_t, int, ncclComm_t, cudaStream_t) = nullptr;
  const char* (*error_string)(ncclResult_t) = nullptr;
};

NcclApi& api() {
  static NcclApi a;
  if (a.ok) return a;
  void* h = dlopen("libnccl.so.2", RTLD_NOW | RTLD_GLOBAL);
  if (!h) h = dlopen("libnccl.so", RTLD_NOW | RTLD_GLOBAL);
  if (!h) return a;
  a.get_unique_id = reinterpret_cast<decltype(a.get_unique_id)>(dlsym(h, "ncclGetUniqueId"));
  a.comm_init_rank = reinterpret_cast<decltype(a.comm_init_rank)>(dlsym(h, "ncclCommInitRank"));
  a.comm_destroy = reinterpret_cast<decltype(a.comm_destroy)>(dlsym(h, "ncclCommDestroy"));
  a.group_start = reinterpret_cast<decltype(a.group_start)>(dlsym(h, "ncclGroupStart"));
  a.group_end = reinterpret_cast<decltype(a.group_end)>(dlsym(h, "ncclGroupEnd"));
  a.send = reinterpret_cast<decltype(a.send)>(dlsym(h, "ncclSend"));
  a.recv = reinterpret_cast<decltype(a.recv)>(dlsym(h, "ncclRecv"));
  a.error_string = reinterpret_cast<decltype(a.error_string)>(dlsym(h, "ncclGetErrorString"));
  a.ok = a.get_unique_id && a.comm_init_rank && a.comm_destroy && a.group_start && a.group_end && a.send &&
         a.recv && a.error_string;
  return a;
}

int nccl_fail(const char* where, ncclResult_t r) {
  return fail("%s: %s", where, api().error_string ? api().error_string(r) : "NCCL error");
}

}  // namespace

extern "C" int fr_nccl_get_unique_id(void* id_out) {
  if (!id_out) return fail("fr_nccl_get_unique_id: NULL output");
  NcclApi& a = api();
  if (!a.ok) return fail("fr_nccl_get_unique_id: libnccl.so.2 not found");
  ncclUniqueId id;
  const ncclResult_t r = a.get_unique_id(&id);
  if (r != ncclSuccess) return nccl_fail("ncclGetUniqueId", r);
  std::memcpy(id_out, &id, sizeof(id));
  return 0;
}

extern "C" int fr_nccl_init(const void* unique_id, int nranks, int rank, fr_comm** out) {
  if (!unique_id || !out || nranks < 1 || rank < 0 || rank >= nranks) return fail("fr_nccl_init: bad arguments");
  NcclApi& a = api();
  if (!a.ok) return fail("fr_nccl_init: libnccl.so.2 not found");
  ncclUniqueId id;
  std::memcpy(&id, unique_id, sizeof(id));
  fr_comm* c = new fr_comm{nullptr, nranks, rank};
  const ncclResult_t r = a.comm_init_rank(&c->comm, nranks, id, rank);
  if (r != ncclSuccess) {
    delete c;
    return nccl_fail("ncclCommInitRank", r);
  }
  *out = c;
  return 0;
}

extern "C" int fr_nccl_destroy(fr_comm* c) {
  if (!c) return 0;
  const ncclResult_t r = api().comm_destroy(c->comm);
  delete c;
  return r == ncclSuccess ? 0 : nccl_fail("ncclCommDestroy", r);
}

// One exchange round: every send and receive of this rank in one NCCL group
// (so all edges progress concurrently and no pair can deadlock on ordering),
// enqueued on `stream`.  Buffers are device pointers of `dtype` elements.
extern "C" int fr_exchange(fr_comm* c, int n_send, const int* send_peers, const void* const* send_bufs,
                           const long long* send_counts, int n_recv, const int* recv_peers,
                           void* const* recv_bufs, const long long* recv_counts, int dtype, fr_stream_t stream) {
  if (!c || n_send < 0 || n_recv < 0 || (n_send && (!send_peers || !send_bufs || !send_counts)) ||
      (n_recv && (!recv_peers || !recv_bufs || !recv_counts)))
    return fail("fr_exchange: bad arguments");
  if (dtype != FR_F32 && dtype != FR_F64) return fail("fr_exchange: unknown dtype %d", dtype);
  const ncclDataType_t t = dtype == FR_F32 ? ncclFloat32 : ncclFloat64;
  for (int i = 0; i < n_send; ++i)
    if (send_peers[i] < 0 || send_peers[i] >= c->nranks || send_counts[i] < 0)
      return fail("fr_exchange: bad send %d (peer %d)", i, send_peers[i]);
  for (int i = 0; i < n_recv; ++i)
    if (recv_peers[i] < 0 || recv_peers[i] >= c->nranks || recv_counts[i] < 0)
      return fail("fr_exchange: bad receive %d (peer %d)", i, recv_peers[i]);
  NcclApi& a = api();
  ncclResult_t r = a.group_start();
  if (r != ncclSuccess) return nccl_fail("ncclGroupStart", r);
  for (int i = 0; i < n_send && r == ncclSuccess; ++i)
    r = a.send(send_bufs[i], size_t(send_counts[i]), t, send_peers[i], c->comm, stream);
  for (int i = 0; i < n_recv && r == ncclSuccess; ++i)
    r = a.recv(recv_bufs[i], size_t(recv_counts[i]), t, recv_peers[i], c->comm, stream);
  const ncclResult_t r2 = a.group_end();
  if (r != ncclSuccess) return nccl_fail("ncclSend/ncclRecv", r);
  if (r2 != ncclSuccess) return nccl_fail("ncclGroupEnd", r2);
  return 0;
}
