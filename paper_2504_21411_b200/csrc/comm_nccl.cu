// NCCL communicators and collectives behind the C ABI (opaque
// ncclComm_t handles created by galv_comm_init / galv_comm_split).  These are the ring
// collectives the cost model charges (collectives.py:49-69: all_gather_time,
// reduce_scatter_time, all_reduce_time; p2p_time :72-89) for callers that drive the kernels
// without torch.distributed.  libnccl.so.2 is resolved lazily with dlopen, so the library
// has no link-time NCCL dependency and, inside a PyTorch process, shares the NCCL that torch
// already loaded.  The Python runtime uses torch.distributed for the same plumbing and the
// NVLink kernels (tp_nvlink.cu, dp_nvlink.cu) for the data-parallel and tensor-parallel hot
// collectives.
#include <dlfcn.h>
#include <nccl.h>

#include <mutex>

#include "common.cuh"

namespace galv {
namespace nccl {

struct Api {
  decltype(&ncclGetUniqueId) get_unique_id = nullptr;
  decltype(&ncclCommInitRank) init_rank = nullptr;
  decltype(&ncclCommSplit) split = nullptr;
  decltype(&ncclCommDestroy) destroy = nullptr;
  decltype(&ncclAllReduce) all_reduce = nullptr;
  decltype(&ncclReduceScatter) reduce_scatter = nullptr;
  decltype(&ncclAllGather) all_gather = nullptr;
  decltype(&ncclSend) send = nullptr;
  decltype(&ncclRecv) recv = nullptr;
  decltype(&ncclGroupStart) group_start = nullptr;
  decltype(&ncclGroupEnd) group_end = nullptr;
  decltype(&ncclGetErrorString) error_string = nullptr;
  bool ok = false;
};

const Api& api() {
  static Api a;
  static std::once_flag once;
  std::call_once(once, [] {
    void* h = dlopen("libnccl.so.2", RTLD_NOW | RTLD_GLOBAL);
    if (!h) h = dlopen("libnccl.so", RTLD_NOW | RTLD_GLOBAL);
    if (!h) return;
#define GALV_SYM(field, name) a.field = reinterpret_cast<decltype(a.field)>(dlsym(h, name))
    GALV_SYM(get_unique_id, "ncclGetUniqueId");
    GALV_SYM(init_rank, "ncclCommInitRank");
    GALV_SYM(split, "ncclCommSplit");
    GALV_SYM(destroy, "ncclCommDestroy");
    GALV_SYM(all_reduce, "ncclAllReduce");
    GALV_SYM(reduce_scatter, "ncclReduceScatter");
    GALV_SYM(all_gather, "ncclAllGather");
    GALV_SYM(send, "ncclSend");
    GALV_SYM(recv, "ncclRecv");
    GALV_SYM(group_start, "ncclGroupStart");
    GALV_SYM(group_end, "ncclGroupEnd");
    GALV_SYM(error_string, "ncclGetErrorString");
#undef GALV_SYM
    a.ok = a.get_unique_id && a.init_rank && a.split && a.destroy && a.all_reduce &&
           a.reduce_scatter && a.all_gather && a.send && a.recv && a.group_start &&
           a.group_end && a.error_string;
  });
  return a;
}

inline ncclDataType_t dtype_of(int32_t d) { return d == 1 ? ncclBfloat16 : ncclFloat32; }

}  // namespace nccl
}  // namespace galv

using namespace galv;

#define GALV_NCCL_API()                                                   \
  const nccl::Api& A = nccl::api();                                       \
  GALV_CHECK_ARG(A.ok, "libnccl.so.2 not found or missing symbols");

#define GALV_NCCL_RET(expr)                                                               \
  do {                                                                                    \
    ncclResult_t _r = (expr);                                                             \
    if (_r != ncclSuccess) {                                                              \
      ::galv::set_error(std::string(__func__) + ": " + A.error_string(_r));               \
      return (int32_t)_r;                                                                 \
    }                                                                                     \
  } while (0)

extern "C" {

int32_t galv_comm_unique_id(void* out) {
  GALV_NCCL_API();
  GALV_CHECK_ARG(out, "bad arguments");
  ncclUniqueId id;
  GALV_NCCL_RET(A.get_unique_id(&id));
  memcpy(out, &id, sizeof(id));
  return 0;
}

int32_t galv_comm_init(const void* unique_id, int32_t nranks, int32_t rank, void** comm) {
  GALV_NCCL_API();
  GALV_CHECK_ARG(unique_id && comm && nranks >= 1 && rank >= 0 && rank < nranks,
                 "bad arguments");
  ncclUniqueId id;
  memcpy(&id, unique_id, sizeof(id));
  ncclComm_t c = nullptr;
  GALV_NCCL_RET(A.init_rank(&c, nranks, id, rank));
  *comm = c;
  return 0;
}

int32_t galv_comm_split(void* comm, int32_t color, int32_t key, void** out) {
  GALV_NCCL_API();
  GALV_CHECK_ARG(comm && out, "bad arguments");
  ncclComm_t c = nullptr;
  GALV_NCCL_RET(A.split(reinterpret_cast<ncclComm_t>(comm), color, key, &c, nullptr));
  *out = c;
  return 0;
}

int32_t galv_comm_destroy(void* comm) {
  GALV_NCCL_API();
  GALV_CHECK_ARG(comm, "bad arguments");
  GALV_NCCL_RET(A.destroy(reinterpret_cast<ncclComm_t>(comm)));
  return 0;
}

int32_t galv_all_reduce(void* comm, const void* send, void* recv, int64_t count, int32_t dtype,
                        void* stream) {
  GALV_NCCL_API();
  GALV_CHECK_ARG(comm && send && recv && count >= 0, "bad arguments");
  GALV_NCCL_RET(A.all_reduce(send, recv, (size_t)count, nccl::dtype_of(dtype), ncclSum,
                             reinterpret_cast<ncclComm_t>(comm), as_stream(stream)));
  return 0;
}

int32_t galv_reduce_scatter(void* comm, const void* send, void* recv, int64_t recv_count,
                            int32_t dtype, void* stream) {
  GALV_NCCL_API();
  GALV_CHECK_ARG(comm && send && recv && recv_count >= 0, "bad arguments");
  GALV_NCCL_RET(A.reduce_scatter(send, recv, (size_t)recv_count, nccl::dtype_of(dtype), ncclSum,
                                 reinterpret_cast<ncclComm_t>(comm), as_stream(stream)));
  return 0;
}

int32_t galv_all_gather(void* comm, const void* send, void* recv, int64_t send_count,
                        int32_t dtype, void* stream) {
  GALV_NCCL_API();
  GALV_CHECK_ARG(comm && send && recv && send_count >= 0, "bad arguments");
  GALV_NCCL_RET(A.all_gather(send, recv, (size_t)send_count, nccl::dtype_of(dtype),
                             reinterpret_cast<ncclComm_t>(comm), as_stream(stream)));
  return 0;
}

// one combined send/recv pair (pipeline boundary exchange, pipesim 1F1B; either side may be
// empty): a single NCCL group so two neighbours exchanging never deadlock
int32_t galv_sendrecv(void* comm, const void* send, int64_t send_bytes, int32_t peer_send,
                      void* recv, int64_t recv_bytes, int32_t peer_recv, void* stream) {
  GALV_NCCL_API();
  GALV_CHECK_ARG(comm && (send || send_bytes == 0) && (recv || recv_bytes == 0), "bad arguments");
  ncclComm_t c = reinterpret_cast<ncclComm_t>(comm);
  GALV_NCCL_RET(A.group_start());
  if (send_bytes > 0)
    GALV_NCCL_RET(A.send(send, (size_t)send_bytes, ncclUint8, peer_send, c, as_stream(stream)));
  if (recv_bytes > 0)
    GALV_NCCL_RET(A.recv(recv, (size_t)recv_bytes, ncclUint8, peer_recv, c, as_stream(stream)));
  GALV_NCCL_RET(A.group_end());
  return 0;
}

}  // extern "C"
