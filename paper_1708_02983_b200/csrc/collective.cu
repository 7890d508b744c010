// The round's packed-buffer allreduce behind the C ABI (SURVEY.md §8(b):
// esgd_nccl_init_all / esgd_allreduce_sum_f32 / esgd_nccl_destroy) for hosts
// that drive libesgd without torch.distributed — the replacement of the
// reference's tree_sum across workers (fabric/collectives.py:18-32) when the
// workers are processes on different GPUs. NCCL is loaded at run time
// (dlopen "libnccl.so.2": the copy the process already has, torch's or the
// system's), so libesgd itself has no link-time NCCL dependency and every
// other entry point works without it.
#include "esgd_common.cuh"

#include <dlfcn.h>
#include <nccl.h>

#include <mutex>

namespace esgd {
namespace {

struct Nccl {
  ncclResult_t (*get_unique_id)(ncclUniqueId*) = nullptr;
  ncclResult_t (*comm_init_rank)(ncclComm_t*, int, ncclUniqueId, int) = nullptr;
  ncclResult_t (*all_reduce)(const void*, void*, size_t, ncclDataType_t, ncclRedOp_t, ncclComm_t,
                             cudaStream_t) = nullptr;
  ncclResult_t (*comm_destroy)(ncclComm_t) = nullptr;
  const char* (*error_string)(ncclResult_t) = nullptr;
  bool ok = false;
};

const Nccl& nccl() {
  static Nccl n;
  static std::once_flag once;
  std::call_once(once, [] {
    void* h = dlopen("libnccl.so.2", RTLD_NOW | RTLD_GLOBAL);
    if (!h) h = dlopen("libnccl.so", RTLD_NOW | RTLD_GLOBAL);
    if (!h) return;
    n.get_unique_id = reinterpret_cast<decltype(n.get_unique_id)>(dlsym(h, "ncclGetUniqueId"));
    n.comm_init_rank = reinterpret_cast<decltype(n.comm_init_rank)>(dlsym(h, "ncclCommInitRank"));
    n.all_reduce = reinterpret_cast<decltype(n.all_reduce)>(dlsym(h, "ncclAllReduce"));
    n.comm_destroy = reinterpret_cast<decltype(n.comm_destroy)>(dlsym(h, "ncclCommDestroy"));
    n.error_string = reinterpret_cast<decltype(n.error_string)>(dlsym(h, "ncclGetErrorString"));
    n.ok = n.get_unique_id && n.comm_init_rank && n.all_reduce && n.comm_destroy && n.error_string;
  });
  return n;
}

int nccl_status(ncclResult_t r, const char* what) {
  if (r == ncclSuccess) return ESGD_OK;
  set_error("%s: NCCL error %d (%s)", what, (int)r, nccl().error_string(r));
  return ESGD_ERR_CUDA;
}

}  // namespace
}  // namespace esgd

static_assert(sizeof(ncclUniqueId) == ESGD_NCCL_ID_BYTES, "ncclUniqueId size");

extern "C" int esgd_nccl_available(void) { return esgd::nccl().ok ? 1 : 0; }

extern "C" int esgd_nccl_unique_id(void* id_out) {
  using namespace esgd;
  ESGD_REQUIRE(id_out, ESGD_ERR_INPUT, "nccl_unique_id: null output");
  ESGD_REQUIRE(nccl().ok, ESGD_ERR_UNSUPPORTED, "nccl_unique_id: libnccl.so.2 not loadable");
  ncclUniqueId id;
  int rc = nccl_status(nccl().get_unique_id(&id), "ncclGetUniqueId");
  if (rc) return rc;
  memcpy(id_out, &id, sizeof(id));
  return ESGD_OK;
}

extern "C" int esgd_nccl_init(esgd_comm_t* comm, const void* id, int32_t world, int32_t rank) {
  using namespace esgd;
  ESGD_REQUIRE(comm && id, ESGD_ERR_INPUT, "nccl_init: null argument");
  ESGD_REQUIRE(world >= 1 && rank >= 0 && rank < world, ESGD_ERR_INPUT,
               "nccl_init: rank %d outside world %d", rank, world);
  ESGD_REQUIRE(nccl().ok, ESGD_ERR_UNSUPPORTED, "nccl_init: libnccl.so.2 not loadable");
  ncclUniqueId uid;
  memcpy(&uid, id, sizeof(uid));
  ncclComm_t c = nullptr;
  int rc = nccl_status(nccl().comm_init_rank(&c, world, uid, rank), "ncclCommInitRank");
  if (rc) return rc;
  *comm = reinterpret_cast<esgd_comm_t>(c);
  return ESGD_OK;
}

extern "C" int esgd_allreduce_sum_f32(esgd_comm_t comm, float* buf, int64_t n, esgd_stream_t stream) {
  using namespace esgd;
  ESGD_REQUIRE(n >= 0, ESGD_ERR_SHAPE, "allreduce_sum: negative length");
  if (n == 0) return ESGD_OK;
  ESGD_REQUIRE(comm && buf, ESGD_ERR_INPUT, "allreduce_sum: null communicator or buffer");
  return nccl_status(nccl().all_reduce(buf, buf, (size_t)n, ncclFloat32, ncclSum,
                                       reinterpret_cast<ncclComm_t>(comm),
                                       reinterpret_cast<cudaStream_t>(stream)),
                     "ncclAllReduce");
}

extern "C" int esgd_nccl_destroy(esgd_comm_t comm) {
  using namespace esgd;
  if (!comm) return ESGD_OK;
  ESGD_REQUIRE(nccl().ok, ESGD_ERR_UNSUPPORTED, "nccl_destroy: libnccl.so.2 not loadable");
  return nccl_status(nccl().comm_destroy(reinterpret_cast<ncclComm_t>(comm)), "ncclCommDestroy");
}
