// The sequence-parallel exchanges of the path as C-ABI entry points over
// NCCL (SURVEY.md §8b "lsrm_allgather_kv / lsrm_dispatch (NCCL comm handle
// passed in)"), so a non-Python host can run block-aware sequence
// parallelism with this library alone:
//
//   lsrm_comm_unique_id / lsrm_comm_init / lsrm_comm_destroy  — communicator
//   lsrm_allgather_kv   — All-gather-KV (`lsrm/seq_parallel.py:181-218`):
//                         all-gather-v of every rank's packed KV shard into a
//                         staging buffer, then the placement segment copies
//                         into the canonical K / V / compressed buffers
//   lsrm_all_to_all_v   — dispatch / return token all-to-all
//                         (`lsrm/seq_parallel.py:146-178`)
//
// NCCL is bound at run time (dlopen "libnccl.so.2", preferring the copy the
// process already loaded, e.g. torch's), so the library has no link-time
// NCCL dependency and shares one NCCL with the host framework. Every call is
// enqueued on the caller's stream (grouped ncclSend / ncclRecv: the shards
// are uneven, so these are all-gather-v / all-to-all-v).
#include <dlfcn.h>
#include <string.h>

#include "common.cuh"

namespace {

// the subset of nccl.h this file uses (ABI-stable since NCCL 2.7)
typedef void* ncclComm_t;
typedef struct { char internal[128]; } ncclUniqueId;
typedef int ncclResult_t;   // 0 = ncclSuccess
constexpr int kNcclUint8 = 1;  // ncclUint8

struct Nccl {
  ncclResult_t (*get_unique_id)(ncclUniqueId*) = nullptr;
  ncclResult_t (*comm_init_rank)(ncclComm_t*, int, ncclUniqueId, int) = nullptr;
  ncclResult_t (*comm_destroy)(ncclComm_t) = nullptr;
  ncclResult_t (*group_start)() = nullptr;
  ncclResult_t (*group_end)() = nullptr;
  ncclResult_t (*send)(const void*, size_t, int, int, ncclComm_t, cudaStream_t) = nullptr;
  ncclResult_t (*recv)(void*, size_t, int, int, ncclComm_t, cudaStream_t) = nullptr;
  const char* (*error_string)(ncclResult_t) = nullptr;
  bool ok = false;
};

Nccl& nccl() {
  static Nccl n = [] {
    Nccl r;
    void* h = dlopen("libnccl.so.2", RTLD_NOW | RTLD_NOLOAD);
    if (!h) h = dlopen("libnccl.so.2", RTLD_NOW | RTLD_GLOBAL);
    if (!h) return r;
    r.get_unique_id = (decltype(r.get_unique_id))dlsym(h, "ncclGetUniqueId");
    r.comm_init_rank = (decltype(r.comm_init_rank))dlsym(h, "ncclCommInitRank");
    r.comm_destroy = (decltype(r.comm_destroy))dlsym(h, "ncclCommDestroy");
    r.group_start = (decltype(r.group_start))dlsym(h, "ncclGroupStart");
    r.group_end = (decltype(r.group_end))dlsym(h, "ncclGroupEnd");
    r.send = (decltype(r.send))dlsym(h, "ncclSend");
    r.recv = (decltype(r.recv))dlsym(h, "ncclRecv");
    r.error_string = (decltype(r.error_string))dlsym(h, "ncclGetErrorString");
    r.ok = r.get_unique_id && r.comm_init_rank && r.comm_destroy && r.group_start &&
           r.group_end && r.send && r.recv && r.error_string;
    return r;
  }();
  return n;
}

#define LSRM_NCCL_LOADED()                                                          \
  do {                                                                              \
    if (!nccl().ok)                                                                 \
      return ::lsrm::set_error(LSRM_E_CUDA, "NCCL (libnccl.so.2) could not be loaded"); \
  } while (0)

#define LSRM_NCCL(expr)                                                              \
  do {                                                                               \
    ncclResult_t _r = (expr);                                                        \
    if (_r != 0)                                                                     \
      return ::lsrm::set_error(LSRM_E_CUDA, "%s failed: %s (%s:%d)", #expr,          \
                               nccl().error_string(_r), __FILE__, __LINE__);         \
  } while (0)

// grouped send/recv of byte ranges: to peer p send [send + so[p], +sn[p]),
// from peer p receive into [recv + ro[p], +rn[p]); own range copied locally
int grouped_exchange(ncclComm_t comm, int rank, int world, const uint8_t* send,
                     const int64_t* so, const int64_t* sn, uint8_t* recv, const int64_t* ro,
                     const int64_t* rn, cudaStream_t st) {
  using namespace lsrm;
  if (rn[rank] > 0) {
    LSRM_REQUIRE(sn[rank] == rn[rank], "exchange: own send (%lld B) != own receive (%lld B)",
                 (long long)sn[rank], (long long)rn[rank]);
    LSRM_CUDA(cudaMemcpyAsync(recv + ro[rank], send + so[rank], (size_t)rn[rank],
                              cudaMemcpyDeviceToDevice, st));
  }
  LSRM_NCCL(nccl().group_start());
  for (int p = 0; p < world; ++p) {
    if (p == rank) continue;
    if (sn[p] > 0) {
      ncclResult_t r = nccl().send(send + so[p], (size_t)sn[p], kNcclUint8, p, comm, st);
      if (r != 0) { nccl().group_end(); LSRM_NCCL(r); }
    }
    if (rn[p] > 0) {
      ncclResult_t r = nccl().recv(recv + ro[p], (size_t)rn[p], kNcclUint8, p, comm, st);
      if (r != 0) { nccl().group_end(); LSRM_NCCL(r); }
    }
  }
  LSRM_NCCL(nccl().group_end());
  return LSRM_OK;
}

}  // namespace

extern "C" int lsrm_comm_unique_id(uint8_t* id_out) {
  using namespace lsrm;
  LSRM_NCCL_LOADED();
  LSRM_REQUIRE(id_out != nullptr, "comm_unique_id: null output");
  ncclUniqueId id;
  LSRM_NCCL(nccl().get_unique_id(&id));
  memcpy(id_out, id.internal, sizeof(id.internal));
  return LSRM_OK;
}

extern "C" int lsrm_comm_init(const uint8_t* id, int world, int rank, void** comm_out) {
  using namespace lsrm;
  LSRM_NCCL_LOADED();
  LSRM_REQUIRE(id && comm_out, "comm_init: null argument");
  LSRM_REQUIRE(world >= 1 && rank >= 0 && rank < world, "comm_init: rank %d of %d", rank, world);
  ncclUniqueId uid;
  memcpy(uid.internal, id, sizeof(uid.internal));
  ncclComm_t c = nullptr;
  LSRM_NCCL(nccl().comm_init_rank(&c, world, uid, rank));
  *comm_out = c;
  return LSRM_OK;
}

extern "C" int lsrm_comm_destroy(void* comm) {
  using namespace lsrm;
  LSRM_NCCL_LOADED();
  if (comm) LSRM_NCCL(nccl().comm_destroy((ncclComm_t)comm));
  return LSRM_OK;
}

extern "C" int lsrm_allgather_kv(void* comm, int rank, int world, const void* shard,
                                 int64_t shard_bytes, void* stage, const int64_t* stage_off,
                                 const int64_t* const* segs, const int64_t* n_segs,
                                 void* const* dst, int n_dst, void* stream) {
  using namespace lsrm;
  LSRM_NCCL_LOADED();
  LSRM_REQUIRE(comm && stage && stage_off, "allgather_kv: null argument");
  LSRM_REQUIRE(world >= 1 && rank >= 0 && rank < world, "allgather_kv: rank %d of %d", rank,
               world);
  LSRM_REQUIRE(stage_off[rank + 1] - stage_off[rank] == shard_bytes,
               "allgather_kv: own shard %lld B != its staging slot %lld B",
               (long long)shard_bytes, (long long)(stage_off[rank + 1] - stage_off[rank]));
  // every peer receives the whole shard: send range = [0, shard_bytes)
  int64_t so[1024], sn[1024], ro[1024], rn[1024];
  LSRM_REQUIRE(world <= 1024, "allgather_kv: world %d > 1024", world);
  for (int p = 0; p < world; ++p) {
    so[p] = 0;
    sn[p] = shard_bytes;
    ro[p] = stage_off[p];
    rn[p] = stage_off[p + 1] - stage_off[p];
  }
  cudaStream_t st = as_stream(stream);
  int rc = grouped_exchange((ncclComm_t)comm, rank, world, (const uint8_t*)shard, so, sn,
                            (uint8_t*)stage, ro, rn, st);
  if (rc != LSRM_OK) return rc;
  // placement: staging -> canonical global buffers (stream-ordered after the
  // receives)
  for (int i = 0; i < n_dst; ++i) {
    rc = lsrm_copy_segments(stage, dst[i], segs[i], n_segs[i], stream);
    if (rc != LSRM_OK) return rc;
  }
  return LSRM_OK;
}

extern "C" int lsrm_all_to_all_v(void* comm, int rank, int world, const void* send,
                                 const int64_t* send_bytes, void* recv,
                                 const int64_t* recv_bytes, void* stream) {
  using namespace lsrm;
  LSRM_NCCL_LOADED();
  LSRM_REQUIRE(comm && send_bytes && recv_bytes, "all_to_all_v: null argument");
  LSRM_REQUIRE(world >= 1 && world <= 1024 && rank >= 0 && rank < world,
               "all_to_all_v: rank %d of %d", rank, world);
  int64_t so[1024], ro[1024];
  int64_t a = 0, b = 0;
  for (int p = 0; p < world; ++p) {
    LSRM_REQUIRE(send_bytes[p] >= 0 && recv_bytes[p] >= 0, "all_to_all_v: negative size");
    so[p] = a;
    ro[p] = b;
    a += send_bytes[p];
    b += recv_bytes[p];
  }
  return grouped_exchange((ncclComm_t)comm, rank, world, (const uint8_t*)send, so, send_bytes,
                          (uint8_t*)recv, ro, recv_bytes, as_stream(stream));
}
