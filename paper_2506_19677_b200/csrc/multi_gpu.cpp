// multi_gpu.cpp — the sweep across GPUs.
//
// Trajectories are independent, so a sweep shards its rows across GPUs with
// no exchange during simulation (rows r ≡ rank mod N, every shard gets every
// cell type).  The one collective is the final statistics reduce: every
// rank's row and completion buffers hold its own rows and zeros elsewhere, so
// an NCCL uint64 SUM onto the root is an exact gather (x + 0 = x for every bit
// pattern, NaN included); the root then runs the bit-exact summary.
//
// Two ways in:
//   * one process per GPU (torchrun / MPI): saber_cuda_nccl_unique_id on one
//     rank, broadcast by the caller, saber_cuda_nccl_init on every rank, then
//     saber_cuda_sweep_plan_gather after each plan launch;
//   * one process driving several GPUs: saber_cuda_sweep_multi (one host
//     thread, stream and plan per device; ncclCommInitAll).
// NCCL is loaded on first use (dlopen): a process that already mapped a
// libnccl.so.2 (e.g. PyTorch's) shares it, so two NCCL builds never mix.
#include <cuda_runtime.h>
#include <dlfcn.h>
#include <nccl.h>

#include <algorithm>
#include <cstdlib>
#include <cstring>
#include <map>
#include <memory>
#include <mutex>
#include <string>
#include <thread>
#include <vector>

#include "saber_internal.h"

using namespace saberb200;

namespace {

saber_status fail(saber_status s, const std::string& m) { return set_error(s, m); }

// ------------------------------------------------------------ NCCL loading --
struct NcclApi {
  bool ok = false;
  std::string why;
  decltype(&ncclGetUniqueId) get_unique_id = nullptr;
  decltype(&ncclCommInitRank) init_rank = nullptr;
  decltype(&ncclCommInitAll) init_all = nullptr;
  decltype(&ncclCommDestroy) destroy = nullptr;
  decltype(&ncclReduce) reduce = nullptr;
  decltype(&ncclGroupStart) group_start = nullptr;
  decltype(&ncclGroupEnd) group_end = nullptr;
  decltype(&ncclGetErrorString) error_string = nullptr;
};

const NcclApi& nccl() {
  static NcclApi api;
  static std::once_flag once;
  std::call_once(once, [] {
    void* h = dlopen("libnccl.so.2", RTLD_NOW | RTLD_NOLOAD);  // already mapped (PyTorch)
    if (!h) {
      const char* env = std::getenv("SABER_NCCL_LIB");
      h = dlopen(env ? env : "libnccl.so.2", RTLD_NOW | RTLD_LOCAL);
    }
    if (!h) {
      api.why = std::string("cannot load libnccl.so.2: ") + dlerror();
      return;
    }
    auto sym = [&](auto& f, const char* name) {
      f = reinterpret_cast<std::remove_reference_t<decltype(f)>>(dlsym(h, name));
      return f != nullptr;
    };
    api.ok = sym(api.get_unique_id, "ncclGetUniqueId") && sym(api.init_rank, "ncclCommInitRank") &&
             sym(api.init_all, "ncclCommInitAll") && sym(api.destroy, "ncclCommDestroy") &&
             sym(api.reduce, "ncclReduce") && sym(api.group_start, "ncclGroupStart") &&
             sym(api.group_end, "ncclGroupEnd") && sym(api.error_string, "ncclGetErrorString");
    if (!api.ok) api.why = "libnccl.so.2 lacks a required symbol";
  });
  return api;
}

#define NCCL_TRY(expr)                                                                 \
  do {                                                                                 \
    const ncclResult_t r_ = (expr);                                                    \
    if (r_ != ncclSuccess)                                                             \
      return fail(SABER_ECUDA, std::string("NCCL: " #expr ": ") + nccl().error_string(r_)); \
  } while (0)

#define CUDA_OK(expr)                                                                  \
  do {                                                                                 \
    const cudaError_t e_ = (expr);                                                     \
    if (e_ != cudaSuccess)                                                             \
      return fail(SABER_ECUDA, std::string(#expr) + ": " + cudaGetErrorString(e_));    \
  } while (0)

}  // namespace

struct saber_nccl {
  ncclComm_t comm = nullptr;
  int n_ranks = 0, rank = 0, device = 0;
};

extern "C" saber_status saber_cuda_nccl_unique_id(uint8_t* id) {
  if (!id) return fail(SABER_EINVAL, "null argument");
  if (!nccl().ok) return fail(SABER_ECUDA, nccl().why);
  ncclUniqueId u;
  NCCL_TRY(nccl().get_unique_id(&u));
  std::memcpy(id, u.internal, NCCL_UNIQUE_ID_BYTES);
  return SABER_OK;
}

extern "C" saber_status saber_cuda_nccl_init(const uint8_t* id, int32_t n_ranks, int32_t rank,
                                             int32_t device, saber_nccl** out) {
  if (!id || !out) return fail(SABER_EINVAL, "null argument");
  *out = nullptr;
  if (n_ranks < 1 || rank < 0 || rank >= n_ranks) return fail(SABER_EINVAL, "bad rank / rank count");
  if (!nccl().ok) return fail(SABER_ECUDA, nccl().why);
  CUDA_OK(cudaSetDevice(device));
  auto c = std::make_unique<saber_nccl>();
  ncclUniqueId u;
  std::memcpy(u.internal, id, NCCL_UNIQUE_ID_BYTES);
  NCCL_TRY(nccl().init_rank(&c->comm, n_ranks, u, rank));
  c->n_ranks = n_ranks;
  c->rank = rank;
  c->device = device;
  *out = c.release();
  return SABER_OK;
}

extern "C" void saber_cuda_nccl_destroy(saber_nccl* c) {
  if (!c) return;
  if (c->comm && nccl().ok) nccl().destroy(c->comm);
  delete c;
}

namespace {

// The final statistics reduce of one rank's plan: rows and completion times
// summed onto `root` (in place there).
saber_status reduce_plan(saber_sweep_plan* plan, ncclComm_t comm, int rank, int root,
                         cudaStream_t s) {
  saber_sweep_buffers b{};
  if (saber_status e = saber_cuda_sweep_plan_buffers(plan, &b)) return e;
  NCCL_TRY(nccl().reduce(b.rows, b.rows, b.rows_bytes / 8, ncclUint64, ncclSum, root, comm, s));
  NCCL_TRY(nccl().reduce(b.completion_times, b.completion_times, b.completion_bytes / 8, ncclUint64,
                         ncclSum, root, comm, s));
  (void)rank;
  return SABER_OK;
}

}  // namespace

extern "C" saber_status saber_cuda_sweep_plan_gather(saber_sweep_plan* plan, saber_nccl* c,
                                                     int32_t root, void* stream) {
  if (!plan || !c) return fail(SABER_EINVAL, "null argument");
  if (root < 0 || root >= c->n_ranks) return fail(SABER_EINVAL, "bad root rank");
  CUDA_OK(cudaSetDevice(c->device));
  NCCL_TRY(nccl().group_start());
  const saber_status s = reduce_plan(plan, c->comm, c->rank, root, static_cast<cudaStream_t>(stream));
  NCCL_TRY(nccl().group_end());
  return s;
}

// ------------------------------------------------- one process, many GPUs --
namespace {

struct CommSet {
  std::vector<int> devices;
  std::vector<ncclComm_t> comms;
};

// Communicators are created once per device list and kept (ncclCommInitAll
// costs tens of milliseconds).
saber_status comms_for(const std::vector<int>& devs, std::vector<ncclComm_t>* out) {
  static std::mutex mu;
  static std::vector<CommSet> cache;
  std::lock_guard<std::mutex> lk(mu);
  for (const CommSet& c : cache)
    if (c.devices == devs) {
      *out = c.comms;
      return SABER_OK;
    }
  if (!nccl().ok) return fail(SABER_ECUDA, nccl().why);
  CommSet c;
  c.devices = devs;
  c.comms.resize(devs.size());
  NCCL_TRY(nccl().init_all(c.comms.data(), static_cast<int>(devs.size()), devs.data()));
  cache.push_back(c);
  *out = c.comms;
  return SABER_OK;
}

}  // namespace

extern "C" saber_status saber_cuda_sweep_multi(const saber_sweep_desc* desc, const int32_t* devices,
                                               int32_t n_devices, saber_sweep_out* out) {
  if (!desc || !out || !devices || n_devices < 1) return fail(SABER_EINVAL, "null argument");
  if (desc->shard_count != 1 || desc->shard_index != 0)
    return fail(SABER_EINVAL, "sweep_multi: the descriptor must describe the whole sweep");
  std::vector<int> devs(devices, devices + n_devices);
  for (int i = 0; i < n_devices; ++i)
    for (int j = 0; j < i; ++j)
      if (devs[static_cast<size_t>(i)] == devs[static_cast<size_t>(j)])
        return fail(SABER_EINVAL, "sweep_multi: a device appears twice (one rank per GPU)");
  const int n = n_devices;
  std::vector<saber_sweep_plan*> plans(static_cast<size_t>(n), nullptr);
  std::vector<cudaStream_t> streams(static_cast<size_t>(n), nullptr);
  struct Cleanup {
    std::vector<saber_sweep_plan*>* p;
    std::vector<cudaStream_t>* s;
    std::vector<int>* d;
    ~Cleanup() {
      for (size_t i = 0; i < p->size(); ++i) {
        cudaSetDevice((*d)[i]);
        if ((*s)[i]) cudaStreamSynchronize((*s)[i]);
        saber_cuda_sweep_plan_destroy((*p)[i]);
        if ((*s)[i]) cudaStreamDestroy((*s)[i]);
      }
    }
  } cleanup{&plans, &streams, &devs};
  std::vector<ncclComm_t> comms;  // (a 1-device communicator too: one code path)
  if (saber_status s = comms_for(devs, &comms)) return s;

  // One host thread per GPU: plan (host prologue + H2D) and the simulation of
  // its shard, concurrently on every device.
  std::vector<saber_status> st(static_cast<size_t>(n), SABER_OK);
  std::vector<std::string> msg(static_cast<size_t>(n));
  auto shard = [&](int r) {
    saber_sweep_desc d = *desc;
    d.device = devs[static_cast<size_t>(r)];
    d.shard_index = r;
    d.shard_count = n;
    saber_status s = SABER_OK;
    if (cudaSetDevice(d.device) != cudaSuccess ||
        cudaStreamCreateWithFlags(&streams[static_cast<size_t>(r)], cudaStreamNonBlocking) != cudaSuccess)
      s = fail(SABER_ECUDA, "sweep_multi: cannot create a stream on device " + std::to_string(d.device));
    if (s == SABER_OK) s = saber_cuda_sweep_plan_create(&d, &plans[static_cast<size_t>(r)]);
    if (s == SABER_OK) s = saber_cuda_sweep_plan_run(plans[static_cast<size_t>(r)], streams[static_cast<size_t>(r)]);
    st[static_cast<size_t>(r)] = s;
    if (s != SABER_OK) msg[static_cast<size_t>(r)] = saber_cuda_last_error();
  };
  std::vector<std::thread> pool;
  for (int r = 1; r < n; ++r) pool.emplace_back(shard, r);
  shard(0);
  for (auto& t : pool) t.join();
  for (int r = 0; r < n; ++r)
    if (st[static_cast<size_t>(r)] != SABER_OK)
      return fail(st[static_cast<size_t>(r)], "device " + std::to_string(devs[static_cast<size_t>(r)]) +
                                                  ": " + msg[static_cast<size_t>(r)]);

  // The final statistics reduce onto device 0 (one NCCL group over all ranks).
  {
    NCCL_TRY(nccl().group_start());
    saber_status s = SABER_OK;
    for (int r = 0; r < n && s == SABER_OK; ++r) {
      cudaSetDevice(devs[static_cast<size_t>(r)]);
      s = reduce_plan(plans[static_cast<size_t>(r)], comms[static_cast<size_t>(r)], r, 0,
                      streams[static_cast<size_t>(r)]);
    }
    NCCL_TRY(nccl().group_end());
    if (s != SABER_OK) return s;
    for (int r = 0; r < n; ++r) {
      CUDA_OK(cudaSetDevice(devs[static_cast<size_t>(r)]));
      CUDA_OK(cudaStreamSynchronize(streams[static_cast<size_t>(r)]));
    }
  }
  // Root: the summary and the results.
  CUDA_OK(cudaSetDevice(devs[0]));
  const bool want_summary = out->summary || out->best_cap_by_rps;
  if (want_summary)
    if (saber_status s = saber_cuda_sweep_plan_summarize(plans[0], streams[0])) return s;
  if (saber_status s = saber_cuda_sweep_plan_fetch(plans[0], out)) return s;
  double ms = 0.0;
  int32_t launches = 0;
  for (int r = 0; r < n; ++r) {
    double d = 0.0;
    int32_t l = 0;
    saber_cuda_sweep_plan_stats(plans[static_cast<size_t>(r)], &d, nullptr, &l);
    ms = std::max(ms, d);
    launches += l;
  }
  out->device_ms = ms;
  out->kernel_launches = launches;
  return SABER_OK;
}
