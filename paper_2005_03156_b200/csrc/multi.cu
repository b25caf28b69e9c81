// multi.cu -- the multi-GPU entry of the C-ABI (fm_multi_*): the
// reference's run_chunked (parallel.hpp:30-82) one level up, for C++ callers
// that own several GPUs in one process.
//
// One index replica per device, built concurrently (every replica is the
// same deterministic build).  A host batch is split into contiguous,
// balanced shards (parallel.shard_range: the first n % N devices take one
// extra point), each device runs the host-buffer pipeline of fm_query_host
// on its shard from its own host thread -- no data-path exchange, a point's
// leaf depends only on the point and the read-only index -- and the
// optional per-block int64 histogram stays on the devices and is summed
// with one ncclAllReduce over NVLink (BASELINE config 5).  NCCL is loaded
// at run time (dlopen "libnccl.so.2": torch's bundled copy when it is
// already mapped, else the system one), so callers that never ask for a
// histogram do not need it; asking for one without NCCL fails loudly.
#include <cuda_runtime.h>
#include <dlfcn.h>
#include <nccl.h>

#include <algorithm>
#include <cstdint>
#include <string>
#include <thread>
#include <vector>

#include "../../include/fastmap_b200.h"

__attribute__((visibility("hidden"))) fm_status fm_set_error(fm_status s, const char* msg);
__attribute__((visibility("hidden"))) fm_status query_host_impl(
    const fm_index* cindex, int mode, const double* h_lonlat, std::uint64_t n, std::int32_t* h_out,
    std::int64_t* h_hist, std::int64_t* d_hist_accum, fm_query_counters* h_counters);

namespace {

struct Nccl {
  void* so = nullptr;
  ncclResult_t (*comm_init_all)(ncclComm_t*, int, const int*) = nullptr;
  ncclResult_t (*all_reduce)(const void*, void*, size_t, ncclDataType_t, ncclRedOp_t, ncclComm_t,
                             cudaStream_t) = nullptr;
  ncclResult_t (*group_start)() = nullptr;
  ncclResult_t (*group_end)() = nullptr;
  ncclResult_t (*comm_destroy)(ncclComm_t) = nullptr;
  const char* (*error_string)(ncclResult_t) = nullptr;

  bool load(std::string* why) {
    if (so) return true;
    so = dlopen("libnccl.so.2", RTLD_NOW | RTLD_GLOBAL);
    if (!so) {
      *why = std::string("libnccl.so.2 not loadable: ") + dlerror();
      return false;
    }
    comm_init_all = reinterpret_cast<decltype(comm_init_all)>(dlsym(so, "ncclCommInitAll"));
    all_reduce = reinterpret_cast<decltype(all_reduce)>(dlsym(so, "ncclAllReduce"));
    group_start = reinterpret_cast<decltype(group_start)>(dlsym(so, "ncclGroupStart"));
    group_end = reinterpret_cast<decltype(group_end)>(dlsym(so, "ncclGroupEnd"));
    comm_destroy = reinterpret_cast<decltype(comm_destroy)>(dlsym(so, "ncclCommDestroy"));
    error_string = reinterpret_cast<decltype(error_string)>(dlsym(so, "ncclGetErrorString"));
    if (!comm_init_all || !all_reduce || !group_start || !group_end || !comm_destroy || !error_string) {
      *why = "libnccl.so.2 lacks the collective entry points";
      return false;
    }
    return true;
  }
};

fm_status fail(fm_status s, const std::string& msg) { return fm_set_error(s, msg.c_str()); }

// the caller's current device is restored on return
struct DeviceRestore {
  int prev = -1;
  DeviceRestore() {
    if (cudaGetDevice(&prev) != cudaSuccess) prev = -1;
  }
  ~DeviceRestore() {
    if (prev >= 0) cudaSetDevice(prev);
  }
};

}  // namespace

struct fm_multi {
  std::vector<int> devices;
  std::vector<fm_index*> replicas;
  std::uint64_t n_polys = 0;
  // histogram reduce (created on first use)
  Nccl nccl;
  std::vector<ncclComm_t> comms;
  std::vector<cudaStream_t> streams;
  std::vector<std::int64_t*> d_hist;
};

namespace {

void release(fm_multi* m) {
  for (std::size_t k = 0; k < m->d_hist.size(); ++k) {
    if (m->d_hist[k]) {
      cudaSetDevice(m->devices[k]);
      cudaFree(m->d_hist[k]);
    }
  }
  for (std::size_t k = 0; k < m->streams.size(); ++k) {
    if (m->streams[k]) {
      cudaSetDevice(m->devices[k]);
      cudaStreamDestroy(m->streams[k]);
    }
  }
  for (ncclComm_t c : m->comms) {
    if (c && m->nccl.comm_destroy) m->nccl.comm_destroy(c);
  }
  for (fm_index* ix : m->replicas) fm_index_destroy(ix);
  delete m;
}

fm_status setup_reduce(fm_multi* m) {
  if (!m->comms.empty()) return FM_OK;
  std::string why;
  if (!m->nccl.load(&why)) return fail(FM_ERR_RUNTIME, "histogram reduce needs NCCL: " + why);
  const int nd = static_cast<int>(m->devices.size());
  std::vector<ncclComm_t> comms(nd, nullptr);
  const ncclResult_t r = m->nccl.comm_init_all(comms.data(), nd, m->devices.data());
  if (r != ncclSuccess) return fail(FM_ERR_RUNTIME, std::string("ncclCommInitAll: ") + m->nccl.error_string(r));
  m->comms = comms;
  m->streams.assign(nd, nullptr);
  m->d_hist.assign(nd, nullptr);
  const std::uint64_t bytes = std::max<std::uint64_t>(1, m->n_polys) * 8;
  for (int k = 0; k < nd; ++k) {
    if (cudaSetDevice(m->devices[k]) != cudaSuccess ||
        cudaStreamCreateWithFlags(&m->streams[k], cudaStreamNonBlocking) != cudaSuccess ||
        cudaMalloc(&m->d_hist[k], bytes) != cudaSuccess) {
      return fail(FM_ERR_CUDA, "histogram buffers: " + std::string(cudaGetErrorString(cudaGetLastError())));
    }
  }
  return FM_OK;
}

}  // namespace

extern "C" {

fm_status fm_multi_build(const double* vertex_lonlat, const std::uint64_t* ring_offsets,
                         std::uint64_t n_rings, const std::uint64_t* poly_ring_offsets,
                         std::uint64_t n_polys, const fm_build_params* params, const int* devices,
                         int n_devices, fm_multi** out) {
  if (!out) return fail(FM_ERR_INVALID_ARGUMENT, "out is null");
  *out = nullptr;
  if (!params || !devices || n_devices < 1) {
    return fail(FM_ERR_INVALID_ARGUMENT, "need build params and at least one device");
  }
  int count = 0;
  if (cudaGetDeviceCount(&count) != cudaSuccess || count == 0) {
    return fail(FM_ERR_NO_DEVICE, "no CUDA device");
  }
  std::vector<int> devs(devices, devices + n_devices);
  for (int k = 0; k < n_devices; ++k) {
    if (devs[k] < 0 || devs[k] >= count) return fail(FM_ERR_INVALID_ARGUMENT, "device ordinal out of range");
    for (int j = 0; j < k; ++j) {
      if (devs[j] == devs[k]) return fail(FM_ERR_INVALID_ARGUMENT, "devices must be distinct");
    }
  }
  DeviceRestore restore;
  fm_multi* m = new fm_multi;
  m->devices = devs;
  m->n_polys = n_polys;
  m->replicas.assign(n_devices, nullptr);
  std::vector<fm_status> st(n_devices, FM_OK);
  std::vector<std::string> err(n_devices);
  std::vector<std::thread> th;
  for (int k = 0; k < n_devices; ++k) {
    th.emplace_back([&, k] {
      fm_build_params p = *params;
      p.device = devs[k];
      st[k] = fm_index_build(vertex_lonlat, ring_offsets, n_rings, poly_ring_offsets, n_polys, &p,
                             &m->replicas[k]);
      if (st[k] != FM_OK) err[k] = fm_last_error();
    });
  }
  for (auto& t : th) t.join();
  for (int k = 0; k < n_devices; ++k) {
    if (st[k] != FM_OK) {
      const fm_status s = st[k];
      const std::string msg = "replica on device " + std::to_string(devs[k]) + ": " + err[k];
      release(m);
      return fail(s, msg);
    }
  }
  *out = m;
  return FM_OK;
}

int fm_multi_size(const fm_multi* m) { return m ? static_cast<int>(m->devices.size()) : 0; }

const fm_index* fm_multi_replica(const fm_multi* m, int k) {
  return (m && k >= 0 && k < static_cast<int>(m->replicas.size())) ? m->replicas[k] : nullptr;
}

fm_status fm_multi_query_host(fm_multi* m, int mode, const double* h_lonlat, std::uint64_t n,
                              std::int32_t* h_out, std::int64_t* h_hist) {
  if (!m) return fail(FM_ERR_INVALID_ARGUMENT, "multi index is null");
  if (n == 0) return FM_OK;
  DeviceRestore restore;
  if (!h_lonlat || !h_out) return fail(FM_ERR_INVALID_ARGUMENT, "null point or output buffer");
  const int nd = static_cast<int>(m->devices.size());
  if (h_hist) {
    const fm_status s = setup_reduce(m);
    if (s != FM_OK) return s;
    for (int k = 0; k < nd; ++k) {
      cudaSetDevice(m->devices[k]);
      if (cudaMemsetAsync(m->d_hist[k], 0, std::max<std::uint64_t>(1, m->n_polys) * 8, m->streams[k]) != cudaSuccess ||
          cudaStreamSynchronize(m->streams[k]) != cudaSuccess) {
        return fail(FM_ERR_CUDA, "histogram reset failed");
      }
    }
  }
  // shard_range: contiguous and balanced, the first n % nd shards one larger
  const std::uint64_t base = n / nd, extra = n % nd;
  std::vector<fm_status> st(nd, FM_OK);
  std::vector<std::string> err(nd);
  std::vector<std::thread> th;
  for (int k = 0; k < nd; ++k) {
    const std::uint64_t start = k * base + std::min<std::uint64_t>(k, extra);
    const std::uint64_t cnt = base + (static_cast<std::uint64_t>(k) < extra ? 1 : 0);
    th.emplace_back([&, k, start, cnt] {
      st[k] = query_host_impl(m->replicas[k], mode, h_lonlat + 2 * start, cnt, h_out + start, nullptr,
                              h_hist ? m->d_hist[k] : nullptr, nullptr);
      if (st[k] != FM_OK) err[k] = fm_last_error();
    });
  }
  for (auto& t : th) t.join();
  for (int k = 0; k < nd; ++k) {
    if (st[k] != FM_OK) return fail(st[k], "shard on device " + std::to_string(m->devices[k]) + ": " + err[k]);
  }
  if (!h_hist) return FM_OK;
  // the one collective: sum the per-device histograms in place over NVLink
  ncclResult_t r = m->nccl.group_start();
  for (int k = 0; k < nd && r == ncclSuccess; ++k) {
    cudaSetDevice(m->devices[k]);
    r = m->nccl.all_reduce(m->d_hist[k], m->d_hist[k], std::max<std::uint64_t>(1, m->n_polys), ncclInt64,
                           ncclSum, m->comms[k], m->streams[k]);
  }
  const ncclResult_t r2 = m->nccl.group_end();
  if (r != ncclSuccess || r2 != ncclSuccess) {
    return fail(FM_ERR_RUNTIME, std::string("ncclAllReduce: ") + m->nccl.error_string(r != ncclSuccess ? r : r2));
  }
  for (int k = 0; k < nd; ++k) {
    cudaSetDevice(m->devices[k]);
    if (cudaStreamSynchronize(m->streams[k]) != cudaSuccess) return fail(FM_ERR_CUDA, "histogram reduce failed");
  }
  std::vector<std::int64_t> tmp(m->n_polys);
  cudaSetDevice(m->devices[0]);
  if (m->n_polys && cudaMemcpy(tmp.data(), m->d_hist[0], m->n_polys * 8, cudaMemcpyDeviceToHost) != cudaSuccess) {
    return fail(FM_ERR_CUDA, "histogram copy failed");
  }
  for (std::uint64_t k = 0; k < m->n_polys; ++k) h_hist[k] += tmp[k];
  return FM_OK;
}

void fm_multi_destroy(fm_multi* m) {
  DeviceRestore restore;
  if (m) release(m);
}

}  // extern "C"
