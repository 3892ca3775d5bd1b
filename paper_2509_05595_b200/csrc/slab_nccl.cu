// slab_nccl.cu — the C4 z-slab path for a C++ host (SURVEY §8(b),(e)ii): one rank per GPU,
// NCCL over NVLink for the only exchange steps.  Per rank:
//   1. SDF of the rank's lattice planes [z0, z1) (udf_run restricted to the slab), written
//      straight into a resident buffer that also has room for the HALO planes of each neighbour
//   2. HALO=2-plane exchange with the z-neighbours: grouped ncclSend / ncclRecv on the context
//      stream, received directly into the resident buffer (no staging copy)
//   3. slab-local DMC of the own cell layers (dmc_extract_slab; identical code to the 1-GPU path)
//   4. ncclAllGather of the (patch vertices, split vertices, faces) counts -> exclusive offsets,
//      rebase of this slab's face indices, and a grouped send of the three arrays straight into
//      place on rank 0.  The assembled mesh is bit-identical to the whole-grid extract (P11 order)
// Mirrors paper_2509_05595_b200/distributed.py (exchange_halo2 / distributed_dmc), which the
// Python host drives over torch.distributed.  NCCL is not linked: its entry points are resolved
// at run time from the NCCL the process already loaded (torch's, or libnccl.so.2).
#include <dlfcn.h>
#include <nccl.h>

#include <algorithm>
#include <mutex>
#include <vector>

#include "common.cuh"
#include "kernels.cuh"

namespace pcu {
namespace {

struct NcclApi {
  ncclResult_t (*send)(const void*, size_t, ncclDataType_t, int, ncclComm_t, cudaStream_t) = nullptr;
  ncclResult_t (*recv)(void*, size_t, ncclDataType_t, int, ncclComm_t, cudaStream_t) = nullptr;
  ncclResult_t (*allgather)(const void*, void*, size_t, ncclDataType_t, ncclComm_t, cudaStream_t) = nullptr;
  ncclResult_t (*group_start)() = nullptr;
  ncclResult_t (*group_end)() = nullptr;
  ncclResult_t (*init_all)(ncclComm_t*, int, const int*) = nullptr;
  ncclResult_t (*destroy)(ncclComm_t) = nullptr;
  const char* (*error_string)(ncclResult_t) = nullptr;
  bool ok = false;
};

const NcclApi& nccl() {
  static NcclApi api;
  static std::once_flag once;
  std::call_once(once, [] {
    void* h = dlopen("libnccl.so.2", RTLD_NOW | RTLD_NOLOAD);  // the copy the process loaded
    if (!h) h = dlopen("libnccl.so.2", RTLD_NOW | RTLD_GLOBAL);
    if (!h) h = dlopen("libnccl.so", RTLD_NOW | RTLD_GLOBAL);
    if (!h) return;
    api.send = reinterpret_cast<decltype(api.send)>(dlsym(h, "ncclSend"));
    api.recv = reinterpret_cast<decltype(api.recv)>(dlsym(h, "ncclRecv"));
    api.allgather = reinterpret_cast<decltype(api.allgather)>(dlsym(h, "ncclAllGather"));
    api.group_start = reinterpret_cast<decltype(api.group_start)>(dlsym(h, "ncclGroupStart"));
    api.group_end = reinterpret_cast<decltype(api.group_end)>(dlsym(h, "ncclGroupEnd"));
    api.init_all = reinterpret_cast<decltype(api.init_all)>(dlsym(h, "ncclCommInitAll"));
    api.destroy = reinterpret_cast<decltype(api.destroy)>(dlsym(h, "ncclCommDestroy"));
    api.error_string = reinterpret_cast<decltype(api.error_string)>(dlsym(h, "ncclGetErrorString"));
    api.ok = api.send && api.recv && api.allgather && api.group_start && api.group_end;
  });
  PCU_REQUIRE(api.ok, PAMOPT_CU_ECUDA, "NCCL (libnccl.so.2) is not available in this process");
  return api;
}

void nccl_check(ncclResult_t r, const char* what) {
  if (r == ncclSuccess) return;
  const char* s = nccl().error_string ? nccl().error_string(r) : "?";
  throw Error(PAMOPT_CU_ECUDA, std::string("NCCL ") + what + ": " + s);
}

constexpr int kHalo = 2;

void slab_range(int R, int world, int rank, int& z0, int& z1) {  // distributed.slab_ranges
  const int n = R + 1, base = n / world, extra = n % world;
  z0 = 0;
  for (int r = 0; r < rank; ++r) z0 += base + (r < extra ? 1 : 0);
  z1 = z0 + base + (rank < extra ? 1 : 0);
}

}  // namespace

void* nccl_comm_init_all(int ndev, const int* devs, void** comms) {
  nccl_check(nccl().init_all(reinterpret_cast<ncclComm_t*>(comms), ndev, devs), "ncclCommInitAll");
  return comms[0];
}

void nccl_comm_destroy(void* comm) {
  if (comm) nccl_check(nccl().destroy(static_cast<ncclComm_t>(comm)), "ncclCommDestroy");
}

void slab_extract_nccl(Ctx& ctx, const double* dV, int64_t nv, const int32_t* dF, int64_t nf, int R, double eps,
                       double beta, int rank, int world, void* comm_, DevBuf<double>& Vout, DevBuf<int32_t>& Fout,
                       int64_t& nv_out, int64_t& nf_out, int64_t counts[3]) {
  PCU_REQUIRE(world >= 1 && rank >= 0 && rank < world, PAMOPT_CU_EINVAL, "slab: bad rank / world");
  PCU_REQUIRE(world == 1 || (R + 1) / world >= kHalo, PAMOPT_CU_EINVAL, "slab: every rank needs >= 2 planes");
  const NcclApi& N = nccl();
  ncclComm_t comm = static_cast<ncclComm_t>(comm_);
  PCU_REQUIRE(comm != nullptr || world == 1, PAMOPT_CU_EINVAL, "slab: null NCCL communicator");
  cudaStream_t st = ctx.stream;
  int z0, z1;
  slab_range(R, world, rank, z0, z1);
  const int pz0 = std::max(z0 - kHalo, 0), pz1 = std::min(z1 + kHalo, R + 1);
  const int64_t plane = static_cast<int64_t>(R + 1) * (R + 1);
  DevBuf<float> res(plane * (pz1 - pz0), st);
  // 1. own planes, written in place inside the resident buffer
  udf_run(ctx, dV, nv, dF, nf, R, 1, eps, res.get() + plane * (z0 - pz0), z0, z1);
  // 2. HALO planes from / to the neighbours
  if (world > 1) {
    nccl_check(N.group_start(), "ncclGroupStart");
    if (rank > 0) {
      nccl_check(N.send(res.get() + plane * (z0 - pz0), plane * kHalo, ncclFloat32, rank - 1, comm, st), "ncclSend");
      nccl_check(N.recv(res.get(), plane * (z0 - pz0), ncclFloat32, rank - 1, comm, st), "ncclRecv");
    }
    if (rank < world - 1) {
      nccl_check(N.send(res.get() + plane * (z1 - kHalo - pz0), plane * kHalo, ncclFloat32, rank + 1, comm, st),
                 "ncclSend");
      nccl_check(N.recv(res.get() + plane * (z1 - pz0), plane * (pz1 - z1), ncclFloat32, rank + 1, comm, st),
                 "ncclRecv");
    }
    nccl_check(N.group_end(), "ncclGroupEnd");
  }
  // 3. slab-local DMC of the own cell layers
  DmcResult d;
  dmc_extract_slab(ctx, res.get(), R, pz0, pz1, z0, std::min(z1, R), beta, d);
  res.release();
  // 4. counts -> offsets -> rebase -> gather on rank 0
  DevBuf<int64_t> mine(3, st), all(3 * static_cast<size_t>(world), st);
  const int64_t c3[3] = {static_cast<int64_t>(d.nvp_own), static_cast<int64_t>(d.n_extra), static_cast<int64_t>(d.nf)};
  PCU_CUDA(cudaMemcpyAsync(mine.get(), c3, sizeof(c3), cudaMemcpyHostToDevice, st));
  if (world > 1) nccl_check(N.allgather(mine.get(), all.get(), 3, ncclInt64, comm, st), "ncclAllGather");
  else PCU_CUDA(cudaMemcpyAsync(all.get(), mine.get(), sizeof(c3), cudaMemcpyDeviceToDevice, st));
  std::vector<int64_t> hc(3 * static_cast<size_t>(world));
  PCU_CUDA(cudaMemcpyAsync(hc.data(), all.get(), hc.size() * 8, cudaMemcpyDeviceToHost, st));
  PCU_CUDA(cudaStreamSynchronize(st));
  int64_t nvp = 0, nex = 0, nft = 0;
  std::vector<int64_t> pb(world), eb(world), fb(world);
  for (int r = 0; r < world; ++r) nvp += hc[3 * r];
  for (int r = 0; r < world; ++r) {
    pb[r] = r ? pb[r - 1] + hc[3 * (r - 1)] : 0;
    eb[r] = r ? eb[r - 1] + hc[3 * (r - 1) + 1] : nvp;
    fb[r] = r ? fb[r - 1] + hc[3 * (r - 1) + 2] : 0;
  }
  nex = eb[world - 1] + hc[3 * (world - 1) + 1] - nvp;
  nft = fb[world - 1] + hc[3 * (world - 1) + 2];
  counts[0] = c3[0];
  counts[1] = c3[1];
  counts[2] = c3[2];
  mesh_rebase(ctx, d.F.get(), 3 * static_cast<int64_t>(d.nf), pb[rank], c3[0], eb[rank]);
  if (rank != 0) {
    nccl_check(N.group_start(), "ncclGroupStart");
    if (c3[0]) nccl_check(N.send(d.V.get(), 3 * c3[0], ncclFloat64, 0, comm, st), "ncclSend");
    if (c3[1]) nccl_check(N.send(d.V.get() + 3 * c3[0], 3 * c3[1], ncclFloat64, 0, comm, st), "ncclSend");
    if (c3[2]) nccl_check(N.send(d.F.get(), 3 * c3[2], ncclInt32, 0, comm, st), "ncclSend");
    nccl_check(N.group_end(), "ncclGroupEnd");
    PCU_CUDA(cudaStreamSynchronize(st));
    nv_out = nf_out = 0;
    return;
  }
  nv_out = nvp + nex;
  nf_out = nft;
  Vout.alloc(3 * (nv_out ? nv_out : 1), st);
  Fout.alloc(3 * (nf_out ? nf_out : 1), st);
  if (c3[0]) PCU_CUDA(cudaMemcpyAsync(Vout.get(), d.V.get(), 3 * c3[0] * 8, cudaMemcpyDeviceToDevice, st));
  if (c3[1])
    PCU_CUDA(cudaMemcpyAsync(Vout.get() + 3 * eb[0], d.V.get() + 3 * c3[0], 3 * c3[1] * 8, cudaMemcpyDeviceToDevice, st));
  if (c3[2]) PCU_CUDA(cudaMemcpyAsync(Fout.get(), d.F.get(), 3 * c3[2] * 4, cudaMemcpyDeviceToDevice, st));
  if (world > 1) {
    nccl_check(N.group_start(), "ncclGroupStart");
    for (int r = 1; r < world; ++r) {
      if (hc[3 * r]) nccl_check(N.recv(Vout.get() + 3 * pb[r], 3 * hc[3 * r], ncclFloat64, r, comm, st), "ncclRecv");
      if (hc[3 * r + 1])
        nccl_check(N.recv(Vout.get() + 3 * eb[r], 3 * hc[3 * r + 1], ncclFloat64, r, comm, st), "ncclRecv");
      if (hc[3 * r + 2])
        nccl_check(N.recv(Fout.get() + 3 * fb[r], 3 * hc[3 * r + 2], ncclInt32, r, comm, st), "ncclRecv");
    }
    nccl_check(N.group_end(), "ncclGroupEnd");
  }
  PCU_CUDA(cudaStreamSynchronize(st));
}

}  // namespace pcu
