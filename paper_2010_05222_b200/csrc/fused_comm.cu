// Collectives fused into the step's kernels over NVLink peer memory (comm_mode
// PFC_COMM_NCCL_FUSED): the NCCL 2.28 device API provides the symmetric exchange region (ncclMemAlloc +
// ncclCommWindowRegister(NCCL_WIN_COLL_SYMMETRIC)), the peers' load/store-accessible (LSA) addresses of it, and a
// device-side LSA barrier. The data movement itself is done by the step's own kernels (pfc_internal.cuh, Peers):
//   K1 normalize_x      stores x_hat rows and labels into every peer's x32 / y      (Alg.1 L2 all-gather)
//   K7 row_combine      stores the row maxima into every peer's xmax slot `rank`     (Alg.1 L6-7)
//   prep_sum            reads the maxima of all ranks (rank order), stores the rescaled sums into the peers' xred
//   finalize            sums the xred slots in rank order                          (the SUM all-reduce)
//   dX split-K reduce   stores each owner's rows into its xdx slot `rank`          (Alg.1 L12-13)
//   xnorm_backward      sums its xdx slots in rank order                           (the reduce-scatter)
// with one LSA barrier kernel after each producer (4 per step). All reductions run in a fixed rank order, so the
// results are deterministic and equal the loopback group's (PFC_COMM_LOOPBACK_FUSED, the same kernels writing into
// the other contexts' regions on one GPU) bit for bit.
//
// Reuse of a region across steps is safe without a fifth barrier: a rank pushes step t+1's x_hat only after passing
// step t's last barrier (after the dX push), which every peer reaches only once it has finished all of its step-t
// reads of x32 / y / xmax / xred; the xdx slots are next written after step t+1's third barrier, which a peer
// reaches only after its step-t x-norm backward (joined into its step stream).
#include <cuda/atomic>
#include <nccl.h>
#include <nccl_device.h>

#include "pfc_internal.cuh"

namespace pfc {

struct FusedNccl {
  void* region = nullptr;
  size_t bytes = 0;
  ncclWindow_t win = nullptr;
  ncclDevComm dev{};
  bool dev_ok = false;
};

namespace {

__global__ void k_peer_bases(ncclWindow_t w, int n, char** out) {
  const int q = threadIdx.x;
  if (q < n) out[q] = static_cast<char*>(ncclGetLsaPointer(w, 0, q));
}

// every rank arrives (release: the stores of the preceding kernels of this stream), then waits for all peers
// (acquire); one CTA
__global__ void k_lsa_barrier(ncclDevComm comm) {
  ncclLsaBarrierSession<ncclCoopCta> bar(ncclCoopCta(), comm, ncclTeamTagLsa(), 0);
  bar.sync(ncclCoopCta(), cuda::memory_order_acq_rel);
}

}  // namespace

pfc_status fused_nccl_create(ncclComm_t comm, const Sizes& sz, FusedNccl** out, char** local_region, Peers* P,
                             std::string* err) {
  *out = nullptr;
  if (sz.world > kMaxLoopback) {
    *err = "fused collectives support at most 16 ranks";
    return PFC_ERR_CONFIG;
  }
  FusedNccl* f = new FusedNccl();
  const SymLayout L = sym_layout(sz);
  f->bytes = (size_t)((L.bytes + 4095) / 4096 * 4096);
  auto fail = [&](pfc_status st, const std::string& m) {
    *err = m;
    fused_nccl_destroy(comm, f);
    return st;
  };
  ncclResult_t r = ncclMemAlloc(&f->region, f->bytes);
  if (r != ncclSuccess) return fail(PFC_ERR_NCCL, std::string("ncclMemAlloc: ") + ncclGetErrorString(r));
  if (cudaMemset(f->region, 0, f->bytes) != cudaSuccess) return fail(PFC_ERR_CUDA, "cudaMemset of the exchange region");
  r = ncclCommWindowRegister(comm, f->region, f->bytes, &f->win, NCCL_WIN_COLL_SYMMETRIC);
  if (r != ncclSuccess) return fail(PFC_ERR_NCCL, std::string("ncclCommWindowRegister: ") + ncclGetErrorString(r));
  ncclDevCommRequirements reqs{};
  reqs.lsaBarrierCount = 1;
  r = ncclDevCommCreate(comm, &reqs, &f->dev);
  if (r != ncclSuccess) return fail(PFC_ERR_NCCL, std::string("ncclDevCommCreate: ") + ncclGetErrorString(r));
  f->dev_ok = true;
  if (f->dev.lsaSize != sz.world || f->dev.lsaRank != sz.rank)
    return fail(PFC_ERR_CONFIG, "fused collectives need every rank in one load/store (NVLink) domain");
  char** d_bases = nullptr;
  if (cudaMalloc(&d_bases, kMaxLoopback * sizeof(char*)) != cudaSuccess) return fail(PFC_ERR_OOM, "cudaMalloc");
  k_peer_bases<<<1, 32>>>(f->win, sz.world, d_bases);
  Peers p{};
  cudaError_t e = cudaMemcpy(p.base, d_bases, sz.world * sizeof(char*), cudaMemcpyDeviceToHost);
  cudaFree(d_bases);
  if (e != cudaSuccess) return fail(PFC_ERR_CUDA, std::string("peer addresses: ") + cudaGetErrorString(e));
  p.n = sz.world;
  p.rank = sz.rank;
  p.lay = L;
  // p.base[rank] is the window's LSA alias of this rank's own region (a second mapping of the same memory): the fused
  // kernels address every rank, this one included, through the LSA aliases; the other kernels use the allocation's
  // own address (c->X32, c->Y) — never both inside one kernel
  *P = p;
  *local_region = static_cast<char*>(f->region);
  *out = f;
  return PFC_OK;
}

void fused_nccl_destroy(ncclComm_t comm, FusedNccl* f) {
  if (!f) return;
  cudaDeviceSynchronize();
  if (f->dev_ok) ncclDevCommDestroy(comm, &f->dev);
  if (f->win) ncclCommWindowDeregister(comm, f->win);
  if (f->region) ncclMemFree(f->region);
  delete f;
}

int launch_lsa_barrier(const FusedNccl* f, cudaStream_t s) {
  k_lsa_barrier<<<1, 32, 0, s>>>(f->dev);
  return 1;
}

}  // namespace pfc
