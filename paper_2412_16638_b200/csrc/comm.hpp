// Inter-rank communication for the slab-decomposed grid.
//
// The k-slab partition (rank r owns planes [r n/P, (r+1) n/P) of the
// x-fastest n^3 vector, a contiguous slice) needs three exchanges:
//   * halo      one n^2 plane to each k-neighbour before every stencil
//               (ring for the periodic advection grid);
//   * alltoall  the FastDiag transpose k-slab <-> j-slab around the
//               contraction along k (T_L, precond.hpp:95-110);
//   * scalars   the Krylov dots/norms (krylov.hpp:43-71) and the stepper's
//               error flags, reduced on the host in RANK ORDER so every rank
//               takes bitwise the same control-flow decision.
//
// Two backends share this interface:
//   NcclComm   one process per GPU (torchrun), NCCL over NVLink/NVSwitch;
//              libnccl is dlopen'ed (the torch-bundled copy when loaded).
//   LocalComm  `size` ranks as threads of one process on one device, the
//              exchanges are stream-ordered device copies between the ranks'
//              buffers, joined by events + host barriers.  It runs every
//              multi-rank code path on a single B200.
#pragma once

#include <memory>
#include <vector>

#include "runtime.hpp"

namespace mprkb {

class Comm {
 public:
  Comm(int rank, int size) : rank_(rank), size_(size) {}
  virtual ~Comm() = default;
  int rank() const { return rank_; }
  int size() const { return size_; }

  // ---- host-blocking collectives on small host arrays ----------------------
  // v[c] <- sum over ranks, added in rank order (0, 1, ..., P-1): identical
  // on every rank and independent of the transport.
  virtual void allreduce_sum(double* v, int count) = 0;
  virtual void allreduce_max(double* v, int count) = 0;
  virtual void bcast_host(double* v, int count, int root) = 0;
  virtual void barrier() = 0;

  // ---- stream-ordered device exchanges (enqueued on `st`) -------------------
  // Plane `lo_src` (my first plane) goes to the lower neighbour's hi ghost,
  // `hi_src` (my last plane) to the upper neighbour's lo ghost.  Neighbours
  // are rank -+ 1, wrapping when `periodic`; a missing neighbour leaves the
  // ghost untouched (the kernels read a Dirichlet zero instead).
  virtual void halo(const void* lo_src, const void* hi_src, void* lo_ghost, void* hi_ghost, size_t bytes,
                    bool periodic, cudaStream_t st) = 0;
  // recv[s*bytes ...] <- rank s's send[rank*bytes ...] for every s (self included)
  virtual void alltoall(const void* send, void* recv, size_t bytes_per_peer, cudaStream_t st) = 0;
  // recv[r*count + c] <- rank r's send[c] (device doubles, stream-ordered on
  // st): the Krylov scalars' per-rank partial sums gathered without a host
  // round trip, so a kernel can complete them in rank order on the device
  virtual void allgather_dev(const double* send, double* recv, int count, cudaStream_t st) = 0;

  int lower(bool periodic) const {
    return rank_ > 0 ? rank_ - 1 : (periodic ? size_ - 1 : -1);
  }
  int upper(bool periodic) const {
    return rank_ < size_ - 1 ? rank_ + 1 : (periodic ? 0 : -1);
  }

 private:
  int rank_, size_;
};

// ---- in-process group (one device, one thread per rank) ------------------------
class LocalGroup;
std::shared_ptr<LocalGroup> make_local_group(int size);
std::unique_ptr<Comm> make_local_comm(const std::shared_ptr<LocalGroup>& g, int rank);

// ---- NCCL (one process per GPU) ---------------------------------------------------
constexpr int kNcclIdBytes = 128;
void nccl_unique_id(unsigned char* id);  // ncclGetUniqueId
std::unique_ptr<Comm> make_nccl_comm(int rank, int size, const unsigned char* id);

// The slab owned by one rank (k-slab for the state, j-slab inside FastDiag).
struct Slab {
  Comm* comm = nullptr;  // null or size 1: the undivided grid
  int n = 0;
  int P = 1, rank = 0;
  int nz = 0, k0 = 0;    // local k-planes [k0, k0 + nz)
  int ny = 0, j0 = 0;    // j-range of the transposed (j-slab) layout
  // split = stepped through a communicator, even a 1-rank one (which then
  // exercises every exchange path against itself)
  bool split() const { return comm != nullptr; }
  size_t local() const { return (size_t)n * n * nz; }
};
// Throws unless n divides evenly into P slabs.
Slab make_slab(int n, Comm* comm);

// Slab + the ghost-plane scratch its stencils share (2 planes of the widest
// scalar).  All users run on one stream, so one pair of planes suffices.
// The exchange runs on its own stream `cs` so the interior planes of a
// stencil (which need no ghost) overlap it; `ready` / `arrived` order it
// against the compute stream.
struct Halo {
  Slab slab;
  DevBuf ghost;
  cudaStream_t cs = nullptr;
  cudaEvent_t ready = nullptr, arrived = nullptr;
  explicit Halo(const Slab& s);
  ~Halo();
  Halo(const Halo&) = delete;
  Halo& operator=(const Halo&) = delete;
};

}  // namespace mprkb
