// Shard collectives of the multi-GPU plan.  The path has exactly two exchange
// steps: the upward exchange after the sharded P2M / M2M --
// an in-place all-gather of the coarse exchange level plus point-to-point
// halo sends / receives of the deep levels' M2L halos -- and the all-reduce
// of the energy/counter vector.
// NCCL is resolved at run time (dlopen of libnccl.so.2 -- in a PyTorch process
// the already-loaded NCCL is reused), so the library has no link-time NCCL
// dependency and single-GPU users never touch it.
#pragma once

#include <cstddef>
#include <vector>
#include <cuda_runtime.h>

namespace ankh_b200 {

/// One peer's share of the halo exchange: this rank's packed rows for the
/// peer (`send`, send_count doubles) and the peer's rows for this rank
/// (`recv`, recv_count doubles).
struct HaloPeer {
  int peer;
  const double* send;
  std::size_t send_count;
  double* recv;
  std::size_t recv_count;
};

class Collective {
 public:
  virtual ~Collective() = default;
  /// recv holds world * count doubles; this rank's contribution already sits at
  /// recv + rank * count (in-place all-gather).
  virtual void allgather_inplace(double* recv, std::size_t count, cudaStream_t st) = 0;
  /// several in-place all-gathers (recv[k] holds world * count[k] doubles),
  /// issued as one group
  virtual void allgather_inplace_group(double* const* recv, const std::size_t* count, int n,
                                       cudaStream_t st) = 0;
  /// The upward exchange as ONE group: in-place all-gathers (as
  /// allgather_inplace_group) plus the halo sends / receives of every peer.
  virtual void upward_exchange(double* const* recv, const std::size_t* count, int n,
                               const std::vector<HaloPeer>& halo, cudaStream_t st) = 0;
  virtual void allreduce_sum(double* buf, std::size_t count, cudaStream_t st) = 0;
  /// sum over `sum[0, n_sum)` and minimum over `mins[0, n_min)`, together
  virtual void allreduce_sum_min(double* sum, std::size_t n_sum, unsigned long long* mins,
                                 std::size_t n_min, cudaStream_t st) = 0;
  virtual int rank() const = 0;
  virtual int world() const = 0;
};

/// 128-byte NCCL unique id for rank 0 to broadcast (throws AnkhError on failure).
void nccl_unique_id(unsigned char out[128]);
/// Communicator over `world` ranks (one GPU each, current device).
Collective* make_nccl_collective(const unsigned char id[128], int rank, int world);
/// One-rank exercise of every NCCL call the plans issue, eager and in a CUDA
/// graph (throws AnkhError on any failure or changed value).
void nccl_selftest();
/// Timing stand-in for a one-GPU box (diagnostics only): the all-gather fills
/// the other shards' rows with device copies of this shard's slab and each
/// halo receive buffer with a device copy of the matching send buffer (the
/// bytes land in HBM as they would over NVLink, at HBM rather than NVLink
/// speed), the all-reduce is the identity.  Reports then hold this shard's
/// partial sums.
Collective* make_loopback_collective(int rank, int world);
/// Test stand-in for G shards in ONE process on one device: at its exchange
/// point shard r copies (stream-ordered) its own slabs into the other shards'
/// expansion arrays (bases[q], same layout); the all-reduces are identities.
/// Halo rows go the same way: shard r copies its packed rows for peer q into
/// q's receive buffer for r (halo_recv[q][r]), which q unpacks at its own
/// exchange point.  Shard r's M2L reads what the others pushed, so from the
/// second evaluation of the same inputs on, every shard holds every slab and
/// halo row it reads and reports its true partial energies.
Collective* make_push_collective(int rank, int world, const std::vector<double*>& bases,
                                 const std::vector<std::vector<double*>>& halo_recv);

}  // namespace ankh_b200
