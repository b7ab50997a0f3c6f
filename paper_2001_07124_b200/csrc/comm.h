// comm.h -- communicators for slab data parallelism (call sites C1-C5).
//
//   NcclComm     : NCCL 2.x loaded at run time (dlopen of the libnccl.so.2 that torch ships),
//                  one rank per GPU, bootstrapped from an ncclUniqueId that the caller
//                  broadcasts (torch.distributed).  Collectives are enqueued on the
//                  handle's stream.
//   LoopbackComm : several ranks on ONE GPU, each driven from its own host thread and
//                  stream; collectives are ordered with CUDA events only (no kernel ever
//                  waits on another), so the multi-rank control flow of the library can be
//                  exercised on a single device.
#pragma once

#include <cuda_runtime.h>

#include <cstddef>
#include <cstdint>
#include <memory>

namespace rt {

class Comm {
 public:
  virtual ~Comm() = default;
  virtual int nranks() const = 0;
  virtual int rank() const = 0;
  // in-place sum over ranks (fp64 or fp32 buffer of n elements)
  virtual void allreduce_sum(double* buf, size_t n, cudaStream_t s) = 0;
  virtual void allreduce_sum(float* buf, size_t n, cudaStream_t s) = 0;
  // recv[r*n .. r*n+n) = send of rank r
  virtual void allgather(const double* send, double* recv, size_t n, cudaStream_t s) = 0;
  // a second communicator over the same ranks whose collectives may run concurrently with this
  // one's on another stream (NCCL: ncclCommSplit; loopback: the group's side group); nullptr if none
  virtual Comm* side() { return nullptr; }
  // a third one (the side stream's R31' unmixing steps of a slab-parallel call, which run while the C3
  // allreduce occupies side()); nullptr if none
  virtual Comm* side2() { return nullptr; }
};

int nccl_get_unique_id(uint8_t id[128]);   // 0 ok, else error (message via nccl_last_error)
const char* nccl_last_error();
std::unique_ptr<Comm> make_nccl_comm(const uint8_t id[128], int nranks, int rank);

struct LoopbackGroup;
LoopbackGroup* loopback_group_create(int nranks);
void loopback_group_destroy(LoopbackGroup* g);
std::unique_ptr<Comm> make_loopback_comm(LoopbackGroup* g, int rank);

}  // namespace rt
