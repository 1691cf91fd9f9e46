// comm.cuh — the exchange layer of the multi-GPU path.
//
// One part of a distributed hierarchy per GPU.  Parts talk through Comm:
//   * CommNccl  one process per GPU, NCCL over NVLink/NVSwitch: grouped
//               ncclSend/ncclRecv for halo rings and ghost DoFs, ncclAllReduce
//               for inner products and setup reductions (libnccl is dlopen'ed,
//               so the library does not pin an NCCL build);
//   * CommLocal P parts driven by P host threads of one process on one device
//               (the same code path, testable on a single B200): mailbox of
//               device pointers + CUDA events + a host barrier; the sum of an
//               all-reduce is formed in part order, so it is deterministic.
// Every operation is stream-ordered on the calling part's stream.
#pragma once

#include <cstdint>
#include <vector>

#include "common.cuh"

namespace auxb200 {

struct Msg {
    int peer;
    void* buf;      // device
    size_t bytes;
};

struct Comm {
    int rank = 0, size = 1;
    bool peers_warm = false;   // the coarse cycle's peer connections exist (solve.cu build_graph)
    Comm();
    virtual ~Comm();
    // in-place element-wise sum over all parts (device doubles)
    virtual void allreduce_sum(double* buf, int count, cudaStream_t s) = 0;
    // in-place element-wise max over all parts (device uint64)
    virtual void allreduce_max(unsigned long long* buf, int count, cudaStream_t s) = 0;
    // a batch of point-to-point messages; a part may appear in both lists
    virtual void exchange(const std::vector<Msg>& sends, const std::vector<Msg>& recvs, cudaStream_t s) = 0;
    virtual void barrier(cudaStream_t s) = 0;
    // every operation is stream-ordered device work with no host round trip,
    // so a sequence of them can be captured into a CUDA graph
    virtual bool graph_capturable() const = 0;
};

// P parts in one process (opaque group shared by the P threads).
struct LocalGroup;
LocalGroup* local_group_create(int parts);
void local_group_destroy(LocalGroup* g);
Comm* make_local_comm(LocalGroup* g, int rank);

// Handle checks of the C ABI's void* transport argument (aux_dist_opts):
// registries of live groups / communicators, no dereference of the pointer.
bool is_local_group(const void* p);
bool is_comm(const void* p);

// NCCL (one process per GPU).
bool nccl_unique_id(unsigned char id[128]);
Comm* make_nccl_comm(const unsigned char id[128], int nranks, int rank);

}  // namespace auxb200
