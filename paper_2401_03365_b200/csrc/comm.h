// comm.h — the collectives a sharded plan needs (lop.cpp:102-119 exchange step).
//
// Two backends:
//  * NCCL (one process per GPU; nccl_dl.h) — the production path;
//  * loopback — R plans of one process sharing a device, driven by R host
//    threads.  A collective is a host rendezvous plus stream events and
//    device-to-device copies, so no kernel ever waits on another rank's kernel.
//    It exists to validate the sharded plan path (ownership, owned query lists,
//    partial updates, exchange, counter reduction) on a single B200; it is not
//    a performance mode.
#pragma once

#include <cuda_runtime.h>

#include <condition_variable>
#include <cstddef>
#include <cstdint>
#include <mutex>
#include <vector>

namespace pcsb {

enum class CDType { F32, F64, U64, U8 };
enum class COp { Sum, Max };

size_t cdtype_size(CDType t);

class Collectives {
public:
    virtual ~Collectives() = default;
    virtual void group_start() {}
    virtual void group_end() {}
    // In place: rank r's `count` elements sit at buf + r * count.
    virtual void allgather(void* buf, size_t count, CDType t, cudaStream_t s) = 0;
    virtual void allreduce(void* buf, size_t count, CDType t, COp op, cudaStream_t s) = 0;
};

// NCCL clique member (comm.cu); `id` is a 128-byte ncclUniqueId.
Collectives* make_nccl_collectives(const uint8_t id[128], int nranks, int rank);

// Shared state of R in-process ranks.
class LoopbackGroup {
public:
    explicit LoopbackGroup(int nranks);
    ~LoopbackGroup();
    int nranks() const { return n_; }

    // Host rendezvous of all ranks (generation counter; reusable).
    void barrier();

    struct Slot {
        void* buf = nullptr;
        cudaEvent_t ready = nullptr;  // rank's data (or its scratch copy) complete
        cudaEvent_t done = nullptr;   // rank's writes into others / reads of others complete
    };
    std::vector<Slot> slots;  // published by each rank before a rendezvous

private:
    int n_;
    std::mutex mu_;
    std::condition_variable cv_;
    int arrived_ = 0;
    uint64_t generation_ = 0;
};

Collectives* make_loopback_collectives(LoopbackGroup* g, int rank);

// No-op collectives: one rank of an N-rank layout computing alone (developer
// knob PCSB_EMULATE_RANK="N:r" — the per-rank compute of an N-GPU run without
// its exchange; the other ranks' points simply stay where they are).
Collectives* make_null_collectives();

}  // namespace pcsb
