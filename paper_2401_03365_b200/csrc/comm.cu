// comm.cu — NCCL and loopback backends of the plan's collectives (comm.h).
#include "comm.h"

#include <cstring>
#include <memory>
#include <string>

#include "nccl_dl.h"
#include "plan.cuh"

namespace pcsb {

size_t cdtype_size(CDType t) {
    switch (t) {
        case CDType::F32: return 4;
        case CDType::F64: return 8;
        case CDType::U64: return 8;
        case CDType::U8: return 1;
    }
    return 1;
}

namespace {

// ---- NCCL ---------------------------------------------------------------------
const NcclApi& nccl_or_throw() {
    std::string err;
    const NcclApi* api = nccl_api(&err);
    if (!api) throw Failure(PCS_ERR_NCCL, err);
    return *api;
}

void nccl_ok(ncclResult_t r, const char* what) {
    if (r != ncclSuccess)
        throw Failure(PCS_ERR_NCCL, std::string(what) + ": " + nccl_or_throw().GetErrorString(r));
}

ncclDataType_t nccl_type(CDType t) {
    switch (t) {
        case CDType::F32: return ncclFloat;
        case CDType::F64: return ncclDouble;
        case CDType::U64: return ncclUint64;
        case CDType::U8: return ncclUint8;
    }
    return ncclUint8;
}

class NcclCollectives : public Collectives {
public:
    NcclCollectives(const uint8_t id[128], int nranks, int rank) : rank_(rank) {
        ncclUniqueId uid;
        static_assert(sizeof(uid) == 128, "ncclUniqueId is 128 bytes");
        std::memcpy(&uid, id, 128);
        nccl_ok(nccl_or_throw().CommInitRank(&comm_, nranks, uid, rank), "ncclCommInitRank");
    }
    ~NcclCollectives() override {
        std::string err;
        if (const NcclApi* api = nccl_api(&err)) api->CommDestroy(comm_);
    }
    void group_start() override { nccl_ok(nccl_or_throw().GroupStart(), "ncclGroupStart"); }
    void group_end() override { nccl_ok(nccl_or_throw().GroupEnd(), "ncclGroupEnd"); }
    void allgather(void* buf, size_t count, CDType t, cudaStream_t s) override {
        char* b = static_cast<char*>(buf);
        nccl_ok(nccl_or_throw().AllGather(b + (size_t)rank_ * count * cdtype_size(t), b, count,
                                          nccl_type(t), comm_, s),
                "ncclAllGather");
    }
    void allreduce(void* buf, size_t count, CDType t, COp op, cudaStream_t s) override {
        nccl_ok(nccl_or_throw().AllReduce(buf, buf, count, nccl_type(t),
                                          op == COp::Sum ? ncclSum : ncclMax, comm_, s),
                "ncclAllReduce");
    }

private:
    ncclComm_t comm_ = nullptr;
    int rank_;
};

// ---- loopback ---------------------------------------------------------------------
constexpr int kMaxLoopRanks = 8;

struct Sources {
    const void* p[kMaxLoopRanks];
};

template <typename T>
__global__ void reduce_sources_kernel(T* __restrict__ dst, Sources src, int n, size_t count, int op) {
    for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < count;
         i += (size_t)gridDim.x * blockDim.x) {
        T v = static_cast<const T*>(src.p[0])[i];
        for (int r = 1; r < n; ++r) {
            const T w = static_cast<const T*>(src.p[r])[i];
            v = op == 0 ? (T)(v + w) : (w > v ? w : v);
        }
        dst[i] = v;
    }
}

class LoopbackCollectives : public Collectives {
public:
    LoopbackCollectives(LoopbackGroup* g, int rank) : g_(g), r_(rank) {
        PCSB_CUDA(cudaEventCreateWithFlags(&g_->slots[r_].ready, cudaEventDisableTiming));
        PCSB_CUDA(cudaEventCreateWithFlags(&g_->slots[r_].done, cudaEventDisableTiming));
    }
    ~LoopbackCollectives() override {
        cudaEventDestroy(g_->slots[r_].ready);
        cudaEventDestroy(g_->slots[r_].done);
        for (void* p : scratch_) cudaFree(p);
    }
    void allgather(void* buf, size_t count, CDType t, cudaStream_t s) override {
        const size_t bytes = count * cdtype_size(t);
        auto& me = g_->slots[r_];
        me.buf = buf;
        PCSB_CUDA(cudaEventRecord(me.ready, s));
        g_->barrier();  // every rank's chunk is final (as seen by its stream)
        for (int q = 0; q < g_->nranks(); ++q) {
            if (q == r_) continue;
            PCSB_CUDA(cudaStreamWaitEvent(s, g_->slots[q].ready, 0));
            PCSB_CUDA(cudaMemcpyAsync(static_cast<char*>(g_->slots[q].buf) + r_ * bytes,
                                      static_cast<char*>(buf) + r_ * bytes, bytes,
                                      cudaMemcpyDeviceToDevice, s));
        }
        PCSB_CUDA(cudaEventRecord(me.done, s));
        g_->barrier();  // every rank has queued its outgoing copies
        for (int q = 0; q < g_->nranks(); ++q)
            if (q != r_) PCSB_CUDA(cudaStreamWaitEvent(s, g_->slots[q].done, 0));
    }
    void allreduce(void* buf, size_t count, CDType t, COp op, cudaStream_t s) override {
        const size_t bytes = count * cdtype_size(t);
        if (bytes > cap_) {
            // never freed before destruction: other ranks' queued reads may still use it
            void* p = nullptr;
            cap_ = std::max<size_t>(bytes, 1u << 20);
            PCSB_CUDA(cudaMalloc(&p, cap_));
            scratch_.push_back(p);
        }
        void* mine = scratch_.back();
        auto& me = g_->slots[r_];
        PCSB_CUDA(cudaMemcpyAsync(mine, buf, bytes, cudaMemcpyDeviceToDevice, s));
        me.buf = mine;
        PCSB_CUDA(cudaEventRecord(me.ready, s));
        g_->barrier();
        Sources src{};
        for (int q = 0; q < g_->nranks(); ++q) {
            src.p[q] = g_->slots[q].buf;
            if (q != r_) PCSB_CUDA(cudaStreamWaitEvent(s, g_->slots[q].ready, 0));
        }
        const int n = g_->nranks(), o = op == COp::Sum ? 0 : 1;
        const int blocks = (int)std::min<size_t>((count + 255) / 256, 1024);
        if (count) {
            switch (t) {
                case CDType::U64:
                    reduce_sources_kernel<unsigned long long>
                        <<<blocks, 256, 0, s>>>((unsigned long long*)buf, src, n, count, o);
                    break;
                case CDType::U8:
                    reduce_sources_kernel<uint8_t><<<blocks, 256, 0, s>>>((uint8_t*)buf, src, n, count, o);
                    break;
                case CDType::F32:
                    reduce_sources_kernel<float><<<blocks, 256, 0, s>>>((float*)buf, src, n, count, o);
                    break;
                case CDType::F64:
                    reduce_sources_kernel<double><<<blocks, 256, 0, s>>>((double*)buf, src, n, count, o);
                    break;
            }
        }
        PCSB_CUDA(cudaEventRecord(me.done, s));
        g_->barrier();  // every rank has queued its reads of the others' scratch
        for (int q = 0; q < g_->nranks(); ++q)
            if (q != r_) PCSB_CUDA(cudaStreamWaitEvent(s, g_->slots[q].done, 0));
    }

private:
    LoopbackGroup* g_;
    int r_;
    std::vector<void*> scratch_;
    size_t cap_ = 0;
};

}  // namespace

LoopbackGroup::LoopbackGroup(int nranks) : slots(nranks), n_(nranks) {
    if (nranks < 1 || nranks > kMaxLoopRanks)
        throw Failure(PCS_ERR_INVALID_PARAM, "loopback groups hold 1..8 ranks");
}

LoopbackGroup::~LoopbackGroup() = default;

void LoopbackGroup::barrier() {
    std::unique_lock<std::mutex> lock(mu_);
    const uint64_t gen = generation_;
    if (++arrived_ == n_) {
        arrived_ = 0;
        ++generation_;
        cv_.notify_all();
        return;
    }
    cv_.wait(lock, [&] { return generation_ != gen; });
}

namespace {
class NullCollectives : public Collectives {
public:
    void allgather(void*, size_t, CDType, cudaStream_t) override {}
    void allreduce(void*, size_t, CDType, COp, cudaStream_t) override {}
};
}  // namespace

Collectives* make_null_collectives() { return new NullCollectives(); }

Collectives* make_nccl_collectives(const uint8_t id[128], int nranks, int rank) {
    return new NcclCollectives(id, nranks, rank);
}

Collectives* make_loopback_collectives(LoopbackGroup* g, int rank) {
    if (!g || rank < 0 || rank >= g->nranks())
        throw Failure(PCS_ERR_INVALID_PARAM, "invalid loopback rank");
    return new LoopbackCollectives(g, rank);
}

}  // namespace pcsb
