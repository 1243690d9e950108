// comm.cu -- row-partitioned multi-GPU plumbing for the CB-GMRES solve.
//
// The reference is single-process (SPEC.md:367 makes multi-GPU a non-goal);
// this is the B200 build's own layer. One process per GPU:
//   * reductions: each rank's partial vector (<= restart+2 doubles) is
//     all-gathered and summed in rank order 0..P-1 by a tiny kernel, so the
//     result is identical on every rank and independent of NCCL's algorithm;
//   * SpMV ghosts: grouped ncclSend/ncclRecv of packed boundary rows into the
//     ghost tail of the local vector (Halo).
// NCCL is loaded with dlopen at first use (the process may already hold
// torch's libnccl.so.2; the same soname is reused). LocalComm runs P ranks
// as P host threads on ONE device with in-process copies -- the partitioned
// solver's test harness, which separates partition/halo bugs from NCCL.
#include <dlfcn.h>
#include <nccl.h>

#include <algorithm>
#include <barrier>
#include <cstring>
#include <memory>
#include <mutex>
#include <thread>
#include <vector>

#include "common.cuh"
#include "solver.h"

namespace cbgx {

namespace {

__global__ void sum_ranks_kernel(const double* __restrict__ g, int P, uint64_t count,
                                 double* __restrict__ out) {
    for (uint64_t k = blockIdx.x * static_cast<uint64_t>(blockDim.x) + threadIdx.x; k < count;
         k += static_cast<uint64_t>(gridDim.x) * blockDim.x) {
        double s = g[k];
        for (int r = 1; r < P; ++r) s = __dadd_rn(s, g[static_cast<uint64_t>(r) * count + k]);
        out[k] = s;
    }
}

// sum_ranks_kernel for a packed vector, element 0 and the rest to two places
__global__ void sum_ranks_split_kernel(const double* __restrict__ g, int P, uint64_t count, double* __restrict__ first,
                                       double* __restrict__ rest) {
    for (uint64_t k = blockIdx.x * static_cast<uint64_t>(blockDim.x) + threadIdx.x; k < count;
         k += static_cast<uint64_t>(gridDim.x) * blockDim.x) {
        double s = g[k];
        for (int r = 1; r < P; ++r) s = __dadd_rn(s, g[static_cast<uint64_t>(r) * count + k]);
        if (k == 0) *first = s;
        else rest[k - 1] = s;
    }
}

__global__ void gather_rows_kernel(const double* __restrict__ v, const int32_t* __restrict__ idx,
                                   uint64_t count, double* __restrict__ out) {
    for (uint64_t k = blockIdx.x * static_cast<uint64_t>(blockDim.x) + threadIdx.x; k < count;
         k += static_cast<uint64_t>(gridDim.x) * blockDim.x)
        out[k] = v[idx[k]];
}

// --------------------------------------------------------------- NCCL
struct NcclApi {
    void* h = nullptr;
    ncclResult_t (*GetUniqueId)(ncclUniqueId*) = nullptr;
    ncclResult_t (*CommInitRank)(ncclComm_t*, int, ncclUniqueId, int) = nullptr;
    ncclResult_t (*CommDestroy)(ncclComm_t) = nullptr;
    ncclResult_t (*AllGather)(const void*, void*, size_t, ncclDataType_t, ncclComm_t, cudaStream_t) = nullptr;
    ncclResult_t (*Send)(const void*, size_t, ncclDataType_t, int, ncclComm_t, cudaStream_t) = nullptr;
    ncclResult_t (*Recv)(void*, size_t, ncclDataType_t, int, ncclComm_t, cudaStream_t) = nullptr;
    ncclResult_t (*GroupStart)() = nullptr;
    ncclResult_t (*GroupEnd)() = nullptr;
    const char* (*GetErrorString)(ncclResult_t) = nullptr;
};

NcclApi& nccl() {
    static NcclApi api;
    static std::once_flag once;
    std::call_once(once, [] {
        void* h = dlopen("libnccl.so.2", RTLD_NOW | RTLD_GLOBAL);
        if (!h) h = dlopen("libnccl.so", RTLD_NOW | RTLD_GLOBAL);
        if (!h) return;
        api.h = h;
        api.GetUniqueId = reinterpret_cast<decltype(api.GetUniqueId)>(dlsym(h, "ncclGetUniqueId"));
        api.CommInitRank = reinterpret_cast<decltype(api.CommInitRank)>(dlsym(h, "ncclCommInitRank"));
        api.CommDestroy = reinterpret_cast<decltype(api.CommDestroy)>(dlsym(h, "ncclCommDestroy"));
        api.AllGather = reinterpret_cast<decltype(api.AllGather)>(dlsym(h, "ncclAllGather"));
        api.Send = reinterpret_cast<decltype(api.Send)>(dlsym(h, "ncclSend"));
        api.Recv = reinterpret_cast<decltype(api.Recv)>(dlsym(h, "ncclRecv"));
        api.GroupStart = reinterpret_cast<decltype(api.GroupStart)>(dlsym(h, "ncclGroupStart"));
        api.GroupEnd = reinterpret_cast<decltype(api.GroupEnd)>(dlsym(h, "ncclGroupEnd"));
        api.GetErrorString = reinterpret_cast<decltype(api.GetErrorString)>(dlsym(h, "ncclGetErrorString"));
    });
    if (!api.h || !api.GetUniqueId || !api.AllGather || !api.Send)
        throw Error(CBGX_ECOMM, "nccl: libnccl.so.2 not loadable");
    return api;
}

void check_nccl(ncclResult_t r, const char* what) {
    if (r != ncclSuccess) {
        const char* s = nccl().GetErrorString ? nccl().GetErrorString(r) : "?";
        throw Error(CBGX_ECOMM, std::string("nccl: ") + s + " (" + what + ")");
    }
}

// Grow-only device scratch.
struct Scratch {
    void* p = nullptr;
    size_t cap = 0;
    void* get(size_t bytes) {
        if (bytes > cap) {
            if (p) CBGX_CUDA(cudaFree(p));
            CBGX_CUDA(cudaMalloc(&p, bytes));
            cap = bytes;
        }
        return p;
    }
    ~Scratch() {
        if (p) cudaFree(p);
    }
};

void sum_gathered(const double* g, int P, size_t count, double* out, cudaStream_t st) {
    CBGX_K(sum_ranks_kernel<<<1, 128, 0, st>>>(g, P, count, out));
    CBGX_CUDA(cudaGetLastError());
}

void sum_gathered_split(const double* g, int P, size_t count, double* first, double* rest, cudaStream_t st) {
    CBGX_K(sum_ranks_split_kernel<<<1, 128, 0, st>>>(g, P, count, first, rest));
    CBGX_CUDA(cudaGetLastError());
}

class NcclComm final : public Comm {
public:
    NcclComm(const ncclUniqueId& id, int nranks, int rank) : rank_(rank), size_(nranks) {
        check_nccl(nccl().CommInitRank(&comm_, nranks, id, rank), "ncclCommInitRank");
    }
    ~NcclComm() override {
        if (comm_) nccl().CommDestroy(comm_);
    }
    int rank() const override { return rank_; }
    int size() const override { return size_; }
    void sum_partials(double* d_vals, size_t count, cudaStream_t st) override {
        double* g = static_cast<double*>(gather_.get(count * size_ * sizeof(double)));
        check_nccl(nccl().AllGather(d_vals, g, count * sizeof(double), ncclChar, comm_, st), "ncclAllGather");
        sum_gathered(g, size_, count, d_vals, st);
    }
    void sum_partials_split(const double* d_src, size_t count, double* d_first, double* d_rest,
                            cudaStream_t st) override {
        double* g = static_cast<double*>(gather_.get(count * size_ * sizeof(double)));
        check_nccl(nccl().AllGather(d_src, g, count * sizeof(double), ncclChar, comm_, st), "ncclAllGather");
        sum_gathered_split(g, size_, count, d_first, d_rest, st);
    }
    void allgather(const void* d_send, void* d_recv, size_t bytes, cudaStream_t st) override {
        check_nccl(nccl().AllGather(d_send, d_recv, bytes, ncclChar, comm_, st), "ncclAllGather");
    }
    void exchange(const std::vector<Msg>& sends, const std::vector<Msg>& recvs, cudaStream_t st) override {
        check_nccl(nccl().GroupStart(), "ncclGroupStart");
        for (const auto& m : sends)
            check_nccl(nccl().Send(m.d_buf, m.bytes, ncclChar, m.peer, comm_, st), "ncclSend");
        for (const auto& m : recvs)
            check_nccl(nccl().Recv(m.d_buf, m.bytes, ncclChar, m.peer, comm_, st), "ncclRecv");
        check_nccl(nccl().GroupEnd(), "ncclGroupEnd");
    }
    void barrier(cudaStream_t st) override {
        uint8_t* b = static_cast<uint8_t*>(bar_.get(static_cast<size_t>(size_) + 1));
        allgather(b + size_, b, 1, st);
        CBGX_CUDA(cudaStreamSynchronize(st));
    }

private:
    int rank_, size_;
    ncclComm_t comm_ = nullptr;
    Scratch gather_, bar_;
};

// ------------------------------------------------ in-process (threads)
struct LocalShared {
    explicit LocalShared(int P) : size(P), bar(P), slots(P), msgs(P) {}
    int size;
    std::barrier<> bar;
    std::vector<const void*> slots;
    std::vector<std::vector<Comm::Msg>> msgs;  // per rank: its sends
};

class LocalComm final : public Comm {
public:
    LocalComm(std::shared_ptr<LocalShared> sh, int rank) : sh_(std::move(sh)), rank_(rank) {}
    int rank() const override { return rank_; }
    int size() const override { return sh_->size; }
    void sum_partials(double* d_vals, size_t count, cudaStream_t st) override {
        double* g = static_cast<double*>(gather_.get(count * sh_->size * sizeof(double)));
        allgather(d_vals, g, count * sizeof(double), st);
        sum_gathered(g, sh_->size, count, d_vals, st);
        CBGX_CUDA(cudaStreamSynchronize(st));
    }
    void sum_partials_split(const double* d_src, size_t count, double* d_first, double* d_rest,
                            cudaStream_t st) override {
        double* g = static_cast<double*>(gather_.get(count * sh_->size * sizeof(double)));
        allgather(d_src, g, count * sizeof(double), st);
        sum_gathered_split(g, sh_->size, count, d_first, d_rest, st);
        CBGX_CUDA(cudaStreamSynchronize(st));
    }
    void allgather(const void* d_send, void* d_recv, size_t bytes, cudaStream_t st) override {
        CBGX_CUDA(cudaStreamSynchronize(st));
        sh_->slots[rank_] = d_send;
        sh_->bar.arrive_and_wait();
        for (int r = 0; r < sh_->size; ++r)
            CBGX_CUDA(cudaMemcpy(static_cast<char*>(d_recv) + r * bytes, sh_->slots[r], bytes, cudaMemcpyDeviceToDevice));
        sh_->bar.arrive_and_wait();
    }
    void exchange(const std::vector<Msg>& sends, const std::vector<Msg>& recvs, cudaStream_t st) override {
        CBGX_CUDA(cudaStreamSynchronize(st));
        sh_->msgs[rank_] = sends;
        sh_->bar.arrive_and_wait();
        for (const auto& m : recvs) {
            const Msg* src = nullptr;
            for (const auto& s : sh_->msgs[m.peer])
                if (s.peer == rank_) src = &s;
            if (!src || src->bytes != m.bytes) throw Error(CBGX_ECOMM, "local comm: unmatched receive");
            CBGX_CUDA(cudaMemcpy(m.d_buf, src->d_buf, m.bytes, cudaMemcpyDeviceToDevice));
        }
        sh_->bar.arrive_and_wait();
    }
    void barrier(cudaStream_t st) override {
        CBGX_CUDA(cudaStreamSynchronize(st));
        sh_->bar.arrive_and_wait();
    }

private:
    std::shared_ptr<LocalShared> sh_;
    int rank_;
    Scratch gather_;
};

}  // namespace

// ------------------------------------------------------------------ Halo
Halo::~Halo() {
    if (d_send_idx) cudaFree(d_send_idx);
    if (d_send_buf) cudaFree(d_send_buf);
}

void Halo::exchange(double* d_vec, cudaStream_t st) const {
    if (!comm || comm->size() == 1) return;
    const uint64_t total = send_offsets.empty() ? 0 : send_offsets.back();
    if (total) {
        CBGX_K(gather_rows_kernel<<<static_cast<int>(std::min<uint64_t>((total + 255) / 256, 1024)), 256, 0, st>>>(
            d_vec + own_offset(), d_send_idx, total, d_send_buf));
        CBGX_CUDA(cudaGetLastError());
    }
    std::vector<Comm::Msg> sends, recvs;
    for (size_t i = 0; i < send_peers.size(); ++i)
        sends.push_back({send_peers[i], d_send_buf + send_offsets[i],
                         (send_offsets[i + 1] - send_offsets[i]) * sizeof(double)});
    for (size_t i = 0; i < recv_peers.size(); ++i) {
        // a peer's ghosts are contiguous and on one side of the own rows
        const uint64_t p = recv_offsets[i];
        const uint64_t at = window ? (p < win_lo ? p : p + n_local) : n_local + p;
        recvs.push_back({recv_peers[i], d_vec + at, (recv_offsets[i + 1] - recv_offsets[i]) * sizeof(double)});
    }
    comm->exchange(sends, recvs, st);
}

// ------------------------------------------------ pure host halo planning
// (no device calls; exposed through the C-ABI so the partition logic is
// testable on CPU with a gloo communicator, tests/test_dist_cpu.py)
struct HaloPlan {
    std::vector<int64_t> ghosts;     // sorted global indices not owned here
    std::vector<uint64_t> need;      // need[o]: ghosts owned by rank o
    std::vector<int32_t> local_cols; // remapped columns
    bool window = false;             // ghosts laid out around the own rows (see below)
    uint64_t win_lo = 0;             // window: ghosts below the own rows (= own rows' offset)
};

HaloPlan plan_halo(int P, int me, const uint64_t* ranges, uint64_t n_global, const int64_t* cols, uint64_t nnz) {
    for (int r = 0; r < P; ++r) {
        if (ranges[2 * r] > ranges[2 * r + 1] || (r > 0 && ranges[2 * r] != ranges[2 * r - 1]))
            throw Error(CBGX_EINVAL, "halo: row blocks must be contiguous and ordered by rank");
    }
    if (ranges[0] != 0 || ranges[2 * P - 1] != n_global) throw Error(CBGX_EINVAL, "halo: row blocks must cover the matrix");
    const uint64_t rb = ranges[2 * me], re = ranges[2 * me + 1];
    auto owner = [&](int64_t c) {
        int lo = 0, hi = P - 1;
        while (lo < hi) {
            const int mid = (lo + hi + 1) / 2;
            if (static_cast<uint64_t>(c) >= ranges[2 * mid]) lo = mid; else hi = mid - 1;
        }
        return lo;
    };
    HaloPlan H;
    for (uint64_t k = 0; k < nnz; ++k) {
        const int64_t c = cols[k];
        if (c < 0 || static_cast<uint64_t>(c) >= n_global) throw Error(CBGX_EINVAL, "csr: column index out of range");
        if (static_cast<uint64_t>(c) < rb || static_cast<uint64_t>(c) >= re) H.ghosts.push_back(c);
    }
    std::sort(H.ghosts.begin(), H.ghosts.end());
    H.ghosts.erase(std::unique(H.ghosts.begin(), H.ghosts.end()), H.ghosts.end());
    H.need.assign(P, 0);
    for (int64_t g : H.ghosts) ++H.need[owner(g)];
    const uint64_t n_local = re - rb;
    // Window layout when the ghosts below the own rows are exactly the rows
    // [rb - n_lo, rb) and those above exactly [re, re + n_hi) (a banded
    // matrix on a slab partition: the neighbouring planes): the local vector
    // is [lower ghosts | own rows | upper ghosts] = the global rows
    // [rb - n_lo, re + n_hi), so every column offset (col - row) of the
    // global matrix survives the remap (shifted by n_lo) and the dictionary
    // SpMV applies. Otherwise the compact layout [own rows | ghosts].
    const uint64_t n_lo = static_cast<uint64_t>(std::lower_bound(H.ghosts.begin(), H.ghosts.end(),
                                                                 static_cast<int64_t>(rb)) - H.ghosts.begin());
    const uint64_t n_hi = H.ghosts.size() - n_lo;
    H.window = (n_lo == 0 || (H.ghosts[0] == static_cast<int64_t>(rb - n_lo) &&
                              H.ghosts[n_lo - 1] == static_cast<int64_t>(rb) - 1)) &&
               (n_hi == 0 || (H.ghosts[n_lo] == static_cast<int64_t>(re) &&
                              H.ghosts.back() == static_cast<int64_t>(re + n_hi) - 1));
    H.win_lo = H.window ? n_lo : 0;
    // own -> own offset + c - rb; ghost at sorted position p -> p (below) or
    // p + n_local (above) in the window layout, n_local + p in the compact
    // one (ghosts sorted by global index == grouped by owner rank); each row
    // keeps its nonzero order, so the local SpMV accumulates in the
    // reference's order.
    H.local_cols.resize(nnz);
    for (uint64_t k = 0; k < nnz; ++k) {
        const int64_t c = cols[k];
        if (static_cast<uint64_t>(c) >= rb && static_cast<uint64_t>(c) < re) {
            H.local_cols[k] = static_cast<int32_t>(H.win_lo + (c - static_cast<int64_t>(rb)));
        } else {
            const uint64_t p = static_cast<uint64_t>(std::lower_bound(H.ghosts.begin(), H.ghosts.end(), c) -
                                                     H.ghosts.begin());
            H.local_cols[k] = static_cast<int32_t>(H.window ? (p < n_lo ? p : p + n_local) : n_local + p);
        }
    }
    return H;
}

std::vector<int32_t> send_index(uint64_t rb, uint64_t re, const int64_t* requested, uint64_t count) {
    std::vector<int32_t> idx(count);
    for (uint64_t k = 0; k < count; ++k) {
        if (requested[k] < static_cast<int64_t>(rb) || requested[k] >= static_cast<int64_t>(re))
            throw Error(CBGX_EINTERNAL, "halo: request for a row this rank does not own");
        idx[k] = static_cast<int32_t>(requested[k] - static_cast<int64_t>(rb));
    }
    return idx;
}

// Collective: builds the halo plan and remaps columns (see cbgx.h).
std::unique_ptr<Halo> make_halo(Comm* comm, uint64_t rb, uint64_t re, uint64_t n_global,
                                const int64_t* d_gcols, uint64_t nnz, int32_t* d_lcols,
                                cudaStream_t st) {
    auto H = std::make_unique<Halo>();
    H->comm = comm;
    H->n_local = re - rb;
    const int P = comm->size(), me = comm->rank();
    std::vector<int64_t> cols(nnz);
    if (nnz) CBGX_CUDA(cudaMemcpy(cols.data(), d_gcols, nnz * 8, cudaMemcpyDeviceToHost));
    // all ranks' row ranges
    std::vector<uint64_t> ranges(2 * P);
    {
        Scratch s;
        uint64_t* d = static_cast<uint64_t*>(s.get((2 * P + 2) * sizeof(uint64_t)));
        const uint64_t mine[2] = {rb, re};
        CBGX_CUDA(cudaMemcpy(d + 2 * P, mine, sizeof(mine), cudaMemcpyHostToDevice));
        comm->allgather(d + 2 * P, d, 2 * sizeof(uint64_t), st);
        CBGX_CUDA(cudaStreamSynchronize(st));
        CBGX_CUDA(cudaMemcpy(ranges.data(), d, 2 * P * sizeof(uint64_t), cudaMemcpyDeviceToHost));
    }
    HaloPlan plan = plan_halo(P, me, ranges.data(), n_global, cols.data(), nnz);
    H->n_ghost = plan.ghosts.size();
    H->window = plan.window;
    H->win_lo = plan.win_lo;
    std::vector<uint64_t> counts(static_cast<size_t>(P) * P);
    {
        Scratch s;
        uint64_t* d = static_cast<uint64_t*>(s.get((static_cast<size_t>(P) * P + P) * sizeof(uint64_t)));
        CBGX_CUDA(cudaMemcpy(d + static_cast<size_t>(P) * P, plan.need.data(), P * sizeof(uint64_t), cudaMemcpyHostToDevice));
        comm->allgather(d + static_cast<size_t>(P) * P, d, P * sizeof(uint64_t), st);
        CBGX_CUDA(cudaStreamSynchronize(st));
        CBGX_CUDA(cudaMemcpy(counts.data(), d, counts.size() * sizeof(uint64_t), cudaMemcpyDeviceToHost));
    }
    // counts[r * P + o] = #rows rank r needs from owner o
    uint64_t off = 0;
    H->recv_offsets.push_back(0);
    for (int o = 0; o < P; ++o) {
        if (o == me || !plan.need[o]) continue;
        H->recv_peers.push_back(o);
        off += plan.need[o];
        H->recv_offsets.push_back(off);
    }
    H->send_offsets.push_back(0);
    uint64_t soff = 0;
    for (int r = 0; r < P; ++r) {
        const uint64_t c = counts[static_cast<size_t>(r) * P + me];
        if (r == me || !c) continue;
        H->send_peers.push_back(r);
        soff += c;
        H->send_offsets.push_back(soff);
    }
    // exchange request lists (global indices) with the owners
    Scratch req_s, req_r;
    int64_t* d_req = static_cast<int64_t*>(req_s.get(std::max<size_t>(plan.ghosts.size(), 1) * 8));
    int64_t* d_got = static_cast<int64_t*>(req_r.get(std::max<uint64_t>(soff, 1) * 8));
    if (!plan.ghosts.empty())
        CBGX_CUDA(cudaMemcpy(d_req, plan.ghosts.data(), plan.ghosts.size() * 8, cudaMemcpyHostToDevice));
    {
        std::vector<Comm::Msg> sends, recvs;
        for (size_t i = 0; i < H->recv_peers.size(); ++i)
            sends.push_back({H->recv_peers[i], d_req + H->recv_offsets[i], (H->recv_offsets[i + 1] - H->recv_offsets[i]) * 8});
        for (size_t i = 0; i < H->send_peers.size(); ++i)
            recvs.push_back({H->send_peers[i], d_got + H->send_offsets[i], (H->send_offsets[i + 1] - H->send_offsets[i]) * 8});
        comm->exchange(sends, recvs, st);
        CBGX_CUDA(cudaStreamSynchronize(st));
    }
    std::vector<int64_t> got(soff);
    if (soff) CBGX_CUDA(cudaMemcpy(got.data(), d_got, soff * 8, cudaMemcpyDeviceToHost));
    const std::vector<int32_t> sidx = send_index(rb, re, got.data(), soff);
    CBGX_CUDA(cudaMalloc(&H->d_send_idx, std::max<uint64_t>(soff, 1) * 4));
    CBGX_CUDA(cudaMalloc(&H->d_send_buf, std::max<uint64_t>(soff, 1) * 8));
    if (soff) CBGX_CUDA(cudaMemcpy(H->d_send_idx, sidx.data(), soff * 4, cudaMemcpyHostToDevice));
    if (nnz) CBGX_CUDA(cudaMemcpy(d_lcols, plan.local_cols.data(), nnz * 4, cudaMemcpyHostToDevice));
    return H;
}

}  // namespace cbgx

using namespace cbgx;

struct cbgx_comm {
    std::unique_ptr<Comm> impl;
};
struct cbgx_halo {
    std::unique_ptr<Halo> impl;
};

extern "C" {

int cbgx_nccl_unique_id(uint8_t out[128]) {
    return guard([&] {
        static_assert(sizeof(ncclUniqueId) == 128, "ncclUniqueId is 128 bytes");
        ncclUniqueId id;
        check_nccl(nccl().GetUniqueId(&id), "ncclGetUniqueId");
        std::memcpy(out, &id, 128);
    });
}

int cbgx_comm_create_nccl(const uint8_t uid[128], int nranks, int rank, cbgx_comm** out) {
    return guard([&] {
        if (!out || nranks < 1 || rank < 0 || rank >= nranks) throw Error(CBGX_EINVAL, "comm: bad arguments");
        ncclUniqueId id;
        std::memcpy(&id, uid, 128);
        auto* c = new cbgx_comm{std::make_unique<NcclComm>(id, nranks, rank)};
        *out = c;
    });
}

int cbgx_comm_create_local_group(int nranks, cbgx_comm** out) {
    return guard([&] {
        if (!out || nranks < 1) throw Error(CBGX_EINVAL, "comm: bad arguments");
        auto shared = std::make_shared<LocalShared>(nranks);
        for (int r = 0; r < nranks; ++r) out[r] = new cbgx_comm{std::make_unique<LocalComm>(shared, r)};
    });
}

int cbgx_comm_destroy(cbgx_comm* c) {
    return guard([&] { delete c; });
}

int cbgx_comm_rank(const cbgx_comm* c, int* rank, int* nranks) {
    return guard([&] {
        if (!c) throw Error(CBGX_EINVAL, "comm: null handle");
        if (rank) *rank = c->impl->rank();
        if (nranks) *nranks = c->impl->size();
    });
}

int cbgx_halo_create(cbgx_comm* c, uint64_t row_begin, uint64_t row_end, uint64_t n_global,
                     const int64_t* d_global_cols, uint64_t nnz, int32_t* d_local_cols_out,
                     cbgx_halo** out) {
    return guard([&] {
        if (!c || !out) throw Error(CBGX_EINVAL, "halo: null argument");
        *out = new cbgx_halo{make_halo(c->impl.get(), row_begin, row_end, n_global, d_global_cols, nnz,
                                       d_local_cols_out, nullptr)};
    });
}

int cbgx_halo_plan(int nranks, int rank, const uint64_t* row_ranges, uint64_t n_global, const int64_t* gcols,
                   uint64_t nnz, int32_t* local_cols_out, int64_t* ghosts_out, uint64_t* n_ghosts,
                   uint64_t* need_per_rank, uint64_t* own_offset) {
    return guard([&] {
        if (nranks < 1 || rank < 0 || rank >= nranks) throw Error(CBGX_EINVAL, "halo: bad rank");
        const HaloPlan p = plan_halo(nranks, rank, row_ranges, n_global, gcols, nnz);
        if (local_cols_out) std::copy(p.local_cols.begin(), p.local_cols.end(), local_cols_out);
        if (ghosts_out) std::copy(p.ghosts.begin(), p.ghosts.end(), ghosts_out);
        if (n_ghosts) *n_ghosts = p.ghosts.size();
        if (need_per_rank) std::copy(p.need.begin(), p.need.end(), need_per_rank);
        if (own_offset) *own_offset = p.win_lo;
    });
}

uint64_t cbgx_halo_own_offset(const cbgx_halo* h) { return h ? h->impl->own_offset() : 0; }

int cbgx_halo_send_index(uint64_t row_begin, uint64_t row_end, const int64_t* requested, uint64_t count,
                         int32_t* send_idx_out) {
    return guard([&] {
        const auto idx = send_index(row_begin, row_end, requested, count);
        std::copy(idx.begin(), idx.end(), send_idx_out);
    });
}

int cbgx_sum_ranks_host(int nranks, uint64_t count, const double* gathered, double* out) {
    return guard([&] {
        // the rank-order combine of sum_ranks_kernel, on the host
        for (uint64_t k = 0; k < count; ++k) {
            double s = gathered[k];
            for (int r = 1; r < nranks; ++r) s += gathered[static_cast<uint64_t>(r) * count + k];
            out[k] = s;
        }
    });
}

int cbgx_halo_destroy(cbgx_halo* h) {
    return guard([&] { delete h; });
}

uint64_t cbgx_halo_ghosts(const cbgx_halo* h) { return h ? h->impl->n_ghost : 0; }

int cbgx_halo_exchange(cbgx_halo* h, double* d_vec, void* stream) {
    return guard([&] {
        if (!h) throw Error(CBGX_EINVAL, "halo: null handle");
        h->impl->exchange(d_vec, as_stream(stream));
    });
}

int cbgx_solver_create_dist(const cbgx_csr* A, cbgx_halo* halo, const cbgx_gmres_config* cfg,
                            cbgx_comm* comm, cbgx_solver** out) {
    return guard([&] {
        if (!A || !halo || !cfg || !comm || !out) throw Error(CBGX_EINVAL, "solver: null argument");
        auto* h = new SolverHandle();
        try {
            h->solver = std::make_unique<Solver>(*A, *cfg, comm->impl.get(), halo->impl.get());
        } catch (...) {
            delete h;
            throw;
        }
        *out = reinterpret_cast<cbgx_solver*>(h);
    });
}

int cbgx_gmres_solve_partitioned_local(uint64_t n, const uint64_t* row_ptrs, const uint64_t* col_idx,
                                       const double* values, const double* b, const double* x0,
                                       const cbgx_gmres_config* cfg, int parts, double* x_out,
                                       cbgx_history* hist, cbgx_solve_stats* stats) {
    return guard([&] {
        if (!cfg || parts < 1) throw Error(CBGX_EINVAL, "partitioned: bad arguments");
        const uint64_t per = (((n + parts - 1) / parts) + 31) / 32 * 32;
        if (per * (parts - 1) >= n) throw Error(CBGX_EINVAL, "partitioned: too many parts for n (32-row blocks)");
        const int dev = current_device();
        auto shared = std::make_shared<LocalShared>(parts);
        std::vector<std::string> errors(parts);
        std::vector<int> codes(parts, CBGX_OK);
        std::vector<uint64_t> err_index(parts, 0);
        auto rank_main = [&](int r) {
            codes[r] = guard([&] {
                CBGX_CUDA(cudaSetDevice(dev));
                cudaStream_t st;
                CBGX_CUDA(cudaStreamCreateWithFlags(&st, cudaStreamNonBlocking));
                LocalComm comm(shared, r);
                const uint64_t rb = std::min<uint64_t>(n, per * r), re = std::min<uint64_t>(n, per * (r + 1));
                const uint64_t k0 = row_ptrs[rb], k1 = row_ptrs[re], nnz = k1 - k0;
                std::vector<int32_t> rp(re - rb + 1);
                for (uint64_t i = rb; i <= re; ++i) rp[i - rb] = static_cast<int32_t>(row_ptrs[i] - k0);
                std::vector<int64_t> gc(col_idx + k0, col_idx + k1);
                void *d_rp = nullptr, *d_gc = nullptr, *d_lc = nullptr, *d_va = nullptr, *d_b = nullptr,
                     *d_x0 = nullptr, *d_x = nullptr;
                auto cleanup = [&] {
                    cudaFree(d_rp); cudaFree(d_gc); cudaFree(d_lc); cudaFree(d_va); cudaFree(d_b);
                    cudaFree(d_x0); cudaFree(d_x); cudaStreamDestroy(st);
                };
                try {
                    const uint64_t nl = re - rb;
                    CBGX_CUDA(cudaMalloc(&d_rp, (nl + 1) * 4));
                    CBGX_CUDA(cudaMalloc(&d_gc, std::max<uint64_t>(nnz, 1) * 8));
                    CBGX_CUDA(cudaMalloc(&d_lc, std::max<uint64_t>(nnz, 1) * 4));
                    CBGX_CUDA(cudaMalloc(&d_va, std::max<uint64_t>(nnz, 1) * 8));
                    CBGX_CUDA(cudaMalloc(&d_b, std::max<uint64_t>(nl, 1) * 8));
                    CBGX_CUDA(cudaMalloc(&d_x0, std::max<uint64_t>(nl, 1) * 8));
                    CBGX_CUDA(cudaMalloc(&d_x, std::max<uint64_t>(nl, 1) * 8));
                    CBGX_CUDA(cudaMemcpy(d_rp, rp.data(), (nl + 1) * 4, cudaMemcpyHostToDevice));
                    CBGX_CUDA(cudaMemcpy(d_gc, gc.data(), nnz * 8, cudaMemcpyHostToDevice));
                    CBGX_CUDA(cudaMemcpy(d_va, values + k0, nnz * 8, cudaMemcpyHostToDevice));
                    CBGX_CUDA(cudaMemcpy(d_b, b + rb, nl * 8, cudaMemcpyHostToDevice));
                    CBGX_CUDA(cudaMemcpy(d_x0, x0 + rb, nl * 8, cudaMemcpyHostToDevice));
                    auto halo = make_halo(&comm, rb, re, n, static_cast<int64_t*>(d_gc), nnz,
                                          static_cast<int32_t*>(d_lc), st);
                    cbgx_csr A{nl, nl + halo->n_ghost, nnz, d_rp, 32, static_cast<int32_t*>(d_lc),
                               static_cast<double*>(d_va)};
                    Solver solver(A, *cfg, &comm, halo.get());
                    cbgx_solve_stats S{};
                    solver.solve(static_cast<double*>(d_b), static_cast<double*>(d_x0), static_cast<double*>(d_x),
                                 r == 0 ? hist : nullptr, &S, st);
                    if (r == 0 && stats) *stats = S;
                    CBGX_CUDA(cudaMemcpy(x_out + rb, d_x, nl * 8, cudaMemcpyDeviceToHost));
                } catch (...) {
                    cleanup();
                    throw;
                }
                cleanup();
            });
            if (codes[r] != CBGX_OK) {
                errors[r] = cbgx_last_error();
                err_index[r] = cbgx_last_error_index();
            }
        };
        std::vector<std::thread> th;
        for (int r = 0; r < parts; ++r) th.emplace_back(rank_main, r);
        for (auto& t : th) t.join();
        for (int r = 0; r < parts; ++r)
            if (codes[r] != CBGX_OK) throw Error(codes[r], errors[r], err_index[r]);
    });
}

}  // extern "C"
