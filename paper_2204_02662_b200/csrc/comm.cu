// Multi-GPU backward aggregation inside the library: one NCCL
// rank per device, destination rows of each execution path sharded by edge
// count, the per-layer y_grad row shards exchanged over NVLink / NVSwitch.
//
// The exchange is the reference caller's "gather_rows(y_grad, ...)" across
// ranks: rank s owns parent-frontier rows [pb[s], pb[s+1]) of the y_grad
// matrix (frontier order, the layout every rank's edge stream indexes). The
// sharded stage issues one ncclBroadcast per owner s, in rank order, on a
// communication stream and records an event after each; the SpMM runs the
// path's source segments — segment s = the edges whose source row lies in
// owner s's rows — on the caller's stream, pass s waiting only for
// broadcast s. Edges are sorted by source row within a destination, so the
// passes in order 0..world-1 are exactly the serial fp32 order: every rank's
// rows are bit-identical to the single-GPU stage while the transfer of later
// shards overlaps the SpMM of earlier ones (tile by tile at shard
// granularity). PG_SHARD_SINGLE_PASS instead waits for the whole exchange
// and runs one pass (no per-segment output re-reads).
//
// NCCL is loaded at first use (dlopen "libnccl.so.2": the copy the host
// process already has — torch's — or the system one), so the library loads
// and runs single-GPU without it.
#include <dlfcn.h>
#include <nccl.h>

#include <cstring>
#include <mutex>
#include <string>
#include <vector>

#include "../../include/pathgcn_b200.h"
#include "pg_internal.h"

namespace pg {

namespace {

struct Nccl {
    decltype(&ncclGetUniqueId) get_unique_id = nullptr;
    decltype(&ncclCommInitRank) init_rank = nullptr;
    decltype(&ncclCommDestroy) destroy = nullptr;
    decltype(&ncclBroadcast) broadcast = nullptr;
    decltype(&ncclGroupStart) group_start = nullptr;
    decltype(&ncclGroupEnd) group_end = nullptr;
    decltype(&ncclSend) send = nullptr;
    decltype(&ncclRecv) recv = nullptr;
    decltype(&ncclGetErrorString) error_string = nullptr;
    decltype(&ncclGetVersion) get_version = nullptr;
    std::string error;
};

const Nccl& nccl() {
    static Nccl n;
    static std::once_flag once;
    std::call_once(once, [] {
        void* h = dlopen("libnccl.so.2", RTLD_NOW | RTLD_GLOBAL);
        if (!h) h = dlopen("libnccl.so", RTLD_NOW | RTLD_GLOBAL);
        if (!h) {
            n.error = std::string("NCCL not loadable: ") + dlerror();
            return;
        }
        auto sym = [&](auto& f, const char* name) {
            f = reinterpret_cast<std::remove_reference_t<decltype(f)>>(dlsym(h, name));
            if (!f && n.error.empty()) n.error = std::string("NCCL symbol missing: ") + name;
        };
        sym(n.get_unique_id, "ncclGetUniqueId");
        sym(n.init_rank, "ncclCommInitRank");
        sym(n.destroy, "ncclCommDestroy");
        sym(n.broadcast, "ncclBroadcast");
        sym(n.group_start, "ncclGroupStart");
        sym(n.group_end, "ncclGroupEnd");
        sym(n.send, "ncclSend");
        sym(n.recv, "ncclRecv");
        sym(n.error_string, "ncclGetErrorString");
        sym(n.get_version, "ncclGetVersion");
    });
    if (!n.error.empty()) fail(kDevice, n.error);
    return n;
}

void nccl_check(ncclResult_t r, const char* what) {
    if (r != ncclSuccess) fail(kDevice, std::string(what) + ": " + nccl().error_string(r));
}

}  // namespace

struct Comm {
    int device = 0, world = 1, rank = 0;
    ncclComm_t comm = nullptr;
    cudaStream_t cs = nullptr;           // communication stream
    cudaEvent_t start = nullptr;         // caller stream -> cs
    std::vector<cudaEvent_t> landed;     // shard s resident
    cudaEvent_t done = nullptr;          // cs -> caller stream
    std::mutex mu;                       // one sharded call at a time per communicator
};

Comm* comm_create(int device, const uint8_t* id, int world, int rank) {
    if (world < 1 || rank < 0 || rank >= world) fail(kConfig, "comm: rank must be in [0, world)");
    const Nccl& n = nccl();
    DeviceGuard dg(device);
    auto c = std::make_unique<Comm>();
    c->device = device;
    c->world = world;
    c->rank = rank;
    ncclUniqueId uid;
    std::memcpy(&uid, id, sizeof(uid));
    nccl_check(n.init_rank(&c->comm, world, uid, rank), "ncclCommInitRank");
    int lo = 0, hi = 0;
    PG_CUDA(cudaDeviceGetStreamPriorityRange(&lo, &hi));
    PG_CUDA(cudaStreamCreateWithPriority(&c->cs, cudaStreamNonBlocking, hi));
    PG_CUDA(cudaEventCreateWithFlags(&c->start, cudaEventDisableTiming));
    PG_CUDA(cudaEventCreateWithFlags(&c->done, cudaEventDisableTiming));
    c->landed.resize(world);
    for (auto& e : c->landed) PG_CUDA(cudaEventCreateWithFlags(&e, cudaEventDisableTiming));
    return c.release();
}

void comm_destroy(Comm* c) {
    if (!c) return;
    DeviceGuard dg(c->device);
    drain_device();
    if (c->comm) nccl().destroy(c->comm);
    for (auto e : c->landed) cudaEventDestroy(e);
    if (c->start) cudaEventDestroy(c->start);
    if (c->done) cudaEventDestroy(c->done);
    if (c->cs) cudaStreamDestroy(c->cs);
    delete c;
}

void comm_unique_id(uint8_t* out) {
    ncclUniqueId uid;
    nccl_check(nccl().get_unique_id(&uid), "ncclGetUniqueId");
    std::memcpy(out, &uid, sizeof(uid));
}

int comm_nccl_version() {
    int v = 0;
    nccl_check(nccl().get_version(&v), "ncclGetVersion");
    return v;
}

// Broadcast the shards of a pitched row matrix (rows [b[s], b[s+1]) owned
// by rank s) in rank order on c.cs after `after` (the caller's stream);
// landed[s] is recorded after shard s. Whole padded rows go over the wire,
// so every shard is one contiguous buffer.
void comm_broadcast_shards(Comm& c, float* rows, uint64_t ld, const uint32_t* b, cudaStream_t after) {
    const Nccl& n = nccl();
    PG_CUDA(cudaEventRecord(c.start, after));
    PG_CUDA(cudaStreamWaitEvent(c.cs, c.start, 0));
    for (int s = 0; s < c.world; ++s) {
        const uint64_t cnt = static_cast<uint64_t>(b[s + 1] - b[s]) * ld;
        if (cnt) {
            float* p = rows + static_cast<uint64_t>(b[s]) * ld;
            nccl_check(n.broadcast(p, p, cnt, ncclFloat32, s, c.comm, c.cs), "ncclBroadcast");
        }
        PG_CUDA(cudaEventRecord(c.landed[s], c.cs));
    }
}

}  // namespace pg

using namespace pg;

namespace {
template <typename F>
int cguard(F&& f) {
    try {
        f();
        return PG_OK;
    } catch (const pg::Error& e) {
        pg::record_error(e);
        return e.code;
    } catch (const std::exception& e) {
        pg::record_error(pg::Error(kConfig, e.what()));
        return PG_ERR_CONFIG;
    }
}
Comm* C_(pg_comm h) {
    if (!h) fail(kConfig, "comm: null handle");
    return reinterpret_cast<Comm*>(h);
}
}  // namespace

extern "C" {

int pg_comm_unique_id(uint8_t* id) {
    return cguard([&] {
        if (!id) fail(kConfig, "comm: null id buffer");
        comm_unique_id(id);
    });
}

int pg_comm_init_rank(int device, const uint8_t* id, int world, int rank, pg_comm* out) {
    return cguard([&] {
        if (!id || !out) fail(kConfig, "comm: null argument");
        *out = reinterpret_cast<pg_comm>(comm_create(device, id, world, rank));
    });
}

int pg_comm_info(pg_comm h, int* world, int* rank, int* nccl_version) {
    return cguard([&] {
        Comm* c = C_(h);
        if (world) *world = c->world;
        if (rank) *rank = c->rank;
        if (nccl_version) *nccl_version = comm_nccl_version();
    });
}

int pg_comm_destroy(pg_comm h) {
    return cguard([&] { comm_destroy(reinterpret_cast<Comm*>(h)); });
}

int pg_comm_allgather_rows(pg_comm h, float* rows, uint64_t ld, const uint32_t* bounds, void* stream) {
    return cguard([&] {
        Comm* c = C_(h);
        if (!bounds) fail(kConfig, "allgather_rows: null bounds");
        for (int s = 0; s < c->world; ++s)
            if (bounds[s + 1] < bounds[s]) fail(kConfig, "allgather_rows: bounds must be non-decreasing");
        if (bounds[c->world] && !rows) fail(kConfig, "allgather_rows: null rows");
        DeviceGuard dg(c->device);
        std::lock_guard<std::mutex> lk(c->mu);
        const cudaStream_t s = static_cast<cudaStream_t>(stream);
        if (c->world > 1) {
            comm_broadcast_shards(*c, rows, ld, bounds, s);
            PG_CUDA(cudaEventRecord(c->done, c->cs));
            PG_CUDA(cudaStreamWaitEvent(s, c->done, 0));
        }
    });
}

int pg_backward_aggregate_sharded(pg_comm h, pg_groups hg, const uint32_t* parent_bounds,
                                  const uint32_t* dest_bounds, float* y_dev, uint64_t y_rows, uint64_t ld_in,
                                  float* x_dev, uint64_t ld_out, uint64_t dim, unsigned flags, void* stream) {
    return cguard([&] {
        Comm* c = C_(h);
        if (!hg) fail(kConfig, "groups: null handle");
        Groups& G = *reinterpret_cast<Groups*>(hg);
        if (!G.path) fail(kConfig, "backward_aggregate: grouping is not over an execution path");
        if (!parent_bounds || !dest_bounds) fail(kConfig, "sharded: null bounds");
        if (flags & PG_AGG_GROUPED) fail(kConfig, "sharded: the grouped Fast kernel runs over whole groupings");
        if (ld_in < dim || ld_out < dim) fail_shape("aggregate_pull: leading dimension smaller than dim");
        Path& p = *G.path;
        if (y_rows != p.P) fail_shape("backward_aggregate: y_grad rows != parent frontier size");
        const int W = c->world;
        if (parent_bounds[0] != 0 || parent_bounds[W] != p.P || dest_bounds[0] != 0 || dest_bounds[W] != p.D)
            fail(kConfig, "sharded: bounds must cover the parent frontier / destination rows");
        for (int s = 0; s < W; ++s)
            if (parent_bounds[s + 1] < parent_bounds[s] || dest_bounds[s + 1] < dest_bounds[s])
                fail(kConfig, "sharded: bounds must be non-decreasing");
        const uint32_t rb = dest_bounds[c->rank], re = dest_bounds[c->rank + 1];
        DeviceGuard dg(c->device);
        std::lock_guard<std::mutex> lk(c->mu);
        std::lock_guard<std::recursive_mutex> glk(G.mu);
        const cudaStream_t s = static_cast<cudaStream_t>(stream);
        if (W == 1) {
            if (re > rb)
                run_aggregate(G, true, rb, re, y_dev, ld_in, x_dev, ld_out, dim, flags & ~PG_SHARD_SINGLE_PASS, s);
            return;
        }
        comm_broadcast_shards(*c, y_dev, ld_in, parent_bounds, s);
        const unsigned f = flags & ~PG_SHARD_SINGLE_PASS;
        if ((flags & PG_SHARD_SINGLE_PASS) || re == rb) {
            PG_CUDA(cudaEventRecord(c->done, c->cs));
            PG_CUDA(cudaStreamWaitEvent(s, c->done, 0));
            if (re > rb) run_aggregate(G, true, rb, re, y_dev, ld_in, x_dev, ld_out, dim, f, s);
            return;
        }
        // source segments at the owners' row cuts (cached on the grouping)
        std::vector<uint64_t> cuts(parent_bounds, parent_bounds + W + 1);
        if (G.seg_cuts != cuts) {
            segment_bounds(p.offsets.get(), p.edges_parent.get(), p.D, cuts.data(), static_cast<uint32_t>(W),
                           G.seg_bnd, lib_stream(G.device));
            G.seg_cuts = cuts;
        }
        for (int k = 0; k < W; ++k) {
            PG_CUDA(cudaStreamWaitEvent(s, c->landed[k], 0));
            run_aggregate(G, true, rb, re, y_dev, ld_in, x_dev, ld_out, dim, k == 0 ? f : (f & ~PG_AGG_OVERWRITE), s,
                          SegSel{G.seg_bnd.get(), k, static_cast<uint32_t>(W)});
        }
        // the caller's later work on y must not race the tail of the exchange
        PG_CUDA(cudaEventRecord(c->done, c->cs));
        PG_CUDA(cudaStreamWaitEvent(s, c->done, 0));
    });
}

}  // extern "C"
