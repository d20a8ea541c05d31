// ring_ipc.cpp -- the ring of vertex sub-parts (O7) moved by
// the copy engines over CUDA IPC instead of NCCL's SM kernels
// (cfg.transport == NE_TRANSPORT_IPC).
//
// Every rank allocates its 2k vertex slots (two ping-pong halves of k
// sub-part slots) and 2k u32 flags as ONE cudaMalloc region, exports it
// (ne_ipc_export), and maps the regions of the ranks it pushes to or credits
// (ne_ipc_connect; the harness all-gathers the handles): g+1 and g-1 on the
// single ring, the group-ring and next-group neighbours with NEXT-3 groups.
// After training (round rho, slot t) rank g pushes the sub-part with one
// cudaMemcpyAsync on its comm stream straight into the other half of slot t of
// D = ring_dest(rho) -- a copy-engine transfer over NVLink between GPUs (a
// plain device copy when two processes share a GPU), no SM involved.
// Ordering uses monotonic counters in flag words, waited on and written by the
// GPU front end (cuStreamWaitValue32 / cuStreamWriteValue32: no kernel, no
// host round trip).  A hop is of kind 0 (along the group's ring) or 1 (to the
// next group, NEXT-3; with one group, the last round's hop); every rank makes
// the same hop kind in the same round, so per-kind, per-slot push counts agree
// on all ranks, and every flag word has exactly one writer (its value never
// goes down -- a flag shared by two writers could be overwritten with an older
// count):
//   * push c of kind k first waits credit[k][t] >= c (D's previous push --
//     the sub-part that occupied the target half -- has left), except the very
//     first push after the ring was set up;
//   * after the copy g writes arrived[k][t] = c at D, and credit[k'][t] =
//     (its next kind-k' push index) at the rank that pushes into g next round;
//   * before training slot t in every round but the first after a load, g
//     waits arrived[k][t] >= (its next expected kind-k arrival).
#include <cuda.h>
#include <cuda_runtime.h>

#include <cstdio>
#include <cstdlib>
#include <cstring>

#include "ne_ctx.h"

namespace {

using WaitFn = CUresult (*)(CUstream, CUdeviceptr, cuuint32_t, unsigned int);
using WriteFn = CUresult (*)(CUstream, CUdeviceptr, cuuint32_t, unsigned int);

struct DriverOps {
    WaitFn wait = nullptr;
    WriteFn write = nullptr;
    bool ok = false;
};

const DriverOps& ops() {
    static DriverOps d = [] {
        DriverOps o;
        cudaDriverEntryPointQueryResult q1, q2;
        void *w = nullptr, *x = nullptr;
        if (cudaGetDriverEntryPoint("cuStreamWaitValue32", &w, cudaEnableDefault, &q1) == cudaSuccess &&
            cudaGetDriverEntryPoint("cuStreamWriteValue32", &x, cudaEnableDefault, &q2) == cudaSuccess &&
            q1 == cudaDriverEntryPointSuccess && q2 == cudaDriverEntryPointSuccess) {
            o.wait = reinterpret_cast<WaitFn>(w);
            o.write = reinterpret_cast<WriteFn>(x);
            o.ok = true;
        }
        cudaGetLastError();
        return o;
    }();
    return d;
}

// The exported description of a rank's region.
struct Blob {
    uint32_t magic, rank, world, subparts;
    uint64_t region_bytes, slot_bytes;
    cudaIpcMemHandle_t handle;
};
constexpr uint32_t kMagic = 0x4E455250u;  // "NERP"

uint32_t* flags_of(const ne_ctx* c, void* region) {
    return reinterpret_cast<uint32_t*>(static_cast<char*>(region) + 2ull * c->cfg.subparts * c->ipc.slot_bytes);
}
// flag words: arrived[kind][t] at [kind * k + t], credit[kind][t] at [2k + kind * k + t]
uint32_t arrived_idx(const ne_ctx* c, uint32_t kind, uint32_t t) { return kind * c->cfg.subparts + t; }
uint32_t credit_idx(const ne_ctx* c, uint32_t kind, uint32_t t) { return (2 + kind) * c->cfg.subparts + t; }

bool ipc_debug() {
    static const bool on = std::getenv("NE_IPC_DEBUG") != nullptr;
    return on;
}

int wait_ge(ne_ctx* c, cudaStream_t s, const uint32_t* flag, uint32_t value) {
    if (ipc_debug()) std::fprintf(stderr, "[ipc rank %d] wait flag %p >= %u\n", c->rank, (const void*)flag, value);
    const CUresult r = ops().wait((CUstream)s, (CUdeviceptr)flag, value, CU_STREAM_WAIT_VALUE_GEQ);
    if (r != CUDA_SUCCESS) return ne_fail(c, NE_ECUDA, "cuStreamWaitValue32 failed (%d)", (int)r);
    return NE_OK;
}

int write_flag(ne_ctx* c, cudaStream_t s, uint32_t* flag, uint32_t value) {
    if (ipc_debug()) std::fprintf(stderr, "[ipc rank %d] write flag %p = %u\n", c->rank, (void*)flag, value);
    const CUresult r = ops().write((CUstream)s, (CUdeviceptr)flag, value, CU_STREAM_WRITE_VALUE_DEFAULT);
    if (r != CUDA_SUCCESS) return ne_fail(c, NE_ECUDA, "cuStreamWriteValue32 failed (%d)", (int)r);
    return NE_OK;
}

void close_peers(ne_ctx* c) {
    for (void*& p : c->ipc.peer)
        if (p && p != c->ipc.region) cudaIpcCloseMemHandle(p);
    c->ipc.peer.clear();
    c->ipc.connected = false;
    c->ipc.blobs.clear();
}

}  // namespace

bool ipc_ring(const ne_ctx* c) { return c->world > 1 && c->cfg.transport == NE_TRANSPORT_IPC; }

int ipc_alloc_slots(ne_ctx* c, size_t slot_bytes, size_t nslots) {
    const uint32_t k = c->cfg.subparts;
    slot_bytes = (slot_bytes + 255) & ~(size_t)255;
    const size_t bytes = nslots * slot_bytes + 4ull * k * sizeof(uint32_t);
    if (!ops().ok) return ne_fail(c, NE_ECUDA, "stream memory operations (cuStreamWaitValue32) unavailable");
    if (c->ipc.region && c->ipc.region_bytes == bytes) {  // same shape: keep region, flags and counters
        for (size_t i = 0; i < nslots; ++i) c->vslot[i] = reinterpret_cast<float*>(static_cast<char*>(c->ipc.region) + i * slot_bytes);
        return NE_OK;
    }
    ipc_release(c);
    NE_CUDA(c, cudaMalloc(&c->ipc.region, bytes));
    c->ipc.region_bytes = bytes;
    c->ipc.slot_bytes = slot_bytes;
    c->ipc.flags = flags_of(c, c->ipc.region);
    // on the compute stream and waited for: the flags must be zero before any
    // peer can write them (the handles are exported after the load returns)
    NE_CUDA(c, cudaMemsetAsync(c->ipc.flags, 0, 4ull * k * sizeof(uint32_t), c->stream));
    NE_CUDA(c, cudaStreamSynchronize(c->stream));
    for (int kind = 0; kind < 2; ++kind) {
        c->ipc.pushed[kind].assign(k, 0);
        c->ipc.waited[kind].assign(k, 0);
    }
    c->ipc.started = false;
    for (size_t i = 0; i < nslots; ++i) c->vslot[i] = reinterpret_cast<float*>(static_cast<char*>(c->ipc.region) + i * slot_bytes);
    return NE_OK;
}

int ipc_reset_on_load(ne_ctx* c) {
    // the previous calls' return-home pushes into this rank were drained; the
    // re-initialised home sub-parts need no arrival
    for (int kind = 0; kind < 2; ++kind) c->ipc.waited[kind] = c->ipc.pushed[kind];
    c->ipc.started = false;
    return NE_OK;
}

int ipc_wait_arrival(ne_ctx* c, uint32_t t, uint32_t kind) {
    return wait_ge(c, c->stream, c->ipc.flags + arrived_idx(c, kind, t), ++c->ipc.waited[kind][t]);
}

int ipc_push(ne_ctx* c, uint32_t t, const void* src, size_t bytes, cudaEvent_t after, uint32_t kind, uint32_t dest,
             uint32_t credit_to, uint32_t next_kind) {
    if (!c->ipc.connected || dest >= c->ipc.peer.size() || credit_to >= c->ipc.peer.size() || !c->ipc.peer[dest] ||
        !c->ipc.peer[credit_to])
        return ne_fail(c, NE_ESTATE, "IPC ring not connected to ranks %u / %u (ne_ipc_export / ne_ipc_connect)", dest,
                       credit_to);
    const uint32_t k = c->cfg.subparts;
    const bool first = c->ipc.pushed[0][t] + c->ipc.pushed[1][t] == 0;
    const uint32_t cnt = ++c->ipc.pushed[kind][t];
    NE_CUDA(c, cudaStreamWaitEvent(c->comm_stream, after, 0));
    if (!first) NE_TRY(wait_ge(c, c->comm_stream, c->ipc.flags + credit_idx(c, kind, t), cnt));  // target half free
    const size_t half = (size_t)(1 - c->cur) * k + t;                                         // the other half of dest
    char* dst = static_cast<char*>(c->ipc.peer[dest]) + half * c->ipc.slot_bytes;
    NE_CUDA(c, cudaMemcpyAsync(dst, src, bytes, cudaMemcpyDeviceToDevice, c->comm_stream));
    NE_TRY(write_flag(c, c->comm_stream, flags_of(c, c->ipc.peer[dest]) + arrived_idx(c, kind, t), cnt));
    NE_TRY(write_flag(c, c->comm_stream, flags_of(c, c->ipc.peer[credit_to]) + credit_idx(c, next_kind, t),
                      c->ipc.pushed[next_kind][t] + 1));
    c->ipc.started = true;
    return NE_OK;
}

int ipc_wait_home(ne_ctx* c, cudaStream_t s, uint32_t t, uint32_t kind) {
    // the push of this call's last round into slot t has landed (no arrival consumed)
    return wait_ge(c, s, c->ipc.flags + arrived_idx(c, kind, t), c->ipc.pushed[kind][t]);
}

int ipc_drain(ne_ctx* c, bool host_sync) {
    if (!c->ipc.region || !c->ipc.connected) return NE_OK;
    const uint32_t k = c->cfg.subparts;
    const uint32_t G = c->cfg.groups > 1 ? c->cfg.groups : 1, L = (uint32_t)c->world / G;
    const uint32_t k0 = L > 1 ? 0u : 1u;  // kind of the round-0 hop's credit (the next call's first push)
    for (uint32_t t = 0; t < k; ++t) {
        if (c->ipc.pushed[0][t] + c->ipc.pushed[1][t] == 0) continue;
        for (uint32_t kind = 0; kind < 2; ++kind)  // every push into me landed
            NE_TRY(wait_ge(c, c->stream, c->ipc.flags + arrived_idx(c, kind, t), c->ipc.pushed[kind][t]));
        // the last credit write into me (after the final round) landed
        NE_TRY(wait_ge(c, c->stream, c->ipc.flags + credit_idx(c, k0, t), c->ipc.pushed[k0][t] + 1));
        for (uint32_t kind = 0; kind < 2; ++kind) c->ipc.waited[kind][t] = c->ipc.pushed[kind][t];
    }
    c->ipc.started = false;
    if (host_sync) {
        NE_CUDA(c, cudaStreamSynchronize(c->comm_stream));
        NE_CUDA(c, cudaStreamSynchronize(c->stream));
    }
    return NE_OK;
}

void ipc_release(ne_ctx* c) {
    close_peers(c);
    if (c->ipc.region) cudaFree(c->ipc.region);
    c->ipc.region = nullptr;
    c->ipc.flags = nullptr;
    c->ipc.region_bytes = c->ipc.slot_bytes = 0;
    c->ipc.started = false;
}

extern "C" {

size_t ne_ipc_blob_size(void) { return sizeof(Blob); }

int ne_ipc_export(ne_ctx* c, void* blob, size_t cap) {
    if (!c || !blob) return NE_EINVAL;
    c->err.clear();
    NE_CUDA(c, cudaSetDevice(c->device));
    if (!ipc_ring(c)) return ne_fail(c, NE_ESTATE, "transport is not NE_TRANSPORT_IPC or world == 1");
    if (!c->ipc.region) return ne_fail(c, NE_ESTATE, "no vertex slots yet (call ne_load_graph first)");
    if (cap < sizeof(Blob)) return ne_fail(c, NE_ERANGE, "blob capacity %zu < %zu", cap, sizeof(Blob));
    Blob b{};
    b.magic = kMagic;
    b.rank = (uint32_t)c->rank;
    b.world = (uint32_t)c->world;
    b.subparts = c->cfg.subparts;
    b.region_bytes = c->ipc.region_bytes;
    b.slot_bytes = c->ipc.slot_bytes;
    NE_CUDA(c, cudaIpcGetMemHandle(&b.handle, c->ipc.region));
    std::memcpy(blob, &b, sizeof b);
    return NE_OK;
}

int ne_ipc_connect(ne_ctx* c, const void* blobs, size_t blob_size) {
    if (!c || !blobs) return NE_EINVAL;
    c->err.clear();
    NE_CUDA(c, cudaSetDevice(c->device));
    if (!ipc_ring(c)) return ne_fail(c, NE_ESTATE, "transport is not NE_TRANSPORT_IPC or world == 1");
    if (blob_size != sizeof(Blob)) return ne_fail(c, NE_EINVAL, "blob size %zu != %zu", blob_size, sizeof(Blob));
    const uint32_t P = (uint32_t)c->world, g = (uint32_t)c->rank;
    const uint32_t G = c->cfg.groups > 1 ? c->cfg.groups : 1;
    // the ranks this one pushes into and credits over the P rounds of a call
    std::vector<bool> need(P, false);
    for (uint32_t rho = 0; rho < P; ++rho) {
        need[ring_dest(P, G, rho, g)] = true;
        need[ring_src(P, G, rho + 1, g)] = true;
    }
    for (uint32_t q = 0; q < P; ++q) {
        if (!need[q]) continue;
        Blob b;
        std::memcpy(&b, static_cast<const char*>(blobs) + (size_t)q * blob_size, sizeof b);
        if (b.magic != kMagic || b.world != P || b.subparts != c->cfg.subparts ||
            b.region_bytes != c->ipc.region_bytes || b.slot_bytes != c->ipc.slot_bytes)
            return ne_fail(c, NE_EINVAL, "IPC blob of rank %u does not match this ring (world %u, subparts %u, "
                                         "region %llu bytes)", q, P, c->cfg.subparts,
                           (unsigned long long)c->ipc.region_bytes);
        if (b.rank != q) return ne_fail(c, NE_EINVAL, "IPC blobs out of rank order (slot %u holds rank %u)", q, b.rank);
    }
    // a reload of a graph of the same shape keeps every region: the handles
    // match the open ones, nothing to re-map
    std::string all(static_cast<const char*>(blobs), (size_t)P * blob_size);
    if (c->ipc.connected && all == c->ipc.blobs) return NE_OK;
    close_peers(c);
    c->ipc.peer.assign(P, nullptr);
    for (uint32_t q = 0; q < P; ++q) {
        if (!need[q]) continue;
        Blob b;
        std::memcpy(&b, static_cast<const char*>(blobs) + (size_t)q * blob_size, sizeof b);
        if (q == g) {  // a one-rank group pushes into itself: its own region
            c->ipc.peer[q] = c->ipc.region;
            continue;
        }
        NE_CUDA(c, cudaIpcOpenMemHandle(&c->ipc.peer[q], b.handle, cudaIpcMemLazyEnablePeerAccess));
    }
    c->ipc.connected = true;
    c->ipc.blobs = std::move(all);
    return NE_OK;
}

}  // extern "C"
