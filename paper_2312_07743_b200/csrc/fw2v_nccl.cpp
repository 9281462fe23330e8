// NCCL for the replica average of data-parallel runs.
//
// libnccl.so.2 is opened at run time (dlopen), so libfw2v.so loads and trains
// on one GPU without it. Inside a Python process that already loaded torch's
// NCCL the soname resolves to that copy; a plain C++ process (ringvec::train
// drop-in) gets the system library. Only the types are taken from <nccl.h>.
//
// A clique is one NCCL communicator per local member:
//   * in-process: ncclCommInitAll over the members' devices (one process
//     driving several GPUs, fw2v_train_corpus_multi / ringvec::train with
//     FW2V_GPUS > 1);
//   * cross-process: ncclCommInitRank with a unique id the caller distributes
//     (one process per GPU, bench.py under torchrun).
// The average is one in-place ncclAllReduce(ncclFloat32, ncclAvg) per matrix —
// NVLink / NVSwitch (NVLS) on a B200 node.
#include <cuda_runtime.h>
#include <dlfcn.h>
#include <nccl.h>

#include <cstdlib>
#include <cstring>
#include <memory>
#include <mutex>
#include <string>
#include <vector>

namespace fw2v {

namespace {

struct NcclApi {
    bool ok = false;
    std::string why;
    ncclResult_t (*GetUniqueId)(ncclUniqueId*) = nullptr;
    ncclResult_t (*CommInitAll)(ncclComm_t*, int, const int*) = nullptr;
    ncclResult_t (*CommInitRank)(ncclComm_t*, int, ncclUniqueId, int) = nullptr;
    ncclResult_t (*CommDestroy)(ncclComm_t) = nullptr;
    ncclResult_t (*AllReduce)(const void*, void*, size_t, ncclDataType_t, ncclRedOp_t, ncclComm_t, cudaStream_t) = nullptr;
    ncclResult_t (*GroupStart)() = nullptr;
    ncclResult_t (*GroupEnd)() = nullptr;
    const char* (*GetErrorString)(ncclResult_t) = nullptr;
};

const NcclApi& api() {
    static NcclApi a;
    static std::once_flag once;
    std::call_once(once, [] {
        // FW2V_NCCL_LIB: an explicit library (the Python binding points it at
        // torch's bundled NCCL so torch, imported later, binds to the same copy).
        void* h = nullptr;
        if (const char* p = std::getenv("FW2V_NCCL_LIB"); p != nullptr && *p != 0) h = dlopen(p, RTLD_NOW | RTLD_GLOBAL);
        if (h == nullptr) h = dlopen("libnccl.so.2", RTLD_NOW | RTLD_GLOBAL);
        if (h == nullptr) h = dlopen("libnccl.so", RTLD_NOW | RTLD_GLOBAL);
        if (h == nullptr) {
            const char* e = dlerror();
            a.why = std::string("libnccl.so.2 not loadable: ") + (e ? e : "?");
            return;
        }
        auto sym = [&](const char* n) { return dlsym(h, n); };
        a.GetUniqueId = reinterpret_cast<decltype(a.GetUniqueId)>(sym("ncclGetUniqueId"));
        a.CommInitAll = reinterpret_cast<decltype(a.CommInitAll)>(sym("ncclCommInitAll"));
        a.CommInitRank = reinterpret_cast<decltype(a.CommInitRank)>(sym("ncclCommInitRank"));
        a.CommDestroy = reinterpret_cast<decltype(a.CommDestroy)>(sym("ncclCommDestroy"));
        a.AllReduce = reinterpret_cast<decltype(a.AllReduce)>(sym("ncclAllReduce"));
        a.GroupStart = reinterpret_cast<decltype(a.GroupStart)>(sym("ncclGroupStart"));
        a.GroupEnd = reinterpret_cast<decltype(a.GroupEnd)>(sym("ncclGroupEnd"));
        a.GetErrorString = reinterpret_cast<decltype(a.GetErrorString)>(sym("ncclGetErrorString"));
        a.ok = a.GetUniqueId && a.CommInitAll && a.CommInitRank && a.CommDestroy && a.AllReduce && a.GroupStart &&
               a.GroupEnd && a.GetErrorString;
        if (!a.ok) a.why = "libnccl.so.2 lacks a required symbol";
    });
    return a;
}

bool check(ncclResult_t r, const char* what, std::string* err) {
    if (r == ncclSuccess) return true;
    *err = std::string(what) + ": " + api().GetErrorString(r);
    return false;
}

} // namespace

struct NcclClique {
    std::vector<int> devices;          // local members' devices
    std::vector<ncclComm_t> comms;     // one per local member
    std::vector<cudaStream_t> streams; // one per local member, on its device
    int world = 1, rank0 = 0;          // cross-process: ranks rank0 .. rank0 + local - 1 of world
    ~NcclClique() {
        for (size_t i = 0; i < comms.size(); ++i) {
            cudaSetDevice(devices[i]);
            if (streams[i]) cudaStreamSynchronize(streams[i]);
            if (comms[i]) api().CommDestroy(comms[i]);
            if (streams[i]) cudaStreamDestroy(streams[i]);
        }
    }
};

bool nccl_available(std::string* why) {
    const NcclApi& a = api();
    if (!a.ok && why) *why = a.why;
    return a.ok;
}

bool nccl_unique_id(uint8_t out[NCCL_UNIQUE_ID_BYTES], std::string* err) {
    if (!nccl_available(err)) return false;
    ncclUniqueId id;
    if (!check(api().GetUniqueId(&id), "ncclGetUniqueId", err)) return false;
    static_assert(sizeof(id) == NCCL_UNIQUE_ID_BYTES, "ncclUniqueId size");
    std::memcpy(out, &id, sizeof(id));
    return true;
}

static bool make_streams(NcclClique& c, std::string* err) {
    c.streams.assign(c.devices.size(), nullptr);
    for (size_t i = 0; i < c.devices.size(); ++i) {
        cudaSetDevice(c.devices[i]);
        cudaError_t e = cudaStreamCreateWithFlags(&c.streams[i], cudaStreamNonBlocking);
        if (e != cudaSuccess) {
            *err = std::string("cudaStreamCreate: ") + cudaGetErrorString(e);
            return false;
        }
    }
    return true;
}

// In-process clique over distinct devices.
std::shared_ptr<NcclClique> nccl_clique_local(const std::vector<int>& devices, std::string* err) {
    if (!nccl_available(err)) return nullptr;
    auto c = std::make_shared<NcclClique>();
    c->devices = devices;
    c->world = static_cast<int>(devices.size());
    c->comms.assign(devices.size(), nullptr);
    if (!check(api().CommInitAll(c->comms.data(), static_cast<int>(devices.size()), devices.data()), "ncclCommInitAll",
               err))
        return nullptr;
    if (!make_streams(*c, err)) return nullptr;
    return c;
}

// Cross-process clique: this process is rank `rank` of `world`, one device.
std::shared_ptr<NcclClique> nccl_clique_rank(int device, const uint8_t id_bytes[NCCL_UNIQUE_ID_BYTES], int world,
                                             int rank, std::string* err) {
    if (!nccl_available(err)) return nullptr;
    auto c = std::make_shared<NcclClique>();
    c->devices = {device};
    c->world = world;
    c->rank0 = rank;
    c->comms.assign(1, nullptr);
    ncclUniqueId id;
    std::memcpy(&id, id_bytes, sizeof(id));
    cudaSetDevice(device);
    if (!check(api().CommInitRank(&c->comms[0], world, id, rank), "ncclCommInitRank", err)) return nullptr;
    if (!make_streams(*c, err)) return nullptr;
    return c;
}

// In place: every member's buffers[i] (count floats each) <- the mean (sum =
// false) or the sum over all members of all processes; u64[i] (may be null) <-
// the sum. Synchronous: returns after every member's stream finished.
bool nccl_allreduce(NcclClique& c, const std::vector<std::vector<float*>>& buffers, size_t count,
                    const std::vector<unsigned long long*>& u64, bool sum, std::string* err) {
    const NcclApi& a = api();
    if (!check(a.GroupStart(), "ncclGroupStart", err)) return false;
    bool ok = true;
    for (size_t i = 0; i < c.comms.size() && ok; ++i) {
        cudaSetDevice(c.devices[i]);
        for (float* b : buffers[i])
            ok = ok && check(a.AllReduce(b, b, count, ncclFloat32, sum ? ncclSum : ncclAvg, c.comms[i], c.streams[i]), "ncclAllReduce", err);
        if (ok && i < u64.size() && u64[i] != nullptr)
            ok = check(a.AllReduce(u64[i], u64[i], 1, ncclUint64, ncclSum, c.comms[i], c.streams[i]), "ncclAllReduce", err);
    }
    ncclResult_t ge = a.GroupEnd();
    if (ok && !check(ge, "ncclGroupEnd", err)) ok = false;
    for (size_t i = 0; i < c.comms.size(); ++i) {
        cudaSetDevice(c.devices[i]);
        cudaError_t e = cudaStreamSynchronize(c.streams[i]);
        if (ok && e != cudaSuccess) {
            *err = std::string("NCCL stream: ") + cudaGetErrorString(e);
            ok = false;
        }
    }
    return ok;
}

} // namespace fw2v
