// cf_api.cu — the C-ABI of include/castfem_b200.h: plan object, upload,
// stepping (CUDA graphs), multi-rank exchange (in-process, NCCL, peer memory or host-staged), and the
// host utilities. Reference interfaces replaced are cited at each entry point
// in include/castfem_b200.h.
#include <cuda.h>
#include <cuda_runtime.h>
#include <dlfcn.h>
#include <nccl.h>

#include <algorithm>
#include <chrono>
#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <memory>
#include <mutex>
#include <numeric>
#include <string>
#include <vector>

#include "cf_devplan.hpp"
#include "cf_internal.hpp"
#include "cf_kernels.cuh"

using namespace cfb;

// ------------------------------------------------------------------ errors
namespace cfb {
static thread_local std::string g_last_error;
bool cuda_device_present() {
    int n = 0;
    const bool ok = cudaGetDeviceCount(&n) == cudaSuccess && n > 0;
    cudaGetLastError();
    return ok;
}
void set_last_error(const std::string& msg) { g_last_error = msg; }
}  // namespace cfb

#define CF_CUDA_CHECK(x)                                                                                   \
    do {                                                                                                   \
        cudaError_t e_ = (x);                                                                              \
        if (e_ != cudaSuccess) raise(CF_CUDA, std::string(#x) + ": " + cudaGetErrorString(e_));            \
    } while (0)

template <class F>
static int guarded(F&& f) {
    try {
        f();
        return CF_OK;
    } catch (const Error& e) {
        set_last_error(e.what());
        return e.code;
    } catch (const std::bad_alloc&) {
        set_last_error("host out of memory");
        return CF_INVALID_ARG;
    } catch (const std::exception& e) {
        set_last_error(e.what());
        return CF_INVALID_ARG;
    }
}

// ------------------------------------------------------------------ NCCL (dlopen)
namespace {
struct NcclApi {
    void* h = nullptr;
    ncclResult_t (*GetUniqueId)(ncclUniqueId*) = nullptr;
    ncclResult_t (*CommInitRank)(ncclComm_t*, int, ncclUniqueId, int) = nullptr;
    ncclResult_t (*CommDestroy)(ncclComm_t) = nullptr;
    ncclResult_t (*Send)(const void*, size_t, ncclDataType_t, int, ncclComm_t, cudaStream_t) = nullptr;
    ncclResult_t (*Recv)(void*, size_t, ncclDataType_t, int, ncclComm_t, cudaStream_t) = nullptr;
    ncclResult_t (*GroupStart)() = nullptr;
    ncclResult_t (*GroupEnd)() = nullptr;
    ncclResult_t (*AllReduce)(const void*, void*, size_t, ncclDataType_t, ncclRedOp_t, ncclComm_t,
                              cudaStream_t) = nullptr;
    const char* (*GetErrorString)(ncclResult_t) = nullptr;
};
NcclApi& nccl() {
    static NcclApi api;
    static std::once_flag once;
    std::call_once(once, [] {
        const char* names[] = {"libnccl.so.2", "libnccl.so"};
        for (const char* n : names)
            if ((api.h = dlopen(n, RTLD_NOW | RTLD_GLOBAL))) break;
        if (!api.h) return;
        api.GetUniqueId = (decltype(api.GetUniqueId))dlsym(api.h, "ncclGetUniqueId");
        api.CommInitRank = (decltype(api.CommInitRank))dlsym(api.h, "ncclCommInitRank");
        api.CommDestroy = (decltype(api.CommDestroy))dlsym(api.h, "ncclCommDestroy");
        api.Send = (decltype(api.Send))dlsym(api.h, "ncclSend");
        api.Recv = (decltype(api.Recv))dlsym(api.h, "ncclRecv");
        api.GroupStart = (decltype(api.GroupStart))dlsym(api.h, "ncclGroupStart");
        api.GroupEnd = (decltype(api.GroupEnd))dlsym(api.h, "ncclGroupEnd");
        api.AllReduce = (decltype(api.AllReduce))dlsym(api.h, "ncclAllReduce");
        api.GetErrorString = (decltype(api.GetErrorString))dlsym(api.h, "ncclGetErrorString");
    });
    if (!api.h || !api.Send || !api.Recv || !api.CommInitRank) raise(CF_NCCL, "libnccl.so.2 not loadable");
    return api;
}
#define CF_NCCL_CHECK(x)                                                                                 \
    do {                                                                                                 \
        ncclResult_t r_ = (x);                                                                           \
        if (r_ != ncclSuccess) raise(CF_NCCL, std::string(#x) + ": " + nccl().GetErrorString(r_));       \
    } while (0)
}  // namespace

struct cf_comm {
    ncclComm_t comm = nullptr;
    int world = 1, rank = 0, device = 0;
    bool host = false;        // host-staged transport (cf_comm_create_host): callbacks instead of NCCL
    bool peer = false;        // peer-memory transport (cf_comm_create_peer): ht only bootstraps the windows
    cf_host_transport ht{};
};

// ------------------------------------------------------------------ plan
namespace {

struct DeviceMem {
    std::vector<void*> ptrs;
    int64_t bytes = 0;
    template <class T>
    T* alloc(size_t n) {
        if (n == 0) n = 1;
        void* p = nullptr;
        CF_CUDA_CHECK(cudaMalloc(&p, n * sizeof(T)));
        ptrs.push_back(p);
        bytes += (int64_t)(n * sizeof(T));
        return (T*)p;
    }
    template <class T, class A>
    T* up(const std::vector<T, A>& v, cudaStream_t s) {
        T* p = alloc<T>(v.size());
        if (!v.empty()) copy_h2d(p, v.data(), v.size() * sizeof(T), s);
        return p;
    }
    // large uploads go through two pinned staging buffers (parallel host copy into one while
    // the other's DMA runs): ~3-4x the pageable rate on the multi-GB tile blobs
    static void copy_h2d(void* dst, const void* src, size_t bytes, cudaStream_t s) {
        constexpr size_t kChunk = 64u << 20;
        if (bytes < 2 * kChunk) {
            CF_CUDA_CHECK(cudaMemcpyAsync(dst, src, bytes, cudaMemcpyHostToDevice, s));
            return;
        }
        if (!std::getenv("CF_UPLOAD_STAGED")) {  // pin the source in place: DMA at link speed
            if (cudaHostRegister((void*)src, bytes, cudaHostRegisterReadOnly) == cudaSuccess) {
                CF_CUDA_CHECK(cudaMemcpyAsync(dst, src, bytes, cudaMemcpyHostToDevice, s));
                CF_CUDA_CHECK(cudaStreamSynchronize(s));
                cudaHostUnregister((void*)src);
                return;
            }
            cudaGetLastError();  // registration refused: fall back to staging
        }
        void* buf[2] = {nullptr, nullptr};
        cudaEvent_t ev[2] = {nullptr, nullptr};
        struct Free {
            void** b;
            cudaEvent_t* e;
            ~Free() {
                for (int k = 0; k < 2; ++k) {
                    if (e[k]) cudaEventSynchronize(e[k]), cudaEventDestroy(e[k]);
                    if (b[k]) cudaFreeHost(b[k]);
                }
            }
        } guard{buf, ev};
        for (int k = 0; k < 2; ++k) {
            CF_CUDA_CHECK(cudaMallocHost(&buf[k], kChunk));
            CF_CUDA_CHECK(cudaEventCreateWithFlags(&ev[k], cudaEventDisableTiming));
        }
        int k = 0;
        for (size_t off = 0; off < bytes; off += kChunk, k ^= 1) {
            const size_t n = std::min(kChunk, bytes - off);
            CF_CUDA_CHECK(cudaEventSynchronize(ev[k]));  // this buffer's previous DMA is done
            const char* from = (const char*)src + off;
            char* to = (char*)buf[k];
            const int parts = 16;
#pragma omp parallel for schedule(static)
            for (int q = 0; q < parts; ++q) {
                const size_t a = n * q / parts, b = n * (q + 1) / parts;
                std::memcpy(to + a, from + a, b - a);
            }
            CF_CUDA_CHECK(cudaMemcpyAsync((char*)dst + off, buf[k], n, cudaMemcpyHostToDevice, s));
            CF_CUDA_CHECK(cudaEventRecord(ev[k], s));
        }
    }
    void release() {
        for (void* p : ptrs) cudaFree(p);
        ptrs.clear();
    }
    void adopt(cfb::DBuf& b) {  // a device-built plan's allocations
        ptrs.insert(ptrs.end(), b.p.begin(), b.p.end());
        bytes += b.bytes;
        b.p.clear();
        b.sz.clear();
        b.bytes = 0;
    }
};

struct Rank {
    int32_t rank = 0;
    RankPlan H;          // host plan (metadata kept; big arrays cleared after upload)
    DeviceMem mem;
    TileArgs ta{};
    UpdArgs ua{};
    PackArgs pa{};
    // T ring: T[cur] = T^k, T[nxt] = T^{k+1} (written during the step, including by
    // the tile kernel's fused private updates), T[old] = T^{k-1} (the lagged
    // interface ambient of refresh_ambient blocked.hpp:441-449; never written
    // during a step — a two-buffer ping-pong would race with the fused updates)
    double* T[3] = {nullptr, nullptr, nullptr};
    double* Tslot[2] = {nullptr, nullptr};  // per-slot T copies (ping-pong)
    int32_t* sched = nullptr;               // dynamic tile-scheduling counter (persistent grids)
    // decomposed plans, border tiles first in one launch (fused_border): completion counter + flag
    // raised by the tile kernel, waited on by the exchange stream; border_seq = steps launched
    bool fused_border = false;
    unsigned long long* border_cnt = nullptr;
    uint32_t* border_flag = nullptr;
    uint32_t border_seq = 0;
    double* recv = nullptr;
    double* send = nullptr;
    double2* acc = nullptr;  // atomic mode: per node (c, r) accumulators
    double2* part = nullptr;
    DevState* st = nullptr;
    // tile launches of one step: tiles grouped by shared-memory footprint, so the common
    // tiles are not sized (and occupancy-limited) by the largest interface tile
    struct TileLaunch {
        TileArgs a;
        size_t smem;
        int grid;
        int phase;  // 0: border tiles (multi-rank), 1: the rest
        int heavy;  // footprint outlier class: concurrent launch on the side stream
    };
    std::vector<TileLaunch> launches;
    int32_t* shared_list = nullptr;
    int4* shared_rec = nullptr;     // packed update records of shared_list
    int2* shared_rec2 = nullptr;    // their slots 6, 7
    int32_t n_shared_list = 0;
    size_t tile_smem = 0;
    int upd_blocks = 0, upd_blocks_all = 0;
    int64_t bytes_per_step = 0;
    int64_t tile_bytes = 0;  // layout bytes of one tile-kernel launch
    int64_t update_bytes = 0;  // algorithmic bytes of the merge + update kernel per step
    int64_t S_tot = 0, E_r = 0;  // slots, elements of this rank
    std::vector<int64_t> nb_send_len, nb_recv_len;
};

}  // namespace

struct cf_plan {
    int device = 0;
    cudaStream_t stream = nullptr;
    cudaStream_t side = nullptr;              // concurrent launch of the heavy tile class
    cudaEvent_t fork = nullptr, join = nullptr;
    cudaStream_t xside = nullptr;             // multi-rank: pack + exchange beside the interior tiles
    DevState** d_states = nullptr;            // in-process ranks' step states (dynamic-dt combine)
    cudaEvent_t xfork = nullptr, xjoin = nullptr;
    cudaEvent_t ev0 = nullptr, ev1 = nullptr;
    int mode = CF_MODE_ATOMIC;
    int tile_threads = 128;      // CTA size of the tile kernel (128 | 256)
    bool pdl = true;             // programmatic dependent launch between the step's kernels (CF_PDL=0: off)
    int stages = 1;              // 1: one tile per CTA; 2: persistent double-buffered TMA pipeline
    // slot temperatures: per-slot copies written by the update (default), or gathered by the tiles
    // from T by node id (CF_SLOT_GATHER=1: update -27 %, tile kernel +7 % at cfg5, net -4 %;
    // saves the 2 x 8 B/slot copies, 4.2 GB at cfg5)
    bool slot_gather = false;
    // the next tile's blob staged into L2 during the reduction (CF_L2_NEXT=0: off): cfg2 tile
    // kernel -4 %, cfg4 / cfg5 unchanged (profiles/r02r_l2_next_ab.txt)
    bool l2_next = true;
    int world = 1, first_rank = 0, local_ranks = 1;
    cf_comm* comm = nullptr;
    DevParams P{};
    DevParams* dP = nullptr;
    bool temp_dep = false, finite_range = false, any_dir = false;
    std::vector<std::unique_ptr<Rank>> ranks;
    int cur = 0;                 // index of the current T buffer (ring of 3)
    int nxt() const { return (cur + 1) % 3; }
    int old() const { return (cur + 2) % 3; }
    int step_parity = 0;
    void advance() {
        cur = (cur + 1) % 3;
        step_parity ^= 1;
    }
    int32_t N_global = 0;
    int64_t E_global = 0;
    bool device_setup = false;
    double loop_seconds = 0;
    double eq13_min = 0;
    double base_min_bound = 0;   // min_e rho c(0) l^2 / k(0) (static dt before the safety factor)
    int64_t launches_per_step = 0;
    int64_t output_every = 0;
    double t_end_setup = 0;
    // graph
    double* h_send = nullptr;    // host-staged transport: pinned copies of the send / recv payloads
    double* h_recv = nullptr;
    bool host_comm() const { return comm && comm->host && world > local_ranks; }
    bool peer_comm() const { return comm && comm->peer && world > local_ranks; }
    // peer-memory transport: this rank's exported window [control | recv x 2 parities] and the
    // other ranks' windows as mapped here (CUDA IPC)
    struct Peer {
        uint8_t* win = nullptr;
        std::vector<uint8_t*> mapped;          // [world]; own entry = win
        uint8_t** d_win = nullptr;             // device copy of mapped
        std::vector<double*> nb_dst;           // per neighbour: its receive region for this rank (parity 0)
        std::vector<int64_t> nb_stride;        // per neighbour: its receive-buffer length (parity stride)
        uint32_t seq = 0, rseq = 0;            // exchanges / reductions issued so far
        bool open = false;
        cf_host_transport boot{};              // bootstrap callbacks (copied: the barrier at destruction)
    } peer;
    double* dTg = nullptr;       // global-order staging (device) for set_temperature / get_fields
    double* dHg = nullptr;
    int64_t graph_steps = 0;
    cudaGraphExec_t graph = nullptr;
    double graph_t_end = 0;
    int graph_cur = -1;
    ~cf_plan() {
        if (graph) cudaGraphExecDestroy(graph);
        peer_close();
        for (auto& r : ranks) r->mem.release();
        if (dP) cudaFree(dP);
        if (dTg) cudaFree(dTg);
        if (dHg) cudaFree(dHg);
        if (ev0) cudaEventDestroy(ev0);
        if (ev1) cudaEventDestroy(ev1);
        if (fork) cudaEventDestroy(fork);
        if (join) cudaEventDestroy(join);
        if (side) cudaStreamDestroy(side);
        if (xfork) cudaEventDestroy(xfork);
        if (xjoin) cudaEventDestroy(xjoin);
        if (xside) cudaStreamDestroy(xside);
        if (d_states) cudaFree(d_states);
        if (h_send) cudaFreeHost(h_send);
        if (h_recv) cudaFreeHost(h_recv);
        if (stream) cudaStreamDestroy(stream);
    }
    // The importers unmap a window before its owner frees it (cudaIpcOpenMemHandle's contract):
    // every rank closes its mappings, then all meet on the bootstrap transport, then the owners free.
    void peer_close() {
        if (!peer.open) return;
        peer.open = false;
        cudaSetDevice(device);
        if (stream) cudaStreamSynchronize(stream);
        if (xside) cudaStreamSynchronize(xside);
        for (size_t q = 0; q < peer.mapped.size(); ++q)
            if (peer.mapped[q] && peer.mapped[q] != peer.win) cudaIpcCloseMemHandle(peer.mapped[q]);
        peer.mapped.clear();
        if (peer.d_win) cudaFree(peer.d_win);
        peer.d_win = nullptr;
        double one = 1.0;
        if (peer.boot.allreduce) peer.boot.allreduce(peer.boot.ctx, &one, 1, CF_REDUCE_MAX);
    }
};

namespace {

// dynamic shared memory of the tile kernel: [stage blobs][stage slot T][(T, H) per slot][contribution
// scratch (coordinates layout only)], for the largest blob / slot count / scratch of the launch's tiles
struct SmemMax {
    int64_t blob = 0, slots = 0, scratch = 0;
};
// blob stage(s), slot-temperature buffer(s) (two with gathered slots), (T, H) per slot, scratch
size_t tile_scratch_off(const SmemMax& m, int stages, bool gather) {
    const int nsT = (stages == 2 || gather) ? 2 : 1;
    return stages * (size_t)cf_round(m.blob, 16) + nsT * 8 * (size_t)m.slots + 16 * (size_t)m.slots;
}
size_t tile_smem_bytes(const SmemMax& m, int stages, bool gather) {
    return tile_scratch_off(m, stages, gather) + 8 * (size_t)cf_round(m.scratch, 2) + 16;
}

#define CF_TILE_VARIANTS_NT(X, NT, G)                                                                          \
    X(true, true, true, true, NT, G) X(true, true, true, false, NT, G) X(true, true, false, true, NT, G)          \
    X(true, true, false, false, NT, G) X(true, false, true, true, NT, G) X(true, false, true, false, NT, G)       \
    X(true, false, false, true, NT, G) X(true, false, false, false, NT, G) X(false, true, true, true, NT, G)      \
    X(false, true, true, false, NT, G) X(false, true, false, true, NT, G) X(false, true, false, false, NT, G)     \
    X(false, false, true, true, NT, G) X(false, false, true, false, NT, G) X(false, false, false, true, NT, G)    \
    X(false, false, false, false, NT, G)
#define CF_TILE_VARIANTS(X)                                                                       \
    CF_TILE_VARIANTS_NT(X, 128, true) CF_TILE_VARIANTS_NT(X, 256, true) CF_TILE_VARIANTS_NT(X, 128, false) \
    CF_TILE_VARIANTS_NT(X, 256, false)

void set_tile_attr(size_t smem) {
#define CF_ATTR(D, T, R, C, NT, G)                                                                \
    CF_CUDA_CHECK(cudaFuncSetAttribute(tile_kernel<D, T, R, C, NT, G>,                                    \
                                       cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
    CF_TILE_VARIANTS(CF_ATTR)
#undef CF_ATTR
}

// kernel launch with programmatic dependent launch (griddepcontrol in the kernels)
template <typename Kern, typename... Args>
void launch_ex(Kern kern, dim3 grid, dim3 block, size_t smem, cudaStream_t st, bool pdl, Args... args) {
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = grid;
    cfg.blockDim = block;
    cfg.dynamicSmemBytes = smem;
    cfg.stream = st;
    cudaLaunchAttribute at[1];
    at[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    at[0].val.programmaticStreamSerializationAllowed = 1;
    cfg.attrs = at;
    cfg.numAttrs = pdl ? 1 : 0;
    CF_CUDA_CHECK(cudaLaunchKernelEx(&cfg, kern, args...));
}

// phase: 0 border tiles, 1 interior tiles, -1 both
void launch_tile(cf_plan* p, Rank& r, double t_end, int phase = -1) {
    if (r.H.n_tiles == 0) return;
    const bool det = p->mode == CF_MODE_DETERMINISTIC;
    const bool dir = r.ua.node_dir != nullptr, cl = p->finite_range, td = p->temp_dep;
    const bool gc = r.H.coords;
    const int nt = p->tile_threads;
    for (int ph = 0; ph < 2; ++ph) {
        if (phase >= 0 && ph != phase) continue;
        // the outlier class (few tiles) runs on a side stream, overlapping the main launch
        // (disjoint outputs: per-slot partials, tile-private nodes); joined before what follows
        bool two = false;
        // (a fused border + interior launch, phase -1, goes with pass 0)
        auto pass_of = [](const Rank::TileLaunch& tl) { return tl.phase < 0 ? 0 : tl.phase; };
        for (const Rank::TileLaunch& tl : r.launches) two = two || (pass_of(tl) == ph && tl.heavy);
        if (two) {
            CF_CUDA_CHECK(cudaEventRecord(p->fork, p->stream));
            CF_CUDA_CHECK(cudaStreamWaitEvent(p->side, p->fork, 0));
        }
        for (size_t k = r.launches.size(); k-- > 0;) {  // outlier class first: its CTAs dispatch first
            const Rank::TileLaunch& tl = r.launches[k];
            if (pass_of(tl) != ph) continue;
            cudaStream_t st = tl.heavy ? p->side : p->stream;
            TileArgs a = tl.a;
            a.T = r.T[p->cur];
            a.Told = r.T[p->old()];
            a.Tn = r.T[p->nxt()];
            a.Tslot = r.Tslot[p->step_parity];
            a.Tslot_n = r.Tslot[p->step_parity ^ 1];
            a.slot_gather = p->slot_gather ? 1 : 0;
            a.l2_next = p->l2_next ? 1 : 0;
            a.t_end = t_end;
            if (a.n_border > 0) {
                r.border_seq += 1;
                a.border_seq = r.border_seq;
                a.border_target = (unsigned long long)r.border_seq * (unsigned long long)a.n_border;
            }
            const dim3 grid(tl.grid), block(nt);
#define CF_LAUNCH(D, T, R, C, NT, G)                                                                  \
    if (det == D && td == T && dir == R && cl == C && nt == NT && gc == G) {                          \
        launch_ex(tile_kernel<D, T, R, C, NT, G>, grid, block, tl.smem, st, p->pdl && !two, a);        \
        continue;                                                                                     \
    }
            CF_TILE_VARIANTS(CF_LAUNCH)
#undef CF_LAUNCH
        }
        if (two) {
            CF_CUDA_CHECK(cudaEventRecord(p->join, p->side));
            CF_CUDA_CHECK(cudaStreamWaitEvent(p->stream, p->join, 0));
        }
    }
}

void reduce_clamp(cf_plan* p, cudaStream_t st);

template <bool DET, bool MULTI>
void launch_update_t(cf_plan* p, Rank& r, const UpdArgs& a, int blocks) {
    // 128-thread CTAs (measured: update 0.0448 -> 0.0434 ms at cfg2 vs 256; CF_UPD_BLOCK overrides)
    static const int ub = std::getenv("CF_UPD_BLOCK") ? std::atoi(std::getenv("CF_UPD_BLOCK")) : 128;
    const dim3 grid(a.list || a.rec ? std::max(1, (a.n_list + ub - 1) / ub) : (blocks * 256 + ub - 1) / ub), block(ub);
    const bool dir = r.ua.node_dir != nullptr;
    const bool cl = p->finite_range;
    const bool td = p->temp_dep;
#define CF_UPD(D, C, T) launch_ex(update_kernel<DET, MULTI, D, C, T>, grid, block, 0, p->stream, p->pdl && !MULTI, a)
    if (dir) {
        if (cl) { if (td) CF_UPD(true, true, true); else CF_UPD(true, true, false); }
        else { if (td) CF_UPD(true, false, true); else CF_UPD(true, false, false); }
    } else {
        if (cl) { if (td) CF_UPD(false, true, true); else CF_UPD(false, true, false); }
        else { if (td) CF_UPD(false, false, true); else CF_UPD(false, false, false); }
    }
#undef CF_UPD
}

void launch_update(cf_plan* p, Rank& r, double t_end) {
    UpdArgs a = r.ua;
    a.T = r.T[p->cur];
    a.Tcur_w = r.T[p->cur];
    a.Tn = r.T[p->nxt()];
    a.Tslot_n = r.Tslot[p->step_parity ^ 1];  // null with gathered slot temperatures
    a.t_end = t_end;
    if (p->peer_comm()) a.recv = r.recv + (size_t)(p->peer.seq & 1) * (size_t)r.H.recv_len;
    int blocks;
    if (p->temp_dep) {  // no fused private updates: every node
        a.list = nullptr;
        a.n_list = r.H.n_local;
        blocks = r.upd_blocks_all;
    } else {
        a.list = r.shared_list;
        a.rec = r.shared_rec;
        a.rec2 = r.shared_rec2;
        a.n_list = r.n_shared_list;
        blocks = r.upd_blocks;
    }
    const bool det = p->mode == CF_MODE_DETERMINISTIC;
    const bool multi = p->world > 1;
    if (det && multi) launch_update_t<true, true>(p, r, a, blocks);
    else if (det) launch_update_t<true, false>(p, r, a, blocks);
    else if (multi) launch_update_t<false, true>(p, r, a, blocks);
    else launch_update_t<false, false>(p, r, a, blocks);
}

void launch_advance(cf_plan* p, Rank& r, double t_end) {
    if (p->temp_dep) launch_ex(advance_kernel<true>, dim3(1), dim3(32), 0, p->stream, p->pdl, r.st, p->dP, t_end, r.sched);
    else launch_ex(advance_kernel<false>, dim3(1), dim3(32), 0, p->stream, p->pdl, r.st, p->dP, t_end, r.sched);
}

// merge + update of every local rank, the cross-rank clamp flag, then the state advance
void launch_update_all(cf_plan* p, double t_end) {
    for (auto& r : p->ranks) launch_update(p, *r, t_end);
    reduce_clamp(p, p->stream);
    for (auto& r : p->ranks) launch_advance(p, *r, t_end);
}

void launch_pack(cf_plan* p, Rank& r, cudaStream_t st) {
    if (r.pa.n_cr + r.pa.n_t == 0) return;
    PackArgs a = r.pa;
    a.T = r.T[p->cur];
    a.u.T = r.T[p->cur];
    // few CTAs (grid-stride): it runs beside the persistent interior tiles in the SM slots they
    // leave free
    const int blocks = std::max(1, std::min<int>(16, (a.n_cr + a.n_t + 255) / 256));
    if (p->mode == CF_MODE_DETERMINISTIC) pack_kernel<true, false><<<blocks, 256, 0, st>>>(a);
    else pack_kernel<false, false><<<blocks, 256, 0, st>>>(a);
}

// ------------------------------------------------------------------ peer-memory transport
struct DriverApi {
    CUresult (*StreamWaitValue32)(CUstream, CUdeviceptr, cuuint32_t, unsigned int) = nullptr;
    CUresult (*StreamBatchMemOp)(CUstream, unsigned int, CUstreamBatchMemOpParams*, unsigned int) = nullptr;
};
DriverApi& driver() {
    static DriverApi api;
    static std::once_flag once;
    std::call_once(once, [] {
        void* fn = nullptr;
        cudaDriverEntryPointQueryResult q;
        if (cudaGetDriverEntryPoint("cuStreamWaitValue32", &fn, cudaEnableDefault, &q) == cudaSuccess &&
            q == cudaDriverEntryPointSuccess)
            api.StreamWaitValue32 = (decltype(api.StreamWaitValue32))fn;
        fn = nullptr;
        if (cudaGetDriverEntryPoint("cuStreamBatchMemOp", &fn, cudaEnableDefault, &q) == cudaSuccess &&
            q == cudaDriverEntryPointSuccess)
            api.StreamBatchMemOp = (decltype(api.StreamBatchMemOp))fn;
        cudaGetLastError();
    });
    if (!api.StreamWaitValue32) raise(CF_CUDA, "cuStreamWaitValue32 not available from this driver");
    return api;
}

// GEQ is a cyclic compare ((int32)(*flag - value) >= 0), so the sequence numbers may wrap. The
// payload stores are ordered before the flag by the sender's system-scope fence + release; where
// the device can also flush third-party remote writes behind a wait, ask for that too.
unsigned wait_geq_flags() {
    static const unsigned flush = [] {
        int dev = 0, can = 0;
        if (cudaGetDevice(&dev) != cudaSuccess ||
            cudaDeviceGetAttribute(&can, cudaDevAttrCanFlushRemoteWrites, dev) != cudaSuccess)
            can = 0;
        cudaGetLastError();
        return can ? (unsigned)CU_STREAM_WAIT_VALUE_FLUSH : 0u;
    }();
    return (unsigned)CU_STREAM_WAIT_VALUE_GEQ | flush;
}
void stream_wait_geq(cudaStream_t st, const uint32_t* flag, uint32_t value) {
    const CUresult r = driver().StreamWaitValue32((CUstream)st, (CUdeviceptr)flag, value, wait_geq_flags());
    if (r != CUDA_SUCCESS) raise(CF_CUDA, "cuStreamWaitValue32 failed (" + std::to_string((int)r) + ")");
}

// send half of the exchange: the pack kernel stores into the neighbours' windows and raises the flags
void launch_pack_peer(cf_plan* p, Rank& r, cudaStream_t st) {
    cf_plan::Peer& x = p->peer;
    PackArgs a = r.pa;
    a.T = r.T[p->cur];
    a.u.T = r.T[p->cur];
    x.seq += 1;
    a.pp.seq = x.seq;
    const size_t nk = r.H.nbrs.size();
    for (size_t k = 0; k < nk; ++k) a.pp.dst[k] = x.nb_dst[k] + (size_t)(x.seq & 1) * (size_t)x.nb_stride[k];
    const int blocks = std::max(1, std::min<int>(16, (a.n_cr + a.n_t + 255) / 256));
    if (p->mode == CF_MODE_DETERMINISTIC) pack_kernel<true, true><<<blocks, 256, 0, st>>>(a);
    else pack_kernel<false, true><<<blocks, 256, 0, st>>>(a);
    CF_CUDA_CHECK(cudaGetLastError());
}

// several flags >= value as ONE stream operation (cuStreamBatchMemOp) where the driver offers it:
// one front-end round instead of one per flag
void stream_wait_geq_all(cudaStream_t st, const std::vector<const uint32_t*>& flags, uint32_t value) {
    if (flags.empty()) return;
    DriverApi& d = driver();
    if (!d.StreamBatchMemOp || flags.size() == 1 || flags.size() > 256) {
        for (const uint32_t* f : flags) stream_wait_geq(st, f, value);
        return;
    }
    std::vector<CUstreamBatchMemOpParams> ops(flags.size());
    for (size_t k = 0; k < flags.size(); ++k) {
        std::memset(&ops[k], 0, sizeof(ops[k]));
        ops[k].waitValue.operation = CU_STREAM_MEM_OP_WAIT_VALUE_32;
        ops[k].waitValue.address = (CUdeviceptr)flags[k];
        ops[k].waitValue.value = value;
        ops[k].waitValue.flags = wait_geq_flags();
    }
    const CUresult r = d.StreamBatchMemOp((CUstream)st, (unsigned)ops.size(), ops.data(), 0);
    if (r != CUDA_SUCCESS) raise(CF_CUDA, "cuStreamBatchMemOp failed (" + std::to_string((int)r) + ")");
}

// receive half: the stream waits until every neighbour's payload of this exchange has landed
void peer_wait_payload(cf_plan* p, Rank& r, cudaStream_t st) {
    const uint32_t* xflag = (const uint32_t*)(p->peer.win + kPeerXflagOff);
    std::vector<const uint32_t*> flags;
    for (const auto& nb : r.H.nbrs) flags.push_back(xflag + nb.rank);
    stream_wait_geq_all(st, flags, p->peer.seq);
}

// all-reduce of n <= 2 scalars at `v` (device) over every rank of the job through the peer windows
template <class V>
void peer_allreduce(cf_plan* p, V* v, int n, int op0, int op1, cudaStream_t st) {
    cf_plan::Peer& x = p->peer;
    x.rseq += 1;
    PeerRed pr{p->world, p->first_rank, x.rseq, x.d_win};
    peer_put_kernel<V><<<1, kPeerMaxWorld, 0, st>>>(pr, v, n);
    CF_CUDA_CHECK(cudaGetLastError());
    const uint32_t* rflag = (const uint32_t*)(x.win + kPeerRflagOff);
    std::vector<const uint32_t*> flags;
    for (int q = 0; q < p->world; ++q)
        if (q != p->first_rank) flags.push_back(rflag + q);
    stream_wait_geq_all(st, flags, x.rseq);
    peer_get_kernel<V><<<1, 32, 0, st>>>(pr, v, n, op0, op1);
    CF_CUDA_CHECK(cudaGetLastError());
}

// windows exported / imported once per plan; the bootstrap transport carries the IPC handles.
// Message to rank q (doubles as raw 8-byte carriers): [0..8) cudaIpcMemHandle_t of this rank's
// window, [8] its receive-buffer length, [9] offset of q's region in it (-1: not a neighbour),
// [10] length of q's region.
void peer_setup(cf_plan* p) {
    cf_plan::Peer& x = p->peer;
    Rank& r = *p->ranks[0];
    const int W = p->world, me = p->first_rank;
    if (p->local_ranks != 1) raise(CF_INVALID_ARG, "peer-memory transport needs one rank per process");
    if (W > kPeerMaxWorld) raise(CF_INVALID_ARG, "peer-memory transport: world_size > " + std::to_string(kPeerMaxWorld));
    if (r.H.nbrs.size() > (size_t)kPeerMaxNbrs)
        raise(CF_INVALID_ARG, "peer-memory transport: more than " + std::to_string(kPeerMaxNbrs) + " neighbours");
    driver();
    static_assert(sizeof(cudaIpcMemHandle_t) == 64, "IPC handle size");
    constexpr int kMsg = 11;
    cudaIpcMemHandle_t mine;
    CF_CUDA_CHECK(cudaIpcGetMemHandle(&mine, x.win));
    std::vector<double> out((size_t)W * kMsg, 0.0), in((size_t)W * kMsg, 0.0);
    std::vector<int32_t> peers;
    std::vector<const double*> sp;
    std::vector<double*> rp;
    std::vector<int64_t> len;
    for (int q = 0; q < W; ++q) {
        if (q == me) continue;
        double* m = out.data() + (size_t)q * kMsg;
        std::memcpy(m, &mine, 64);
        int64_t v[3] = {r.H.recv_len, -1, 0};
        for (size_t k = 0; k < r.H.nbrs.size(); ++k)
            if (r.H.nbrs[k].rank == q) {
                v[1] = r.H.recv_off[k];
                v[2] = r.nb_recv_len[k];
            }
        std::memcpy(m + 8, v, sizeof v);
        peers.push_back(q);
        sp.push_back(m);
        rp.push_back(in.data() + (size_t)q * kMsg);
        len.push_back(kMsg);
    }
    const cf_host_transport& t = p->comm->ht;
    x.boot = t;
    if (t.sendrecv(t.ctx, (int32_t)peers.size(), peers.data(), sp.data(), len.data(), rp.data(), len.data()) != 0)
        raise(CF_PROTOCOL, "peer-memory transport: handle exchange failed");
    x.mapped.assign((size_t)W, nullptr);
    x.mapped[(size_t)me] = x.win;
    x.open = true;
    for (int q = 0; q < W; ++q) {
        if (q == me) continue;
        cudaIpcMemHandle_t h;
        std::memcpy(&h, in.data() + (size_t)q * kMsg, 64);
        void* base = nullptr;
        CF_CUDA_CHECK(cudaIpcOpenMemHandle(&base, h, cudaIpcMemLazyEnablePeerAccess));
        x.mapped[(size_t)q] = (uint8_t*)base;
    }
    CF_CUDA_CHECK(cudaMalloc(&x.d_win, sizeof(uint8_t*) * (size_t)W));
    CF_CUDA_CHECK(cudaMemcpy(x.d_win, x.mapped.data(), sizeof(uint8_t*) * (size_t)W, cudaMemcpyHostToDevice));
    PackArgs& pk = r.pa;
    pk.pp.n_nbrs = (int32_t)r.H.nbrs.size();
    pk.pp.ticket = (unsigned*)(x.win + kPeerCtrlBytes - 64);
    for (size_t k = 0; k < r.H.nbrs.size(); ++k) {
        const int q = r.H.nbrs[k].rank;
        int64_t v[3];
        std::memcpy(v, in.data() + (size_t)q * kMsg + 8, sizeof v);
        if (v[1] < 0) raise(CF_PROTOCOL, "asymmetric neighbour lists");
        if (v[2] != r.nb_send_len[k]) raise(CF_PROTOCOL, "payload length mismatch");
        x.nb_dst.push_back((double*)(x.mapped[(size_t)q] + kPeerCtrlBytes) + v[1]);
        x.nb_stride.push_back(v[0]);
        pk.pp.send_off[k] = r.H.send_off[k];
        pk.pp.flag[k] = (uint32_t*)(x.mapped[(size_t)q] + kPeerXflagOff) + me;
    }
    pk.pp.send_off[r.H.nbrs.size()] = r.H.send_len;
}

void host_allreduce(cf_plan* p, double* v, int64_t n, int32_t op) {
    const cf_host_transport& t = p->comm->ht;
    if (t.allreduce(t.ctx, v, n, op) != 0) raise(CF_PROTOCOL, "host transport: allreduce failed");
}

void exchange(cf_plan* p, cudaStream_t st) {
    if (p->world == 1) return;
    if (p->local_ranks == p->world) {
        // in-process transport: every rank's send region for q -> q's recv region for r
        for (auto& rp : p->ranks) {
            Rank& r = *rp;
            for (size_t k = 0; k < r.H.nbrs.size(); ++k) {
                const int q = r.H.nbrs[k].rank;
                Rank& dst = *p->ranks[q - p->first_rank];
                size_t kk = 0;
                while (kk < dst.H.nbrs.size() && dst.H.nbrs[kk].rank != r.rank) ++kk;
                if (kk == dst.H.nbrs.size()) raise(CF_PROTOCOL, "asymmetric neighbour lists");
                const int64_t len = r.nb_send_len[k];
                if (len != dst.nb_recv_len[kk]) raise(CF_PROTOCOL, "payload length mismatch");
                if (len)
                    CF_CUDA_CHECK(cudaMemcpyAsync(dst.recv + dst.H.recv_off[kk], r.send + r.H.send_off[k],
                                                  len * sizeof(double), cudaMemcpyDeviceToDevice, st));
            }
        }
        return;
    }
    if (!p->comm) raise(CF_NCCL, "world_size > local ranks but no communicator");
    if (p->peer_comm()) {  // the pack kernel already stored into the neighbours' windows
        peer_wait_payload(p, *p->ranks[0], st);
        return;
    }
    if (p->host_comm()) {
        // host-staged: send payload -> pinned host -> caller's sendrecv -> pinned host -> recv buffer.
        // The previous step's H2D from h_recv is complete: it precedes this D2H on the same stream.
        Rank& r = *p->ranks[0];
        const size_t nk = r.H.nbrs.size();
        if (r.H.send_len) CF_CUDA_CHECK(cudaMemcpyAsync(p->h_send, r.send, r.H.send_len * sizeof(double),
                                                        cudaMemcpyDeviceToHost, st));
        CF_CUDA_CHECK(cudaStreamSynchronize(st));
        std::vector<int32_t> peers(nk);
        std::vector<const double*> sp(nk);
        std::vector<double*> rp(nk);
        for (size_t k = 0; k < nk; ++k) {
            peers[k] = r.H.nbrs[k].rank;
            sp[k] = p->h_send + r.H.send_off[k];
            rp[k] = p->h_recv + r.H.recv_off[k];
        }
        const cf_host_transport& t = p->comm->ht;
        if (t.sendrecv(t.ctx, (int32_t)nk, peers.data(), sp.data(), r.nb_send_len.data(), rp.data(),
                       r.nb_recv_len.data()) != 0)
            raise(CF_PROTOCOL, "host transport: sendrecv failed");
        if (r.H.recv_len) CF_CUDA_CHECK(cudaMemcpyAsync(r.recv, p->h_recv, r.H.recv_len * sizeof(double),
                                                        cudaMemcpyHostToDevice, st));
        return;
    }
    NcclApi& n = nccl();
    Rank& r = *p->ranks[0];
    CF_NCCL_CHECK(n.GroupStart());
    for (size_t k = 0; k < r.H.nbrs.size(); ++k) {
        const int q = r.H.nbrs[k].rank;
        if (r.nb_send_len[k])
            CF_NCCL_CHECK(n.Send(r.send + r.H.send_off[k], r.nb_send_len[k], ncclFloat64, q, p->comm->comm, st));
        if (r.nb_recv_len[k])
            CF_NCCL_CHECK(n.Recv(r.recv + r.H.recv_off[k], r.nb_recv_len[k], ncclFloat64, q, p->comm->comm, st));
    }
    CF_NCCL_CHECK(n.GroupEnd());
}

// one blocked_step for every local rank
// dynamic dt across ranks (blocked.hpp:477-480 is a min over every element of the mesh): after all
// tiles, min of each rank's per-step bound (both parity slots; the idle slot is +inf everywhere)
__global__ void min_bound_combine_kernel(DevState* const* st, int n) {
    const int k = threadIdx.x;
    if (k >= 2) return;
    unsigned long long m = ~0ull;
    for (int r = 0; r < n; ++r) m = st[r]->min_bound[k] < m ? st[r]->min_bound[k] : m;
    for (int r = 0; r < n; ++r) st[r]->min_bound[k] = m;
}

void reduce_min_bound(cf_plan* p, cudaStream_t st) {
    if (!p->temp_dep || p->world == 1) return;
    if (p->local_ranks == p->world) {
        min_bound_combine_kernel<<<1, 32, 0, st>>>(p->d_states, (int)p->ranks.size());
        CF_CUDA_CHECK(cudaGetLastError());
        return;
    }
    unsigned long long* mb = p->ranks[0]->st->min_bound;  // positive doubles: bit order == value order
    if (p->peer_comm()) {
        peer_allreduce(p, mb, 2, kPeerMin, kPeerMin, st);
        return;
    }
    if (p->host_comm()) {
        double v[2];
        CF_CUDA_CHECK(cudaMemcpyAsync(v, mb, sizeof v, cudaMemcpyDeviceToHost, st));
        CF_CUDA_CHECK(cudaStreamSynchronize(st));
        host_allreduce(p, v, 2, CF_REDUCE_MIN);
        CF_CUDA_CHECK(cudaMemcpyAsync(mb, v, sizeof v, cudaMemcpyHostToDevice, st));
        CF_CUDA_CHECK(cudaStreamSynchronize(st));  // v is a stack array
        return;
    }
    NcclApi& n = nccl();
    if (!n.AllReduce) raise(CF_NCCL, "ncclAllReduce not available");
    CF_NCCL_CHECK(n.AllReduce(mb, mb, 2, ncclUint64, ncclMin, p->comm->comm, st));
}

// clamp accounting over the whole mesh (update_fields blocked.hpp:526-534 counts a step as clamped
// when any node clamps): OR of every rank's per-step flag before the advance kernels count it
__global__ void clamp_combine_kernel(DevState* const* st, int n) {
    int f = 0;
    for (int r = 0; r < n; ++r) f |= st[r]->clamp_flag;
    for (int r = 0; r < n; ++r) st[r]->clamp_flag = f;
}

void reduce_clamp(cf_plan* p, cudaStream_t st) {
    if (!p->finite_range || p->world == 1) return;
    if (p->local_ranks == p->world) {
        clamp_combine_kernel<<<1, 1, 0, st>>>(p->d_states, (int)p->ranks.size());
        CF_CUDA_CHECK(cudaGetLastError());
        return;
    }
    int* flag = &p->ranks[0]->st->clamp_flag;
    if (p->peer_comm()) {
        peer_allreduce(p, flag, 1, kPeerMax, kPeerMax, st);
        return;
    }
    if (p->host_comm()) {
        int f = 0;
        CF_CUDA_CHECK(cudaMemcpyAsync(&f, flag, sizeof f, cudaMemcpyDeviceToHost, st));
        CF_CUDA_CHECK(cudaStreamSynchronize(st));
        double v = f;
        host_allreduce(p, &v, 1, CF_REDUCE_MAX);
        f = v > 0 ? 1 : 0;
        CF_CUDA_CHECK(cudaMemcpyAsync(flag, &f, sizeof f, cudaMemcpyHostToDevice, st));
        CF_CUDA_CHECK(cudaStreamSynchronize(st));
        return;
    }
    NcclApi& n = nccl();
    CF_NCCL_CHECK(n.AllReduce(flag, flag, 1, ncclInt32, ncclMax, p->comm->comm, st));
}

// multi-rank (SURVEY 8(e) overlap): border tiles -> [side stream: pack -> exchange] while the
// interior tiles run on the main stream -> join -> update
void enqueue_step(cf_plan* p, double t_end) {
    bool fused = p->world > 1;
    for (auto& r : p->ranks) fused = fused && r->fused_border;
    if (p->world == 1) {
        for (auto& r : p->ranks) launch_tile(p, *r, t_end);
    } else if (fused) {
        // one tile launch per rank, border tiles first; the exchange stream waits for the flag the
        // kernel raises when its last border tile has flushed, then packs and exchanges while the
        // same kernel goes on with the interior tiles
        for (auto& r : p->ranks) launch_tile(p, *r, t_end);
        for (auto& r : p->ranks) {  // each rank's pack as soon as its own border tiles are done
            if (r->border_flag) stream_wait_geq(p->xside, r->border_flag, r->border_seq);
            if (p->peer_comm()) launch_pack_peer(p, *r, p->xside);
            else launch_pack(p, *r, p->xside);
        }
        exchange(p, p->xside);
        CF_CUDA_CHECK(cudaEventRecord(p->xjoin, p->xside));
        reduce_min_bound(p, p->stream);
        CF_CUDA_CHECK(cudaStreamWaitEvent(p->stream, p->xjoin, 0));
    } else {
        for (auto& r : p->ranks) launch_tile(p, *r, t_end, 0);
        CF_CUDA_CHECK(cudaEventRecord(p->xfork, p->stream));
        CF_CUDA_CHECK(cudaStreamWaitEvent(p->xside, p->xfork, 0));
        if (p->peer_comm()) launch_pack_peer(p, *p->ranks[0], p->xside);
        else
            for (auto& r : p->ranks) launch_pack(p, *r, p->xside);
        if (p->host_comm()) {  // the host blocks in the exchange: enqueue the interior tiles first
            for (auto& r : p->ranks) launch_tile(p, *r, t_end, 1);
            exchange(p, p->xside);
            CF_CUDA_CHECK(cudaEventRecord(p->xjoin, p->xside));
        } else {
            exchange(p, p->xside);
            CF_CUDA_CHECK(cudaEventRecord(p->xjoin, p->xside));
            for (auto& r : p->ranks) launch_tile(p, *r, t_end, 1);
        }
        reduce_min_bound(p, p->stream);
        CF_CUDA_CHECK(cudaStreamWaitEvent(p->stream, p->xjoin, 0));
    }
    launch_update_all(p, t_end);
    p->advance();
}

// the device-resident arrays of one rank's plan (uploaded host plan or device-built plan)
struct RankDev {
    uint8_t* blob = nullptr;
    int32_t* slot_node = nullptr;
    const uint8_t* node_region = nullptr;
    const int8_t* node_dir = nullptr;
    const int32_t* local_global = nullptr;
    int32_t* merge_off = nullptr;
    int32_t* merge_idx = nullptr;
    int32_t* shared_list = nullptr;
    int4* shared_rec = nullptr;
    int2* shared_rec2 = nullptr;
    int64_t n_shared_list = 0, merge_parts = 0, S_tot = 0, E_r = 0;
    int32_t *node_shared = nullptr, *shared_off = nullptr, *shared_src = nullptr, *shared_src_r = nullptr,
            *ghost_src = nullptr;
};
void finish_rank(cf_plan* p, Rank& r, const RankDev& d);

void upload_rank(cf_plan* p, Rank& r, const SetupData& S) {
    (void)S;
    RankPlan& h = r.H;
    DeviceMem& M = r.mem;
    cudaStream_t s = p->stream;
    RankDev d;
    d.S_tot = h.tile_slot_off.empty() ? 0 : h.tile_slot_off.back();
    d.E_r = (int64_t)h.elem_global.size();
    d.slot_node = M.up(h.slot_node, s);
    {
        // device-side packing: the host staged only the non-geometry sections; the geometry
        // is computed here from the oriented tets and node coordinates (bitwise the host's)
        uint8_t* blob = M.alloc<uint8_t>((size_t)std::max<int64_t>(16, h.blob_bytes));
        DeviceMem tmp;
        FillArgs f{};
        f.meta = tmp.up(h.tile_meta, s);
        f.blob_off = tmp.up(h.blob_off, s);
        f.rest_off = tmp.up(h.rest_off, s);
        f.rest = tmp.up(h.blob, s);
        f.elem_off = tmp.up(h.elem_off, s);
        f.tets_ord = tmp.up(h.tets_ord, s);
        f.coords = tmp.up(h.coords_local, s);
        f.slot_off = tmp.up(h.tile_slot_off, s);
        f.slot_node = d.slot_node;
        f.blob = blob;
        f.tdep = p->temp_dep;
        f.coords_layout = h.coords;
        if (h.n_tiles) fill_tiles_kernel<<<h.n_tiles, 128, 0, s>>>(f);
        CF_CUDA_CHECK(cudaGetLastError());
        CF_CUDA_CHECK(cudaStreamSynchronize(s));
        tmp.release();
        d.blob = blob;
        decltype(h.tets_ord)().swap(h.tets_ord);
        decltype(h.coords_local)().swap(h.coords_local);
    }
    d.node_region = M.up(h.node_region, s);
    d.node_dir = h.node_dir.empty() ? nullptr : M.up(h.node_dir, s);
    d.local_global = M.up(h.local_global, s);
    d.merge_off = M.up(h.merge_off, s);
    d.merge_idx = M.up(h.merge_idx, s);
    d.shared_list = M.up(h.shared_list, s);
    d.n_shared_list = (int64_t)h.shared_list.size();
    {
        std::vector<int4> rec(2 * std::max<size_t>(1, h.shared_list.size()));
        std::vector<int2> rec2(std::max<size_t>(1, h.shared_list.size()));
        for (size_t k = 0; k < h.shared_list.size(); ++k) {
            const int32_t i = h.shared_list[k];
            const int32_t b = h.merge_off[i], cnt = h.merge_off[i + 1] - b;
            int32_t sl[8] = {0, 0, 0, 0, 0, 0, 0, 0};
            for (int q = 0; q < 8 && q < cnt; ++q) sl[q] = h.merge_idx[b + q];
            rec[2 * k] = make_int4(i, cnt, sl[0], sl[1]);
            rec[2 * k + 1] = make_int4(sl[2], sl[3], sl[4], sl[5]);
            rec2[k] = make_int2(sl[6], sl[7]);
            d.merge_parts += cnt;
        }
        d.shared_rec = M.up(rec, s);
        d.shared_rec2 = M.up(rec2, s);
    }
    if (p->world > 1) {
        d.node_shared = M.up(h.node_shared, s);
        d.shared_off = M.up(h.shared_off, s);
        d.shared_src = M.up(h.shared_src, s);
        d.shared_src_r = M.up(h.shared_src_r, s);
        d.ghost_src = M.up(h.ghost_src, s);
    }
    CF_CUDA_CHECK(cudaStreamSynchronize(s));
    finish_rank(p, r, d);
    // drop the big host arrays (metadata kept)
    decltype(h.blob)().swap(h.blob);
    std::vector<int32_t>().swap(h.merge_idx);
    std::vector<int32_t>().swap(h.slot_node);
    std::vector<int32_t>().swap(h.elem_global);
}

// a device-built plan (cf_devplan.cu): its allocations move into the rank
void adopt_rank(cf_plan* p, Rank& r, DevRankPlan& dp) {
    r.H = std::move(dp.H);
    RankDev d;
    d.blob = dp.blob;
    d.slot_node = dp.slot_node;
    d.node_region = dp.node_region;
    d.node_dir = dp.node_dir;
    d.local_global = dp.local_global;
    d.merge_off = dp.merge_off;
    d.merge_idx = dp.merge_idx;
    d.shared_list = dp.shared_list;
    d.shared_rec = dp.shared_rec;
    d.shared_rec2 = dp.shared_rec2;
    d.n_shared_list = dp.n_shared_list;
    d.merge_parts = dp.merge_parts;
    d.S_tot = dp.S_tot;
    d.E_r = dp.E_r;
    d.node_shared = dp.node_shared;
    d.shared_off = dp.shared_off;
    d.shared_src = dp.shared_src;
    d.shared_src_r = dp.shared_src_r;
    d.ghost_src = dp.ghost_src;
    r.mem.adopt(dp.mem);
    finish_rank(p, r, d);
}

void finish_rank(cf_plan* p, Rank& r, const RankDev& d) {
    RankPlan& h = r.H;
    DeviceMem& M = r.mem;
    cudaStream_t s = p->stream;
    const int64_t S_tot = d.S_tot;
    const int64_t Er = d.E_r;
    r.S_tot = S_tot;
    r.E_r = Er;
    const bool det = p->mode == CF_MODE_DETERMINISTIC;

    r.T[0] = M.alloc<double>((size_t)h.n_local + h.n_ghost);
    r.T[1] = M.alloc<double>((size_t)h.n_local + h.n_ghost);
    r.T[2] = M.alloc<double>((size_t)h.n_local + h.n_ghost);
    if (!p->slot_gather) {  // per-slot T copies (default); CF_SLOT_GATHER=1: tiles gather T by node id
        r.Tslot[0] = M.alloc<double>(S_tot + 2);
        r.Tslot[1] = M.alloc<double>(S_tot + 2);
    }
    r.st = M.alloc<DevState>(1);
    TileArgs& a = r.ta;
    a.n_local = h.n_local;
    a.n_T = h.n_local + h.n_ghost;
    a.n_slots = S_tot;
    a.meta = M.up(h.tile_meta, s);
    a.slot_off = M.up(h.tile_slot_off, s);
    a.blob_off = M.up(h.blob_off, s);
    a.slot_node = d.slot_node;
    a.blob = d.blob;
    const uint8_t* node_region = d.node_region;
    const int8_t* node_dir = d.node_dir;
    const int32_t* local_global = d.local_global;
    a.node_region = node_region;
    a.node_dir = node_dir;
    a.local_global = local_global;
    if (det) {
        r.part = M.alloc<double2>(S_tot);
    } else {
        r.acc = M.alloc<double2>(h.n_local);
        CF_CUDA_CHECK(cudaMemsetAsync(r.acc, 0, sizeof(double2) * std::max<int64_t>(1, h.n_local), s));
    }
    a.part = r.part;
    a.acc = r.acc;
    a.P = p->dP;
    a.st = r.st;
    a.n_tiles = h.n_tiles;
    a.max_slots = h.max_slots;
    a.blob_smem = (int32_t)cf_round(h.max_blob, 16);
    a.stages = p->stages;
#ifdef CF_DIAG
    if (const char* e = std::getenv("CF_PROBE")) a.probe = std::atoi(e);
#endif
    // tile classes: "light" = tiles whose footprint is within the 97th percentile,
    // "heavy" = the rest (e.g. a given block map's interface blocks), own concurrent launch
    {
        const int S = p->stages;
        std::vector<SmemMax> need(h.n_tiles);
        std::vector<size_t> bytes(h.n_tiles);
        for (int32_t t = 0; t < h.n_tiles; ++t) {
            const TileMeta& tm = h.tile_meta[t];
            const TileLayout L(tm, p->temp_dep, h.coords);
            need[t] = SmemMax{L.bytes, cf_round(tm.ns, 2), L.scratch};
            bytes[t] = tile_smem_bytes(need[t], S, p->slot_gather);
        }
        auto occupancy = [&](size_t smem) {
            int per_sm = 0;
#define CF_OCC(NT, G)                                                                                \
    if (p->tile_threads == NT && h.coords == G)                                                      \
        CF_CUDA_CHECK(cudaOccupancyMaxActiveBlocksPerMultiprocessor(                                 \
            &per_sm, tile_kernel<true, false, false, false, NT, G>, NT, smem));
            CF_OCC(128, true) CF_OCC(256, true) CF_OCC(128, false) CF_OCC(256, false)
#undef CF_OCC
            return std::max(1, per_sm);
        };
        set_tile_attr(220 * 1024);  // per function (shared by every plan): the opt-in maximum
        size_t cut = 0;
        if (h.n_tiles) {
            std::vector<size_t> sorted = bytes;
            const size_t q = std::min<size_t>(sorted.size() - 1, (size_t)(0.97 * (double)sorted.size()));
            std::nth_element(sorted.begin(), sorted.begin() + q, sorted.end());
            cut = sorted[q];
            // one launch unless the outliers would lower the occupancy of every tile (tiles
            // formed from an element order are already split to a common budget; given block
            // maps are not)
            const size_t mx_all = *std::max_element(bytes.begin(), bytes.end());
            if (occupancy(cut) == occupancy(mx_all)) cut = mx_all;
        }
        if (const char* e = std::getenv("CF_TILE_CLASSES"))
            if (std::atoi(e) == 1) cut = SIZE_MAX;  // diagnostics: one launch for every tile
        // groups: phase (multi-rank: 0 = border tiles, whose partials feed the exchange;
        // 1 = interior tiles, computed while the exchange is in flight) x footprint class
        std::vector<int32_t> lists[4];
        SmemMax mx[4];
        for (int32_t t = 0; t < h.n_tiles; ++t) {
            const int phase = (p->world > 1 && h.tile_border[t]) ? 0 : 1;
            const int c = 2 * phase + (bytes[t] <= cut ? 0 : 1);
            lists[c].push_back(t);
            mx[c].blob = std::max(mx[c].blob, need[t].blob);
            mx[c].slots = std::max(mx[c].slots, need[t].slots);
            mx[c].scratch = std::max(mx[c].scratch, need[t].scratch);
        }
        int sms = 148;
        cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, p->device);
        const bool heavy_any = !lists[1].empty() || !lists[3].empty();
        // CF_BORDER_FUSED=1 (decomposed plans without an outlier class): ONE launch, border tiles
        // first (each part in its own processing order); the kernel raises a flag when the border
        // tiles are done and the exchange stream waits on its value. Default: two launches, border
        // then interior, joined by an event -- in the in-process proxy (R ranks on one GPU) the
        // stream's flag wait costs more than the saved border tail (cfg4 R = 8: 2.61 vs 2.44 ms per
        // step, profiles/r02an_fused_border_ab.txt); to be re-measured with one GPU per rank.
        bool fuse = false;
        if (const char* e = std::getenv("CF_BORDER_FUSED"))
            fuse = std::atoi(e) != 0 && p->world > 1 && !heavy_any && S == 1 && !lists[0].empty();
        int32_t n_border = 0;
        for (int c = 0; c < 4; ++c) {
            if (lists[c].empty()) continue;
            if (fuse && c == 2) continue;  // appended to class 0 below
            Rank::TileLaunch tl;
            tl.phase = c / 2;
            tl.heavy = c & 1;
            tl.a = a;
            // heavy-first processing order (longest processing time first, for the dynamic
            // scheduler of single-rank persistent grids: -0.5 % tile time at cfg2; results do not
            // depend on the order). CF_TILE_ORDER=heavy | morton overrides.
            bool heavy_first = !heavy_any && p->stages == 1;
            if (const char* e = std::getenv("CF_TILE_ORDER")) heavy_first = std::string(e) == "heavy";
            if (heavy_first)
                    std::stable_sort(lists[c].begin(), lists[c].end(), [&](int32_t x, int32_t y) {
                        const TileMeta &mx_ = h.tile_meta[x], &my_ = h.tile_meta[y];
                        return 4 * mx_.nf + mx_.ns > 4 * my_.nf + my_.ns;
                    });
            if (fuse && c == 0) {
                bool hf = p->stages == 1;
                if (const char* e = std::getenv("CF_TILE_ORDER")) hf = std::string(e) == "heavy";
                if (hf)
                    std::stable_sort(lists[2].begin(), lists[2].end(), [&](int32_t x, int32_t y) {
                        const TileMeta &mx_ = h.tile_meta[x], &my_ = h.tile_meta[y];
                        return 4 * mx_.nf + mx_.ns > 4 * my_.nf + my_.ns;
                    });
                n_border = (int32_t)lists[0].size();
                lists[0].insert(lists[0].end(), lists[2].begin(), lists[2].end());
                mx[0].blob = std::max(mx[0].blob, mx[2].blob);
                mx[0].slots = std::max(mx[0].slots, mx[2].slots);
                mx[0].scratch = std::max(mx[0].scratch, mx[2].scratch);
                tl.phase = -1;
                r.fused_border = true;
                r.border_cnt = M.alloc<unsigned long long>(1);
                r.border_flag = M.alloc<uint32_t>(1);
                CF_CUDA_CHECK(cudaMemsetAsync(r.border_cnt, 0, sizeof(unsigned long long), s));
                CF_CUDA_CHECK(cudaMemsetAsync(r.border_flag, 0, sizeof(uint32_t), s));
                tl.a.n_border = n_border;
                tl.a.border_cnt = r.border_cnt;
                tl.a.border_flag = r.border_flag;
            }
            std::vector<TileDesc> desc(lists[c].size());
            for (size_t i = 0; i < lists[c].size(); ++i) {
                const int32_t t = lists[c][i];
                desc[i] = TileDesc{h.tile_meta[t], h.tile_slot_off[t],
                                   TileLayout(h.tile_meta[t], p->temp_dep, h.coords).bytes, h.blob_off[t]};
            }
            tl.a.desc = M.up(desc, s);
            tl.a.n_tiles = (int32_t)lists[c].size();
            tl.a.max_slots = (int32_t)mx[c].slots;
            tl.a.blob_smem = (int32_t)cf_round(mx[c].blob, 16);
            tl.a.scratch_off = (int32_t)tile_scratch_off(mx[c], S, p->slot_gather);
            tl.smem = tile_smem_bytes(mx[c], S, p->slot_gather);
            if (tl.smem > 220 * 1024)
                raise(CF_INVALID_ARG, "tile shared-memory footprint exceeds 220 KB; use smaller tiles");
            const int per_sm = occupancy(tl.smem);
            // persistent CTAs (one per resident slot, each walking tiles it, it + grid, ...): the
            // CTA prologue is paid once and the next tile's copy is issued right after the previous
            // tile's reduction (cfg2: -2.9 % tile time). Not with a concurrent outlier-class launch,
            // whose CTAs could only become resident after the persistent grid drained. On
            // decomposed meshes the grid leaves CTA slots for the exchange kernels (below).
            bool persist = S == 2 || !heavy_any;
            if (const char* e = std::getenv("CF_TILE_PERSIST")) persist = S == 2 || std::atoi(e) != 0;
            // decomposed plans leave a few CTA slots free so the exchange's pack and NCCL kernels
            // (side stream) run beside the persistent interior tiles instead of after them
            const int reserve = p->world > 1 ? 8 : 0;
            tl.grid = persist ? std::max(1, std::min<int>(tl.a.n_tiles, sms * per_sm - reserve)) : tl.a.n_tiles;
            // persistent single-stage grids schedule tiles dynamically (ticket counter reset by
            // the advance kernel of every step); CF_TILE_DYNAMIC=0: static round-robin
            tl.a.sched = nullptr;
            const char* dyn_env = std::getenv("CF_TILE_DYNAMIC");
            if (persist && S == 1 && tl.grid < tl.a.n_tiles && !(dyn_env && std::atoi(dyn_env) == 0)) {
                if (!r.sched) {  // one counter per launch class (border / interior x light / heavy)
                    r.sched = M.alloc<int32_t>(4);
                    CF_CUDA_CHECK(cudaMemsetAsync(r.sched, 0, 4 * sizeof(int32_t), s));
                }
                tl.a.sched = r.sched + c;
            }
            // one tile per CTA: CTA it stages tile it + (resident CTAs) into L2 (CF_TILE_PREFETCH=k: k x that)
            tl.a.prefetch = 0;  // measured: no gain (the wait is occupancy, not DRAM latency)
            if (const char* e = std::getenv("CF_TILE_PREFETCH"))
                if (!persist) tl.a.prefetch = (int)(std::atof(e) * sms * per_sm);
            r.launches.push_back(tl);
            if (std::getenv("CF_TRACE_SETUP") && std::atoi(std::getenv("CF_TRACE_SETUP")))
                std::fprintf(stderr, "[cf setup] rank %d class %d: %zu tiles, blob max %lld, slots max %lld, "
                             "scratch max %lld, smem/CTA %zu B, %d CTAs/SM\n", h.rank, c, lists[c].size(),
                             (long long)mx[c].blob, (long long)mx[c].slots, (long long)mx[c].scratch, tl.smem, per_sm);
        }
        r.tile_smem = r.launches.empty() ? 0 : r.launches[0].smem;
    }

    UpdArgs& u = r.ua;
#ifdef CF_DIAG
    if (const char* e = std::getenv("CF_PROBE")) u.probe = std::atoi(e);
#endif
    u.n_local = h.n_local;
    u.n_ghost = h.n_ghost;
    u.n_slots = S_tot;
    u.merge_off = d.merge_off;  // partial merge (deterministic) + Tslot scatter (both modes)
    u.merge_idx = d.merge_idx;
    u.part = r.part;
    u.acc = r.acc;
    u.node_dir = node_dir;
    u.node_region = node_region;
    u.local_global = local_global;
    u.P = p->dP;
    u.st = r.st;
    r.shared_list = d.shared_list;
    r.n_shared_list = (int32_t)d.n_shared_list;
    r.shared_rec = d.shared_rec;
    r.shared_rec2 = d.shared_rec2;
    if (p->world > 1) {
        u.node_shared = d.node_shared;
        u.shared_off = d.shared_off;
        u.shared_src_c = d.shared_src;
        u.shared_src_r = d.shared_src_r;
        if (p->peer_comm()) {  // receive buffer (two step parities) inside the exported window
            const size_t bytes = (size_t)kPeerCtrlBytes + 2 * sizeof(double) * (size_t)std::max<int64_t>(1, h.recv_len);
            p->peer.win = M.alloc<uint8_t>(bytes);
            CF_CUDA_CHECK(cudaMemsetAsync(p->peer.win, 0, bytes, s));
            r.recv = (double*)(p->peer.win + kPeerCtrlBytes);
        } else {
            r.recv = M.alloc<double>(h.recv_len);
        }
        r.send = M.alloc<double>(h.send_len);
        u.recv = r.recv;
        u.n_recv = h.recv_len;
        u.ghost_src = d.ghost_src;
        std::vector<int32_t> cr_node, t_node;
        std::vector<int64_t> cr_dst, cr_dst_r, t_dst;
        for (size_t k = 0; k < h.nbrs.size(); ++k) {
            const auto& x = h.nbrs[k];
            const int64_t base = h.send_off[k];
            const int64_t ns = (int64_t)x.shared.size();
            for (int64_t j = 0; j < ns; ++j) {
                cr_node.push_back(x.shared[j]);
                cr_dst.push_back(base + j);
                cr_dst_r.push_back(base + ns + j);
            }
            for (size_t j = 0; j < x.ext_to.size(); ++j) {
                t_node.push_back(x.ext_to[j]);
                t_dst.push_back(base + 2 * ns + (int64_t)j);
            }
            r.nb_send_len.push_back(2 * ns + (int64_t)x.ext_to.size());
            r.nb_recv_len.push_back(2 * ns + (int64_t)x.ext_from.size());
        }
        PackArgs& pk = r.pa;
        pk.n_cr = (int32_t)cr_node.size();
        pk.n_t = (int32_t)t_node.size();
        pk.cr_node = M.up(cr_node, s);
        pk.cr_dst = M.up(cr_dst, s);
        pk.cr_dst_r = M.up(cr_dst_r, s);
        pk.t_node = M.up(t_node, s);
        pk.t_dst = M.up(t_dst, s);
        pk.send = r.send;
        pk.u = u;
    }
    int sms = 148;
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, p->device);
    r.upd_blocks = std::max(1, (int)((r.n_shared_list + 255) / 256));  // one record per thread
    r.upd_blocks_all = std::max(1, std::min<int>(sms * 8, (int)((h.n_local + 255) / 256)));
    // canonical algorithmic bytes: 105 E + 48 N + 24 F_bc + 56 F_if
    r.bytes_per_step = 105 * Er + 48 * (int64_t)h.n_local + 24 * h.n_bc_facets + 56 * h.n_if_facets;
    r.tile_bytes = (h.blob_off.empty() ? 0 : h.blob_off.back()) + (8 + 16) * S_tot;
    {
        // update kernel: per merged node its 32 B record (or CSR offsets), T read + Tn write, per
        // partial a 16 B read (deterministic; atomic: the node's two accumulators read + zeroed)
        // and the 8 B slot-copy write
        const bool all = p->temp_dep;
        const int64_t nodes = all ? h.n_local : d.n_shared_list;
        const int64_t parts = all ? S_tot : d.merge_parts;
        r.update_bytes = nodes * (32 + 16) + parts * 8 + (det ? parts * 16 : nodes * 32);
    }
    CF_CUDA_CHECK(cudaStreamSynchronize(s));
}

void scatter_state(cf_plan* p);

void init_state(cf_plan* p, const double* T_global_host) {
    // one H2D of the global field, then on-device scatter into every rank's T ring and slot copies
    if (!p->dTg) CF_CUDA_CHECK(cudaMalloc(&p->dTg, std::max<int64_t>(1, p->N_global) * sizeof(double)));
    CF_CUDA_CHECK(cudaMemcpyAsync(p->dTg, T_global_host, (size_t)p->N_global * sizeof(double), cudaMemcpyHostToDevice,
                                  p->stream));
    scatter_state(p);
}

// (re)initialise every rank's state from the global field staged in dTg
void scatter_state(cf_plan* p) {
    for (auto& rp : p->ranks) {
        Rank& r = *rp;
        const int32_t nT = r.H.n_local + r.H.n_ghost;
        const int blocks = std::max(1, std::min(1184, (nT + 255) / 256));
        scatter_init_kernel<<<blocks, 256, 0, p->stream>>>(nT, r.ta.local_global, p->dTg, r.T[0], r.T[1], r.T[2]);
        const int64_t S_tot = r.S_tot;
        const int sb = (int)std::max<int64_t>(1, std::min<int64_t>(1184, (S_tot + 255) / 256));
        if (r.Tslot[0]) slot_init_kernel<<<sb, 256, 0, p->stream>>>(S_tot, r.ta.slot_node, r.T[0], r.Tslot[0], r.Tslot[1]);
        if (r.acc) {  // atomic mode: no partial sums survive a re-initialisation
            const size_t nb = sizeof(double2) * std::max<int64_t>(1, r.H.n_local);
            CF_CUDA_CHECK(cudaMemsetAsync(r.acc, 0, nb, p->stream));
        }
        DevState st{};
        st.min_bound[0] = st.min_bound[1] = 0x7ff0000000000000ull;
        st.err_node = INT32_MAX;
        CF_CUDA_CHECK(cudaMemcpyAsync(r.st, &st, sizeof st, cudaMemcpyHostToDevice, p->stream));
    }
    CF_CUDA_CHECK(cudaGetLastError());
    CF_CUDA_CHECK(cudaStreamSynchronize(p->stream));  // st is a stack object
    p->cur = 0;
    p->step_parity = 0;
    if (p->graph) {
        cudaGraphExecDestroy(p->graph);
        p->graph = nullptr;
    }
}

DevState read_state(cf_plan* p, int k = 0) {
    DevState st;
    CF_CUDA_CHECK(cudaMemcpyAsync(&st, p->ranks[k]->st, sizeof st, cudaMemcpyDeviceToHost, p->stream));
    CF_CUDA_CHECK(cudaStreamSynchronize(p->stream));
    return st;
}

void check_device_errors(cf_plan* p) {
#ifdef CF_DIAG
    if (std::getenv("CF_PROBE")) return;  // diagnostics runs skip the physics
#endif
    for (size_t k = 0; k < p->ranks.size(); ++k) {
        const DevState st = read_state(p, (int)k);
        if (st.err_node != INT32_MAX)
            raise(CF_VALIDATION, "zero lumped capacitance at active node " + std::to_string(st.err_node));
    }
}

void run_steps(cf_plan* p, int64_t n, double t_end) {
    if (n <= 0) return;
    CF_CUDA_CHECK(cudaSetDevice(p->device));
    CF_CUDA_CHECK(cudaEventRecord(p->ev0, p->stream));
    int64_t done = 0;
    // host-staged steps synchronise, peer-memory steps wait on per-step flag values: never captured
    bool flag_waits = false;  // fused border launches: the exchange stream waits on per-step flag values
    for (auto& r : p->ranks) flag_waits = flag_waits || r->fused_border;
    if (p->graph_steps > 0 && !p->host_comm() && !p->peer_comm() && !flag_waits) {
        const int state_key = p->cur * 2 + p->step_parity;
        if (p->graph && (p->graph_t_end != t_end || p->graph_cur != state_key)) {
            cudaGraphExecDestroy(p->graph);
            p->graph = nullptr;
        }
        if (!p->graph && n >= p->graph_steps) {
            const int cur0 = p->cur, par0 = p->step_parity;
            cudaGraph_t g;
            CF_CUDA_CHECK(cudaStreamBeginCapture(p->stream, cudaStreamCaptureModeThreadLocal));
            for (int64_t s = 0; s < p->graph_steps; ++s) enqueue_step(p, t_end);
            CF_CUDA_CHECK(cudaStreamEndCapture(p->stream, &g));
            CF_CUDA_CHECK(cudaGraphInstantiate(&p->graph, g, 0));
            cudaGraphDestroy(g);
            p->cur = cur0;  // capture did not execute
            p->step_parity = par0;
            p->graph_t_end = t_end;
            p->graph_cur = cur0 * 2 + par0;
        }
        while (p->graph && n - done >= p->graph_steps) {
            CF_CUDA_CHECK(cudaGraphLaunch(p->graph, p->stream));
            for (int64_t s = 0; s < p->graph_steps; ++s) p->advance();
            done += p->graph_steps;
            if (p->graph_cur != p->cur * 2 + p->step_parity) break;  // length not a multiple of 6: recapture
        }
    }
    for (; done < n; ++done) enqueue_step(p, t_end);
    CF_CUDA_CHECK(cudaGetLastError());
    CF_CUDA_CHECK(cudaEventRecord(p->ev1, p->stream));
    CF_CUDA_CHECK(cudaEventSynchronize(p->ev1));
    float ms = 0;
    CF_CUDA_CHECK(cudaEventElapsedTime(&ms, p->ev0, p->ev1));
    p->loop_seconds += ms * 1e-3;
    check_device_errors(p);
}

// ------------------------------------------------------------------ lambda_max kernels
struct LamArgs {
    TileArgs a;
    bool tdep, coords;
    const double* cval;  // per region rho*c(T0)
    const double* kval;  // per region k(T0)
    const double* hval;  // per facet kind
    const double* x;
    double* y;
    double* M;
    double* D;
};

// element i of a tile blob (global memory): gradients and volume, stored or recomputed
__device__ void lam_geom(const LamArgs& L, const uint8_t* B, const TileLayout& Ly, int i, ushort4 cn,
                         double (&g)[4][3], double& vol) {
    if (L.coords) {
        const double* X = (const double*)(B + Ly.xyz);
        const unsigned short sl[4] = {cn.x, cn.y, cn.z, cn.w};
        double p[4][3];
        for (int k = 0; k < 4; ++k)
            for (int c = 0; c < 3; ++c) p[k][c] = X[4 * sl[k] + c];
        dev_tet_grads(p, g, vol);
        return;
    }
    const double* G = (const double*)(B + Ly.geom);  // pairs (g1x g1y) (g1z g2x) (g2y g2z) (g3x g3y) (g3z vol)
    const int S = Ly.ne2;
    const double v[10] = {G[2 * i], G[2 * i + 1], G[2 * (S + i)], G[2 * (S + i) + 1], G[2 * (2 * S + i)],
                          G[2 * (2 * S + i) + 1], G[2 * (3 * S + i)], G[2 * (3 * S + i) + 1], G[2 * (4 * S + i)],
                          G[2 * (4 * S + i) + 1]};
    for (int k = 0; k < 3; ++k) {
        g[1][k] = v[k];
        g[2][k] = v[3 + k];
        g[3][k] = v[6 + k];
        g[0][k] = ((g[1][k] + g[2][k]) + g[3][k]) * -1.0;
    }
    vol = v[9];
}

// lambda_max operator on the tile blobs (global reads, no shared memory)
__global__ void lam_setup(LamArgs L) {
    const TileArgs& a = L.a;
    const int t = blockIdx.x;
    const TileMeta tm = a.meta[t];
    const TileLayout Ly(tm, L.tdep, L.coords);
    const uint8_t* B = a.blob + a.blob_off[t];
    const int s0 = a.slot_off[t];
    for (int i = threadIdx.x; i < tm.ne; i += blockDim.x) {
        const ushort4 cn = *(const ushort4*)(B + Ly.conn_of(i));
        double g[4][3], vol;
        lam_geom(L, B, Ly, i, cn, g, vol);
        const double w = L.cval[B[Ly.region + i]] * vol * 0.25;
        const unsigned short sl[4] = {cn.x, cn.y, cn.z, cn.w};
        for (int k = 0; k < 4; ++k) atomicAdd(&L.M[a.slot_node[s0 + sl[k]] & 0x0fffffff], w);
    }
    for (int i = threadIdx.x; i < tm.nf; i += blockDim.x) {
        const ushort4 fs = *(const ushort4*)(B + Ly.fac_slots(i));
        const double w = L.hval[fs.w] * (*(const double*)(B + Ly.fac_area(i)) / 3.0);
        const unsigned short sl[3] = {fs.x, fs.y, fs.z};
        for (int k = 0; k < 3; ++k) atomicAdd(&L.D[a.slot_node[s0 + sl[k]] & 0x0fffffff], w);
    }
}

__global__ void lam_apply(LamArgs L) {
    const TileArgs& a = L.a;
    const int t = blockIdx.x;
    const TileMeta tm = a.meta[t];
    const TileLayout Ly(tm, L.tdep, L.coords);
    const uint8_t* B = a.blob + a.blob_off[t];
    const int s0 = a.slot_off[t];
    for (int i = threadIdx.x; i < tm.ne; i += blockDim.x) {
        const ushort4 cn = *(const ushort4*)(B + Ly.conn_of(i));
        const int32_t n[4] = {a.slot_node[s0 + cn.x] & 0x0fffffff, a.slot_node[s0 + cn.y] & 0x0fffffff,
                              a.slot_node[s0 + cn.z] & 0x0fffffff, a.slot_node[s0 + cn.w] & 0x0fffffff};
        double g[4][3], vol;
        lam_geom(L, B, Ly, i, cn, g, vol);
        const double kv = L.kval[B[Ly.region + i]] * vol;
        double gx = 0, gy = 0, gz = 0;
        for (int b = 0; b < 4; ++b) {
            const double xb = L.x[n[b]];
            gx += g[b][0] * xb;
            gy += g[b][1] * xb;
            gz += g[b][2] * xb;
        }
        for (int k = 0; k < 4; ++k) atomicAdd(&L.y[n[k]], kv * (g[k][0] * gx + g[k][1] * gy + g[k][2] * gz));
    }
}

__global__ void lam_init_x(int32_t n, const int32_t* gid, const int8_t* dir, uint64_t seed, double* x) {
    for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < n; i += gridDim.x * blockDim.x) {
        const uint64_t key = (uint64_t)gid[i];
        uint64_t z = seed * 0x9E3779B97F4A7C15ull + key + 0x632BE59BD9B4E019ull;
        z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ull;
        z = (z ^ (z >> 27)) * 0x94D049BB133111EBull;
        z ^= z >> 31;
        const double u = (double)(z >> 11) * (1.0 / 9007199254740992.0);
        x[i] = (dir && dir[i] >= 0) ? 0.0 : (u - 0.5);
    }
}
__global__ void lam_diag(int32_t n, const double* D, const double* x, double* y) {
    for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < n; i += gridDim.x * blockDim.x) y[i] = D[i] * x[i];
}
// num = x.y, den = x.M.x ; y <- y / M ; nrm2 = y.M.y
__global__ void lam_reduce(int32_t n, const int8_t* dir, const double* M, const double* x, double* y, double* acc) {
    double a0 = 0, a1 = 0, a2 = 0;
    for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < n; i += gridDim.x * blockDim.x) {
        double yi = y[i];
        if (dir && dir[i] >= 0) yi = 0;
        a0 += x[i] * yi;
        a1 += x[i] * M[i] * x[i];
        yi = yi / M[i];
        a2 += yi * M[i] * yi;
        y[i] = yi;
    }
    for (int o = 16; o > 0; o >>= 1) {
        a0 += __shfl_xor_sync(0xffffffffu, a0, o);
        a1 += __shfl_xor_sync(0xffffffffu, a1, o);
        a2 += __shfl_xor_sync(0xffffffffu, a2, o);
    }
    if ((threadIdx.x & 31) == 0) {
        atomicAdd(&acc[0], a0);
        atomicAdd(&acc[1], a1);
        atomicAdd(&acc[2], a2);
    }
}
__global__ void lam_scale(int32_t n, const double* y, const double* acc, double* x) {
    const double inv = 1.0 / sqrt(acc[2]);
    for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < n; i += gridDim.x * blockDim.x) x[i] = y[i] * inv;
}

__global__ void minmax_kernel(int32_t n, const double* T, double* out) {
    double lo = __longlong_as_double(0x7ff0000000000000ll), hi = -lo;
    for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < n; i += gridDim.x * blockDim.x) {
        lo = fmin(lo, T[i]);
        hi = fmax(hi, T[i]);
    }
    for (int o = 16; o > 0; o >>= 1) {
        lo = fmin(lo, __shfl_xor_sync(0xffffffffu, lo, o));
        hi = fmax(hi, __shfl_xor_sync(0xffffffffu, hi, o));
    }
    if ((threadIdx.x & 31) == 0) {
        // min/max of doubles via ordered integer atomics on a sign-aware encoding
        auto enc = [](double v) {
            long long b = __double_as_longlong(v);
            return (unsigned long long)(b < 0 ? ~b : (b | 0x8000000000000000ll));
        };
        atomicMin((unsigned long long*)&out[0], enc(lo));
        atomicMax((unsigned long long*)&out[1], enc(hi));
    }
}
double dec_ordered(unsigned long long u) {
    long long b = (u & 0x8000000000000000ull) ? (long long)(u & 0x7fffffffffffffffull) : (long long)~u;
    double d;
    std::memcpy(&d, &b, 8);
    return d;
}

}  // namespace

// ================================================================== C-ABI
extern "C" {

int cf_abi_version(void) { return CF_ABI_VERSION; }

int cf_last_error(char* buf, size_t len) {
    if (!buf || !len) return CF_INVALID_ARG;
    std::snprintf(buf, len, "%s", g_last_error.c_str());
    return CF_OK;
}

}  // extern "C"

namespace {
struct FixtureArgs {  // cf_plan_create_fixture: the mesh generated on the device
    int32_t kind, n;
    double radius, jitter;
    uint64_t seed;
    double t0_noise;
    uint64_t noise_seed;
    int32_t rcm;
};

cf_run_opts normalized_opts(const cf_run_opts* opts, int& tile) {
    cf_run_opts o{};
    o.world_size = 1;
    o.local_ranks = 1;
    o.node_order = CF_NODE_ORDER_RCM;
    o.elem_order = CF_ELEM_ORDER_MORTON;
    if (opts) o = *opts;
    if (o.world_size < 1) o.world_size = 1;
    if (o.local_ranks < 1) o.local_ranks = 1;
    if (o.rank < 0 || o.rank + o.local_ranks > o.world_size) raise(CF_INVALID_ARG, "bad rank / local_ranks");
    if (o.local_ranks != 1 && o.local_ranks != o.world_size)
        raise(CF_INVALID_ARG, "local_ranks must be 1 or world_size");
    if (o.mode != CF_MODE_ATOMIC && o.mode != CF_MODE_DETERMINISTIC) raise(CF_INVALID_ARG, "bad mode");
    if (o.geometry != CF_GEOM_COORDS && o.geometry != CF_GEOM_STORED) raise(CF_INVALID_ARG, "bad geometry mode");
    if (o.fast_math != 0) raise(CF_CONFIG, "fast_math is reserved (kernels are built without FMA contraction)");
    tile = o.tile_elems > 0 ? o.tile_elems : 384;
    if (tile > kMaxTileElems) raise(CF_INVALID_ARG, "tile_elems must be <= 2048");
    int ndev = 0;
    if (cudaGetDeviceCount(&ndev) != cudaSuccess || ndev == 0) raise(CF_CUDA, "no CUDA device available");
    if (o.device < 0 || o.device >= ndev) raise(CF_INVALID_ARG, "bad device ordinal");
    CF_CUDA_CHECK(cudaSetDevice(o.device));
    return o;
}

PlanOptions plan_options(const cf_run_opts& o, int tile) {
    PlanOptions po;
    po.mode = o.mode;
    po.node_order = o.node_order;
    po.elem_order = o.elem_order;
    po.geometry = o.geometry;
    po.tile_elems = tile;
    po.tile_of_element = o.tile_of_element;
    po.n_tiles_given = o.n_tiles_given;
    po.world_size = o.world_size;
    return po;
}

// the plan object before its ranks: streams, parameters, static dt bound
std::unique_ptr<cf_plan> new_plan(const cf_run_opts& o, const cf_setup_desc* setup, const SetupData& S, int32_t N,
                                  const std::vector<double>& region_min_edge) {
    auto p = std::make_unique<cf_plan>();
    p->device = o.device;
    p->mode = o.mode;
    if (const char* e = std::getenv("CF_TILE_THREADS")) {
        const int v = std::atoi(e);
        p->tile_threads = v == 256 ? 256 : 128;
    }
    if (const char* e = std::getenv("CF_TILE_STAGES")) p->stages = std::atoi(e) == 2 ? 2 : 1;
    if (const char* e = std::getenv("CF_PDL")) p->pdl = std::atoi(e) != 0;
    if (const char* e = std::getenv("CF_SLOT_GATHER")) p->slot_gather = std::atoi(e) != 0;
    if (const char* e = std::getenv("CF_L2_NEXT")) p->l2_next = std::atoi(e) != 0;
    if (p->stages == 2) p->slot_gather = false;
    p->world = o.world_size;
    p->first_rank = o.rank;
    p->local_ranks = o.local_ranks;
    p->comm = (cf_comm*)o.comm;
    if (p->world > p->local_ranks && !p->comm) raise(CF_NCCL, "world_size > local_ranks needs a cf_comm");
    p->P = S.P;
    p->temp_dep = S.temp_dep;
    p->finite_range = S.P.finite_range != 0;
    p->N_global = N;
    p->output_every = setup->output_every;
    p->t_end_setup = setup->t_end;
    CF_CUDA_CHECK(cudaStreamCreateWithFlags(&p->stream, cudaStreamNonBlocking));
    CF_CUDA_CHECK(cudaStreamCreateWithFlags(&p->side, cudaStreamNonBlocking));
    CF_CUDA_CHECK(cudaEventCreateWithFlags(&p->fork, cudaEventDisableTiming));
    CF_CUDA_CHECK(cudaEventCreateWithFlags(&p->join, cudaEventDisableTiming));
    CF_CUDA_CHECK(cudaStreamCreateWithFlags(&p->xside, cudaStreamNonBlocking));
    CF_CUDA_CHECK(cudaEventCreateWithFlags(&p->xfork, cudaEventDisableTiming));
    CF_CUDA_CHECK(cudaEventCreateWithFlags(&p->xjoin, cudaEventDisableTiming));
    CF_CUDA_CHECK(cudaEventCreate(&p->ev0));
    CF_CUDA_CHECK(cudaEventCreate(&p->ev1));
    CF_CUDA_CHECK(cudaMalloc(&p->dP, sizeof(DevParams)));
    CF_CUDA_CHECK(cudaMemcpy(p->dP, &p->P, sizeof(DevParams), cudaMemcpyHostToDevice));
    double e13 = INFINITY;  // monotone in the minimum edge per region (see resolve_setup)
    for (int32_t rg = 0; rg < (int32_t)region_min_edge.size(); ++rg) {
        if (!std::isfinite(region_min_edge[rg])) continue;
        const DevMaterial& mm = S.P.mat[rg];
        const double c0 = pl_eval(S.P, mm.c, 0), k0 = pl_eval(S.P, mm.k, 0), me = region_min_edge[rg];
        e13 = std::min(e13, mm.rho * c0 * me * me / k0);
    }
    p->eq13_min = e13;
    p->base_min_bound = S.min_bound;
    return p;
}

// after the ranks: multi-rank state table, optional L2 window, host buffers, launch count
void finish_plan(cf_plan* p) {
    if (p->ranks.size() > 1) {
        std::vector<DevState*> sts;
        for (const auto& rk : p->ranks) sts.push_back(rk->st);
        CF_CUDA_CHECK(cudaMalloc(&p->d_states, sizeof(DevState*) * sts.size()));
        CF_CUDA_CHECK(cudaMemcpy(p->d_states, sts.data(), sizeof(DevState*) * sts.size(), cudaMemcpyHostToDevice));
    }
    // Optional L2 residency of the per-slot partials between their writer (tile kernel) and
    // reader (update kernel), CF_L2_PERSIST=fraction. Measured on cfg2 and left off: update
    // 0.049 -> 0.058 ms with the whole 67 MB persisting, tile kernel unchanged.
    if (p->ranks.size() == 1 && p->ranks[0]->part) {
        const char* e = std::getenv("CF_L2_PERSIST");
        const double frac = e ? std::atof(e) : 0.0;
        int max_win = 0, max_pers = 0;
        cudaDeviceGetAttribute(&max_win, cudaDevAttrMaxAccessPolicyWindowSize, p->device);
        cudaDeviceGetAttribute(&max_pers, cudaDevAttrMaxPersistingL2CacheSize, p->device);
        const Rank& rk = *p->ranks[0];
        const size_t bytes = sizeof(double2) * (size_t)rk.H.tile_slot_off.back();
        if (frac > 0 && max_win > 0 && max_pers > 0 && bytes > 0) {
            const size_t pers = std::min<size_t>((size_t)(frac * (double)bytes), (size_t)max_pers);
            CF_CUDA_CHECK(cudaDeviceSetLimit(cudaLimitPersistingL2CacheSize, pers));
            cudaStreamAttrValue v = {};
            v.accessPolicyWindow.base_ptr = (void*)rk.part;
            v.accessPolicyWindow.num_bytes = std::min<size_t>(bytes, (size_t)max_win);
            v.accessPolicyWindow.hitRatio =
                (float)std::min(1.0, (double)pers / (double)v.accessPolicyWindow.num_bytes);
            v.accessPolicyWindow.hitProp = cudaAccessPropertyPersisting;
            v.accessPolicyWindow.missProp = cudaAccessPropertyStreaming;
            CF_CUDA_CHECK(cudaStreamSetAttribute(p->stream, cudaStreamAttributeAccessPolicyWindow, &v));
        }
    }
    if (p->peer_comm()) peer_setup(p);
    if (p->host_comm()) {
        const RankPlan& h = p->ranks[0]->H;
        CF_CUDA_CHECK(cudaMallocHost(&p->h_send, sizeof(double) * std::max<int64_t>(1, h.send_len)));
        CF_CUDA_CHECK(cudaMallocHost(&p->h_recv, sizeof(double) * std::max<int64_t>(1, h.recv_len)));
    }
    p->launches_per_step = 0;
    for (const auto& rk : p->ranks)
        p->launches_per_step += (int64_t)rk->launches.size() + 2 + (p->world > 1 ? 1 : 0);
}

bool use_device_setup(const cf_run_opts& o) {
    const char* e = std::getenv("CF_HOST_SETUP");
    if (e && std::atoi(e)) return false;
    return !o.tile_of_element && o.partition != CF_PARTITION_GRAPH && o.world_size <= 64;
}

// host setup pipeline (cf_mesh.cpp / cf_plan.cpp): given block maps, graph partitions, > 64
// ranks, or CF_HOST_SETUP=1
void create_host(const cf_mesh_desc* mesh, const cf_setup_desc* setup, const cf_run_opts& o, int tile, cf_plan** out) {
    trace_stage("plan_create: start");
    MeshData m;
    finalize_mesh(mesh, m);
    SetupData S;
    resolve_setup(m, setup, S);
    trace_stage("resolve: rest");
    std::vector<int32_t> label(m.N);
    if (o.node_order == CF_NODE_ORDER_RCM) {
        label = rcm_permutation_device(m.N, m.E, m.tets.data(), -1, o.device);  // the RCM pass on the B200
    } else {
        std::iota(label.begin(), label.end(), 0);
    }
    std::vector<int32_t> part;
    PlanOptions po = plan_options(o, tile);
    if (o.world_size > 1) {
        if (o.partition == CF_PARTITION_GIVEN) {
            if (!o.part_of_element) raise(CF_INVALID_ARG, "part_of_element required");
            part.assign(o.part_of_element, o.part_of_element + m.E);
            for (int32_t v : part)
                if (v < 0 || v >= o.world_size) raise(CF_VALIDATION, "part id out of range");
        } else if (o.partition == CF_PARTITION_GRAPH) {
            part = partition_elements(m, o.world_size, 0.05, true);
        } else {
            part = partition_rcb(m, o.world_size);
        }
        po.part_of_element = part.data();
    }
    trace_stage("labels + partition");
    auto p = new_plan(o, setup, S, m.N, m.region_min_edge);
    p->E_global = m.E;
    for (int r = o.rank; r < o.rank + o.local_ranks; ++r) {
        auto rk = std::make_unique<Rank>();
        rk->rank = r;
        build_rank_plan(m, S, po, label, r, rk->H);
        upload_rank(p.get(), *rk, S);
        trace_stage("upload");
        p->ranks.push_back(std::move(rk));
    }
    finish_plan(p.get());
    init_state(p.get(), S.T0.data());
    CF_CUDA_CHECK(cudaStreamSynchronize(p->stream));
    trace_stage("init state");
    *out = p.release();
}

// device setup pipeline (cf_devplan.cu): the mesh lives only in device memory
void create_device(const cf_mesh_desc* mesh, const FixtureArgs* fx, const cf_setup_desc* setup, const cf_run_opts& o,
                   int tile, cf_plan** out) {
    trace_stage("plan_create: start (device setup)");
    cudaStream_t s;
    CF_CUDA_CHECK(cudaStreamCreateWithFlags(&s, cudaStreamNonBlocking));
    struct SG {
        cudaStream_t s;
        ~SG() { cudaStreamDestroy(s); }
    } sg{s};
    DevMesh dm;
    T0Noise noise;
    if (fx) {
        devmesh_fixture(fx->kind, fx->n, fx->radius, fx->jitter, fx->seed, fx->rcm != 0, s, dm);
        noise.amp = fx->t0_noise;
        noise.seed = fx->noise_seed;
    } else {
        devmesh_from_desc(mesh, s, dm);
    }
    trace_stage("device: mesh + finalize");
    DevSetup ds;
    resolve_setup_device(dm, setup, noise, s, ds);
    trace_stage("device: resolve");
    DBuf work;
    int32_t* d_label = nullptr;
    if (o.node_order == CF_NODE_ORDER_RCM) {
        d_label = work.alloc<int32_t>(dm.N);
        rcm_labels_device(dm.N, dm.E, dm.tets, -1, s, d_label);
        trace_stage("device: rcm");
    }
    int32_t* d_part = nullptr;
    if (o.world_size > 1) {
        d_part = work.alloc<int32_t>(dm.E);
        if (o.partition == CF_PARTITION_GIVEN) {
            if (!o.part_of_element) raise(CF_INVALID_ARG, "part_of_element required");
            for (int64_t e = 0; e < dm.E; ++e)
                if (o.part_of_element[e] < 0 || o.part_of_element[e] >= o.world_size)
                    raise(CF_VALIDATION, "part id out of range");
            CF_CUDA_CHECK(cudaMemcpyAsync(d_part, o.part_of_element, sizeof(int32_t) * dm.E, cudaMemcpyHostToDevice, s));
        } else {
            partition_rcb_device(dm, o.world_size, s, d_part);
        }
        trace_stage("device: partition");
    }
    const PlanOptions po = plan_options(o, tile);
    auto p = new_plan(o, setup, ds.S, dm.N, dm.region_min_edge);
    p->E_global = dm.E;
    p->device_setup = true;
    for (int r = o.rank; r < o.rank + o.local_ranks; ++r) {
        auto rk = std::make_unique<Rank>();
        rk->rank = r;
        DevRankPlan dp;
        build_rank_plan_device(dm, ds, po, d_label, d_part, r, s, dp);
        trace_stage("device: rank plan");
        adopt_rank(p.get(), *rk, dp);
        p->ranks.push_back(std::move(rk));
    }
    finish_plan(p.get());
    if (!p->dTg) CF_CUDA_CHECK(cudaMalloc(&p->dTg, std::max<int64_t>(1, p->N_global) * sizeof(double)));
    CF_CUDA_CHECK(cudaMemcpyAsync(p->dTg, ds.T0, (size_t)p->N_global * sizeof(double), cudaMemcpyDeviceToDevice, s));
    CF_CUDA_CHECK(cudaStreamSynchronize(s));
    scatter_state(p.get());
    CF_CUDA_CHECK(cudaStreamSynchronize(p->stream));
    trace_stage("init state");
    *out = p.release();
}
}  // namespace

extern "C" {
int cf_plan_create(const cf_mesh_desc* mesh, const cf_setup_desc* setup, const cf_run_opts* opts, cf_plan** out) {
    return guarded([&] {
        if (!mesh || !setup || !out) raise(CF_INVALID_ARG, "null argument");
        *out = nullptr;
        int tile = 384;
        const cf_run_opts o = normalized_opts(opts, tile);
        if (use_device_setup(o)) create_device(mesh, nullptr, setup, o, tile, out);
        else create_host(mesh, setup, o, tile, out);
    });
}

int cf_plan_create_fixture(const cf_fixture_spec* fx, const cf_setup_desc* setup, const cf_run_opts* opts,
                           cf_plan** out) {
    return guarded([&] {
        if (!fx || !setup || !out) raise(CF_INVALID_ARG, "null argument");
        if (fx->perm_seed != 0) raise(CF_INVALID_ARG, "device fixtures keep the generator numbering (perm_seed 0)");
        *out = nullptr;
        int tile = 384;
        const cf_run_opts o = normalized_opts(opts, tile);
        if (o.tile_of_element || o.partition == CF_PARTITION_GRAPH || o.world_size > 64)
            raise(CF_INVALID_ARG, "device fixtures need RCB or given partitions and no given tile map");
        const FixtureArgs a{fx->kind, fx->n, fx->radius, fx->jitter, fx->seed, fx->t0_noise, fx->noise_seed, fx->rcm};
        create_device(nullptr, &a, setup, o, tile, out);
    });
}

int cf_plan_destroy(cf_plan* plan) {
    return guarded([&] {
        if (!plan) return;
        cudaSetDevice(plan->device);
        cudaStreamSynchronize(plan->stream);
        delete plan;
    });
}

int cf_set_temperature(cf_plan* p, const double* T_host) {
    return guarded([&] {
        if (!p || !T_host) raise(CF_INVALID_ARG, "null argument");
        CF_CUDA_CHECK(cudaSetDevice(p->device));
        init_state(p, T_host);
        p->loop_seconds = 0;
    });
}

int cf_step(cf_plan* p, int64_t n_steps, double t_end) {
    return guarded([&] {
        if (!p) raise(CF_INVALID_ARG, "null plan");
        run_steps(p, n_steps, t_end);
    });
}

int cf_time_phases(cf_plan* p, int64_t n, double* ms_out) {
    return guarded([&] {
        if (!p || !ms_out) raise(CF_INVALID_ARG, "null argument");
        CF_CUDA_CHECK(cudaSetDevice(p->device));
        cudaEvent_t ev[5];
        for (auto& e : ev) CF_CUDA_CHECK(cudaEventCreate(&e));
        double acc[4] = {0, 0, 0, 0};
        for (int64_t s = 0; s < n; ++s) {
            CF_CUDA_CHECK(cudaEventRecord(ev[0], p->stream));
            for (auto& r : p->ranks) launch_tile(p, *r, 0.0);
            CF_CUDA_CHECK(cudaEventRecord(ev[1], p->stream));
            if (p->peer_comm()) launch_pack_peer(p, *p->ranks[0], p->stream);
            else if (p->world > 1)
                for (auto& r : p->ranks) launch_pack(p, *r, p->stream);
            CF_CUDA_CHECK(cudaEventRecord(ev[2], p->stream));
            exchange(p, p->stream);
            reduce_min_bound(p, p->stream);
            CF_CUDA_CHECK(cudaEventRecord(ev[3], p->stream));
            launch_update_all(p, 0.0);
            CF_CUDA_CHECK(cudaEventRecord(ev[4], p->stream));
            p->advance();
            CF_CUDA_CHECK(cudaEventSynchronize(ev[4]));
            for (int k = 0; k < 4; ++k) {
                float ms = 0;
                CF_CUDA_CHECK(cudaEventElapsedTime(&ms, ev[k], ev[k + 1]));
                acc[k] += ms;
            }
            float tot = 0;
            CF_CUDA_CHECK(cudaEventElapsedTime(&tot, ev[0], ev[4]));
            p->loop_seconds += tot * 1e-3;
        }
        CF_CUDA_CHECK(cudaGetLastError());
        for (auto& e : ev) cudaEventDestroy(e);
        for (int k = 0; k < 4; ++k) ms_out[k] = n > 0 ? acc[k] / (double)n : 0.0;
        check_device_errors(p);
    });
}

int cf_set_dt_safety(cf_plan* p, double s) {
    return guarded([&] {
        if (!p) raise(CF_INVALID_ARG, "null plan");
        if (!(s > 0 && s <= 1)) raise(CF_CONFIG, "safety must be in (0, 1]");
        CF_CUDA_CHECK(cudaSetDevice(p->device));
        p->P.dt_safety = s;
        if (!p->temp_dep) p->P.static_dt = p->base_min_bound * s;
        CF_CUDA_CHECK(cudaMemcpyAsync(p->dP, &p->P, sizeof(DevParams), cudaMemcpyHostToDevice, p->stream));
        CF_CUDA_CHECK(cudaStreamSynchronize(p->stream));
    });
}

int cf_enable_graph(cf_plan* p, int64_t steps) {
    return guarded([&] {
        if (!p) raise(CF_INVALID_ARG, "null plan");
        if (p->graph) {
            cudaGraphExecDestroy(p->graph);
            p->graph = nullptr;
        }
        p->graph_steps = std::max<int64_t>(0, steps);
    });
}

int cf_solve(cf_plan* p, int64_t max_steps, double* series, int64_t cap, int64_t* n_series) {
    return guarded([&] {
        if (!p) raise(CF_INVALID_ARG, "null plan");
        CF_CUDA_CHECK(cudaSetDevice(p->device));
        int64_t ns = 0;
        const int64_t every = p->output_every;
        double* mm = nullptr;
        if (every > 0) CF_CUDA_CHECK(cudaMalloc(&mm, 2 * sizeof(double)));
        auto sample = [&]() {
            unsigned long long init[2] = {~0ull, 0ull};
            CF_CUDA_CHECK(cudaMemcpyAsync(mm, init, sizeof init, cudaMemcpyHostToDevice, p->stream));
            for (auto& r : p->ranks)
                minmax_kernel<<<148, 256, 0, p->stream>>>(r->H.n_local, r->T[p->cur], mm);
            // the series covers the whole mesh (solve_serial blocked.hpp:678-681): min / max over
            // every rank of the job
            if (p->peer_comm()) {
                peer_allreduce(p, (unsigned long long*)mm, 2, kPeerMin, kPeerMax, p->stream);
            } else if (p->world > p->local_ranks && !p->host_comm()) {
                NcclApi& n = nccl();
                CF_NCCL_CHECK(n.AllReduce(mm, mm, 1, ncclUint64, ncclMin, p->comm->comm, p->stream));
                CF_NCCL_CHECK(n.AllReduce((unsigned long long*)mm + 1, (unsigned long long*)mm + 1, 1, ncclUint64,
                                          ncclMax, p->comm->comm, p->stream));
            }
            unsigned long long res[2];
            CF_CUDA_CHECK(cudaMemcpyAsync(res, mm, sizeof res, cudaMemcpyDeviceToHost, p->stream));
            const DevState st = read_state(p);
            double lo = dec_ordered(res[0]), hi = dec_ordered(res[1]);
            if (p->host_comm()) {
                host_allreduce(p, &lo, 1, CF_REDUCE_MIN);
                host_allreduce(p, &hi, 1, CF_REDUCE_MAX);
            }
            if (series && ns < cap) {
                series[3 * ns] = st.time;
                series[3 * ns + 1] = lo;
                series[3 * ns + 2] = hi;
            }
            ++ns;
        };
        if (max_steps > 0) {
            DevState st = read_state(p);
            int64_t left = max_steps - st.step_index;
            while (left > 0) {
                int64_t chunk = left;
                if (every > 0) chunk = std::min<int64_t>(left, every - (int64_t)(st.step_index % every));
                run_steps(p, chunk, 0.0);
                left -= chunk;
                st.step_index += chunk;
                if (every > 0 && st.step_index % every == 0) sample();
            }
        } else {
            const double t_end = p->t_end_setup;
            for (;;) {
                DevState st = read_state(p);
                if (!(st.time < t_end)) break;
                const int64_t chunk = every > 0 ? every - (int64_t)(st.step_index % every) : 256;
                run_steps(p, chunk, t_end);
                const DevState s2 = read_state(p);
                if (every > 0 && s2.step_index % every == 0 && s2.step_index != st.step_index) sample();
            }
        }
        if (mm) cudaFree(mm);
        if (n_series) *n_series = ns;
    });
}

int cf_get_fields(cf_plan* p, double* T_host, double* H_host) {
    return guarded([&] {
        if (!p) raise(CF_INVALID_ARG, "null plan");
        CF_CUDA_CHECK(cudaSetDevice(p->device));
        const size_t bytes = std::max<int64_t>(1, p->N_global) * sizeof(double);
        if (!p->dTg) CF_CUDA_CHECK(cudaMalloc(&p->dTg, bytes));
        if (H_host && !p->dHg) CF_CUDA_CHECK(cudaMalloc(&p->dHg, bytes));
        if (p->ranks.size() > 1 || p->world > 1) {  // nodes owned by other processes keep the host value
            if (T_host) CF_CUDA_CHECK(cudaMemcpyAsync(p->dTg, T_host, bytes, cudaMemcpyHostToDevice, p->stream));
            if (H_host) CF_CUDA_CHECK(cudaMemcpyAsync(p->dHg, H_host, bytes, cudaMemcpyHostToDevice, p->stream));
        }
        for (auto& rp : p->ranks) {
            Rank& r = *rp;
            const int32_t n = r.H.n_local;
            const int blocks = std::max(1, std::min(1184, (n + 255) / 256));
            double* tg = T_host ? p->dTg : nullptr;
            double* hg = H_host ? p->dHg : nullptr;
            if (p->temp_dep)
                gather_fields_kernel<true><<<blocks, 256, 0, p->stream>>>(n, r.ta.local_global, r.T[p->cur],
                                                                          r.ua.node_region, p->dP, tg, hg);
            else
                gather_fields_kernel<false><<<blocks, 256, 0, p->stream>>>(n, r.ta.local_global, r.T[p->cur],
                                                                           r.ua.node_region, p->dP, tg, hg);
        }
        CF_CUDA_CHECK(cudaGetLastError());
        if (T_host) CF_CUDA_CHECK(cudaMemcpyAsync(T_host, p->dTg, (size_t)p->N_global * sizeof(double),
                                                  cudaMemcpyDeviceToHost, p->stream));
        if (H_host) CF_CUDA_CHECK(cudaMemcpyAsync(H_host, p->dHg, (size_t)p->N_global * sizeof(double),
                                                  cudaMemcpyDeviceToHost, p->stream));
        CF_CUDA_CHECK(cudaStreamSynchronize(p->stream));
    });
}

int cf_get_stats(cf_plan* p, cf_stats* out) {
    return guarded([&] {
        if (!p || !out) raise(CF_INVALID_ARG, "null argument");
        CF_CUDA_CHECK(cudaSetDevice(p->device));
        const DevState st = read_state(p);
        std::memset(out, 0, sizeof *out);
        out->time = st.time;
        out->dt = st.dt;
        out->step_index = st.step_index;
        out->clamp_steps = st.clamp_steps;
        out->loop_seconds = p->loop_seconds;
        out->static_dt = p->temp_dep ? 0 : p->P.static_dt;
        out->dynamic_dt = p->temp_dep;
        for (auto& r : p->ranks) {
            out->n_tiles += r->H.n_tiles;
            out->n_elems_local += r->E_r;
            out->n_nodes_local += r->H.n_local;
            out->total_slots += r->H.tile_slot_off.empty() ? 0 : r->H.tile_slot_off.back();
            out->n_shared_nodes += r->H.n_shared;
            out->n_ghost_nodes += r->H.n_ghost;
            out->device_bytes += r->mem.bytes;
            out->bytes_per_step += r->bytes_per_step;
            out->tile_bytes_per_launch += r->tile_bytes;
            out->update_bytes_per_step += r->update_bytes;
        }
        out->launches_per_step = p->launches_per_step;
        out->n_nodes_global = p->N_global;
        out->n_elems_global = p->E_global;
        out->device_setup = p->device_setup ? 1 : 0;
    });
}

int cf_device_temperature(cf_plan* p, int32_t k, double** dptr, int64_t* n) {
    return guarded([&] {
        if (!p || !dptr || !n || k < 0 || k >= (int32_t)p->ranks.size()) raise(CF_INVALID_ARG, "bad argument");
        *dptr = p->ranks[k]->T[p->cur];
        *n = p->ranks[k]->H.n_local;
    });
}

int cf_choose_tile_elems(const int32_t* candidates, const double* seconds, int32_t n, int32_t* chosen) {
    return guarded([&] {
        // choose_block_count blocked.hpp:566-575
        if (n <= 0 || !candidates || !seconds || !chosen) raise(CF_VALIDATION, "autotune needs one timing per candidate");
        int32_t best = 0;
        for (int32_t i = 1; i < n; ++i)
            if (seconds[i] < seconds[best]) best = i;
        *chosen = candidates[best];
    });
}

int cf_default_tile_candidates(int64_t n_elems, int32_t* out, int32_t cap, int32_t* count) {
    return guarded([&] {
        if (!count) raise(CF_INVALID_ARG, "null argument");
        int32_t c = 0;
        for (int32_t te : {192, 384, 768, 1536}) {  // 6 * 2^k, multiples of 32 (whole warps)
            if (c > 0 && n_elems / te < 148) break;  // keep at least one CTA per SM
            if (out && c < cap) out[c] = te;
            ++c;
        }
        *count = c;
    });
}

int cf_autotune_tiles(const cf_mesh_desc* mesh, const cf_setup_desc* setup, const cf_run_opts* opts,
                      const int32_t* candidates, int32_t n_candidates, int32_t trial_steps,
                      double projected_total_steps, double* seconds_out, cf_tune_report* out) {
    return guarded([&] {
        if (!mesh || !setup || !opts || !out) raise(CF_INVALID_ARG, "null argument");
        const auto t0 = std::chrono::steady_clock::now();
        std::vector<int32_t> cand;
        if (candidates && n_candidates > 0) {
            cand.assign(candidates, candidates + n_candidates);
        } else {
            int32_t n = 0;
            cand.resize(8);
            if (cf_default_tile_candidates(mesh->n_elems, cand.data(), 8, &n) != CF_OK) raise(CF_INVALID_ARG, "candidates");
            cand.resize(n);
        }
        if (trial_steps < 1) raise(CF_INVALID_ARG, "trial_steps must be >= 1");
        std::vector<double> secs(cand.size(), INFINITY);
        for (size_t i = 0; i < cand.size(); ++i) {
            cf_run_opts o = *opts;
            o.tile_elems = cand[i];
            o.tile_of_element = nullptr;
            cf_plan* p = nullptr;
            const int st = cf_plan_create(mesh, setup, &o, &p);
            if (st == CF_INVALID_ARG) continue;  // tiles too large for shared memory: +inf
            if (st != CF_OK) raise(st, std::string("autotune candidate ") + std::to_string(cand[i]) + ": " +
                                           g_last_error);
            std::unique_ptr<cf_plan, int (*)(cf_plan*)> guard(p, cf_plan_destroy);
            CF_CUDA_CHECK(cudaSetDevice(p->device));
            for (int rep = 0; rep < 2; ++rep) {  // best of 2 from the initial field (autotune_block_count)
                if (rep) scatter_state(p);       // dTg still holds the plan's initial field
                p->loop_seconds = 0;
                run_steps(p, trial_steps, 0.0);
                secs[i] = std::min(secs[i], p->loop_seconds);
            }
        }
        int32_t chosen = 0;
        if (cf_choose_tile_elems(cand.data(), secs.data(), (int32_t)cand.size(), &chosen) != CF_OK)
            raise(CF_VALIDATION, g_last_error);
        out->n_candidates = (int32_t)cand.size();
        out->chosen = chosen;
        out->overhead_fraction = 0;
        const double wall = std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count();
        if (projected_total_steps > 0) {
            const size_t k = (size_t)(std::find(cand.begin(), cand.end(), chosen) - cand.begin());
            const double projected = secs[k] / trial_steps * projected_total_steps;
            out->overhead_fraction = wall / (wall + projected);
        }
        if (seconds_out) std::copy(secs.begin(), secs.end(), seconds_out);
    });
}

int cf_estimate_lambda_max(cf_plan* p, int32_t iterations, uint64_t seed, double* lambda, double* eq13) {
    return guarded([&] {
        if (!p || !lambda) raise(CF_INVALID_ARG, "null argument");
        if (p->ranks.size() != 1 || p->world != 1) raise(CF_INVALID_ARG, "lambda_max needs a single-rank plan");
        CF_CUDA_CHECK(cudaSetDevice(p->device));
        Rank& r = *p->ranks[0];
        const int32_t n = r.H.n_local;
        DeviceMem M;
        std::vector<double> cval(kMaxRegions, 0), kval(kMaxRegions, 0), hval(kMaxFacetKinds, 0);
        // properties at the region's initial temperature (no latent heat);
        // h of an interface table: its largest value (conservative)
        for (int g = 0; g < p->P.n_materials; ++g) {
            const DevMaterial& mm = p->P.mat[g];
            if (!(mm.rho > 0)) continue;
            cval[g] = mm.rho * pl_eval(p->P, mm.c, mm.T0);
            kval[g] = pl_eval(p->P, mm.k, mm.T0);
        }
        for (int k = 0; k < p->P.n_kinds; ++k) {
            const DevFacetKind& K = p->P.kind[k];
            if (K.interface) {
                double hm = -INFINITY;
                for (int j = 0; j < K.htab.n; ++j) hm = std::max(hm, p->P.pool[K.htab.off + K.htab.n + j]);
                hval[k] = hm;
            } else {
                hval[k] = K.h;
            }
        }
        LamArgs L;
        L.a = r.ta;
        L.tdep = p->temp_dep;
        L.coords = r.H.coords;
        L.cval = M.up(cval, p->stream);
        L.kval = M.up(kval, p->stream);
        L.hval = M.up(hval, p->stream);
        double* x = M.alloc<double>(n);
        double* y = M.alloc<double>(n);
        L.M = M.alloc<double>(n);
        L.D = M.alloc<double>(n);
        double* acc = M.alloc<double>(3);
        CF_CUDA_CHECK(cudaMemsetAsync(L.M, 0, n * sizeof(double), p->stream));
        CF_CUDA_CHECK(cudaMemsetAsync(L.D, 0, n * sizeof(double), p->stream));
        L.x = x;
        L.y = y;
        lam_setup<<<r.H.n_tiles, 256, 0, p->stream>>>(L);  // one CTA per tile (blob in global)
        const int blocks = std::max(1, std::min(1184, (n + 255) / 256));
        lam_init_x<<<blocks, 256, 0, p->stream>>>(n, r.ta.local_global, r.ta.node_dir, seed, x);
        double h_acc[3] = {0, 0, 0};
        for (int it = 0; it < iterations; ++it) {
            lam_diag<<<blocks, 256, 0, p->stream>>>(n, L.D, x, y);
            lam_apply<<<r.H.n_tiles, 256, 0, p->stream>>>(L);
            CF_CUDA_CHECK(cudaMemsetAsync(acc, 0, 3 * sizeof(double), p->stream));
            lam_reduce<<<blocks, 256, 0, p->stream>>>(n, r.ta.node_dir, L.M, x, y, acc);
            lam_scale<<<blocks, 256, 0, p->stream>>>(n, y, acc, x);
        }
        CF_CUDA_CHECK(cudaMemcpyAsync(h_acc, acc, sizeof h_acc, cudaMemcpyDeviceToHost, p->stream));
        CF_CUDA_CHECK(cudaStreamSynchronize(p->stream));
        M.release();
        *lambda = h_acc[0] / h_acc[1];
        if (eq13) *eq13 = p->eq13_min;
    });
}

int cf_comm_unique_id(uint8_t out[128]) {
    return guarded([&] {
        ncclUniqueId id;
        CF_NCCL_CHECK(nccl().GetUniqueId(&id));
        static_assert(sizeof(id) == 128, "ncclUniqueId size");
        std::memcpy(out, &id, 128);
    });
}

int cf_comm_create(int32_t world, int32_t rank, int32_t device, const uint8_t uid[128], cf_comm** out) {
    return guarded([&] {
        if (!out || !uid) raise(CF_INVALID_ARG, "null argument");
        CF_CUDA_CHECK(cudaSetDevice(device));
        auto c = std::make_unique<cf_comm>();
        ncclUniqueId id;
        std::memcpy(&id, uid, 128);
        CF_NCCL_CHECK(nccl().CommInitRank(&c->comm, world, id, rank));
        c->world = world;
        c->rank = rank;
        c->device = device;
        *out = c.release();
    });
}

int cf_comm_create_host(int32_t world, int32_t rank, int32_t device, const cf_host_transport* t, cf_comm** out) {
    return guarded([&] {
        if (!out || !t || !t->sendrecv || !t->allreduce) raise(CF_INVALID_ARG, "null argument");
        if (world < 1 || rank < 0 || rank >= world) raise(CF_INVALID_ARG, "bad world / rank");
        auto c = std::make_unique<cf_comm>();
        c->world = world;
        c->rank = rank;
        c->device = device;
        c->host = true;
        c->ht = *t;
        *out = c.release();
    });
}

int cf_comm_create_peer(int32_t world, int32_t rank, int32_t device, const cf_host_transport* t, cf_comm** out) {
    return guarded([&] {
        if (!out || !t || !t->sendrecv || !t->allreduce) raise(CF_INVALID_ARG, "null argument");
        if (world < 1 || rank < 0 || rank >= world) raise(CF_INVALID_ARG, "bad world / rank");
        if (world > kPeerMaxWorld) raise(CF_INVALID_ARG, "peer-memory transport: world_size > " + std::to_string(kPeerMaxWorld));
        auto c = std::make_unique<cf_comm>();
        c->world = world;
        c->rank = rank;
        c->device = device;
        c->peer = true;
        c->ht = *t;
        *out = c.release();
    });
}

int cf_comm_destroy(cf_comm* c) {
    return guarded([&] {
        if (!c) return;
        if (c->comm) nccl().CommDestroy(c->comm);
        delete c;
    });
}

// ------------------------------------------------------------------ host utilities
int cf_rcm_permutation(const cf_mesh_desc* d, int32_t seed, int32_t* out) {
    return guarded([&] {
        if (!d || !out) raise(CF_INVALID_ARG, "null argument");
        const Graph g = build_node_graph(d->n_nodes, d->n_elems, d->tets);
        const auto p = rcm_permutation(g, seed);
        std::memcpy(out, p.data(), sizeof(int32_t) * p.size());
    });
}

int cf_rcm_permutation_device(const cf_mesh_desc* d, int32_t seed, int32_t device, int32_t* out) {
    return guarded([&] {
        if (!d || !out) raise(CF_INVALID_ARG, "null argument");
        if (d->n_nodes < 0 || d->n_elems < 0) raise(CF_INVALID_ARG, "negative size");
        for (int64_t k = 0; k < 4 * (int64_t)d->n_elems; ++k)
            if (d->tets[k] < 0 || d->tets[k] >= d->n_nodes) raise(CF_VALIDATION, "tet node id out of range");
        const auto p = rcm_permutation_device(d->n_nodes, d->n_elems, d->tets, seed, device);
        std::memcpy(out, p.data(), sizeof(int32_t) * p.size());
    });
}

int cf_bandwidth(const cf_mesh_desc* d, const int32_t* perm, int64_t* out) {
    return guarded([&] {
        if (!d || !out) raise(CF_INVALID_ARG, "null argument");
        const Graph g = build_node_graph(d->n_nodes, d->n_elems, d->tets);
        *out = bandwidth(g, perm);
    });
}

int cf_finalize_mesh(const cf_mesh_desc* d, int32_t* tets_out, int32_t* owner_out) {
    return guarded([&] {
        MeshData m;
        finalize_mesh(d, m);
        if (tets_out) std::memcpy(tets_out, m.tets.data(), sizeof(int32_t) * m.tets.size());
        if (owner_out) std::memcpy(owner_out, m.owner.data(), sizeof(int32_t) * m.owner.size());
    });
}

int cf_pair_sister_facets(const cf_mesh_desc* d, int32_t* out, int64_t cap, int64_t* n) {
    return guarded([&] {
        MeshData m;
        finalize_mesh(d, m);
        const auto pairs = pair_sister_facets(m);
        if (n) *n = (int64_t)pairs.size();
        if (out)
            for (size_t i = 0; i < pairs.size() && (int64_t)i < cap; ++i) {
                out[3 * i] = pairs[i].facet;
                out[3 * i + 1] = pairs[i].sister;
                out[3 * i + 2] = pairs[i].contact;
            }
    });
}

int cf_partition_rcb(const cf_mesh_desc* d, int32_t parts, int32_t* out) {
    return guarded([&] {
        MeshData m;
        finalize_mesh(d, m);
        const auto p = partition_rcb(m, parts);
        std::memcpy(out, p.data(), sizeof(int32_t) * p.size());
    });
}

int cf_partition_graph(const cf_mesh_desc* d, int32_t parts, double balance_tol, int32_t augment, int32_t* out) {
    return guarded([&] {
        if (!d || !out) raise(CF_INVALID_ARG, "null argument");
        MeshData m;
        finalize_mesh(d, m);
        const auto p = partition_elements(m, parts, balance_tol, augment != 0);
        std::memcpy(out, p.data(), sizeof(int32_t) * p.size());
    });
}

int cf_partition_metrics(const cf_mesh_desc* d, const int32_t* part, int32_t parts, int64_t* edge_cut,
                         double* imbalance, int32_t* neighbor_counts, int64_t* split_interface_pairs) {
    return guarded([&] {
        if (!d || !part) raise(CF_INVALID_ARG, "null argument");
        if (parts < 1) raise(CF_VALIDATION, "part count must be >= 1");
        for (int32_t e = 0; e < d->n_elems; ++e)
            if (part[e] < 0 || part[e] >= parts) raise(CF_VALIDATION, "part id out of range");
        MeshData m;
        finalize_mesh(d, m);
        const PartitionQuality q = partition_metrics(m, part, parts);
        if (edge_cut) *edge_cut = q.edge_cut;
        if (imbalance) *imbalance = q.imbalance;
        if (neighbor_counts) std::memcpy(neighbor_counts, q.neighbor_counts.data(), sizeof(int32_t) * parts);
        if (split_interface_pairs) *split_interface_pairs = count_split_interface_pairs(m, part);
    });
}

int cf_tile_map(const cf_mesh_desc* mesh, const cf_setup_desc* setup, const cf_run_opts* opts,
                int32_t* tile_of_element, int32_t* n_tiles) {
    return guarded([&] {
        if (!mesh || !setup || !opts || !tile_of_element) raise(CF_INVALID_ARG, "null argument");
        MeshData m;
        finalize_mesh(mesh, m);
        SetupData S;
        resolve_setup(m, setup, S);
        std::vector<int32_t> label(m.N);
        if (opts->node_order == CF_NODE_ORDER_RCM)  // the plan's own pass where a B200 is present
            label = cuda_device_present() ? rcm_permutation_device(m.N, m.E, m.tets.data(), -1, opts->device)
                                          : rcm_permutation(build_node_graph(m.N, m.E, m.tets.data()), -1);
        else
            std::iota(label.begin(), label.end(), 0);
        PlanOptions po;
        po.mode = opts->mode;
        po.elem_order = opts->elem_order;
        po.geometry = opts->geometry;
        po.tile_elems = opts->tile_elems > 0 ? opts->tile_elems : 384;
        po.tile_of_element = opts->tile_of_element;
        po.world_size = std::max(1, opts->world_size);
        std::vector<int32_t> part;
        if (po.world_size > 1) {
            part = opts->partition == CF_PARTITION_GIVEN && opts->part_of_element
                       ? std::vector<int32_t>(opts->part_of_element, opts->part_of_element + m.E)
                   : opts->partition == CF_PARTITION_GRAPH ? partition_elements(m, po.world_size, 0.05, true)
                                                           : partition_rcb(m, po.world_size);
            po.part_of_element = part.data();
        }
        for (int32_t e = 0; e < m.E; ++e) tile_of_element[e] = -1;
        int32_t base = 0;
        const int r0 = opts->rank, r1 = opts->local_ranks > 1 ? po.world_size : opts->rank + 1;
        for (int r = r0; r < r1; ++r) {
            RankPlan rp;
            build_rank_plan(m, S, po, label, r, rp);
            int64_t pos = 0;
            for (int32_t t = 0; t < rp.n_tiles; ++t)
                for (int32_t i = 0; i < rp.tile_meta[t].ne; ++i) tile_of_element[rp.elem_global[pos++]] = base + t;
            base += rp.n_tiles;
        }
        if (n_tiles) *n_tiles = base;
    });
}

int cf_exchange_plan(const cf_mesh_desc* mesh, const cf_setup_desc* setup, const cf_run_opts* opts, int32_t* n_nbrs,
                     int32_t* nbr_rank, int64_t* counts, int32_t* shared, int32_t* ext_to, int32_t* ext_from) {
    return guarded([&] {
        if (!mesh || !setup || !opts || !n_nbrs) raise(CF_INVALID_ARG, "null argument");
        if (opts->world_size < 2) raise(CF_INVALID_ARG, "exchange plan needs world_size >= 2");
        trace_stage("exchange_plan: start");
        MeshData m;
        finalize_mesh(mesh, m);
        SetupData S;
        resolve_setup(m, setup, S);
        trace_stage("resolve: rest");
        std::vector<int32_t> label(m.N);
        std::iota(label.begin(), label.end(), 0);
        PlanOptions po;
        po.elem_order = opts->elem_order;
        po.geometry = opts->geometry;
        po.node_order = CF_NODE_ORDER_GIVEN;
        po.tile_elems = opts->tile_elems > 0 ? opts->tile_elems : 384;
        po.world_size = opts->world_size;
        std::vector<int32_t> part = opts->partition == CF_PARTITION_GIVEN && opts->part_of_element
                                        ? std::vector<int32_t>(opts->part_of_element, opts->part_of_element + m.E)
                                    : opts->partition == CF_PARTITION_GRAPH ? partition_elements(m, po.world_size, 0.05, true)
                                                                            : partition_rcb(m, po.world_size);
        trace_stage("partition");
        po.part_of_element = part.data();
        RankPlan rp;
        build_rank_plan(m, S, po, label, opts->rank, rp);
        *n_nbrs = (int32_t)rp.nbrs.size();
        int64_t os = 0, ot = 0, of = 0;
        for (size_t k = 0; k < rp.nbrs.size(); ++k) {
            const auto& x = rp.nbrs[k];
            if (nbr_rank) nbr_rank[k] = x.rank;
            if (counts) {
                counts[3 * k] = (int64_t)x.shared.size();
                counts[3 * k + 1] = (int64_t)x.ext_to.size();
                counts[3 * k + 2] = (int64_t)x.ext_from.size();
            }
            for (int32_t l : x.shared) if (shared) shared[os++] = rp.local_global[l];
            for (int32_t l : x.ext_to) if (ext_to) ext_to[ot++] = rp.local_global[l];
            for (int32_t l : x.ext_from) if (ext_from) ext_from[of++] = rp.local_global[l];
        }
    });
}

}  // extern "C"
// Digest of one rank's tiled plan (host builder, or the device builder with device != 0): one
// FNV-1a 64 per plan array, in the order of cf_plan_digest_names (castfem_b200.h). Test
// instrumentation: the two builders must agree array for array.
static uint64_t fnv(const void* p, size_t n, uint64_t h = 1469598103934665603ull) {
    const uint8_t* b = (const uint8_t*)p;
    for (size_t i = 0; i < n; ++i) h = (h ^ b[i]) * 1099511628211ull;
    return h;
}
template <class V>
static uint64_t fnv_vec(const V& v) {
    return fnv(v.data(), v.size() * sizeof(typename V::value_type), fnv(&v, 0) ^ (uint64_t)v.size());
}
static void digest_rank_plan(const RankPlan& rp, uint64_t* d) {
    int k = 0;
    const int64_t scal[] = {rp.n_tiles, rp.n_local, rp.n_ghost, rp.n_if_facets, rp.n_bc_facets, rp.n_private,
                            rp.max_slots, rp.max_elems, rp.max_facets, rp.max_blob, rp.blob_bytes, rp.n_shared,
                            rp.send_len, rp.recv_len};
    d[k++] = fnv(scal, sizeof scal);
    d[k++] = fnv_vec(rp.tile_meta);
    d[k++] = fnv_vec(rp.tile_border);
    d[k++] = fnv_vec(rp.tile_slot_off);
    d[k++] = fnv_vec(rp.blob_off);
    d[k++] = fnv_vec(rp.elem_off);
    uint64_t hb = 0;  // the staged (non-geometry) part of every tile, tile by tile
    for (int32_t t = 0; t < rp.n_tiles; ++t) hb = fnv(rp.blob.data() + rp.rest_off[t], rp.rest_off[t + 1] - rp.rest_off[t], hb ^ (uint64_t)t);
    d[k++] = hb;
    d[k++] = fnv_vec(rp.tets_ord);
    d[k++] = fnv_vec(rp.elem_global);
    d[k++] = fnv_vec(rp.slot_node);
    d[k++] = fnv_vec(rp.local_global);
    d[k++] = fnv_vec(rp.node_region);
    d[k++] = fnv_vec(rp.node_dir);
    d[k++] = fnv_vec(rp.merge_off);
    d[k++] = fnv_vec(rp.merge_idx);
    d[k++] = fnv_vec(rp.shared_list);
    uint64_t hn = 0;
    for (const auto& x : rp.nbrs) {
        hn = fnv(&x.rank, 4, hn);
        hn ^= fnv_vec(x.shared) + 3 * fnv_vec(x.ext_to) + 7 * fnv_vec(x.ext_from);
    }
    d[k++] = hn;
    d[k++] = fnv_vec(rp.node_shared) ^ 3 * fnv_vec(rp.shared_off) ^ 5 * fnv_vec(rp.shared_src) ^
             7 * fnv_vec(rp.shared_src_r) ^ 11 * fnv_vec(rp.send_off) ^ 13 * fnv_vec(rp.recv_off) ^
             17 * fnv_vec(rp.ghost_src);
    while (k < CF_DIGEST_LEN) d[k++] = 0;
}

extern "C" {
int cf_plan_digest(const cf_mesh_desc* mesh, const cf_setup_desc* setup, const cf_run_opts* opts, int32_t rank,
                   uint64_t* digest) {
    return guarded([&] {
        if (!mesh || !setup || !opts || !digest) raise(CF_INVALID_ARG, "null argument");
        MeshData m;
        finalize_mesh(mesh, m);
        SetupData S;
        resolve_setup(m, setup, S);
        std::vector<int32_t> label(m.N);
        if (opts->node_order == CF_NODE_ORDER_RCM)
            label = rcm_permutation(build_node_graph(m.N, m.E, m.tets.data()), -1);
        else
            std::iota(label.begin(), label.end(), 0);
        PlanOptions po;
        po.mode = opts->mode;
        po.node_order = opts->node_order;
        po.elem_order = opts->elem_order;
        po.geometry = opts->geometry;
        po.tile_elems = opts->tile_elems > 0 ? opts->tile_elems : 384;
        po.tile_of_element = opts->tile_of_element;
        po.n_tiles_given = opts->n_tiles_given;
        po.world_size = std::max(1, opts->world_size);
        std::vector<int32_t> part;
        if (po.world_size > 1) {
            part = opts->partition == CF_PARTITION_GIVEN && opts->part_of_element
                       ? std::vector<int32_t>(opts->part_of_element, opts->part_of_element + m.E)
                       : partition_rcb(m, po.world_size);
            po.part_of_element = part.data();
        }
        RankPlan rp;
        build_rank_plan(m, S, po, label, rank, rp);
        digest_rank_plan(rp, digest);
    });
}

// the same digests from the device setup pipeline (needs a B200)
int cf_plan_digest_device(const cf_mesh_desc* mesh, const cf_setup_desc* setup, const cf_run_opts* opts, int32_t rank,
                          uint64_t* digest) {
    return guarded([&] {
        if (!mesh || !setup || !opts || !digest) raise(CF_INVALID_ARG, "null argument");
        int tile = 384;
        cf_run_opts o = normalized_opts(opts, tile);
        cudaStream_t s;
        CF_CUDA_CHECK(cudaStreamCreateWithFlags(&s, cudaStreamNonBlocking));
        struct SG {
            cudaStream_t s;
            ~SG() { cudaStreamDestroy(s); }
        } sg{s};
        DevMesh dm;
        devmesh_from_desc(mesh, s, dm);
        DevSetup ds;
        resolve_setup_device(dm, setup, T0Noise{}, s, ds);
        DBuf work;
        int32_t* d_label = nullptr;
        if (o.node_order == CF_NODE_ORDER_RCM) {
            d_label = work.alloc<int32_t>(dm.N);
            rcm_labels_device(dm.N, dm.E, dm.tets, -1, s, d_label);
        }
        int32_t* d_part = nullptr;
        if (o.world_size > 1) {
            d_part = work.alloc<int32_t>(dm.E);
            if (o.partition == CF_PARTITION_GIVEN && o.part_of_element)
                CF_CUDA_CHECK(cudaMemcpyAsync(d_part, o.part_of_element, sizeof(int32_t) * dm.E, cudaMemcpyHostToDevice, s));
            else
                partition_rcb_device(dm, o.world_size, s, d_part);
        }
        DevRankPlan dp;
        build_rank_plan_device(dm, ds, plan_options(o, tile), d_label, d_part, rank, s, dp);
        RankPlan rp;
        download_dev_rank_plan(dp, ds.S.temp_dep, o.geometry == CF_GEOM_COORDS, s, rp);
        digest_rank_plan(rp, digest);
    });
}

// device partition (test instrumentation: equal to cf_partition_rcb)
int cf_partition_rcb_device(const cf_mesh_desc* mesh, int32_t parts, int32_t* out) {
    return guarded([&] {
        if (!mesh || !out) raise(CF_INVALID_ARG, "null argument");
        cudaStream_t s;
        CF_CUDA_CHECK(cudaStreamCreateWithFlags(&s, cudaStreamNonBlocking));
        struct SG {
            cudaStream_t s;
            ~SG() { cudaStreamDestroy(s); }
        } sg{s};
        DevMesh dm;
        devmesh_from_desc(mesh, s, dm);
        DBuf work;
        int32_t* d = work.alloc<int32_t>(dm.E);
        partition_rcb_device(dm, parts, s, d);
        CF_CUDA_CHECK(cudaMemcpy(out, d, sizeof(int32_t) * dm.E, cudaMemcpyDeviceToHost));
    });
}

int cf_generate_fixture(int32_t kind, int32_t n, double radius, double jitter, uint64_t seed, uint64_t perm_seed,
                        cf_fixture* out) {
    return guarded([&] {
        if (!out) raise(CF_INVALID_ARG, "null argument");
        generate_fixture(kind, n, radius, jitter, seed, perm_seed, out);
    });
}

int cf_counter_uniform(uint64_t seed, const int64_t* keys, int64_t n, double lo, double hi, double* out) {
    return guarded([&] {
        if (n && (!keys || !out)) raise(CF_INVALID_ARG, "null argument");
        for (int64_t i = 0; i < n; ++i) out[i] = lo + (hi - lo) * counter_uniform(seed, (uint64_t)keys[i]);
    });
}

}  // extern "C"
