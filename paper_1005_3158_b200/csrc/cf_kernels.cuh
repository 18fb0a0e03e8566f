// cf_kernels.cuh — sm_100a kernels of the castfem explicit step.
//
// One step (blocked_step blocked.hpp:542-550) is two kernels:
//   tile_kernel    assemble_blocks (blocked.hpp:454-498), one CTA per tile (the
//                  paper's cache block recast as a thread-block tile):
//                    - one elected thread streams the tile's packed blob (element
//                      geometry, connectivity, facets, reduction CSR;
//                      cf_tileblob.hpp) into shared memory with TMA bulk copies
//                      (cp.async.bulk + mbarrier complete_tx), while
//                    - all threads gather the tile's nodal T (L2-resident) and
//                      derive H = enthalpy(T) once per tile slot;
//                    - element physics (Lemmon C_app, lumped capacitance,
//                      conduction residual) and facet fluxes (convective, and
//                      interface with the one-step-lagged sister ambient read from
//                      the previous T buffer) write their contributions in place
//                      over the consumed blob columns;
//                    - a fixed-order per-slot reduction through the tile CSR (no
//                      shared-memory fp64 atomics: those are CAS loops on sm_100a);
//                    - flush: tile-private nodes are UPDATED right here (merge is
//                      the identity for them: merge_blocks :502-515), tile-shared
//                      nodes write per-(tile, slot) partials (deterministic) or
//                      fp64 RED into node accumulators (atomic).
//   update_kernel  merge_blocks + update_fields (:519-538) for the shared nodes
//                  only: ascending-tile merge, ascending-rank combine across GPUs,
//                  T += (dt*r)/c, Dirichlet, clamp flag; the last CTA advances time.
// With temperature-dependent tables (dynamic dt, :477-480) dt is a global min
// known only after assembly, so no node is updated in the tile kernel.
#pragma once

#include <cuda_runtime.h>

#include <cstdint>

#include "cf_physics.cuh"
#include "cf_tileblob.hpp"

namespace cfb {

// Diagnostics (CF_PROBE: skip phases, L2-resident replay) exist only in a -DCF_DIAG build
// (`make DIAG=1`, results invalid); the production kernels compile every probe branch away.
#ifdef CF_DIAG
#define CF_PRB(a) ((a).probe)
#else
#define CF_PRB(a) 0
#endif
// Bounds assertions (a -DCF_BOUNDS build, `make BOUNDS=1`): every shared-memory index the tile
// kernel derives from plan data and every global index of the step kernels is checked against
// its array, trapping on violation -- the memcheck substitute where compute-sanitizer is
// unavailable (tests run against such a build, scripts/bounds_check.sh). Compiled out otherwise.
#ifdef CF_BOUNDS
#define CF_ASSERT(c) do { if (!(c)) __trap(); } while (0)
#else
#define CF_ASSERT(c) do { } while (0)
#endif

struct DevState {
    double time;
    double dt;
    long long step_index;
    long long clamp_steps;
    unsigned long long min_bound[2];  // positive doubles as bits (atomicMin)
    int clamp_flag;
    unsigned int ticket;
    int err_node;                     // INT32_MAX: none
    int done;
};

// ------------------------------------------------------------------ PTX helpers
__device__ __forceinline__ uint32_t smem_u32(const void* p) {
    return (uint32_t)__cvta_generic_to_shared(p);
}
__device__ __forceinline__ void mbar_init(uint64_t* bar, uint32_t count) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count) : "memory");
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
}
__device__ __forceinline__ void mbar_expect_tx(uint64_t* bar, uint32_t bytes) {
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)), "r"(bytes)
                 : "memory");
}
__device__ __forceinline__ void bulk_g2s(void* dst, const void* src, uint32_t bytes, uint64_t* bar) {
    asm volatile(
        "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
            smem_u32(dst)),
        "l"(src), "r"(bytes), "r"(smem_u32(bar))
        : "memory");
}
__device__ __forceinline__ void bulk_prefetch_l2(const void* src, uint32_t bytes) {
    asm volatile("cp.async.bulk.prefetch.L2.global [%0], %1;" ::"l"(src), "r"(bytes) : "memory");
}
// programmatic dependent launch: wait for the preceding kernel's completion (and memory);
// a no-op without the launch attribute. No kernel triggers early (griddepcontrol.
// launch_dependents): early-resident waiting CTAs measured slower than the implicit trigger
// at CTA exit, which still hides the launch latency between the step's kernels.
__device__ __forceinline__ void griddep_wait() { asm volatile("griddepcontrol.wait;" ::: "memory"); }
__device__ __forceinline__ void mbar_wait(uint64_t* bar, uint32_t parity) {
    asm volatile(
        "{\n .reg .pred p;\n WAIT_%=:\n mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n @!p bra WAIT_%=;\n}" ::"r"(
            smem_u32(bar)),
        "r"(parity)
        : "memory");
}
__device__ __forceinline__ void st_release_sys(uint32_t* p, uint32_t v) {
    asm volatile("st.release.sys.global.u32 [%0], %1;" ::"l"(p), "r"(v) : "memory");
}
__device__ __forceinline__ void atomic_min_pos(unsigned long long* addr, double v) {
    atomicMin(addr, (unsigned long long)__double_as_longlong(v));
}

// dt of the current step (blocked_step blocked.hpp:547-548) and the done flag
// (solve_serial's loop condition :674-675 for the t_end mode).
template <bool TDEP>
__device__ __forceinline__ void step_dt(const DevParams* __restrict__ P, const DevState* st, double t_end,
                                        double& dt, double& t_next, bool& done) {
    const double time = st->time;
    dt = TDEP ? __longlong_as_double((long long)st->min_bound[st->step_index & 1]) * P->dt_safety : P->static_dt;
    done = false;
    if (t_end > 0) {
        const double remaining = t_end - time;
        if (!(time < t_end)) done = true;
        if (remaining > 0) dt = dt < remaining ? dt : remaining;
    }
    t_next = time + dt;
}

// update_fields for one node (blocked.hpp:519-538): explicit_update, Dirichlet, clamp
template <bool DIR, bool CLAMP>
__device__ __forceinline__ double node_update(const DevParams* __restrict__ P, DevState* st, double T, double c,
                                              double r, double dt, double t_next, int dir_id, int region,
                                              const int32_t* gid, int& clamped) {
    double Tn;
    if (!(c > 0)) {
        atomicMin(&st->err_node, *gid);  // explicit_update throws (fem.hpp:110-111); id loaded lazily
        Tn = T;
    } else {
        Tn = T + dt * r / c;
    }
    if (DIR && dir_id >= 0) Tn = dev_pl_eval(P, P->dir_tab[dir_id], t_next);
    if (CLAMP) {
        const DevMaterial& m = P->mat[region];
        if (Tn < m.range_lo || Tn > m.range_hi) clamped = 1;
    }
    return Tn;
}

// ------------------------------------------------------------------ tile kernel
struct TileArgs {
    const TileMeta* meta;
    const int32_t* slot_off;
    const int64_t* blob_off;
    const uint8_t* blob;
    const int32_t* slot_node;
    const uint8_t* node_region;
    const int8_t* node_dir;
    const int32_t* local_global;
    const double* T;     // current (unused by the tile kernel except through Tslot)
    const double* Told;  // previous step (ambient lag of interface facets)
    double* Tn;          // next (tile-private nodes)
    const double* Tslot; // current T of every tile slot
    double* Tslot_n;     // next T of every tile slot (tile-private slots written here)
    double2* part;       // per (tile, slot) partial (c, r)   [deterministic]
    double2* acc;        // per node (c, r) RED accumulators, one 16-byte pair per node  [atomic]
    const DevParams* P;
    DevState* st;
    const TileDesc* desc;      // tiles of this launch (metadata + offsets, one 32 B record each)
    int32_t n_tiles;           // tiles of this launch
    int32_t max_slots;
    int32_t blob_smem;   // bytes reserved per blob stage in shared memory
    int32_t stages;      // 1: one tile per CTA; 2: persistent, double-buffered
    int32_t prefetch;    // stages == 1: tile it + prefetch is staged into L2 by CTA it (0: off)
    int32_t scratch_off; // coordinates layout: byte offset of the contribution scratch in shared memory
    int32_t probe;       // diagnostics only (CF_PROBE; results invalid): 1 = copies only, 3 = no
                         // reduction phase, 4 = no element phase, 5 = no enthalpy evaluation,
                         // 7 = no Lemmon divide / sqrt, 8 = bank-conflict-free reduction operand
                         // reads (wrong operands); + 16: every CTA re-reads one of 1184
                         // L2-resident tiles (compute-side time)
    double t_end;
    int32_t* sched;            // dynamic tile scheduling counter (persistent single-stage grids), or null
    int32_t slot_gather;       // 1: slot temperatures gathered from T by node id (no slot copies)
    int32_t l2_next;           // persistent grids: stage the next tile's blob into L2 at phase 3's start
    // decomposed plans, one launch for every tile with the border tiles (those holding a
    // rank-shared node) first: when the last of them has flushed its partials the kernel raises
    // border_flag = border_seq, on which the exchange stream waits before it packs
    int32_t n_border;               // leading tiles of this launch that are border tiles (0: none)
    uint32_t border_seq;            // this step's flag value
    unsigned long long border_target;  // border_cnt after this step's last border tile (cumulative)
    unsigned long long* border_cnt;
    uint32_t* border_flag;
    int32_t n_local;           // bounds (CF_BOUNDS builds): local nodes (+ ghosts below n_T)
    int32_t n_T;
    int64_t n_slots;
};

constexpr uint32_t kBulkChunk = 32768;

struct TileHdr {  // per stage: the metadata of the tile in flight (written before the barrier arrive)
    TileMeta tm;
    int32_t s0;
    int64_t boff;  // blob byte offset (the stored layout's max_edge tail is read from global memory)
    // the tile's section layout, computed once by the issuing thread (raw storage: TileLayout
    // has a constructor, which __shared__ variables cannot run)
    alignas(8) unsigned char L[sizeof(TileLayout)];
    __device__ __forceinline__ const TileLayout& layout() const { return *reinterpret_cast<const TileLayout*>(L); }
};

// `it` indexes the launch's tile descriptors
// (slots == false: the slot temperatures -- written by the preceding kernel -- are left to
// issue_slot_copy after griddep_wait; the barrier already expects their bytes)
__device__ __forceinline__ void load_desc(const TileArgs& a, int it, int4& d0, int4& d1) {
    if (CF_PRB(a) & 16) it %= 1184;  // diagnostics: L2-resident tiles (compute-side time)
    d0 = __ldg((const int4*)(a.desc + it));
    d1 = __ldg((const int4*)(a.desc + it) + 1);
}
__device__ __forceinline__ void issue_tile_copy(const TileArgs& a, int4 d0, int4 d1, bool tdep, bool coords,
                                                uint8_t* dst, double* sTdst, uint64_t* bar, TileHdr* hdr,
                                                bool slots = true) {
    const TileMeta tm{d0.x, d0.y, d0.z, d0.w};
    const int32_t s0 = d1.x, bytes = d1.y;
    const int64_t boff = (int64_t)(uint32_t)d1.z | (int64_t)d1.w << 32;
    const uint32_t tbytes = 8u * (uint32_t)cf_round32(tm.ns, 2);
    // copies first (their complete_tx may precede the expect_tx: the barrier's phase also waits
    // for the arrive below), then the header, published by that arrive (release)
    const uint8_t* src = a.blob + boff;
    for (int32_t o = 0; o < bytes; o += (int32_t)kBulkChunk) {
        const uint32_t n = (uint32_t)(bytes - o < (int32_t)kBulkChunk ? bytes - o : (int32_t)kBulkChunk);
        bulk_g2s(dst + o, src + o, n, bar);
    }
    if (a.slot_gather) {
        hdr->tm = tm;
        hdr->s0 = s0;
        hdr->boff = boff;
        *reinterpret_cast<TileLayout*>(hdr->L) = TileLayout(tm, tdep, coords);
        mbar_expect_tx(bar, (uint32_t)bytes);
        return;
    }
    if (slots && tbytes) bulk_g2s(sTdst, a.Tslot + s0, tbytes, bar);
    hdr->tm = tm;
    hdr->s0 = s0;
    hdr->boff = boff;
    *reinterpret_cast<TileLayout*>(hdr->L) = TileLayout(tm, tdep, coords);
    mbar_expect_tx(bar, (uint32_t)bytes + tbytes);
}
// slot temperatures gathered from the node array by the tile's slot node ids (read from the
// tile's blob in global memory, so the gathers need not wait for its bulk copy): one 8-byte
// cp.async per slot into sTdst, one commit group per thread (possibly empty)
template <int NT>
__device__ __forceinline__ void gather_slot_T(const TileArgs& a, int4 d0, int4 d1, bool tdep, bool coords, double* sTdst,
                                              int tid) {
    const TileMeta tm{d0.x, d0.y, d0.z, d0.w};
    const int64_t boff = (int64_t)(uint32_t)d1.z | (int64_t)d1.w << 32;
    const TileLayout L(tm, tdep, coords);
    const int32_t* gsn = (const int32_t*)(a.blob + boff + L.snode);
    for (int s = tid; s < tm.ns; s += NT) {
        const int32_t node = __ldg(gsn + s);
        asm volatile("cp.async.ca.shared.global [%0], [%1], 8;" ::"r"(smem_u32(sTdst + s)), "l"(a.T + node) : "memory");
    }
    asm volatile("cp.async.commit_group;" ::: "memory");
}
// the next tile's descriptor, staged asynchronously into shared memory (no registers held)
__device__ __forceinline__ void prefetch_desc(const TileArgs& a, int it, int4* sdesc) {
    if (CF_PRB(a) & 16) it %= 1184;
    const int4* g = (const int4*)(a.desc + it);
    asm volatile("cp.async.ca.shared.global [%0], [%1], 16;" ::"r"(smem_u32(sdesc)), "l"(g) : "memory");
    asm volatile("cp.async.ca.shared.global [%0], [%1], 16;" ::"r"(smem_u32(sdesc + 1)), "l"(g + 1) : "memory");
    asm volatile("cp.async.commit_group;" ::: "memory");
}
__device__ __forceinline__ void staged_desc(const int4* sdesc, int4& d0, int4& d1, bool keep_last = false) {
    // keep_last: the most recent group (the next tile's slot-temperature gathers) may stay in flight
    if (keep_last) asm volatile("cp.async.wait_group 1;" ::: "memory");
    else asm volatile("cp.async.wait_all;" ::: "memory");
    d0 = sdesc[0];
    d1 = sdesc[1];
}
__device__ __forceinline__ void issue_slot_copy(const TileArgs& a, const TileHdr* hdr, double* sTdst, uint64_t* bar) {
    const uint32_t tbytes = 8u * (uint32_t)cf_round32(hdr->tm.ns, 2);
    if (tbytes) bulk_g2s(sTdst, a.Tslot + hdr->s0, tbytes, bar);
}

// L2 prefetch of the tile a CTA launched about one resident-grid width later will fetch
__device__ __forceinline__ void prefetch_tile(const TileArgs& a, int it, bool tdep, bool coords) {
    const int4 d0 = __ldg((const int4*)(a.desc + it)), d1 = __ldg((const int4*)(a.desc + it) + 1);
    const TileMeta tm{d0.x, d0.y, d0.z, d0.w};
    const int64_t boff = (int64_t)(uint32_t)d1.z | (int64_t)d1.w << 32;
    const TileLayout L(tm, tdep, coords);
    const uint8_t* src = a.blob + boff;
    for (int32_t o = 0; o < L.bytes; o += (int32_t)kBulkChunk)
        bulk_prefetch_l2(src + o, (uint32_t)(L.bytes - o < (int32_t)kBulkChunk ? L.bytes - o : kBulkChunk));
    const uint32_t tbytes = 8u * (uint32_t)cf_round32(tm.ns, 2);
    if (tbytes && a.Tslot) bulk_prefetch_l2(a.Tslot + d1.x, tbytes);
}

// Each CTA walks tiles blockIdx.x, +gridDim.x, ...; with stages == 2 it is a
// persistent two-stage TMA pipeline (the blob of tile k+1 streams in while
// tile k is computed), with stages == 1 the grid covers the tiles one-to-one.
#ifndef CF_GC_MINB
#define CF_GC_MINB 5  // min resident CTAs per SM requested from ptxas (coordinates layout: 96 regs;
                      // its light tiles fit 5 CTAs/SM in shared memory -- measured +3 %)
#endif
#ifndef CF_GS_MINB
#define CF_GS_MINB 1  // min resident CTAs per SM requested from ptxas (stored layout)
#endif
template <bool DET, bool TDEP, bool DIR, bool CLAMP, int kTileThreads, bool GC>
__global__ void __launch_bounds__(kTileThreads, GC ? CF_GC_MINB : CF_GS_MINB) tile_kernel(TileArgs a) {
    constexpr bool FUSE = !TDEP;
    extern __shared__ __align__(16) unsigned char smem[];
    __shared__ uint64_t bar[2];
    __shared__ TileHdr hdr[2];
    __shared__ int4 ndesc[2];  // next tile's descriptor (thread 0 only)
    __shared__ int s_issue;     // the tile whose copy follows this one in the stage buffer
    __shared__ DevMaterial sMat[kMaxRegions];
    const int tid = threadIdx.x;
    const DevParams* __restrict__ P = a.P;
    uint8_t* const buf0 = smem;
    uint8_t* const buf1 = smem + (a.stages - 1) * a.blob_smem;
    // slot-temperature buffers: one per stage; gathered slots (single stage) alternate between two,
    // the next tile's gathers landing while this tile computes
    const bool gather = a.slot_gather && a.stages == 1;
    const int nsT = (a.stages == 2 || gather) ? 2 : 1;
    double* const sT0 = (double*)(smem + a.stages * (size_t)a.blob_smem);
    double* const sT1 = sT0 + (nsT - 1) * a.max_slots;
    double2* sTH = (double2*)(sT0 + nsT * a.max_slots);  // (T, H) per slot, 16 B aligned

    // the first copy is the CTA's critical path: thread 0 initialises the barriers and issues it
    // before anything else; the material table, the step's dt and the scratch zeros overlap it
    // (the other threads touch the barriers only after the __syncthreads below)
    // With programmatic dependent launch this prologue (static blob) overlaps the previous
    // kernel's completion; the slot temperatures and the step state follow griddep_wait.
    const bool first0 = blockIdx.x < a.n_tiles, first1 = a.stages == 2 && blockIdx.x + gridDim.x < a.n_tiles;
    if (tid == 0) {
        mbar_init(&bar[0], 1);
        mbar_init(&bar[1], 1);
        int4 d0, d1;
        if (first0) {
            load_desc(a, blockIdx.x, d0, d1);
            issue_tile_copy(a, d0, d1, TDEP, GC, buf0, sT0, &bar[0], &hdr[0], false);
        }
        if (first1) {
            load_desc(a, blockIdx.x + gridDim.x, d0, d1);
            issue_tile_copy(a, d0, d1, TDEP, GC, buf1, sT1, &bar[1], &hdr[1], false);
        }
        griddep_wait();
        if (first0 && !gather) issue_slot_copy(a, &hdr[0], sT0, &bar[0]);
        if (first1) issue_slot_copy(a, &hdr[1], sT1, &bar[1]);
        if (a.stages == 1 && a.prefetch && (int)blockIdx.x + a.prefetch < a.n_tiles)
            prefetch_tile(a, blockIdx.x + a.prefetch, TDEP, GC);
    }
    // dynamic tile scheduling (persistent single-stage grids): after its first tile (blockIdx.x)
    // a CTA takes tickets from a.sched (reset to 0 by the update kernel); tile = grid + ticket.
    // Thread 0 draws the ticket one tile ahead, so the atomic's latency overlaps a whole tile.
    const bool dyn = a.sched != nullptr && a.stages == 1;
    int ticket = 0;
    if (dyn && tid == 0 && first0) ticket = atomicAdd(a.sched, 1);
    for (int i = tid; i < P->n_materials; i += kTileThreads) sMat[i] = P->mat[i];
    if (GC && tid < 2) ((double*)(smem + a.scratch_off))[tid] = 0.0;  // the facet entries' lump operand
    if (tid != 0) griddep_wait();  // before any thread reads the step state
    if (gather && first0) {  // the first tile's slot temperatures (T is final for this step)
        int4 d0, d1;
        load_desc(a, blockIdx.x, d0, d1);
        gather_slot_T<kTileThreads>(a, d0, d1, TDEP, GC, sT0, tid);
    }
    double dt = 0, t_next = 0;
    bool done = false;
    if (FUSE) step_dt<TDEP>(P, a.st, a.t_end, dt, t_next, done);
    const double time = a.st->time;
    __syncthreads();  // barriers initialised, material table staged
    int clamped = 0;
    double local_min = __longlong_as_double(0x7ff0000000000000ll);

    // a border tile is complete once every thread's flush has been fenced and the CTA has met at a
    // barrier; thread 0 then counts it and the CTA finishing the launch's last one raises the flag
    auto border_done = [&]() {
        __threadfence();
        const unsigned long long old = atomicAdd(a.border_cnt, 1ull);
        if (old + 1 == a.border_target) {
            __threadfence();
            st_release_sys(a.border_flag, a.border_seq);
        }
    };
    bool pending_border = false;  // the previous tile of this CTA was a border tile (CTA-uniform)
    int k = 0;
    for (int t = blockIdx.x; t < a.n_tiles; ++k) {
        const int stage = a.stages == 2 ? (k & 1) : 0;
        uint8_t* B = stage ? buf1 : buf0;
        double* sT = (gather ? (k & 1) : stage) ? sT1 : sT0;
        mbar_wait(&bar[stage], a.stages == 2 ? ((k >> 1) & 1) : (k & 1));
        if (gather) asm volatile("cp.async.wait_all;" ::: "memory");  // this thread's slot gathers
        const TileMeta tm = hdr[stage].tm;
        const int s0 = hdr[stage].s0;
        const TileLayout& L = hdr[stage].layout();
        const int ne = tm.ne, ns = tm.ns, nf = tm.nf;
        // t_follow: this CTA's next tile; t_issue: the tile copied into this stage's buffer next
        const int t_follow = dyn ? -1 : t + (int)gridDim.x;
        if (tid == 0) {
            int nx = t + a.stages * (int)gridDim.x;
            if (dyn) {
                nx = ticket + (int)gridDim.x;
                if (nx < a.n_tiles) ticket = atomicAdd(a.sched, 1);
            }
            s_issue = nx;
            if (nx < a.n_tiles) prefetch_desc(a, nx, ndesc);
        }
        int4 nd0, nd1;
        if ((CF_PRB(a) & 15) == 1) {  // diagnostics: memory-path timing without the physics
            __syncthreads();
            const int t_issue = s_issue;
            if (tid == 0 && t_issue < a.n_tiles) {
                staged_desc(ndesc, nd0, nd1);
                issue_tile_copy(a, nd0, nd1, TDEP, GC, B, sT, &bar[stage], &hdr[stage]);
            }
            t = dyn ? t_issue : t_follow;
            __syncthreads();  // s_issue read by every thread before its next write
            continue;
        }
        // interface facets: the 4 sister temperatures of the lagged ambient (T^{k-1}, global) are
        // gathered by cp.async into the facet record's sister/pad bytes (the ids are read first),
        // overlapping phases 1 and 2a; the same thread consumes them in phase 2b
        for (int i = tid; i < nf; i += kTileThreads) {
            double2* rec = (double2*)(B + L.fac + 48 * i);
            const ushort4 fs = *(const ushort4*)(B + L.fac_slots(i));
            if (!P->kind[fs.w].interface) continue;
            const int4 sn = *(const int4*)(rec + 1);
            CF_ASSERT(sn.x >= 0 && sn.y >= 0 && sn.z >= 0 && sn.w >= 0 && sn.x < a.n_T && sn.y < a.n_T && sn.z < a.n_T &&
                      sn.w < a.n_T);
            const uint32_t dst = smem_u32(rec + 1);
            asm volatile("cp.async.ca.shared.global [%0], [%1], 8;" ::"r"(dst), "l"(a.Told + sn.x) : "memory");
            asm volatile("cp.async.ca.shared.global [%0], [%1], 8;" ::"r"(dst + 8), "l"(a.Told + sn.y) : "memory");
            asm volatile("cp.async.ca.shared.global [%0], [%1], 8;" ::"r"(dst + 16), "l"(a.Told + sn.z) : "memory");
            asm volatile("cp.async.ca.shared.global [%0], [%1], 8;" ::"r"(dst + 24), "l"(a.Told + sn.w) : "memory");
        }
        asm volatile("cp.async.commit_group;" ::: "memory");
        // phase 1: H = enthalpy(T) per slot (blocked.hpp:462-467) from the streamed slot temperatures
        const uint8_t* sinfo = B + L.sinfo;
        for (int s = tid; s < ns; s += kTileThreads) {
            const double T = sT[s];
            sTH[s] = make_double2(T, (CF_PRB(a) & 15) == 5 ? T : dev_enthalpy<TDEP>(P, sMat[sinfo[s] & 0x3f], T));
        }
        __syncthreads();
        if (pending_border && tid == 0) border_done();  // every thread's fenced flush precedes the barrier
        pending_border = false;

        // phase 2a: elements (element_accumulate fem.hpp:57-70). Stored layout: the element's
        // four (lump, rc_q) pairs go over its own consumed geometry pairs (columns 0..3);
        // coordinates layout: lump / rc columns of the shared-memory scratch R
        const int S = L.ne2;
        double* R = (double*)(smem + a.scratch_off);  // coordinates layout only
        const uint8_t* ereg = B + L.region;
        const uint8_t* gblob = a.blob + hdr[stage].boff;  // this tile's blob in global memory
        // the tile's section offsets in registers for the whole element loop (the layout lives in
        // shared memory, which the loop's contribution stores may alias)
        const ushort4* connp = (const ushort4*)(B + L.conn);
        const double2* G2p = (const double2*)(B + L.geom);
        const uint8_t* metail = gblob + L.bytes;
        for (int i = tid; i < ((CF_PRB(a) & 15) == 4 ? 0 : ne); i += kTileThreads) {
            double g[4][3], vol, max_edge = 0;
            const ushort4 cn = connp[i];
            CF_ASSERT(cn.x < ns && cn.y < ns && cn.z < ns && cn.w < ns);
            if (GC) {
                const double2* X = (const double2*)(B + L.xyz);  // slot (x, y) (z, 0)
                const unsigned short sl[4] = {cn.x, cn.y, cn.z, cn.w};
                double p[4][3];
#pragma unroll
                for (int k = 0; k < 4; ++k) {
                    const double2 xy = X[2 * sl[k]], z0 = X[2 * sl[k] + 1];
                    p[k][0] = xy.x;
                    p[k][1] = xy.y;
                    p[k][2] = z0.x;
                }
                dev_tet_grads(p, g, vol);
                max_edge = ((const double*)(B + L.geom))[i];
            } else {
                const double2* G2 = G2p;
                const double2 c0 = G2[i], c1 = G2[S + i], c2 = G2[2 * S + i], c3 = G2[3 * S + i],
                              c4 = G2[4 * S + i];
                g[1][0] = c0.x;
                g[1][1] = c0.y;
                g[1][2] = c1.x;
                g[2][0] = c1.y;
                g[2][1] = c2.x;
                g[2][2] = c2.y;
                g[3][0] = c3.x;
                g[3][1] = c3.y;
                g[3][2] = c4.x;
                vol = c4.y;
#pragma unroll
                for (int c = 0; c < 3; ++c) g[0][c] = ((g[1][c] + g[2][c]) + g[3][c]) * -1.0;
            }
            const double2 th0 = sTH[cn.x], th1 = sTH[cn.y], th2 = sTH[cn.z], th3 = sTH[cn.w];
            const double T[4] = {th0.x, th1.x, th2.x, th3.x};
            const double H[4] = {th0.y, th1.y, th2.y, th3.y};
            const DevMaterial& m = sMat[ereg[i]];
            double lump, rc[4];
            dev_element<TDEP, !GC>(
                P, m, g, vol, [&]() { return GC ? max_edge : __ldg((const double*)metail + i); },
                T, H, lump, rc, (CF_PRB(a) & 15) == 7);
            if (TDEP)
                local_min = fmin(local_min, dev_stable_bound<TDEP>(P, m, ((const double*)(B + L.minedge))[i], T));
            if (GC) {
                R[L.lump_idx(i)] = lump;
#pragma unroll
                for (int c = 0; c < 4; ++c) R[L.rc_idx(i, c)] = rc[c];
            } else {
                double2* W = (double2*)B;
#pragma unroll
                for (int c = 0; c < 4; ++c) W[c * S + i] = make_double2(lump, rc[c]);  // L.pair_elem(i, c)
            }
        }
        // phase 2b: facets (facet_flux_accumulate fem.hpp:74-79; interface blocked.hpp:485-490);
        // terms stored negated (the reduction does r -= v for every entry: r - (-f) == r + f
        // exactly): stored layout as (0.0, -term_a) pairs over the facet's own consumed record,
        // coordinates layout into the scratch's facet-term columns
        for (int i = tid; i < nf; i += kTileThreads) {
            const double2* rec = (const double2*)(B + L.fac + 48 * i);  // (area, slots+kind), sisters
            const double2 rec0 = rec[0];
            const double area = rec0.x;
            const long long fb = __double_as_longlong(rec0.y);
            const ushort4 fs = make_ushort4((unsigned short)fb, (unsigned short)(fb >> 16), (unsigned short)(fb >> 32),
                                            (unsigned short)(fb >> 48));
            const DevFacetKind& K = P->kind[fs.w];
            CF_ASSERT(fs.x < ns && fs.y < ns && fs.z < ns);
            const double ts[3] = {sT[fs.x], sT[fs.y], sT[fs.z]};
            double q, h, tinf;
            if (K.interface) {
                const double var = K.var == CF_VAR_TIME ? time : (ts[0] + ts[1] + ts[2]) / 3.0;
                q = 0.0;
                h = dev_pl_eval(P, K.htab, var);
                // interface_ambient from the PRE-update T of the previous step (refresh_ambient lag),
                // gathered before phase 1 (this thread's cp.async group)
                asm volatile("cp.async.wait_all;" ::: "memory");
                const double2 t01 = rec[1], t23 = rec[2];
                double sum = 0;
                sum += t01.x;
                sum += t01.y;
                sum += t23.x;
                sum += t23.y;
                tinf = 0.25 * sum;
            } else {
                q = K.q;
                h = K.h;
                tinf = K.t_inf;
            }
            const double third = area / 3.0;
            const double f0 = third * (-q + h * (tinf - ts[0]));
            const double f1 = third * (-q + h * (tinf - ts[1]));
            const double f2 = third * (-q + h * (tinf - ts[2]));
            if (GC) {
                R[L.fac_idx(i, 0)] = -f0;
                R[L.fac_idx(i, 1)] = -f1;
                R[L.fac_idx(i, 2)] = -f2;
            } else {
                double2* W = (double2*)B;
                W[L.pair_facet(i, 0)] = make_double2(0.0, -f0);
                W[L.pair_facet(i, 1)] = make_double2(0.0, -f1);
                W[L.pair_facet(i, 2)] = make_double2(0.0, -f2);
            }
        }
        __syncthreads();

        // the next tile's slot temperatures, gathered into the other buffer while this tile reduces
        // and its blob streams in (after phase 2b: the facet threads' wait_all there covers only
        // the ambient gathers)
        if (gather) {
            const int t_iss = s_issue;
            if (t_iss < a.n_tiles) {
                int4 d0, d1;
                load_desc(a, t_iss, d0, d1);
                gather_slot_T<kTileThreads>(a, d0, d1, TDEP, GC, (k & 1) ? sT0 : sT1, tid);
            } else {
                asm volatile("cp.async.commit_group;" ::: "memory");
            }
        }
        // the next tile of this CTA into L2 while this one reduces: its bulk copy, issued after the
        // reduction, then reads L2 instead of waiting out the DRAM latency. Issued by the last warp,
        // whose reduction lists are the shortest (sperm), not by warp 0 on the critical path; the
        // descriptor is read from global memory (L2-hot: thread 0 staged it at the tile's start)
        if (a.l2_next && tid == kTileThreads - 32 && s_issue < a.n_tiles) {
            int4 d0, d1;
            load_desc(a, s_issue, d0, d1);
            const TileMeta tm{d0.x, d0.y, d0.z, d0.w};
            const int64_t boff = (int64_t)(uint32_t)d1.z | (int64_t)d1.w << 32;
            const uint8_t* src = a.blob + boff;
            for (int32_t o = 0; o < d1.y; o += (int32_t)kBulkChunk)
                bulk_prefetch_l2(src + o, (uint32_t)(d1.y - o < (int32_t)kBulkChunk ? d1.y - o : kBulkChunk));
            const uint32_t tbytes = 8u * (uint32_t)cf_round32(tm.ns, 2);
            if (tbytes && a.Tslot) bulk_prefetch_l2(a.Tslot + d1.x, tbytes);
        }
        // phase 3: per-slot fixed-order reduction (ascending element, then facets) + flush,
        // through the slot's 16-bit operand codes (cf_tileblob.hpp)
        const uint16_t* cend = (const uint16_t*)(B + L.csr_end);
        const uint16_t* sperm = (const uint16_t*)(B + L.sperm);
        const uint16_t* csr = (const uint16_t*)(B + L.csr);
        const int32_t* snode = (const int32_t*)(B + L.snode);
        const double2* W = (const double2*)B;
        // per-slot reduction (reads the tile's shared memory) ...
        auto reduce = [&](int s, double& c, double& r) {
            const int beg = s == 0 ? 0 : cend[s - 1];
            const int end = cend[s];
            CF_ASSERT(s < ns && beg <= end && (end - beg) % 4 == 0);
            c = 0;
            r = 0;
            for (int j = beg; j < end; j += 4) {  // lists padded to 4 with exact (0.0, 0.0) no-ops
                const uint2 pr = *(const uint2*)(csr + j);
                const uint32_t v[4] = {pr.x & 0xffffu, pr.x >> 16, pr.y & 0xffffu, pr.y >> 16};
                CF_ASSERT(GC || (v[0] < (uint32_t)(L.bytes >> 4) && v[1] < (uint32_t)(L.bytes >> 4) &&
                                 v[2] < (uint32_t)(L.bytes >> 4) && v[3] < (uint32_t)(L.bytes >> 4)));
                double l[4], q[4];
                if (GC) {
                    const int32_t rz = L.r_zero, rl = L.r_lump;
#pragma unroll
                    for (int k = 0; k < 4; ++k) {
                        const bool op = v[k] & 0x8000u;
                        const int li = rl + (int)(v[k] & 0x3ffu);
                        l[k] = R[op ? rz : li];
                        q[k] = R[op ? (int)(v[k] & 0x7fffu) : li + ((int)(v[k] >> 10) + 1) * S];
                    }
                } else {
#pragma unroll
                    for (int k = 0; k < 4; ++k) {
                        const double2 w = W[(CF_PRB(a) & 15) == 8 ? ((v[k] & ~7u) | (s & 7)) : v[k]];
                        l[k] = w.x;
                        q[k] = w.y;
                    }
                }
#pragma unroll
                for (int k = 0; k < 4; ++k) {
                    c += l[k];
                    r -= q[k];
                }
            }
        };
        // ... and its flush (global memory only, so it may follow the next tile's copy issue)
        auto flush = [&](int s, double c, double r, int info, int32_t node, double Ts) {
            CF_ASSERT(node >= 0 && node < a.n_local && (int64_t)s0 + s < a.n_slots);
            if (FUSE && (info & 0x80)) {
                // tile-private node: its merge is the identity, update it now
                double Tn;
                if (done) {
                    Tn = Ts;
                } else {
                    const int dir = (DIR && (info & 0x40)) ? a.node_dir[node] : -1;
                    Tn = node_update<DIR, CLAMP>(P, a.st, Ts, c, r, dt, t_next, dir, info & 0x3f,
                                                 a.local_global + node, clamped);
                }
                a.Tn[node] = Tn;
                if (!gather) a.Tslot_n[s0 + s] = Tn;
            } else if (DET) {
                a.part[s0 + s] = make_double2(c, r);
            } else {
                atomicAdd(&a.acc[node].x, c);  // both REDs land in the node's one sector
                atomicAdd(&a.acc[node].y, r);
            }
        };
        // the first slot of every thread keeps its result in registers and flushes after the next
        // tile's copy is issued; further slots (tiles of > 128 slots) flush inline
        const int nred = (CF_PRB(a) & 15) == 3 ? 0 : ns;
        constexpr int KD = 1;
        double kc[KD], kr[KD], kT[KD];
        int ks[KD], kinfo[KD];
        int32_t knode[KD];
        bool kv[KD];
#pragma unroll
        for (int k = 0; k < KD; ++k) {
            const int j = tid + k * kTileThreads;
            kv[k] = j < nred;
            if (kv[k]) {
                const int sl = sperm[j];  // threads take slots by list length (similar trip counts per warp)
                ks[k] = sl;
                reduce(sl, kc[k], kr[k]);
                kinfo[k] = sinfo[sl];
                knode[k] = snode[sl];
                kT[k] = sT[sl];
            }
        }
        for (int j = tid + KD * kTileThreads; j < nred; j += kTileThreads) {
            const int sl = sperm[j];
            double c, r;
            reduce(sl, c, r);
            flush(sl, c, r, sinfo[sl], snode[sl], sT[sl]);
        }
        const int t_issue = s_issue;  // written before the phase-1 barrier
        const int t_nxt = dyn ? t_issue : t_follow;
        if (t_nxt < a.n_tiles) {
            __syncthreads();  // stage buffer and sT/sH free again; s_issue read by every thread
            if (tid == 0 && t_issue < a.n_tiles) {
                // generic-proxy writes to B (in-place contributions) must be ordered
                // before the async-proxy (TMA) overwrite of the same buffer
                asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
                staged_desc(ndesc, nd0, nd1, gather);
                issue_tile_copy(a, nd0, nd1, TDEP, GC, B, sT, &bar[stage], &hdr[stage]);
            }
        }
#pragma unroll
        for (int k = 0; k < KD; ++k)
            if (kv[k]) flush(ks[k], kc[k], kr[k], kinfo[k], knode[k], kT[k]);
        if (t < a.n_border) {  // partials of a border tile: visible device-wide before it is counted
            __threadfence();
            pending_border = true;
        }
        if (t_nxt >= a.n_tiles) break;  // last tile of this CTA: no trailing barrier
        t = t_nxt;
    }
    if (pending_border) {
        __syncthreads();
        if (tid == 0) border_done();
    }
    if (TDEP) {
        for (int o = 16; o > 0; o >>= 1) local_min = fmin(local_min, __shfl_xor_sync(0xffffffffu, local_min, o));
        if ((tid & 31) == 0) atomic_min_pos(&a.st->min_bound[a.st->step_index & 1], local_min);
    }
    if (CLAMP && clamped) a.st->clamp_flag = 1;
}

// ------------------------------------------------------------------ update kernel
struct UpdArgs {
    int32_t n_list, n_local, n_ghost;
    int64_t n_slots;      // bounds (CF_BOUNDS builds)
    int64_t n_recv;       // bounds: doubles in one parity of the receive buffer
    int32_t probe;        // diagnostics only (CF_PROBE; results invalid): 8 = no slot-copy writes,
                          // 9 = no partial reads
    const int32_t* list;  // nodes to merge + update (NULL: all local nodes)
    const int4* rec;      // packed per listed node: {node, count, slot0, slot1}, {slot2 .. slot5}
                          // (count > 8: slots via merge_off/merge_idx); NULL: use list + merge CSR
    const int2* rec2;     // per listed node: {slot6, slot7} (tile corners of structured meshes)
    const double* T;      // current (ghost slots written here)
    double* Tn;           // next
    const int32_t* merge_off;
    const int32_t* merge_idx;
    const double2* part;
    double2* acc;
    const int8_t* node_dir;
    const uint8_t* node_region;
    const int32_t* local_global;
    // multi-rank
    const int32_t* node_shared;
    const int32_t* shared_off;
    const int32_t* shared_src_c;
    const int32_t* shared_src_r;
    const double* recv;
    const int32_t* ghost_src;
    double* Tcur_w;  // == T, writable (ghost slots)
    double* Tslot_n; // next per-slot T copies (every slot of an updated node)
    const DevParams* P;
    DevState* st;
    double t_end;
};

template <bool DET>
__device__ __forceinline__ void own_partial(const UpdArgs& a, int i, double& c, double& r) {
    if (DET) {
        c = 0;
        r = 0;
        for (int j = a.merge_off[i]; j < a.merge_off[i + 1]; ++j) {
            const double2 pr = a.part[a.merge_idx[j]];
            c += pr.x;
            r += pr.y;
        }
    } else {
        const double2 v = a.acc[i];
        c = v.x;
        r = v.y;
    }
}

template <bool DET, bool MULTI, bool DIR, bool CLAMP, bool TDEP>
__global__ void __launch_bounds__(256) update_kernel(UpdArgs a) {
    const DevParams* __restrict__ P = a.P;
    griddep_wait();  // the tile kernel's partials / private updates are complete and visible
    double dt, t_next;
    bool done;
    step_dt<TDEP>(P, a.st, a.t_end, dt, t_next, done);
    int clamped = 0;
    const int stride = gridDim.x * blockDim.x;
    for (int k = blockIdx.x * blockDim.x + threadIdx.x; k < a.n_list; k += stride) {
        int i, cnt = -1;
        int4 r0, r1;
        int2 r2 = make_int2(0, 0);
        if (a.rec) {  // coalesced records: node + up to 8 slot (= partial) indices
            r0 = __ldg(a.rec + 2 * k);
            r1 = __ldg(a.rec + 2 * k + 1);
            i = r0.x;
            cnt = r0.y;
            if (cnt > 6) r2 = __ldg(a.rec2 + k);
        } else {
            i = a.list ? a.list[k] : k;
        }
        const int sl[8] = {r0.z, r0.w, r1.x, r1.y, r1.z, r1.w, r2.x, r2.y};
        const bool packed = cnt >= 0 && cnt <= 8;
        CF_ASSERT(i >= 0 && i < a.n_local);
#pragma unroll
        for (int q = 0; q < 8; ++q) CF_ASSERT(!packed || q >= cnt || (sl[q] >= 0 && sl[q] < a.n_slots));
        const double T = __ldg(a.T + i);
        if (done) {
            if (!DET) {  // the tile kernel still accumulated this (no-op) step: drop it
                a.acc[i] = make_double2(0.0, 0.0);
            }
            a.Tn[i] = T;
            if (!a.Tslot_n) continue;
            if (packed) {
#pragma unroll
                for (int q = 0; q < 8; ++q)
                    if (q < cnt) a.Tslot_n[sl[q]] = T;
            } else {
                for (int j = a.merge_off[i]; j < a.merge_off[i + 1]; ++j) a.Tslot_n[a.merge_idx[j]] = T;
            }
            continue;
        }
        double c, r;
        if (DET && packed) {
            // all partial loads issued before the in-order (ascending tile) sums
            double2 pr[8];
#pragma unroll
            for (int q = 0; q < 8; ++q) pr[q] = (q < cnt && CF_PRB(a) != 9) ? __ldg(a.part + sl[q]) : make_double2(1.0, 0.0);
            c = 0;
            r = 0;
#pragma unroll
            for (int q = 0; q < 8; ++q)
                if (q < cnt) {
                    c += pr[q].x;
                    r += pr[q].y;
                }
        } else {
            own_partial<DET>(a, i, c, r);
        }
        if (!DET) {
            a.acc[i] = make_double2(0.0, 0.0);
        }
        if (MULTI) {
            const int32_t sh = a.node_shared[i];
            double ct = 0, rt = 0;
            if (sh >= 0) {
                for (int j = a.shared_off[sh]; j < a.shared_off[sh + 1]; ++j) {
                    const int32_t sc = a.shared_src_c[j];
                    if (sc < 0) {
                        ct += c;
                        rt += r;
                    } else {
                        CF_ASSERT(sc < a.n_recv && a.shared_src_r[j] >= 0 && a.shared_src_r[j] < a.n_recv);
                        ct += a.recv[sc];
                        rt += a.recv[a.shared_src_r[j]];
                    }
                }
            } else {
                ct += c;
                rt += r;
            }
            c = ct;
            r = rt;
        }
        const double Tn = node_update<DIR, CLAMP>(P, a.st, T, c, r, dt, t_next, DIR ? a.node_dir[i] : -1,
                                                  CLAMP ? a.node_region[i] : 0, a.local_global + i, clamped);
        a.Tn[i] = Tn;
        if (CF_PRB(a) == 8 || !a.Tslot_n) continue;
        if (packed) {
#pragma unroll
            for (int q = 0; q < 8; ++q)
                if (q < cnt) a.Tslot_n[sl[q]] = Tn;
        } else {
            for (int j = a.merge_off[i]; j < a.merge_off[i + 1]; ++j) a.Tslot_n[a.merge_idx[j]] = Tn;
        }
    }
    if (MULTI)
        for (int g = blockIdx.x * blockDim.x + threadIdx.x; g < a.n_ghost; g += stride) {
            CF_ASSERT(a.ghost_src[g] >= 0 && a.ghost_src[g] < a.n_recv);
            a.Tcur_w[a.n_local + g] = a.recv[a.ghost_src[g]];
        }
    if (CLAMP && clamped) a.st->clamp_flag = 1;
}

// advances the step state after the update (a separate one-warp launch: the update's CTAs
// exit without a grid-wide ticket; every kernel of the step has read the state by then)
template <bool TDEP>
__global__ void advance_kernel(DevState* st, const DevParams* __restrict__ P, double t_end, int32_t* sched) {
    griddep_wait();
    if (threadIdx.x != 0) return;
    if (sched)  // the tile kernel's scheduling tickets (one counter per launch class) restart every step
        for (int c = 0; c < 4; ++c) sched[c] = 0;
    double dt, t_next;
    bool done;
    step_dt<TDEP>(P, st, t_end, dt, t_next, done);
    if (!done) {
        const int par = (int)(st->step_index & 1);
        st->time = t_next;
        st->dt = dt;
        st->step_index += 1;
        if (st->clamp_flag) st->clamp_steps += 1;
        st->min_bound[par ^ 1] = 0x7ff0000000000000ull;
    } else {
        st->done = 1;
    }
    st->clamp_flag = 0;
}

// ------------------------------------------------------------------ plan upload (device-side packing)
struct FillArgs {
    const TileMeta* meta;
    const int64_t* blob_off;
    const int64_t* rest_off;
    const uint8_t* rest;          // host-packed [conn, bytes) sections, staged on the device
    const int64_t* elem_off;
    const int32_t* tets_ord;      // oriented tets, local node ids, tile order
    const double* coords;         // local node coordinates
    const int32_t* slot_off;
    const int32_t* slot_node;
    uint8_t* blob;
    bool tdep, coords_layout;
};

// one CTA per tile: the staged sections into place, then the geometry (stored: the five
// 16-byte pair columns g1 g2 g3 vol + the max_edge tail; coordinates: slot xyz + max_edge),
// min_edge for dynamic dt
__global__ void __launch_bounds__(128) fill_tiles_kernel(FillArgs f) {
    const int t = blockIdx.x;
    const TileMeta tm = f.meta[t];
    const TileLayout L(tm, f.tdep, f.coords_layout);
    uint8_t* B = f.blob + f.blob_off[t];
    const uint8_t* stg = f.rest + f.rest_off[t];
    const int S = L.ne2;
    const int4* src = (const int4*)stg;
    int4* dst = (int4*)(B + L.stage);
    for (int j = threadIdx.x; j < (L.bytes - L.stage) / 16; j += blockDim.x) dst[j] = src[j];
    __syncthreads();  // the minedge section (dynamic dt) lies in the copied range
    const int64_t e0 = f.elem_off[t];
    for (int i = threadIdx.x; i < S; i += blockDim.x) {
        double g[4][3], vol = 0, mn = 0, mx = 0;
        if (i < tm.ne) {
            double p[4][3];
#pragma unroll
            for (int a = 0; a < 4; ++a) {
                const int32_t l = f.tets_ord[4 * (e0 + i) + a];
#pragma unroll
                for (int k = 0; k < 3; ++k) p[a][k] = f.coords[3 * (int64_t)l + k];
            }
            dev_tet_geometry(p, g, vol, mn, mx);
        } else {
#pragma unroll
            for (int a = 0; a < 4; ++a) g[a][0] = g[a][1] = g[a][2] = 0.0;
        }
        if (f.coords_layout) {
            ((double*)(B + L.geom))[i] = mx;
        } else {
            double2* G2 = (double2*)(B + L.geom);
            G2[i] = make_double2(g[1][0], g[1][1]);
            G2[S + i] = make_double2(g[1][2], g[2][0]);
            G2[2 * S + i] = make_double2(g[2][1], g[2][2]);
            G2[3 * S + i] = make_double2(g[3][0], g[3][1]);
            G2[4 * S + i] = make_double2(g[3][2], vol);
            *(double*)(B + L.max_edge_of(i)) = mx;  // uncopied tail
        }
        if (f.tdep) ((double*)(B + L.minedge))[i] = mn;
    }
    if (f.coords_layout) {
        double* xyz = (double*)(B + L.xyz);
        const int s0 = f.slot_off[t];
        for (int k = threadIdx.x; k < tm.ns; k += blockDim.x) {
            const int32_t l = f.slot_node[s0 + k] & 0x0fffffff;
            xyz[4 * k] = f.coords[3 * (int64_t)l];
            xyz[4 * k + 1] = f.coords[3 * (int64_t)l + 1];
            xyz[4 * k + 2] = f.coords[3 * (int64_t)l + 2];
            xyz[4 * k + 3] = 0.0;
        }
    }
}

// ------------------------------------------------------------------ pack kernel
// Peer-memory transport (NVLink / NVSwitch P2P; CUDA IPC between the rank processes): every rank
// owns one exported window = [control block | receive buffer x 2 step parities]. The control block
// holds, per sending rank, the payload flag (the sender's exchange sequence number), the flag of
// the scalar reductions and their 2-parity value slots.
constexpr int kPeerMaxNbrs = 32;
constexpr int kPeerMaxWorld = 64;
constexpr int kPeerXflagOff = 0;      // u32[kPeerMaxWorld]: payload of exchange #seq from rank q has landed
constexpr int kPeerRflagOff = 256;    // u32[kPeerMaxWorld]: reduction #seq operands of rank q have landed
constexpr int kPeerRedOff = 512;      // u64[2 parities][kPeerMaxWorld][2]
constexpr int kPeerCtrlBytes = 4096;  // the receive buffer starts here

struct PeerPack {
    int32_t n_nbrs;
    uint32_t seq;                      // this exchange's sequence number (1, 2, ...)
    unsigned* ticket;                  // CTAs done (last one raises the flags)
    int64_t send_off[kPeerMaxNbrs + 1];  // payload offsets per neighbour (the send-buffer layout)
    double* dst[kPeerMaxNbrs];         // the neighbour's receive region for this rank, this step's parity
    uint32_t* flag[kPeerMaxNbrs];      // the neighbour's payload flag for this rank
};

struct PackArgs {
    int32_t n_cr, n_t;
    const int32_t* cr_node;  // local ids
    const int64_t* cr_dst;   // c offset
    const int64_t* cr_dst_r; // r offset
    const int32_t* t_node;
    const int64_t* t_dst;
    const double* T;
    double* send;
    UpdArgs u;               // merge inputs
    PeerPack pp;             // peer-memory transport only
};

// PEER: exchange_and_merge's send half fused with the pack -- each value is stored
// straight into the neighbour's receive buffer over NVLink, and the last CTA to finish raises this
// rank's flag in every neighbour's control block (release at system scope after every CTA's
// system-scope fence), on which the neighbour's stream waits before its update.
template <bool DET, bool PEER>
__global__ void __launch_bounds__(256) pack_kernel(PackArgs a) {
    const int stride = gridDim.x * blockDim.x;
    auto out = [&](int64_t off) -> double* {
        if (!PEER) return a.send + off;
        CF_ASSERT(off >= 0 && off < a.pp.send_off[a.pp.n_nbrs]);  // inside this rank's payload layout
        int k = 0;
        while (k + 1 < a.pp.n_nbrs && off >= a.pp.send_off[k + 1]) ++k;
        return a.pp.dst[k] + (off - a.pp.send_off[k]);
    };
    for (int j = blockIdx.x * blockDim.x + threadIdx.x; j < a.n_cr + a.n_t; j += stride) {
        if (j < a.n_cr) {
            double c, r;
            CF_ASSERT(a.cr_node[j] >= 0 && a.cr_node[j] < a.u.n_local);
            own_partial<DET>(a.u, a.cr_node[j], c, r);
            *out(a.cr_dst[j]) = c;
            *out(a.cr_dst_r[j]) = r;
        } else {
            const int k = j - a.n_cr;
            *out(a.t_dst[k]) = a.T[a.t_node[k]];
        }
    }
    if (PEER) {
        __threadfence_system();
        __syncthreads();
        if (threadIdx.x == 0) {
            const unsigned done = atomicAdd(a.pp.ticket, 1u);
            if (done == gridDim.x - 1) {
                *a.pp.ticket = 0;
                __threadfence_system();
                for (int k = 0; k < a.pp.n_nbrs; ++k) st_release_sys(a.pp.flag[k], a.pp.seq);
            }
        }
    }
}

// Scalar all-reduce over the peer windows (dynamic dt: min of the per-step bound, blocked.hpp:477-480;
// clamp flag: max, :526-534; series T min / max, :678-681). put: this rank's operands into its slot
// of every other rank's control block + flag; the stream then waits for every rank's flag; get:
// combine the slots of this rank's own block. Slots alternate by sequence parity: a rank can be at
// most one reduction ahead of any other (it waited for everyone's previous operands).
struct PeerRed {
    int32_t world, rank;
    uint32_t seq;
    uint8_t* const* win;  // [world] window bases as mapped in this process (own included)
};
enum { kPeerMin = 0, kPeerMax = 1 };

template <class V>
__global__ void peer_put_kernel(PeerRed pr, const V* src, int n) {
    const int q = threadIdx.x;
    if (q >= pr.world || q == pr.rank) return;
    unsigned long long* slot = (unsigned long long*)(pr.win[q] + kPeerRedOff) +
                               (((size_t)(pr.seq & 1) * kPeerMaxWorld + pr.rank) * 2);
    for (int k = 0; k < n; ++k) slot[k] = (unsigned long long)src[k];
    __threadfence_system();
    st_release_sys((uint32_t*)(pr.win[q] + kPeerRflagOff) + pr.rank, pr.seq);
}

template <class V>
__global__ void peer_get_kernel(PeerRed pr, V* dst, int n, int op0, int op1) {
    if (threadIdx.x >= n) return;
    const int k = threadIdx.x;
    const int op = k == 0 ? op0 : op1;
    unsigned long long v = (unsigned long long)dst[k];
    const volatile unsigned long long* base = (const volatile unsigned long long*)(pr.win[pr.rank] + kPeerRedOff) +
                                              (size_t)(pr.seq & 1) * kPeerMaxWorld * 2;
    for (int q = 0; q < pr.world; ++q) {
        if (q == pr.rank) continue;
        const unsigned long long w = base[q * 2 + k];
        v = op == kPeerMin ? (w < v ? w : v) : (w > v ? w : v);
    }
    dst[k] = (V)v;
}

// global-order host field -> rank-local T ring (all 3 buffers) and slot copies
__global__ void scatter_init_kernel(int32_t n_nodes, const int32_t* local_global, const double* Tg, double* T0,
                                    double* T1, double* T2) {
    for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < n_nodes; i += gridDim.x * blockDim.x) {
        const double v = Tg[local_global[i]];
        T0[i] = v;
        T1[i] = v;
        T2[i] = v;
    }
}
__global__ void slot_init_kernel(int64_t n_slots, const int32_t* slot_node, const double* T, double* S0, double* S1) {
    for (int64_t s = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; s < n_slots; s += (int64_t)gridDim.x * blockDim.x) {
        const int32_t sn = slot_node[s];
        const double v = sn >= 0 ? T[(uint32_t)sn & 0x0fffffffu] : 0.0;
        S0[s] = v;
        S1[s] = v;
    }
}
// rank-local T (and H = enthalpy(T)) -> global order (blocked.hpp:686-691)
template <bool TDEP>
__global__ void gather_fields_kernel(int32_t n, const int32_t* local_global, const double* T, const uint8_t* reg,
                                     const DevParams* P, double* Tg, double* Hg) {
    for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < n; i += gridDim.x * blockDim.x) {
        const int32_t g = local_global[i];
        const double t = T[i];
        if (Tg) Tg[g] = t;
        if (Hg) Hg[g] = dev_enthalpy<TDEP>(P, P->mat[reg[i]], t);
    }
}

// H = enthalpy(T) per local node (output only)
template <bool TDEP>
__global__ void enthalpy_kernel(int32_t n, const double* T, const uint8_t* reg, const DevParams* P, double* H) {
    for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < n; i += gridDim.x * blockDim.x)
        H[i] = dev_enthalpy<TDEP>(P, P->mat[reg[i]], T[i]);
}

}  // namespace cfb
