// cf_kernels.cuh — sm_100a kernels of the castfem explicit step.
//
// One step (blocked_step blocked.hpp:542-550) is:
//   tile_kernel    assemble_blocks (blocked.hpp:454-498): one CTA per tile (the
//                  paper's cache block); gathers the tile's nodal T into shared
//                  memory, derives H = enthalpy(T) once per tile slot, runs the
//                  element physics (Lemmon C_app, lumped capacitance, conduction
//                  residual) and the facet fluxes (convective + interface with the
//                  one-step-lagged sister ambient read from the previous T buffer),
//                  then reduces each slot's contributions in a fixed order through
//                  a tile-local CSR — no shared-memory fp64 atomics (those are CAS
//                  loops on sm_100a). Flush: deterministic mode writes per-(tile,
//                  slot) partials; atomic mode stores tile-private nodes and
//                  fp64-REDs tile-shared ones.
//   pack_kernel    (multi-rank) shared-node partials + pre-update T of external
//                  nodes into the per-neighbour send buffer.
//   update_kernel  merge_blocks (:502-515) + update_fields (:519-538): per node,
//                  ascending-tile merge of partials (or the RED accumulators),
//                  ascending-rank combine for shared nodes, T += (dt*r)/c,
//                  Dirichlet overwrite, clamp flag; the last CTA advances time.
#pragma once

#include <cuda_runtime.h>

#include <cstdint>

#include "cf_physics.cuh"

namespace cfb {

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

struct TileArgs {
    const int32_t* tile_elem_off;
    const int32_t* tile_slot_off;
    const int64_t* tile_csr_off;
    const int32_t* tile_facet_off;
    const ushort4* conn;
    const uint8_t* ereg;
    const double* geom;  // [11][E]
    const double* min_edge;
    int64_t E;
    const int32_t* slot_node;
    const uint8_t* slot_info;
    const uint16_t* slot_csr_end;
    const uint16_t* csr;
    const ushort4* fslots;
    const double* farea;
    const int4* fsister;
    const double* T;     // current
    const double* Told;  // previous step (ambient lag)
    double* part_c;
    double* part_r;
    double* acc_c;
    double* acc_r;
    const DevParams* P;
    DevState* st;
    int max_slots, max_elems, max_facets;
};

__device__ __forceinline__ void atomic_min_pos(unsigned long long* addr, double v) {
    atomicMin(addr, (unsigned long long)__double_as_longlong(v));
}

template <bool DET, bool TDEP>
__global__ void __launch_bounds__(256) tile_kernel(TileArgs a) {
    extern __shared__ double smem[];
    const int t = blockIdx.x;
    const int tid = threadIdx.x;
    const int e0 = a.tile_elem_off[t];
    const int ne = a.tile_elem_off[t + 1] - e0;
    const int s0 = a.tile_slot_off[t];
    const int ns = a.tile_slot_off[t + 1] - s0;
    const int f0 = a.tile_facet_off[t];
    const int nf = a.tile_facet_off[t + 1] - f0;
    const int64_t c0 = a.tile_csr_off[t];
    const DevParams* __restrict__ P = a.P;

    double* sT = smem;
    double* sH = sT + a.max_slots;
    double* sl = sH + a.max_slots;          // lump per element
    double* sr = sl + a.max_elems;          // rc[4][max_elems]
    double* sf = sr + 4 * a.max_elems;      // facet terms [3*nf]

    // phase 1: gather T, derive H per slot (H is always enthalpy(T): blocked.hpp:427,529)
    for (int s = tid; s < ns; s += blockDim.x) {
        const int32_t node = a.slot_node[s0 + s];
        const double T = a.T[node];
        const int reg = a.slot_info[s0 + s] & 0x7f;
        sT[s] = T;
        sH[s] = dev_enthalpy<TDEP>(P, P->mat[reg], T);
    }
    __syncthreads();

    // phase 2a: elements
    double local_min = __longlong_as_double(0x7ff0000000000000ll);
    for (int i = tid; i < ne; i += blockDim.x) {
        const int64_t p = (int64_t)e0 + i;
        const ushort4 cn = a.conn[p];
        const int reg = a.ereg[p];
        double g[4][3];
#pragma unroll
        for (int k = 0; k < 3; ++k) {
            g[1][k] = a.geom[(int64_t)k * a.E + p];
            g[2][k] = a.geom[(int64_t)(3 + k) * a.E + p];
            g[3][k] = a.geom[(int64_t)(6 + k) * a.E + p];
        }
        const double vol = a.geom[9 * a.E + p];
        const double max_edge = a.geom[10 * a.E + p];
#pragma unroll
        for (int k = 0; k < 3; ++k) g[0][k] = ((g[1][k] + g[2][k]) + g[3][k]) * -1.0;
        const double T[4] = {sT[cn.x], sT[cn.y], sT[cn.z], sT[cn.w]};
        const double H[4] = {sH[cn.x], sH[cn.y], sH[cn.z], sH[cn.w]};
        const DevMaterial& m = P->mat[reg];
        double lump, rc[4];
        dev_element<TDEP>(P, m, g, vol, max_edge, T, H, lump, rc);
        sl[i] = lump;
#pragma unroll
        for (int k = 0; k < 4; ++k) sr[k * a.max_elems + i] = rc[k];
        if (TDEP) local_min = fmin(local_min, dev_stable_bound<TDEP>(P, m, a.min_edge[p], T));
    }
    // phase 2b: facets (facet_flux_accumulate fem.hpp:74-79; interface blocked.hpp:485-490)
    const double time = a.st->time;
    for (int i = tid; i < nf; i += blockDim.x) {
        const ushort4 fs = a.fslots[f0 + i];
        const DevFacetKind& K = P->kind[fs.w];
        const double ts[3] = {sT[fs.x], sT[fs.y], sT[fs.z]};
        double q, h, tinf;
        if (K.interface) {
            const double var = K.var == CF_VAR_TIME ? time : (ts[0] + ts[1] + ts[2]) / 3.0;
            q = 0.0;
            h = dev_pl_eval(P, K.htab, var);
            const int4 sn = a.fsister[f0 + i];
            // interface_ambient / refresh_ambient from the PRE-update T of the previous step
            double sum = 0;
            sum += a.Told[sn.x];
            sum += a.Told[sn.y];
            sum += a.Told[sn.z];
            sum += a.Told[sn.w];
            tinf = 0.25 * sum;
        } else {
            q = K.q;
            h = K.h;
            tinf = K.t_inf;
        }
        const double third = a.farea[f0 + i] / 3.0;
#pragma unroll
        for (int k = 0; k < 3; ++k) sf[3 * i + k] = third * (-q + h * (tinf - ts[k]));
    }
    if (TDEP) {
        // block min then one atomic per CTA
        for (int o = 16; o > 0; o >>= 1) local_min = fmin(local_min, __shfl_xor_sync(0xffffffffu, local_min, o));
        if ((tid & 31) == 0) atomic_min_pos(&a.st->min_bound[a.st->step_index & 1], local_min);
    }
    __syncthreads();

    // phase 3: per-slot fixed-order reduction (ascending element, then facets)
    const int e4 = 4 * ne;
    for (int s = tid; s < ns; s += blockDim.x) {
        const int beg = s == 0 ? 0 : a.slot_csr_end[s0 + s - 1];
        const int end = a.slot_csr_end[s0 + s];
        double c = 0, r = 0;
        for (int j = beg; j < end; ++j) {
            const int code = a.csr[c0 + j];
            if (code < e4) {
                const int e = code >> 2;
                c += sl[e];
                r -= sr[(code & 3) * a.max_elems + e];
            } else {
                r += sf[code - e4];
            }
        }
        if (DET) {
            a.part_c[s0 + s] = c;
            a.part_r[s0 + s] = r;
        } else {
            const int32_t node = a.slot_node[s0 + s];
            if (a.slot_info[s0 + s] & 0x80) {
                a.acc_c[node] = c;
                a.acc_r[node] = r;
            } else {
                atomicAdd(&a.acc_c[node], c);
                atomicAdd(&a.acc_r[node], r);
            }
        }
    }
}

struct UpdArgs {
    int32_t n_local, n_ghost;
    const double* T;   // current (ghost slots written here)
    double* Tn;        // next
    const int32_t* merge_off;
    const int32_t* merge_idx;
    const double* part_c;
    const double* part_r;
    double* acc_c;
    double* acc_r;
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
    double* Tcur_w;    // == T, writable (ghost slots)
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
            const int32_t s = a.merge_idx[j];
            c += a.part_c[s];
            r += a.part_r[s];
        }
    } else {
        c = a.acc_c[i];
        r = a.acc_r[i];
    }
}

template <bool DET, bool MULTI, bool DIR, bool CLAMP, bool TDEP>
__global__ void __launch_bounds__(256) update_kernel(UpdArgs a) {
    const DevParams* __restrict__ P = a.P;
    const double time = a.st->time;
    double dt = TDEP ? __longlong_as_double((long long)a.st->min_bound[a.st->step_index & 1]) * P->dt_safety
                     : P->static_dt;
    bool done = false;
    if (a.t_end > 0) {
        const double remaining = a.t_end - time;
        if (!(time < a.t_end)) done = true;
        if (remaining > 0) dt = dt < remaining ? dt : remaining;
    }
    const double t_next = time + dt;
    int clamped = 0;
    const int stride = gridDim.x * blockDim.x;
    for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < a.n_local; i += stride) {
        const double T = a.T[i];
        if (done) {
            a.Tn[i] = T;
            continue;
        }
        double c, r;
        own_partial<DET>(a, i, c, r);
        if (!DET) {
            a.acc_c[i] = 0;
            a.acc_r[i] = 0;
        }
        if (MULTI) {
            const int32_t sh = a.node_shared[i];
            if (sh >= 0) {
                double ct = 0, rt = 0;
                for (int j = a.shared_off[sh]; j < a.shared_off[sh + 1]; ++j) {
                    const int32_t sc = a.shared_src_c[j];
                    if (sc < 0) {
                        ct += c;
                        rt += r;
                    } else {
                        ct += a.recv[sc];
                        rt += a.recv[a.shared_src_r[j]];
                    }
                }
                c = ct;
                r = rt;
            } else {
                c = 0 + c;
                r = 0 + r;
            }
        }
        double Tn;
        if (!(c > 0)) {
            atomicMin(&a.st->err_node, a.local_global[i]);
            Tn = T;
        } else {
            Tn = T + dt * r / c;
        }
        if (DIR) {
            const int d = a.node_dir[i];
            if (d >= 0) Tn = dev_pl_eval(P, P->dir_tab[d], t_next);
        }
        if (CLAMP) {
            const DevMaterial& m = P->mat[a.node_region[i]];
            if (Tn < m.range_lo || Tn > m.range_hi) clamped = 1;
        }
        a.Tn[i] = Tn;
    }
    if (MULTI)
        for (int g = blockIdx.x * blockDim.x + threadIdx.x; g < a.n_ghost; g += stride)
            a.Tcur_w[a.n_local + g] = a.recv[a.ghost_src[g]];
    if (CLAMP && clamped) a.st->clamp_flag = 1;
    // last CTA advances the step state (all CTAs have read it by then)
    __shared__ bool last;
    __syncthreads();
    if (threadIdx.x == 0) {
        __threadfence();
        const unsigned int tk = atomicAdd(&a.st->ticket, 1u);
        last = tk == gridDim.x - 1;
    }
    __syncthreads();
    if (last && threadIdx.x == 0) {
        __threadfence();
        DevState* s = a.st;
        if (!done) {
            const int par = (int)(s->step_index & 1);
            s->time = t_next;
            s->dt = dt;
            s->step_index += 1;
            if (s->clamp_flag) s->clamp_steps += 1;
            s->min_bound[par ^ 1] = 0x7ff0000000000000ull;
        } else {
            s->done = 1;
        }
        s->clamp_flag = 0;
        s->ticket = 0;
        __threadfence();
    }
}

struct PackArgs {
    int32_t n_cr, n_t;
    const int32_t* cr_node;  // local ids
    const int64_t* cr_dst;   // c offset; r at cr_dst_r
    const int64_t* cr_dst_r;
    const int32_t* t_node;
    const int64_t* t_dst;
    const double* T;
    double* send;
    UpdArgs u;               // merge inputs
};

template <bool DET>
__global__ void __launch_bounds__(256) pack_kernel(PackArgs a) {
    const int stride = gridDim.x * blockDim.x;
    for (int j = blockIdx.x * blockDim.x + threadIdx.x; j < a.n_cr + a.n_t; j += stride) {
        if (j < a.n_cr) {
            double c, r;
            own_partial<DET>(a.u, a.cr_node[j], c, r);
            a.send[a.cr_dst[j]] = c;
            a.send[a.cr_dst_r[j]] = r;
        } else {
            const int k = j - a.n_cr;
            a.send[a.t_dst[k]] = a.T[a.t_node[k]];
        }
    }
}

// H = enthalpy(T) per local node (output only)
template <bool TDEP>
__global__ void enthalpy_kernel(int32_t n, const double* T, const uint8_t* reg, const DevParams* P, double* H) {
    for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < n; i += gridDim.x * blockDim.x)
        H[i] = dev_enthalpy<TDEP>(P, P->mat[reg[i]], T[i]);
}

}  // namespace cfb
