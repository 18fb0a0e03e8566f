// cf_tileblob.hpp — byte layout of one tile (cache block) in HBM.
//
// Every tile's element, facet and reduction data is one contiguous,
// 16-byte-aligned blob so the tile kernel fetches it with a single TMA bulk
// copy (cp.async.bulk) into shared memory. Sections (each 16 B aligned):
//   geom      11 x ne2 f64   SoA: g1x g1y g1z g2x g2y g2z g3x g3y g3z vol max_edge
//   conn      ne2 x ushort4  tile-local slots of the 4 nodes
//   minedge   ne2 f64        (only with temperature-dependent tables: dynamic dt)
//   farea     nf2 f64        facet area
//   fsister   nf x int4      sister-element nodes (local / ghost ids) of interface facets
//   fslots    nf2 x ushort4  facet slots s0 s1 s2 + facet kind
//   snode     ns4 i32        local node id of each slot (flush target)
//   csr_end   ns8 u16        per-slot end of its contribution list (tile relative)
//   csr       ncsr8 u16      contribution codes: 4*e+a (elements), 4*ne+4*f+a (facets)
//   sinfo     ns16 u8        region | 0x40 Dirichlet | 0x80 tile-private node
//   region    ne16 u8        element region
//   zero      16 B           0.0 (c-operand of facet entries in the slot reduction)
// The slots' current temperatures are NOT in the blob: they live in a per-slot
// copy Tslot[s0 .. s0+ns) (ping-ponged per step, written by the update of the
// previous step) fetched by a second bulk copy, so no tile ever gathers T.
// (nX = n rounded up to a multiple of X.) Host packing (cf_plan.cpp) and the
// device view (cf_kernels.cuh) both use TileLayout, so they cannot disagree.
#pragma once

#include <cstdint>

#ifdef __CUDACC__
#define CF_HD __host__ __device__ __forceinline__
#else
#define CF_HD inline
#endif

namespace cfb {

struct TileMeta {
    int32_t ne, ns, nf, ncsr;
};

CF_HD int64_t cf_round(int64_t n, int64_t m) { return (n + m - 1) & ~(m - 1); }  // m: power of two

struct TileLayout {
    int64_t geom, conn, minedge, farea, fsister, fslots, snode, csr_end, csr, sinfo, region, zero, bytes;
    int32_t ne2;  // SoA stride of geom
    CF_HD TileLayout(const TileMeta& m, bool tdep) {
        ne2 = (int32_t)cf_round(m.ne, 2);
        const int64_t nf2 = cf_round(m.nf, 2);
        int64_t o = 0;
        geom = o;
        o += 11 * 8 * (int64_t)ne2;
        conn = o;
        o += 8 * (int64_t)ne2;
        minedge = o;
        if (tdep) o += 8 * (int64_t)ne2;
        farea = o;
        o += 8 * nf2;
        fsister = o;
        o += 16 * (int64_t)m.nf;
        fslots = o;
        o += 8 * nf2;
        snode = o;
        o += 4 * cf_round(m.ns, 4);
        csr_end = o;
        o += 2 * cf_round(m.ns, 8);
        csr = o;
        o += 2 * cf_round(m.ncsr, 8);
        sinfo = o;
        o += cf_round(m.ns, 16);
        region = o;
        o += cf_round(m.ne, 16);
        zero = o;  // 16 zero bytes: the "lump" operand of facet entries in the reduction
        o += 16;
        bytes = o;
    }
};

}  // namespace cfb
