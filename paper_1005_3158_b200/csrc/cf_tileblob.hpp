// cf_tileblob.hpp — byte layout of one tile (cache block) in HBM.
//
// Every tile's element, facet and reduction data is one contiguous,
// 16-byte-aligned blob so the tile kernel fetches it with a single TMA bulk
// copy (cp.async.bulk) into shared memory. Sections (each 16 B aligned):
//   xyz       ns x 4 f64     slot coordinates (x, y, z, 0)       [CF_GEOM_COORDS only]
//   geom      11 x ne2 f64   SoA: g1x g1y g1z g2x g2y g2z g3x g3y g3z vol max_edge
//                            [CF_GEOM_COORDS: max_edge only, 1 x ne2 f64]
//   conn      ne2 x ushort4  tile-local slots of the 4 nodes
//   minedge   ne2 f64        (only with temperature-dependent tables: dynamic dt)
//   farea     nf2 f64        facet area
//   fsister   nf x int4      sister-element nodes (local / ghost ids) of interface facets
//   fslots    nf2 x ushort4  facet slots s0 s1 s2 + facet kind
//   snode     ns4 i32        local node id of each slot (flush target)
//   csr_end   ns8 u16        per-slot end of its contribution list (tile relative)
//   csr       ncsr4 u32      contribution pairs (lump index | residual index << 16), double
//                            indices from the operand base R (see TileLayout::lump_idx ...);
//                            each slot's list padded to a multiple of 4 with (0.0, 0.0) pairs
//   sinfo     ns16 u8        region | 0x40 Dirichlet | 0x80 tile-private node
//   region    ne16 u8        element region
//   zero      16 B           0.0 (c-operand of facet entries in the slot reduction)
// The element phase writes its (lump, rc0..rc3) contribution columns over the
// consumed geometry columns (stored layout) or into a shared-memory scratch that
// is never streamed (coordinates layout).
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
    int32_t ne, ns, nf, ncsr;  // ncsr: padded contribution entries
};

struct alignas(16) TileDesc {  // one tile of a launch: metadata + slot offset + blob byte offset
    TileMeta tm;
    int32_t s0, pad;
    int64_t blob_off;
};

CF_HD int64_t cf_round(int64_t n, int64_t m) { return (n + m - 1) & ~(m - 1); }  // m: power of two
CF_HD int32_t cf_round32(int32_t n, int32_t m) { return (n + m - 1) & ~(m - 1); }

struct TileLayout {
    // byte offsets (a tile is at most ~220 KB: 32-bit offsets keep the kernel's registers down)
    int32_t geom, xyz, conn, minedge, farea, fsister, fslots, snode, csr_end, csr, sinfo, region, zero, bytes;
    int32_t ne2, nf2;  // SoA strides (elements, facets)
    bool coords;
    // Reduction operands, as double indices from the tile's operand base R (the stage
    // blob for the stored layout, the shared-memory scratch for the coordinates layout):
    //   zero, lump(e), rc(e, q), facet term(f, a)  -- precomputed into the CSR pairs
    int32_t r_zero, r_lump;
    int32_t scratch;   // coordinates layout: scratch doubles (zero pair, 5 x ne2, 3 x nf2)
    CF_HD int32_t lump_idx(int e) const { return r_lump + e; }
    CF_HD int32_t rc_idx(int e, int q) const { return r_lump + (1 + q) * ne2 + e; }
    CF_HD int32_t fac_idx(int f, int a) const {
        if (coords) return r_lump + 5 * ne2 + a * nf2 + f;
        return a == 0 ? (farea >> 3) + f : (fsister >> 3) + 2 * f + a - 1;
    }
    CF_HD TileLayout(const TileMeta& m, bool tdep, bool coords_) : coords(coords_) {
        ne2 = cf_round32(m.ne, 2);
        nf2 = cf_round32(m.nf, 2);
        int32_t o = 0;
        geom = xyz = o;
        if (coords) {
            o += 32 * m.ns;  // slot (x, y, z, 0)
            geom = o;                 // max_edge only
            o += 8 * ne2;
        } else {
            o += 11 * 8 * ne2;
        }
        conn = o;
        o += 8 * ne2;
        minedge = o;
        if (tdep) o += 8 * ne2;
        farea = o;
        o += 8 * nf2;
        fsister = o;
        o += 16 * m.nf;
        fslots = o;
        o += 8 * nf2;
        snode = o;
        o += 4 * cf_round32(m.ns, 4);
        csr_end = o;
        o += 2 * cf_round32(m.ns, 8);
        csr = o;
        o += 4 * cf_round32(m.ncsr, 4);
        sinfo = o;
        o += cf_round32(m.ns, 16);
        region = o;
        o += cf_round32(m.ne, 16);
        zero = o;  // 16 zero bytes: the "lump" operand of facet entries in the reduction
        o += 16;
        bytes = o;
        r_zero = coords ? 0 : (zero >> 3);
        r_lump = coords ? 2 : (geom >> 3);
        scratch = coords ? 2 + 5 * ne2 + 3 * (int32_t)nf2 : 0;
    }
};

}  // namespace cfb
