// cf_tileblob.hpp — byte layout of one tile (cache block) in HBM.
//
// Every tile's element, facet and reduction data is one contiguous,
// 16-byte-aligned blob so the tile kernel fetches it with a single TMA bulk
// copy (cp.async.bulk) into shared memory. Sections (each 16 B aligned):
//   CF_GEOM_STORED (default):
//   geom      5 x ne8 x 16 B SoA of 16-byte pairs, one pair per element per column:
//                            (g1x g1y) (g1z g2x) (g2y g2z) (g3x g3y) (g3z vol)
//   conn      ne8 x ushort4  tile-local slots of the 4 nodes
//   (max_edge is not streamed: the degeneracy test bounds it by 1/|g1| and reads the exact
//    value, ne8 f64 in an uncopied tail after `bytes`, only when that bound cannot decide)
//   CF_GEOM_COORDS:
//   xyz       ns x 4 f64     slot coordinates (x, y, z, 0)
//   geom      ne2 f64        max_edge
//   conn      ne2 x ushort4  tile-local slots of the 4 nodes
//   both:
//   minedge   ne2 f64        (only with temperature-dependent tables: dynamic dt)
//   fac       nf x 48 B      per facet: (area f64, slots s0 s1 s2 + kind as ushort4),
//                            sister-element nodes (local / ghost ids) as int4, 16 B pad
//   snode     ns4 i32        local node id of each slot (flush target)
//   csr_end   ns8 u16        per-slot end of its contribution list (tile relative)
//   sperm     ns8 u16        phase-3 thread order: thread j reduces slot sperm[j] (slots sorted by
//                            list length; the slots themselves are private first, then shared by
//                            node id)
//   csr       ncsr8 u16      per-slot contribution codes in reduction order (see below); each
//                            slot's list padded to a multiple of 4 with the zero operand
//   sinfo     ns16 u8        region | 0x40 Dirichlet | 0x80 tile-private node
//   region    ne16 u8        element region
//   zero      16 B           (0.0, 0.0)
// Reduction operands. Stored layout: the element phase writes each element's four
// (lump, rc_q) pairs over its own consumed geometry pairs (column q), each facet's three
// (0.0, -term_a) pairs over its own consumed 48-byte record, so a code is simply the
// 16-byte pair index from the blob base (one 16-byte load per contribution).
// Coordinates layout: lump / rc / facet terms go to a shared-memory scratch of doubles
// (zero pair, lump column, 4 rc columns, 3 facet-term columns); a code is e | q << 10 for an
// element contribution (operands lump[e], rc_q[e]) or 0x8000 | the residual operand's
// double index (lump operand: the zero) for a facet term or padding.
// The slots' current temperatures are NOT in the blob: they live in a per-slot
// copy Tslot[s0 .. s0+ns) (ping-ponged per step, written by the update of the
// previous step) fetched by a second bulk copy, so no tile ever gathers T.
// (nX = n rounded up to a multiple of X.) Host packing (cf_plan.cpp) and the
// device view (cf_kernels.cuh) both use TileLayout, so they cannot disagree.
// Host staging (cf_plan.cpp -> fill_tiles_kernel) holds the sections [conn, bytes) verbatim;
// the geometry (and the stored layout's max_edge tail) is computed on the device.
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

struct alignas(16) TileDesc {  // one tile of a launch: metadata + slot offset + blob bytes + offset
    TileMeta tm;
    int32_t s0, bytes;  // bytes: TileLayout(tm).bytes (the copy is issued before the layout is built)
    int64_t blob_off;
};

CF_HD int64_t cf_round(int64_t n, int64_t m) { return (n + m - 1) & ~(m - 1); }  // m: power of two
CF_HD int32_t cf_round32(int32_t n, int32_t m) { return (n + m - 1) & ~(m - 1); }

struct TileLayout {
    // byte offsets (a tile is at most ~220 KB: 32-bit offsets keep the kernel's registers down)
    int32_t geom, xyz, conn, minedge, fac, snode, csr_end, sperm, csr, sinfo, region, zero, bytes;
    int32_t stage;     // first byte of the host-staged part (= conn)
    int32_t total;     // bytes in HBM: `bytes` (copied to shared memory) + the stored layout's
                       // uncopied max_edge tail (ne2 f64 at offset `bytes`)
    int32_t ne2;       // SoA stride (elements)
    int32_t nf;
    bool coords;
    int32_t r_zero, r_lump;  // reduction operand indices (stored: 16 B pairs; coords: scratch doubles)
    int32_t scratch;   // coordinates layout: scratch doubles (zero pair, 5 x ne2, 3 x nf2)
    // stored layout: pair index of (lump, rc_q) of element e / (0, -term_a) of facet f
    CF_HD int32_t pair_elem(int e, int q) const { return q * ne2 + e; }
    CF_HD int32_t pair_facet(int f, int a) const { return (fac >> 4) + 3 * f + a; }
    // coordinates layout: scratch double indices
    CF_HD int32_t lump_idx(int e) const { return r_lump + e; }
    CF_HD int32_t rc_idx(int e, int q) const { return r_lump + (1 + q) * ne2 + e; }
    CF_HD int32_t fac_idx(int f, int a) const { return r_lump + 5 * ne2 + a * cf_round32(nf, 2) + f; }
    // 16-bit reduction code of element e corner q / facet f corner a / the padding no-op
    CF_HD uint16_t code_elem(int e, int q) const {
        return coords ? (uint16_t)(e | q << 10) : (uint16_t)pair_elem(e, q);
    }
    CF_HD uint16_t code_facet(int f, int a) const {
        return coords ? (uint16_t)(0x8000 | fac_idx(f, a)) : (uint16_t)pair_facet(f, a);
    }
    CF_HD uint16_t code_zero() const { return coords ? (uint16_t)(0x8000 | r_zero) : (uint16_t)r_zero; }
    // largest operand index a code carries (must stay below 0x8000)
    CF_HD int32_t max_operand() const {
        return coords ? fac_idx(nf, 2) : (bytes >> 4);
    }
    CF_HD TileLayout(const TileMeta& m, bool tdep, bool coords_) : coords(coords_) {
        ne2 = cf_round32(m.ne, coords ? 2 : 8);  // stored: pair columns 8-aligned (bank groups, cf_plan.cpp)
        nf = m.nf;
        int32_t o = 0;
        geom = xyz = conn = o;
        if (coords) {
            o += 32 * m.ns;  // slot (x, y, z, 0)
            geom = o;        // max_edge only
            o += 8 * ne2;
            conn = o;
            o += 8 * ne2;
        } else {
            o += 5 * 16 * ne2;
            conn = o;
            o += 8 * ne2;
        }
        minedge = o;
        stage = conn;
        if (tdep) o += 8 * ne2;
        fac = o;
        o += 48 * m.nf;
        snode = o;
        o += 4 * cf_round32(m.ns, 4);
        csr_end = o;
        o += 2 * cf_round32(m.ns, 8);
        sperm = o;
        o += 2 * cf_round32(m.ns, 8);
        csr = o;
        o += 2 * cf_round32(m.ncsr, 8);
        sinfo = o;
        o += cf_round32(m.ns, 16);
        region = o;
        o += cf_round32(m.ne, 16);
        zero = o;  // 16 zero bytes
        o += 16;
        bytes = o;
        total = coords ? bytes : bytes + 8 * ne2;
        r_zero = coords ? 0 : (zero >> 4);
        r_lump = coords ? 2 : 0;
        scratch = coords ? 2 + 5 * ne2 + 3 * cf_round32(m.nf, 2) : 0;
    }
    // byte offsets of element i's connectivity (ushort4), its exact max_edge (stored layout: in the
    // uncopied tail) and of facet f's record fields
    CF_HD int32_t conn_of(int i) const { return conn + 8 * i; }
    CF_HD int32_t max_edge_of(int i) const { return coords ? geom + 8 * i : bytes + 8 * i; }
    CF_HD int32_t fac_area(int f) const { return fac + 48 * f; }
    CF_HD int32_t fac_slots(int f) const { return fac + 48 * f + 8; }
    CF_HD int32_t fac_sister(int f) const { return fac + 48 * f + 16; }
    // bytes of the host staging of this tile, and the staging offset of a blob offset >= stage
    CF_HD int32_t staged_bytes() const { return bytes - stage; }
    CF_HD int32_t stage_of(int32_t off) const { return off - stage; }
};

}  // namespace cfb
