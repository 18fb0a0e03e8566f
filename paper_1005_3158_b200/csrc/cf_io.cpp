// cf_io.cpp — the text formats either side of the step:
//   femesh 1 mesh       parse_mesh / write_mesh      mesh.hpp:256-343
//   solver config       parse_config                 material.hpp:186-345
//   partmap             load_partmap / write_partmap partition.hpp:424-449
//   binary mesh         this repo's fast path for large meshes (same validation as parse_mesh)
// Same lexical rules ('#' comments, whitespace-separated words, blank lines skipped,
// 1-based line numbers), the same number syntax (std::from_chars), the same
// section semantics and defaults, and the same error classes and messages (the first
// defect in file order, as a sequential reader would meet it):
// CF_PARSE "line N: ..." for syntax, CF_VALIDATION "mesh validation failed: ..."
// for a mesh finalize_mesh rejects, CF_CONFIG for table / material checks.
// Structure (this repo's own): the buffer is indexed into logical lines once; the mesh parser
// plans its sections from the header lines, converts every section's records in parallel (OpenMP)
// and numbers the tags in a last ordered pass (1.6 M tets of text: 0.16 s, the reference's stream
// reader 3.7 s); the config grammar is a table of sections and keys, each key with its assignment.
#include <algorithm>
#include <cctype>
#include <charconv>
#include <cstdio>
#include <cstring>
#include <iterator>
#include <map>
#include <memory>
#include <mutex>
#include <string>
#include <string_view>
#include <vector>

#include "cf_internal.hpp"

namespace cfb {
namespace {

// ---- text front end ------------------------------------------------------------------------
// The buffer is indexed once into its logical lines (comment cut at '#', blank lines dropped,
// physical line numbers kept). The parsers work on that index: the mesh parser plans its sections
// from the header lines alone (a section's records are the next N logical lines) and then converts
// the record lines of every section in parallel; the first defect in file order is the one
// reported, with the line number the reference's sequential reader would report.
struct LogicalLine {
    const char* b;
    const char* e;  // [b, e): comment removed; may still carry blanks at either end
    long no;        // 1-based physical line number
};

inline bool blank(char c) { return std::isspace((unsigned char)c) != 0; }

struct LineIndex {
    std::vector<LogicalLine> lines;
    long physical = 0;  // physical lines in the buffer: what an end-of-input error reports
    explicit LineIndex(std::string_view text) {
        const char* p = text.data();
        const char* const end = p + text.size();
        while (p < end) {
            const char* nl = (const char*)std::memchr(p, '\n', (size_t)(end - p));
            const char* stop = nl ? nl : end;
            ++physical;
            if (const char* hash = (const char*)std::memchr(p, '#', (size_t)(stop - p))) stop = hash;
            const char* q = p;
            while (q < stop && blank(*q)) ++q;
            if (q < stop) lines.push_back(LogicalLine{q, stop, physical});
            p = nl ? nl + 1 : end;
        }
    }
};

// whitespace-separated words of a logical line: stores up to cap of them, returns how many there are
int words(const LogicalLine& L, std::string_view* out, int cap) {
    int n = 0;
    for (const char* p = L.b; p < L.e;) {
        while (p < L.e && blank(*p)) ++p;
        const char* q = p;
        while (q < L.e && !blank(*q)) ++q;
        if (q > p) {
            if (n < cap) out[n] = std::string_view(p, (size_t)(q - p));
            ++n;
        }
        p = q;
    }
    return n;
}

[[noreturn]] void parse_fail(const std::string& what, long line) {
    raise(CF_PARSE, "line " + std::to_string(line) + ": " + what);
}

template <class T>
T number(std::string_view t, long line, const char* kind) {
    T v{};
    const auto r = std::from_chars(t.data(), t.data() + t.size(), v);
    if (r.ec != std::errc{} || r.ptr != t.data() + t.size())
        parse_fail(std::string("expected ") + kind + ", got '" + std::string(t) + "'", line);
    return v;
}
double to_double(std::string_view t, long line) { return number<double>(t, line, "a number"); }
long to_long(std::string_view t, long line) { return number<long>(t, line, "an integer"); }

void append_g17(std::string& s, double v) {
    char b[40];
    const int n = std::snprintf(b, sizeof b, "%.17g", v);
    s.append(b, (size_t)n);
}

// The earliest defect in file order wins, whichever pass or thread met it.
struct FirstDefect {
    size_t at = SIZE_MAX;  // position in the line index (lines.size() = end of input)
    Error err{CF_OK, ""};
    std::mutex mu;
    void offer(size_t where, const Error& e) {
        std::lock_guard<std::mutex> g(mu);
        if (where < at) {
            at = where;
            err = e;
        }
    }
    void rethrow() const {
        if (at != SIZE_MAX) throw err;
    }
};

}  // namespace

// ------------------------------------------------------------------ mesh
struct TextMesh {
    std::vector<double> coords;
    std::vector<int32_t> tets, region, facets, facet_tag, contacts;
    std::vector<std::string> tags;
    std::vector<const char*> tag_ptrs;
    cf_mesh_desc desc{};
    int32_t tag_id(std::string_view name) {  // first use numbers a tag (Mesh::add_tag mesh.hpp:62-67)
        const auto it = std::find(tags.begin(), tags.end(), name);
        if (it != tags.end()) return (int32_t)(it - tags.begin());
        tags.emplace_back(name);
        return (int32_t)tags.size() - 1;
    }
    void make_desc() {
        tag_ptrs.clear();
        for (const auto& t : tags) tag_ptrs.push_back(t.c_str());
        desc = cf_mesh_desc{(int32_t)(coords.size() / 3), coords.data(),   (int32_t)region.size(), tets.data(),
                            region.data(),                 (int32_t)facet_tag.size(), facets.data(),
                            facet_tag.data(),              (int32_t)tags.size(),      tag_ptrs.data(),
                            (int32_t)(contacts.size() / 2), contacts.data()};
    }
};

namespace {
// the femesh record sections (mesh.hpp:256-262): keyword, words per record, and the reference's messages
struct RecordKind {
    const char* keyword;
    int fields;
    const char* usage;
    const char* cut_short;
    const char* shape;
};
constexpr RecordKind kRecordKinds[] = {
    {"nodes", 3, "usage: nodes N", "unexpected end of node list", "node line needs 'x y z'"},
    {"tets", 5, "usage: tets M", "unexpected end of element list", "element line needs 'n0 n1 n2 n3 region'"},
    {"facets", 4, "usage: facets B", "unexpected end of facet list", "facet line needs 'n0 n1 n2 tag'"},
};
enum { kNodes = 0, kTets = 1, kFacets = 2, kContact = 3 };

struct Section {   // one header line and the logical lines it owns
    int kind;      // kNodes .. kContact
    size_t first;  // contact: the header line itself; records: the first record line
    size_t count;  // records present (a list cut short by the end of input keeps what is there)
    size_t base;   // index of its first record in the mesh arrays
};
}  // namespace

std::unique_ptr<TextMesh> parse_mesh_text(std::string_view text) {
    const LineIndex idx(text);
    const auto& L = idx.lines;
    std::string_view w[6];
    if (L.empty() || words(L[0], w, 6) != 2 || w[0] != "femesh" || w[1] != "1")
        parse_fail("expected header 'femesh 1'", L.empty() ? idx.physical : L[0].no);

    // pass 1: the section plan, from the header lines alone
    FirstDefect defect;
    std::vector<Section> plan;
    size_t totals[3] = {0, 0, 0};
    for (size_t i = 1; i < L.size();) {
        try {
            const int nw = words(L[i], w, 6);
            if (w[0] == "contact") {
                if (nw != 3) parse_fail("usage: contact tagA tagB", L[i].no);
                plan.push_back(Section{kContact, i, 0, 0});
                ++i;
                continue;
            }
            int kind = -1;
            for (int k = 0; k < 3; ++k)
                if (w[0] == kRecordKinds[k].keyword) kind = k;
            if (kind < 0) parse_fail("unknown section '" + std::string(w[0]) + "'", L[i].no);
            if (nw != 2) parse_fail(kRecordKinds[kind].usage, L[i].no);
            const long n = to_long(w[1], L[i].no);
            if (n < 0) raise(CF_INVALID_ARG, "line " + std::to_string(L[i].no) + ": negative count");
            const size_t have = std::min<size_t>((size_t)n, L.size() - (i + 1));
            plan.push_back(Section{kind, i + 1, have, totals[kind]});
            totals[kind] += have;
            if (have < (size_t)n) {  // reported only if every record that is there converts
                defect.offer(L.size(), Error(CF_PARSE, "line " + std::to_string(idx.physical) + ": " +
                                                           kRecordKinds[kind].cut_short));
                break;
            }
            i += 1 + have;
        } catch (const Error& e) {
            defect.offer(i, e);
            break;
        }
    }

    // pass 2: the records of every planned section, converted in parallel
    auto m = std::make_unique<TextMesh>();
    m->coords.resize(3 * totals[kNodes]);
    m->tets.resize(4 * totals[kTets]);
    m->region.resize(totals[kTets]);
    m->facets.resize(3 * totals[kFacets]);
    std::vector<std::string_view> facet_word(totals[kFacets]);
    for (const Section& sec : plan) {
        if (sec.kind == kContact) continue;
        const RecordKind& rk = kRecordKinds[sec.kind];
        const int64_t n = (int64_t)sec.count;
#pragma omp parallel for schedule(static) if (n > 4096)
        for (int64_t r = 0; r < n; ++r) {
            const LogicalLine& rec = L[sec.first + (size_t)r];
            const size_t o = sec.base + (size_t)r;
            try {
                std::string_view f[6];
                if (words(rec, f, 6) != rk.fields) parse_fail(rk.shape, rec.no);
                if (sec.kind == kNodes) {
                    for (int k = 0; k < 3; ++k) m->coords[3 * o + k] = to_double(f[k], rec.no);
                } else if (sec.kind == kTets) {
                    for (int k = 0; k < 4; ++k) m->tets[4 * o + k] = (int32_t)to_long(f[k], rec.no);
                    m->region[o] = (int32_t)to_long(f[4], rec.no);
                } else {
                    for (int k = 0; k < 3; ++k) m->facets[3 * o + k] = (int32_t)to_long(f[k], rec.no);
                    facet_word[o] = f[3];
                }
            } catch (const Error& e) {
                defect.offer(sec.first + (size_t)r, e);
            }
        }
    }
    defect.rethrow();

    // pass 3: tags numbered by first appearance in file order, over facet records and contact lines
    m->facet_tag.resize(totals[kFacets]);
    for (const Section& sec : plan) {
        if (sec.kind == kFacets) {
            for (size_t r = 0; r < sec.count; ++r) m->facet_tag[sec.base + r] = m->tag_id(facet_word[sec.base + r]);
        } else if (sec.kind == kContact) {
            words(L[sec.first], w, 6);
            m->contacts.push_back(m->tag_id(w[1]));
            m->contacts.push_back(m->tag_id(w[2]));
        }
    }
    m->make_desc();
    // the mesh must pass finalize_mesh (validation + orientation), as parse_mesh requires (mesh.hpp:318-322)
    MeshData md;
    try {
        finalize_mesh(&m->desc, md);
    } catch (const Error& e) {
        raise(CF_VALIDATION, std::string("mesh validation failed: ") + e.what());
    }
    std::memcpy(m->tets.data(), md.tets.data(), sizeof(int32_t) * m->tets.size());  // oriented
    return m;
}

std::string format_mesh(const cf_mesh_desc* d) {  // write_mesh mesh.hpp:327-343
    std::string s = "femesh 1\nnodes " + std::to_string(d->n_nodes) + "\n";
    for (int64_t i = 0; i < d->n_nodes; ++i) {
        for (int k = 0; k < 3; ++k) {
            if (k) s.push_back(' ');
            append_g17(s, d->coords[3 * i + k]);
        }
        s.push_back('\n');
    }
    s += "tets " + std::to_string(d->n_elems) + "\n";
    for (int64_t e = 0; e < d->n_elems; ++e) {
        for (int k = 0; k < 4; ++k) s += std::to_string(d->tets[4 * e + k]) + " ";
        s += std::to_string(d->region[e]) + "\n";
    }
    auto tag = [&](int32_t t) -> std::string {
        if (t < 0 || t >= d->n_tags) raise(CF_INVALID_ARG, "tag index out of range");
        return d->tags[t];
    };
    if (d->n_facets > 0) {
        s += "facets " + std::to_string(d->n_facets) + "\n";
        for (int64_t f = 0; f < d->n_facets; ++f) {
            for (int k = 0; k < 3; ++k) s += std::to_string(d->facets[3 * f + k]) + " ";
            s += tag(d->facet_tag[f]) + "\n";
        }
    }
    for (int64_t c = 0; c < d->n_contacts; ++c)
        s += "contact " + tag(d->contacts[2 * c]) + " " + tag(d->contacts[2 * c + 1]) + "\n";
    return s;
}

// ------------------------------------------------------------------ binary mesh (fast path)
// "CFMESHB1" | i64 N E F n_tags n_contacts | f64 coords[3N] | i32 tets[4E] region[E]
// facets[3F] facet_tag[F] contacts[2C] | per tag: i32 length + bytes. Little-endian.
namespace {
constexpr char kMagic[8] = {'C', 'F', 'M', 'E', 'S', 'H', 'B', '1'};
}

std::string mesh_binary(const cf_mesh_desc* d) {
    std::string s(kMagic, 8);
    auto put = [&](const void* p, size_t n) { s.append((const char*)p, n); };
    const int64_t hdr[5] = {d->n_nodes, d->n_elems, d->n_facets, d->n_tags, d->n_contacts};
    put(hdr, sizeof hdr);
    put(d->coords, 24 * (size_t)d->n_nodes);
    put(d->tets, 16 * (size_t)d->n_elems);
    put(d->region, 4 * (size_t)d->n_elems);
    put(d->facets, 12 * (size_t)d->n_facets);
    put(d->facet_tag, 4 * (size_t)d->n_facets);
    put(d->contacts, 8 * (size_t)d->n_contacts);
    for (int32_t t = 0; t < d->n_tags; ++t) {
        const int32_t n = (int32_t)std::strlen(d->tags[t]);
        put(&n, 4);
        put(d->tags[t], (size_t)n);
    }
    return s;
}

std::unique_ptr<TextMesh> parse_mesh_binary(std::string_view b) {
    size_t pos = 0;
    auto take = [&](void* dst, size_t n) {
        if (b.size() - pos < n) raise(CF_PARSE, "binary mesh truncated at byte " + std::to_string(pos));
        if (n) std::memcpy(dst, b.data() + pos, n);
        pos += n;
    };
    char magic[8];
    if (b.size() < 8) raise(CF_PARSE, "binary mesh: missing header");
    take(magic, 8);
    if (std::memcmp(magic, kMagic, 8) != 0) raise(CF_PARSE, "binary mesh: bad magic (expected CFMESHB1)");
    int64_t h[5];
    take(h, sizeof h);
    for (int k = 0; k < 5; ++k)
        if (h[k] < 0 || h[k] > INT32_MAX) raise(CF_PARSE, "binary mesh: bad count in header");
    // the fixed-size sections the header announces must be present before anything is allocated
    // (counts <= INT32_MAX: the byte total fits in 64 bits); tags add at least 4 bytes each
    const uint64_t need = 24ull * (uint64_t)h[0] + 20ull * (uint64_t)h[1] + 16ull * (uint64_t)h[2] +
                          4ull * (uint64_t)h[3] + 8ull * (uint64_t)h[4];
    if (need > b.size() - pos) raise(CF_PARSE, "binary mesh truncated at byte " + std::to_string(b.size()));
    auto m = std::make_unique<TextMesh>();
    m->coords.resize(3 * (size_t)h[0]);
    m->tets.resize(4 * (size_t)h[1]);
    m->region.resize((size_t)h[1]);
    m->facets.resize(3 * (size_t)h[2]);
    m->facet_tag.resize((size_t)h[2]);
    m->contacts.resize(2 * (size_t)h[4]);
    take(m->coords.data(), 8 * m->coords.size());
    take(m->tets.data(), 4 * m->tets.size());
    take(m->region.data(), 4 * m->region.size());
    take(m->facets.data(), 4 * m->facets.size());
    take(m->facet_tag.data(), 4 * m->facet_tag.size());
    take(m->contacts.data(), 4 * m->contacts.size());
    for (int64_t t = 0; t < h[3]; ++t) {
        int32_t n = 0;
        take(&n, 4);
        if (n < 0) raise(CF_PARSE, "binary mesh: bad tag length");
        std::string tag((size_t)n, '\0');
        take(tag.data(), (size_t)n);
        m->tags.push_back(tag);
    }
    if (pos != b.size()) raise(CF_PARSE, "binary mesh: trailing bytes");
    for (int32_t v : m->facet_tag)
        if (v < 0 || v >= (int32_t)m->tags.size()) raise(CF_VALIDATION, "mesh validation failed: facet tag out of range");
    for (int32_t v : m->contacts)
        if (v < 0 || v >= (int32_t)m->tags.size()) raise(CF_VALIDATION, "mesh validation failed: contact tag out of range");
    m->make_desc();
    MeshData md;  // the text parser's finalize_mesh contract: validation + orientation
    try {
        finalize_mesh(&m->desc, md);
    } catch (const Error& e) {
        raise(CF_VALIDATION, std::string("mesh validation failed: ") + e.what());
    }
    std::memcpy(m->tets.data(), md.tets.data(), sizeof(int32_t) * m->tets.size());
    return m;
}

// ------------------------------------------------------------------ config
struct TextSetup {
    struct Table {
        std::vector<double> x, y;
    };
    struct Mat {
        double rho = 0, latent = 0, solidus = 0, liquidus = 0, T0 = 0;
        Table c, k;
    };
    struct Bc {
        int kind = CF_BC_FLUX;
        Table T;
        double q = 0, h = 0, t_inf = 0;
    };
    struct Coeff {
        std::string a, b;
        int var = CF_VAR_TIME;
        Table h{{0.0}, {0.0}};  // PiecewiseLinear::constant(0)
    };
    std::vector<Mat> mats;
    std::map<std::string, Bc> bcs;  // ordered by tag, as the reference's std::map
    std::vector<Coeff> coeffs;
    double safety = 0.5, t_end = 0;
    long output_every = 0;
    // views
    std::vector<cf_material> vmat;
    std::vector<cf_boundary_condition> vbc;
    std::vector<cf_interface_coeff> vco;
    cf_setup_desc desc{};
    static cf_table view(const Table& t) { return cf_table{(int32_t)t.x.size(), t.x.data(), t.y.data()}; }
    void make_desc() {
        vmat.clear();
        for (const auto& m : mats)
            vmat.push_back(cf_material{m.rho, view(m.c), view(m.k), m.latent, m.solidus, m.liquidus, m.T0});
        vbc.clear();
        for (const auto& [tag, b] : bcs) vbc.push_back(cf_boundary_condition{tag.c_str(), b.kind, view(b.T), b.q, b.h, b.t_inf});
        vco.clear();
        for (const auto& c : coeffs) vco.push_back(cf_interface_coeff{c.a.c_str(), c.b.c_str(), c.var, view(c.h)});
        desc = cf_setup_desc{(int32_t)vmat.size(), vmat.data(), (int32_t)vbc.size(), vbc.data(), (int32_t)vco.size(),
                             vco.data(), safety, t_end, (int64_t)output_every, nullptr};
    }
};

namespace {
using Words = std::vector<std::string_view>;

// a table value (material.hpp:188-202): one bare number is a constant, otherwise x:y pairs
TextSetup::Table table_from(const Words& w, long line) {
    TextSetup::Table t;
    if (w.size() == 2 && w[1].find(':') == std::string_view::npos) {
        t.x = {0.0};
        t.y = {to_double(w[1], line)};
        return t;
    }
    for (size_t i = 1; i < w.size(); ++i) {
        const size_t colon = w[i].find(':');
        if (colon == std::string_view::npos) parse_fail("expected x:y pair, got '" + std::string(w[i]) + "'", line);
        t.x.push_back(to_double(w[i].substr(0, colon), line));
        t.y.push_back(to_double(w[i].substr(colon + 1), line));
    }
    return t;
}

// the checks PiecewiseLinear::validate makes (material.hpp:40-46)
void require_table(const TextSetup::Table& t, const std::string& name) {
    if (t.x.empty() || t.x.size() != t.y.size()) raise(CF_CONFIG, name + ": empty or inconsistent table");
    if (std::adjacent_find(t.x.begin(), t.x.end(), [](double a, double b) { return !(b > a); }) != t.x.end())
        raise(CF_CONFIG, name + ": table abscissae must be strictly increasing");
}

std::string_view value_of(const Words& w, long line) {  // the word after the key
    if (w.size() < 2) raise(CF_INVALID_ARG, "line " + std::to_string(line) + ": missing value");
    return w[1];
}

// Where key lines currently land: the open section's objects.
struct ConfigCursor {
    TextSetup* S = nullptr;
    TextSetup::Mat* mat = nullptr;
    TextSetup::Bc* bc = nullptr;
    TextSetup::Coeff* coeff = nullptr;
};

// The grammar as data: every section lists its keys, each with the assignment it performs.
struct KeyRule {
    const char* key;
    void (*assign)(ConfigCursor&, const Words&, long);
};
struct SectionRule {
    const char* name;
    size_t header_words;  // words inside the brackets, the name included
    const char* noun;     // "unknown <noun> key '...'"
    void (*open)(ConfigCursor&, const std::vector<std::string>&, long);
    std::vector<KeyRule> keys;
};

#define CF_NUM(target) [](ConfigCursor& c, const Words& w, long ln) { target = to_double(value_of(w, ln), ln); }
#define CF_TAB(target) [](ConfigCursor& c, const Words& w, long ln) { target = table_from(w, ln); }

const std::vector<SectionRule>& grammar() {
    static const std::vector<SectionRule> g = {
        {"material", 2, "material",
         [](ConfigCursor& c, const std::vector<std::string>& h, long ln) {
             const long r = to_long(h[1], ln);
             if (r < 0) raise(CF_INVALID_ARG, "line " + std::to_string(ln) + ": negative region id");
             if (c.S->mats.size() <= (size_t)r) c.S->mats.resize((size_t)r + 1);
             c.mat = &c.S->mats[(size_t)r];
         },
         {{"rho", CF_NUM(c.mat->rho)}, {"c", CF_TAB(c.mat->c)}, {"k", CF_TAB(c.mat->k)},
          {"latent_heat", CF_NUM(c.mat->latent)}, {"solidus", CF_NUM(c.mat->solidus)},
          {"liquidus", CF_NUM(c.mat->liquidus)}, {"T0", CF_NUM(c.mat->T0)}}},
        {"bc", 2, "bc",
         [](ConfigCursor& c, const std::vector<std::string>& h, long) { c.bc = &c.S->bcs[h[1]]; },  // flux by default
         {{"kind",
           [](ConfigCursor& c, const Words& w, long ln) {
               const std::string_view v = value_of(w, ln);
               if (v == "fixed") c.bc->kind = CF_BC_FIXED;
               else if (v == "flux") c.bc->kind = CF_BC_FLUX;
               else parse_fail("bc kind must be fixed or flux", ln);
           }},
          {"T", CF_TAB(c.bc->T)}, {"q", CF_NUM(c.bc->q)}, {"h", CF_NUM(c.bc->h)}, {"T_inf", CF_NUM(c.bc->t_inf)}}},
        {"interface", 3, "interface",
         [](ConfigCursor& c, const std::vector<std::string>& h, long) {
             c.S->coeffs.emplace_back();
             c.coeff = &c.S->coeffs.back();
             c.coeff->a = h[1];
             c.coeff->b = h[2];
         },
         {{"h", CF_TAB(c.coeff->h)},
          {"h_time", [](ConfigCursor& c, const Words& w, long ln) { c.coeff->var = CF_VAR_TIME, c.coeff->h = table_from(w, ln); }},
          {"h_temp",
           [](ConfigCursor& c, const Words& w, long ln) { c.coeff->var = CF_VAR_TEMPERATURE, c.coeff->h = table_from(w, ln); }}}},
        {"solver", 1, "solver", [](ConfigCursor&, const std::vector<std::string>&, long) {},
         {{"safety", CF_NUM(c.S->safety)}, {"t_end", CF_NUM(c.S->t_end)},
          {"output_every", [](ConfigCursor& c, const Words& w, long ln) { c.S->output_every = to_long(value_of(w, ln), ln); }}}},
    };
    return g;
}
#undef CF_NUM
#undef CF_TAB

// "[bc outer]", "[ bc outer ]", "[bc] outer": the brackets carry no meaning of their own -- they are
// dropped wherever they stand and what is left of each word counts
std::vector<std::string> header_words(const Words& w) {
    std::vector<std::string> out;
    for (std::string_view t : w) {
        std::string bare;
        std::copy_if(t.begin(), t.end(), std::back_inserter(bare), [](char ch) { return ch != '[' && ch != ']'; });
        if (!bare.empty()) out.push_back(std::move(bare));
    }
    return out;
}
}  // namespace

std::unique_ptr<TextSetup> parse_config_text(std::string_view text) {
    auto S = std::make_unique<TextSetup>();
    const LineIndex idx(text);
    ConfigCursor cur;
    cur.S = S.get();
    const SectionRule* open = nullptr;
    Words w;
    for (const LogicalLine& line : idx.lines) {
        std::string_view first[1];
        w.resize((size_t)words(line, first, 1));
        words(line, w.data(), (int)w.size());
        if (w[0].front() == '[') {
            const std::vector<std::string> head = header_words(w);
            if (head.empty()) parse_fail("empty section header", line.no);
            open = nullptr;
            for (const SectionRule& r : grammar())
                if (head[0] == r.name && head.size() == r.header_words) open = &r;
            if (!open) parse_fail("unknown section '" + head[0] + "'", line.no);
            open->open(cur, head, line.no);
            continue;
        }
        if (!open) parse_fail("key '" + std::string(w[0]) + "' outside any section", line.no);
        const auto rule = std::find_if(open->keys.begin(), open->keys.end(), [&](const KeyRule& k) { return w[0] == k.key; });
        if (rule == open->keys.end())
            parse_fail(std::string("unknown ") + open->noun + " key '" + std::string(w[0]) + "'", line.no);
        rule->assign(cur, w, line.no);
    }
    // what MaterialTable::finalize checks (material.hpp:104-119), for every region that was given a density
    for (const auto& m : S->mats) {
        if (!(m.rho > 0)) continue;  // a region never configured: the plan builder reports it if a tet uses it
        require_table(m.c, "c");
        require_table(m.k, "k");
        if (std::any_of(m.c.y.begin(), m.c.y.end(), [](double v) { return v <= 0; })) raise(CF_CONFIG, "c(T) must be positive");
        if (std::any_of(m.k.y.begin(), m.k.y.end(), [](double v) { return v <= 0; })) raise(CF_CONFIG, "k(T) must be positive");
        if (m.latent < 0) raise(CF_CONFIG, "latent_heat must be non-negative");
        if (m.latent > 0 && !(m.solidus < m.liquidus)) raise(CF_CONFIG, "phase change requires solidus < liquidus");
    }
    if (!(S->safety > 0 && S->safety <= 1)) raise(CF_CONFIG, "safety must be in (0, 1]");
    for (const auto& c : S->coeffs) require_table(c.h, "interface h");
    S->make_desc();
    return S;
}

// ------------------------------------------------------------------ partmap
void parse_partmap_text(std::string_view text, int32_t n_elems, int32_t* parts, int32_t* part_count) {
    // load_partmap partition.hpp:424-445: one integer per line (trimmed), '#' lines and blanks skipped
    size_t pos = 0, k = 0;
    long line_no = 0;
    int32_t count = 0;
    bool negative = false;
    while (pos < text.size()) {
        size_t end = text.find('\n', pos);
        if (end == std::string_view::npos) end = text.size();
        std::string_view v = text.substr(pos, end - pos);
        pos = end + 1;
        ++line_no;
        while (!v.empty() && std::isspace((unsigned char)v.back())) v.remove_suffix(1);
        while (!v.empty() && std::isspace((unsigned char)v.front())) v.remove_prefix(1);
        if (v.empty() || v[0] == '#') continue;
        const long p = to_long(v, line_no);
        if (k < (size_t)n_elems && parts) parts[k] = (int32_t)p;
        ++k;
        if (p < 0) negative = true;
        else if (p + 1 > count) count = (int32_t)(p + 1);
    }
    if (k != (size_t)n_elems)
        raise(CF_VALIDATION, "partmap has " + std::to_string(k) + " entries for " + std::to_string(n_elems) +
                                 " elements");
    if (negative) raise(CF_VALIDATION, "negative part id in partmap");
    if (part_count) *part_count = count;
}

std::string format_partmap(const int32_t* parts, int32_t n) {
    std::string s;
    for (int32_t i = 0; i < n; ++i) s += std::to_string(parts[i]) + "\n";
    return s;
}

}  // namespace cfb

// ------------------------------------------------------------------ C-ABI
using namespace cfb;

struct cf_text_mesh : TextMesh {};
struct cf_text_setup : TextSetup {};

namespace {
template <class F>
int io_guarded(F&& f) {
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
void copy_out(const std::string& s, char* buf, int64_t cap, int64_t* len) {
    if (len) *len = (int64_t)s.size();
    if (buf && cap > 0) {
        const size_t n = std::min<size_t>(s.size(), (size_t)cap - 1);
        std::memcpy(buf, s.data(), n);
        buf[n] = 0;
    }
}
}  // namespace

extern "C" {

int cf_mesh_parse(const char* text, int64_t len, cf_text_mesh** out) {
    return io_guarded([&] {
        if (!out || (len && !text) || len < 0) raise(CF_INVALID_ARG, "null argument");
        auto m = parse_mesh_text(std::string_view(text ? text : "", (size_t)len));
        auto r = std::make_unique<cf_text_mesh>();
        static_cast<TextMesh&>(*r) = std::move(*m);
        r->make_desc();
        *out = r.release();
    });
}

int cf_mesh_view(const cf_text_mesh* m, cf_mesh_desc* out) {
    return io_guarded([&] {
        if (!m || !out) raise(CF_INVALID_ARG, "null argument");
        *out = m->desc;
    });
}

void cf_mesh_free(cf_text_mesh* m) { delete m; }

int cf_mesh_parse_binary(const void* data, int64_t len, cf_text_mesh** out) {
    return io_guarded([&] {
        if (!out || (len && !data) || len < 0) raise(CF_INVALID_ARG, "null argument");
        auto m = parse_mesh_binary(std::string_view((const char*)data, (size_t)len));
        auto r = std::make_unique<cf_text_mesh>();
        static_cast<TextMesh&>(*r) = std::move(*m);
        r->make_desc();
        *out = r.release();
    });
}

int cf_mesh_format_binary(const cf_mesh_desc* d, void* buf, int64_t cap, int64_t* len) {
    return io_guarded([&] {
        if (!d) raise(CF_INVALID_ARG, "null argument");
        const std::string s = mesh_binary(d);
        if (len) *len = (int64_t)s.size();
        if (buf && cap >= (int64_t)s.size()) std::memcpy(buf, s.data(), s.size());
        else if (buf) raise(CF_INVALID_ARG, "buffer too small for the binary mesh");
    });
}

int cf_mesh_format(const cf_mesh_desc* d, char* buf, int64_t cap, int64_t* len) {
    return io_guarded([&] {
        if (!d) raise(CF_INVALID_ARG, "null argument");
        copy_out(format_mesh(d), buf, cap, len);
    });
}

int cf_config_parse(const char* text, int64_t len, cf_text_setup** out) {
    return io_guarded([&] {
        if (!out || (len && !text) || len < 0) raise(CF_INVALID_ARG, "null argument");
        auto S = parse_config_text(std::string_view(text ? text : "", (size_t)len));
        auto r = std::make_unique<cf_text_setup>();
        static_cast<TextSetup&>(*r) = std::move(*S);
        r->make_desc();
        *out = r.release();
    });
}

int cf_config_view(const cf_text_setup* s, cf_setup_desc* out) {
    return io_guarded([&] {
        if (!s || !out) raise(CF_INVALID_ARG, "null argument");
        *out = s->desc;
    });
}

void cf_config_free(cf_text_setup* s) { delete s; }

int cf_partmap_parse(const char* text, int64_t len, int32_t n_elems, int32_t* parts_out, int32_t* part_count) {
    return io_guarded([&] {
        if ((len && !text) || len < 0 || n_elems < 0) raise(CF_INVALID_ARG, "bad argument");
        parse_partmap_text(std::string_view(text ? text : "", (size_t)len), n_elems, parts_out, part_count);
    });
}

int cf_partmap_format(const int32_t* parts, int32_t n, char* buf, int64_t cap, int64_t* len) {
    return io_guarded([&] {
        if (n < 0 || (n && !parts)) raise(CF_INVALID_ARG, "bad argument");
        copy_out(format_partmap(parts, n), buf, cap, len);
    });
}

}  // extern "C"
