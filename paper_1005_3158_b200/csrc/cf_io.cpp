// cf_io.cpp — the text formats either side of the step:
//   femesh 1 mesh       parse_mesh / write_mesh      mesh.hpp:256-343
//   solver config       parse_config                 material.hpp:186-345
//   partmap             load_partmap / write_partmap partition.hpp:424-449
//   binary mesh         this repo's fast path for large meshes (same validation as parse_mesh)
// Same tokenizer ('#' comments, whitespace-separated tokens, blank lines skipped,
// 1-based line numbers), the same number syntax (std::from_chars), the same
// section semantics and defaults, and the same error classes and messages:
// CF_PARSE "line N: ..." for syntax, CF_VALIDATION "mesh validation failed: ..."
// for a mesh finalize_mesh rejects, CF_CONFIG for table / material checks.
#include <algorithm>
#include <cctype>
#include <charconv>
#include <cstdio>
#include <cstring>
#include <map>
#include <memory>
#include <string>
#include <string_view>
#include <vector>

#include "cf_internal.hpp"

namespace cfb {
namespace {

struct Lines {  // LineReader mesh.hpp:211-235
    std::string_view text;
    size_t pos = 0;
    long line_no = 0;
    bool next(std::vector<std::string_view>& tok) {
        while (pos < text.size()) {
            size_t end = text.find('\n', pos);
            if (end == std::string_view::npos) end = text.size();
            std::string_view v = text.substr(pos, end - pos);
            pos = end + 1;
            ++line_no;
            if (const size_t h = v.find('#'); h != std::string_view::npos) v = v.substr(0, h);
            tok.clear();
            size_t i = 0;
            while (i < v.size()) {
                while (i < v.size() && std::isspace((unsigned char)v[i])) ++i;
                size_t j = i;
                while (j < v.size() && !std::isspace((unsigned char)v[j])) ++j;
                if (j > i) tok.push_back(v.substr(i, j - i));
                i = j;
            }
            if (!tok.empty()) return true;
        }
        return false;
    }
};

[[noreturn]] void parse_fail(const std::string& what, long line) {
    raise(CF_PARSE, "line " + std::to_string(line) + ": " + what);
}

double to_double(std::string_view t, long line) {
    double v = 0;
    const auto r = std::from_chars(t.data(), t.data() + t.size(), v);
    if (r.ec != std::errc{} || r.ptr != t.data() + t.size())
        parse_fail("expected a number, got '" + std::string(t) + "'", line);
    return v;
}

long to_long(std::string_view t, long line) {
    long v = 0;
    const auto r = std::from_chars(t.data(), t.data() + t.size(), v);
    if (r.ec != std::errc{} || r.ptr != t.data() + t.size())
        parse_fail("expected an integer, got '" + std::string(t) + "'", line);
    return v;
}

// a count from a section header: the reference reserves it (negative -> length error)
size_t to_count(std::string_view t, long line) {
    const long n = to_long(t, line);
    if (n < 0) raise(CF_INVALID_ARG, "line " + std::to_string(line) + ": negative count");
    return (size_t)n;
}

void append_g17(std::string& s, double v) {
    char b[40];
    const int n = std::snprintf(b, sizeof b, "%.17g", v);
    s.append(b, (size_t)n);
}

}  // namespace

// ------------------------------------------------------------------ mesh
struct TextMesh {
    std::vector<double> coords;
    std::vector<int32_t> tets, region, facets, facet_tag, contacts;
    std::vector<std::string> tags;
    std::vector<const char*> tag_ptrs;
    cf_mesh_desc desc{};
    int32_t add_tag(std::string_view name) {  // Mesh::add_tag mesh.hpp:62-67
        for (size_t i = 0; i < tags.size(); ++i)
            if (tags[i] == name) return (int32_t)i;
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

std::unique_ptr<TextMesh> parse_mesh_text(std::string_view text) {
    Lines rd{text};
    std::vector<std::string_view> tok;
    if (!rd.next(tok) || tok.size() != 2 || tok[0] != "femesh" || tok[1] != "1")
        parse_fail("expected header 'femesh 1'", rd.line_no);
    auto m = std::make_unique<TextMesh>();
    while (rd.next(tok)) {
        if (tok[0] == "nodes") {
            if (tok.size() != 2) parse_fail("usage: nodes N", rd.line_no);
            const size_t n = to_count(tok[1], rd.line_no);
            m->coords.reserve(m->coords.size() + 3 * n);
            for (size_t i = 0; i < n; ++i) {
                if (!rd.next(tok)) parse_fail("unexpected end of node list", rd.line_no);
                if (tok.size() != 3) parse_fail("node line needs 'x y z'", rd.line_no);
                for (int k = 0; k < 3; ++k) m->coords.push_back(to_double(tok[k], rd.line_no));
            }
        } else if (tok[0] == "tets") {
            if (tok.size() != 2) parse_fail("usage: tets M", rd.line_no);
            const size_t n = to_count(tok[1], rd.line_no);
            m->tets.reserve(m->tets.size() + 4 * n);
            for (size_t i = 0; i < n; ++i) {
                if (!rd.next(tok)) parse_fail("unexpected end of element list", rd.line_no);
                if (tok.size() != 5) parse_fail("element line needs 'n0 n1 n2 n3 region'", rd.line_no);
                for (int k = 0; k < 4; ++k) m->tets.push_back((int32_t)to_long(tok[k], rd.line_no));
                m->region.push_back((int32_t)to_long(tok[4], rd.line_no));
            }
        } else if (tok[0] == "facets") {
            if (tok.size() != 2) parse_fail("usage: facets B", rd.line_no);
            const size_t n = to_count(tok[1], rd.line_no);
            for (size_t i = 0; i < n; ++i) {
                if (!rd.next(tok)) parse_fail("unexpected end of facet list", rd.line_no);
                if (tok.size() != 4) parse_fail("facet line needs 'n0 n1 n2 tag'", rd.line_no);
                for (int k = 0; k < 3; ++k) m->facets.push_back((int32_t)to_long(tok[k], rd.line_no));
                m->facet_tag.push_back(m->add_tag(tok[3]));
            }
        } else if (tok[0] == "contact") {
            if (tok.size() != 3) parse_fail("usage: contact tagA tagB", rd.line_no);
            const int32_t a = m->add_tag(tok[1]);
            const int32_t b = m->add_tag(tok[2]);
            m->contacts.push_back(a);
            m->contacts.push_back(b);
        } else {
            parse_fail("unknown section '" + std::string(tok[0]) + "'", rd.line_no);
        }
    }
    m->make_desc();
    // finalize_mesh: validation and orientation, errors wrapped like parse_mesh (mesh.hpp:318-322)
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
// parse_table material.hpp:188-202: one bare number = constant, else x:y pairs
TextSetup::Table parse_table(const std::vector<std::string_view>& tok, size_t first, long line) {
    TextSetup::Table t;
    if (tok.size() == first + 1 && tok[first].find(':') == std::string_view::npos) {
        t.x = {0.0};
        t.y = {to_double(tok[first], line)};
        return t;
    }
    for (size_t i = first; i < tok.size(); ++i) {
        const size_t c = tok[i].find(':');
        if (c == std::string_view::npos) parse_fail("expected x:y pair, got '" + std::string(tok[i]) + "'", line);
        t.x.push_back(to_double(tok[i].substr(0, c), line));
        t.y.push_back(to_double(tok[i].substr(c + 1), line));
    }
    return t;
}

// PiecewiseLinear::validate material.hpp:40-46
void validate_table(const TextSetup::Table& t, const std::string& name) {
    if (t.x.empty() || t.x.size() != t.y.size()) raise(CF_CONFIG, name + ": empty or inconsistent table");
    for (size_t i = 1; i < t.x.size(); ++i)
        if (!(t.x[i] > t.x[i - 1])) raise(CF_CONFIG, name + ": table abscissae must be strictly increasing");
}

std::string_view arg1(const std::vector<std::string_view>& tok, long line) {  // tok.at(1)
    if (tok.size() < 2) raise(CF_INVALID_ARG, "line " + std::to_string(line) + ": missing value");
    return tok[1];
}
}  // namespace

std::unique_ptr<TextSetup> parse_config_text(std::string_view text) {
    auto S = std::make_unique<TextSetup>();
    Lines rd{text};
    std::vector<std::string_view> tok;
    enum { NONE, MATERIAL, BC, INTERFACE, SOLVER } sec = NONE;
    long region = -1;
    std::string bc_tag;
    auto material_at = [&](long r) -> TextSetup::Mat& {
        if (r < 0) raise(CF_INVALID_ARG, "line " + std::to_string(rd.line_no) + ": negative region id");
        if ((long)S->mats.size() <= r) S->mats.resize((size_t)r + 1);
        return S->mats[(size_t)r];
    };
    while (rd.next(tok)) {
        if (tok.front().front() == '[') {  // section header: brackets dropped, tokens re-split
            std::vector<std::string> head;
            std::string cur;
            for (const auto& t : tok) {
                for (char ch : t) {
                    if (ch == '[' || ch == ']') continue;
                    cur.push_back(ch);
                }
                if (!cur.empty()) head.push_back(cur);
                cur.clear();
            }
            if (head.empty()) parse_fail("empty section header", rd.line_no);
            if (head[0] == "material" && head.size() == 2) {
                sec = MATERIAL;
                region = to_long(head[1], rd.line_no);
                material_at(region);
            } else if (head[0] == "bc" && head.size() == 2) {
                sec = BC;
                bc_tag = head[1];
                S->bcs[bc_tag];  // default flux bc
            } else if (head[0] == "interface" && head.size() == 3) {
                sec = INTERFACE;
                TextSetup::Coeff c;
                c.a = head[1];
                c.b = head[2];
                S->coeffs.push_back(c);
            } else if (head[0] == "solver" && head.size() == 1) {
                sec = SOLVER;
            } else {
                parse_fail("unknown section '" + head[0] + "'", rd.line_no);
            }
            continue;
        }
        const std::string key(tok[0]);
        const long ln = rd.line_no;
        switch (sec) {
            case MATERIAL: {
                auto& m = material_at(region);
                if (key == "rho") m.rho = to_double(arg1(tok, ln), ln);
                else if (key == "c") m.c = parse_table(tok, 1, ln);
                else if (key == "k") m.k = parse_table(tok, 1, ln);
                else if (key == "latent_heat") m.latent = to_double(arg1(tok, ln), ln);
                else if (key == "solidus") m.solidus = to_double(arg1(tok, ln), ln);
                else if (key == "liquidus") m.liquidus = to_double(arg1(tok, ln), ln);
                else if (key == "T0") m.T0 = to_double(arg1(tok, ln), ln);
                else parse_fail("unknown material key '" + key + "'", ln);
                break;
            }
            case BC: {
                auto& b = S->bcs[bc_tag];
                if (key == "kind") {
                    const std::string_view v = arg1(tok, ln);
                    if (v == "fixed") b.kind = CF_BC_FIXED;
                    else if (v == "flux") b.kind = CF_BC_FLUX;
                    else parse_fail("bc kind must be fixed or flux", ln);
                } else if (key == "T") b.T = parse_table(tok, 1, ln);
                else if (key == "q") b.q = to_double(arg1(tok, ln), ln);
                else if (key == "h") b.h = to_double(arg1(tok, ln), ln);
                else if (key == "T_inf") b.t_inf = to_double(arg1(tok, ln), ln);
                else parse_fail("unknown bc key '" + key + "'", ln);
                break;
            }
            case INTERFACE: {
                auto& c = S->coeffs.back();
                if (key == "h") {
                    c.h = parse_table(tok, 1, ln);
                } else if (key == "h_time") {
                    c.var = CF_VAR_TIME;
                    c.h = parse_table(tok, 1, ln);
                } else if (key == "h_temp") {
                    c.var = CF_VAR_TEMPERATURE;
                    c.h = parse_table(tok, 1, ln);
                } else {
                    parse_fail("unknown interface key '" + key + "'", ln);
                }
                break;
            }
            case SOLVER: {
                if (key == "safety") S->safety = to_double(arg1(tok, ln), ln);
                else if (key == "t_end") S->t_end = to_double(arg1(tok, ln), ln);
                else if (key == "output_every") S->output_every = to_long(arg1(tok, ln), ln);
                else parse_fail("unknown solver key '" + key + "'", ln);
                break;
            }
            case NONE:
                parse_fail("key '" + key + "' outside any section", ln);
        }
    }
    // MaterialTable::finalize material.hpp:104-119 for the materials that were set
    for (const auto& m : S->mats) {
        if (!(m.rho > 0)) continue;  // untouched slots are caught at bind time
        validate_table(m.c, "c");
        validate_table(m.k, "k");
        for (double v : m.c.y)
            if (v <= 0) raise(CF_CONFIG, "c(T) must be positive");
        for (double v : m.k.y)
            if (v <= 0) raise(CF_CONFIG, "k(T) must be positive");
        if (m.latent < 0) raise(CF_CONFIG, "latent_heat must be non-negative");
        if (m.latent > 0 && !(m.solidus < m.liquidus)) raise(CF_CONFIG, "phase change requires solidus < liquidus");
    }
    if (!(S->safety > 0 && S->safety <= 1)) raise(CF_CONFIG, "safety must be in (0, 1]");
    for (const auto& c : S->coeffs) validate_table(c.h, "interface h");
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
