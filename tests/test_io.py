"""Text formats either side of the step: the product's
femesh / config / partmap parsers (C-ABI, paper_1005_3158_b200/csrc/cf_io.cpp)
against the reference's own parse_mesh / write_mesh / parse_config /
load_partmap (unmodified headers in oracle/_ref): identical output text,
identical error class and message (line numbers included)."""
import numpy as np
import pytest

from oracle import oracle as orc
from paper_1005_3158_b200 import castfem as cf

need_ref = pytest.mark.skipif(not orc.ref_available(), reason="oracle/_ref not built (needs /root/reference)")


def ours_mesh(text: bytes):
    try:
        return 0, cf.write_mesh(cf.parse_mesh(text))
    except cf.CastfemError as e:
        return e.code, str(e)


def ours_config(text: bytes):
    try:
        S = cf.parse_config(text)
    except cf.CastfemError as e:
        return e.code, str(e)
    g = lambda v: "%.17g" % v
    tab = lambda t: "[" + ",".join(f"{g(x)}:{g(y)}" for x, y in zip(t.xs, t.ys)) + "]"
    s = ""
    for i, m in enumerate(S.materials):
        s += (f"material {i} rho={g(m.rho)} c={tab(m.c_of_T)} k={tab(m.k_of_T)} L={g(m.latent_heat)} "
              f"Ts={g(m.solidus)} Tl={g(m.liquidus)} T0={g(m.initial_temperature)}\n")
    for tag in sorted(S.boundary_conditions):
        b = S.boundary_conditions[tag]
        s += f"bc {tag} kind={b.kind} T={tab(b.fixed_T)} q={g(b.q)} h={g(b.h)} t_inf={g(b.t_inf)}\n"
    for c in S.interface_coeffs:
        s += f"interface {c.tag_a} {c.tag_b} var={c.var} h={tab(c.h)}\n"
    s += f"solver safety={g(S.solver.dt_safety)} t_end={g(S.solver.t_end)} output_every={S.solver.output_every}\n"
    return 0, s


def _casting_text(n=5, jitter=0.2, perm=3):
    m = cf.generate_fixture("casting", n, jitter=jitter, seed=4, perm_seed=perm)
    return cf.write_mesh(m).encode(), m


# ---------------------------------------------------------------- mesh
def test_mesh_roundtrip_self():
    text, m = _casting_text()
    p = cf.parse_mesh(text)
    assert np.array_equal(p.nodes, m.nodes) and np.array_equal(p.region, m.region)
    assert p.element_count() == m.element_count() and len(p.facets) == len(m.facets)
    again = cf.parse_mesh(cf.write_mesh(p))  # a finalized mesh round-trips exactly
    assert np.array_equal(again.tets, p.tets) and again.tags == p.tags and again.contacts == p.contacts


@need_ref
@pytest.mark.parametrize("n,jitter,perm", [(4, 0.0, 0), (5, 0.2, 3), (7, 0.1, 9)])
def test_mesh_matches_reference(n, jitter, perm):
    text, _ = _casting_text(n, jitter, perm)
    assert ours_mesh(text) == orc.ref_mesh_roundtrip(text)


MESH_CASES = [
    b"",
    b"femesh 2\n",
    b"# comment only\n\n   \nfemesh 1 # trailing\n",
    b"femesh 1\nnodes\n",
    b"femesh 1\nnodes 2\n0 0 0\n",
    b"femesh 1\nnodes 1\n0 0\n",
    b"femesh 1\nnodes 1\n0 0 x\n",
    b"femesh 1\nnodes 1\n0 0 +1\n",
    b"femesh 1\nnodes 1\n0 0 1e400\n",
    b"femesh 1\nnodes 4\n0 0 0\n1 0 0\n0 1 0\n0 0 1\ntets 1\n0 1 2 3\n",
    b"femesh 1\nnodes 4\n0 0 0\n1 0 0\n0 1 0\n0 0 1\ntets 1\n0 1 2 3 0.5\n",
    b"femesh 1\nnodes 4\n0 0 0\n1 0 0\n0 1 0\n0 0 1\ntets 1\n0 1 2 3 0\n",
    b"femesh 1\nnodes 4\n0 0 0\n1 0 0\n0 1 0\n0 0 1\ntets 1\n0 1 3 2 0\nfacets 1\n0 1 2 outer\n",
    b"femesh 1\nnodes 4\n0 0 0\n1 0 0\n0 1 0\n0 0 1\ntets 1\n0 1 2 3 0\nfacets 1\n0 1 outer\n",
    b"femesh 1\nnodes 4\n0 0 0\n1 0 0\n0 1 0\n0 0 1\ntets 1\n0 1 2 3 0\ncontact a\n",
    b"femesh 1\nnodes 4\n0 0 0\n1 0 0\n0 1 0\n0 0 1\ntets 1\n0 1 2 3 0\ncontact a b\nfoo\n",
    b"femesh 1\nnodes 4\n0 0 0\n1 0 0\n0 1 0\n0 0 1\ntets 1\n0 1 2 9 0\n",
    b"femesh 1\nnodes 4\n0 0 0\n1 0 0\n0 1 0\n2 0 0\ntets 1\n0 1 2 3 0\n",
    b"femesh 1\nnodes 5\n0 0 0\n1 0 0\n0 1 0\n0 0 1\n5 5 5\ntets 1\n0 1 2 3 0\n",
    b"femesh 1\nnodes 4\n0 0 0\n1 0 0\n0 1 0\n0 0 1\ntets 1\n0 1 2 3 0\nfacets 1\n0 1 3 x\n",
    b"femesh 1\nnodes 4\n0 0 0\n1 0 0\n0 1 0\n0 0 1\ntets 1\n0 1 2 3 0\nfacets 1\n0 1 7 x\n",
    # several defects: the first in file order is the one reported (the product plans the sections
    # first and converts the records afterwards, in parallel)
    b"femesh 1\nnodes 2\n0 0 0\n0 0 oops\nbogus 3\n",                      # bad record before a bad header
    b"femesh 1\nnodes 2\n0 0 0\n1 1 1\nbogus 3\ntets 1\n0 1 2 x 0\n",      # bad header before a bad record
    b"femesh 1\nnodes 3\n0 0 0\n0 0\n",                                     # malformed record inside a list cut short
    b"femesh 1\nnodes 3\n0 0 0\n0 0 1\n\n# tail\n",                        # list cut short: the last physical line
    b"femesh 1\nnodes 2\n0 0 0\ntets 1\n",                                  # a header line consumed as a record
    b"femesh 1\nnodes x\n0 0 0\n",                                          # count is not an integer
    b"femesh 1\nnodes 1 2\n0 0 0\n",                                        # usage
    b"femesh 1\ncontact a b c\nnodes 1\n0 0 z\n",                           # contact usage before a bad record
    b"femesh 1\nnodes 4\n0 0 0\n1 0 0\n0 1 0\n0 0 1\ntets 1\n0 1 2 3 0\ncontact q p\nfacets 2\n0 1 2 p\n0 1 3 zz\n"
    b"contact zz q\n",                                                       # tags numbered by first appearance
    b"femesh 1\n nodes 1 \n\t0 0\t0 # c\r\n",                              # blanks, tabs, CR, comments
    b"femesh 1\nnodes 2\n0 0 0\n1 1 1\nnodes 2\n2 2 2\n0 0 1\ntets 1\n0 1 2 3 0\n",  # a section given twice appends
]


@need_ref
@pytest.mark.parametrize("i", range(len(MESH_CASES)))
def test_mesh_edge_cases_match_reference(i):
    text = MESH_CASES[i]
    ours, ref = ours_mesh(text), orc.ref_mesh_roundtrip(text)
    assert ours == ref  # same status, same text / message (line numbers, validation wording)


@need_ref
def test_large_mesh_parallel_conversion_matches_reference():
    """Lists longer than the parallel threshold (4096 records): same text out as the reference,
    and with one bad record deep inside each list the same first error."""
    m = cf.generate_fixture("casting", 12, jitter=0.1, seed=2, perm_seed=5)
    text = cf.write_mesh(m).encode()
    assert m.element_count() > 4096
    assert ours_mesh(text) == orc.ref_mesh_roundtrip(text)
    lines = text.split(b"\n")
    tets_at = lines.index(b"tets %d" % m.element_count())
    for at, repl in ((tets_at + 5000, b"1 2 3"), (tets_at + 9000, b"1 2 3 4 x"), (1 + 700, b"0 0 nan?")):
        bad = list(lines)
        bad[at] = repl
        bad[tets_at + 9500] = b"7 7"  # a later defect must not win
        t = b"\n".join(bad)
        ours, ref = ours_mesh(t), orc.ref_mesh_roundtrip(t)
        assert ours == ref and ours[0] != 0


# ---------------------------------------------------------------- config
CONFIG_OK = [
    b"",
    b"[solver]\nsafety 0.14 # comment\nt_end 100\noutput_every 7\n",
    b"""# casting, config 2
[material 1]
rho 1500
c 1000
k 1
T0 300
[material 0]
rho 2700
c 900
k 200
latent_heat 3.9e5
solidus 821
liquidus 913
T0 973
[bc outer]
h 20
T_inf 300
[bc hot]
kind fixed
T 0:650 50:950
[ interface cast_if mold_if ]
h 1000
[interface a b]
h_temp 300:10 900:2000
[interface c d]
[solver]
safety 0.138
""",
    b"[material 2]\nrho 7800\nc 300:450 900:700\nk 300:45 900:30\n[bc outer]\nkind flux\nq 5\n",
    # header forms: the brackets are dropped wherever they stand
    b"[ bc   outer ]\nh 3\n[bc] inner\nq 1\n[[bc] outer]\nT_inf 9\n",
    b"[interface a b]\nh_temp 300:5 900:7\n[interface] c [d\nh_time 4\n[solver ]\nsafety 0.25\n",
    # a section reopened continues the same object; regions out of order leave untouched slots
    b"[material 3]\nrho 2\nc 5\nk 6\n[bc w]\nq 2\n[material 3]\nT0 77\nlatent_heat 4\nsolidus 1\nliquidus 2\n"
    b"[bc w]\nkind fixed\nT 0:1 10:2\n[material 1]\nrho 9\nc 1\nk 1\n",
    b"[material 0]\nrho 1 2 3\nc 1\nk 0:1 5:2 # extra words after a scalar are ignored\n",
]

CONFIG_BAD = [
    b"rho 5\n",
    b"[]\n",
    b"[material]\n",
    b"[material x]\n",
    b"[material 0 1]\n",
    b"[bogus]\n",
    b"[material 0]\nrho abc\n",
    b"[material 0]\ncolor red\n",
    b"[material 0]\nrho 1\nc 1 2\nk 1\n",
    b"[material 0]\nrho 1\nc 2:1 1:2\nk 1\n",
    b"[material 0]\nrho 1\nc 0\nk 1\n",
    b"[material 0]\nrho 1\nc 1\nk 1\nlatent_heat 5\nsolidus 10\nliquidus 10\n",
    b"[material 0]\nrho 1\nc 1\nk 1\nlatent_heat -1\n",
    b"[material 0]\nrho 1\nk 1\n",
    b"[bc x]\nkind other\n",
    b"[bc x]\nwhat 1\n",
    b"[interface a b]\nh 5:1 4:2\n",
    b"[interface a b]\nbeta 1\n",
    b"[solver]\nsafety 0\n",
    b"[solver]\nsafety 1.5\n",
    b"[solver]\noutput_every 2.5\n",
    b"[solver]\nfoo 1\n",
    b"[ ]\n",
    b"[bc]\n",
    b"[bc a b]\n",
    b"[interface a]\n",
    b"[solver now]\n",
    b"[Material 0]\n",
    b"[material 0]\nrho 1\nc 1:\nk 1\n",
    b"[material 0]\nrho 1\nc :1\nk 1\n",
    b"[material 0]\nrho 1\nc 1:2:3\nk 1\n",
    b"[material 0]\nrho 1\nc\nk 1\n",
    b"[material 0]\nrho 1\nc 1\nk -2\n",
    b"[solver]\nsafety 0.5\nt_end x\n[bogus]\n",
]


def test_config_inputs_the_reference_mishandles_are_rejected_cleanly():
    """Where the reference has undefined behaviour (a negative region indexes before the material
    array) or leaks a library message (tok.at(1) on a key without a value throws std::out_of_range
    with libstdc++'s wording), this parser reports an invalid argument with the line number."""
    from paper_1005_3158_b200 import _abi
    for text, msg in ((b"[material -1]\n", "line 1: negative region id"),
                      (b"[bc x]\nkind\n", "line 2: missing value"),
                      (b"[solver]\n\nsafety\n", "line 3: missing value")):
        code, what = ours_config(text)
        assert code == _abi.CF_INVALID_ARG and what == msg


@need_ref
@pytest.mark.parametrize("i", range(len(CONFIG_OK)))
def test_config_matches_reference(i):
    text = CONFIG_OK[i]
    ours, ref = ours_config(text), orc.ref_config_dump(text)
    assert ref[0] == 0, ref
    assert ours == ref


@need_ref
@pytest.mark.parametrize("i", range(len(CONFIG_BAD)))
def test_config_errors_match_reference(i):
    text = CONFIG_BAD[i]
    ours, ref = ours_config(text), orc.ref_config_dump(text)
    assert ours[0] == ref[0] and ref[0] != 0, (ours, ref)
    assert ours[1] == ref[1]


def test_config_drives_the_solver_setup():
    """A parsed config is a SimulationSetup the plan accepts (binding checked at plan build)."""
    S = cf.parse_config(CONFIG_OK[2])
    assert [m.rho for m in S.materials] == [2700.0, 1500.0]
    assert S.boundary_conditions["hot"].kind == "fixed" and S.boundary_conditions["hot"].fixed_T.xs == [0.0, 50.0]
    assert S.interface_coeffs[1].var == "temperature" and S.interface_coeffs[2].h.ys == [0.0]
    assert S.solver.dt_safety == 0.138


# ---------------------------------------------------------------- partmap
PARTMAPS = [
    (b"0\n1\n1\n0\n", 4),
    (b"# parts\n 2 \n\n0\n1\n3\n", 4),
    (b"0\n1\n", 3),
    (b"0\n-1\n1\n", 3),
    (b"0\nx\n1\n", 3),
    (b"", 0),
]


@need_ref
@pytest.mark.parametrize("i", range(len(PARTMAPS)))
def test_partmap_matches_reference(i):
    text, n = PARTMAPS[i]
    ref = orc.ref_load_partmap(text, n)
    try:
        parts, count = cf.load_partmap(text, n)
        ours = (0, (parts, count))
    except cf.CastfemError as e:
        ours = (e.code, str(e))
    assert ours[0] == ref[0], (ours, ref)
    if ref[0] == 0:
        assert np.array_equal(ours[1][0], ref[1][0]) and ours[1][1] == ref[1][1]
    else:
        assert ours[1] == ref[1]


def test_partmap_roundtrip():
    p = np.array([3, 0, 2, 2, 1], dtype=np.int32)
    parts, count = cf.load_partmap(cf.write_partmap(p), len(p))
    assert np.array_equal(parts, p) and count == 4


# ---------------------------------------------------------------- binary fast path
def test_binary_mesh_roundtrip_equals_text(tmp_path):
    """The binary fast path holds exactly what the text format holds (after the same
    finalize_mesh), and read_mesh dispatches on the magic."""
    text, m = _casting_text(6, 0.2, 4)
    from_text = cf.parse_mesh(text)
    blob = cf.write_mesh_binary(m)
    assert blob[:8] == cf.MESH_BINARY_MAGIC
    from_bin = cf.parse_mesh_binary(blob)
    for a, b in [(from_text.nodes, from_bin.nodes), (from_text.tets, from_bin.tets), (from_text.region, from_bin.region),
                 (from_text.facets, from_bin.facets)]:
        assert np.array_equal(a, b)
    assert [from_text.tags[t] for t in from_text.facet_tag] == [from_bin.tags[t] for t in from_bin.facet_tag]
    p = tmp_path / "m.cfmb"
    p.write_bytes(blob)
    assert np.array_equal(cf.read_mesh(str(p)).tets, from_bin.tets)
    p2 = tmp_path / "m.femesh"
    p2.write_bytes(text)
    assert np.array_equal(cf.read_mesh(str(p2)).tets, from_text.tets)


def test_binary_mesh_errors():
    _, m = _casting_text(3, 0.0, 0)
    blob = cf.write_mesh_binary(m)
    for bad in [b"", b"NOTAMESH" + blob[8:], blob[:-3], blob + b"x"]:
        with pytest.raises(cf.ParseError):
            cf.parse_mesh_binary(bad)
    bad_tet = bytearray(blob)  # first tet's first node -> out of range: validation like parse_mesh
    off = 8 + 40 + 24 * m.node_count()
    bad_tet[off:off + 4] = (10 ** 6).to_bytes(4, "little")
    with pytest.raises(cf.ValidationError, match="mesh validation failed"):
        cf.parse_mesh_binary(bytes(bad_tet))


def test_binary_mesh_header_counts_bounded_by_buffer():
    """A 48-byte header announcing INT32_MAX nodes/tets is rejected as truncated before any
    section is allocated (no multi-GB resize on a malformed file)."""
    import struct
    hdr = b"CFMESHB1" + struct.pack("<5q", 2**31 - 1, 2**31 - 1, 0, 0, 0)
    import time
    t0 = time.time()
    with pytest.raises(cf.ParseError, match="truncated"):
        cf.parse_mesh_binary(hdr)
    assert time.time() - t0 < 1.0
