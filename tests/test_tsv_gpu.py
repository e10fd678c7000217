"""LoadTableTSV on the B200: the device parser gives the
host parser's values and errors (tables.py:246-284 semantics: universal
newlines, exact field count, int() per field, first bad line reported)."""

import numpy as np
import pytest

from paper_1503_07881_b200.errors import ParseError
from paper_1503_07881_b200.tables import INT, STRING, Schema, load_tsv

pytestmark = pytest.mark.gpu
S2 = Schema([("src", INT), ("dst", INT)])


def _both(tmp_path, text: bytes, schema=S2):
    p = tmp_path / "t.tsv"
    p.write_bytes(text)
    host_exc = dev_exc = None
    try:
        host = load_tsv(p, schema)
    except (ParseError, OverflowError) as e:
        host_exc = e
    try:
        dev = load_tsv(p, schema, device="cuda")
    except (ParseError, OverflowError) as e:
        dev_exc = e
    if host_exc is not None or dev_exc is not None:
        assert type(host_exc) is type(dev_exc), (host_exc, dev_exc)
        assert str(host_exc) == str(dev_exc)
        if isinstance(host_exc, ParseError):
            assert getattr(host_exc, "line", None) == getattr(dev_exc, "line", None)
        return None
    assert dev.n_rows == host.n_rows
    for name in schema.names:
        assert np.array_equal(dev.column(name).cpu().numpy(), host.column(name))
    return dev


def test_random_table_round_trip(tmp_path):
    rng = np.random.default_rng(3)
    a = rng.integers(-10**12, 10**12, size=20000)
    b = rng.integers(-5, 10**6, size=20000)
    text = "".join(f"{x}\t{y}\n" for x, y in zip(a.tolist(), b.tolist())).encode()
    t = _both(tmp_path, text)
    assert np.array_equal(t.column("src").cpu().numpy(), a)


@pytest.mark.parametrize("text", [
    b"", b"1\t2", b"1\t2\n3\t4", b"1\t2\r\n3\t4\r\n", b"1\t2\r3\t4\r", b"1\t2\n\r\n3\t4\n",
    b" 1 \t+2\n007\t-0\n", b"1_000\t2_3_4\n", b"-9223372036854775808\t9223372036854775807\n",
    b"1\t2\n\n3\t4\n", b"1\t2\t3\n", b"1\n", b"1\tx\n", b"1\t2_\n", b"1\t_2\n", b"1\t2__3\n",
    b"1\t\n", b"\t1\n", b"1\t-\n", b"1\t+-2\n", b"1\t9223372036854775808\n",
    b"1\t99999999999999999999999\n2\tz\n", b"5\t6\n7\t8\n9\t1 0\n", b"1\t2\x0b\n",
])
def test_edge_cases_match_host(tmp_path, text):
    _both(tmp_path, text)


def test_single_int_column_and_errors(tmp_path):
    s1 = Schema([("x", INT)])
    _both(tmp_path, b"1\n2\n3\n", s1)
    _both(tmp_path, b"1\n\n3\n", s1)
    _both(tmp_path, b"1\n2\t3\n", s1)


def test_non_int_schema_is_refused(tmp_path):
    from paper_1503_07881_b200.errors import TypeMismatchError

    p = tmp_path / "t.tsv"
    p.write_bytes(b"a\t1\n")
    with pytest.raises(TypeMismatchError):
        load_tsv(p, Schema([("s", STRING), ("x", INT)]), device="cuda")


def test_ingest_feeds_tograph(tmp_path):
    import paper_1503_07881_b200 as gt
    from oracle import reference_port as ref
    from paper_1503_07881_b200.synth import rmat_edges

    src, dst = rmat_edges(12, 50000, seed=2, permute=True)
    p = tmp_path / "e.tsv"
    p.write_text("".join(f"{a}\t{b}\n" for a, b in zip(src.tolist(), dst.tolist())))
    t = load_tsv(p, S2, device="cuda")
    g = gt.table_to_graph(t, gt.EdgeSpec("src", "dst"))
    want = ref.build_csr(src, dst)
    assert np.array_equal(g.csr().out_off, want.out_off)
    assert gt.triangle_count(g) == ref.triangle_count_fast(want)
