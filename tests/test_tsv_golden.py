"""LoadTableTSV parity against the REAL reference's load_tsv (tables.py:
246-284), recorded by tests/golden/make_golden_tsv.py into tsv.npz: the host
parser restatement (CPU), the device parser and the front-end routing (GPU)
give the same values, or the same exception class, message and line."""

from pathlib import Path

import numpy as np
import pytest

from paper_1503_07881_b200 import graphdesk
from paper_1503_07881_b200.errors import ParseError, TypeMismatchError
from paper_1503_07881_b200.tables import INT, Schema, load_tsv

GOLD = np.load(Path(__file__).resolve().parent / "golden" / "tsv.npz")
NAMES = GOLD["names"].tolist()


def _case(name):
    i = NAMES.index(name)
    text = GOLD["texts"][GOLD["text_off"][i]:GOLD["text_off"][i + 1]].tobytes()
    nc = int(GOLD["ncols"][i])
    cols = GOLD["cols"][GOLD["col_off"][i]:GOLD["col_off"][i + 1]]
    n = int(GOLD["counts"][i])
    want = [cols[j * n:(j + 1) * n] for j in range(nc)]
    return text, nc, str(GOLD["status"][i]), str(GOLD["messages"][i]), int(GOLD["lines"][i]), want


def _check(load, tmp_path, name):
    text, nc, status, msg, line, want = _case(name)
    p = tmp_path / f"{name}.tsv"
    p.write_bytes(text)
    schema = Schema([(f"c{j}", INT) for j in range(nc)])
    if status != "ok":
        with pytest.raises((ParseError, OverflowError)) as ei:
            load(p, schema)
        assert type(ei.value).__name__ == status
        assert str(ei.value) == msg
        if status == "ParseError":
            assert getattr(ei.value, "line", None) == line
        return None
    t = load(p, schema)
    assert t.n_rows == len(want[0]) if want else True
    for j in range(nc):
        got = t.column(f"c{j}")
        got = got.cpu().numpy() if hasattr(got, "cpu") else np.asarray(got)
        assert np.array_equal(got, want[j]), (name, j)
    return t


@pytest.mark.parametrize("name", NAMES)
def test_host_parser_matches_reference(tmp_path, name):
    _check(load_tsv, tmp_path, name)


@pytest.mark.gpu
@pytest.mark.parametrize("name", NAMES)
def test_device_parser_matches_reference(tmp_path, name):
    text = _case(name)[0]
    if any(b >= 0x80 for b in text):  # the device parser takes ASCII only
        p = tmp_path / "x.tsv"
        p.write_bytes(text)
        with pytest.raises(TypeMismatchError):
            load_tsv(p, Schema([("c0", INT), ("c1", INT)]), device="cuda")
        return
    t = _check(lambda p, s: load_tsv(p, s, device="cuda"), tmp_path, name)
    if t is not None and t.n_rows:
        assert t.column("c0").is_cuda


@pytest.mark.gpu
@pytest.mark.parametrize("name", NAMES)
def test_frontend_load_table_tsv_matches_reference(tmp_path, name):
    """graphdesk.LoadTableTSV routes all-int ASCII files to the GPU parser
    (columns land in HBM) and everything else to the host parser; errors are
    wrapped in FrontendError with the engine error attached (front-end
    __init__.py:35-42)."""
    text, nc, status, msg, line, want = _case(name)
    p = tmp_path / f"{name}.tsv"
    p.write_bytes(text)
    spec = ",".join(f"c{j}:int" for j in range(nc))
    if status == "OverflowError":  # not an EngineError/ValueError/OSError: not wrapped
        with pytest.raises(OverflowError, match=msg):
            graphdesk.LoadTableTSV(spec, str(p))
        return
    if status != "ok":
        with pytest.raises(graphdesk.FrontendError) as ei:
            graphdesk.LoadTableTSV(spec, str(p))
        eng = ei.value.engine_error
        assert type(eng).__name__ == status and str(eng) == msg
        return
    h = graphdesk.LoadTableTSV(spec, str(p))
    t = h._table
    for j in range(nc):
        got = t.column(f"c{j}")
        ascii_text = all(b < 0x80 for b in text)
        if ascii_text and t.n_rows:
            assert got.is_cuda
        got = got.cpu().numpy() if hasattr(got, "cpu") else np.asarray(got)
        assert np.array_equal(got, want[j])
