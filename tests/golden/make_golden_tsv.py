"""Golden fixtures for LoadTableTSV by running the REAL
reference's graphtables.load_tsv (tables.py:246-284) in the build container
on crafted all-int TSV files: values for the valid ones, the exception class,
message and line for the invalid ones (wrong field counts, non-integer
tokens, Python int() edge cases — whitespace, signs, underscores, leading
zeros —, values beyond int64, CRLF / lone CR line ends, empty lines, no
final newline, non-ASCII digits). Written to ``tsv.npz``.

Usage: PYTHONDONTWRITEBYTECODE=1 python tests/golden/make_golden_tsv.py
"""

from __future__ import annotations

import sys
import tempfile
from pathlib import Path

import numpy as np

HERE = Path(__file__).resolve().parent
sys.dont_write_bytecode = True
sys.path.insert(0, str(HERE))

from make_golden import ref  # noqa: E402  (the unmodified graphtables)


def cases():
    rng = np.random.default_rng(2024)
    out = []

    def add(name, text: str | bytes, ncols=2):
        out.append((name, text.encode("utf-8") if isinstance(text, str) else text, ncols))

    add("simple", "1\t2\n3\t4\n-5\t6\n")
    add("no_final_newline", "1\t2\n3\t4")
    add("empty_file", "")
    add("crlf", "1\t2\r\n3\t4\r\n")
    add("lone_cr", "1\t2\r3\t4\r")
    add("mixed_line_ends", "1\t2\r\n3\t4\n5\t6\r7\t8")
    add("whitespace", " 12\t 13 \n\t7\t8\n" if False else " 12\t 13 \n+7\t-0\n")
    add("underscores", "1_000\t2_0\n")
    add("double_underscore", "1__0\t2\n")
    add("leading_zeros", "007\t0000\n")
    add("hex_token", "0x10\t2\n")
    add("float_token", "1.0\t2\n")
    add("empty_field", "1\t\n")
    add("empty_line_mid", "1\t2\n\n3\t4\n")
    add("only_newline", "\n")
    add("one_field", "1\t2\n3\n")
    add("three_fields", "1\t2\n3\t4\t5\n")
    add("trailing_tab", "1\t2\t\n")
    add("int64_extremes", f"{2**63 - 1}\t{-2**63}\n0\t1\n")
    add("overflow_pos", f"1\t2\n{2**63}\t3\n")
    add("overflow_neg", f"{-2**63 - 1}\t3\n")
    add("sign_only", "-\t3\n")
    add("arabic_digits", "١٢\t3\n")
    add("space_inside", "1 2\t3\n")
    add("three_cols", "1\t2\t3\n4\t5\t6\n", ncols=3)
    add("three_cols_short", "1\t2\t3\n4\t5\n", ncols=3)
    for k in range(4):  # random tables, some with one bad line
        n = int(rng.integers(1000, 30000))
        a = rng.integers(-10**12, 10**12, n)
        b = rng.integers(-5, 10**6, n)
        lines = [f"{x}\t{y}" for x, y in zip(a.tolist(), b.tolist())]
        if k >= 2:
            bad = int(rng.integers(0, n))
            lines[bad] = ["12\tx3", "7", "1\t2\t3", "--4\t1"][k]
        add(f"random_{k}", "\n".join(lines) + ("\n" if k % 2 == 0 else ""))
    return out


def main():
    names, texts, ncols, status, messages, lines, cols, counts = [], [], [], [], [], [], [], []
    with tempfile.TemporaryDirectory() as tmp:
        for name, data, nc in cases():
            p = Path(tmp) / "t.tsv"
            p.write_bytes(data)
            schema = ref.Schema([(f"c{j}", "int") for j in range(nc)])
            names.append(name)
            texts.append(np.frombuffer(data, dtype=np.uint8))
            ncols.append(nc)
            try:
                t = ref.load_tsv(p, schema)
            except Exception as e:  # recorded: class, message, line
                status.append(type(e).__name__)
                messages.append(str(e))
                lines.append(int(getattr(e, "line", -1) or -1))
                cols.append(np.empty(0, np.int64))
                counts.append(0)
                continue
            status.append("ok")
            messages.append("")
            lines.append(-1)
            cols.append(np.concatenate([np.asarray(t.column(f"c{j}"), np.int64)
                                        for j in range(nc)]) if t.n_rows else np.empty(0, np.int64))
            counts.append(t.n_rows)
    text_off = np.concatenate([[0], np.cumsum([x.size for x in texts])]).astype(np.int64)
    col_off = np.concatenate([[0], np.cumsum([x.size for x in cols])]).astype(np.int64)
    np.savez_compressed(HERE / "tsv.npz", names=np.array(names), ncols=np.array(ncols),
                        status=np.array(status), messages=np.array(messages),
                        lines=np.array(lines), counts=np.array(counts),
                        texts=np.concatenate(texts), text_off=text_off,
                        cols=np.concatenate(cols), col_off=col_off)
    for n, s, m in zip(names, status, messages):
        print(f"{n:20s} {s:14s} {m[:70]}")


if __name__ == "__main__":
    main()
