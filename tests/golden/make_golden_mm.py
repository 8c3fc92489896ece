"""Golden Matrix Market parses from the UNMODIFIED reference (run in the build container).

    python tests/golden/make_golden_mm.py   # writes tests/golden/reference_mm_golden.json

Each case is a text fed to kernelpick.sparse.parse_matrix_market (sparse.py:106-196); the
JSON stores either the canonical CSR (offsets, cols, values as float.hex) or the exact
ParseError message.
"""
import json
import os
import sys

OUT = os.path.join(os.path.dirname(os.path.abspath(__file__)), "reference_mm_golden.json")
H = "%%MatrixMarket matrix coordinate real general\n"
CASES = {
    "general": H + "% comment\n\n3 4 4\n1 1 1.5\n3 4 -2e-3\n1 1 0.25\n2 3 7\n",
    "crlf_and_cr": "%%MatrixMarket matrix coordinate real general\r\n3 3 2\r\n1 2 1.0\r3 3 2.5\r\n",
    "vt_ff_breaks": "%%MatrixMarket matrix coordinate real general\n2 2 2\x0b1 1 1\x0c2 2 2\n",
    "unicode_breaks": "%%MatrixMarket matrix coordinate real general\n2 2 2 1 1 1\x852 2 2 ",
    "fs_gs_rs_breaks": "%%MatrixMarket matrix coordinate real general\x1c2 2 2\x1d1 1 1\x1e2 2 2\n",
    "symmetric": "%%MatrixMarket matrix coordinate real symmetric\n3 3 3\n2 1 4.0\n3 3 1.5\n3 1 -1\n",
    "skew": "%%MatrixMarket matrix coordinate real skew-symmetric\n3 3 2\n2 1 4.0\n3 2 0.5\n",
    "pattern": "%%MatrixMarket matrix coordinate pattern general\n2 3 3\n1 1\n2 3\n1 1\n",
    "integer_field": "%%MatrixMarket matrix coordinate integer symmetric\n2 2 2\n1 1 3\n2 1 -4\n",
    "header_case_ws": "  %%MATRIXMARKET  Matrix COORDINATE Real GENERAL  \n 2   2  1 \n\t1\t2\t 5.5  \n",
    "float_forms": H + "2 9 9\n1 1 1_000.5\n1 2 .5\n1 3 5.\n1 4 +1E+2\n1 5 -0.0\n1 6 1e-400\n1 7 1e1_0\n"
                       "1 8 0.1\n2 9 3.141592653589793238462643383279\n",
    "int_forms": H + "3 3 3\n+1 0_1 1\n003 2 2\n2 +3 3\n",
    "dup_heavy": H + "2 2 10\n" + "1 1 0.1\n" * 9 + "2 2 1\n",
    "empty_matrix": H + "4 5 0\n",
    "trailing_comments": H + "2 2 1\n% c\n1 1 1\n%end\n\n",
    "no_final_newline": H + "2 2 2\n1 1 1\n2 2 2",
    # errors
    "err_empty": "",
    "err_header": "%%MatrixMarket matrix coordinate real\n1 1 0\n",
    "err_object": "%%MatrixMarket vector coordinate real general\n",
    "err_format": "%%MatrixMarket matrix array real general\n",
    "err_field": "%%MatrixMarket matrix coordinate complex general\n",
    "err_symmetry": "%%MatrixMarket matrix coordinate real hermitian\n",
    "err_no_size": "%%MatrixMarket matrix coordinate real general\n% only comments\n\n",
    "err_header_only": "%%MatrixMarket matrix coordinate real general\n",
    "err_size_fields": H + "3 3\n",
    "err_size_int": H + "3 x 1\n",
    "err_size_neg": H + "3 -3 1\n",
    "err_fields": H + "2 2 1\n1 1\n",
    "err_malformed": H + "2 2 1\n1 1 abc\n",
    "err_hex": H + "2 2 1\n1 1 0x1p3\n",
    "err_nonfinite": H + "2 2 1\n1 1 inf\n",
    "err_nan": H + "2 2 1\n1 1 NaN\n",
    "err_overflow_value": H + "2 2 1\n1 1 1e400\n",
    "err_range": H + "2 2 1\n3 1 1.0\n",
    "err_range0": H + "2 2 1\n0 1 1.0\n",
    "err_skew_diag": "%%MatrixMarket matrix coordinate real skew-symmetric\n2 2 1\n1 1 1.0\n",
    "err_extra": H + "2 2 1\n1 1 1\n2 2 2\n",
    "err_truncated": H + "2 2 3\n1 1 1\n2 2 2\n",
    "err_truncated_trailing_blank": H + "2 2 3\n1 1 1\n\n\n",
    "err_underscore": H + "2 2 1\n1 1 1__0\n",
    "err_float_exp": H + "2 2 1\n1 1 1e\n",
    "err_late": H + "3 3 5\n1 1 1\n2 2 2\n3 3 3\n1 2 4\n1 3 x\n",
    "err_quote_in_entry": H + "2 2 1\n1 1 it's\n",
}


def long_case(n_lines: int = 30000, seed: int = 7) -> str:
    """A larger file (several parser chunks): symmetric, comments and blank lines mixed in,
    duplicates; regenerated identically by the tests."""
    import random
    rnd = random.Random(seed)
    out = ["%%MatrixMarket matrix coordinate real symmetric", "% generated", f"500 500 {n_lines}"]
    for k in range(n_lines):
        i = rnd.randint(1, 500)
        j = rnd.randint(1, i)
        out.append(f"{i} {j} {rnd.uniform(-10, 10)!r}")
        if k % 97 == 0:
            out.append("% mid comment")
        if k % 131 == 0:
            out.append("")
    return "\r\n".join(out) + "\r\n"


def main():
    sys.path.insert(0, "/root/reference/pkg/src")
    os.environ["KERNELPICK_PURE_KERNELS"] = "1"
    from kernelpick import errors, sparse
    out = {}
    cases = dict(CASES)
    cases["long_symmetric_crlf"] = long_case()
    for name, text in cases.items():
        rec = {} if name == "long_symmetric_crlf" else {"text": text}
        try:
            m = sparse.parse_matrix_market(text)
            rec.update({"row_offsets": [int(v) for v in m.row_offsets], "col_indices": [int(v) for v in m.col_indices],
                        "values": [float(v).hex() for v in m.values], "n_rows": m.n_rows, "n_cols": m.n_cols})
        except errors.ParseError as e:
            rec["error"] = str(e)
        out[name] = rec
    with open(OUT, "w") as f:
        json.dump({"generator": "tests/golden/make_golden_mm.py",
                   "reference": "kernelpick.sparse.parse_matrix_market (sparse.py:106-196)", "cases": out}, f)
    print(f"wrote {len(out)} cases")


if __name__ == "__main__":
    main()
