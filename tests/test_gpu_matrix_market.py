"""Matrix Market ingest / output against the unmodified reference (matrix_market.cpp):
the B200 reader (parallel host parse + device CSR assembly) returns bit-identical CSR for
every file form the reference accepts, the same error text and line number for the ones it
rejects, and the writer's bytes equal the reference writer's (17 significant digits)."""
import os

import numpy as np
import pytest

from paper_1403_1649_b200 import aggmg as M

from helpers import assert_csr_bits, random_sparse

pytestmark = pytest.mark.gpu

CASES = {
    "general": "%%MatrixMarket matrix coordinate real general\n% comment\n\n3 4 5\n1 1 2.5\n"
               "2 3 -1e-3\n3 4 7\n1 2 -0.0\n3 1 +4.25\n",
    "duplicates": "%%MatrixMarket matrix coordinate real general\n2 2 5\n1 1 0.1\n1 1 0.2\n"
                  "2 2 1\n1 1 0.3\n2 1 -0.0\n",
    "symmetric": "%%MatrixMarket matrix coordinate real symmetric\n3 3 4\n1 1 4\n2 1 -1\n"
                 "3 2 -1\n3 3 4\n",
    "integer": "%%MatrixMarket matrix coordinate integer general\n2 2 2\n1 2 3\n2 1 -4\n",
    "pattern": "%%MatrixMarket matrix coordinate pattern general\n2 3 3\n1 1\n2 3\n1 3\n",
    "array": "%%MatrixMarket matrix array real general\n2 2\n1.5\n0\n-2\n3\n",
    "array_sym": "%%MatrixMarket Matrix Array Real Symmetric\n3 3\n1\n2\n0\n4\n5\n6\n",
    "extra_lines": "%%MatrixMarket matrix coordinate real general\n2 2 1\n1 1 1\nnot parsed\n",
    "crlf": "%%MatrixMarket matrix coordinate real general\r\n2 2 2\r\n1 1 1.25\r\n2 2 -3\r\n",
}
ERRORS = {
    "%%MatrixMarket vector coordinate real general\n1 1 1\n1 1 1\n": "line 1: unsupported object",
    "%%MatrixMarket matrix coordinate complex general\n1 1 1\n1 1 1\n": "unsupported field",
    "%%MatrixMarket matrix coordinate real general\n2 2 3\n1 1 1\n3 1 2\n": "line 4: index out of range",
    "%%MatrixMarket matrix coordinate real symmetric\n2 2 1\n1 2 1\n": "line 3: symmetric entry above",
    "%%MatrixMarket matrix coordinate real general\n2 2 3\n1 1 1\n2 2 2\n": "line 5: unexpected end",
    "%%MatrixMarket matrix coordinate real general\n2 2 1\n1 x 1\n": "line 3: expected column index",
    "%%MatrixMarket matrix coordinate real general\n2 2 1\n1 1 abc\n": "line 3: expected numeric",
    "%%MatrixMarket matrix coordinate pattern general\n1 1 1\n1 1\n": "pattern option",
    "%%MatrixMarket matrix coordinate real general\n% only comments\n": "missing size line",
}


def test_reader_matches_reference(gpu, ref):
    for name, text in CASES.items():
        pat = name == "pattern"
        A = gpu.read_matrix_market_text(text, allow_pattern=pat)
        B = ref.read_matrix_market_text(text, allow_pattern=pat)
        assert_csr_bits(A, B, name)


def test_reader_errors_match_reference(gpu, ref):
    for text, msg in ERRORS.items():
        with pytest.raises(M.Error) as eg:
            gpu.read_matrix_market_text(text)
        with pytest.raises(M.Error) as er:
            ref.read_matrix_market_text(text)
        assert str(eg.value) == str(er.value), (str(eg.value), str(er.value))
        assert msg in str(eg.value)


def test_writer_bytes_and_round_trip(gpu, ref, tmp_path):
    A = random_sparse(400, 350, 0.03, 5)
    A.values[::7] *= 1e-300
    A.values[::11] = -0.0
    pg, pr = tmp_path / "g.mtx", tmp_path / "r.mtx"
    gpu.write_matrix_market(pg, A)
    ref.write_matrix_market(pr, A)
    assert pg.read_bytes() == pr.read_bytes()
    assert_csr_bits(gpu.read_matrix_market(pg), ref.read_matrix_market(pr), "round trip")
    x = np.random.default_rng(2).standard_normal(1000)
    gpu.write_vector_market(tmp_path / "x.mtx", x)
    ref.write_vector_market(tmp_path / "y.mtx", x)
    assert (tmp_path / "x.mtx").read_bytes() == (tmp_path / "y.mtx").read_bytes()
    assert np.array_equal(gpu.read_vector_market(tmp_path / "x.mtx").view(np.uint64), x.view(np.uint64))


def test_large_file_parallel_parse(gpu, ref, tmp_path):
    """> 4 MB of data lines: the chunked parallel parse (errors found in file order)."""
    A = gpu.generate_poisson(3, 40, 40, 40)  # 440 k entries, ~20 MB of text
    p = tmp_path / "big.mtx"
    gpu.write_matrix_market(p, A)
    assert_csr_bits(gpu.read_matrix_market(p), A, "big")
    lines = p.read_bytes().split(b"\n")
    bad = len(lines) * 3 // 4
    lines[bad] = b"1 1 nope"
    lines[bad + 1000] = b"1 1"  # a later error must not win
    q = tmp_path / "bad.mtx"
    q.write_bytes(b"\n".join(lines))
    with pytest.raises(M.Error, match=f"line {bad + 1}: expected numeric value"):
        gpu.read_matrix_market(q)
