"""Input side: the product's multithreaded host CSV
loader and median-of-ratios offsets against the reference's own load_counts
(P:src/io.cpp:125-164) and estimate_offsets (P:src/model.cpp:21-68), run
from oracle/_ref.  Host-only code, so these run without a GPU.  The bar is
exact: identical counts, labels, duplicate flag and LoadError message; the
offsets bit-identical."""
import numpy as np
import pytest

import oracle
from paper_1606_06659_b200 import (CountMatrix, LoadError, NormalizationError,
                                   estimate_offsets, load_counts)

from helpers import heterosis, mismatch

pytestmark = pytest.mark.usefixtures("ref")


def _write(tmp_path, text, name="counts.csv", binary=False):
    p = tmp_path / name
    if binary:
        p.write_bytes(text)
    else:
        p.write_text(text)
    return str(p)


def _csv(counts, genes=None, samples=None, crlf=False):
    G, N = counts.shape
    genes = genes or [f"gene{g + 1}" for g in range(G)]
    samples = samples or [f"s{n + 1}" for n in range(N)]
    nl = "\r\n" if crlf else "\n"
    rows = ["gene," + ",".join(samples)]
    rows += [genes[g] + "," + ",".join(str(v) for v in counts[g]) for g in range(G)]
    return nl.join(rows) + nl


def _same_as_reference(path):
    ours = load_counts(path)
    rc, rg, rs, rd = oracle.ref_load_counts(path)
    assert np.array_equal(ours.counts, rc)
    assert ours.genes == rg and ours.samples == rs
    assert ours.duplicate_genes == rd
    return ours


def _same_error(path):
    with pytest.raises(oracle.RefLoadError) as ref_e:
        oracle.ref_load_counts(path)
    with pytest.raises(LoadError) as our_e:
        load_counts(path)
    assert str(our_e.value) == str(ref_e.value)
    return str(our_e.value)


def test_load_simulated_matrix(tmp_path):
    counts, _, _ = heterosis(5000, seed=4)
    m = _same_as_reference(_write(tmp_path, _csv(counts)))
    assert m.counts.shape == (5000, 16) and not m.duplicate_genes


def test_load_quoting_crlf_blank_rows_and_duplicates(tmp_path):
    text = ('"gene","s,1","s""2",s3\r\n'
            '"a,b",1,2,3\r\n'
            '\r\n'
            'x"y,4,5,6\r\n'
            '\n'
            '"a,b",7,8,9\r\n'
            '"q""""",0,0,9223372036854775807')  # no trailing newline
    m = _same_as_reference(_write(tmp_path, text))
    assert m.samples == ["s,1", 's"2', "s3"]
    assert m.genes == ["a,b", 'x"y', "a,b", 'q""']
    assert m.duplicate_genes
    assert m.counts[-1, -1] == 2**63 - 1


def test_load_many_rows_parallel_parse(tmp_path):
    rng = np.random.default_rng(3)
    counts = rng.integers(0, 10**12, size=(60000, 7))
    m = _same_as_reference(_write(tmp_path, _csv(counts, crlf=True)))
    assert np.array_equal(m.counts, counts)


@pytest.mark.parametrize("text", [
    "",                                   # empty file
    "\n",                                 # header with a single (empty) cell
    "gene\n",                             # no sample columns
    "gene,s1,s2\n",                       # no gene rows
    "gene,s1,s2\n\n\n",                   # only blank rows
    "gene,s1,s2\ng1,1\n",                 # too few cells
    "gene,s1,s2\ng1,1,2,3\n",             # too many cells
    "gene,s1,s2\ng1,1,x\n",               # non-integer
    "gene,s1,s2\ng1,1, 2\n",              # leading blank: strtoll skips it (valid)
    "gene,s1,s2\ng1,1,2 \n",              # trailing garbage
    "gene,s1,s2\ng1,1,\n",                # empty cell
    "gene,s1,s2\ng1,1,-3\n",              # negative
    "gene,s1,s2\ng1,1,99999999999999999999\n",  # overflow (ERANGE)
    "gene,s1,s2\ng1,1,2.5\n",             # real
    "gene,s1,s2\ng1,1,0x10\n",            # base-10 only
])
def test_load_errors_match_reference(tmp_path, text):
    path = _write(tmp_path, text)
    try:
        ref = oracle.ref_load_counts(path)
    except oracle.RefLoadError:
        _same_error(path)
        return
    ours = load_counts(path)
    assert np.array_equal(ours.counts, ref[0]) and ours.genes == ref[1]


def test_first_bad_row_in_file_order_wins(tmp_path):
    # bad rows spread over the parallel parse chunks: the reference throws on
    # the first one in file order, and so must we
    counts = np.ones((40000, 4), dtype=np.int64)
    lines = _csv(counts).splitlines()
    lines[30001] = "late,1,2,3,x"
    lines[20001] = "middle,1,2"
    lines[25001] = "other,-1,2,3,4"
    msg = _same_error(_write(tmp_path, "\n".join(lines) + "\n"))
    assert msg == "row 20002 has 3 cells, expected 5"


def test_missing_file(tmp_path):
    with pytest.raises(LoadError, match="cannot open counts file"):
        load_counts(str(tmp_path / "absent.csv"))


@pytest.mark.parametrize("G,N,seed", [(1, 1, 0), (2, 16, 1), (3, 5, 2), (2000, 16, 3),
                                      (20001, 12, 4)])
def test_offsets_bit_identical(G, N, seed):
    rng = np.random.default_rng(seed)
    counts = rng.poisson(rng.gamma(2.0, 50.0, size=(G, 1)) * rng.uniform(0.5, 2, size=(1, N)))
    counts[rng.random(size=counts.shape) < 0.05] = 0
    counts[0] = np.maximum(counts[0], 1)  # at least one gene positive everywhere
    ours = estimate_offsets(CountMatrix(counts))
    ref = oracle.ref_estimate_offsets(counts)
    assert not len(mismatch(ours, ref))


def test_offsets_large_counts():
    # counts past the memoised log range go through log() directly
    rng = np.random.default_rng(7)
    counts = rng.integers(1, 10**9, size=(3001, 9))
    counts[::3] = rng.integers(1, 70000, size=counts[::3].shape)
    assert not len(mismatch(estimate_offsets(counts), oracle.ref_estimate_offsets(counts)))


def test_offsets_simulated_heterosis_shape():
    counts, _, h = heterosis(39656, seed=1)
    ours = estimate_offsets(counts)
    assert not len(mismatch(ours, oracle.ref_estimate_offsets(counts)))
    assert abs(ours.sum()) < 1e-12


def test_offsets_even_and_odd_kept_counts():
    # k odd -> middle ratio; k even -> midpoint of the two middle ratios
    for G in (4, 5):
        counts = np.arange(1, 1 + G * 3, dtype=np.int64).reshape(G, 3) ** 2
        assert not len(mismatch(estimate_offsets(counts), oracle.ref_estimate_offsets(counts)))


def test_offsets_need_a_gene_positive_everywhere():
    counts = np.array([[0, 1], [1, 0]])
    with pytest.raises(oracle.ConfigErr) as ref_e:
        oracle.ref_estimate_offsets(counts)
    with pytest.raises(NormalizationError) as our_e:
        estimate_offsets(counts)
    assert str(our_e.value) == str(ref_e.value)


def test_loaded_file_drives_offsets(tmp_path):
    counts, _, _ = heterosis(3000, seed=9)
    m = load_counts(_write(tmp_path, _csv(counts)))
    assert not len(mismatch(estimate_offsets(m), oracle.ref_estimate_offsets(counts)))


# ---- load_model_matrix / load_offsets (P:src/io.cpp:178-243)

def _same_table(path, which, fn):
    try:
        ref = oracle.ref_load_table(path, which)
    except oracle.RefLoadError as e:
        with pytest.raises(LoadError) as ours:
            fn(path)
        assert str(ours.value) == str(e)
        return None
    got = fn(path)
    got = got.X if which == 0 else got[:, None]
    assert got.shape == ref.shape and not len(mismatch(got.ravel(), ref.ravel()))
    return got


@pytest.mark.parametrize("text", [
    "a,b,c\n1,0,1\n1,1,-1\n1,-1,0.5\n",
    "\"x,1\",y\r\n1,2.5e-3\r\n\r\n1,-0x1p3\r\n1, 7\n",   # quoted header, CRLF, hex, blank
    "a,b\n1,inf\n1,nan\n",                             # strtod accepts these (validation is later)
    "",
    "a,b\n",
    "a,b\n1,2,3\n",
    "a,b\n1,x\n",
    "a,b\n1,\n",
    "a,b\n1,2 \n",
])
def test_model_matrix_loader_matches_reference(tmp_path, text):
    from paper_1606_06659_b200 import load_model_matrix
    p = _write(tmp_path, text)
    got = _same_table(p, 0, load_model_matrix)
    if got is not None and text.startswith('"x,1"'):
        assert load_model_matrix(p).effects == ["x,1", "y"]


@pytest.mark.parametrize("text", [
    "sample,offset\ns1,0.1\ns2,-0.25\n\ns3,1e-300\n",
    "sample,offset\r\n\"s,1\",2\r\n",
    "",
    "sample,offset\n",
    "sample,offset\ns1\n",
    "sample,offset\ns1,0.1,3\n",
    "sample,offset\ns1,abc\n",
])
def test_offsets_loader_matches_reference(tmp_path, text):
    from paper_1606_06659_b200 import load_offsets
    p = _write(tmp_path, text)
    _same_table(p, 1, load_offsets)


def test_table_loaders_missing_files(tmp_path):
    from paper_1606_06659_b200 import load_model_matrix, load_offsets
    with pytest.raises(LoadError, match="cannot open model matrix file"):
        load_model_matrix(str(tmp_path / "no.csv"))
    with pytest.raises(LoadError, match="cannot open offsets file"):
        load_offsets(str(tmp_path / "no.csv"))
