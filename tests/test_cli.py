"""CLI / report parity with the reference CLI (golden files produced by the
real reference): partition reports byte-identical (CPU); spmm-bench ledger,
metrics and confront reports byte-identical (GPU: the multiply runs on the
device); error JSON + exit code 2."""

import json
import os

import numpy as np
import pytest

from paper_2504_04673_b200.cli import main
from conftest import Golden


def _run(tmp_path, name, g):
    argv = [str(x) for x in g[name + "__argv"]]
    assert main(argv + ["--out-dir", str(tmp_path)]) == 0
    return sorted(k.split("__", 1)[1] for k in g.z.files if k.startswith(name + "__")
                  and not k.endswith("__argv"))


@pytest.mark.parametrize("name", ["part_gvb", "part_block"])
def test_partition_reports_byte_identical(tmp_path, name):
    g = Golden("cli_golden.npz")
    for fn in _run(tmp_path, name, g):
        assert open(os.path.join(tmp_path, fn), "rb").read() == g[f"{name}__{fn}"].tobytes(), fn


@pytest.mark.gpu
@pytest.mark.parametrize("name", ["spmm_15d", "spmm_1d_obl", "spmm_1d_rand"])
def test_spmm_bench_reports_byte_identical(tmp_path, name):
    g = Golden("cli_golden.npz")
    for fn in _run(tmp_path, name, g):
        assert open(os.path.join(tmp_path, fn), "rb").read() == g[f"{name}__{fn}"].tobytes(), fn


def test_cli_errors_exit_2_with_json(capsys, tmp_path):
    rc = main(["spmm-bench", "--gen", "sbm", "--n", "40", "--p", "6", "--c", "2",
               "--variant", "15d-sparse", "--out-dir", str(tmp_path)])
    assert rc == 2
    err = json.loads(capsys.readouterr().err)
    assert "c*c to divide p" in err["error"] and err["p"] == 6
    rc = main(["partition", "--graph", str(tmp_path / "missing.mtx"), "--k", "2",
               "--out-dir", str(tmp_path)])
    assert rc == 2
    assert "cannot read graph file" in json.loads(capsys.readouterr().err)["error"]


def test_matrix_market_roundtrip(tmp_path):
    from paper_2504_04673_b200 import io
    from paper_2504_04673_b200.graphgen import star_augmented
    a = star_augmented(60, seed=2)
    io.save_matrix_market(tmp_path / "g.mtx", a)
    b = io.load_matrix_market(tmp_path / "g.mtx")
    assert np.array_equal(a.col_idx, b.col_idx) and np.array_equal(a.values, b.values)
    io.save_edge_list_tsv(tmp_path / "g.tsv", a)
    c = io.load_edge_list_tsv(tmp_path / "g.tsv")
    assert np.array_equal(a.row_ptr, c.row_ptr)
    with pytest.raises(io.ParseError, match="missing %%MatrixMarket"):
        (tmp_path / "bad.mtx").write_text("1 1 1\n")
        io.load_matrix_market(tmp_path / "bad.mtx")
