"""On-device autotuner (sgnn_tune_spmm / ops.run_tuning) -- the replacement
for run_tuning (autotune.hpp:99-164): every candidate is checked bitwise
against the default plan inside the sweep; the report keeps the reference's
shape (entries per K, speedup, tie-broken best_k, skipped Ks) and round-trips
through the report.cpp CSV dialect."""
import numpy as np
import pytest

from conftest import rand_csr

pytestmark = pytest.mark.gpu


def _graph():
    from paper_2403_14853_b200 import graphs, ops
    rp, ci = graphs.rmat(13, 8192 * 16, seed=4)
    v = graphs.uniform(len(ci), -1, 1, seed=4)
    return ops.CsrMatrix.from_numpy(rp, ci, v, 8192)


def test_tune_spmm_returns_fastest_bitwise_equal_plan(cuda):
    import torch

    from paper_2403_14853_b200 import ops
    a = _graph()
    plan, table = ops.tune_spmm(a, 64, "sum", reps=3)
    assert len(table) >= 4
    assert plan.params["lanes"] in (4, 8, 16, 32)
    best = min(e["ms"] for e in table)
    assert any(e["params"] == plan.params and e["ms"] == best for e in table)
    x = torch.randn(8192, 64, device="cuda")
    np.testing.assert_array_equal(ops.spmm_plan(a, x, "sum", plan).cpu().numpy().view(np.uint32),
                                  ops.spmm_plan(a, x, "sum", ops.Plan(a, 64)).cpu().numpy().view(np.uint32))
    with pytest.raises(ops.ConfigError):
        ops.tune_spmm(a, 64, "sum", reps=2)


def test_run_tuning_report_and_csv_roundtrip(cuda, tmp_path):
    from paper_2403_14853_b200 import ops, report
    a = _graph()
    rep = ops.run_tuning(a, [32, 48, 32, 128], reps=3, graph_id="rmat13")
    assert [e.k for e in rep.entries] == [32, 128] and rep.skipped == [48]
    top = max(rep.entries, key=lambda e: (e.speedup, -e.k))
    assert rep.best_k == top.k
    for e in rep.entries:
        assert e.t_trusted_ms > 0 and e.t_specialized_ms > 0
        assert abs(e.speedup - e.t_trusted_ms / e.t_specialized_ms) < 1e-9
    path = tmp_path / "r.csv"
    report.save_report(rep, path)
    back = report.load_report(path)
    assert back.best_k == rep.best_k and back.graph_id == "rmat13" and back.skipped == [48]
    # "%.9g" (report.cpp:14-18) keeps 9 significant digits
    assert [e.k for e in back.entries] == [e.k for e in rep.entries]
    for b, e in zip(back.entries, rep.entries):
        assert b.t_trusted_ms == pytest.approx(e.t_trusted_ms, rel=1e-8)
        assert b.t_specialized_ms == pytest.approx(e.t_specialized_ms, rel=1e-8)
    assert back.plans == {k: rep.plans[k].params for k in rep.plans}
    # a tuned plan registered on the matrix is what spmm(..., specialized) uses
    a.register_plan(32, rep.plans[32])
    assert a.plan(32, "tuned") is rep.plans[32]
