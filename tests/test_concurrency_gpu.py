"""Concurrent callers ("Multiple calls may run concurrently against one immutable
model and one store"): host threads issuing prefill_with_reuse on one model, each on its own CUDA
stream, get exactly the results of the same calls made one after another.  The run uses the
deterministic split-K reduction (Runner.deterministic): without it, red.add arrival order makes
runs differ at bf16-rounding scale, which would hide a real race."""
import threading

import numpy as np
import pytest

from scenes import Scene

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu


@pytest.mark.timeout(600)
def test_two_threads_match_serial_results(cuda_ok):
    import paper_2512_12977_b200 as P
    from paper_2512_12977_b200.engine import _runner
    sc = Scene(P, "C1", 2, export=False)
    L = sc.cfg.num_layers
    runner = _runner(sc.model)
    runner.deterministic = True
    runner.graphs.clear()
    plans = [P.plan_static(0.05, L), P.RecomputePlan((0.3, 0.2, 0.1, 0.0)), P.plan_static(0.0, L),
             P.RecomputePlan((1.0, 0.1, 0.1, 0.0))]
    serial = [P.prefill_with_reuse(sc.model, sc.request(p), sc.store).logits for p in plans]
    out = {}
    errors = []

    def worker(tid):
        try:
            s = torch.cuda.Stream()
            with torch.cuda.stream(s):
                for rep in range(6):
                    k = (tid + rep) % len(plans)
                    res = P.prefill_with_reuse(sc.model, sc.request(plans[k]), sc.store)
                    out[(tid, rep)] = (k, res.logits, res.last_logits())
        except Exception as exc:           # surfaced below
            errors.append(exc)

    th = [threading.Thread(target=worker, args=(t,)) for t in range(2)]
    try:
        for t in th:
            t.start()
        for t in th:
            t.join()
    finally:
        runner.deterministic = False
        runner.graphs.clear()
    assert not errors, errors
    for (tid, rep), (k, lg, last) in out.items():
        assert np.array_equal(lg, serial[k]), (tid, rep, k, float(np.max(np.abs(lg - serial[k]))))
        assert np.array_equal(last, lg[-1])
