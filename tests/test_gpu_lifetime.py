"""GPU: device handles are released on the last reference, without waiting
for Python's cycle collector (a hierarchy is 5-6 GB at C3, so a reference
cycle would hold it until a full collection runs)."""

import gc
import weakref

import pytest
import torch


@pytest.mark.gpu
def test_handles_released_without_cycle_collector():
    from paper_2010_12879_b200 import Session, SolveConfig, amg_setup, workloads
    from paper_2010_12879_b200.pipeline import _OpRef
    w = workloads.c2_small()
    gc.collect()
    gc.disable()
    try:
        sess = Session(w.model, w.frequency_hz, SolveConfig(rel_tol=1e-8))
        vox, rep, _ = sess.snapshot(torch.from_numpy(w.a).cuda())
        assert rep.converged
        h = amg_setup(_OpRef(sess.op), SolveConfig())
        lvl = h.levels[0]
        assert lvl.aggregates.shape[0] == h.level_sizes[0]
        refs = [weakref.ref(x) for x in (sess, sess.hierarchy, sess.op, h)]
        del sess, h
        alive = [r() is not None for r in refs]
        assert alive == [False] * 4, alive
        with pytest.raises(ReferenceError):
            lvl.matrix
    finally:
        gc.enable()
