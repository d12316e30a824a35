"""Demand-driven oracle: the same plain definition as pmg_oracle.evaluate, evaluated only at the points a
set of requested liveout points depends on — TEST INFRASTRUCTURE ONLY (see pmg_oracle.py header).

Used by the full-size parity tests (BASELINE.json sizes, e.g. Harris 6400x6400, local Laplacian
2560x1536x8 planes), where evaluating every stage over its whole domain would take minutes.

Definition followed (§2.2; reading R1): the value of stage S at point p is
expr_S evaluated at p, every read P(q) := P[clamp(q, domain(P))].  Nothing about the arithmetic changes:
each needed point is computed by the Evaluator's own expression semantics (pmg_oracle.Evaluator._ev), on
1-D arrays of points instead of whole-domain grids.

Steps:
  1. backward, consumers before producers (reverse topological order): the needed points of every stage
     are the clamped read coordinates of its consumers' needed points.  An index expression that itself
     reads data (the local Laplacian's intensity-dependent plane index) cannot be evaluated before the
     data exist, so that dimension is taken whole (a superset: every plane);
  2. forward, topological order: evaluate each stage at its needed points; reads of other stages look the
     value up among the producer's computed points (which step 1 guarantees contain every read).

Pinned in tests/test_oracle.py against pmg_oracle.evaluate at random points of small images (every
pipeline), which is the definition it restates."""
from __future__ import annotations

import numpy as np

from .pmg_oracle import Access, Bin, Call, Evaluator, TableRead, Un, _V, parse


def _reads_data(e) -> bool:
    if isinstance(e, (Access, TableRead)):
        return True
    if isinstance(e, Call):
        return any(_reads_data(a) for a in e.args)
    if isinstance(e, Bin):
        return _reads_data(e.a) or _reads_data(e.b)
    if isinstance(e, Un):
        return _reads_data(e.a)
    return False


def _accesses(e, out):
    """Accesses of a stage expression, outermost first (nested index reads included)."""
    if isinstance(e, Access):
        out.append(e)
        for a in e.args:
            _accesses(a, out)
    elif isinstance(e, TableRead):
        _accesses(e.index, out)
    elif isinstance(e, Call):
        for a in e.args:
            _accesses(a, out)
    elif isinstance(e, Bin):
        _accesses(e.a, out)
        _accesses(e.b, out)
    elif isinstance(e, Un):
        _accesses(e.a, out)


class _Sparse:
    """A stage known at a sorted set of linear indices."""

    def __init__(self, shape, lin):
        self.shape = tuple(shape)
        self.lin = lin
        self.vals = None


class PointEvaluator(Evaluator):
    def __init__(self, prog, params, precision="f32"):
        super().__init__(prog, params, precision)
        self.sparse = {}

    def _coords(self, name, lin):
        return np.unravel_index(lin, self.shape_of(name))

    def _env(self, name, lin):
        s = self.p.stages[name]
        return {v: _V(c.astype(np.int32), "i") for v, c in zip(s.vars, self._coords(name, lin))}

    # step 1: needed points (backward)
    def _needed(self, liveout, points):
        shape = self.shape_of(liveout)
        need = {liveout: [np.ravel_multi_index(tuple(np.asarray(c) for c in points), shape)]}
        for name in reversed(self.p.topo_order()):
            if name not in need:
                continue
            lin = np.unique(np.concatenate(need.pop(name)))
            self.sparse[name] = _Sparse(self.shape_of(name), lin)
            env = self._env(name, lin)
            accs = []
            _accesses(self.p.stages[name].expr, accs)
            for a in accs:
                if a.target not in self.p.stages:
                    continue
                pshape = self.shape_of(a.target)
                cols = []
                for d, ie in enumerate(a.args):
                    if _reads_data(ie):
                        cols.append(None)                   # data-dependent: the whole dimension
                        continue
                    iv = self._ev(ie, env)
                    cols.append(np.clip(np.broadcast_to(np.asarray(iv.a, dtype=np.int64), lin.shape), 0, pshape[d] - 1))
                n = lin.shape[0]
                for d, c in enumerate(cols):
                    if c is None:
                        full = np.arange(pshape[d], dtype=np.int64)
                        cols = [np.repeat(x, pshape[d]) if x is not None else None for x in cols]
                        cols[d] = np.tile(full, n)
                        n *= pshape[d]
                need.setdefault(a.target, []).append(np.ravel_multi_index(tuple(cols), pshape))

    # step 2: evaluate (forward); reads of sparse stages are lookups
    def _ev(self, e, env):
        if isinstance(e, Access) and e.target in self.sparse:
            sp = self.sparse[e.target]
            idx = []
            for d, a in enumerate(e.args):
                iv = self._ev(a, env)
                idx.append(np.clip(np.asarray(iv.a, dtype=np.int64), 0, sp.shape[d] - 1))
            idx = np.broadcast_arrays(*idx)
            lin = np.ravel_multi_index(tuple(idx), sp.shape)
            pos = np.searchsorted(sp.lin, lin)
            pos = np.minimum(pos, sp.lin.shape[0] - 1)
            if not np.all(sp.lin[pos] == lin):
                raise AssertionError(f"point oracle: read of {e.target} outside its needed set")
            return self._read(e.target, sp.vals[pos])
        return super()._ev(e, env)

    def run_points(self, inputs, liveout, points):
        for name in list(self.p.images) + list(self.p.tables):
            self.values[name] = np.asarray(inputs[name])
        self._needed(liveout, points)
        for name in self.p.topo_order():
            if name not in self.sparse:
                continue
            sp = self.sparse[name]
            val = self._ev(self.p.stages[name].expr, self._env(name, sp.lin))
            sp.vals = np.broadcast_to(self._store(val, self.p.stages[name].dtype), sp.lin.shape).copy()
        shape = self.shape_of(liveout)
        lin = np.ravel_multi_index(tuple(np.asarray(c) for c in points), shape)
        sp = self.sparse[liveout]
        return sp.vals[np.searchsorted(sp.lin, lin)]


def evaluate_points(text_or_prog, params: dict, inputs: dict, liveout: str, points, precision: str = "f32"):
    """Values of `liveout` at `points` (a tuple of coordinate arrays, one per dimension, outermost first)."""
    prog = parse(text_or_prog) if isinstance(text_or_prog, str) else text_or_prog
    return PointEvaluator(prog, params, precision).run_points(inputs, liveout, points)
