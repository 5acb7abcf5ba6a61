"""Model check (CPU, threads) of the multi-GPU peer-memory exchange protocol of wnnc_iterate
(csrc/capi.cu:run_iterations, csrc/traverse.cu epilogue, csrc/comm.cu).

Each rank runs the iteration's steps in stream order.  A traversal stores its owned rows into EVERY rank's
replica and then signals every rank (one count per rank and exchange); a wait blocks until the rank's
counter has reached world × (exchanges so far).  Ranks run at random, independent speeds.  Every replica
row carries the version (array, iteration) of the value last stored into it, and every read asserts that
all rows hold exactly the version the algorithm needs — a row not yet written, or already overwritten by
a faster rank, fails the run.  The ping-pong μ buffers are what make the protocol race-free: with a
single μ buffer a fast rank's G epilogue overwrites the μ a slow rank's axpy (μ' = μ + αr) still reads,
and the model finds it.
"""
import random
import threading

import pytest


class Model:
    def __init__(self, world, n_rows, pingpong, seed):
        self.world, self.n, self.pingpong = world, n_rows, pingpong
        nb = 2 if pingpong else 1
        # replica[r][name] = list of per-row versions
        self.rep = [{"s": [None] * n_rows, "r": [None] * n_rows, "p0": [None] * world, "p1": [None] * world,
                     "p2": [None] * world, "acc": [None] * n_rows,
                     **{f"mu{b}": [("mu", 0)] * n_rows for b in range(nb)}}
                    for _ in range(world)]
        self.sig = [0] * world
        self.cv = threading.Condition()
        self.errors = []
        self.rng = [random.Random(seed * 100 + r) for r in range(world)]
        bounds = [round(k * n_rows / world) for k in range(world + 1)]
        self.shard = [(bounds[k], bounds[k + 1]) for k in range(world)]

    def _delay(self, rank):
        if self.rng[rank].random() < 0.3:
            threading.Event().wait(self.rng[rank].random() * 0.002)

    def _mu(self, k):
        return f"mu{k % 2}" if self.pingpong else "mu0"

    def read(self, rank, name, want, step):
        self._delay(rank)
        got = self.rep[rank][name]
        bad = [v for v in got if v != want]
        if bad:
            self.errors.append(f"rank {rank} {step}: read {name} expecting {want}, saw {bad[0]}")

    def traverse(self, rank, name, version, part):
        """owned rows into every replica (epilogue stores), block partial likewise, then signal all ranks"""
        b, e = self.shard[rank]
        for r in range(self.world):
            self._delay(rank)
            if name:
                for i in range(b, e):
                    self.rep[r][name][i] = version
            if part:
                self.rep[r][part][rank] = (part, version[1])
        with self.cv:
            for r in range(self.world):
                self.sig[r] += 1
            self.cv.notify_all()

    def scatter(self, rank, k, signal=True):
        """transpose-mode adjoint: memset + scatter of this rank's shard into its OWN accumulators (node and
        point accumulators cover every row), then signal all ranks"""
        for i in range(self.n):
            self._delay(rank)
            self.rep[rank]["acc"][i] = ("acc", k)
        if signal:
            with self.cv:
                for r in range(self.world):
                    self.sig[r] += 1
                self.cv.notify_all()

    def reduce_pushdown(self, rank, k):
        """every rank's accumulators (peer reads, rank order), then r and all Σ|r|² slots into its own replica"""
        for r in range(self.world):
            self._delay(rank)
            bad = [v for v in self.rep[r]["acc"] if v != ("acc", k)]
            if bad:
                self.errors.append(f"rank {rank} reduce: rank {r}'s accumulators expecting {('acc', k)}, saw {bad[0]}")
        for i in range(self.n):
            self.rep[rank]["r"][i] = ("r", k)
        for r in range(self.world):
            self.rep[rank]["p1"][r] = ("p1", k)

    def wait(self, rank, count):
        with self.cv:
            ok = self.cv.wait_for(lambda: self.sig[rank] >= self.world * count, timeout=10)
        if not ok:
            self.errors.append(f"rank {rank}: wait timed out")

    def run_rank(self, rank, iters, transpose=False, scatter_signal=True):
        ex = 0
        for k in range(iters):
            mu = self._mu(k)
            self.read(rank, mu, ("mu", k), "m1")                    # moments of μ
            self.read(rank, mu, ("mu", k), "A(mu) leaves")
            self.traverse(rank, "s", ("s", k), "p0")                 # s = ½ − Aμ, Σ s²
            ex += 1
            self.wait(rank, ex)
            if transpose:                                            # r = Aᵀ s by scatter + push-down
                self.read(rank, "s", ("s", k), "scatter")
                self.scatter(rank, k, signal=scatter_signal)
                if scatter_signal:
                    ex += 1
                    self.wait(rank, ex)
                self.reduce_pushdown(rank, k)
            else:
                self.read(rank, "s", ("s", k), "m2")
                self.read(rank, "s", ("s", k), "AT leaves")
                self.traverse(rank, "r", ("r", k), "p1")             # r = Aᵀ s, Σ|r|²
                ex += 1
                self.wait(rank, ex)
            self.read(rank, "r", ("r", k), "m3")
            self.traverse(rank, None, ("q", k), "p2")                # Σ (A r)²
            ex += 1
            self.wait(rank, ex)
            for p in ("p0", "p1", "p2"):
                self.read(rank, p, (p, k), "alpha")
            self.read(rank, mu, ("mu", k), "m4 axpy")                # μ' = μ + α r
            self.read(rank, "r", ("r", k), "m4 axpy")
            self.traverse(rank, self._mu(k + 1), ("mu", k + 1), None)  # G epilogue: the next μ, no partial
            ex += 1
            self.wait(rank, ex)
        self.read(rank, self._mu(iters), ("mu", iters), "result")


def _run(world, pingpong, seed, iters=6, n_rows=23, transpose=False, scatter_signal=True):
    m = Model(world, n_rows, pingpong, seed)
    th = [threading.Thread(target=m.run_rank, args=(r, iters, transpose, scatter_signal)) for r in range(world)]
    for t in th:
        t.start()
    for t in th:
        t.join()
    return m.errors


@pytest.mark.parametrize("world", [1, 2, 3, 4, 8])
def test_peer_protocol_is_race_free(world):
    for seed in range(12):
        errs = _run(world, pingpong=True, seed=seed)
        assert not errs, errs[:3]


def test_empty_shards_still_signal():
    # more ranks than rows: a rank with no queries still takes part in every exchange (k_peer_signal)
    for seed in range(6):
        assert not _run(8, pingpong=True, seed=seed, n_rows=5)


def test_single_mu_buffer_races():
    # the model is sharp enough to see the hazard the ping-pong buffers remove
    found = any(_run(4, pingpong=False, seed=s) for s in range(40))
    assert found


@pytest.mark.parametrize("world", [1, 2, 3, 8])
def test_transpose_adjoint_protocol_is_race_free(world):
    # transpose mode across ranks: each rank's own accumulators, one signal / wait, then every rank reads all
    # ranks' accumulators; a fast rank's next memset of its accumulators comes after two more exchanges
    # (Σ(Ar)², G), which a slow rank only passes once it has finished reading them
    for seed in range(12):
        errs = _run(world, pingpong=True, seed=seed, transpose=True)
        assert not errs, errs[:3]


def test_transpose_adjoint_needs_its_signal():
    # without the exchange after the scatter a rank reads a peer's accumulators before the peer wrote them
    found = any(_run(3, pingpong=True, seed=s, transpose=True, scatter_signal=False) for s in range(40))
    assert found
