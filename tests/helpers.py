"""Test-only back-ends (mirrors of the reference's test fakes)."""
import threading
import time

import numpy as np

import oracle as O
import paper_2502_11129_b200 as hb


class OracleExecutor(hb.BatchExecutor):
    """CPU back-end over the C restatement (tests only; never the product)."""

    def __init__(self, threads=2):
        self.threads = threads

    def name(self):
        return "oracle"

    def run(self, request):
        hb.validate_request(request)
        t0 = time.perf_counter()
        b = O.simulate_batch(int(request.kind), request.seeds, request.steps, self.threads)
        if np.any(b.fail_step):
            bad = np.nonzero(b.fail_step)[0]
            raise hb.BatchFailure([(int(request.seeds[i]), O.blowup_message(int(request.seeds[i]),
                                                                             int(b.fail_step[i])))
                                   for i in bad], b.results[b.fail_step == 0])
        return hb.BatchResult(b.results, max(time.perf_counter() - t0, 1e-9), [])


class StubExecutor(hb.BatchExecutor):
    """test_scheduler.cpp:16-42: fixed wall, optional sleep or failure."""

    def __init__(self, wall, sleep_s=0.0, fail=False):
        self.wall, self.sleep_s, self.fail = wall, sleep_s, fail
        self.calls = 0
        self._lock = threading.Lock()

    def name(self):
        return "stub"

    def run(self, request):
        with self._lock:
            self.calls += 1
        if self.fail:
            raise RuntimeError("stub back-end failure")
        if self.sleep_s > 0:
            time.sleep(self.sleep_s)
        n = len(request.seeds)
        r = np.zeros(n, dtype=hb.RESULT_DTYPE)
        r["seed"] = request.seeds
        r["checksum"] = request.seeds ^ np.uint64(0xABCD)
        r["steps_executed"] = request.steps
        return hb.BatchResult(r, self.wall, [])


class FailingExecutor(hb.BatchExecutor):
    def name(self):
        return "broken"

    def run(self, request):
        raise RuntimeError("executor down")


class NoisyStubExecutor(StubExecutor):
    """StubExecutor whose reported wall is base x (1 + U(-noise, noise)),
    seeded: the timing jitter of identical devices."""

    def __init__(self, wall, noise=0.03, seed=0):
        super().__init__(wall)
        self.noise = noise
        self.rng = np.random.default_rng(seed)

    def run(self, request):
        r = super().run(request)
        r.wall_time_s = self.wall * (1.0 + self.rng.uniform(-self.noise, self.noise))
        return r
