"""A deterministic CPU stand-in for B200Runner used by the CPU tests of the
sharding logic (multigpu.ShardedRunner): test infrastructure only."""
import zlib


class FakeRunner:
    def __init__(self, device=0, fail_on=None, **opts):
        self.device = device
        self.fail_on = fail_on
        self.e0 = None
        self.workloads = 0

    def set_workload(self, e0, inputs=None):
        self.e0 = e0
        self.workloads += 1

    def _result(self, text):
        return {"status": "OK", "family": "fake", "repeats": 1, "cfg": [0] * 13,
                "latency_ns": 1000.0 + zlib.crc32(text.encode()) % 9000, "max_abs_err": 0.0,
                "mismatches": 0, "workloads": self.workloads}

    def measure_programs(self, texts):
        if self.fail_on is not None and any(self.fail_on in t for t in texts):
            raise ValueError(f"device {self.device}: injected failure")
        return [self._result(t) for t in texts]

    def baseline_result(self):
        return self._result("e0")

    def elapsed_ms(self):
        return 0.0

    def launch_count(self):
        return 0


def fake_factory(device, **opts):
    return FakeRunner(device, **opts)
