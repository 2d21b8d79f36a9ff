"""bench.py host-side helpers (no GPU): the communication object of the bench
line follows the reference's accounting (CommStats; bench.cpp:79-87)."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import bench  # noqa: E402


class _Ex:
    def __init__(self, ar, rd, mx):
        self._s = {"allreduce_volume": ar, "redistribute_volume": rd, "max_rank_sent": mx}

    def stats(self):
        return dict(self._s)


def test_communication_sums_modes_against_the_bound():
    c = bench._communication([_Ex(3072, 0, 1024), _Ex(0, 134217728, 33554432)], 2.0e8)
    assert c["allreduce_elems"] == 3072 and c["redistribute_elems"] == 134217728
    assert c["volume_total_elems"] == 134220800
    assert c["volume_total_bytes"] == 8 * 134220800
    assert c["max_rank_sent_bytes"] == 8 * (1024 + 33554432)
    assert abs(c["volume_to_bound_ratio"] - 134220800 / 2.0e8) < 1e-12


def test_communication_without_a_bound():
    c = bench._communication([_Ex(0, 0, 0)], 0.0)
    assert c["volume_total_elems"] == 0 and c["volume_to_bound_ratio"] is None


def _bench(args, env_extra=None):
    import subprocess
    env = dict(os.environ)
    env.pop("WORLD_SIZE", None)
    env.update(env_extra or {})
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    return subprocess.run([sys.executable, os.path.join(root, "bench.py"), *args],
                          capture_output=True, text=True, timeout=300, env=env)


def test_gpus_n_refuses_a_box_with_fewer_gpus():
    """`bench.py --gpus 2` never prints an n_gpus=1 line: on a box with fewer
    GPUs (none here) it exits 2 with the reason on stderr."""
    r = _bench(["--gpus", "2", "--steps", "1", "--warmup", "1"])
    assert r.returncode == 2, (r.returncode, r.stderr[-500:])
    assert "needs 2 GPUs" in r.stderr
    assert not [l for l in r.stdout.splitlines() if l.startswith("{")]


def test_gpus_must_match_world_size():
    """Launched under torchrun, --gpus and WORLD_SIZE must agree."""
    r = _bench(["--gpus", "2", "--steps", "1", "--warmup", "1"],
               {"WORLD_SIZE": "4", "RANK": "0", "LOCAL_RANK": "0"})
    assert r.returncode == 2, (r.returncode, r.stderr[-500:])
    assert "WORLD_SIZE=4" in r.stderr
