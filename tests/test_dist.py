"""Multi-rank host logic of the sharded bootstrap (paper_2109_02731_b200/dist.py) on CPU
with the gloo backend, world size 2."""
import json
import os
import socket
import subprocess
import sys

import pytest
from paper_2109_02731_b200.dist import broadcast_keys, gather_outputs, max_over_ranks, shard_range


def test_shard_range_partitions_exactly():
    for total in (0, 1, 7, 4096, 65536, 65537):
        for world in (1, 2, 3, 8):
            seen = []
            for r in range(world):
                s, c = shard_range(total, world, r)
                seen.extend(range(s, s + c))
            assert seen == list(range(total))
            counts = [shard_range(total, world, r)[1] for r in range(world)]
            assert max(counts) - min(counts) <= 1
    with pytest.raises(ValueError):
        shard_range(10, 2, 2)


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


@pytest.mark.parametrize("total", [4096, 4097])
def test_two_rank_broadcast_shard_gather(total):
    port = _free_port()
    here = os.path.dirname(os.path.abspath(__file__))
    procs = []
    for r in range(2):
        env = dict(os.environ, RANK=str(r), WORLD_SIZE="2", MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
        procs.append(subprocess.Popen([sys.executable, os.path.join(here, "dist_worker.py"), str(total)],
                                      env=env, stdout=subprocess.PIPE, stderr=subprocess.PIPE, text=True))
    outs = [p.communicate(timeout=300) for p in procs]
    for p, (o, e) in zip(procs, outs):
        assert p.returncode == 0, e[-2000:]
        res = json.loads(o.strip().splitlines()[-1])
        assert res["keys"] and res["gather"] and res["max"] == 11.0, res
