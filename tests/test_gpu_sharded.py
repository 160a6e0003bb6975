"""Box-scale sharding ("sharded over G GPUs == single-GPU == oracle, byte for
byte"; the paper parallelises over independent activations).

Two rank processes share the one GPU (FDFB_SHARE_DEVICE=1, gloo for the host-side collectives;
the ranks never wait on each other inside a kernel): rank 0's keys are broadcast, each rank
encrypts its contiguous shard with global object indices and bootstraps it.  The gathered bytes
must equal one process bootstrapping the whole batch.  Single == oracle is asserted by the
sampled Large tests of test_gpu_parity.py on the same code path."""
import os
import socket
import subprocess
import sys

import numpy as np
import pytest

torch = pytest.importorskip("torch")

import synth  # noqa: E402

pytestmark = pytest.mark.gpu

if not torch.cuda.is_available():  # pragma: no cover
    pytest.skip("needs a CUDA device", allow_module_level=True)

from paper_2109_02731_b200 import Context  # noqa: E402


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


@pytest.mark.parametrize("name,total,backend,world", [("tiny", 37, "gloo", 2), ("large", 2 * 296 + 37, "gloo", 2),
                                                     ("tiny", 37, "nccl", 1)])
def test_sharded_bootstrap_equals_single_rank_bytes(name, total, backend, world, tmp_path):
    """gloo: two ranks share the GPU.  nccl: the key broadcast and output all-gather go through
    NCCL on device tensors (a world of one rank: one GPU per rank, and the box has one)."""
    here = os.path.dirname(os.path.abspath(__file__))
    port = _free_port()
    out_path = str(tmp_path / "sharded.npz")
    procs = []
    for r in range(world):
        env = dict(os.environ, RANK=str(r), WORLD_SIZE=str(world), MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port),
                   FDFB_SHARE_DEVICE="1", FDFB_TEST_BACKEND=backend)
        procs.append(subprocess.Popen([sys.executable, os.path.join(here, "sharded_worker.py"), name, str(total),
                                       out_path], env=env, stdout=subprocess.PIPE, stderr=subprocess.PIPE, text=True))
    outs = [p.communicate(timeout=900) for p in procs]
    for p, (o, e) in zip(procs, outs):
        assert p.returncode == 0, e[-3000:]
    got = np.load(out_path)
    cfg = synth.load_config(name)
    ctx = Context(cfg, 0)
    dev = torch.device("cuda", 0)
    keys = ctx.keygen(cfg["seeds"]["keys"], which=0x0F)
    msgs = synth.messages(cfg, total)
    ct = ctx.lwe_encrypt(cfg["seeds"]["err"], keys["s"], torch.from_numpy(msgs.copy()).to(dev))
    out = ctx.bootstrap_batch(keys, ctx.setup_lut(synth.lut(cfg)), ct)
    torch.cuda.synchronize()
    assert np.array_equal(got["ct"], ct.cpu().numpy())          # shards encrypt the global batch
    assert np.array_equal(got["out"], out.cpu().numpy())        # and bootstrap to the same bytes
