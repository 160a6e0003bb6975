"""Host-side logic of bench.py (no GPU): the algorithmic work counts behind the roofline,
the modmul slot normalisation, the Box-scale sharding and the reference arm's JSON line."""
import json
import os
import subprocess
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import bench  # noqa: E402
import synth  # noqa: E402


def test_algorithmic_work_matches_design_counts():
    """DESIGN.md §7 / SURVEY §8(d.3): one Large CMux is (2l+2) NTTs of (N/2) log2 N butterflies
    plus 2l * 2 * N MACs = 145,408 modmul; a Large bootstrap is (l_boot + 1) n u = 12,288 CMux."""
    cfg = synth.load_config("large")
    per_cmux, cmux_per_bs = bench.algorithmic_work(cfg)
    assert per_cmux == (2 * 4 + 2) * (2048 // 2) * 11 + 2 * 4 * 2 * 2048 == 145408
    assert cmux_per_bs == (5 + 1) * 1024 * 2 == 12288
    tiny = synth.load_config("tiny")
    assert bench.algorithmic_work(tiny) == ((2 * 3 + 2) * 128 * 8 + 2 * 3 * 2 * 256, (3 + 1) * 64 * 1)


def test_modmul_slot_normalisation_by_word_size():
    assert bench.imad_per_modmul(synth.load_config("large")) == 16
    assert bench.imad_per_modmul(synth.load_config("fhew")) == 6      # 2^31 <= Q < 2^32: 64-bit Shoup
    assert bench.imad_per_modmul(synth.load_config("tiny")) == 4


def test_box_scale_sharding_covers_65536():
    from paper_2109_02731_b200.dist import shard_range
    for world in (1, 2, 4, 8):
        per = 65536 // world
        spans = [shard_range(per * world, world, r) for r in range(world)]
        assert [c for _, c in spans] == [per] * world
        assert spans[0][0] == 0 and spans[-1][0] + spans[-1][1] == 65536


@pytest.mark.timeout(300)
def test_reference_arm_prints_the_contract_line():
    """--impl reference (the CPU oracle on a bounded sample) prints one JSON line with the keys
    the driver reads; small sample so the CPU suite stays fast."""
    out = subprocess.run([sys.executable, os.path.join(ROOT, "bench.py"), "--impl", "reference", "--steps", "1",
                          "--warmup", "3", "--cpu-seconds", "2"], capture_output=True, text=True, timeout=280,
                         cwd=ROOT)
    assert out.returncode == 0, out.stderr[-2000:]
    line = json.loads(out.stdout.strip().splitlines()[-1])
    for key in ("impl", "metric", "value", "unit", "n_gpus", "steps", "warmup", "ms_per_step", "higher_is_better",
                "scaling", "vs_baseline", "dtype", "data", "config", "cpu_baseline", "e2e"):
        assert key in line, key
    assert line["impl"] == "reference" and line["value"] > 0
    assert line["cpu_baseline"]["kind"] == "oracle" and line["cpu_baseline"]["cores"] >= 1
    assert line["e2e"]["h2d_bytes_per_step"] == 0 and line["e2e"]["value"] == line["value"]


def test_reference_arm_config_matches_gpu_arm_and_times_its_sample():
    """Both arms print the same config dict (bootstrap_config), and the reference arm's
    ms_per_step is the measured duration of its (bounded) sample step, not a projection."""
    out = subprocess.run([sys.executable, os.path.join(ROOT, "bench.py"), "--impl", "reference", "--steps", "2",
                          "--warmup", "3", "--cpu-seconds", "2"], capture_output=True, text=True, timeout=280,
                         cwd=ROOT)
    assert out.returncode == 0, out.stderr[-2000:]
    line = json.loads(out.stdout.strip().splitlines()[-1])
    assert line["config"] == bench.bootstrap_config(synth.load_config("large"), 4096, 1)
    assert 0.5 < line["ms_per_step"] / 1000.0 < 60.0
    assert line["steps"] == 2
