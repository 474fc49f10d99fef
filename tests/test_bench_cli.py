"""bench.py command-line contract on CPU (no GPU needed): `--gpus N` without a torchrun environment
re-launches itself under torch.distributed.run and fails loudly (one JSON error line, exit 2) when
fewer than N GPUs are visible -- never a silent 1-rank run reported as N."""
import json
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def test_gpus_n_without_torchrun_fails_loudly_on_too_few_gpus():
    env = {k: v for k, v in os.environ.items() if k not in ("WORLD_SIZE", "RANK", "LOCAL_RANK")}
    env["CUDA_VISIBLE_DEVICES"] = ""
    r = subprocess.run([sys.executable, os.path.join(ROOT, "bench.py"), "--gpus", "2", "--steps", "1", "--warmup", "3"],
                       capture_output=True, text=True, env=env, timeout=300)
    assert r.returncode == 2, (r.returncode, r.stdout[-500:], r.stderr[-500:])
    line = json.loads(r.stdout.strip().splitlines()[-1])
    assert "error" in line and "--gpus 2" in line["error"]
