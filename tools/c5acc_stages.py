"""Stage times and per-kernel launch list of one BASELINE config (default C5 with tau = eps/10)."""
import json
import os
import statistics
import sys

os.environ["HFMM_PROFILE_STAGES"] = "1"
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402
import paper_0911_4114_b200 as hf  # noqa: E402
from workloads import CONFIGS, points_and_charges  # noqa: E402

name = sys.argv[1] if len(sys.argv) > 1 else "C5"
acc = len(sys.argv) > 2 and sys.argv[2] == "acc"
serial = len(sys.argv) > 3 and sys.argv[3] == "serial"
cfg = CONFIGS[name]
x, q = points_and_charges(cfg)
g = hf.HFMM(0)
g.build_tree(x, cfg.depth, cfg.lo, cfg.size)
g.precompute(cfg.kappa, cfg.eps, cfg.alpha, tau=cfg.eps / 10 if acc else 0.0)
qd = torch.from_numpy(q).cuda()
y = torch.empty_like(qd)
for _ in range(2):
    g.matvec(qd, out=y, serial=serial)
st = []
for _ in range(3):
    g.matvec(qd, out=y, serial=serial)
    torch.cuda.synchronize()
    st.append(g.stage_times())
info = g.info()
print(json.dumps({"config": name, "acc": acc, "serial": serial, "L_f": info["L_f"], "D_s": info["source_level"],
                  "stages_ms": {k: statistics.mean(s[k] for s in st) for k in st[0]},
                  "levels": [(lv["level"], lv["n_theta"], lv["n_phi"], lv["boxes"], lv["m2l_pairs"], lv["active"]) for lv in info["levels"]],
                  "p2p_pairs": info["p2p_pairs"], "s2m_evals": info["s2m_evals"], "p2p_tile": info["p2p_tile"]}))
