"""Per-rank M exchange volume of a BASELINE config under the multi-rank plan: for R virtual ranks
(one device, hfmm_set_dist_virtual), every active level's boxes received per matvec by the halo
(levels >= HFMM_HALO_LEVEL) or the all-gather, and the all-gather volume for comparison.
    python tools/halo_volume.py C4 8 [halo_level]"""
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
name = sys.argv[1]
R = int(sys.argv[2])
if len(sys.argv) > 3:
    os.environ["HFMM_HALO_LEVEL"] = sys.argv[3]
import torch  # noqa: E402,F401
import paper_0911_4114_b200 as hf  # noqa: E402
from workloads import CONFIGS, points_and_charges  # noqa: E402

cfg = CONFIGS[name]
x, _ = points_and_charges(cfg)
vg = hf.VirtualGroup(R)
out = {"config": name, "ranks": R, "halo_level": os.environ.get("HFMM_HALO_LEVEL", "4"), "levels": {}}
for r in range(R):
    g = hf.HFMM(0)
    vg.bind(g, r)
    g.build_tree(x, cfg.depth, cfg.lo, cfg.size)
    g.precompute(cfg.kappa, cfg.eps, cfg.alpha)
    for lv in g.info()["levels"]:
        if not lv["active"]:
            continue
        d = out["levels"].setdefault(lv["level"], {"K": lv["K"], "boxes": lv["boxes"], "halo": lv["halo"],
                                                   "recv_boxes": [], "send_boxes": []})
        d["recv_boxes"].append(lv["m_recv_boxes"])
        d["send_boxes"].append(lv["m_send_boxes"])
    g.close()    # plans are freed one by one: only the plan statistics are needed
for l, d in out["levels"].items():
    d["recv_MB_max"] = max(d["recv_boxes"]) * d["K"] * 16 / 1e6
    d["allgather_recv_MB_max_est"] = d["boxes"] * (R - 1) / R * d["K"] * 16 / 1e6
print(json.dumps(out))
