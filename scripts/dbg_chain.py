import os, sys
sys.path.insert(0, '/root/repo')
import numpy as np
import paper_2101_11157_b200 as wv
ids = {name: vid for vid, name, cls in wv.kernel_variants()}
for items in ["0.001", "4", "1000000"]:
    os.environ["WV_LANE_ITEMS"] = items
    wv.set_kernel_variant(0, ids["c0 int s2/2 pairs"])
    _, ref = wv.search(5, 20000, 1)
    wv.set_kernel_variant(0, ids["c0 lane2"])
    _, got = wv.search(5, 20000, 1)
    bad = np.nonzero(got["res_w"] != ref["res_w"])[0]
    print(items, "bad", len(bad), "idx", bad[:40].tolist(), "p", got["p"][bad[:10]].tolist(), flush=True)
