"""Debug helper: per golden profile case, max error and first mismatching windows."""
import json, os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import paper_2401_13680_b200 as P
from oracle import pastila_oracle as O
root = os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "tests", "golden")
meta = json.load(open(os.path.join(root, "golden.json")))
g = np.load(os.path.join(root, "golden.npz"))
for c, cs in enumerate(meta["prof"]):
    x = g[f"prof{c}_x"]
    s = P.TimeSeries(x)
    params = P.MPdistParams(cs["m"], cs["l"], cs["k"])
    for si, seg in enumerate(cs["segs"]):
        got = P.mpdist_profile(s, seg, params).values
        ref = g[f"prof{c}_D"][si]
        err = np.abs(got - ref)
        bad = np.nonzero(err > 1e-6)[0]
        print(c, cs, "n", x.size, "seg", seg, "maxerr %.3g" % err.max(), "nbad", bad.size, bad[:10], got[bad[:3]], ref[bad[:3]])
