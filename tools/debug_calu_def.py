"""Diagnostics: device CALU_PRRP vs the oracle on a deficient-node fixture."""
import json, sys
import numpy as np
sys.path.insert(0, ".")
import paper_1208_2451_b200 as dev
from paper_1208_2451_b200 import matgen
from oracle import prrp_oracle as orc
name = sys.argv[1]
meta = json.load(open(f"tests/golden/full/{name}.json"))
arr = dict(np.load(f"tests/golden/full/{name}.npz"))
a = matgen.gen_deficient_block(meta["n"], meta["seed"], meta["blocks"], meta["b"])
b = meta["b"]
tree = dev.binary_tree(meta["P"]) if meta["P"] else dev.flat_tree()
f = dev.caluprrp_factor(a, b, meta["tau"], tree)
d = np.nonzero(f.perm != arr["perm"])[0]
print("first diff", d[:10], "panel", d[0] // b if len(d) else None)
print("swaps dev", f.stats.swap_counts[:10], "ref", meta["stats"]["swap_counts"][:10])
print("charged dev", f.stats.flops_charged, "ref", meta["stats"]["flops_charged"])
for k in range(min(8, meta["n"] // b)):
    print(k, np.array_equal(f.perm[k*b:(k+1)*b], arr["perm"][k*b:(k+1)*b]))
if len(d):
    k = d[0] // b
    # the oracle panel by panel: factor the first k panels, then the tournament of panel k
    fo = orc.calu_prrp(a, b, meta["tau"], "binary", meta["P"], panel_limit=k)
    print("oracle prefix equals ref:", np.array_equal(fo.perm[:k*b], arr["perm"][:k*b]))
tp, trace = dev.tournament_select(np.asfortranarray(a[:, :b]), b, meta["tau"], tree, "srrqr")
print("tournament_select perm equal:", np.array_equal(tp, arr["t0_perm"]))
for nd, rd in zip(trace.nodes, meta["t0_trace"]):
    print(nd.level, nd.index, len(nd.members), len(rd["members"]), np.array_equal(nd.members, rd["members"]),
          len(nd.selected), len(rd["selected"]), np.array_equal(nd.selected, rd["selected"]))
# fused path: the first panel's pivots vs the reference's tournament winners
print("fused first-panel pivots equal the ref tournament winners:", np.array_equal(f.perm[:b], arr["t0_perm"][:b]))
print("fused first-panel pivot SET equal:", set(f.perm[:b]) == set(arr["t0_perm"][:b]))
