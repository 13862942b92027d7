import sys; sys.path.insert(0, '/root/repo'); sys.path.insert(0, '/root/repo/tests')
import numpy as np
from conftest import load_case, rel
from cases import hierarchy
import paper_1412_0464_b200 as hb
d = load_case("wedge2d")
hh = hierarchy("wedge2d", device=True)
print("x", rel(hb.prec_x(hh.partition, d["probe_xc"]), d["sweep_x"]))
