"""32-qubit single-GPU check of the widest 32-bit-index tile base (a tile with qubit 31):
the supremacy circuit followed by its inverse returns |0...0> (complex64, 32 GiB)."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import workloads as W  # noqa: E402
import paper_2106_13995_b200 as P  # noqa: E402

c = W.supremacy(7, 5, 20, 0, n=32)
m = W.concat(c, W.inverse(c))
with P.StateVector(32, "c64") as sv:
    st = sv.apply_circuit(W.to_text(m))
    a0 = sv.amplitudes(0, 4)
    nrm = sv.norm()
print({"passes": st["passes"], "amp0": complex(a0[0]), "amp1..3": [abs(x) for x in a0[1:]], "norm": nrm})
assert abs(a0[0] - 1) < 1e-3 and np.max(np.abs(a0[1:])) < 1e-4 and abs(nrm - 1) < 1e-3
print("mirror32 ok")
