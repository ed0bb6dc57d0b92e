"""One load_metis_graph + load_coords + evaluate of a side x side grid (for ncu captures).

    python tools/graphio_once.py [side]
"""
import io
import os
import sys
import tempfile

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, os.path.dirname(os.path.abspath(__file__)))
import graphio_bench as B  # noqa: E402
from paper_1805_01208_b200 import fileio, metrics  # noqa: E402
from paper_1805_01208_b200.types import Partition  # noqa: E402

side = int(sys.argv[1]) if len(sys.argv) > 1 else 2048
n, off, nbrs, _ = B.grid_csr_device(side)
text = B.metis_text_device(n, off, nbrs)
xs, ys = np.arange(n) % side, np.arange(n) // side
tmp = tempfile.mkdtemp(prefix="graphio_once_")
gpath, cpath = os.path.join(tmp, "g.graph"), os.path.join(tmp, "g.xyz")
with open(gpath, "wb") as f:
    f.write(text)
s = io.StringIO()
np.savetxt(s, np.stack([xs * 0.125 + 0.1, ys * 0.3 - 7.7], 1)[: 1 << 20], fmt="%.17g")
with open(cpath, "w") as f:
    f.write(s.getvalue())
g = fileio.load_metis_graph(gpath)
c = fileio.load_coords(cpath)
tiles = (side + 127) // 128
part = Partition(assignment=(ys // 128) * tiles + xs // 128, k=tiles * tiles)
rep = metrics.evaluate(g, part)
print("n", n, "bytes", len(text), "cut", rep.edge_cut, "diameter", max(rep.block_diameters),
      "coords", c.shape)
os.remove(gpath)
os.remove(cpath)
os.rmdir(tmp)
