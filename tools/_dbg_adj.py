import sys, time, numpy as np, torch
sys.path.insert(0, "/root/repo")
from paper_2009_07226_b200 import geometry, pipeline, matrixstore
import os
os.environ["XCT_VERBOSE"] = "1"
g = geometry.make_geometry(2048, 16, 2048)
cfg = pipeline.SystemConfig(precision="mixed", ffactor=16)
sa = pipeline.StreamedAssembly(g, cfg)
dev = sa.dev
counts = torch.zeros(g.num_voxels, dtype=torch.int64, device=dev)
ta = matrixstore.forward_tile_height(g.grid_n, sa.rw, cfg.warps_per_cta, 1)
chunks = sa._chunks(ta)
from paper_2009_07226_b200 import _lib
st = _lib.stream_handle(dev)
for k0, k1 in chunks:
    ip, ix, v = sa._siddon(k0, k1)
    _lib.call("xct_csr_col_counts", ip.data_ptr(), ix.data_ptr(), (k1-k0)*g.grid_n, 0, g.num_voxels, counts.data_ptr(), st)
sa.BAND_NNZ_DEV = 6e8
t0 = time.time()
try:
    sa._adjoint_device(0, chunks, counts)
except matrixstore.DeviceBuildUnsupported as e:
    print("declined:", e)
print("adjoint", time.time() - t0)
