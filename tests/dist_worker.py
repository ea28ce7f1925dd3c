"""Worker for tests/test_parallel_cpu.py (run as a subprocess per rank):
rank 0 builds a staged side on the host, rank 1 receives it over gloo."""
import json
import os
import sys
from pathlib import Path

ROOT = Path(__file__).resolve().parents[1]
sys.path[:0] = [str(ROOT), str(ROOT / "oracle")]

import numpy as np  # noqa: E402
import torch  # noqa: E402
import torch.distributed as dist  # noqa: E402

import xct_oracle as O  # noqa: E402
from paper_2009_07226_b200 import matrixstore, parallel  # noqa: E402


def main():
    rank = int(os.environ["RANK"])
    dist.init_process_group("gloo", rank=rank, world_size=int(os.environ["WORLD_SIZE"]))
    cpu = torch.device("cpu")
    side = None
    if rank == 0:
        g = O.make_geom(20, 1, 16)
        A = O.system_matrix(g)
        plan = matrixstore.adjoint_plan(g.num_angles, g.n, 16, 2)
        T = O.transpose_block(O.whole_block(A))
        side = matrixstore.build_device_side(T.indptr, T.indices.astype(np.int32), T.values,
                                             T.num_rows, T.num_cols, plan, "single", 16, 0,
                                             dev=cpu)
    got = parallel._bcast_side(side, 0, rank, cpu)
    digest = {k: float(v.double().sum()) for k, v in got.tensors.items()}
    out = dict(rank=rank, digest=digest, nnz=int(got.info.nnz), smem=got.smem_bytes,
               groups=int(got.staged.n_groups))
    Path(sys.argv[1]).write_text(json.dumps(out))
    dist.destroy_process_group()


if __name__ == "__main__":
    main()
