import sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
import paper_2106_00124_b200 as ex
from oracle import oracle as orc
rng = np.random.default_rng(0)
for shape, box in [((1, 7), (1, 2)), ((2, 7), (1, 2)), ((3, 4), (2, 2)), ((1, 7), (1, 1)), ((4, 1), (2, 1)), ((3, 3, 3), (2, 2, 2))]:
    a = rng.integers(-9, 9, size=shape).astype(np.int64)
    got = ex.corners_excluded(ex.Tensor(ex.IntAddOps(), torch.from_numpy(a).cuda()), box).data.cpu().numpy()
    want = orc.corners_excluded(a, box)
    bc = orc.box_complement_excluded(a, box)
    print(shape, box, np.array_equal(got, want), np.array_equal(want, bc))
    if not np.array_equal(got, want):
        print(a); print(got); print(want)
