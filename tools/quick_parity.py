import os, sys, time, numpy as np
sys.path.insert(0, os.getcwd())
sys_path_fix = None
sys.path.insert(0, "oracle/_ref")
import fmmkit
import paper_1301_1704_b200 as fb
from paper_1301_1704_b200.workloads import generate
from tests.parity import compare_structures
for (n, L, dist) in [(3000, 4, "uniform"), (65536, 4, "uniform"), (2**18, 7, "uniform"), (4096, 5, "sphere")]:
    src, q, recv = generate(n, n, dist, 1)
    t0 = time.time(); want = fmmkit.build_all(src, q, recv, max_level=L); t1 = time.time()
    got = fb.build_all(src, q, recv, max_level=L); t2 = time.time()
    errs = compare_structures(got, want)
    print(n, L, dist, "ref %.3fs gpu %.3fs" % (t1-t0, t2-t1), "OK" if not errs else errs[:10], flush=True)
from paper_1301_1704_b200 import kernels as K
ck = fmmkit.backend.get_kernels("compiled")
rng = np.random.default_rng(3)
pts = rng.random((5000, 3))
for L in (0, 3, 7, 20):
    a = K.encode_points(pts[:, 0], pts[:, 1], pts[:, 2], L); b = ck.encode_points(pts[:, 0], pts[:, 1], pts[:, 2], L)
    print("encode", L, np.array_equal(a, b), a.dtype)
bx = ck.encode_points(pts[:, 0], pts[:, 1], pts[:, 2], 3)
a = K.assign_box_ranks(bx, 512); b = ck.assign_box_ranks(bx, 512)
print("ranks", all(np.array_equal(x, y) for x, y in zip(a, b)))
s = fmmkit.sort_points(pts, None, 4); r = fmmkit.sort_points(rng.random((3000, 3)), None, 4)
a = K.adjacent_segments(r.non_empty_index, s.non_empty_index, 4); b = ck.adjacent_segments(r.non_empty_index, s.non_empty_index, 4)
print("adjacent", all(np.array_equal(x, y) for x, y in zip(a, b)))
a = K.stencil_segments(r.non_empty_index, s.non_empty_index, 4); b = ck.stencil_segments(r.non_empty_index, s.non_empty_index, 4)
print("stencil", all(np.array_equal(x, y) and x.dtype == y.dtype for x, y in zip(a, b)))
print("parents", np.array_equal(K.propagate_to_parents(s.non_empty_index), fmmkit.lists.propagate_to_parents(s.non_empty_index)))
