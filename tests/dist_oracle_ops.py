"""Test infrastructure only: the per-rank steps of the partitioned build
(paper_1301_1704_b200.distributed.DeviceOps) restated on the CPU oracle
(oracle/), so the partition / exchange / offset logic of the driver can run
under gloo on a machine without a GPU."""

import numpy as np
import torch

from oracle import oracle as orc
from paper_1301_1704_b200.distributed import DistLists
from paper_1301_1704_b200.pseudosort import SortedPointSet


def _t(a):
    return torch.from_numpy(np.ascontiguousarray(a))


def _keys(points, level):
    pts = points.numpy() if isinstance(points, torch.Tensor) else points
    return orc.encode(np.ascontiguousarray(pts.reshape(-1, 3)), level)


def _bits_to_keys(words):
    w = words.numpy().view(np.uint64)
    bits = np.unpackbits(w.view(np.uint8), bitorder="little")
    return np.flatnonzero(bits).astype(np.uint64)


class OracleOps:
    def part_histogram(self, src, recv, level, pbits):
        sh = np.uint64(3 * level - pbits)
        keys = np.concatenate([_keys(src, level), _keys(recv, level)])
        return _t(np.bincount((keys >> sh).astype(np.int64), minlength=1 << pbits).astype(np.int64))

    def part_pack(self, src, q, recv, level, pbits, bin_rank, nranks, gbase_src, gbase_recv):
        sh = np.uint64(3 * level - pbits)
        br = bin_rank.numpy()
        out = []
        for pts, gbase in ((src.numpy(), gbase_src), (recv.numpy(), gbase_recv)):
            dest = br[(_keys(pts, level) >> sh).astype(np.int64)]
            order = np.argsort(dest, kind="stable")
            out.append((pts[order], order + gbase, np.bincount(dest, minlength=nranks), order))
        (sx, sg, sc, so), (rx, rg, rc, _) = out
        sq = _t(q.numpy()[so]) if q is not None else None
        return _t(sx), sq, _t(sg), _t(rx), _t(rg), sc.tolist(), rc.tolist()

    def dist_sort(self, src, q, sgid, recv, rgid, level):
        words = max(1, (8 ** level) // 64)
        bmp = np.zeros(2 * words, dtype=np.uint64)
        sets = []
        for k, (pts, qq, gid) in enumerate(((src, q, sgid), (recv, None, rgid))):
            s = orc.sort_points(pts.numpy(), None if qq is None else qq.numpy(), level)
            ne = s.non_empty_index.astype(np.uint64)
            np.bitwise_or.at(bmp, k * words + (ne >> np.uint64(6)).astype(np.int64),
                             np.left_shift(np.uint64(1), ne & np.uint64(63)))
            sets.append(SortedPointSet(
                level=level, points=_t(s.points),
                charges=None if s.charges is None else _t(s.charges),
                permutation=_t(gid.numpy()[s.permutation]), bookmarks=_t(s.bookmarks),
                non_empty_index=_t(s.non_empty_index), boxes=_t(s.boxes)))
        return sets[0], sets[1], _t(bmp.view(np.int64))

    def dist_lists(self, gbmp, level, key_lo, key_hi):
        L = level
        words = max(1, (8 ** L) // 64)
        src_L = _bits_to_keys(gbmp[:words])
        recv_L = _bits_to_keys(gbmp[words:])

        def lvl(keys, l):
            return np.unique(keys >> np.uint64(3 * (L - l)))

        def owned(keys, l):
            first = keys << np.uint64(3 * (L - l))
            return keys[(first >= np.uint64(key_lo)) & (first < np.uint64(key_hi))]

        rows_L = owned(recv_L, L)
        nb, nl = orc.adjacent_segments(rows_L, src_L, L)
        dsrc, drecv, sb, sr, sc = {}, {}, {}, {}, {}
        for l in range(2, L + 1):
            s_l, r_l = lvl(src_L, l), lvl(recv_L, l)
            rows = owned(r_l, l)
            b, r, c = orc.stencil_segments(rows, s_l, l)
            sb[l], sr[l], sc[l] = _t(b), _t(r), _t(c)
            if l < L:
                dsrc[l], drecv[l] = _t(owned(s_l, l)), _t(rows)
        return DistLists(neighbor_bookmark=_t(nb), neighbor_list=_t(nl), dir_src=dsrc,
                         dir_recv=drecv, st_bookmark=sb, st_ranks=sr, st_codes=sc)
