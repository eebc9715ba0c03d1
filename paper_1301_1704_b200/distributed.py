"""Multi-GPU build of ONE problem by contiguous Morton-key ranges.

The paper's scheme (reference ownership by key range:
pkg/src/fmmkit/partition.py:22-61, distributed build: exchange.py:183-272),
one process per GPU, the collectives through `torch.distributed` (NCCL over
NVLink on the B200 box):

 1. every rank holds an index-contiguous shard of the sources and receivers;
 2. histogram of the top `pbits` level-L key bits (device), all-reduce, and a
    deterministic cut of the bins into P contiguous ranges balancing src+recv
    points -- a box never straddles two ranks;
 3. stable pack by destination (device) and an all-to-all of (xyz, q, global
    index); receive order is (source rank, index) = global index order, so
    the local stable sort reproduces the global order;
 4. local sort phase (`fmmb_dist_sort`): sorted points, permutation in global
    indices, rank-local bookmarks, level-L occupancy bitmaps;
 5. all-reduce (SUM = OR: the ranks' bits are disjoint) of the bitmaps;
 6. lists of the receiver rows the rank owns (a level-l box is owned by the
    rank whose key range holds its first level-L key), with global source
    ranks (`fmmb_dist_lists`);
 7. an all-gather of the shard sizes turns rank-local CSR / bookmark offsets
    into global ones.

Every rank ends up with a contiguous shard of every `FmmStructures` array;
`concat_shards` of the shards in rank order is bit-identical to the
single-GPU `build_all` of the whole problem.

The collectives go through a small `Comm` interface: `TorchComm` (one rank
per process, torch.distributed -- NCCL, or gloo with host staging) and
`SimComm` (all ranks driven by one process; used to test and measure the
partitioned path on a single GPU).  The per-rank device steps go through an
`ops` object (`DeviceOps`, the libfmmb200 kernels; there is no CPU fallback).
"""

from __future__ import annotations

import ctypes as C
import os
from dataclasses import dataclass, field

import numpy as np
import torch

from . import _lib
from .errors import DomainError
from .lists import FmmStructures, LevelDirectory, NeighborTable, TranslationStencils
from .pseudosort import SortedPointSet, _point_set_from_c, check_level

__all__ = [
    "Comm", "TorchComm", "SimComm", "DeviceOps", "DistShard", "PhaseTimer", "build_all_distributed",
    "cut_bins", "concat_shards", "partition_bits",
]


# ------------------------------------------------------------------ comms
class Comm:
    """Collectives over `size` ranks; `ranks` are the ranks this process
    drives (one for TorchComm, all of them for SimComm).  Every method takes
    one entry per driven rank, in `ranks` order, and returns the same."""

    size: int
    ranks: list

    def allreduce_sum(self, xs: list) -> list:
        raise NotImplementedError

    def all_to_all(self, chunks: list, recv_rows: list | None = None) -> list:
        """chunks[i][d] = tensor from driven rank i to rank d; returns
        out[i][s] = tensor rank ranks[i] received from rank s.  recv_rows[i][s]
        (optional) = its row count, when already known (no size exchange)."""
        raise NotImplementedError

    def exchange_counts(self, counts: list) -> list:
        """counts[i] = k host ints per destination rank (k*size, destination
        major) from driven rank i -> out[i][k*s + j] = value j rank ranks[i]
        got from rank s."""
        raise NotImplementedError

    def all_gather(self, xs: list) -> list:
        """out[i] = [x of rank 0, ..., x of rank size-1] (same shapes)."""
        raise NotImplementedError

    def peer_tables(self, bufs: list) -> list:
        """Fused pack + exchange: bufs[i] = {name: device tensor} of driven
        rank i's receive arrays.  Returns tables[i][name] = [device pointer
        of rank d's array, usable from rank ranks[i]'s device, for d in
        range(size)] (CUDA IPC across processes; P2P / same device in one)."""
        raise NotImplementedError

    def peer_barrier(self) -> None:
        """Every rank's peer stores are complete and visible."""
        raise NotImplementedError


class SimComm(Comm):
    """All `size` ranks in this process (their tensors may share a device)."""

    def __init__(self, size: int):
        self.size = size
        self.ranks = list(range(size))

    def allreduce_sum(self, xs):
        tot = xs[0].clone()
        for x in xs[1:]:
            tot += x
        return [tot.clone() for _ in xs]

    def all_to_all(self, chunks, recv_rows=None):
        return [[chunks[s][d] for s in range(self.size)] for d in range(self.size)]

    def exchange_counts(self, counts):
        k = len(counts[0]) // self.size
        return [[counts[s][k * d + j] for s in range(self.size) for j in range(k)]
                for d in range(self.size)]

    def all_gather(self, xs):
        return [list(xs) for _ in xs]

    def peer_tables(self, bufs):
        tab = {k: [b[k].data_ptr() if b[k] is not None and b[k].numel() else 0 for b in bufs]
               for k in bufs[0]}
        return [tab for _ in bufs]

    def peer_barrier(self):
        for d in range(torch.cuda.device_count()):
            torch.cuda.synchronize(d)


class TorchComm(Comm):
    """One rank per process over a torch.distributed process group (NCCL for
    CUDA tensors; gloo stages CUDA tensors through the host)."""

    def __init__(self, group=None):
        import torch.distributed as dist

        self.dist = dist
        self.group = group
        self.size = dist.get_world_size(group)
        self.ranks = [dist.get_rank(group)]
        self.stage = dist.get_backend(group) == "gloo"

    def _to(self, x):
        return x.cpu() if self.stage else x

    def allreduce_sum(self, xs):
        (x,) = xs
        y = self._to(x).clone()
        self.dist.all_reduce(y, group=self.group)
        return [y.to(x.device)]

    def exchange_counts(self, counts):
        (row,) = counts
        x = torch.tensor([int(c) for c in row], dtype=torch.int64)
        if not self.stage:
            x = x.cuda()
        y = torch.empty_like(x)
        self.dist.all_to_all_single(y, x, group=self.group)
        return [[int(v) for v in y.cpu().tolist()]]

    def all_to_all(self, chunks, recv_rows=None):
        (row,) = chunks
        dev = row[0].device
        dtype = row[0].dtype
        tail = tuple(row[0].shape[1:])
        width = int(np.prod(tail)) if tail else 1
        if recv_rows is not None:
            rs = [int(v) for v in recv_rows[0]]
        else:
            rs = self.exchange_counts([[int(c.shape[0]) for c in row]])[0]
        send = self._to(torch.cat([c.reshape(-1) for c in row]))
        recv = torch.empty(sum(rs) * width, dtype=dtype, device=send.device)
        self.dist.all_to_all_single(recv, send, [r * width for r in rs],
                                    [int(c.shape[0]) * width for c in row], group=self.group)
        recv = recv.to(dev)
        out, at = [], 0
        for r in rs:
            out.append(recv[at: at + r * width].reshape((r,) + tail))
            at += r * width
        return [out]

    def peer_tables(self, bufs):
        """CUDA IPC: every rank shares its receive arrays' storages, opens the
        others' (torch's own IPC path, lazily enabled peer access)."""
        (b,) = bufs
        mine = {k: (v.untyped_storage()._share_cuda_(), v.storage_offset() * v.element_size())
                if v is not None and v.numel() else None for k, v in b.items()}
        allm = [None] * self.size
        self.dist.all_gather_object(allm, mine, group=self.group)
        me = self.ranks[0]
        self._peer_keep = []
        tab = {}
        for k in b:
            ptrs = []
            for d, md in enumerate(allm):
                if md[k] is None:
                    ptrs.append(0)
                elif d == me:
                    ptrs.append(b[k].data_ptr())
                else:
                    meta, off = md[k]
                    st = torch.UntypedStorage._new_shared_cuda(*meta)
                    self._peer_keep.append(st)
                    ptrs.append(st.data_ptr() + off)
            tab[k] = ptrs
        return [tab]

    def peer_barrier(self):
        torch.cuda.synchronize()
        self.dist.barrier(group=self.group)

    def all_gather(self, xs):
        (x,) = xs
        outs = [torch.empty_like(self._to(x)) for _ in range(self.size)]
        self.dist.all_gather(outs, self._to(x).contiguous(), group=self.group)
        return [[o.to(x.device) for o in outs]]


# ------------------------------------------------------------- device ops
@dataclass
class DistLists:
    neighbor_bookmark: torch.Tensor
    neighbor_list: torch.Tensor
    dir_src: dict
    dir_recv: dict
    st_bookmark: dict
    st_ranks: dict
    st_codes: dict


class DeviceOps:
    """The per-rank device steps, on libfmmb200 (include/fmmb200.h).
    `launches` counts the library's kernel launches."""

    def __init__(self):
        self.launches = 0

    def _count(self, h):
        self.launches += int(_lib.load().fmmb_last_launch_count(h))

    def part_histogram(self, src, recv, level, pbits):
        dev = _lib.device_of(src.device)
        h = _lib.handle(dev)
        hist = torch.empty(1 << pbits, dtype=torch.int32, device=dev)  # u32 counts < 2^31
        n, m = int(src.shape[0]), int(recv.shape[0])
        st = _lib.load().fmmb_part_histogram(
            h, src.data_ptr() if n else None, n, recv.data_ptr() if m else None, m, level,
            pbits, hist.data_ptr(), _lib.stream_of(dev))
        _lib.check(st, h)
        self._count(h)
        return hist.to(torch.int64)

    def part_pack(self, src, q, recv, level, pbits, bin_rank, nranks, gbase_src, gbase_recv):
        dev = _lib.device_of(src.device)
        h = _lib.handle(dev)
        n, m = int(src.shape[0]), int(recv.shape[0])
        sxyz = torch.empty((n, 3), dtype=torch.float64, device=dev)
        sq = torch.empty(n, dtype=torch.float64, device=dev) if q is not None else None
        sgid = torch.empty(n, dtype=torch.int64, device=dev)
        rxyz = torch.empty((m, 3), dtype=torch.float64, device=dev)
        rgid = torch.empty(m, dtype=torch.int64, device=dev)
        counts = (C.c_int64 * (2 * nranks))()
        br = bin_rank.to(device=dev, dtype=torch.int32).contiguous()
        p = lambda t: t.data_ptr() if (t is not None and t.numel()) else None  # noqa: E731
        st = _lib.load().fmmb_part_pack(
            h, p(src), p(q), n, p(recv), m, level, pbits, br.data_ptr(), nranks, gbase_src,
            gbase_recv, p(sxyz), p(sq), p(sgid), p(rxyz), p(rgid), counts, _lib.stream_of(dev))
        _lib.check(st, h)
        self._count(h)
        c = list(counts)
        return sxyz, sq, sgid, rxyz, rgid, c[:nranks], c[nranks:]

    def part_counts(self, src, recv, level, pbits, bin_rank, nranks):
        dev = _lib.device_of(src.device)
        h = _lib.handle(dev)
        n, m = int(src.shape[0]), int(recv.shape[0])
        counts = (C.c_int64 * (2 * nranks))()
        br = bin_rank.to(device=dev, dtype=torch.int32).contiguous()
        p = lambda t: t.data_ptr() if (t is not None and t.numel()) else None  # noqa: E731
        st = _lib.load().fmmb_part_counts(h, p(src), n, p(recv), m, level, pbits, br.data_ptr(),
                                          nranks, counts, _lib.stream_of(dev))
        _lib.check(st, h)
        self._count(h)
        return list(counts)

    def part_pack_peer(self, src, q, recv, level, pbits, bin_rank, nranks, gbase_src,
                       gbase_recv, table, soff, roff):
        dev = _lib.device_of(src.device)
        h = _lib.handle(dev)
        n, m = int(src.shape[0]), int(recv.shape[0])
        br = bin_rank.to(device=dev, dtype=torch.int32).contiguous()
        p = lambda t: t.data_ptr() if (t is not None and t.numel()) else None  # noqa: E731
        P = C.c_void_p * nranks
        arr = {k: P(*[v or None for v in table[k]]) for k in ("sxyz", "sq", "sgid", "rxyz", "rgid")}
        st = _lib.load().fmmb_part_pack_peer(
            h, p(src), p(q), n, p(recv), m, level, pbits, br.data_ptr(), nranks, gbase_src,
            gbase_recv, arr["sxyz"], arr["sq"] if q is not None else None, arr["sgid"],
            arr["rxyz"], arr["rgid"], (C.c_int64 * nranks)(*soff), (C.c_int64 * nranks)(*roff),
            _lib.stream_of(dev))
        _lib.check(st, h)
        self._count(h)

    def dist_sort(self, src, q, sgid, recv, rgid, level):
        dev = _lib.device_of(src.device)
        h = _lib.handle(dev)
        n, m = int(src.shape[0]), int(recv.shape[0])
        words = max(1, (8 ** level) // 64)
        bmp = torch.empty(2 * words, dtype=torch.int64, device=dev)
        alloc = _lib.Allocator(dev)
        so, ro = _lib.PointSetC(), _lib.PointSetC()
        p = lambda t: t.data_ptr() if (t is not None and t.numel()) else None  # noqa: E731
        st = _lib.load().fmmb_dist_sort(
            h, p(src), p(q), n, p(sgid), p(recv), m, p(rgid), level, alloc.fn, None,
            C.byref(so), C.byref(ro), bmp.data_ptr(), _lib.stream_of(dev))
        if alloc.error is not None:
            raise alloc.error
        _lib.check(st, h)
        self._count(h)
        return (_point_set_from_c(so, alloc, level, q is not None),
                _point_set_from_c(ro, alloc, level, False), bmp)

    def dist_join(self, device):
        """Order the current stream after the local pass of the last dist_sort."""
        dev = _lib.device_of(device)
        h = _lib.handle(dev)
        _lib.check(_lib.load().fmmb_dist_join(h, _lib.stream_of(dev)), h)

    def dist_lists(self, gbmp, level, key_lo, key_hi):
        dev = _lib.device_of(gbmp.device)
        h = _lib.handle(dev)
        alloc = _lib.Allocator(dev)
        out = _lib.StructuresC()
        st = _lib.load().fmmb_dist_lists(h, gbmp.data_ptr(), level, key_lo, key_hi, alloc.fn,
                                         None, C.byref(out), _lib.stream_of(dev))
        if alloc.error is not None:
            raise alloc.error
        _lib.check(st, h)
        self._count(h)
        L = level
        rows_L = int(out.recv.k)
        v = _lib.view
        dsrc, drecv, sb, sr, sc = {}, {}, {}, {}, {}
        rows = {L: rows_L}
        for l in range(2, L):
            dsrc[l] = v(alloc, out.dir_src[l], int(out.n_dir_src[l]), "u8")
            drecv[l] = v(alloc, out.dir_recv[l], int(out.n_dir_recv[l]), "u8")
            rows[l] = int(out.n_dir_recv[l])
        for l in range(2, L + 1):
            sb[l] = v(alloc, out.st_bookmark[l], rows[l] + 1, "i8")
            sr[l] = v(alloc, out.st_ranks[l], int(out.n_st[l]), "i8")
            sc[l] = v(alloc, out.st_codes[l], int(out.n_st[l]), "i2")
        return DistLists(
            neighbor_bookmark=v(alloc, out.neighbor_bookmark, rows_L + 1, "i8"),
            neighbor_list=v(alloc, out.neighbor_list, int(out.n_neighbor), "i8"),
            dir_src=dsrc, dir_recv=drecv, st_bookmark=sb, st_ranks=sr, st_codes=sc)


# ------------------------------------------------------------ partition
def partition_bits(level: int) -> int:
    """Histogram resolution of the cut: the top min(14, 3L) key bits."""
    return min(14, 3 * level)


def cut_bins(hist: torch.Tensor, nranks: int) -> torch.Tensor:
    """Rank of every histogram bin: contiguous bin ranges with balanced point
    counts, rank(b) = min(P-1, floor(P * points-before-b / total)).  A pure
    function of the all-reduced histogram, so every rank computes the same."""
    # on the host: one small read-back instead of a chain of device ops and
    # syncs (the all-reduced histogram has <= 2^14 bins)
    h = hist.detach().to("cpu", torch.int64).numpy()
    excl = np.cumsum(h) - h
    tot = int(h.sum())
    if tot == 0:
        out = np.zeros_like(h)
    else:
        out = np.minimum((excl * nranks) // tot, nranks - 1)
    return torch.from_numpy(out).to(hist.device)


def key_windows(bin_rank: torch.Tensor, nranks: int, level: int, pbits: int) -> list:
    """[key_lo, key_hi) of every rank's level-L key range."""
    br = bin_rank.cpu()
    nb = br.numel()
    sh = 3 * level - pbits
    starts = torch.searchsorted(br, torch.arange(nranks + 1, dtype=br.dtype)).tolist()
    starts[-1] = nb
    return [(starts[g] << sh, starts[g + 1] << sh) for g in range(nranks)]


# ----------------------------------------------------------------- driver
@dataclass
class DistShard:
    """One rank's contiguous shard of every FmmStructures array (global
    offsets applied; the CSR/bookmark trailing entry only on the last rank)."""

    rank: int
    nranks: int
    max_level: int
    key_window: tuple
    sorted_src: SortedPointSet
    sorted_recv: SortedPointSet
    neighbor_table: NeighborTable
    directory: LevelDirectory
    stencils: TranslationStencils
    exchanged: dict = field(default_factory=dict)  # points sent to other ranks

    def to_numpy(self) -> "DistShard":
        """Host copy of the shard (numpy arrays, reference dtypes): every
        array copied into pinned host memory on the build stream, one sync."""
        from ._host import HostBatch

        batch = HostBatch()
        staged = {}

        def npy(v):
            if not isinstance(v, torch.Tensor):
                return v
            if not v.is_cuda:
                return v.numpy()
            key = (v.data_ptr(), v.numel(), v.dtype)
            if key not in staged:
                staged[key] = batch.add(v.contiguous())
            return staged[key]

        out = self._to_host(npy)
        batch.finish()

        def fin(v):
            return v.numpy() if isinstance(v, torch.Tensor) else v

        return out._to_host(fin)

    def _to_host(self, npy) -> "DistShard":

        def ps(p):
            return SortedPointSet(level=p.level, points=npy(p.points), charges=npy(p.charges),
                                  permutation=npy(p.permutation), bookmarks=npy(p.bookmarks),
                                  non_empty_index=npy(p.non_empty_index), boxes=npy(p.boxes))

        d, st = self.directory, self.stencils
        return DistShard(
            rank=self.rank, nranks=self.nranks, max_level=self.max_level,
            key_window=self.key_window, sorted_src=ps(self.sorted_src),
            sorted_recv=ps(self.sorted_recv),
            neighbor_table=NeighborTable(npy(self.neighbor_table.neighbor_bookmark),
                                         npy(self.neighbor_table.neighbor_list)),
            directory=LevelDirectory(d.max_level, {l: npy(v) for l, v in d.src_boxes.items()},
                                     {l: npy(v) for l, v in d.recv_boxes.items()}),
            stencils=TranslationStencils({l: npy(v) for l, v in st.bookmark.items()},
                                         {l: npy(v) for l, v in st.ranks.items()},
                                         {l: npy(v) for l, v in st.codes.items()}),
            exchanged=dict(self.exchanged))


def _cat(parts: list) -> torch.Tensor:
    """torch.cat of received pieces; no copy when they are already adjacent
    slices of one receive buffer (TorchComm) or a single piece."""
    if len(parts) == 1:
        return parts[0]
    p0 = parts[0]
    at = p0.data_ptr()
    adjacent = all(t.is_contiguous() and t.dtype == p0.dtype for t in parts)
    for t in parts:
        if not adjacent:
            break
        if t.numel() and t.data_ptr() != at:
            adjacent = False
        at += t.numel() * t.element_size()
    if adjacent and p0.untyped_storage().data_ptr() <= p0.data_ptr():
        rows = sum(int(t.shape[0]) for t in parts)
        base = p0.untyped_storage()
        off = (p0.data_ptr() - base.data_ptr()) // p0.element_size()
        full = torch.empty(0, dtype=p0.dtype, device=p0.device).set_(
            base, off, (rows,) + tuple(p0.shape[1:]), p0.stride())
        if all(t.untyped_storage().data_ptr() == base.data_ptr() for t in parts):
            return full
    return torch.cat(parts)


def _shard_csr(bm: torch.Tensor, offset: int, last: bool) -> torch.Tensor:
    x = bm + offset
    return x if last else x[:-1]


class PhaseTimer:
    """CUDA events at the partitioned build's phase boundaries, on the
    current stream of the driven rank's device (collectives issued through
    torch.distributed order that stream after their completion).  `ms()`
    synchronises and returns {phase: ms}; phases repeated over several
    builds accumulate."""

    def __init__(self):
        self.marks = []  # (name, event) in order

    def mark(self, name: str) -> None:
        e = torch.cuda.Event(enable_timing=True)
        e.record()
        self.marks.append((name, e))

    def ms(self) -> dict:
        out = {}
        if not self.marks:
            return out
        self.marks[-1][1].synchronize()
        for (_, a), (name, b) in zip(self.marks, self.marks[1:]):
            if name != "start":
                out[name] = out.get(name, 0.0) + a.elapsed_time(b)
        return out


def _mark(timer, name):
    if timer is not None:
        timer.mark(name)


def build_all_distributed(shards: list, max_level: int, comm: Comm, ops=None,
                          pbits: int | None = None, exchange: str | None = None,
                          timer: PhaseTimer | None = None) -> list:
    """Partitioned build.  `shards[i] = (src, charges, recv)` of the rank
    comm.ranks[i]: device tensors, index-contiguous pieces of the global
    arrays in rank order.  Returns one DistShard per driven rank.  `timer`
    (optional, one driven rank) records the phase boundaries."""
    _mark(timer, "start")
    check_level(max_level)
    if max_level < 2:
        raise DomainError("the partitioned build needs max_level >= 2")
    ops = ops or DeviceOps()
    L = max_level
    P = comm.size
    pb = pbits or partition_bits(L)
    nd = len(comm.ranks)
    dev = [s[0].device for s in shards]
    # 1. global index bases
    sizes = [torch.tensor([int(s[0].shape[0]), int(s[2].shape[0])], dtype=torch.int64,
                          device=dev[i]) for i, s in enumerate(shards)]
    allsz = [[int(v) for t in g for v in t.cpu().tolist()] for g in comm.all_gather(sizes)]
    gb = []
    for i, r in enumerate(comm.ranks):
        ns, ms = allsz[i][0::2], allsz[i][1::2]
        gb.append((sum(ns[:r]), sum(ms[:r])))
    # 2. histogram -> cut
    hists = [ops.part_histogram(s[0], s[2], L, pb) for s in shards]
    hists = comm.allreduce_sum(hists)
    br_host = cut_bins(hists[0].cpu(), P)
    windows = key_windows(br_host, P, L, pb)
    bin_rank = br_host.to(dev[0], non_blocking=True)
    _mark(timer, "partition (histogram, all-reduce, cut)")
    exchange = exchange or os.environ.get("FMMB_DIST_EXCHANGE", "a2a")
    if exchange == "peer":  # 3'. fused pack + exchange over peer memory
        return _finish(shards, L, comm, ops, P, dev, gb, windows,
                       _exchange_peer(shards, L, comm, ops, P, pb, bin_rank, gb, dev, timer),
                       timer)
    # 3. pack + exchange
    packs = [ops.part_pack(s[0], s[1], s[2], L, pb, bin_rank, P, gb[i][0], gb[i][1])
             for i, s in enumerate(shards)]
    _mark(timer, "pack")

    def split(t, cnts):
        out, at = [], 0
        for c in cnts:
            out.append(t[at: at + c])
            at += c
        return out

    with_q = shards[0][1] is not None
    # one count exchange (src and recv counts per destination), then the five
    # payload exchanges with known sizes: no host round trip between them
    cnt = comm.exchange_counts([[v for d in range(P) for v in (pk[5][d], pk[6][d])]
                                for pk in packs])
    rsrc = [[c[2 * s] for s in range(P)] for c in cnt]
    rrecv = [[c[2 * s + 1] for s in range(P)] for c in cnt]
    ex = {}
    for key, idx, cidx, rr in (("sxyz", 0, 5, rsrc), ("sgid", 2, 5, rsrc), ("rxyz", 3, 6, rrecv),
                               ("rgid", 4, 6, rrecv)):
        ex[key] = comm.all_to_all([split(pk[idx], pk[cidx]) for pk in packs], rr)
    if with_q:
        ex["sq"] = comm.all_to_all([split(pk[1], pk[5]) for pk in packs], rsrc)
    received = []
    for i, r in enumerate(comm.ranks):
        sent = sum(int(t.shape[0]) for d, t in enumerate(split(packs[i][0], packs[i][5])) if d != r)
        sent_r = sum(int(t.shape[0]) for d, t in enumerate(split(packs[i][3], packs[i][6])) if d != r)
        received.append({"sxyz": _cat(ex["sxyz"][i]), "sgid": _cat(ex["sgid"][i]),
                         "rxyz": _cat(ex["rxyz"][i]), "rgid": _cat(ex["rgid"][i]),
                         "sq": _cat(ex["sq"][i]) if with_q else None,
                         "sent_points": sent + sent_r,
                         # payload bytes leaving this rank: xyz + gid (+ q) per point
                         "sent_bytes": sent * (40 if with_q else 32) + sent_r * 32})
    _mark(timer, "exchange (all-to-all)")
    return _finish(shards, L, comm, ops, P, dev, gb, windows, received, timer)


def _exchange_peer(shards, L, comm, ops, P, pb, bin_rank, gb, dev, timer=None) -> list:
    """Fused pack + exchange: counts, one all-gather of them, receive arrays
    sized and shared, then every rank stores its points straight into the
    destinations' arrays (fmmb_part_pack_peer) -- no send buffers, no
    separate all-to-all.  Receive order = (source rank, input index), as
    with the all-to-all."""
    with_q = shards[0][1] is not None
    cnts = [ops.part_counts(s[0], s[2], L, pb, bin_rank, P) for s in shards]
    allc = comm.all_gather([torch.tensor(c, dtype=torch.int64, device=dev[i])
                            for i, c in enumerate(cnts)])
    bufs, offs, received = [], [], []
    for i, r in enumerate(comm.ranks):
        mat = torch.stack([t.cpu() for t in allc[i]]).tolist()  # mat[s] = counts of rank s
        n_in = sum(mat[s][r] for s in range(P))
        m_in = sum(mat[s][P + r] for s in range(P))
        soff = [sum(mat[s][d] for s in range(r)) for d in range(P)]
        roff = [sum(mat[s][P + d] for s in range(r)) for d in range(P)]
        f64, i64 = dict(dtype=torch.float64, device=dev[i]), dict(dtype=torch.int64, device=dev[i])
        bufs.append({"sxyz": torch.empty((n_in, 3), **f64),
                     "sq": torch.empty(n_in, **f64) if with_q else None,
                     "sgid": torch.empty(n_in, **i64), "rxyz": torch.empty((m_in, 3), **f64),
                     "rgid": torch.empty(m_in, **i64)})
        offs.append((soff, roff))
        c = cnts[i]
        received.append({"sent_points": sum(c[d] + c[P + d] for d in range(P) if d != r),
                         "sent_bytes": sum(c[d] * (40 if with_q else 32) + c[P + d] * 32
                                           for d in range(P) if d != r)})
    _mark(timer, "pack (counts, receive tables)")
    tables = comm.peer_tables(bufs)
    for i, s in enumerate(shards):
        ops.part_pack_peer(s[0], s[1], s[2], L, pb, bin_rank, P, gb[i][0], gb[i][1], tables[i],
                           *offs[i])
    comm.peer_barrier()
    for i in range(len(shards)):
        received[i].update(bufs[i])
    _mark(timer, "exchange (peer stores)")
    return received


def _finish(shards, L, comm, ops, P, dev, gb, windows, received, timer=None) -> list:
    """Local sort, global occupancy, owned lists, global offsets (steps 4-7)."""
    nd = len(comm.ranks)
    results = []
    sorted_sets = []
    bmps = []
    for i, r in enumerate(comm.ranks):
        rv = received[i]
        # 4. local sort phase
        ss, sr, bmp = ops.dist_sort(rv["sxyz"], rv["sq"], rv["sgid"], rv["rxyz"], rv["rgid"], L)
        sorted_sets.append((ss, sr))
        bmps.append(bmp)
        results.append({"sent_points": rv["sent_points"], "sent_bytes": rv.get("sent_bytes", 0)})
    _mark(timer, "local sort")
    # 5. global occupancy
    gbmps = comm.allreduce_sum(bmps)
    _mark(timer, "occupancy all-reduce")
    # 6. owned lists
    lists = [ops.dist_lists(gbmps[i], L, *windows[r]) for i, r in enumerate(comm.ranks)]
    for i in range(nd):  # the local passes ran beside the all-reduce and the lists
        if hasattr(ops, "dist_join"):
            ops.dist_join(dev[i])
    _mark(timer, "owned lists")
    # 7. global offsets from every rank's shard sizes
    def stats(i):  # host-known sizes (a CSR's last bookmark is its list length)
        ss, sr = sorted_sets[i]
        dl = lists[i]
        v = [ss.points.shape[0], sr.points.shape[0], dl.neighbor_list.shape[0]]
        for l in range(2, L + 1):
            v.append(dl.st_ranks[l].shape[0])
        return torch.tensor([int(x) for x in v], dtype=torch.int64, device=dev[i])

    allst = comm.all_gather([stats(i) for i in range(nd)])
    _mark(timer, "offsets (all-gather)")
    out = []
    for i, r in enumerate(comm.ranks):
        st = torch.stack([t.cpu() for t in allst[i]])  # (P, 3 + L - 1)
        before = st[:r].sum(0) if r else torch.zeros(st.shape[1], dtype=torch.int64)
        last = r == P - 1
        ss, sr = sorted_sets[i]
        dl = lists[i]
        ss.bookmarks = _shard_csr(ss.bookmarks, int(before[0]), last)
        sr.bookmarks = _shard_csr(sr.bookmarks, int(before[1]), last)
        nt = NeighborTable(_shard_csr(dl.neighbor_bookmark, int(before[2]), last),
                           dl.neighbor_list)
        dsrc = {L: ss.non_empty_index, **dl.dir_src}
        drecv = {L: sr.non_empty_index, **dl.dir_recv}
        sb = {l: _shard_csr(dl.st_bookmark[l], int(before[3 + l - 2]), last)
              for l in range(2, L + 1)}
        out.append(DistShard(
            rank=r, nranks=P, max_level=L, key_window=windows[r], sorted_src=ss,
            sorted_recv=sr, neighbor_table=nt, directory=LevelDirectory(L, dsrc, drecv),
            stencils=TranslationStencils(sb, dl.st_ranks, dl.st_codes), exchanged=results[i]))
    return out


def concat_shards(shards: list) -> FmmStructures:
    """The global FmmStructures from every rank's shard (rank order)."""
    shards = sorted(shards, key=lambda s: s.rank)
    L = shards[0].max_level

    def cat(get):
        parts = [get(s) for s in shards]
        if isinstance(parts[0], torch.Tensor):
            return torch.cat([p.to(parts[0].device) for p in parts])
        return np.concatenate(parts)

    def ps(side):
        first = getattr(shards[0], side)
        return SortedPointSet(
            level=L,
            points=cat(lambda s: getattr(s, side).points),
            charges=None if first.charges is None else cat(lambda s: getattr(s, side).charges),
            permutation=cat(lambda s: getattr(s, side).permutation),
            bookmarks=cat(lambda s: getattr(s, side).bookmarks),
            non_empty_index=cat(lambda s: getattr(s, side).non_empty_index),
            boxes=cat(lambda s: getattr(s, side).boxes))

    levels = range(2, L + 1)
    return FmmStructures(
        max_level=L, sorted_src=ps("sorted_src"), sorted_recv=ps("sorted_recv"),
        neighbor_table=NeighborTable(cat(lambda s: s.neighbor_table.neighbor_bookmark),
                                     cat(lambda s: s.neighbor_table.neighbor_list)),
        directory=LevelDirectory(
            L, {l: cat(lambda s: s.directory.src_boxes[l]) for l in levels},
            {l: cat(lambda s: s.directory.recv_boxes[l]) for l in levels}),
        stencils=TranslationStencils(
            {l: cat(lambda s: s.stencils.bookmark[l]) for l in levels},
            {l: cat(lambda s: s.stencils.ranks[l]) for l in levels},
            {l: cat(lambda s: s.stencils.codes[l]) for l in levels}))
