"""CPU restatement of one partition of the partitioned BFS (test
infrastructure only — imported by tests/, never by the product).

``EmuPart`` has the step methods of ``paper_1604_02844_b200.distributed.
PartitionedGraph`` and the same observable semantics (the word-cyclic
partition of the degree-ordered ids, the exchange buffer layouts, the
per-level counts), computed with numpy on CPU torch tensors. The gloo tests
drive it with the product's level loop (``bfs_partitioned`` +
``TorchExchange``) in world_size-2 process groups, which exercises the
driver and the exchange protocol without a GPU; the GPU tests then check the
device partitions against the single-GPU BFS and this oracle.

Algorithm per level (csrc/partition.cu): expand the owned frontier (owned
neighbours: visited + parent; others: visited mark only), pack marks by
owner, merge the received marks (parent = first neighbour in F_L), compact
the owned words (level L+1), all-gather F_{L+1}, visited |= F_{L+1}.
The search itself is the reference's top-down BFS (traversal.py:80-104).
"""

from __future__ import annotations

import numpy as np
import torch

SENTINEL = 0x7FFFFFFF


def _words(bits: np.ndarray) -> np.ndarray:
    return np.packbits(bits.astype(np.uint8), bitorder="little").view("<u4")


def _bits(words: np.ndarray) -> np.ndarray:
    return np.unpackbits(np.ascontiguousarray(words).view(np.uint8), bitorder="little").astype(bool)


class EmuPart:
    def __init__(self, n: int, colstarts: np.ndarray, rows: np.ndarray, rank: int, nparts: int):
        assert nparts >= 1 and (nparts & (nparts - 1)) == 0 and 0 <= rank < nparts
        self.num_vertices = n
        self.rank, self.nparts = rank, nparts
        cs = np.asarray(colstarts, dtype=np.int64)
        rw = np.asarray(rows, dtype=np.int64)
        deg = np.diff(cs)
        # internal ids: descending degree, ties by original id (layout.cu step 1)
        self.new2old = np.argsort(-deg, kind="stable").astype(np.int64)
        self.old2new = np.empty(n, dtype=np.int64)
        self.old2new[self.new2old] = np.arange(n)
        self.deg = deg[self.new2old]
        self.rows = [np.sort(self.old2new[rw[cs[o]:cs[o + 1]]]) for o in self.new2old]
        self.nwords = ((n + 31) // 32 + nparts - 1) // nparts * nparts
        self.words_per_peer = self.nwords // nparts
        self.nbits = self.nwords * 32
        ids = np.arange(self.nbits)
        self.owned = ((ids >> 5) % nparts == rank) & (ids < n)
        gw = np.arange(self.nwords)
        self.slot = (gw % nparts) * self.words_per_peer + gw // nparts  # global word -> exchange slot
        self.resolved = 0

    # -- buffers (CPU torch tensors, as the gloo collectives need) -----------
    def new_buffers(self) -> dict:
        W, P = self.words_per_peer, self.nparts
        return {"send": torch.zeros(P * W, dtype=torch.int32), "recv": torch.zeros(P * W, dtype=torch.int32),
                "fsend": torch.zeros(W + 4, dtype=torch.int32), "fgath": torch.zeros(P * (W + 4), dtype=torch.int32),
                "red": torch.zeros(2, dtype=torch.int64)}

    def new_outputs(self):
        n = self.num_vertices
        pad = (n + 31) // 32 * 32
        return torch.empty(pad, dtype=torch.int32), torch.empty(n, dtype=torch.int32)

    # -- steps ------------------------------------------------------------------
    def start(self, root: int, red) -> None:
        assert 0 <= root < self.num_vertices
        self.visited = np.zeros(self.nbits, dtype=bool)
        self.level = np.full(self.nbits, -1, dtype=np.int64)
        self.pred = np.full(self.nbits, SENTINEL, dtype=np.int64)
        r = int(self.old2new[root])
        self.visited[r] = True
        self.prev = self.visited.copy()
        self.F = self.visited.copy()
        self.frontier = []
        c = (0, 0)
        if self.owned[r]:
            self.level[r] = 0
            self.pred[r] = root
            self.frontier = [r]
            c = (1, int(self.deg[r]))
        red.copy_(torch.tensor(c, dtype=torch.int64))
        self.L = -1
        self.resolved = 0

    def expand(self) -> None:
        for u in self.frontier:
            pu = int(self.new2old[u])
            for v in self.rows[u]:
                if not self.visited[v]:
                    self.visited[v] = True
                    if self.owned[v]:
                        self.pred[v] = pu

    def pack(self, send) -> None:
        marks = _words(self.visited & ~self.prev & ~self.owned_word_mask())
        out = np.zeros(self.nwords, dtype="<u4")
        out[self.slot] = marks
        send.copy_(torch.from_numpy(out.view(np.int32)))

    def owned_word_mask(self) -> np.ndarray:
        ids = np.arange(self.nbits)
        return (ids >> 5) % self.nparts == self.rank

    def merge(self, recv, fsend) -> None:
        W = self.words_per_peer
        rv = recv.numpy().view("<u4")
        inc_w = np.zeros(W, dtype="<u4")
        for p in range(self.nparts):
            if p != self.rank:
                inc_w |= rv[p * W:(p + 1) * W]
        gwords = np.zeros(self.nwords, dtype="<u4")
        gwords[np.arange(W) * self.nparts + self.rank] = inc_w
        inc = _bits(gwords) & self.owned
        for v in np.nonzero(inc & ~self.visited)[0]:
            self.visited[v] = True
            par = SENTINEL
            for u in self.rows[v]:
                self.resolved += 1
                if self.F[u]:
                    par = int(self.new2old[u])
                    break
            assert par != SENTINEL, "no frontier neighbour for a remote discovery"
            self.pred[v] = par
        new = self.visited & ~self.prev & self.owned
        self.level[new] = self.L + 1
        self.frontier = list(np.nonzero(new)[0])
        fs = _words(new)[np.arange(W) * self.nparts + self.rank]
        counts = np.array([len(self.frontier), int(self.deg[new[:self.num_vertices]].sum())], dtype="<u8")
        fsend.copy_(torch.from_numpy(np.concatenate([fs, counts.view("<u4")]).view(np.int32)))

    def sync(self, fgath) -> None:
        W, P = self.words_per_peer, self.nparts
        g = fgath.numpy().view("<u4").reshape(P, W + 4)
        self.summed = tuple(int(x) for x in g[:, W:].copy().view("<u8").sum(axis=0))
        words = g[:, :W].reshape(-1)[self.slot]
        self.F = _bits(words)
        self.visited |= self.F
        self.prev = self.visited.copy()

    def level_done(self, red=None):
        from paper_1604_02844_b200.traversal import LayerStats
        disc, edges = (int(x) for x in red.tolist()) if red is not None else self.summed
        if self.L < 0:
            self.L = 0
            self.cur = (disc, edges)
            return LayerStats(0, 0, 0), disc == 0
        ly = LayerStats(self.cur[0], self.cur[1], disc)
        self.cur = (disc, edges)
        self.L += 1
        return ly, disc == 0

    def finish(self, pred, level) -> None:
        n = self.num_vertices
        pr = np.full(len(pred), SENTINEL, dtype=np.int32)
        lv = np.full(n, -1, dtype=np.int32)
        own = np.nonzero(self.owned[:n] & (self.level[:n] >= 0))[0]
        orig = self.new2old[own]
        pr[orig] = self.pred[own]
        lv[orig] = self.level[own]
        pred.copy_(torch.from_numpy(pr))
        level.copy_(torch.from_numpy(lv))

    def resolve_count(self) -> int:
        return self.resolved
