"""Stream-K decomposition and mapping of LeanTiles (§4.3, Alg. 2).  TEST INFRASTRUCTURE ONLY.

Integer work; the C++ planner must reproduce it bit-exactly.

* Linearisation: units (output tiles) in batch -> heads order, each unit's C_n
  LeanTile iterations contiguous ("crossing the head and query boundary as it may").  For
  the ragged packed layout the order is heads -> total context.  Reading C14: the
  caller passes the per-unit C_n list already in memory order of its KV layout.
* Eq. 2 / Alg. 2 §4-7: I = sum_u C_n(u), I_G = I / G.
  Reading C8: the first r = I mod G CTAs take ceil(I/G), the rest floor(I/G)
  (cta_start = g*floor(I/G) + min(g, r)).
* Alg. 2 §8-18 + §41: each CTA walks its range segment by segment
  (reading C10: while-loop, iter jumps to tile_iter_end).  host-block iff iter == tile_iter
  (§17); finishing-block iff cta_end >= tile_iter_end (§18).
* Alg. 2 §26 ``last_cta = tile_iter_end / C_n`` is garbled (it is a tile index);
  reading C9: last_cta = owner(tile_iter_end - 1), the CTA holding the tile's last
  iteration.  :func:`last_cta_literal` keeps the literal formula so a test can show it
  drops a contributor on the paper's own Fig. 1 example.

Two independent constructions are provided and tested against each other:
:func:`stream_k_segments` (Alg. 2's per-CTA walk) and :func:`segments_from_owner_table`
(brute force: the owner of every single global iteration, grouped into maximal runs).
"""
from __future__ import annotations

import math
from dataclasses import dataclass
from typing import List, Sequence, Tuple


@dataclass(frozen=True)
class Segment:
    """One call of LeanTile() by one CTA: Alg. 2 §11-18 quantities for that call."""

    cta: int           # g
    unit: int          # tile_idx (output tile = work unit)
    begin: int         # local_iter
    end: int           # local_iter_end (exclusive)
    host: bool         # iter == tile_iter                     (§17)
    finishing: bool    # cta_end >= tile_iter_end              (§18)
    last_cta: int      # owner(tile_iter_end - 1)              (§26, reading C9)

    def row(self) -> Tuple[int, int, int, int, int, int, int]:
        return (self.cta, self.unit, self.begin, self.end, int(self.host),
                int(self.finishing), self.last_cta)


def iters_per_cta(total_iters: int, grid: int) -> List[int]:
    """Per-CTA iteration counts: Eq. 2 / Alg. 2 §7 with reading C8's remainder rule."""
    if grid < 1:
        raise ValueError("grid must be >= 1")
    q, r = divmod(total_iters, grid)
    return [q + 1 if g < r else q for g in range(grid)]


def cta_range(total_iters: int, grid: int, g: int) -> Tuple[int, int]:
    """Alg. 2 §9: [cta_start, cta_end) of CTA g."""
    q, r = divmod(total_iters, grid)
    start = g * q + min(g, r)
    return start, start + (q + 1 if g < r else q)


def owner(total_iters: int, grid: int, it: int) -> int:
    """The CTA whose range contains global iteration ``it`` (closed form of reading C8)."""
    q, r = divmod(total_iters, grid)
    if it < r * (q + 1):
        return it // (q + 1)
    return r + (it - r * (q + 1)) // q


def _offsets(c_n: Sequence[int]) -> List[int]:
    off = [0]
    for c in c_n:
        if c < 1:
            raise ValueError("every unit needs >= 1 LeanTile (reading C6)")
        off.append(off[-1] + c)
    return off


def stream_k_segments(c_n: Sequence[int], grid: int) -> List[Segment]:
    """Alg. 2 §8-18, §41 executed for every CTA in index order."""
    off = _offsets(c_n)
    total = off[-1]
    segs: List[Segment] = []
    unit = 0
    for g in range(grid):                                   # fork CTA_g       (§8)
        cta_start, cta_end = cta_range(total, grid, g)      #                  (§9)
        it = cta_start
        while it < cta_end:                                 # (§10, reading C10)
            while off[unit + 1] <= it:                      # tile_idx         (§11)
                unit += 1
            tile_iter = off[unit]                           #                  (§12)
            tile_iter_end = tile_iter + c_n[unit]           #                  (§13)
            local_iter = it - tile_iter                     #                  (§14)
            local_iter_end = min(tile_iter_end, cta_end) - tile_iter  #        (§15)
            segs.append(Segment(
                cta=g, unit=unit, begin=local_iter, end=local_iter_end,
                host=(it == tile_iter),                     #                  (§17)
                finishing=(cta_end >= tile_iter_end),       #                  (§18)
                last_cta=owner(total, grid, tile_iter_end - 1)))   # (§26, reading C9)
            it = tile_iter_end                              #                  (§41)
    return segs


def segments_from_ranges(c_n: Sequence[int], begins: Sequence[int]) -> List[Segment]:
    """Alg. 2 §10-18, §41 for arbitrary contiguous per-CTA ranges [begins[v], begins[v+1])
    (§9's equal split replaced by a table); last_cta = the range holding the unit's last
    iteration (reading C9)."""
    off = _offsets(c_n)
    assert begins[0] == 0 and begins[-1] == off[-1] and all(a <= b for a, b in zip(begins, begins[1:]))

    def own(it):  # the range containing global iteration it
        lo, hi = 0, len(begins) - 2
        while lo < hi:
            mid = (lo + hi + 1) // 2
            if begins[mid] <= it:
                lo = mid
            else:
                hi = mid - 1
        return lo

    segs: List[Segment] = []
    unit = 0
    for v in range(len(begins) - 1):
        cta_start, cta_end = begins[v], begins[v + 1]
        it = cta_start
        while it < cta_end:
            while off[unit + 1] <= it:
                unit += 1
            tile_iter, tile_iter_end = off[unit], off[unit + 1]
            segs.append(Segment(cta=v, unit=unit, begin=it - tile_iter,
                                end=min(tile_iter_end, cta_end) - tile_iter,
                                host=(it == tile_iter), finishing=(cta_end >= tile_iter_end),
                                last_cta=own(tile_iter_end - 1)))
            it = tile_iter_end
    return segs


def balanced_ranges(total_iters: int, grid: int, head_permille: int = 940, min_chunk: int = 2,
                    max_chunks: int = 8) -> Tuple[List[int], List[int]]:
    """Virtual-CTA ranges and claim order of the DYNAMIC schedule (this build's
    extension, not in the paper).  Every range of Eq. 2 (Alg. 2 §7-9, reading C8) is cut
    into a HEAD -- its first part -- and a TAIL of k chunks of s LeanTiles:

        L = |range g|,  T0 = floor(L (1000 - head_permille) / 1000)
        s = max(min_chunk, ceil(T0 / max_chunks)),  k = floor(T0 / s),  tail = the last k s

    Returns (begins, claim): ``begins`` the boundaries of all pieces in iteration order
    (range 0's head, its chunks, range 1's head, ...; empty ranges contribute nothing) and
    ``claim`` the order in which persistent CTAs take them: every head (in range order),
    then chunk 0 of every range that has one, chunk 1 of every range, ...  head_permille =
    1000 leaves no tail: exactly Alg. 2's equal ranges, claimed in range order."""
    begins: List[int] = [0]
    heads: List[int] = []
    tails: List[List[int]] = []
    v = 0
    for g in range(grid):
        b, e = cta_range(total_iters, grid, g)
        L = e - b
        if L == 0:
            continue
        t0 = L * (1000 - head_permille) // 1000
        s = max(min_chunk, -(-t0 // max_chunks))
        k = min(t0 // s, (L - 1) // s)          # the head keeps >= 1 LeanTile
        heads.append(v)                           # head [b, e - k s)
        begins.append(e - k * s)
        v += 1
        chunks = []
        for j in range(1, k + 1):                 # chunk j-1: [e - (k - j + 1) s, e - (k - j) s)
            chunks.append(v)
            begins.append(e - (k - j) * s)
            v += 1
        tails.append(chunks)
    claim = list(heads)
    for j in range(max((len(t) for t in tails), default=0)):
        claim.extend(t[j] for t in tails if j < len(t))
    assert len(begins) == v + 1 and sorted(claim) == list(range(v))
    return begins, claim


def weighted_ranges(total_iters: int, weights: Sequence[int]) -> List[int]:
    """Range boundaries of the SM-rate-weighted stream-K schedule (this
    build's extension of Eq. 2, not in the paper): Eq. 2 hands every CTA I / G
    LeanTiles; here CTA g's share is proportional to its weight w_g (its SM's measured
    streaming rate) on top of one LeanTile each,

        R = max(I - G, 0),  begins[g] = min(g, I) + floor(R * (w_0 + ... + w_{g-1}) / W),

    W = w_0 + ... + w_{G-1}, in exact integer arithmetic.  Every CTA g < I gets >= 1
    LeanTile (an empty range inside a unit would leave its host waiting for a partial
    nobody writes; with I < G the trailing CTAs idle, as Alg. 2's).  The ranges stay
    contiguous, so Alg. 2 §10-18 runs over them unchanged (``segments_from_ranges``)."""
    assert len(weights) >= 1 and all(1 <= int(w) <= (1 << 20) for w in weights)
    G, W = len(weights), sum(int(w) for w in weights)
    R = max(total_iters - G, 0)
    begins, acc = [], 0
    for g, w in enumerate(list(weights) + [0]):
        begins.append(min(g, total_iters) + R * acc // W)
        acc += int(w)
    return begins


def fixed_split_ranges(c_n: Sequence[int], split: int) -> List[int]:
    """Range boundaries of FlashDecoding's fixed split: unit u cut into
    s = min(split, C_n(u)) chunks, the first C_n mod s of them one LeanTile longer."""
    begins = [0]
    pos = 0
    for c in c_n:
        s = max(1, min(split, c))
        q, r = divmod(c, s)
        for j in range(s):
            pos += q + (1 if j < r else 0)
            begins.append(pos)
    return begins


def fa2_num_splits(units: int, max_cn: int, sms: int) -> int:
    """FlashAttention-2's split heuristic used by FlashDecoding (the paper's FD baseline,
    P:505): no split if the units fill 80% of the SMs, else the smallest s whose wave
    efficiency units*s / (ceil(units*s/sms) * sms) reaches 85% of the best s <= 128."""
    if units >= int(0.8 * sms):
        return 1
    max_s = min(128, sms, max_cn)
    eff = {}
    for s in range(1, max_s + 1):
        waves = units * s / sms
        eff[s] = waves / math.ceil(waves)
    best = max(eff.values())
    for s in range(1, max_s + 1):
        if eff[s] >= 0.85 * best:
            return s
    return 1


def owner_table(total_iters: int, grid: int) -> List[int]:
    """Brute force: hand out iterations CTA by CTA, counts from :func:`iters_per_cta`."""
    table: List[int] = []
    for g, n in enumerate(iters_per_cta(total_iters, grid)):
        table.extend([g] * n)
    assert len(table) == total_iters
    return table


def segments_from_owner_table(c_n: Sequence[int], grid: int) -> List[Segment]:
    """Independent construction: maximal runs of equal (owner, unit) over all iterations."""
    off = _offsets(c_n)
    own = owner_table(off[-1], grid)
    segs: List[Segment] = []
    for u in range(len(c_n)):
        first, last = off[u], off[u + 1] - 1
        run_start = first
        for it in range(first, last + 1):
            if it == last or own[it + 1] != own[it]:
                segs.append(Segment(
                    cta=own[it], unit=u, begin=run_start - first, end=it + 1 - first,
                    host=(run_start == first), finishing=(it == last),
                    last_cta=own[last]))
                run_start = it + 1
    segs.sort(key=lambda s: (s.cta, s.unit))
    return segs


def last_cta_literal(c_n_uniform: int, unit: int) -> int:
    """Alg. 2 §26 read literally: tile_iter_end / C_n (= unit + 1).  Kept only to test that
    it is NOT the CTA index (reading C9)."""
    tile_iter_end = (unit + 1) * c_n_uniform
    return tile_iter_end // c_n_uniform


def fixed_split_segments(c_n: Sequence[int], grid: int, split: int) -> List[Segment]:
    """FlashDecoding's fixed-split decomposition: each unit's C_n
    iterations cut into ``split`` near-equal chunks (first chunks take the extra iteration,
    S:271), chunks dealt round-robin to the grid in launch order; host = chunk 0.
    ``cta`` is the worker; a worker may hold several chunks (successive waves)."""
    segs: List[Segment] = []
    chunk_id = 0
    for u, c in enumerate(c_n):
        s = min(split, c)
        q, r = divmod(c, s)
        begin = 0
        chunk_owner = []
        for j in range(s):
            n = q + 1 if j < r else q
            chunk_owner.append((chunk_id % grid, begin, begin + n))
            chunk_id += 1
            begin += n
        last_owner = chunk_owner[-1][0]
        for j, (w, b0, b1) in enumerate(chunk_owner):
            segs.append(Segment(cta=w, unit=u, begin=b0, end=b1, host=(j == 0),
                                finishing=(j == s - 1), last_cta=last_owner))
    return segs


def quantization_efficiency(segs: Sequence[Segment], grid: int) -> float:
    """I / (G * max per-worker iterations)."""
    load = [0] * grid
    for s in segs:
        load[s.cta] += s.end - s.begin
    return sum(load) / (grid * max(load))
