"""fp64 CPU oracle for LeanAttention decode attention (arXiv 2405.10480).

TEST INFRASTRUCTURE ONLY.  Only ``tests/``, ``__graft_entry__.smoke()`` and ``bench.py``'s
``cpu_baseline`` leg / ``--impl reference`` arm may import or execute anything under
``oracle/``.  The product path (``paper_2405_10480_b200``) never imports it and shares no
code, header, table or constant generator with it.

Citations: ``P:n`` = line n of the paper text; ``S:n`` = line n of SPEC.md.

Modules
-------
* :mod:`oracle.attention`  -- Eq. 1, the plain definition of decode attention,
  materialising S in fp64.  This is THE parity reference: LeanAttention is exact attention
  ("same exact attention output"), reached faster.
* :mod:`oracle.rescale`    -- §4.1: un-scaled partial (O~, m, l), the softmax
  re-scaling operator f(x, y), its neutral element and finalisation (Alg. 2 §38-39).
* :mod:`oracle.leantile`   -- Alg. 1 LeanTile(), step by step, in fp64.
* :mod:`oracle.schedule`   -- Alg. 2 §4-18/§41 stream-K segment walk and
  an independent per-iteration owner enumeration (the planner's bit-exact reference).
* :mod:`oracle.lean_attention` -- Alg. 2 executed serially in fp64 (partials, host folds).
* :mod:`oracle.fp8`         -- E4M3 byte -> value (the OCP format definition) and the
  per-tensor dequantisation of an FP8 KV cache (NEXT-4; not in the paper).
* :mod:`oracle.shard_combine` -- the sequence-shard combine of normalised (O_r, L_r) pairs
  (BASELINE.json north star; exact by §4.1's associativity).

Parity status of every function is listed in DESIGN.md §"Oracle and pins"; all are pinned.
"""
from .attention import (decode_attention, decode_attention_unit, decode_attention_multi, decode_attention_varq,
                        paged_rows, scores)
from .rescale import PartialState, neutral, partial, combine, finalize, fold
from .leantile import lean_tile
from .schedule import (Segment, iters_per_cta, cta_range, owner, stream_k_segments,
                       owner_table, segments_from_owner_table, last_cta_literal,
                       fixed_split_segments, quantization_efficiency, segments_from_ranges,
                       balanced_ranges, fixed_split_ranges, fa2_num_splits, weighted_ranges)
from .lean_attention import lean_attention
from .shard_combine import combine_shards
from .fp8 import e4m3_decode, dequantize

__all__ = [
    "decode_attention", "decode_attention_unit", "decode_attention_multi", "decode_attention_varq", "scores",
    "PartialState", "neutral", "partial", "combine", "finalize", "fold",
    "lean_tile",
    "Segment", "iters_per_cta", "cta_range", "owner", "stream_k_segments", "owner_table",
    "segments_from_owner_table", "last_cta_literal", "fixed_split_segments",
    "quantization_efficiency", "segments_from_ranges", "balanced_ranges", "fixed_split_ranges",
    "fa2_num_splits",
    "lean_attention", "combine_shards", "e4m3_decode", "dequantize",
]
