"""Multi-GPU partitioning of the evaluation.

The path partitions without a data-path collective: independent input value
sets are sharded across the ranks (one process per GPU, the device plan
replicated on each), every rank evaluates its shard with ``run_batch_csr``,
and NCCL is used only when one rank needs every CSR block afterwards
(``gather_csr``).  Timing across ranks is the max (``max_over_ranks``).

Works with any ``torch.distributed`` backend: NCCL on the B200 box, gloo in the
CPU tests (tests/test_shard.py, world size 2).
"""

from __future__ import annotations


def shard_value_sets(total: int, world: int, rank: int) -> tuple[int, int]:
    """(first value set, count) of ``rank``: contiguous, sizes differ by at most one."""
    if total < 0 or world < 1 or not 0 <= rank < world:
        raise ValueError("need total >= 0, world >= 1, 0 <= rank < world")
    base, extra = divmod(total, world)
    count = base + (1 if rank < extra else 0)
    first = rank * base + min(rank, extra)
    return first, count


def gather_csr(out_shard, total: int, dst: int = 0, group=None):
    """Gather every rank's [n_out, count] CSR block into [n_out, total] on ``dst`` (None elsewhere).

    Blocks are padded to the largest shard so one ``gather`` moves them all; the
    value-set order of the result is the global order of ``shard_value_sets``.
    """
    import torch
    import torch.distributed as dist

    world = dist.get_world_size(group)
    rank = dist.get_rank(group)
    counts = [shard_value_sets(total, world, r)[1] for r in range(world)]
    if out_shard.shape[1] != counts[rank]:
        raise ValueError(f"rank {rank} holds {out_shard.shape[1]} value sets, expected {counts[rank]}")
    width = max(counts) if counts else 0
    send = out_shard.new_zeros((out_shard.shape[0], width))
    send[:, : counts[rank]] = out_shard
    recv = [torch.empty_like(send) for _ in range(world)] if rank == dst else None
    dist.gather(send, recv, dst=dst, group=group)
    if rank != dst:
        return None
    return torch.cat([recv[r][:, : counts[r]] for r in range(world)], dim=1)


def max_over_ranks(value: float, device=None, group=None) -> float:
    """The slowest rank's time (the job's time)."""
    import torch
    import torch.distributed as dist

    if not dist.is_initialized() or dist.get_world_size(group) == 1:
        return float(value)
    t = torch.tensor([float(value)], dtype=torch.float64, device=device)
    dist.all_reduce(t, op=dist.ReduceOp.MAX, group=group)
    return float(t.item())


# -- one large evaluation: output nonzeros partitioned, each rank its producer cone ----------


class _OutputSlice:
    """An ExecutionPlan view whose outputs are the CSR positions [lo, hi) (codegen.py:88-98 fields)."""

    def __init__(self, plan, lo: int, hi: int):
        import numpy as np

        self._plan = plan
        self.outputs = np.asarray(plan.outputs, np.int64)[lo:hi]
        self.output_range = (lo, hi)

    def __getattr__(self, name):
        return getattr(self._plan, name)


def shard_outputs(total: int, world: int, rank: int) -> tuple[int, int]:
    """[lo, hi) of the CSR value array ``rank`` evaluates: contiguous, sizes differ by at most one."""
    first, count = shard_value_sets(total, world, rank)
    return first, first + count


def shard_bounds(lowered, n_out: int, world: int, rank: int) -> tuple[int, int]:
    """[lo, hi) of ``rank``'s CSR outputs: the even split of ``shard_outputs``, moved to the nearest
    CSR-window boundary when the plan assembles its outputs in windows (lower._csr_windows), so
    every window belongs to one rank."""
    import numpy as np

    wn = getattr(lowered, "windows", None)
    if wn is None:
        return shard_outputs(n_out, world, rank)
    k = np.asarray(wn.k, np.int64)

    def snap(p):
        j = int(np.argmin(np.abs(k - p)))
        return int(k[j])

    lo, hi = shard_outputs(n_out, world, rank)
    return (0 if rank == 0 else snap(lo)), (n_out if rank == world - 1 else snap(hi))


def output_cone(plan, lo: int, hi: int):
    """Per plan kernel, the instances the CSR outputs [lo, hi) depend on (bool mask of length N).

    Walks the dependency waves backwards from the output addresses: an instance
    is needed when one of its results (``dest_base + r*N + i``, codegen.py:265)
    is needed, and then every address its slots load (``slot_addresses``,
    codegen.py:373-388) is needed.
    """
    import numpy as np

    from .lower import compute_waves
    from .plan import slot_addresses

    need = np.zeros(int(plan.value_array_size), bool)
    need[np.asarray(plan.outputs, np.int64)[lo:hi]] = True
    waves = compute_waves(plan)
    masks = {}
    for k in sorted(range(len(plan.kernels)), key=lambda j: -waves[j]):
        kp = plan.kernels[k]
        n, r = kp.instances, kp.n_roots
        if n == 0:
            masks[k] = np.zeros(0, bool)
            continue
        m = need[kp.dest_base: kp.dest_base + r * n].reshape(r, n).any(axis=0)
        masks[k] = m
        if m.any():
            for col in slot_addresses(plan, kp):
                need[col[m]] = True
    return masks


def shard_device_plan(plan, lowered, lo: int, hi: int):
    """(plan view, lowered view) computing only the CSR outputs [lo, hi): every launch unit keeps the
    tiles that hold an instance of the outputs' producer cone, the gather only those outputs.  The
    value-array layout is unchanged (addresses, index tables and the specialised kernels are the
    full plan's), so the shard's CSR values equal the full evaluation's [lo, hi) bit for bit.
    CSR-mode single-set calls only (run_csr / capture_csr / run_outputs_host)."""
    import dataclasses

    import numpy as np

    from . import lower as L

    if getattr(lowered, "csr_layout", None):
        raise ValueError("output sharding needs the reference value-array layout (csr_layout off)")
    if int(lowered.needs_zero) == 2:
        raise ValueError("output sharding needs a plan without reads before writes")
    # the value-mode twins of CSR-window members carry output positions for batched CSR only (not a
    # mode of the shard): the view drops them
    twins = np.zeros(len(lowered.groups), bool)
    for u in range(len(lowered.units)):
        ur = lowered.unit(u)
        if ur["flags"] & L.UNIT_VALUE_ONLY:
            twins[ur["group_begin"]: ur["group_end"]] = True
    opos_flags = L.FLAG_OPOS16 | L.FLAG_OPOS32
    if np.any((lowered.groups["flags"] & opos_flags) & ~twins):
        raise ValueError("output sharding supports the gather and CSR-window output modes only")
    groups = np.array(lowered.groups, copy=True)
    groups["flags"] = np.where(twins, groups["flags"] & ~opos_flags, groups["flags"])
    wn = getattr(lowered, "windows", None)
    w0 = w1 = 0
    if wn is not None:  # keep the windows [w0, w1) that make up [lo, hi), re-based to the shard
        k = np.asarray(wn.k, np.int64)
        w0, w1 = int(np.searchsorted(k, lo)), int(np.searchsorted(k, hi))
        if k[w0] != lo or k[w1] != hi:
            raise ValueError("a CSR-window plan shards at window boundaries (shard_bounds)")
    masks = output_cone(plan, lo, hi)
    by_base = {int(kp.dest_base): k for k, kp in enumerate(plan.kernels) if kp.instances}
    tiles = np.asarray(lowered.tiles).reshape(-1, 2)
    units = np.array(lowered.units, np.int64, copy=True)
    keep_t, t_cur = [], 0
    for u in range(len(units)):
        ur = lowered.unit(u)
        if ur["flags"] & L.UNIT_WINDOW:  # its "tiles" are windows
            units[u, UNIT_TB], units[u, UNIT_TE] = 0, w1 - w0
            continue
        t = tiles[ur["tile_begin"]: ur["tile_end"]]
        keep = np.zeros(len(t), bool)
        for j, (gi, s) in enumerate(t.tolist()):
            g = lowered.groups[gi]
            k = by_base.get(int(g["dest_base"]))
            if k is None:  # not a plan kernel: keep
                keep[j] = True
                continue
            if g["flags"] & L.FLAG_SERIAL:
                keep[j] = bool(masks[k].any())
                continue
            size = (32 * L.sop_vec(int(g["variant"])) if g["kind"] == L.KIND_SOP
                    else ur["block_size"] * ur["variant"])
            keep[j] = bool(masks[k][s: s + size].any())
        kt = t[keep]
        units[u, UNIT_TB], units[u, UNIT_TE] = t_cur, t_cur + len(kt)
        t_cur += len(kt)
        keep_t.append(kt)
    new_tiles = np.concatenate(keep_t).astype(np.int32) if keep_t else np.zeros((0, 2), np.int32)
    view = _OutputSlice(plan, lo, hi)
    swn = None
    if wn is not None:
        c0, c1 = int(wn.copy_off[w0]), int(wn.copy_off[w1])
        swn = dataclasses.replace(wn, k=np.asarray(wn.k[w0: w1 + 1], np.int64) - lo, pieces=wn.pieces[w0:w1],
                                  copy_off=np.asarray(wn.copy_off[w0: w1 + 1], np.int64) - c0,
                                  copy_src=wn.copy_src[c0:c1], copy_pos=wn.copy_pos[c0:c1])
    lw = dataclasses.replace(lowered, tiles=new_tiles.reshape(-1, 2), units=units, groups=groups,
                             outputs=np.asarray(lowered.outputs, np.int64)[lo:hi], tiles_alt=None, windows=swn)
    return view, lw


UNIT_TB, UNIT_TE = 5, 6  # lower.UNIT_FIELDS tile_begin / tile_end


def shard_device(shard, relayout="auto", **lower_kw):
    """(plan, lowered) one rank runs for a plan shard (``shard_plan``): the shard's own lowering and,
    where it keeps the reference value-array layout, its launch tiles filtered to the instances its
    outputs need -- shard_plan keeps multi-root and self-referencing kernels whole (their result
    stride is N), the tile filter (``shard_device_plan`` over all of the shard's outputs) then skips
    their unneeded instances (C2's face kernel: every rank evaluated all 2M faces)."""
    from .lower import lower_plan

    lw = lower_plan(shard, relayout=relayout, **lower_kw)
    if int(lw.needs_zero) == 2:
        return shard, lw
    if getattr(lw, "csr_layout", None):  # the tile filter needs the reference layout; whole multi-root
        lw = lower_plan(shard, relayout=False, **lower_kw)  # kernels per rank would cost more (C3)
    return shard_device_plan(shard, lw, 0, len(shard.outputs))


def shard_plan(plan, lo: int, hi: int):
    """The plan shard of the CSR outputs [lo, hi): an ExecutionPlan of its own (codegen.py:88-98
    fields), every kernel cut to the instance range its outputs' producer cone needs.

    A kernel outside the cone is dropped; a single-root kernel keeps instances [a, b) -- the first
    to the last needed -- with ``dest_base + a``, so its results stay at the full plan's addresses
    (``dest_base + i``, codegen.py:265) and its position / constant columns are sliced to [a, b);
    multi-root and self-referencing kernels are kept whole (their result stride is N).  Value-array
    addresses are unchanged, so the shard lowers and runs like any plan and its CSR values equal
    the full evaluation's [lo, hi) bit for bit -- while the rank uploads only its share of the
    index tables ("each GPU holds its own plan shard").
    """
    import dataclasses

    import numpy as np

    from .plan import ExecutionPlan

    masks = output_cone(plan, lo, hi)
    positions = np.asarray(plan.positions)
    constants = np.asarray(plan.constants)
    kernels, pos, con = [], [], []
    p_next = c_next = 0
    for k, kp in enumerate(plan.kernels):
        m = masks[k]
        n = kp.instances
        if n == 0 or not m.any():
            continue
        need = np.flatnonzero(m)
        a, b = int(need[0]), int(need[-1]) + 1
        if kp.n_roots != 1 or kp.self_referencing:
            a, b = 0, n
        r, c = len(kp.retained), len(kp.const_vars)
        seg = positions[kp.p_base: kp.p_base + r * n]
        cols = seg.reshape(r, n) if kp.layout == "coalesced" else seg.reshape(n, r).T
        cseg = constants[kp.c_base: kp.c_base + c * n]
        ccols = cseg.reshape(c, n) if kp.layout == "coalesced" else cseg.reshape(n, c).T
        cut = cols[:, a:b]
        ccut = ccols[:, a:b]
        pos.append((cut if kp.layout == "coalesced" else cut.T).reshape(-1))
        con.append((ccut if kp.layout == "coalesced" else ccut.T).reshape(-1))
        kernels.append(dataclasses.replace(kp, instances=b - a, dest_base=kp.dest_base + a, p_base=p_next,
                                           c_base=c_next))
        p_next += cut.size
        c_next += ccut.size
    return ExecutionPlan(
        value_array_size=int(plan.value_array_size), input_count=int(plan.input_count),
        vector_width=int(plan.vector_width), outputs=np.asarray(plan.outputs, np.int64)[lo:hi],
        kernels=kernels,
        positions=np.concatenate(pos).astype(np.uint32) if pos else np.zeros(0, np.uint32),
        constants=np.concatenate(con).astype(np.float64) if con else np.zeros(0, np.float64),
        metadata=dict(getattr(plan, "metadata", {}) or {}, shard=[int(lo), int(hi)]))
