"""Algorithmic (compulsory) traffic and op counts of a plan -- SURVEY.md §8(d).

Per launch (one dependency wave, or the output gather) the compulsory bytes
are what any implementation of that launch must move through HBM at least
once:

    index tables     4 * (retained position entries of the wave's groups)
  + constants        8 * (constant entries)
  + reads            8 * (distinct value-array addresses the wave loads)
  + writes           8 * (result slots the wave writes: sum N*R)

and for the output gather ``4 * n_out`` (u32 index) + ``8 * distinct output
addresses`` + ``8 * n_out`` (CSR values written).  Summed over a plan this is
the §8(d) ``B_alg`` with intermediates counted once per launch that touches
them (they cross HBM between launches), so it is >= the single-pass figure
and is the right denominator for a per-kernel roofline.

FP64 op count per instance follows §8(d): ADD/MUL count children-1, every
other op 1 (DIV/SQRT/transcendentals are 1 op each though they cost more).
"""

from __future__ import annotations

from dataclasses import dataclass

import numpy as np

from .plan import slot_addresses, unique_addresses


@dataclass
class LaunchTraffic:
    name: str
    index_bytes: int
    const_bytes: int
    read_bytes: int
    write_bytes: int
    fp64_ops: int

    @property
    def bytes(self) -> int:
        return self.index_bytes + self.const_bytes + self.read_bytes + self.write_bytes


def wave_traffic(plan, lowered, batch: int = 1) -> list[LaunchTraffic]:
    """One record per wave launch, then one for the output gather."""
    out = []
    by_wave: dict[int, list] = {}
    for kl in lowered.kernels:
        by_wave.setdefault(kl.wave, []).append(kl)
    for w in range(lowered.n_waves):
        idx = con = wr = ops = 0
        addrs = []
        for kl in by_wave.get(w, []):
            kp = plan.kernels[kl.index]
            idx += 4 * len(kp.retained) * kp.instances
            con += 8 * len(kp.const_vars) * kp.instances
            wr += 8 * kp.n_roots * kp.instances * batch
            ops += kl.ops * kp.instances * batch
            if kp.pos_vars:
                addrs.append(unique_addresses(np.concatenate(slot_addresses(plan, kp))))
        reads = int(unique_addresses(np.concatenate(addrs)).size) if addrs else 0
        out.append(LaunchTraffic(f"wave{w}", idx, con, 8 * reads * batch, wr, ops))
    outs = np.asarray(plan.outputs, dtype=np.int64)
    n_out = int(outs.size)
    out.append(LaunchTraffic("gather_outputs", 4 * n_out, 0, 8 * int(unique_addresses(outs).size) * batch,
                             8 * n_out * batch, 0))
    return out


def csr_wave_traffic(plan, lowered, batch: int = 1) -> list[LaunchTraffic]:
    """Per CSR-mode wave (sgb_run_csr): compulsory bytes of each launch wave.

    index + constants as above; reads = 8 B per distinct address loaded by the
    wave's groups and copy groups; writes = 8 B per result slot a later wave
    re-reads plus 8 B per output value stored (first occurrence by its
    producer, the rest by copy groups).  Output-position tables are an
    encoding overhead of this backend, not algorithmic bytes.
    """
    outs = np.asarray(plan.outputs, dtype=np.int64)
    uniq = unique_addresses(outs)
    waves = max([lowered.n_waves] + [w + 1 for w, _, _ in lowered.copies])
    wn = getattr(lowered, "windows", None)
    members = set(getattr(lowered, "window_members", []) or [])
    out = []
    for w in range(waves):
        idx = con = wr = ops = 0
        addrs = []
        for kl in lowered.kernels:
            if kl.wave != w:
                continue
            kp = plan.kernels[kl.index]
            idx += 4 * len(kp.retained) * kp.instances
            con += 8 * len(kp.const_vars) * kp.instances
            ops += kl.ops * kp.instances * batch
            lo, hi = kp.dest_base, kp.dest_base + kp.n_roots * kp.instances
            if kl.index in members:  # CSR windows: every output is written once, below
                pass
            elif kl.flags & 16:  # FLAG_STREAM: only the outputs are stored
                a, b = np.searchsorted(uniq, [lo, hi])
                wr += 8 * int(b - a) * batch
            else:
                wr += 8 * kp.n_roots * kp.instances * batch
            if kp.pos_vars:
                addrs.append(unique_addresses(np.concatenate(slot_addresses(plan, kp))))
        for cw, src, _ in lowered.copies:
            if cw == w:
                idx += 4 * src.size
                wr += 8 * src.size * batch
                addrs.append(unique_addresses(src))
        if wn is not None and w == lowered.n_waves - 1:  # the window unit: copies + every output once
            src = np.asarray(wn.copy_src, np.int64)
            idx += 4 * src.size
            wr += 8 * int(outs.size) * batch
            if src.size:
                addrs.append(unique_addresses(src))
        reads = int(unique_addresses(np.concatenate(addrs)).size) if addrs else 0
        out.append(LaunchTraffic(f"csr_wave{w}", idx, con, 8 * reads * batch, wr, ops))
    return out


def plan_balg(plan) -> int:
    """SURVEY §8(d) single-evaluation B_alg of the plan (intermediates once)."""
    P = int(np.asarray(plan.positions).size)
    C = int(np.asarray(plan.constants).size)
    n_res = sum(kp.n_roots * kp.instances for kp in plan.kernels)
    reread = []
    for kp in plan.kernels:
        for col in slot_addresses(plan, kp):
            reread.append(col[col >= plan.input_count])
    n_reread = int(unique_addresses(np.concatenate(reread)).size) if reread else 0
    outs = np.asarray(plan.outputs, dtype=np.int64)
    dup = int(outs.size - unique_addresses(outs).size)
    return 4 * P + 8 * C + 8 * (int(plan.input_count) + n_res + n_reread + dup)
