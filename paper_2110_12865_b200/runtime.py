"""Drop-in GPU backend for the reference evaluators (ctypes over libsgb.so).

Mirrors the reference's evaluation API:

* ``interpret_plan(plan, inputs, record_loads=False, check_schedule=False)
  -> InterpretResult`` -- codegen.py:404-446, same arguments, same result
  fields, same ``ValueError`` on an input-length mismatch (:415-418); the
  values come from the B200.
* ``compile_plan(plan, work_dir=None, parallel="none", device=0) -> run`` --
  emit.py:198-245: ``run(inputs)`` returns the FULL value array like the
  emitted ``sg_run``; ``run.outputs(inputs)`` returns only the CSR values;
  ``run.library_path`` names the loaded native library.  Unlike the
  reference (which returns None without a C compiler) a missing CUDA
  extension or GPU raises: there is no CPU fallback.
* ``DevicePlan`` -- the device-resident plan for stream-ordered use on torch
  tensors (``run_values``, ``gather_outputs``, ``run_batch``).
"""

from __future__ import annotations

import ctypes
import threading
from dataclasses import dataclass, field
from pathlib import Path
from typing import Sequence

import numpy as np

from .lower import GROUP_DTYPE, lower_plan
from .plan import slot_addresses

_PKG = Path(__file__).resolve().parent
LIB_PATH = _PKG / "libsgb.so"

_lib = None
_lib_lock = threading.Lock()


class SgbError(RuntimeError):
    pass


class _Desc(ctypes.Structure):
    _fields_ = [
        ("value_array_size", ctypes.c_int64),
        ("input_count", ctypes.c_int64),
        ("n_groups", ctypes.c_int32),
        ("n_waves", ctypes.c_int32),
        ("n_units", ctypes.c_int32),
        ("needs_zero", ctypes.c_int32),
        ("groups", ctypes.c_void_p),
        ("units", ctypes.c_void_p),
        ("tiles", ctypes.c_void_p),
        ("n_tiles", ctypes.c_int64),
        ("tape", ctypes.c_void_p),
        ("tape_rows", ctypes.c_int64),
        ("imm", ctypes.c_void_p),
        ("n_imm", ctypes.c_int64),
        ("sop", ctypes.c_void_p),
        ("n_sop", ctypes.c_int64),
        ("slot_col", ctypes.c_void_p),
        ("slot_delta", ctypes.c_void_p),
        ("n_slot", ctypes.c_int64),
        ("positions", ctypes.c_void_p),
        ("n_positions", ctypes.c_int64),
        ("constants", ctypes.c_void_p),
        ("n_constants", ctypes.c_int64),
        ("cbase", ctypes.c_void_p),
        ("n_cbase", ctypes.c_int64),
        ("coff", ctypes.c_void_p),
        ("n_coff", ctypes.c_int64),
        ("obase", ctypes.c_void_p),
        ("n_obase", ctypes.c_int64),
        ("ooff", ctypes.c_void_p),
        ("n_ooff", ctypes.c_int64),
        ("opos32", ctypes.c_void_p),
        ("n_opos32", ctypes.c_int64),
        ("outputs", ctypes.c_void_p),
        ("n_outputs", ctypes.c_int64),
        ("jit_cubin", ctypes.c_void_p),
        ("jit_cubin_size", ctypes.c_int64),
        ("win_pieces", ctypes.c_void_p),
        ("n_win_pieces", ctypes.c_int64),
        ("win_k", ctypes.c_void_p),
        ("n_win_k", ctypes.c_int64),
        ("win_copy", ctypes.c_void_p),
        ("n_win_copy", ctypes.c_int64),
        ("copy_src", ctypes.c_void_p),
        ("copy_pos", ctypes.c_void_p),
        ("n_copy", ctypes.c_int64),
        ("win_meta", ctypes.c_void_p),
        ("n_win_meta", ctypes.c_int64),
        ("win_meta_off", ctypes.c_void_p),
        ("win_iv", ctypes.c_void_p),
        ("n_win_iv", ctypes.c_int64),
        ("win_iv_off", ctypes.c_void_p),
        ("win_bulk", ctypes.c_void_p),
        ("win_ring", ctypes.c_int64),
        ("win_slot_meta", ctypes.c_int64),
        ("win_slot_x", ctypes.c_int64),
        ("win_bw", ctypes.c_int64),
    ]


SYMBOLS = (
    "sgb_plan_create", "sgb_plan_destroy", "sgb_run_values", "sgb_run_csr", "sgb_gather_outputs",
    "sgb_sg_run", "sgb_run_outputs_host", "sgb_run_outputs_host_many", "sgb_run_batch", "sgb_run_batch_csr", "sgb_gather_outputs_batch",
    "sgb_plan_waves", "sgb_last_error", "sgb_run_wave", "sgb_plan_units", "sgb_plan_set_tiles",
    "sgb_plan_set_wave_grid", "sgb_plan_value_slots", "sgb_run_inputs_csr",
)


def load_library(path: Path | str | None = None):
    """Load libsgb.so (raises if it is missing: the product has no fallback)."""
    global _lib
    with _lib_lock:
        if _lib is not None and path is None:
            return _lib
        p = Path(path) if path else LIB_PATH
        if not p.exists():
            raise SgbError(f"{p} is missing; build it with __graft_entry__.build() "
                           "(python -m paper_2110_12865_b200._build)")
        lib = ctypes.CDLL(str(p))
        vp, i64, i32 = ctypes.c_void_p, ctypes.c_int64, ctypes.c_int
        sig = {
            "sgb_plan_create": (i32, [ctypes.POINTER(_Desc), i32, ctypes.POINTER(vp)]),
            "sgb_plan_destroy": (None, [vp]),
            "sgb_run_values": (i32, [vp, vp, vp]),
            "sgb_run_csr": (i32, [vp, vp, vp, vp]),
            "sgb_run_wave": (i32, [vp, vp, vp, i32, vp]),
            "sgb_gather_outputs": (i32, [vp, vp, vp, vp]),
            "sgb_sg_run": (i32, [vp, vp, vp, vp]),
            "sgb_run_outputs_host": (i32, [vp, vp, vp]),
            "sgb_run_outputs_host_many": (i32, [vp, i64, vp, i64, vp, i64]),
            "sgb_run_batch": (i32, [vp, vp, i64, i64, vp]),
            "sgb_run_batch_csr": (i32, [vp, vp, i64, i64, vp, i64, vp]),
            "sgb_gather_outputs_batch": (i32, [vp, vp, i64, i64, vp, i64, vp]),
            "sgb_plan_waves": (i32, [vp, i32]),
            "sgb_plan_units": (i32, [vp, i32]),
            "sgb_plan_set_tiles": (i32, [vp, vp, i64]),
            "sgb_plan_set_wave_grid": (i32, [vp, i32, i32]),
            "sgb_plan_value_slots": (i64, [vp]),
            "sgb_run_inputs_csr": (i32, [vp, vp, vp, vp]),
            "sgb_last_error": (ctypes.c_char_p, []),
        }
        for name, (res, args) in sig.items():
            fn = getattr(lib, name)
            fn.restype = res
            fn.argtypes = args
        if path is None:
            _lib = lib
        return lib


def _check(rc: int, what: str):
    if rc != 0:
        msg = load_library().sgb_last_error().decode(errors="replace")
        raise SgbError(f"{what} failed ({rc}): {msg}")


def _ptr(a: np.ndarray):
    return ctypes.c_void_p(a.ctypes.data) if a.size else ctypes.c_void_p(0)


def _stream_handle(stream) -> ctypes.c_void_p:
    if stream is None:
        import torch

        return ctypes.c_void_p(torch.cuda.current_stream().cuda_stream)
    if isinstance(stream, int):
        return ctypes.c_void_p(stream)
    return ctypes.c_void_p(stream.cuda_stream)


class DevicePlan:
    """A reference ExecutionPlan lowered and uploaded to one B200."""

    def __init__(self, plan, device: int = 0, lowered=None, csr_layout: bool = False):
        """``csr_layout``: lower with the CSR layout (lower.choose_relayout) -- CSR-mode
        calls only (run_csr, capture_csr, run_outputs_host, run_batch_csr); the
        value-mode calls raise SgbError.  ``SGB_RELAYOUT`` = auto (default) / all / 0."""
        import os

        import torch

        if not torch.cuda.is_available():
            raise SgbError("no CUDA device: the B200 backend has no CPU fallback")
        self.plan = plan
        self.device = int(device)
        if lowered is None:
            mode = os.environ.get("SGB_RELAYOUT", "auto") if csr_layout else False
            lowered = lower_plan(plan, relayout=False if mode in ("0", "") else mode)
        self.lowered = lowered
        self.csr_layout = bool(getattr(lowered, "csr_layout", None))
        self.value_array_size = int(plan.value_array_size)
        self.input_count = int(plan.input_count)
        self.n_outputs = len(plan.outputs)
        self._lib = load_library()
        self._handle = ctypes.c_void_p(0)
        lw = self.lowered
        keep = dict(
            groups=np.ascontiguousarray(lw.groups, GROUP_DTYPE),
            units=np.ascontiguousarray(lw.units, np.int64),
            tiles=np.ascontiguousarray(lw.tiles, np.int32).reshape(-1, 2),
            tape=np.ascontiguousarray(lw.tape, np.uint32).reshape(-1, 4),
            imm=np.ascontiguousarray(lw.imm, np.float64),
            sop=np.ascontiguousarray(lw.sop, np.uint32),
            scol=np.ascontiguousarray(lw.slot_col, np.int32),
            sdel=np.ascontiguousarray(lw.slot_delta, np.int64),
            pos=np.ascontiguousarray(lw.positions, np.uint32),
            con=np.ascontiguousarray(lw.constants, np.float64),
            cbase=np.ascontiguousarray(lw.cbase, np.uint32),
            coff=np.ascontiguousarray(lw.coff, np.uint16),
            obase=np.ascontiguousarray(lw.obase, np.uint32),
            ooff=np.ascontiguousarray(lw.ooff, np.uint16),
            opos32=np.ascontiguousarray(lw.opos32, np.uint32),
            outs=np.ascontiguousarray(lw.outputs, np.int64),
            cubin=np.frombuffer(lw.jit_cubin, dtype=np.uint8).copy() if lw.jit_cubin else np.zeros(0, np.uint8),
        )
        wn = getattr(lw, "windows", None)
        keep.update(
            wpieces=np.ascontiguousarray(wn.pieces if wn is not None else np.zeros((0, 2)), np.int32).reshape(-1, 2),
            wk=np.ascontiguousarray(wn.k if wn is not None else np.zeros(0), np.int64),
            wcopy=np.ascontiguousarray(wn.copy_off if wn is not None else np.zeros(0), np.int64),
            csrc=np.ascontiguousarray(wn.copy_src if wn is not None else np.zeros(0), np.uint32),
            cpos=np.ascontiguousarray(wn.copy_pos if wn is not None else np.zeros(0), np.uint16),
        )
        wb = getattr(lw, "wbulk", None)
        bulk_flags = np.zeros(wn.pieces.shape[1] if wn is not None else 0, np.int32)
        if wb is not None:
            bulk_flags[wb.members] = 1
        keep.update(
            wmeta=np.ascontiguousarray(wb.meta if wb is not None else np.zeros(0), np.uint8),
            wmeta_off=np.ascontiguousarray(wb.meta_off if wb is not None else np.zeros(0), np.int64),
            wiv=np.ascontiguousarray(wb.iv if wb is not None else np.zeros((0, 2)), np.uint32).reshape(-1, 2),
            wiv_off=np.ascontiguousarray(wb.iv_off if wb is not None else np.zeros(0), np.int64),
            wbulk=bulk_flags,
        )
        d = _Desc(
            value_array_size=self.value_array_size, input_count=self.input_count,
            n_groups=len(keep["groups"]), n_waves=lw.n_waves, n_units=len(keep["units"]),
            needs_zero=int(lw.needs_zero),
            groups=_ptr(keep["groups"]), units=_ptr(keep["units"]), tiles=_ptr(keep["tiles"]),
            n_tiles=keep["tiles"].shape[0], tape=_ptr(keep["tape"]),
            tape_rows=keep["tape"].shape[0], imm=_ptr(keep["imm"]), n_imm=keep["imm"].size,
            sop=_ptr(keep["sop"]), n_sop=keep["sop"].size, slot_col=_ptr(keep["scol"]),
            slot_delta=_ptr(keep["sdel"]), n_slot=keep["scol"].size, positions=_ptr(keep["pos"]),
            n_positions=keep["pos"].size, constants=_ptr(keep["con"]), n_constants=keep["con"].size,
            cbase=_ptr(keep["cbase"]), n_cbase=keep["cbase"].size, coff=_ptr(keep["coff"]),
            n_coff=keep["coff"].size, obase=_ptr(keep["obase"]), n_obase=keep["obase"].size,
            ooff=_ptr(keep["ooff"]), n_ooff=keep["ooff"].size, opos32=_ptr(keep["opos32"]),
            n_opos32=keep["opos32"].size, outputs=_ptr(keep["outs"]), n_outputs=keep["outs"].size,
            jit_cubin=_ptr(keep["cubin"]), jit_cubin_size=keep["cubin"].size,
            win_pieces=_ptr(keep["wpieces"]), n_win_pieces=keep["wpieces"].shape[0],
            win_k=_ptr(keep["wk"]), n_win_k=keep["wk"].size, win_copy=_ptr(keep["wcopy"]),
            n_win_copy=keep["wcopy"].size, copy_src=_ptr(keep["csrc"]), copy_pos=_ptr(keep["cpos"]),
            n_copy=keep["csrc"].size,
            win_meta=_ptr(keep["wmeta"]), n_win_meta=keep["wmeta"].size, win_meta_off=_ptr(keep["wmeta_off"]),
            win_iv=_ptr(keep["wiv"]), n_win_iv=keep["wiv"].shape[0], win_iv_off=_ptr(keep["wiv_off"]),
            win_bulk=_ptr(keep["wbulk"]),
            win_ring=wb.ring if wb is not None else 0, win_slot_meta=wb.slot_meta if wb is not None else 0,
            win_slot_x=wb.slot_x if wb is not None else 0, win_bw=wb.bw if wb is not None else 0,
        )
        torch.cuda.init()
        _check(self._lib.sgb_plan_create(ctypes.byref(d), self.device, ctypes.byref(self._handle)),
               "sgb_plan_create")
        self.launches = int(self._lib.sgb_plan_waves(self._handle, 0))  # value-mode waves
        self.csr_launches = int(self._lib.sgb_plan_waves(self._handle, 1))  # CSR-mode waves
        self.units = int(self._lib.sgb_plan_units(self._handle, 0))  # kernel launches per evaluation
        self.value_slots = int(self._lib.sgb_plan_value_slots(self._handle))  # CSR workspace doubles
        self.csr_units = int(self._lib.sgb_plan_units(self._handle, 1))
        self.tile_order = {}  # wave -> (schedule, grid) kept by autotune
        if os.environ.get("SGB_AUTOTUNE", "1") != "0":
            self.autotune()

    def set_tiles(self, tiles: np.ndarray):
        """Swap in another schedule of the plan's tiles (sgb_plan_set_tiles)."""
        t = np.ascontiguousarray(tiles, np.int32).reshape(-1, 2)
        _check(self._lib.sgb_plan_set_tiles(self._handle, _ptr(t), t.shape[0]), "sgb_plan_set_tiles")

    def set_wave_grid(self, wave: int, tiles: bool) -> int:
        """Specialised units of ``wave``: persistent grid (False) or one block per tile (True)."""
        rc = int(self._lib.sgb_plan_set_wave_grid(self._handle, int(wave), int(bool(tiles))))
        if rc < 0:
            _check(rc, "sgb_plan_set_wave_grid")
        return rc

    def autotune(self, reps: int = 5, gain: float = 0.98):
        """Per wave, keep the fastest launch configuration of its specialised units: tile schedule
        instance- (``tiles``) or fraction-interleaved (``tiles_alt``, when lower_plan offers one) x
        grid persistent or one block per tile.  Each wave is timed alone with CUDA events in CSR
        mode, every candidate twice, min over ``reps`` launches; a candidate replaces the default
        (instance order, persistent) only when ``gain`` x faster.  Results never depend on it."""
        import torch

        from .lower import UNIT_JIT, UNIT_WINDOW

        lw = self.lowered
        base = np.ascontiguousarray(lw.tiles, np.int32).reshape(-1, 2)
        alt = (np.ascontiguousarray(lw.tiles_alt, np.int32).reshape(-1, 2)
               if getattr(lw, "tiles_alt", None) is not None else None)
        waves, ranges = set(), {}
        for u in range(len(lw.units)):
            r = lw.unit(u)
            t0, t1 = r["tile_begin"], r["tile_end"]
            if r["flags"] & UNIT_JIT and not r["flags"] & UNIT_WINDOW and t1 > t0:
                waves.add(r["wave"])
                if alt is not None and not np.array_equal(base[t0:t1], alt[t0:t1]):
                    ranges.setdefault(r["wave"], []).append((t0, t1))
        if not waves or not self.n_outputs:
            return
        rng = np.random.default_rng(0)
        x = self.new_values(rng.uniform(0.5, 2.0, self.input_count))
        out = torch.empty(self.n_outputs, dtype=torch.float64, device=x.device)
        self.run_csr(x, out)
        stream = torch.cuda.current_stream(x.device)
        evs = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(reps)]

        def time_wave(w):
            for e0, e1 in evs:
                e0.record(stream)
                self.run_wave(x, w, out, stream)
                e1.record(stream)
            torch.cuda.synchronize(x.device)
            return min(e0.elapsed_time(e1) for e0, e1 in evs)

        cands = [("inst", False), ("inst", True)] + ([("frac", False), ("frac", True)] if ranges else [])
        best = {w: {} for w in waves}
        for _ in range(2):
            for order, tiles in cands:
                self.set_tiles(alt if order == "frac" else base)
                for w in waves:
                    if order == "frac" and w not in ranges:
                        continue
                    self.set_wave_grid(w, tiles)
                    key = (order, tiles)
                    best[w][key] = min(best[w].get(key, np.inf), time_wave(w))
        final = base.copy()
        for w in sorted(waves):
            t_def = best[w][("inst", False)]
            key = min(best[w], key=best[w].get)
            if best[w][key] >= gain * t_def:
                key = ("inst", False)
            self.set_wave_grid(w, key[1])
            if key[0] == "frac":
                for t0, t1 in ranges[w]:
                    final[t0:t1] = alt[t0:t1]
            self.tile_order[w] = f"{key[0]}/{'tiles' if key[1] else 'persistent'}"
        self.tile_timings = {w: {f"{o}/{'tiles' if g else 'persistent'}": v for (o, g), v in d.items()}
                             for w, d in best.items()}
        self.set_tiles(final)
        self.tiles = final

    def close(self):
        if self._handle:
            self._lib.sgb_plan_destroy(self._handle)
            self._handle = ctypes.c_void_p(0)

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    # -- device-resident API (torch tensors, stream-ordered) ------------------------

    def _check_tensor(self, t, rows: int, name: str):
        import torch

        if not isinstance(t, torch.Tensor) or t.dtype != torch.float64 or not t.is_cuda:
            raise TypeError(f"{name} must be a float64 CUDA tensor")
        if t.device.index != self.device:
            raise ValueError(f"{name} lives on cuda:{t.device.index}, plan on cuda:{self.device}")
        if not t.is_contiguous() or t.shape[0] != rows:
            raise ValueError(f"{name} must be contiguous with {rows} rows, got {tuple(t.shape)}")

    def _check_workspace(self, x):
        """CSR-mode value arrays of a plan with a bulk-fed window unit must span value_slots doubles
        (the 16-byte bulk copies may read one padding slot; DevicePlan.new_values allocates it)."""
        if self.value_slots > self.value_array_size:
            span = x.untyped_storage().nbytes() // 8 - x.storage_offset()
            if span < self.value_slots:
                raise ValueError(f"x must span {self.value_slots} doubles (sgb_plan_value_slots), got {span}: "
                                 "allocate it with DevicePlan.new_values")

    def new_values(self, inputs=None):
        """Zeroed device value array with ``inputs`` placed at [0, input_count)."""
        import torch

        # a bulk-fed window unit may read one padding slot past the value array (sgb_plan_value_slots)
        x = torch.zeros(self.value_slots, dtype=torch.float64, device=f"cuda:{self.device}")[: self.value_array_size]
        if inputs is not None:
            x[: self.input_count] = torch.as_tensor(inputs, dtype=torch.float64).to(x.device)
        return x

    def run_values(self, x, stream=None):
        """sg_run on a device value array (in place)."""
        self._check_tensor(x, self.value_array_size, "x")
        _check(self._lib.sgb_run_values(self._handle, ctypes.c_void_p(x.data_ptr()),
                                        _stream_handle(stream)), "sgb_run_values")
        return x

    def run_csr(self, x, out=None, stream=None):
        """inputs (placed in x) -> CSR values in one pass; x is scratch for intermediates."""
        import torch

        self._check_tensor(x, self.value_array_size, "x")
        self._check_workspace(x)
        if out is None:
            out = torch.empty(self.n_outputs, dtype=torch.float64, device=x.device)
        self._check_tensor(out, self.n_outputs, "out")
        _check(self._lib.sgb_run_csr(self._handle, ctypes.c_void_p(x.data_ptr()), ctypes.c_void_p(out.data_ptr()),
                                     _stream_handle(stream)), "sgb_run_csr")
        return out

    def run_inputs_csr(self, inputs, out=None, stream=None):
        """Device inputs [input_count] -> CSR values [n_outputs] through the plan's own workspace
        (sgb_run_inputs_csr; no value array on the caller's side)."""
        import torch

        if not isinstance(inputs, torch.Tensor) or inputs.dtype != torch.float64 or not inputs.is_cuda \
                or not inputs.is_contiguous() or inputs.numel() != self.input_count:
            raise ValueError(f"inputs must be a contiguous float64 CUDA tensor of {self.input_count} values")
        if out is None:
            out = torch.empty(self.n_outputs, dtype=torch.float64, device=inputs.device)
        self._check_tensor(out, self.n_outputs, "out")
        _check(self._lib.sgb_run_inputs_csr(self._handle, ctypes.c_void_p(inputs.data_ptr()),
                                            ctypes.c_void_p(out.data_ptr()), _stream_handle(stream)),
               "sgb_run_inputs_csr")
        return out

    def capture_csr(self, x, out, batch: bool = False):
        """A CUDA graph of one CSR-mode evaluation on these buffers (``graph.replay()`` re-runs it).

        All launches of the evaluation -- every wave's units on the caller's stream and the
        forked aux streams, and the output gather -- are captured once, so a replay costs one
        graph launch instead of one launch per unit (launch-bound plans such as C1).
        """
        import torch

        g = torch.cuda.CUDAGraph()
        s = torch.cuda.Stream(device=x.device)
        rezero = self.lowered.needs_zero == 2  # reads precede writes: every evaluation starts from zeros

        def body():
            if rezero:
                x[self.input_count:].zero_()
            self.run_batch_csr(x, out) if batch else self.run_csr(x, out)

        s.wait_stream(torch.cuda.current_stream(x.device))
        with torch.cuda.stream(s):  # warm the launch path outside the capture
            body()
        torch.cuda.current_stream(x.device).wait_stream(s)
        with torch.cuda.graph(g):
            body()
        return g

    def run_wave(self, x, wave: int, out=None, stream=None):
        """One dependency wave (profiling / per-launch timing); ``out`` given = CSR mode."""
        if out is not None:
            self._check_workspace(x)
        _check(self._lib.sgb_run_wave(self._handle, ctypes.c_void_p(x.data_ptr()),
                                      ctypes.c_void_p(out.data_ptr() if out is not None else 0), int(wave),
                                      _stream_handle(stream)), "sgb_run_wave")
        return x

    def gather_outputs(self, x, out=None, stream=None):
        import torch

        self._check_tensor(x, self.value_array_size, "x")
        if out is None:
            out = torch.empty(self.n_outputs, dtype=torch.float64, device=x.device)
        self._check_tensor(out, self.n_outputs, "out")
        _check(self._lib.sgb_gather_outputs(self._handle, ctypes.c_void_p(x.data_ptr()),
                                            ctypes.c_void_p(out.data_ptr()), _stream_handle(stream)),
               "sgb_gather_outputs")
        return out

    def run_batch(self, X, stream=None):
        """B independent evaluations: X[value_array_size, B] (batch-fastest), in place."""
        self._check_tensor(X, self.value_array_size, "X")
        if X.dim() != 2:
            raise ValueError("X must be [value_array_size, batch]")
        _check(self._lib.sgb_run_batch(self._handle, ctypes.c_void_p(X.data_ptr()), X.stride(0),
                                       X.shape[1], _stream_handle(stream)), "sgb_run_batch")
        return X

    def run_batch_csr(self, X, out=None, stream=None):
        """Batched CSR mode: out[k, b] = value of output k in value set b (CSR-window plans: the members'
        value-mode twins store their outputs directly, only the copied outputs are gathered; otherwise
        batched values + one gather)."""
        import torch

        self._check_tensor(X, self.value_array_size, "X")
        if X.dim() != 2:
            raise ValueError("X must be [value_array_size, batch]")
        if out is None:
            out = torch.empty((self.n_outputs, X.shape[1]), dtype=torch.float64, device=X.device)
        if out.dim() != 2 or out.shape[1] < X.shape[1] or out.shape[0] != self.n_outputs or out.stride(1) != 1:
            raise ValueError("out must be [n_outputs, >= batch] with unit column stride")
        _check(self._lib.sgb_run_batch_csr(self._handle, ctypes.c_void_p(X.data_ptr()), X.stride(0), X.shape[1],
                                           ctypes.c_void_p(out.data_ptr()), out.stride(0), _stream_handle(stream)),
               "sgb_run_batch_csr")
        return out

    def run_batch_outputs_host(self, inputs, out):
        """Value sets through host buffers in chunks, pipelined: ``inputs`` a pinned float64 tensor
        (chunks, input_count, cb), ``out`` (chunks, n_outputs, cb).  Chunk c's inputs copy in on a
        copy stream while chunk c-1 evaluates (sgb_run_batch_csr, current stream) and chunk c-2's
        CSR values copy out on another; two device workspaces.  Synchronous."""
        import torch

        if inputs.dim() != 3 or inputs.shape[1] != self.input_count or inputs.dtype != torch.float64:
            raise ValueError(f"inputs must be float64 (chunks, {self.input_count}, cb)")
        n_chunks, _, cb = inputs.shape
        if tuple(out.shape) != (n_chunks, self.n_outputs, cb) or out.dtype != torch.float64:
            raise ValueError(f"out must be float64 ({n_chunks}, {self.n_outputs}, {cb})")
        dev = torch.device(f"cuda:{self.device}")
        comp = torch.cuda.current_stream(dev)
        h2d, d2h = torch.cuda.Stream(dev), torch.cuda.Stream(dev)
        nj = min(2, n_chunks)
        ws = getattr(self, "_batch_ws", None)
        if ws is None or ws[0] != cb or len(ws[1]) < nj:
            # kept across calls: CSR evaluations never write the slots a plan reads as zero
            X = [torch.zeros((self.value_array_size, cb), dtype=torch.float64, device=dev) for _ in range(nj)]
            O = [torch.empty((self.n_outputs, cb), dtype=torch.float64, device=dev) for _ in range(nj)]
            self._batch_ws = ws = (cb, X, O)
        X, O = ws[1], ws[2]
        ev_in, ev_run, ev_out = ([torch.cuda.Event() for _ in range(nj)] for _ in range(3))
        comp.synchronize()  # the workspaces are zeroed / free before the copy streams touch them
        rezero = int(self.lowered.needs_zero) == 2
        for c in range(n_chunks):
            j = c % nj
            if c >= nj:
                h2d.wait_event(ev_run[j])  # chunk c-2 has finished reading X[j]
            with torch.cuda.stream(h2d):
                X[j][: self.input_count].copy_(inputs[c], non_blocking=True)
            ev_in[j].record(h2d)
            comp.wait_event(ev_in[j])
            if c >= nj:
                comp.wait_event(ev_out[j])  # chunk c-2's CSR values are out of O[j]
            if rezero:
                X[j][self.input_count:].zero_()
            self.run_batch_csr(X[j], O[j], stream=comp)
            ev_run[j].record(comp)
            d2h.wait_event(ev_run[j])
            with torch.cuda.stream(d2h):
                out[c].copy_(O[j], non_blocking=True)
            ev_out[j].record(d2h)
        torch.cuda.synchronize(dev)
        return out

    def gather_outputs_batch(self, X, out=None, stream=None):
        import torch

        self._check_tensor(X, self.value_array_size, "X")
        if out is None:
            out = torch.empty((self.n_outputs, X.shape[1]), dtype=torch.float64, device=X.device)
        _check(self._lib.sgb_gather_outputs_batch(
            self._handle, ctypes.c_void_p(X.data_ptr()), X.stride(0), X.shape[1],
            ctypes.c_void_p(out.data_ptr()), out.stride(0), _stream_handle(stream)),
            "sgb_gather_outputs_batch")
        return out

    # -- host-buffer API (the reference's sg_run contract) ------------------------

    def sg_run(self, x_host: np.ndarray) -> np.ndarray:
        """Reference ABI: full host value array in, evaluated in place."""
        if x_host.dtype != np.float64 or not x_host.flags.c_contiguous or x_host.size != self.value_array_size:
            raise ValueError("x must be a contiguous float64 array of value_array_size")
        _check(self._lib.sgb_sg_run(self._handle, _ptr(x_host), ctypes.c_void_p(0), ctypes.c_void_p(0)),
               "sgb_sg_run")
        return x_host

    def run_outputs_host(self, inputs: np.ndarray, out: np.ndarray | None = None) -> np.ndarray:
        inputs = np.ascontiguousarray(inputs, dtype=np.float64)
        if inputs.shape != (self.input_count,):
            raise ValueError(f"plan expects {self.input_count} input values, got {inputs.size}")
        if out is None:
            out = np.empty(self.n_outputs, np.float64)
        _check(self._lib.sgb_run_outputs_host(self._handle, _ptr(inputs), _ptr(out)),
               "sgb_run_outputs_host")
        return out

    def run_outputs_host_many(self, inputs: np.ndarray, out: np.ndarray | None = None) -> np.ndarray:
        """A stream of value sets, host buffers in and out: ``inputs`` is (n_sets, input_count)
        (or (input_count,) for the same inputs every set), ``out`` (n_sets, n_outputs).  Copies
        in, evaluation and copies out of consecutive sets overlap (sgb_run_outputs_host_many);
        pass pinned arrays for the overlap."""
        if inputs.dtype != np.float64 or not inputs.flags.c_contiguous:
            inputs = np.ascontiguousarray(inputs, dtype=np.float64)
        if inputs.ndim == 1:
            if inputs.shape != (self.input_count,):
                raise ValueError(f"plan expects {self.input_count} input values, got {inputs.size}")
            if out is None:
                raise ValueError("out (n_sets, n_outputs) is required when one input set is repeated")
            in_stride = 0
        elif inputs.ndim == 2 and inputs.shape[1] == self.input_count:
            in_stride = self.input_count
        else:
            raise ValueError(f"inputs must be (n_sets, {self.input_count}), got {inputs.shape}")
        n_sets = out.shape[0] if out is not None else inputs.shape[0]
        if out is None:
            out = np.empty((n_sets, self.n_outputs), np.float64)
        if (out.dtype != np.float64 or not out.flags.c_contiguous or out.shape != (n_sets, self.n_outputs)
                or (in_stride and inputs.shape[0] != n_sets)):
            raise ValueError("out must be a contiguous float64 (n_sets, n_outputs) array matching inputs")
        _check(self._lib.sgb_run_outputs_host_many(self._handle, n_sets, _ptr(inputs), in_stride, _ptr(out),
                                                   self.n_outputs), "sgb_run_outputs_host_many")
        return out


# -- the reference-facing API -------------------------------------------------------


@dataclass
class InterpretResult:
    """codegen.py:365-370"""

    outputs: np.ndarray
    values: np.ndarray
    loads: list | None = None
    violations: list = field(default_factory=list)


def compile_plan(plan, work_dir=None, parallel: str = "none", device: int = 0):
    """GPU counterpart of ``compile_plan`` (emit.py:198-245).

    ``work_dir`` and ``parallel`` are accepted for signature compatibility
    (the device plan needs no source files and always runs every instance in
    parallel).  Returns ``run(inputs) -> full value array`` (host numpy).
    """
    if parallel not in ("none", "pragma"):
        raise ValueError(f"parallel must be 'none' or 'pragma', got {parallel!r}")
    dp = DevicePlan(plan, device=device)

    def run(inputs) -> np.ndarray:
        inputs = np.asarray(inputs, dtype=np.float64)
        if inputs.shape != (plan.input_count,):
            raise ValueError(f"plan expects {plan.input_count} input values, got {inputs.size}")
        x = np.zeros(plan.value_array_size, dtype=np.float64)
        x[: plan.input_count] = inputs
        return dp.sg_run(x)

    run.outputs = dp.run_outputs_host
    run.device_plan = dp
    run.library_path = LIB_PATH
    run.source_path = _PKG / "csrc" / "sgb.cu"
    return run


def interpret_plan(plan, inputs: Sequence[float], record_loads: bool = False,
                   check_schedule: bool = False, device: int = 0,
                   device_plan: DevicePlan | None = None) -> InterpretResult:
    """GPU counterpart of ``interpret_plan`` (codegen.py:404-446)."""
    if len(inputs) != plan.input_count:
        raise ValueError(f"plan expects {plan.input_count} input values, got {len(inputs)}")
    dp = device_plan or DevicePlan(plan, device=device)
    x = np.zeros(plan.value_array_size, dtype=np.float64)
    x[: plan.input_count] = np.asarray(inputs, dtype=np.float64)
    dp.sg_run(x)
    loads = [] if record_loads else None
    violations: list[str] = []
    if record_loads or check_schedule:
        # the address trace / write-before-read tracer are plan properties
        # (codegen.py:423-443); they do not depend on the evaluated values
        written = np.zeros(plan.value_array_size, dtype=bool)
        written[: plan.input_count] = True
        for kp in plan.kernels:
            cols = slot_addresses(plan, kp)
            if record_loads:
                for s, col in enumerate(cols):
                    loads.extend((kp.name, s, int(a)) for a in col)
            if check_schedule:
                for s, col in enumerate(cols):
                    bad = ~written[col]
                    if bad.any() and not kp.self_referencing:
                        violations.append(f"{kp.name}: slot {s} reads {int(bad.sum())} unwritten addresses")
                written[kp.dest_base: kp.dest_base + kp.n_roots * kp.instances] = True
    outputs = x[np.asarray(plan.outputs, dtype=np.int64)] if len(plan.outputs) else np.zeros(0)
    return InterpretResult(outputs=outputs, values=x, loads=loads, violations=violations)
