"""Public layer-level API: one LSRM sparse-attention layer (the four gated NSA
uses of a Stage-2 block, `lsrm/recon_pipeline.py:477-488`) on the GPU.

    inst  = build_instance("c3")                 # fixture geometry -> tokens, routing
    layer = SparseAttentionLayer(inst)
    outs  = layer.forward_host(x_hat, y_hat)     # NumPy in -> NumPy out (f32)

`forward_host` is the end-to-end path a reference user calls (host buffers,
H2D + permute/cast + fused layer + un-permute/cast + D2H).  The device path
(`engine.forward` on block-major bf16 tensors) is what `bench.py` times as
`value`; `time_host_path` is its `e2e`.
"""

from dataclasses import dataclass

import numpy as np
import torch

from . import _dev as D
from . import _ops
from .block_partition import BlockPartition, partition
from .block_routing import RoutingBudgets, build_routing_plan, volume_token_coords
from .engine import USES, USE_GEOM, SparseLayerEngine
from .tensor_core import AttentionParams
from .tokenizer import upsample_select_tokens
from .workloads import coarse_inputs, load_workload, nsa_use_weights, params_of


@dataclass
class Instance:
    name: str
    params: AttentionParams
    part_vol: BlockPartition
    part_img: BlockPartition
    plan_rows: dict
    weights: dict
    x_hat: np.ndarray     # [Nv, d] f32 LayerNorm'd volume tokens (token order)
    y_hat: np.ndarray     # [Ni, d] f32
    n_vol: int
    n_img: int


def build_instance(name: str = "c3", seed: int = 0, params: AttentionParams = None) -> Instance:
    """GPU instance setup: compaction -> partition -> 3D routing (all on the
    device, bit-exact with the reference), LN'd fine tokens as layer input.
    `params` overrides the workload's head geometry (e.g. paper heads on the
    C1 geometry, which the bf16 engine needs: head_dim 32/64)."""
    wl = load_workload(name)
    params = params or params_of(name)
    d = params.model_dim
    x_d, y_d, pe_v, pe_i = coarse_inputs(wl, d, seed)
    x_up, y_up = upsample_select_tokens(D.dev(x_d), D.dev(y_d), wl.vol_mask, wl.img_mask,
                                        pe_v, pe_i, wl.factor_vol, wl.factor_img)
    pv, pi = partition(x_up), partition(y_up)
    plan = build_routing_plan(volume_token_coords(x_up), wl.img_points, pv, pi, wl.cameras,
                              RoutingBudgets(), host_lists=False)
    ones = D.dev(np.ones(d, np.float32))
    zeros = D.dev(np.zeros(d, np.float32))
    xh = _ops.layer_norm(x_up.features, ones, zeros)
    yh = _ops.layer_norm(y_up.features, ones, zeros)
    return Instance(name, params, pv, pi, plan.device_rows, nsa_use_weights(params, seed),
                    D.host(xh), D.host(yh), x_up.count, y_up.count)


class SparseAttentionLayer:
    def __init__(self, inst: Instance):
        self.inst = inst
        self.engine = SparseLayerEngine(inst.part_vol, inst.part_img, inst.plan_rows,
                                        inst.weights, inst.params)
        self.tok = {"x": inst.part_vol.dev("block_token_ids"),
                    "y": inst.part_img.dev("block_token_ids")}
        d = inst.params.model_dim
        self._stage = {"x": D.empty((inst.n_vol, d), torch.float32),
                       "y": D.empty((inst.n_img, d), torch.float32)}
        self._out32 = {u: D.empty((self.engine.meta[USE_GEOM[u][0]].n, d), torch.float32)
                       for u in USES}
        self._bm = {"x": D.empty((inst.n_vol, d), torch.bfloat16),
                    "y": D.empty((inst.n_img, d), torch.bfloat16)}

    def device_inputs(self, x_hat, y_hat):
        """token-order f32 -> block-major bf16 (gather + cast kernels)."""
        out = []
        for s, a in (("x", x_hat), ("y", y_hat)):
            t = D.dev(a, torch.float32)
            g = _ops.gather_rows(t, self.tok[s])
            out.append(_ops.cast(g, torch.bfloat16))
        return out

    def _forward_from_stage(self):
        for s in ("x", "y"):
            bm32 = _ops.gather_rows(self._stage[s], self.tok[s])
            from ._native import call
            call("lsrm_cast", 1, bm32.data_ptr(), self._bm[s].data_ptr(), bm32.numel(),
                 D.stream())
        outs = self.engine.forward(self._bm["x"], self._bm["y"])
        res = {}
        from ._native import call
        for u in USES:
            qs = USE_GEOM[u][0]
            o32 = _ops.cast(outs[u], torch.float32)
            _ops.scatter_rows(o32, self.tok[qs], self._out32[u])
            res[u] = self._out32[u]
        return res

    def forward_host(self, x_hat: np.ndarray, y_hat: np.ndarray, pinned_out=None) -> dict:
        """NumPy in -> dict use -> NumPy [Nq, d] f32 (token order)."""
        self._stage["x"].copy_(torch.from_numpy(np.ascontiguousarray(x_hat, np.float32)),
                               non_blocking=True)
        self._stage["y"].copy_(torch.from_numpy(np.ascontiguousarray(y_hat, np.float32)),
                               non_blocking=True)
        res = self._forward_from_stage()
        outs = {}
        for u in USES:
            dst = pinned_out[u] if pinned_out is not None else torch.empty(
                tuple(res[u].shape), dtype=torch.float32, pin_memory=True)
            dst.copy_(res[u], non_blocking=True)
            outs[u] = dst
        torch.cuda.current_stream().synchronize()
        return {u: outs[u].numpy() for u in USES}

    def time_host_path(self, x_hat, y_hat, steps=5):
        """End-to-end throughput of the host API path over `steps` layer calls.

        Every step copies its f32 inputs from pinned host memory, runs the
        layer (permute/cast, four NSA uses, un-permute/cast) and copies the
        four f32 outputs back to pinned host memory. Steps are pipelined two
        deep: H2D, compute and D2H run on their own streams, with double-
        buffered device staging. Step k's D2H therefore overlaps step k+1's
        H2D and compute. Returns (mean ms per step from the first H2D to the
        last D2H, H2D bytes per step, D2H bytes per step)."""
        xp = torch.from_numpy(np.ascontiguousarray(x_hat, np.float32)).pin_memory()
        yp = torch.from_numpy(np.ascontiguousarray(y_hat, np.float32)).pin_memory()
        pipe = HostPipeline(self, n_slots=2)
        pipe.run(xp, yp, 2)          # warm-up (graph capture inside)
        torch.cuda.synchronize()
        ms = pipe.run(xp, yp, steps)
        h2d = xp.numel() * 4 + yp.numel() * 4
        d2h = sum(t.numel() * 4 for t in pipe.host_out[0].values())
        return ms, h2d, d2h

    def profile_breakdown(self, x_bm, y_bm, reps=5):
        """Device time per kernel class (events on the launching stream)."""
        e = self.engine
        st = torch.cuda.current_stream()
        names = ["project_gemm", "kv_prep", "attention", "wo_gemm"]
        acc = {n: 0.0 for n in names}
        per_use = {u: 0.0 for u in USES}
        for _ in range(reps):
            ev = [torch.cuda.Event(enable_timing=True) for _ in range(2)]
            ev[0].record(st)
            e.project(x_bm, y_bm)
            ev[1].record(st)
            torch.cuda.synchronize()
            acc["project_gemm"] += ev[0].elapsed_time(ev[1])
            ev = [torch.cuda.Event(enable_timing=True) for _ in range(2)]
            ev[0].record(st)
            e.prepare_kv()
            ev[1].record(st)
            torch.cuda.synchronize()
            acc["kv_prep"] += ev[0].elapsed_time(ev[1])
            # the layer's attention: one launch for all four uses (LPT queue)
            ev = [torch.cuda.Event(enable_timing=True) for _ in range(2)]
            ev[0].record(st)
            e.attend_all()
            ev[1].record(st)
            torch.cuda.synchronize()
            acc["attention"] += ev[0].elapsed_time(ev[1])
            ev = [torch.cuda.Event(enable_timing=True) for _ in range(2)]
            ev[0].record(st)
            e.output_all()         # the four W_o GEMMs: one grouped launch
            ev[1].record(st)
            torch.cuda.synchronize()
            acc["wo_gemm"] += ev[0].elapsed_time(ev[1])
            for u in USES:
                ev = [torch.cuda.Event(enable_timing=True) for _ in range(2)]
                ev[0].record(st)
                e.attend(u)        # informational: each use alone
                ev[1].record(st)
                torch.cuda.synchronize()
                per_use[u] += ev[0].elapsed_time(ev[1])
        out = {f"{n}_ms": v / reps for n, v in acc.items()}
        out["attention_per_use_ms"] = {u: v / reps for u, v in per_use.items()}
        out["attention_per_use_note"] = "each use launched alone; the layer runs one merged launch"
        return out


class HostPipeline:
    """Two-deep pipeline of host-API layer calls (H2D | compute | D2H streams).

    Slot s owns device staging (f32 inputs, f32 outputs) and pinned host
    outputs. Its compute is one CUDA graph: gather/cast to block-major bf16,
    the engine's four NSA uses, cast/scatter back to token order. Engine
    buffers are shared, because compute is serialised on one stream."""

    def __init__(self, layer: SparseAttentionLayer, n_slots: int = 2):
        self.layer, self.n = layer, n_slots
        inst, eng = layer.inst, layer.engine
        d = inst.params.model_dim
        self.stage = [{"x": D.empty((inst.n_vol, d), torch.float32),
                       "y": D.empty((inst.n_img, d), torch.float32)} for _ in range(n_slots)]
        self.dev_out = [{u: D.empty((eng.meta[USE_GEOM[u][0]].n, d), torch.float32) for u in USES}
                        for _ in range(n_slots)]
        self.host_out = [{u: torch.empty(tuple(t.shape), dtype=torch.float32, pin_memory=True)
                          for u, t in slot.items()} for slot in self.dev_out]
        self.s_in, self.s_comp, self.s_out = (torch.cuda.Stream() for _ in range(3))
        self.graphs = None

    def _compute(self, slot: int):
        lay, eng = self.layer, self.layer.engine
        from ._native import call
        for s in ("x", "y"):
            bm32 = _ops.gather_rows(self.stage[slot][s], lay.tok[s])
            call("lsrm_cast", 1, bm32.data_ptr(), lay._bm[s].data_ptr(), bm32.numel(), D.stream())
        outs = eng.forward(lay._bm["x"], lay._bm["y"])
        for u in USES:
            o32 = _ops.cast(outs[u], torch.float32)
            _ops.scatter_rows(o32, lay.tok[USE_GEOM[u][0]], self.dev_out[slot][u])

    def _capture(self):
        self.graphs = []
        with torch.cuda.stream(self.s_comp):
            for slot in range(self.n):          # warm-up outside capture
                self._compute(slot)
        torch.cuda.synchronize()
        for slot in range(self.n):
            g = torch.cuda.CUDAGraph()
            with torch.cuda.graph(g, stream=self.s_comp):
                self._compute(slot)
            self.graphs.append(g)
        torch.cuda.synchronize()

    def run(self, xp: torch.Tensor, yp: torch.Tensor, steps: int) -> float:
        if self.graphs is None:
            self._capture()
        ev = lambda: torch.cuda.Event(enable_timing=False)   # noqa: E731
        consumed = [None] * self.n     # compute finished with the slot's staging
        drained = [None] * self.n      # D2H finished with the slot's outputs
        t0, t1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        t0.record(self.s_in)
        for k in range(steps):
            s = k % self.n
            with torch.cuda.stream(self.s_in):
                if consumed[s] is not None:
                    self.s_in.wait_event(consumed[s])
                self.stage[s]["x"].copy_(xp, non_blocking=True)
                self.stage[s]["y"].copy_(yp, non_blocking=True)
                e_in = ev()
                e_in.record(self.s_in)
            with torch.cuda.stream(self.s_comp):   # replay() launches on the current stream
                self.s_comp.wait_event(e_in)
                if drained[s] is not None:
                    self.s_comp.wait_event(drained[s])
                self.graphs[s].replay()
                e_c = ev()
                e_c.record(self.s_comp)
            consumed[s] = e_c
            with torch.cuda.stream(self.s_out):
                self.s_out.wait_event(e_c)
                for u in USES:
                    self.host_out[s][u].copy_(self.dev_out[s][u], non_blocking=True)
                e_o = ev()
                e_o.record(self.s_out)
                drained[s] = e_o
        t1.record(self.s_out)
        torch.cuda.synchronize()
        return t0.elapsed_time(t1) / steps
