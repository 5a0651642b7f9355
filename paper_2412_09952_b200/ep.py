"""Expert parallelism for the E8T2 layer: one process per GPU, E/R experts per
rank (reference ownership rule moefold/upcycle.py:207-208, byte
model moefold/plan.py:246-247).  Two transports:

* "p2p" (default, `_EPPeerFunction`): the exchange is fused into the kernels
  over NVLink peer memory (torch symmetric memory, device barriers): the
  permute and combine-backward kernels store rows straight into the expert
  owners' planes, and the owners' FWD2 / BWD1 epilogues TMA-store their
  output tiles straight into the source ranks' planes, so combine and the
  router backward read locally.  Counts never leave the device; no host
  synchronisation.
* "nccl" (`_EPFunction`, the comparison baseline): separate kernels around
  NCCL all_to_all_single with exact splits (one host round trip for the
  counts), per rank r (T_local tokens, rank-local capacity, so routing equals
  the single-GPU oracle on that rank's batch):

  forward   K1 router -> K1b dispatch (compact layout) -> K2 permute into the
            send buffer -> all_to_all(counts) -> all_to_all(rows, exact
            splits) -> grouped GEMMs over R * E_local received segments
            -> all_to_all back -> K5 combine
  backward  K6 combine' -> all_to_all(dO) -> BWD2 / WGRAD / BWD1 over the
            received segments -> all_to_all(dxp) back -> router' ->
            all_reduce(dW_g, dW_noise)  (the router is replicated)

The fixed-capacity data-movement plan (`EPPlan`, used by the p2p receive
buffers) is plain torch and is exercised on CPU with the gloo backend in
tests/test_ep_gloo.py; the compute runs only in the CUDA library.
"""

from __future__ import annotations

from dataclasses import dataclass

import os

import torch
import torch.distributed as dist

from . import _lib
from .errors import ConfigError, ShapeError
from .moe import (DeviceRoutingStats, GateConfig, SEG_PAD, _acc_targets, _arange_i32, _dispatch_ws, _ep, _noise,
                  _router_ws, _swizzled, _wgrad_call, _wgrad_outputs, _wgrad_tickets, expert_capacity)


_TOKENS_CHECKED: set = set()   # (group id, T_local) pairs every rank agreed on (ExpertParallelMoE._check_tokens)
_INDEX_CACHE: dict = {}   # EPPlan key -> {(kind, device): index tensors}; read-only after creation


@dataclass
class EPPlan:
    """Static layout of one EP step (identical on every rank)."""

    world: int
    rank: int
    n_experts: int
    tokens: int          # T_local
    capacity: int | None
    cap_pad: int         # rows per (rank, expert) segment, multiple of 128

    @classmethod
    def make(cls, world: int, rank: int, n_experts: int, tokens: int, capacity_factor: float | None) -> "EPPlan":
        if n_experts % world != 0:
            raise ConfigError(f"n_experts ({n_experts}) not divisible by ep={world}")
        cap = expert_capacity(tokens, n_experts, capacity_factor)
        c = tokens if cap is None else min(cap, tokens)
        cap_pad = max(SEG_PAD, (c + SEG_PAD - 1) // SEG_PAD * SEG_PAD)
        return cls(world, rank, n_experts, tokens, cap, cap_pad)

    @property
    def e_local(self) -> int:
        return self.n_experts // self.world

    @property
    def owned(self) -> range:
        return range(self.rank * self.e_local, (self.rank + 1) * self.e_local)

    @property
    def send_rows(self) -> int:
        return self.n_experts * self.cap_pad

    def recv_segments(self, device):
        """(base, expert) of the R * E_local received segments: segment
        (src, el) starts at (src * E_local + el) * cap_pad.  Built once per
        (plan, device) and cached (no per-step index kernels)."""
        key = ("recv", device)
        if key not in _INDEX_CACHE.setdefault(self._key(), {}):
            n = self.world * self.e_local
            base = torch.arange(n, dtype=torch.int32, device=device) * self.cap_pad
            expert = torch.arange(n, dtype=torch.int32, device=device) % self.e_local
            _INDEX_CACHE[self._key()][key] = (base, expert)
        return _INDEX_CACHE[self._key()][key]

    def peer_seg_base(self, device) -> torch.Tensor:
        """[E] row of (this rank, expert e) inside expert e's owner receive buffer:
        (rank * E_local + e % E_local) * cap_pad (cached like recv_segments)."""
        key = ("peer", device)
        if key not in _INDEX_CACHE.setdefault(self._key(), {}):
            e = torch.arange(self.n_experts, dtype=torch.int32, device=device)
            _INDEX_CACHE[self._key()][key] = ((self.rank * self.e_local + e % self.e_local) *
                                              self.cap_pad).to(torch.int32)
        return _INDEX_CACHE[self._key()][key]

    def _key(self):
        return (self.world, self.rank, self.n_experts, self.cap_pad)

    def exchange_counts(self, counts: torch.Tensor, group=None) -> torch.Tensor:
        """counts[E] (tokens this rank sends to each expert) -> recv[R * E_local]
        (tokens each source rank sends to each of my experts)."""
        recv = torch.empty(self.world * self.e_local, dtype=counts.dtype, device=counts.device)
        dist.all_to_all_single(recv, counts.contiguous(), group=group)
        return recv

    def exchange_rows(self, out: torch.Tensor, inp: torch.Tensor, group=None) -> torch.Tensor:
        """Equal-split all-to-all of [E * cap_pad, D] row blocks (expert-major)."""
        dist.all_to_all_single(out, inp, group=group)
        return out


class _Splits:
    """Exact all-to-all splits of the NCCL transport.  Send side: the compact
    dispatch layout (segments padded to 128 rows, experts in order), so the
    rows for destination d are the padded segments of d's experts, contiguous.
    Receive side: source-major, local-expert-minor padded segments.  Only kept
    rows (+ <128 pad rows per segment) cross the wire, also when dropless."""

    def __init__(self, counts, rcounts, plan: "EPPlan", device):
        El = plan.e_local
        ch = torch.stack([counts, rcounts]) if counts.numel() == rcounts.numel() else None
        if ch is not None:
            c_h, r_h = ch.cpu().tolist()
        else:
            c_h, r_h = counts.cpu().tolist(), rcounts.cpu().tolist()
        pad = lambda c: (c + SEG_PAD - 1) // SEG_PAD * SEG_PAD  # noqa: E731
        self.send = [sum(pad(c_h[d * El + el]) for el in range(El)) for d in range(plan.world)]
        self.recv = [sum(pad(r_h[src * El + el]) for el in range(El)) for src in range(plan.world)]
        self.rows_send, self.rows_recv = sum(self.send), sum(self.recv)
        base, acc = [], 0
        for c in r_h:
            base.append(acc)
            acc += pad(c)
        self.rbase = torch.tensor(base, dtype=torch.int32, device=device)
        self.rexp = torch.arange(plan.world * El, dtype=torch.int32, device=device) % El

    def to_owners(self, rows_send: torch.Tensor, H: int, group) -> torch.Tensor:
        out = torch.empty(max(self.rows_recv, 1), H, dtype=rows_send.dtype, device=rows_send.device)
        dist.all_to_all_single(out[:self.rows_recv], rows_send[:self.rows_send], output_split_sizes=self.recv,
                               input_split_sizes=self.send, group=group)
        return out

    def to_sources(self, rows_recv: torch.Tensor, H: int, group) -> torch.Tensor:
        out = torch.empty(max(self.rows_send, 1), H, dtype=rows_recv.dtype, device=rows_recv.device)
        dist.all_to_all_single(out[:self.rows_send], rows_recv[:self.rows_recv], output_split_sizes=self.send,
                               input_split_sizes=self.recv, group=group)
        return out


class _EPFunction(torch.autograd.Function):
    @staticmethod
    def forward(ctx, x, w_g, w_noise, W1, W2, W3, z, st):
        cfg, plan, group = st["cfg"], st["plan"], st["group"]
        T, H = x.shape
        E = w_g.shape[1]
        El = plan.e_local
        F = W1.shape[1]
        dev = x.device
        s = _lib.stream_ptr()
        f32 = dict(dtype=torch.float32, device=dev)
        bf = dict(dtype=torch.bfloat16, device=dev)
        rt = _lib.ROUTER[cfg.router_type]

        logits = torch.empty(T, E, **f32)
        gates = torch.empty(T, E, **f32)
        probs = torch.empty(T, E, **f32) if cfg.router_type == "st" else None
        noise_act = torch.empty(T, E, **f32) if z is not None else None
        err = None          # gate errors reach the host through the dispatch stats (stats[2])
        ws = _router_ws(H, E, dev)      # left holding the swizzled W_g / W_noise (reused below)
        ctx.router_ws = ws
        _lib.call("b200moe_router_fwd", x.data_ptr(), w_g.data_ptr(), w_noise.data_ptr(), _lib.ptr(z), T, H, E,
                  cfg.top_k, rt, logits.data_ptr(), gates.data_ptr(), _lib.ptr(probs), _lib.ptr(noise_act),
                  ws.data_ptr(), None, s)
        slot_rank = torch.empty(T, E, dtype=torch.int32, device=dev)
        counts = torch.empty(E, dtype=torch.int32, device=dev)
        seg_base = torch.empty(E, dtype=torch.int32, device=dev)
        gate_mass = torch.empty(E, **f32)
        imp = torch.empty(E, **f32)
        imp_loss = torch.empty(1, **f32)
        stats = torch.empty(3, dtype=torch.int64, device=dev)
        _lib.call("b200moe_dispatch", gates.data_ptr(), T, E, -1 if plan.capacity is None else plan.capacity,
                  _lib.POLICY[cfg.drop_policy], _lib.LAYOUT_COMPACT, 0, slot_rank.data_ptr(),
                  counts.data_ptr(), seg_base.data_ptr(), gate_mass.data_ptr(), imp.data_ptr(), stats.data_ptr(),
                  imp_loss.data_ptr(), None, _dispatch_ws(dev, T).data_ptr(), s)
        # exact splits: the compact layout keeps each destination's experts
        # contiguous; one host round trip fetches both count vectors
        rcounts = plan.exchange_counts(counts, group)
        sp = _Splits(counts, rcounts, plan, dev)
        xs = torch.empty(max(sp.rows_send, 1), H, **bf)
        _lib.call("b200moe_permute", x.data_ptr(), slot_rank.data_ptr(), seg_base.data_ptr(), counts.data_ptr(), T,
                  H, E, xs.data_ptr(), s)
        xr = sp.to_owners(xs, H, group)
        Rs = max(sp.rows_recv, 1)
        rbase, rexp = sp.rbase, sp.rexp
        nseg = plan.world * El
        A = torch.empty(Rs, F, **bf)
        B = torch.empty(Rs, F, **bf)
        Hh = torch.empty(Rs, F, **bf)
        _lib.call("b200moe_expert_fwd1", xr.data_ptr(), W1.data_ptr(), W3.data_ptr(), rbase.data_ptr(),
                  rcounts.data_ptr(), rexp.data_ptr(), nseg, Rs, H, F, El, A.data_ptr(), B.data_ptr(), Hh.data_ptr(), s)
        Or = torch.empty(Rs, H, **bf)
        _lib.call("b200moe_expert_fwd2", Hh.data_ptr(), W2.data_ptr(), rbase.data_ptr(), rcounts.data_ptr(),
                  rexp.data_ptr(), nseg, Rs, H, F, El, Or.data_ptr(), s)
        Os = sp.to_sources(Or, H, group)
        y = torch.empty(T, H, **bf)
        _lib.call("b200moe_combine", Os.data_ptr(), gates.data_ptr(), slot_rank.data_ptr(), seg_base.data_ptr(), T,
                  H, E, y.data_ptr(), s)
        st["routing"] = dict(logits=logits, slot_rank=slot_rank, counts=counts, seg_base=seg_base,
                             gate_mass=gate_mass, importance=imp, importance_loss=imp_loss, stats=stats, err=err,
                             recv_counts=rcounts)
        ctx.st = st
        ctx.acc_targets = _acc_targets(W1, W2, W3)
        ctx.splits = sp
        ctx.save_for_backward(x, w_g, w_noise, W1, W2, W3, z, gates, probs, noise_act, slot_rank, counts, seg_base,
                              rcounts, xr, A, B, Hh, Os)
        return y, gates

    @staticmethod
    def backward(ctx, dy, dgates):
        (x, w_g, w_noise, W1, W2, W3, z, gates, probs, noise_act, slot_rank, counts, seg_base, rcounts, xr, A, B,
         Hh, Os) = ctx.saved_tensors
        st = ctx.st
        cfg, plan, group = st["cfg"], st["plan"], st["group"]
        T, H = x.shape
        E = w_g.shape[1]
        El = plan.e_local
        F = W1.shape[1]
        sp = ctx.splits
        Rs = max(sp.rows_recv, 1)
        dev = x.device
        s = _lib.stream_ptr()
        f32 = dict(dtype=torch.float32, device=dev)
        bf = dict(dtype=torch.bfloat16, device=dev)
        nseg = plan.world * El
        rbase, rexp = sp.rbase, sp.rexp

        dy = (torch.zeros(T, H, **bf) if dy is None else dy).to(torch.bfloat16).contiguous()
        dOs = torch.empty(max(sp.rows_send, 1), H, **bf)
        dg = torch.empty(T, E, **f32)
        _lib.call("b200moe_combine_bwd", dy.data_ptr(), Os.data_ptr(), gates.data_ptr(), slot_rank.data_ptr(),
                  seg_base.data_ptr(), counts.data_ptr(), T, H, E, dOs.data_ptr(), dg.data_ptr(), s)
        dOr = sp.to_owners(dOs, H, group)
        dA = torch.empty(Rs, F, **bf)
        dB = torch.empty(Rs, F, **bf)
        _lib.call("b200moe_expert_bwd2", dOr.data_ptr(), W2.data_ptr(), A.data_ptr(), B.data_ptr(), rbase.data_ptr(),
                  rcounts.data_ptr(), rexp.data_ptr(), nseg, Rs, H, F, El, dA.data_ptr(), dB.data_ptr(), s)
        dW1, dW2, dW3, acc = _wgrad_outputs(ctx.acc_targets, W1, W2, W3)
        _wgrad_call(acc, xr.data_ptr(), Hh.data_ptr(), dOr.data_ptr(), dA.data_ptr(),
                  dB.data_ptr(), rbase.data_ptr(), rcounts.data_ptr(), rexp.data_ptr(), nseg, Rs, H, F, El,
                  dW1.data_ptr(), dW2.data_ptr(), dW3.data_ptr(), s)
        if acc:
            dW1 = dW2 = dW3 = None
        dxr = torch.empty(Rs, H, **bf)
        _lib.call("b200moe_expert_bwd1", dA.data_ptr(), dB.data_ptr(), W1.data_ptr(), W3.data_ptr(), rbase.data_ptr(),
                  rcounts.data_ptr(), rexp.data_ptr(), nseg, Rs, H, F, El, dxr.data_ptr(), s)
        dxs = sp.to_sources(dxr, H, group)
        dx = torch.empty(T, H, **bf)
        dh = torch.empty(T, E, **f32)
        dn = torch.empty(T, E, **f32) if z is not None else None
        dgx, sx_t, sx_e = None, 0, 0
        if dgates is not None:
            dgx = dgates.to(torch.float32)
            sx_t, sx_e = dgx.stride()
        ws = torch.empty(2 * H * _ep(E) + T * _ep(E), **f32)
        _lib.call("b200moe_router_bwd", dxs.data_ptr(), slot_rank.data_ptr(), seg_base.data_ptr(), dg.data_ptr(),
                  _lib.ptr(dgx), sx_t, sx_e, gates.data_ptr(), _lib.ptr(probs), w_g.data_ptr(), w_noise.data_ptr(),
                  _lib.ptr(z), _lib.ptr(noise_act), *_swizzled(ctx, H, E, z), T, H, E, cfg.top_k,
                  _lib.ROUTER[cfg.router_type],
                  dx.data_ptr(), dh.data_ptr(), _lib.ptr(dn), ws.data_ptr(), s)
        dwg = torch.empty(H, E, **f32)
        dwn = torch.empty(H, E, **f32) if z is not None else None
        wsw = torch.empty((T + 63) // 64 * H * E, **f32)
        _lib.call("b200moe_router_wgrad", x.data_ptr(), dh.data_ptr(), _lib.ptr(dn), T, H, E, dwg.data_ptr(),
                  _lib.ptr(dwn), wsw.data_ptr(), _wgrad_tickets(dev, H).data_ptr(), s)
        if st.get("reduce_router", True):
            dist.all_reduce(dwg, group=group)
            if dwn is not None:
                dist.all_reduce(dwn, group=group)
        return dx, dwg, dwn, dW1, dW2, dW3, None, None


class _PeerBuffers:
    """Symmetric-memory receive buffers of the p2p transport.  A *forward*
    set per (buffer slot, receive rows, hidden, group) holds xr (tokens in,
    [R*E_local*cap_pad, H] bf16) plus the int32 receive-count table; xr is
    saved for the layer's backward (WGRAD's operand, and the recompute FWD1's
    input), so every layer alive in one autograd graph needs its own slot (the
    model forward uses the layer index).  The *shared* set (slot -1) holds two
    planes that are live only transiently: O (expert outputs: written by FWD2,
    read by the peers' combine right after, never in the backward, which uses
    the combine's local row mirror `og`) and dO / dxp (inside one layer's
    backward).  Every user of a shared plane is preceded by a device barrier
    of all ranks, so one set serves every layer's forward and backward.  Peers
    address the planes through device arrays of per-rank base pointers; canary
    bands surround every plane."""

    _cache: dict = {}
    GUARD = 4096          # canary bytes before, between and after the planes
    CANARY = 0xA5

    @classmethod
    def get(cls, rows: int, H: int, n_counts: int, group, device, slot: int = 0):
        grp = group if group is not None else dist.group.WORLD
        key = (slot, rows, H, n_counts, grp.group_name, device.index)
        b = cls._cache.get(key)
        if b is None:
            b = cls(rows, H, n_counts, grp, device)
            cls._cache[key] = b
        return b

    @classmethod
    def backward_set(cls, rows: int, H: int, group, device):
        """The shared set (O in the forward, dO / dxp in the backward)."""
        return cls.get(rows, H, 0, group, device, slot=-1)

    def __init__(self, rows, H, n_counts, grp, device):
        import torch.distributed._symmetric_memory as symm
        self.generation = 0   # bumped by every forward that (re)fills xr
        G = self.GUARD
        plane = rows * H * 2
        nplanes = 1 if n_counts else 2      # forward set: xr;  shared set: O / dO and dxp
        offs = [G + i * (plane + G) for i in range(nplanes)]
        cnt_off = offs[-1] + plane + G
        cnt_bytes = ((n_counts * 4 + 255) // 256) * 256
        total = cnt_off + cnt_bytes + G
        self.raw = symm.empty(total, dtype=torch.uint8, device=device)
        self.raw.fill_(self.CANARY)
        self.handle = symm.rendezvous(self.raw, grp.group_name)
        self.views = [self.raw[o:o + plane].view(torch.bfloat16).view(rows, H) for o in offs]
        self.counts = self.raw[cnt_off:cnt_off + n_counts * 4].view(torch.int32)
        self._guards = [(0, G)] + [(o + plane, G) for o in offs] + [(cnt_off + cnt_bytes, G)]
        ptrs = list(self.handle.buffer_ptrs)
        mk = lambda off: torch.tensor([p + off for p in ptrs], dtype=torch.int64, device=device)  # noqa: E731
        self.peer = [mk(o) for o in offs]   # the planes' base pointers on every rank (device arrays)
        self.peer_host = [[p + o for p in ptrs] for o in offs]   # the same, host lists (GEMM store maps)
        me = self.raw.data_ptr()
        # this rank's own plane base repeated per rank: the peer kernels' row addressing with every
        # "owner" local (consumers of rows the owners' GEMMs pushed here)
        self.local_rep = [torch.tensor([me + o] * len(ptrs), dtype=torch.int64, device=device) for o in offs]
        self.peer_counts = mk(cnt_off)

    def guards_intact(self) -> bool:
        """True if no kernel (local or a peer's, over NVLink) wrote into the
        canary bands around this rank's planes (checked by tools/ep_check.py)."""
        return all(bool((self.raw[o:o + n] == self.CANARY).all()) for o, n in self._guards)

    def barrier(self):
        self.handle.barrier(channel=0)

    # forward set: plane 0 = xr;  shared set: plane 0 = O (forward) / dO (backward), plane 1 = dxp
    @property
    def xr(self):
        return self.views[0]

    @property
    def o(self):
        return self.views[0]

    @property
    def do(self):
        return self.views[0]

    @property
    def dxp(self):
        return self.views[1]


class _EPPeerFunction(torch.autograd.Function):
    """Expert parallelism with the dispatch / combine exchange fused into the
    permute / combine kernels over NVLink peer memory (no NCCL all-to-all)."""

    @staticmethod
    def forward(ctx, x, w_g, w_noise, W1, W2, W3, z, st):
        cfg, plan, group = st["cfg"], st["plan"], st["group"]
        T, H = x.shape
        E = w_g.shape[1]
        El = plan.e_local
        F = W1.shape[1]
        dev = x.device
        s = _lib.stream_ptr()
        f32 = dict(dtype=torch.float32, device=dev)
        bf = dict(dtype=torch.bfloat16, device=dev)
        rt = _lib.ROUTER[cfg.router_type]
        Rs = plan.send_rows
        pb = _PeerBuffers.get(Rs, H, plan.world * El, group, dev, st.get("buffer_slot", 0))
        pbs = _PeerBuffers.backward_set(Rs, H, group, dev)   # O lives in the shared set's first plane

        logits = torch.empty(T, E, **f32)
        gates = torch.empty(T, E, **f32)
        probs = torch.empty(T, E, **f32) if cfg.router_type == "st" else None
        noise_act = torch.empty(T, E, **f32) if z is not None else None
        err = None          # gate errors reach the host through the dispatch stats (stats[2])
        ws = _router_ws(H, E, dev)      # left holding the swizzled W_g / W_noise (reused below)
        ctx.router_ws = ws
        _lib.call("b200moe_router_fwd", x.data_ptr(), w_g.data_ptr(), w_noise.data_ptr(), _lib.ptr(z), T, H, E,
                  cfg.top_k, rt, logits.data_ptr(), gates.data_ptr(), _lib.ptr(probs), _lib.ptr(noise_act),
                  ws.data_ptr(), None, s)
        slot_rank = torch.empty(T, E, dtype=torch.int32, device=dev)
        counts = torch.empty(E, dtype=torch.int32, device=dev)
        seg_local = torch.empty(E, dtype=torch.int32, device=dev)
        gate_mass = torch.empty(E, **f32)
        imp = torch.empty(E, **f32)
        imp_loss = torch.empty(1, **f32)
        stats = torch.empty(3, dtype=torch.int64, device=dev)
        _lib.call("b200moe_dispatch", gates.data_ptr(), T, E, -1 if plan.capacity is None else plan.capacity,
                  _lib.POLICY[cfg.drop_policy], _lib.LAYOUT_FIXED, plan.cap_pad, slot_rank.data_ptr(),
                  counts.data_ptr(), seg_local.data_ptr(), gate_mass.data_ptr(), imp.data_ptr(), stats.data_ptr(),
                  imp_loss.data_ptr(), None, _dispatch_ws(dev, T).data_ptr(), s)
        seg_peer = plan.peer_seg_base(dev)      # row of (this rank, expert e) in e's owner buffer
        pb.barrier()                            # every rank is done with the previous use of the buffers
        pb.generation += 1
        _lib.call("b200moe_permute_peer", x.data_ptr(), slot_rank.data_ptr(), seg_peer.data_ptr(),
                  counts.data_ptr(), T, H, E, El, plan.rank, pb.peer[0].data_ptr(), pb.peer_counts.data_ptr(), s)
        pb.barrier()                            # all tokens and counts have landed
        rbase, rexp = plan.recv_segments(dev)
        nseg = plan.world * El
        rcounts = pb.counts
        A = torch.empty(Rs, F, **bf)
        B = torch.empty(Rs, F, **bf)
        Hh = torch.empty(Rs, F, **bf)
        _lib.call("b200moe_expert_fwd1", pb.xr.data_ptr(), W1.data_ptr(), W3.data_ptr(), rbase.data_ptr(),
                  rcounts.data_ptr(), rexp.data_ptr(), nseg, Rs, H, F, El, A.data_ptr(), B.data_ptr(), Hh.data_ptr(), s)
        push = st.get("gemm_push", True)
        if push:
            # FWD2 pushes every output tile straight into its source rank's receive plane
            # (the shared set's first plane, expert-major: the source's own dispatch layout)
            arr, dst = _lib.host_u64(pbs.peer_host[0])
            _lib.call("b200moe_expert_fwd2_peer", Hh.data_ptr(), W2.data_ptr(), rbase.data_ptr(), rcounts.data_ptr(),
                      rexp.data_ptr(), nseg, Rs, H, F, El, dst, plan.world, plan.rank, plan.cap_pad, Rs, s)
        else:
            _lib.call("b200moe_expert_fwd2", Hh.data_ptr(), W2.data_ptr(), rbase.data_ptr(), rcounts.data_ptr(),
                      rexp.data_ptr(), nseg, Rs, H, F, El, pbs.o.data_ptr(), s)
        if st.get("recompute"):
            # selective recompute: a, b, h ([rows, F] x 3, the layer's largest
            # activations) are dropped here and rebuilt by one FWD1 launch at the
            # start of the backward from xr (kept in the forward set anyway)
            A = B = Hh = None
        elif st.get("drop_h"):
            # keep a, b only: BWD2 rebuilds h = silu(a) * b for WGRAD (b200moe_expert_bwd2_h)
            Hh = None
        pb.barrier()                            # all expert outputs are ready (pushed: landed here)
        y = torch.empty(T, H, **bf)
        # the gathered expert rows are kept for the backward (read locally there
        # instead of over NVLink again; O's plane is reused by the next layer)
        og = torch.empty(T * cfg.top_k, H, **bf)
        if push:   # this rank's tokens' expert rows are local now, at seg_local[e] + slot
            _lib.call("b200moe_combine_peer", pbs.local_rep[0].data_ptr(), El, gates.data_ptr(),
                      slot_rank.data_ptr(), seg_local.data_ptr(), T, H, E, y.data_ptr(), _lib.ptr(og), cfg.top_k, s)
        else:
            _lib.call("b200moe_combine_peer", pbs.peer[0].data_ptr(), El, gates.data_ptr(), slot_rank.data_ptr(),
                      seg_peer.data_ptr(), T, H, E, y.data_ptr(), _lib.ptr(og), cfg.top_k, s)
        ctx.og = og
        st["routing"] = dict(logits=logits, slot_rank=slot_rank, counts=counts, seg_base=seg_peer,
                             gate_mass=gate_mass, importance=imp, importance_loss=imp_loss, stats=stats, err=err,
                             recv_counts=rcounts.clone())
        ctx.st = st
        ctx.acc_targets = _acc_targets(W1, W2, W3)
        ctx.pb = pb
        ctx.generation = pb.generation
        ctx.recompute = A is None
        ctx.rebuild_h = A is not None and Hh is None
        ctx.push = push
        ctx.save_for_backward(x, w_g, w_noise, W1, W2, W3, z, gates, probs, noise_act, slot_rank, counts, seg_peer,
                              A, B, Hh, seg_local)
        return y, gates

    @staticmethod
    def backward(ctx, dy, dgates):
        (x, w_g, w_noise, W1, W2, W3, z, gates, probs, noise_act, slot_rank, counts, seg_peer, A, B,
         Hh, seg_local) = ctx.saved_tensors
        st, pb = ctx.st, ctx.pb
        if pb.generation != ctx.generation:
            # another forward on the same buffer slot overwrote the saved xr
            raise RuntimeError(f"EP symmetric buffer slot {st.get('buffer_slot', 0)} was refilled by a later forward "
                               f"before this backward; give layers that are alive in one graph distinct buffer_slot "
                               f"values")
        cfg, plan, group = st["cfg"], st["plan"], st["group"]
        T, H = x.shape
        E = w_g.shape[1]
        El = plan.e_local
        F = W1.shape[1]
        Rs = plan.send_rows
        dev = x.device
        s = _lib.stream_ptr()
        f32 = dict(dtype=torch.float32, device=dev)
        bf = dict(dtype=torch.bfloat16, device=dev)
        nseg = plan.world * El
        rbase, rexp = plan.recv_segments(dev)
        rcounts = pb.counts
        pbb = _PeerBuffers.backward_set(Rs, H, group, dev)   # dO, dxp: shared by every layer's backward
        if ctx.recompute:
            A, B, Hh = (torch.empty(Rs, F, **bf) for _ in range(3))
            _lib.call("b200moe_expert_fwd1", pb.xr.data_ptr(), W1.data_ptr(), W3.data_ptr(), rbase.data_ptr(),
                      rcounts.data_ptr(), rexp.data_ptr(), nseg, Rs, H, F, El, A.data_ptr(), B.data_ptr(),
                      Hh.data_ptr(), s)

        dy = (torch.zeros(T, H, **bf) if dy is None else dy).to(torch.bfloat16).contiguous()
        dg = torch.empty(T, E, **f32)
        pbb.barrier()                           # every rank is done with the previous layer's dO / dxp
        _lib.call("b200moe_combine_bwd_peer", dy.data_ptr(), pbb.peer[0].data_ptr(), gates.data_ptr(),
                  slot_rank.data_ptr(), seg_peer.data_ptr(), counts.data_ptr(), T, H, E, El, pbb.peer[0].data_ptr(),
                  dg.data_ptr(), _lib.ptr(ctx.og), cfg.top_k, s)
        ctx.og = None
        pbb.barrier()                           # all output gradients have landed
        dA = torch.empty(Rs, F, **bf)
        dB = torch.empty(Rs, F, **bf)
        if ctx.rebuild_h:
            Hh = torch.empty(Rs, F, **bf)
            _lib.call("b200moe_expert_bwd2_h", pbb.do.data_ptr(), W2.data_ptr(), A.data_ptr(), B.data_ptr(),
                      rbase.data_ptr(), rcounts.data_ptr(), rexp.data_ptr(), nseg, Rs, H, F, El, dA.data_ptr(),
                      dB.data_ptr(), Hh.data_ptr(), 0, s)
        else:
            _lib.call("b200moe_expert_bwd2", pbb.do.data_ptr(), W2.data_ptr(), A.data_ptr(), B.data_ptr(),
                      rbase.data_ptr(), rcounts.data_ptr(), rexp.data_ptr(), nseg, Rs, H, F, El, dA.data_ptr(),
                      dB.data_ptr(), s)
        dW1, dW2, dW3, acc = _wgrad_outputs(ctx.acc_targets, W1, W2, W3)
        _wgrad_call(acc, pb.xr.data_ptr(), Hh.data_ptr(), pbb.do.data_ptr(), dA.data_ptr(),
                  dB.data_ptr(), rbase.data_ptr(), rcounts.data_ptr(), rexp.data_ptr(), nseg, Rs, H, F, El,
                  dW1.data_ptr(), dW2.data_ptr(), dW3.data_ptr(), s)
        if acc:
            dW1 = dW2 = dW3 = None
        if ctx.push:   # BWD1 pushes dxp tiles into the source ranks' planes (expert-major, as in the forward)
            arr, dst = _lib.host_u64(pbb.peer_host[1])
            _lib.call("b200moe_expert_bwd1_peer", dA.data_ptr(), dB.data_ptr(), W1.data_ptr(), W3.data_ptr(),
                      rbase.data_ptr(), rcounts.data_ptr(), rexp.data_ptr(), nseg, Rs, H, F, El, dst, plan.world,
                      plan.rank, plan.cap_pad, Rs, s)
        else:
            _lib.call("b200moe_expert_bwd1", dA.data_ptr(), dB.data_ptr(), W1.data_ptr(), W3.data_ptr(),
                      rbase.data_ptr(), rcounts.data_ptr(), rexp.data_ptr(), nseg, Rs, H, F, El, pbb.dxp.data_ptr(),
                      s)
        pbb.barrier()                           # all input gradients are ready
        dx = torch.empty(T, H, **bf)
        dh = torch.empty(T, E, **f32)
        dn = torch.empty(T, E, **f32) if z is not None else None
        dgx, sx_t, sx_e = None, 0, 0
        if dgates is not None:
            dgx = dgates.to(torch.float32)
            sx_t, sx_e = dgx.stride()
        ws = torch.empty(2 * H * _ep(E) + T * _ep(E), **f32)
        dxp_bufs, dxp_base = (pbb.local_rep[1], seg_local) if ctx.push else (pbb.peer[1], seg_peer)
        _lib.call("b200moe_router_bwd_peer", dxp_bufs.data_ptr(), El, slot_rank.data_ptr(), dxp_base.data_ptr(),
                  dg.data_ptr(), _lib.ptr(dgx), sx_t, sx_e, gates.data_ptr(), _lib.ptr(probs), w_g.data_ptr(),
                  w_noise.data_ptr(), _lib.ptr(z), _lib.ptr(noise_act), *_swizzled(ctx, H, E, z), T, H, E,
                  cfg.top_k, _lib.ROUTER[cfg.router_type], dx.data_ptr(), dh.data_ptr(), _lib.ptr(dn), ws.data_ptr(), s)
        dwg = torch.empty(H, E, **f32)
        dwn = torch.empty(H, E, **f32) if z is not None else None
        wsw = torch.empty((T + 63) // 64 * H * E, **f32)
        _lib.call("b200moe_router_wgrad", x.data_ptr(), dh.data_ptr(), _lib.ptr(dn), T, H, E, dwg.data_ptr(),
                  _lib.ptr(dwn), wsw.data_ptr(), _wgrad_tickets(dev, H).data_ptr(), s)
        if st.get("reduce_router", True):
            dist.all_reduce(dwg, group=group)
            if dwn is not None:
                dist.all_reduce(dwn, group=group)
        return dx, dwg, dwn, dW1, dW2, dW3, None, None


class ExpertParallelMoE:
    """EP-sharded E8T2 layer on this rank.  `w_g`, `w_noise`: replicated
    router [H, E] fp32; W1, W3 [E_local, F, H], W2 [E_local, H, F] bf16: the
    experts this rank owns (e.g. from upcycle_shard / upcycle_experts)."""

    TRANSPORTS = ("p2p", "nccl")

    def __init__(self, w_g, w_noise, W1, W2, W3, cfg: GateConfig, group=None, transport: str = "p2p",
                 buffer_slot: int = 0, recompute: bool = False, drop_h: bool = False, gemm_push: bool = True):
        """transport: "p2p" (default) fuses the dispatch/combine exchange into the
        permute/combine kernels over NVLink symmetric memory; "nccl" uses
        all_to_all_single between separate kernels (the comparison baseline).
        buffer_slot: which symmetric receive buffers the p2p transport uses;
        layers whose forwards are alive in the same autograd graph need
        distinct slots (a slot's xr is saved for its backward)."""
        if transport not in self.TRANSPORTS:
            raise ConfigError(f"transport must be one of {self.TRANSPORTS}, got {transport!r}")
        self.transport = transport
        self.group = group
        self.world = dist.get_world_size(group)
        self.rank = dist.get_rank(group)
        if cfg.n_experts % self.world != 0:
            raise ConfigError(f"n_experts ({cfg.n_experts}) not divisible by ep={self.world}")
        if W1.shape[0] != cfg.n_experts // self.world:
            raise ShapeError(f"rank holds {W1.shape[0]} experts, expected {cfg.n_experts // self.world}")
        if cfg.n_experts > 32:
            raise ConfigError("the B200 router supports up to 32 experts")
        self.w_g, self.w_noise, self.W1, self.W2, self.W3, self.cfg = w_g, w_noise, W1, W2, W3, cfg
        self.buffer_slot = buffer_slot
        self.recompute = recompute   # p2p: rebuild a, b, h in the backward instead of keeping them
        self.drop_h = drop_h         # p2p: keep a, b only; BWD2 rebuilds h (one third of the memory of a, b, h)
        self.gemm_push = gemm_push   # p2p: FWD2 / BWD1 push their rows to the sources (else peers pull them)

    def _check_tokens(self, T: int, device) -> None:
        """The p2p transport sizes every rank's receive segments from T_local
        (EPPlan.cap_pad), so all ranks must agree on T.  Checked once per
        (group, T) in the process -- with one all_reduce (max of T and of -T)
        and a host read -- not per layer object: a model builds its layers'
        ExpertParallelMoE views on every forward, and a per-layer check was a
        host synchronisation per layer and micro-batch.  Like every collective
        decision, this assumes SPMD ranks: each rank meets a new T_local in the
        same call (a rank that alone switched to a T another rank already
        checked would not join that rank's all_reduce)."""
        key = (id(self.group) if self.group is not None else None, T)
        if key in _TOKENS_CHECKED:
            return
        t = torch.tensor([T, -T], dtype=torch.int64, device=device if dist.get_backend(self.group) == "nccl" else "cpu")
        dist.all_reduce(t, op=dist.ReduceOp.MAX, group=self.group)
        hi, lo = int(t[0]), -int(t[1])
        if hi != T or lo != T:
            raise ShapeError(f"expert-parallel ranks disagree on tokens per rank (this rank {T}, range [{lo}, {hi}]); "
                             f"the p2p transport needs equal T_local on every rank")
        _TOKENS_CHECKED.add(key)

    def forward(self, x: torch.Tensor, rng=None, training: bool = False, noise=None, reduce_router: bool = True):
        T, H = x.shape
        if H % 256 or self.W1.shape[1] % 256:
            raise ShapeError("the EP path needs hidden and ffn multiples of 256")
        if self.transport == "p2p":
            self._check_tokens(T, x.device)
        plan = EPPlan.make(self.world, self.rank, self.cfg.n_experts, T, self.cfg.capacity_factor)
        z = _noise(T, self.cfg.n_experts, x.device, self.cfg.noise_enabled and training, rng, noise)
        st = dict(cfg=self.cfg, plan=plan, group=self.group, reduce_router=reduce_router, buffer_slot=self.buffer_slot,
                  recompute=self.recompute, drop_h=self.drop_h, gemm_push=self.gemm_push)
        fn = _EPPeerFunction if self.transport == "p2p" else _EPFunction
        y, gates = fn.apply(x.to(torch.bfloat16).contiguous(), self.w_g.to(torch.float32).contiguous(),
                            self.w_noise.to(torch.float32).contiguous(), self.W1, self.W2, self.W3, z, st)
        r = st["routing"]
        from .moe import MoEForwardResult
        gates._b200_importance = (r["importance"], gates._version, r["importance_loss"])
        out = MoEForwardResult(output=y, stats=DeviceRoutingStats(r["counts"], r["stats"], r["gate_mass"], plan.capacity,
                                                            r["err"]), gates=gates)
        out.routing = r
        out.plan = plan
        return out

    __call__ = forward


def run_ep_bench(args, rank: int, world: int, dev, measured: dict):
    """bench.py --gpus N under torchrun: weak scaling, T_local tokens per rank."""
    import json
    import bench as B
    import paper_2412_09952_b200 as P
    from .upcycle import router_weights, upcycle_experts

    H, F, E, K = B.H, B.F, B.E, B.K_TOP
    T = args.tokens
    _lib.call("b200moe_gemm_set_debug", getattr(args, "gemm_debug", 0))
    if E % world:
        raise ConfigError(f"{E} experts cannot be split over {world} ranks")
    torch.manual_seed(0)  # same dense FFN on every rank (upcycling is rank-local copying)
    w1 = (torch.randn(H, F, device=dev) * 0.02).to(torch.bfloat16)
    w2 = (torch.randn(F, H, device=dev) * 0.02).to(torch.bfloat16)
    w3 = (torch.randn(H, F, device=dev) * 0.02).to(torch.bfloat16)
    W1, W2, W3 = (w.requires_grad_() for w in upcycle_experts(w1, w2, w3, E // world))
    del w1, w2, w3
    cfg_m = P.ModelConfig(vocab=32, hidden=H, layers=1, heads=32, kv_heads=8, ffn_hidden=F, seq_len=T)
    wg, wn = router_weights(cfg_m, E, 0, 1, torch.float32, dev)
    wg.requires_grad_()
    wn.requires_grad_()
    gate = P.GateConfig(n_experts=E, top_k=K, router_type=args.router, capacity_factor=args.cf,
                        drop_policy=args.policy)
    layer = ExpertParallelMoE(wg, wn, W1, W2, W3, gate, transport=args.transport,
                              gemm_push=not getattr(args, "ep_pull", False))
    g = torch.Generator(device=dev).manual_seed(1000 + rank)
    x = torch.randn(T, H, device=dev, generator=g).to(torch.bfloat16).requires_grad_()
    dy = torch.randn(T, H, device=dev, generator=g).to(torch.bfloat16)
    lam = torch.tensor(0.01, device=dev)
    params = [W1, W2, W3, wg, wn, x]

    def step(xin, dyin, on_forward=None):
        for p in params:
            p.grad = None
        out = layer(xin)
        if on_forward is not None:
            on_forward(out.output)
        aux = P.importance_penalty(out.gates)
        torch.autograd.backward([out.output, aux], [dyin, lam])
        return out, aux

    try:
        step(x, dy)
        torch.cuda.synchronize()
    except Exception as exc:   # noqa: BLE001 -- symmetric-memory setup failed on this box
        if args.transport != "p2p":
            raise
        import sys
        print(f"[bench] p2p transport unavailable ({exc!r}); measuring the NCCL all-to-all transport",
              file=sys.stderr, flush=True)
        args.transport = "nccl"   # reported in the JSON line's config
        layer = ExpertParallelMoE(wg, wn, W1, W2, W3, gate, transport="nccl")
    def agree(n):   # the same number of warm-up steps on every rank (EP steps synchronise the ranks)
        t = torch.tensor([n], device=dev, dtype=torch.int64)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        return int(t)

    clk = B.ClockSampler(dev.index)   # started before the warm-up (see bench.run_single)
    warm = B.warmup(args, lambda: step(x, dy), agree)
    out = step(x, dy)[0]
    warm += 1
    torch.cuda.synchronize()
    S = int(out.routing["recv_counts"].sum().item())
    s_send = int(out.routing["counts"].sum().item())
    del out          # no autograd graph of an eager step may outlive it into a capture (graphs.py)
    # timed region: GEMM spans recorded inside the same steps (see bench.py).
    # Default: the K steps are captured into one CUDA graph per rank (device
    # barriers, peer kernels and the dW_g all_reduce are all stream work) and
    # replayed once untimed, once timed; --eager launches them from Python.
    prof = _lib.Profiler(spans=_lib.GEMM_SPANS)
    cap = None
    eager = getattr(args, "eager", False)
    if not eager:
        from .graphs import capture
        _lib.PROFILER = prof
        err = None
        try:
            cap = capture(lambda: step(x, dy), repeat=args.steps, warmup=0)
        except Exception as exc:   # noqa: BLE001 -- all ranks fall back together (below)
            err, cap = exc, None
            torch.cuda.synchronize()
        _lib.PROFILER = None
        ok = torch.tensor([0 if cap is None else 1], device=dev)
        dist.all_reduce(ok, op=dist.ReduceOp.MIN)     # a graph only if every rank captured one
        if int(ok) == 0:
            if err is not None:
                import sys
                print(f"[bench] CUDA-graph capture failed ({err!r}); timing the eager loop", file=sys.stderr,
                      flush=True)
            cap, eager = None, True
            args.eager = True
            prof = _lib.Profiler(spans=_lib.GEMM_SPANS)
    if cap is not None:
        dist.barrier()
        cap.replay()
        torch.cuda.synchronize()
        warm += args.steps
    else:
        _lib.PROFILER = prof
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    with clk:
        dist.barrier()
        torch.cuda.synchronize()
        e0.record()
        if cap is not None:
            cap.replay()
        else:
            for _ in range(args.steps):
                step(x, dy)
        e1.record()
        torch.cuda.synchronize()
        dist.barrier()
    _lib.PROFILER = None
    del cap
    ms = e0.elapsed_time(e1) / args.steps
    gemm_ms = prof.span_ms() / args.steps
    t = torch.tensor([ms, float(S)], device=dev, dtype=torch.float64)
    tmax = t.clone()
    dist.all_reduce(tmax[:1], op=dist.ReduceOp.MAX)
    ssum = t[1:].clone()
    dist.all_reduce(ssum, op=dist.ReduceOp.SUM)
    ms_max = float(tmax[0])
    S_tot = float(ssum[0])
    s_all = [torch.zeros(1, device=dev, dtype=torch.float64) for _ in range(world)]
    dist.all_gather(s_all, t[1:].clone())
    s_ranks = [int(v) for v in s_all]

    # e2e: host-resident x / dy copied in, y / dx / aux loss copied out, every step
    dist.barrier()
    e2e_rank = B.run_e2e(args.steps, T, x, dy, step, graphed=not eager)
    e2e_t = torch.tensor([e2e_rank["ms_per_step"]], device=dev, dtype=torch.float64)
    dist.all_reduce(e2e_t, op=dist.ReduceOp.MAX)
    clocks = clk.summary()
    # attribution pass on this rank: per-entry-point events (exchange kernels)
    kp = _lib.Profiler(events=True)
    _lib.PROFILER = kp
    n_prof = 3
    for _ in range(n_prof):
        step(x, dy)
    torch.cuda.synchronize()
    _lib.PROFILER = None
    kt = kp.times_ms()
    achieved = 18.0 * H * F * S / (gemm_ms * 1e-3) / 1e12 if gemm_ms > 0 else None
    # NVLink side of the fused exchange (p2p): bytes each peer kernel moves to or
    # from other ranks' buffers per step -- (R-1)/R of this rank's kept rows
    # (S_send of them, H bf16 each) one way -- against the measured 770 GB/s per
    # direction (B200_PROFILING.md).  Event times include the kernels' local work.
    exchange = None
    if args.transport == "p2p" and world > 1:
        remote = s_send * H * 2 * (world - 1) / world
        # permute and combine-backward store rows into the owners' planes; the return
        # direction rides in FWD2's / BWD1's epilogues (TMA stores into the sources'
        # planes, inside the GEMM time), so combine and the router backward read locally
        per = {"b200moe_permute_peer": remote, "b200moe_combine_bwd_peer": remote,
               "b200moe_combine_peer": 0, "b200moe_router_bwd_peer": 0}
        exchange = {"return_exchange": "pushed by the FWD2 / BWD1 epilogues over NVLink, overlapped with their MMAs "
                                      f"({int(remote)} bytes each way per GEMM; inside gemm_ms_per_step)"}
        for name, nbytes in per.items():
            if name in kt:
                t_ms = kt[name][0] / n_prof
                exchange[name.replace("b200moe_", "")] = {
                    "ms": round(t_ms, 4), "nvlink_bytes": int(nbytes),
                    "GBps": round(nbytes / (t_ms * 1e-3) / 1e9, 1),
                    "frac_of_770": round(nbytes / (t_ms * 1e-3) / 1e9 / 770.0, 3)} if nbytes else {
                    "ms": round(t_ms, 4), "nvlink_bytes": 0, "note": "reads rows the owners' GEMMs pushed here"}
    # CPU baseline: the oracle on the R rank-local batches, run
    # one after the other on rank 0's host cores, each a bounded sample of
    # cpu_tokens tokens; tokens/s = R * sample / total time.
    cpu = None
    # the other ranks wait on a gloo barrier (a blocking socket read) instead of
    # spinning in an NCCL barrier on host cores rank 0's BLAS threads need, and
    # rank 0 leaves one core per other rank
    cpu_group = dist.new_group(backend="gloo")
    if not getattr(args, "no_cpu_baseline", False) and rank == 0:
        spare = max(1, len(os.sched_getaffinity(0)) - (world - 1))
        times, cores = B.cpu_sample(args.cpu_tokens, args.cf, args.router, args.policy, world, threads=spare)
        cpu = {"value": round(world * args.cpu_tokens / sum(times), 3), "unit": "tokens/s", "cores": cores,
               "kind": "port",
               "sample": f"{world} rank-local batches of {args.cpu_tokens} tokens, fwd+bwd at the Llama-3 shape run "
                         f"sequentially, numpy/OpenBLAS fp32 on {cores} threads, {B.cpu_model()}"}
    dist.barrier(group=cpu_group)
    if rank == 0:
        tps = world * T / (ms_max * 1e-3)
        flops = 18.0 * H * F * S_tot + 6.0 * world * T * H * E
        peak = measured["bf16_tflops"]
        peak_s = measured.get("bf16_tflops_sustained", peak)
        burst = ms_max * args.steps < 1000.0
        roof_peak = peak if burst else peak_s
        line = {
            "metric": "E8T2 MoE-layer fwd+bwd tokens/s", "value": round(tps, 1), "unit": "tokens/s",
            "n_gpus": world, "steps": args.steps, "warmup": warm, "ms_per_step": round(ms_max, 4),
            "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "bf16", "data": "synthetic",
            "config": {"workload": "Llama-3-8B-shape E8T2 MoE layer fwd+bwd, expert parallel (configs[2])",
                       "hidden": H, "ffn": F, "experts": E, "top_k": K, "tokens_per_gpu": T,
                       "capacity_factor": args.cf, "router": args.router, "drop_policy": args.policy,
                       "kept_slots_total": int(S_tot), "parallelism": f"ep{world}",
                       "comm": ("dispatch/combine fused into permute/combine kernels over NVLink symmetric memory "
                                "(device barriers) + NCCL all_reduce(dW_g)" if args.transport == "p2p" else
                                "NCCL all_to_all_single (exact splits) + all_reduce(dW_g)"),
                       "transport": args.transport,
                       "return_exchange": ("peers pull expert rows in combine / router backward"
                                           if getattr(args, "ep_pull", False) else
                                           "pushed from the FWD2 / BWD1 epilogues (TMA stores over NVLink)"),
                       "launch": ("eager (one Python call chain per step)" if eager else
                                  f"CUDA graph of the {args.steps} timed steps per rank, replayed once untimed "
                                  f"before the timed replay"),
                       "l2": "inputs > L2, no flush (expert weights + activations)"},
            "mfu": {"measured_peak": round(flops / (ms_max * 1e-3) / (world * peak * 1e12), 4),
                    "spec_2250": round(flops / (ms_max * 1e-3) / (world * 2.25e15), 4)},
            "roofline": {"kernel": "moe_gemm (tcgen05 grouped GEMM, rank 0's 5 launches/step)", "bound": "tensor",
                         "achieved": None if achieved is None else round(achieved, 1), "peak": roof_peak,
                         "unit": "TFLOP/s", "frac": None if achieved is None else round(achieved / roof_peak, 4),
                         "peak_kind": f"measured {'burst' if burst else 'sustained'} bf16",
                         "frac_of_sustained": None if achieved is None else round(achieved / peak_s, 4),
                         "traffic": None,
                         "traffic_note": "no multi-GPU ncu capture; N=1 capture in profiles/",
                         "algorithmic_dram_bytes_per_step": B.gemm_min_bytes(S),
                         "gemm_ms_per_step": round(gemm_ms, 4), "gemm_share_of_step": round(gemm_ms / ms, 4),
                         "kernel_timing": "events around the two GEMM runs of every timed step (rank 0)"},
            "e2e": {"value": round(world * T / (float(e2e_t[0]) * 1e-3), 1), "unit": "tokens/s",
                    "h2d_bytes_per_step": world * e2e_rank["h2d_bytes_per_step"],
                    "d2h_bytes_per_step": world * e2e_rank["d2h_bytes_per_step"],
                    "h2d": e2e_rank["h2d"], "d2h": e2e_rank["d2h"]},
            "cpu_baseline": cpu, "clocks": clocks, "gpu_launches": prof.launches,
            "exchange": exchange,
            "kernels_ms_per_step": {n.replace("b200moe_", ""): round(t_ / n_prof, 4) for n, (t_, c) in kt.items()},
            "kept_slots_per_rank": s_ranks,
        }
        print(json.dumps(line), flush=True)
