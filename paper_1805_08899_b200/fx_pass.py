"""Automatic Echo pass over an arbitrary PyTorch model (PAPER.md:31, 404-415:
Echo is an automatic graph pass that needs no model changes).

    em = EchoModule(model, example_inputs)            # torch.fx trace + the C++ estimator's plan
    loss = em(*inputs); loss.backward()               # same gradients, fewer bytes kept

1. `torch.fx` traces the model (its forward must return the scalar training loss) and ShapeProp
   records every tensor's shape / dtype.
2. The traced graph is written in the estimator's graph schema (the op set of
   oracle/footprint.py) -- Linear / F.linear -> fully_connected, Conv2d -> conv2d, relu / tanh / sigmoid / gelu /
   silu, LayerNorm / F.layer_norm -> layer_norm (three outputs: y, mean, rstd), elementwise add / mul,
   multiplication or division by a constant -> scale, matmul, softmax, dropout (two outputs: y,
   keep-mask), sum -> sum_reduce -- and
   echo_footprint_estimate (a8, Alg. 1) decides per feature map: stash, 1-bit, or
   recompute (mirrored) -- dead FC mirrors are never recomputed.
3. The model runs through an fx Interpreter inside torch.autograd.graph.saved_tensors_hooks: every
   tensor autograd saves is mapped back to its graph edge and
     stash     -> kept as is (and referenced, as a recomputation frontier);
     1-bit     -> packed to one bit per element by libecho (echo_sign_pack: a ReLU's output sign,
                  a dropout's keep-mask; Alg. 1 line 18) and unpacked to
                  a 0 / 1 tensor for the backward (ReLU's backward reads only result > 0);
     recompute -> not kept; regenerated in the backward from the kept frontier by re-running the
                  mirrored nodes (no_grad, memoised per backward; a mirrored dropout re-applies its
                  kept mask, it is never re-drawn: reading R26).
   The gradients are those of the unmodified model (Echo changes no math).
`kept_bytes()` measures what the hooks actually kept (unique storages, parameters excluded), to be
compared with the estimator's `stash_bytes`.
"""
from __future__ import annotations

import json
import operator

import torch
import torch.fx as fx
import torch.nn as nn
import torch.nn.functional as F
from torch.fx.passes.shape_prop import ShapeProp

from . import abi

_DT = {torch.float32: "f32", torch.bfloat16: "bf16", torch.float64: "f64"}


class Unsupported(ValueError):
    pass


def _kind(gm, n):
    """The estimator op of fx node n (or None for placeholders / outputs / parameters)."""
    if n.op == "call_module":
        m = gm.get_submodule(n.target)
        if isinstance(m, nn.Linear):
            return "fully_connected"
        if isinstance(m, nn.Conv2d):
            return "conv2d"
        if isinstance(m, nn.ReLU):
            return "relu"
        if isinstance(m, nn.Tanh):
            return "tanh"
        if isinstance(m, nn.Sigmoid):
            return "sigmoid"
        if isinstance(m, nn.Dropout):
            return "dropout"
        if isinstance(m, nn.GELU):
            return "gelu"
        if isinstance(m, nn.SiLU):
            return "silu"
        if isinstance(m, nn.LayerNorm):
            return "layer_norm"
        raise Unsupported(f"module {type(m).__name__}")
    if n.op == "call_function":
        t = n.target
        if t in (operator.mul, torch.mul, operator.truediv, torch.div) and len(n.args) == 2 and not n.kwargs:
            a, b = n.args
            scalar = lambda x: isinstance(x, (int, float)) and not isinstance(x, bool)
            if isinstance(a, fx.Node) and scalar(b) or (t in (operator.mul, torch.mul) and scalar(a) and isinstance(b, fx.Node)):
                return "scale"                                  # y = c x: a constant factor (or divisor)
        table = {F.linear: "fully_connected", torch.relu: "relu", F.relu: "relu", torch.tanh: "tanh",
                 torch.sigmoid: "sigmoid", operator.add: "add", torch.add: "add", operator.mul: "mul",
                 torch.mul: "mul", torch.matmul: "matmul", operator.matmul: "matmul", F.softmax: "softmax",
                 torch.softmax: "softmax", torch.sum: "sum_reduce", F.dropout: "dropout", F.gelu: "gelu",
                 F.silu: "silu", F.layer_norm: "layer_norm"}
        if t in table:
            return table[t]
        raise Unsupported(f"function {getattr(t, '__name__', t)}")
    if n.op == "call_method":
        table = {"relu": "relu", "tanh": "tanh", "sigmoid": "sigmoid", "sum": "sum_reduce", "softmax": "softmax"}
        if n.target in table:
            return table[n.target]
        raise Unsupported(f"method {n.target}")
    return None


class EchoPlan:
    """The traced model in the estimator's schema, the estimator's decisions and the fx <-> edge maps."""

    def __init__(self, model: nn.Module, example_inputs, strategy="echo", enable_binarization=True):
        self.gm = fx.symbolic_trace(model)
        ShapeProp(self.gm).propagate(*example_inputs)
        self.doc, self.node_id, self.param_ids = self._to_doc()
        cfg = {"strategy": strategy, "enable_binarization": bool(enable_binarization)}
        self.report = json.loads(abi.echo_footprint_estimate(json.dumps(self.doc), json.dumps(cfg)))
        self.decision = {(int(i), int(k)): d for i, k, d in self.report["decisions"]}
        self.by_id = {i: n for n, i in self.node_id.items()}

    def _meta(self, n):
        tm = n.meta.get("tensor_meta")
        if tm is None:
            raise Unsupported(f"no shape for {n.name}")
        if tm.dtype not in _DT and tm.dtype != torch.bool:
            raise Unsupported(f"dtype {tm.dtype} of {n.name}")
        return list(tm.shape), _DT.get(tm.dtype, "u8")

    def _to_doc(self):
        gm = self.gm
        ph, nodes, outputs = [], [], []
        ids, pids = {}, {}
        nid = 0

        def param(name, t):
            nonlocal nid
            if name not in pids:
                pids[name] = nid
                ph.append({"id": nid, "name": name, "shape": list(t.shape), "dtype": _DT[t.dtype], "trainable": True,
                           "tag": "param"})
                nid += 1
            return [pids[name], 0]

        for n in gm.graph.nodes:
            if n.op == "placeholder":
                shp, dt = self._meta(n)
                ids[n] = nid
                ph.append({"id": nid, "name": n.name, "shape": shp, "dtype": dt, "trainable": False, "tag": "input"})
                nid += 1
            elif n.op == "get_attr":
                ids[n] = param(n.target, getattr(gm, n.target) if "." not in n.target else gm.get_parameter(n.target))[0]
            elif n.op == "output":
                arg = n.args[0]
                if not isinstance(arg, fx.Node):
                    raise Unsupported("the model must return one scalar loss tensor")
                outputs.append([ids[arg], 0])
            else:
                op = _kind(gm, n)
                ins, attrs = [], {}
                if op == "fully_connected" and n.op == "call_module":
                    m = gm.get_submodule(n.target)
                    ins = [[ids[n.args[0]], 0], param(f"{n.target}.weight", m.weight)]
                    if m.bias is not None:
                        ins.append(param(f"{n.target}.bias", m.bias))
                elif op == "conv2d":
                    m = gm.get_submodule(n.target)
                    st, pd = m.stride, m.padding
                    if (m.groups != 1 or m.dilation != (1, 1) or isinstance(pd, str) or st[0] != st[1] or pd[0] != pd[1]
                            or m.padding_mode != "zeros"):
                        raise Unsupported(f"{n.name}: conv2d needs groups 1, dilation 1, square stride / zero padding")
                    ins = [[ids[n.args[0]], 0], param(f"{n.target}.weight", m.weight)]
                    if m.bias is not None:
                        ins.append(param(f"{n.target}.bias", m.bias))
                    attrs.update(stride=int(st[0]), padding=int(pd[0]))
                elif op == "layer_norm":
                    if n.op == "call_module":
                        m = gm.get_submodule(n.target)
                        shape = tuple(m.normalized_shape)
                        ins = [[ids[n.args[0]], 0]]
                        if m.weight is not None:
                            ins.append(param(f"{n.target}.weight", m.weight))
                        if m.bias is not None:
                            ins.append(param(f"{n.target}.bias", m.bias))
                    else:
                        shape = n.args[1] if len(n.args) > 1 else n.kwargs["normalized_shape"]
                        if any(isinstance(a, fx.Node) for a in list(n.args[2:]) + list(n.kwargs.values())):
                            raise Unsupported(f"{n.name}: functional layer_norm with weight / bias tensors")
                        ins = [[ids[n.args[0]], 0]]
                    attrs["norm_ndim"] = len(shape) if isinstance(shape, (tuple, list)) else 1
                elif op == "dropout":
                    m = gm.get_submodule(n.target) if n.op == "call_module" else None
                    attrs["p"] = m.p if m is not None else n.kwargs.get("p", n.args[1] if len(n.args) > 1 else 0.5)
                    ins = [[ids[n.args[0]], 0]]
                else:
                    for a in n.args:
                        if isinstance(a, fx.Node):
                            ins.append([ids[a], 0])
                        elif op not in ("softmax", "sum_reduce", "scale"):
                            raise Unsupported(f"{n.name}: non-tensor operand {a!r}")
                    if op in ("add", "mul"):
                        shapes = [self._meta(a)[0] for a in n.args if isinstance(a, fx.Node)]
                        if len(shapes) != 2 or shapes[0] != shapes[1]:
                            raise Unsupported(f"{n.name}: broadcasting {op}")
                ids[n] = nid
                nodes.append({"id": nid, "op": op, "inputs": ins, "attrs": attrs, "tag": n.name})
                nid += 1
        return {"version": 1, "placeholders": ph, "nodes": nodes, "outputs": outputs}, ids, pids

    def stash_bytes(self):
        return int(self.report["stash_bytes"])


class _Run(fx.Interpreter):
    """Runs the traced model; records which edge every output tensor is."""

    def __init__(self, owner):
        super().__init__(owner.plan.gm)
        self.o = owner

    def run_node(self, n):
        self.o.current = n
        self.o.ln_stat = 0
        out = super().run_node(n)
        if isinstance(out, torch.Tensor) and n in self.o.plan.node_id:
            self.o._record(n, out)
        return out


class EchoModule(nn.Module):
    """`model` with Echo's feature-map plan applied automatically (see the module docstring)."""

    def __init__(self, model: nn.Module, example_inputs, strategy="echo", enable_binarization=True):
        super().__init__()
        self.model = model
        self.plan = EchoPlan(model, example_inputs, strategy, enable_binarization)
        self.params = {p.untyped_storage().data_ptr() for p in model.parameters()}
        self._reset()

    def _reset(self):
        self.env = {}            # edge -> kept tensor (stash edges, inputs, kept masks): the frontier
        self.bits = {}           # edge -> (bits, shape, dtype) of binarized edges
        self.ptr_of = {}         # fx node -> storage ptr of its output (no reference held)
        self.kept = {}           # storage ptr -> bytes actually kept (tensors, bits, frontier refs)
        self.cache = {}          # recomputed edges (per backward)
        self.current = None

    # ------------------------------------------------------------ forward bookkeeping
    def _record(self, n, t):
        e = (self.plan.node_id[n], 0)
        self.ptr_of[n] = t.untyped_storage().data_ptr()
        if self.plan.decision.get(e) == "stash":                           # frontier: referenced
            self.env[e] = t
            self._keep(t)

    def _keep(self, t, nbytes=None):
        k = t.untyped_storage().data_ptr()
        if k not in self.params:
            self.kept[k] = nbytes if nbytes is not None else t.untyped_storage().nbytes()

    def kept_bytes(self):
        return sum(self.kept.values())

    # ------------------------------------------------------------ saved-tensor hooks
    def _edge_of(self, t):
        """A tensor saved while fx node `current` runs is one of its inputs, its output, or (dropout)
        its keep-mask; the inputs are alive, so their storage identifies them."""
        n = self.current
        k = t.untyped_storage().data_ptr()
        for a in n.all_input_nodes:
            if self.ptr_of.get(a) == k:
                return (self.plan.node_id[a], 0)
        kind = _kind(self.plan.gm, n)
        if kind == "dropout" and t.dtype == torch.bool:
            return (self.plan.node_id[n], 1)
        if kind == "layer_norm":                               # native_layer_norm saves x, then mean, rstd
            self.ln_stat = getattr(self, "ln_stat", 0) + 1
            return (self.plan.node_id[n], self.ln_stat)
        return (self.plan.node_id[n], 0)

    def _pack(self, t):
        k = t.untyped_storage().data_ptr()
        if k in self.params or self.current is None:
            return ("T", t)
        e = self._edge_of(t)
        d = self.plan.decision.get(e)
        if d == "bit" and not t.is_cuda:                      # no host path: the 1-bit pack is a libecho kernel
            raise RuntimeError(f"EchoModule: edge {e} is kept as 1 bit, which needs a CUDA tensor (got {t.device})")
        if d == "bit":
            if e in self.bits:
                bits = self.bits[e][0]
            else:
                bits = torch.empty((t.numel() + 7) // 8, dtype=torch.uint8, device=t.device)
                abi.echo_sign_pack(t.contiguous(), bits)
                self.bits[e] = (bits, t.shape, t.dtype)
                self._keep(bits, bits.numel())
            return ("B", bits, t.shape, t.dtype)
        if e[1] >= 1 and d not in ("bit", "recompute"):      # a kept (byte) mask / statistic is a frontier too
            self.env[e] = t
        if d == "recompute":                                  # (never a keep-mask: masks are random, R26)
            return ("R", e, t.shape, t.stride(), t.storage_offset())
        self._keep(t)
        return ("T", t)

    def _unpack(self, obj):
        if obj[0] == "T":
            return obj[1]
        if obj[0] == "B":
            _, bits, shape, dtype = obj
            out = torch.empty(shape, dtype=dtype, device=bits.device)
            abi.echo_bits_unpack(bits, out)
            return out
        _, e, shape, stride, off = obj
        base = self._value(e)
        if tuple(base.shape) == tuple(shape) and base.stride() == tuple(stride):
            return base
        return base.as_strided(shape, stride, off)

    def _value(self, e):
        """The tensor of edge e in the backward: a kept one, or regenerated from the frontier."""
        if e in self.cache:
            return self.cache[e]
        d = self.plan.decision.get(e)
        n = self.plan.by_id.get(e[0])
        if e in self.bits and e[1] == 1:                      # a binarized keep-mask: decode it
            bits, shape, dtype = self.bits[e]
            v = torch.empty(shape, dtype=dtype, device=bits.device)
            abi.echo_bits_unpack(bits, v)
        elif n is None or n.op in ("placeholder", "get_attr") or d in ("stash", None):
            v = self.env[e]
        elif d == "bit":
            raise RuntimeError(f"edge {e} was binarized but is needed by value")
        else:
            with torch.no_grad():
                v = self._rerun(n)
            if isinstance(v, tuple):                           # layer_norm: (y, mean, rstd), all cached
                for k, x in enumerate(v):
                    self.cache[(e[0], k)] = x
                v = v[e[1]]
        self.cache[e] = v
        return v

    def _arg(self, a):
        if isinstance(a, fx.Node):
            if a.op == "get_attr":
                return self.plan.gm.get_parameter(a.target)
            return self._value((self.plan.node_id[a], 0))
        if isinstance(a, (tuple, list)):
            return type(a)(self._arg(x) for x in a)
        return a

    def _rerun(self, n):
        gm = self.plan.gm
        args = [self._arg(a) for a in n.args]
        kwargs = {k: self._arg(v) for k, v in n.kwargs.items()}
        if _kind(gm, n) == "dropout":                         # mirrored dropout: re-apply the kept mask
            m = gm.get_submodule(n.target) if n.op == "call_module" else None
            p = m.p if m is not None else kwargs.get("p", args[1] if len(args) > 1 else 0.5)
            training = m.training if m is not None else kwargs.get("training", True)
            if p == 0.0 or not training:                      # identity: no mask was drawn
                return args[0]
            mask = self._value((self.plan.node_id[n], 1))
            return args[0] * mask * (1.0 / (1.0 - p))
        if _kind(gm, n) == "layer_norm":                      # all three outputs (the same kernel as the forward)
            if n.op == "call_module":
                m = gm.get_submodule(n.target)
                return tuple(torch.native_layer_norm(args[0], m.normalized_shape, m.weight, m.bias, m.eps))
            shape = args[1] if len(args) > 1 else kwargs["normalized_shape"]
            eps = kwargs.get("eps", args[4] if len(args) > 4 else 1e-5)
            return tuple(torch.native_layer_norm(args[0], list(shape), None, None, eps))
        if n.op == "call_module":
            return gm.get_submodule(n.target)(*args, **kwargs)
        if n.op == "call_method":
            return getattr(args[0], n.target)(*args[1:], **kwargs)
        return n.target(*args, **kwargs)

    def forward(self, *inputs):
        self._reset()
        with torch.autograd.graph.saved_tensors_hooks(self._pack, self._unpack):
            out = _Run(self).run(*inputs)
        self.current = None
        return out


def baseline_saved_bytes(model: nn.Module, *inputs):
    """Bytes autograd keeps for the unmodified model's backward (unique storages, parameters excluded):
    the Baseline the estimator's "baseline" strategy models (reading R11)."""
    params = {p.untyped_storage().data_ptr() for p in model.parameters()}
    kept = {}

    def pack(t):
        k = t.untyped_storage().data_ptr()
        if k not in params:
            kept[k] = t.untyped_storage().nbytes()
        return t
    with torch.autograd.graph.saved_tensors_hooks(pack, lambda t: t):
        out = model(*inputs)
    return out, sum(kept.values())
