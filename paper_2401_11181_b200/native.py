"""ctypes binding of libtetri.so (include/tetri.h).

This is the only door from Python to the device path.  There is no fallback:
if the library is missing or has no CUDA device, calls raise ``NativeError``.
Status codes map to exceptions the way SURVEY.md §8(b) prescribes:
``TK_EINVAL`` -> ValueError, ``TK_ECAPACITY`` -> SimulationError (a KV
capacity break, as pdsim/decode.py:63-66), everything else -> NativeError.
"""

from __future__ import annotations

import ctypes as C
import os
import time
from dataclasses import dataclass
from pathlib import Path

from .engine import SimulationError

LIB_PATH = Path(__file__).resolve().parent / "lib" / "libtetri.so"

TK_OK, TK_EINVAL, TK_ECUDA, TK_ENOMEM, TK_ECAPACITY, TK_EUNSUPPORTED = 0, -1, -2, -3, -4, -5
TK_ARCH_OPT, TK_ARCH_LLAMA = 0, 1
EPI_BF16, EPI_BF16_BIAS, EPI_BF16_BIAS_RELU, EPI_F32_BIAS_RESID, EPI_F32 = range(5)


class NativeError(RuntimeError):
    pass


class tk_model_desc(C.Structure):
    _fields_ = [("arch", C.c_int32), ("n_layers", C.c_int32), ("hidden", C.c_int32),
                ("n_heads", C.c_int32), ("head_dim", C.c_int32), ("ffn", C.c_int32),
                ("vocab", C.c_int32), ("max_positions", C.c_int32), ("n_labels", C.c_int32),
                ("init_std", C.c_float), ("norm_eps", C.c_float), ("rope_theta", C.c_float)]


class tk_slice(C.Structure):
    _fields_ = [("start", C.c_int32), ("len", C.c_int32), ("bt_offset", C.c_int32),
                ("n_pages", C.c_int32), ("emit", C.c_int32)]


_P = C.c_void_p
_I32P = C.POINTER(C.c_int32)
_I64P = C.POINTER(C.c_int64)

_SIGNATURES = {
    "tk_last_error": ([], C.c_char_p),
    "tk_version": ([], C.c_int),
    "tk_device_count": ([_I32P], C.c_int),
    "tk_device_memory": ([C.c_int32, _I64P, _I64P], C.c_int),
    "tk_instance_create": ([C.c_int32, C.POINTER(tk_model_desc), C.c_uint64, C.c_int32, C.c_int32,
                            C.c_int32, C.POINTER(_P)], C.c_int),
    "tk_instance_destroy": ([_P], C.c_int),
    "tk_instance_info": ([_P, _I64P, _I64P, _I64P], C.c_int),
    "tk_weight_numel": ([_P, C.c_char_p, _I64P], C.c_int),
    "tk_weight_read": ([_P, C.c_char_p, _P, C.c_int64], C.c_int),
    "tk_weight_write": ([_P, C.c_char_p, _P, C.c_int64], C.c_int),
    "tk_kv_read": ([_P, C.c_int32, _P], C.c_int),
    "tk_prefill_chunk": ([_P, C.c_int32, _I32P, C.POINTER(tk_slice), C.c_int32, _I32P, C.c_int32,
                          _I32P, C.POINTER(C.c_float), C.POINTER(_P)], C.c_int),
    "tk_decode_step": ([_P, C.c_int32, _I32P, _I32P, _I32P, C.c_int32, _I32P,
                        C.POINTER(C.c_float), C.POINTER(_P)], C.c_int),
    "tk_kv_send": ([_P, _I32P, _P, _I32P, C.c_int32, C.POINTER(_P)], C.c_int),
    "tk_kv_send_ex": ([_P, _I32P, _P, _I32P, C.c_int32, C.c_int32, C.POINTER(_P)], C.c_int),
    "tk_predict": ([_P, _I32P, _I32P, C.c_int32, C.c_int32, _I32P, C.POINTER(_P)], C.c_int),
    "tk_predict_scores": ([_P, _I32P, _I32P, C.c_int32, C.c_int32, _I32P, C.POINTER(C.c_float),
                           C.POINTER(_P)], C.c_int),
    "tk_swap_out": ([_P, _I32P, C.c_int32, _P, C.POINTER(_P)], C.c_int),
    "tk_swap_in": ([_P, _I32P, C.c_int32, _P, C.POINTER(_P)], C.c_int),
    "tk_host_alloc": ([C.c_int64, C.POINTER(_P)], C.c_int),
    "tk_host_free": ([_P], C.c_int),
    "tk_event_query": ([_P, _I64P], C.c_int),
    "tk_event_wait": ([_P, _I64P], C.c_int),
    "tk_event_release": ([_P], C.c_int),
    "tk_instance_sync": ([_P], C.c_int),
    "tk_event_elapsed": ([_P, _P, _I64P], C.c_int),
    "tk_event_anchor": ([C.c_int32, C.POINTER(_P)], C.c_int),
    "tk_launch_count": ([_I64P], C.c_int),
    "tk_last_staged_bytes": ([_P, _I64P, _I64P], C.c_int),
    "tk_profile_enable": ([_P, C.c_int32], C.c_int),
    "tk_profile_read": ([_P, C.c_int32, _I64P, C.POINTER(C.c_double), C.POINTER(C.c_double),
                         C.POINTER(C.c_double)], C.c_int),
    "tk_gemm_bf16": ([_P, _P, _P, _P, C.c_int32, C.c_int32, C.c_int32, C.c_int32, _P, C.c_int64,
                      _P], C.c_int),
    "tk_gemm_workspace_bytes": ([C.c_int32, C.c_int32, C.c_int32, _I64P], C.c_int),
    "tk_layernorm": ([_P, _P, _P, _P, C.c_int32, C.c_int32, C.c_float, _P], C.c_int),
    "tk_argmax": ([_P, C.c_int32, C.c_int32, C.c_int32, _P, _P], C.c_int),
    "tk_paged_decode_attention": ([_P, _P, _P, C.c_int32, C.c_int32, C.c_int32, C.c_int32,
                                   C.c_int32, _P, C.c_int32, _P, C.c_int32, C.c_float, _P,
                                   C.c_int64, _P], C.c_int),
    "tk_chunk_attention": ([_P, C.c_int32, _P, _P, C.c_int32, C.c_int32, C.c_int32, C.c_int32,
                            C.c_int32, C.POINTER(tk_slice), C.c_int32, _I32P, C.c_int32,
                            C.c_float, _P], C.c_int),
    "tk_debug_fa_trace": ([C.POINTER(C.c_uint64), C.c_int32], C.c_int),
    "tk_debug_gemm_trace": ([C.POINTER(C.c_uint64), C.c_int32], C.c_int),
    "tk_debug_gemm_cta_trace": ([C.POINTER(C.c_uint64), C.c_int32], C.c_int),
    "tk_fa_plan": ([C.POINTER(tk_slice), C.c_int32, C.c_int32, C.c_int32, _I32P, _I32P, C.c_int32,
                    _I32P, C.c_int32, _I32P, C.c_int32, C.c_int32], C.c_int),
    "tk_chunk_attention_timed": ([_P, C.c_int32, _P, _P, C.c_int32, C.c_int32, C.c_int32,
                                  C.c_int32, C.c_int32, C.POINTER(tk_slice), C.c_int32, _I32P,
                                  C.c_int32, C.c_float, _P, C.c_int32, C.POINTER(C.c_float)],
                                 C.c_int),
}

EXPORTED = tuple(_SIGNATURES)
SEND_ENGINES = {"auto": 0, "sm": 1, "ce": 2}  # TK_SEND_* in include/tetri.h

_lib: C.CDLL | None = None


def load(path: str | Path | None = None) -> C.CDLL:
    """Load (once) and type the library; raises NativeError if absent."""
    global _lib
    if _lib is not None:
        return _lib
    p = Path(path) if path else Path(os.environ["TK_LIB"]) if os.environ.get("TK_LIB") else LIB_PATH
    if not p.exists():
        raise NativeError(f"{p} not built; run `python -m paper_2401_11181_b200.build`")
    lib = C.CDLL(str(p))
    for name, (args, res) in _SIGNATURES.items():
        fn = getattr(lib, name)
        fn.argtypes = args
        fn.restype = res
    _lib = lib
    return lib


def check(rc: int, what: str = "") -> int:
    if rc >= 0:
        return rc
    msg = f"{what}: {load().tk_last_error().decode()}" if what else load().tk_last_error().decode()
    if rc == TK_EINVAL:
        raise ValueError(msg)
    if rc == TK_ECAPACITY:
        raise SimulationError(msg)
    raise NativeError(f"[{rc}] {msg}")


def i32(values) -> C.Array:
    """int32 C array from a sequence (array.array fills it in C: a decode step's
    block table of ~20k entries converts in ~0.4 ms instead of ~3 ms through
    ctypes argument unpacking)."""
    import array
    buf = array.array("i", values)
    if not buf:
        return (C.c_int32 * 1)()
    return (C.c_int32 * len(buf)).from_buffer(buf)  # keeps `buf` alive


# ---------------------------------------------------------------- model shapes

@dataclass(frozen=True)
class ModelShape:
    name: str
    arch: int
    n_layers: int
    hidden: int
    n_heads: int
    ffn: int
    vocab: int
    max_positions: int = 2048
    n_labels: int = 0
    init_std: float = 0.02
    norm_eps: float = 1e-5
    rope_theta: float = 10000.0

    @property
    def head_dim(self) -> int:
        return self.hidden // self.n_heads

    @property
    def kv_bytes_per_token(self) -> int:
        return 2 * self.n_layers * self.hidden * 2

    @property
    def params(self) -> int:
        h, f = self.hidden, self.ffn
        if self.arch == TK_ARCH_OPT:
            per = 4 * h * h + 3 * h + h + 2 * h * f + f + h + 4 * h
            head = 0 if not self.n_labels else ((self.n_labels + 7) // 8 * 8) * h
            return self.vocab * h + (self.max_positions + 2) * h + self.n_layers * per + 2 * h + head
        per = 4 * h * h + 3 * h * f + 2 * h
        return 2 * self.vocab * h + self.n_layers * per + h

    def gemm_flops_per_token(self) -> int:
        """Dense GEMM FLOPs per token across all layers (excl. attention / head)."""
        h, f = self.hidden, self.ffn
        mult = 2 if self.arch == TK_ARCH_OPT else 3
        return 2 * self.n_layers * (4 * h * h + mult * h * f)

    def desc(self) -> tk_model_desc:
        return tk_model_desc(self.arch, self.n_layers, self.hidden, self.n_heads, self.head_dim,
                             self.ffn, self.vocab, self.max_positions, self.n_labels,
                             self.init_std, self.norm_eps, self.rope_theta)


# OPT-13B shape with the learned-position table extended to cover 8k prompts
# plus 2k decodes (random weights; SURVEY.md §7 "hard parts").
OPT_13B = ModelShape("opt-13b", TK_ARCH_OPT, 40, 5120, 40, 20480, 50272, max_positions=10240)
# OPT-125M ("the tiny decoder", BASELINE.json configs[0]) with the position table
# extended like OPT-13B's so the four-class workload's 8k+2k requests fit.
OPT_125M = ModelShape("opt-125m", TK_ARCH_OPT, 12, 768, 12, 3072, 50272, max_positions=10240)
LLAMA2_7B = ModelShape("llama-2-7b", TK_ARCH_LLAMA, 32, 4096, 32, 11008, 32000,
                       max_positions=4096, norm_eps=1e-5)
# OPT-125M-shaped predictor with the 41-bucket score head (g=200, 8192 max).
PREDICTOR_125M = ModelShape("opt-125m-cls", TK_ARCH_OPT, 12, 768, 12, 3072, 50272,
                            max_positions=2048, n_labels=41)
# Small shapes for parity tests (fast on the fp32 CPU oracle).
TINY_OPT = ModelShape("tiny", TK_ARCH_OPT, 2, 256, 2, 1024, 1024, max_positions=1024)
TINY_LLAMA = ModelShape("tiny-llama", TK_ARCH_LLAMA, 2, 256, 2, 768, 1024, max_positions=1024)
# Tiny OPT whose position table covers pdsim's longest request (8192-token prompt +
# 2048 decodes): replays of the reference's default workloads (executor "replay").
TINY_LONG = ModelShape("tiny-long", TK_ARCH_OPT, 2, 256, 2, 1024, 1024, max_positions=10240)

MODELS = {m.name: m for m in (OPT_13B, OPT_125M, LLAMA2_7B, PREDICTOR_125M, TINY_OPT, TINY_LLAMA,
                              TINY_LONG)}


# ---------------------------------------------------------------- handles

class Event:
    """A device completion handle (``done()`` for the engine, ``wait()``)."""

    def __init__(self, ptr: C.c_void_p, keep=(), device: int | None = None):
        self._ptr = ptr
        self._keep = keep  # host buffers that must outlive publication
        self._done = False
        self.elapsed_ns = 0
        self.device = device
        self._t_done: float | None = None

    def done_time(self) -> float | None:
        """Host ``time.perf_counter()`` of the device completion (the end marker
        mapped through the device's anchor event), or None if not done."""
        if not self._done or self.device is None:
            return None
        if self._t_done is None:
            anchor, t0 = _anchor(self.device)
            ns = C.c_int64()
            check(load().tk_event_elapsed(anchor._ptr, self._ptr, C.byref(ns)),
                  "tk_event_elapsed")
            self._t_done = t0 + ns.value / 1e9
        return self._t_done

    def done(self) -> bool:
        if self._done:
            return True
        ns = C.c_int64(0)
        rc = check(load().tk_event_query(self._ptr, C.byref(ns)), "tk_event_query")
        if rc == 1:
            self._done = True
            self.elapsed_ns = ns.value
        return self._done

    def wait(self) -> int:
        if not self._done:
            ns = C.c_int64(0)
            check(load().tk_event_wait(self._ptr, C.byref(ns)), "tk_event_wait")
            self._done = True
            self.elapsed_ns = ns.value
        return self.elapsed_ns

    def __del__(self):
        try:
            if self._ptr and _lib is not None:
                _lib.tk_event_release(self._ptr)
        except Exception:
            pass


class Instance:
    """One device-side serving instance (weights + KV page pool + streams)."""

    def __init__(self, shape: ModelShape, device: int = 0, seed: int = 0, kv_pages: int = 64,
                 page_tokens: int = 16, max_chunk: int = 512):
        lib = load()
        self.shape = shape
        self.device = device
        self.page_tokens = page_tokens
        self.kv_pages = kv_pages
        self.max_chunk = max_chunk
        self._desc = shape.desc()
        h = C.c_void_p()
        check(lib.tk_instance_create(device, C.byref(self._desc), seed, kv_pages, page_tokens,
                                     max_chunk, C.byref(h)), "tk_instance_create")
        self._h = h
        wb, pb, kb = C.c_int64(), C.c_int64(), C.c_int64()
        check(lib.tk_instance_info(h, C.byref(wb), C.byref(pb), C.byref(kb)))
        self.weight_bytes, self.page_bytes, self.pool_bytes = wb.value, pb.value, kb.value

    @property
    def handle(self):
        return self._h

    def close(self) -> None:
        if self._h:
            load().tk_instance_destroy(self._h)
            self._h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    # -- weights (parity tests) --------------------------------------------------
    def weight_numel(self, name: str) -> int:
        n = C.c_int64()
        check(load().tk_weight_numel(self._h, name.encode(), C.byref(n)), "tk_weight_numel")
        return n.value

    def read_weight(self, name: str):
        import numpy as np
        n = self.weight_numel(name)
        buf = np.empty(n, dtype=np.uint16)
        check(load().tk_weight_read(self._h, name.encode(), buf.ctypes.data, n), "tk_weight_read")
        return buf

    def write_weight(self, name: str, bf16_bits) -> None:
        import numpy as np
        arr = np.ascontiguousarray(bf16_bits, dtype=np.uint16).ravel()
        check(load().tk_weight_write(self._h, name.encode(), arr.ctypes.data, arr.size),
              "tk_weight_write")

    def read_page(self, page: int):
        import numpy as np
        buf = np.empty(self.page_bytes // 2, dtype=np.uint16)
        check(load().tk_kv_read(self._h, page, buf.ctypes.data), "tk_kv_read")
        return buf

    # -- data path ---------------------------------------------------------------------
    def prefill_chunk(self, token_ids, slices, block_tables, want_logits: bool = False):
        """slices: [(start, len, bt_offset, n_pages, emit)].  Returns (event, tokens[, logits])."""
        import numpy as np
        n = len(token_ids)
        ids = i32(token_ids)
        sl = (tk_slice * len(slices))(*[tk_slice(*s) for s in slices])
        bt = i32(block_tables)
        out = (C.c_int32 * len(slices))()
        n_emit = sum(1 for s in slices if s[4])
        logits = np.empty((n_emit, self.shape.vocab), dtype=np.float32) if want_logits else None
        ev = C.c_void_p()
        check(load().tk_prefill_chunk(
            self._h, n, ids, sl, len(slices), bt, len(block_tables), out,
            logits.ctypes.data_as(C.POINTER(C.c_float)) if want_logits and n_emit else None,
            C.byref(ev)), "tk_prefill_chunk")
        e = Event(ev, keep=(ids, sl, bt, out), device=self.device)
        return (e, out, logits) if want_logits else (e, out)

    def decode_step(self, last_tokens, ctx_lens, block_tables, bt_stride, want_logits=False):
        import numpy as np
        b = len(last_tokens)
        out = (C.c_int32 * b)()
        logits = np.empty((b, self.shape.vocab), dtype=np.float32) if want_logits else None
        ids, lens, bt = i32(last_tokens), i32(ctx_lens), i32(block_tables)
        ev = C.c_void_p()
        check(load().tk_decode_step(
            self._h, b, ids, lens, bt, bt_stride, out,
            logits.ctypes.data_as(C.POINTER(C.c_float)) if want_logits else None,
            C.byref(ev)), "tk_decode_step")
        e = Event(ev, keep=(ids, lens, bt, out), device=self.device)
        return (e, out, logits) if want_logits else (e, out)

    def kv_send(self, src_pages, dst: "Instance", dst_pages, engine: str = "auto") -> Event:
        """engine: "auto" (tk_kv_send), "sm" (page-copy kernel; peer stores over
        NVLink across devices) or "ce" (copy engines)."""
        if engine not in SEND_ENGINES:
            raise ValueError(f"engine must be one of {sorted(SEND_ENGINES)}")
        sp, dp = i32(src_pages), i32(dst_pages)
        ev = C.c_void_p()
        if engine == "auto":
            check(load().tk_kv_send(self._h, sp, dst._h, dp, len(src_pages), C.byref(ev)),
                  "tk_kv_send")
        else:
            check(load().tk_kv_send_ex(self._h, sp, dst._h, dp, len(src_pages),
                                       SEND_ENGINES[engine], C.byref(ev)), "tk_kv_send_ex")
        return Event(ev, keep=(sp, dp), device=self.device)

    def predict(self, token_ids, lens, max_len: int = 512):
        out = (C.c_int32 * len(lens))()
        ids, ls = i32(token_ids), i32(lens)
        ev = C.c_void_p()
        check(load().tk_predict(self._h, ids, ls, len(lens), max_len, out, C.byref(ev)),
              "tk_predict")
        return Event(ev, keep=(ids, ls, out), device=self.device), out

    def predict_scores(self, token_ids, lens, max_len: int = 512):
        """(buckets, fp32 scores [n, n_labels]) -- waits for the device."""
        import numpy as np
        out = (C.c_int32 * len(lens))()
        scores = np.empty((len(lens), self.shape.n_labels), dtype=np.float32)
        ids, ls = i32(token_ids), i32(lens)
        ev = C.c_void_p()
        check(load().tk_predict_scores(self._h, ids, ls, len(lens), max_len, out,
                                       scores.ctypes.data_as(C.POINTER(C.c_float)), C.byref(ev)),
              "tk_predict_scores")
        e = Event(ev, keep=(ids, ls, out), device=self.device)
        e.wait()
        return list(out), scores

    def swap_out(self, pages, host_ptr) -> Event:
        p = i32(pages)
        ev = C.c_void_p()
        check(load().tk_swap_out(self._h, p, len(pages), host_ptr, C.byref(ev)), "tk_swap_out")
        return Event(ev, keep=(p,), device=self.device)

    def swap_in(self, pages, host_ptr) -> Event:
        p = i32(pages)
        ev = C.c_void_p()
        check(load().tk_swap_in(self._h, p, len(pages), host_ptr, C.byref(ev)), "tk_swap_in")
        return Event(ev, keep=(p,), device=self.device)

    def sync(self) -> None:
        check(load().tk_instance_sync(self._h), "tk_instance_sync")

    # -- instrumentation ----------------------------------------------------------------
    def staged_bytes(self) -> tuple[int, int]:
        a, b = C.c_int64(), C.c_int64()
        check(load().tk_last_staged_bytes(self._h, C.byref(a), C.byref(b)))
        return a.value, b.value

    def profile(self, on: bool) -> None:
        check(load().tk_profile_enable(self._h, 1 if on else 0))

    def profile_read(self) -> dict:
        """Per kernel class: launches, ms, algorithmic flops and bytes (resets)."""
        out = {}
        for kind, name in enumerate(PROFILE_KINDS):
            n, ms, fl, by = C.c_int64(), C.c_double(), C.c_double(), C.c_double()
            check(load().tk_profile_read(self._h, kind, C.byref(n), C.byref(ms), C.byref(fl),
                                         C.byref(by)), "tk_profile_read")
            out[name] = {"launches": n.value, "ms": ms.value, "flops": fl.value,
                         "bytes": by.value}
        return out


PROFILE_KINDS = ("qkv_gemm", "o_gemm", "fc1_gemm", "fc2_gemm", "attention", "head_gemm", "other")


_anchors: dict[int, tuple[Event, float]] = {}


def _anchor(device: int) -> tuple[Event, float]:
    """Per-device (anchor event, host perf_counter at its completion)."""
    a = _anchors.get(device)
    if a is None:
        ev = C.c_void_p()
        check(load().tk_event_anchor(device, C.byref(ev)), "tk_event_anchor")
        t0 = time.perf_counter()
        a = _anchors[device] = (Event(ev, device=device), t0)
        a[0]._done = True
    return a


def event_elapsed_ns(first: Event, last: Event) -> int:
    """Device time from first's start marker to last's end marker."""
    first.wait()
    last.wait()
    ns = C.c_int64()
    check(load().tk_event_elapsed(first._ptr, last._ptr, C.byref(ns)), "tk_event_elapsed")
    return ns.value


def launch_count() -> int:
    n = C.c_int64()
    check(load().tk_launch_count(C.byref(n)))
    return n.value


def host_alloc(nbytes: int) -> int:
    p = C.c_void_p()
    check(load().tk_host_alloc(nbytes, C.byref(p)), "tk_host_alloc")
    return p.value


def host_free(ptr: int) -> None:
    check(load().tk_host_free(C.c_void_p(ptr)), "tk_host_free")


def device_count() -> int:
    n = C.c_int32()
    check(load().tk_device_count(C.byref(n)), "tk_device_count")
    return n.value


def device_memory(device: int) -> tuple[int, int]:
    """(free, total) HBM bytes of ``device``."""
    f, t = C.c_int64(), C.c_int64()
    check(load().tk_device_memory(device, C.byref(f), C.byref(t)), "tk_device_memory")
    return f.value, t.value


# ---------------------------------------------------------------- raw kernels (torch tensors)

def _ptr(t) -> C.c_void_p:
    return C.c_void_p(0 if t is None else t.data_ptr())


def _stream(stream=None) -> C.c_void_p:
    if stream is None:
        import torch
        stream = torch.cuda.current_stream()
    return C.c_void_p(stream.cuda_stream)


def gemm(a, b, bias=None, epilogue: int = EPI_BF16, out=None, workspace=None, stream=None):
    """C = A[M,K] . B[N,K]^T with a fused epilogue, on the tcgen05 kernel."""
    import torch
    M, K = a.shape
    N = b.shape[0]
    if out is None:
        dt = torch.float32 if epilogue in (EPI_F32, EPI_F32_BIAS_RESID) else torch.bfloat16
        out = torch.zeros((M, N), dtype=dt, device=a.device)
    ws_bytes = C.c_int64()
    check(load().tk_gemm_workspace_bytes(M, N, K, C.byref(ws_bytes)))
    if workspace is None:
        workspace = torch.zeros(ws_bytes.value, dtype=torch.uint8, device=a.device)
    check(load().tk_gemm_bf16(_ptr(a), _ptr(b), _ptr(out), _ptr(bias), M, N, K, epilogue,
                              _ptr(workspace), workspace.numel(), _stream(stream)), "tk_gemm_bf16")
    return out


def layernorm(x, w, b, eps=1e-5, stream=None):
    import torch
    y = torch.empty(x.shape, dtype=torch.bfloat16, device=x.device)
    check(load().tk_layernorm(_ptr(x), _ptr(w), _ptr(b), _ptr(y), x.shape[0], x.shape[1], eps,
                              _stream(stream)), "tk_layernorm")
    return y


def argmax(logits, cols=None, stream=None):
    import torch
    rows, stride = logits.shape
    out = torch.empty(rows, dtype=torch.int32, device=logits.device)
    check(load().tk_argmax(_ptr(logits), rows, cols or stride, stride, _ptr(out), _stream(stream)),
          "tk_argmax")
    return out


def paged_decode_attention(q, pool, layer, n_layers, block_tables, ctx_lens, page_tokens=16,
                           scale=None, stream=None):
    import torch
    B, H, D = q.shape
    o = torch.empty_like(q)
    max_ctx = int(ctx_lens.max().item())
    splits = (max_ctx + 255) // 256
    ws = torch.empty(max(1, B * H * splits * (D + 2) * 4), dtype=torch.uint8, device=q.device)
    check(load().tk_paged_decode_attention(
        _ptr(q), _ptr(o), _ptr(pool), layer, n_layers, H, D, page_tokens, _ptr(block_tables),
        block_tables.shape[1], _ptr(ctx_lens), B, scale if scale else D ** -0.5, _ptr(ws),
        ws.numel(), _stream(stream)), "tk_paged_decode_attention")
    return o


def chunk_attention(q, q_stride, pool, layer, n_layers, n_heads, head_dim, slices, block_tables,
                    page_tokens=16, scale=None, stream=None):
    import torch
    n = sum(s[1] for s in slices)
    o = torch.empty((n, n_heads * head_dim), dtype=torch.bfloat16, device=q.device)
    sl = (tk_slice * len(slices))(*[tk_slice(*s) for s in slices])
    check(load().tk_chunk_attention(
        _ptr(q), q_stride, _ptr(o), _ptr(pool), layer, n_layers, n_heads, head_dim, page_tokens,
        sl, len(slices), i32(block_tables), n, scale if scale else head_dim ** -0.5,
        _stream(stream)), "tk_chunk_attention")
    return o


def chunk_attention_timed(q, q_stride, pool, layer, n_layers, n_heads, head_dim, slices,
                          block_tables, iters=20, page_tokens=16, scale=None, stream=None):
    """(o, mean device microseconds per launch) -- microbenchmarks only."""
    import torch
    n = sum(s[1] for s in slices)
    o = torch.empty((n, n_heads * head_dim), dtype=torch.bfloat16, device=q.device)
    sl = (tk_slice * len(slices))(*[tk_slice(*s) for s in slices])
    us = C.c_float()
    check(load().tk_chunk_attention_timed(
        _ptr(q), q_stride, _ptr(o), _ptr(pool), layer, n_layers, n_heads, head_dim, page_tokens,
        sl, len(slices), i32(block_tables), n, scale if scale else head_dim ** -0.5,
        _stream(stream), iters, C.byref(us)), "tk_chunk_attention_timed")
    return o, us.value


def fa_plan(slices, n_heads, max_ctas=148, span=256):
    """Chunk-attention work plan (host only): (pairs, units, cta_off, n_pieces).
    span 512: the CTA-pair kernel's quads, max_ctas counting 2-CTA clusters."""
    n = len(slices)
    n_tok = sum(sl[1] for sl in slices)
    pcap = n + n_tok // 256 + 1
    ucap = pcap * n_heads + max_ctas + 1
    counts = (C.c_int32 * 5)()
    pairs = (C.c_int32 * (pcap * 6))()
    units = (C.c_int32 * (ucap * 5))()
    off = (C.c_int32 * (max_ctas + 1))()
    sl = (tk_slice * n)(*[tk_slice(*x) for x in slices])
    check(load().tk_fa_plan(sl, n, n_heads, max_ctas, counts, pairs, pcap, units, ucap, off,
                            max_ctas + 1, span), "tk_fa_plan")
    n_pairs, n_units, n_ctas, n_pieces = counts[0], counts[1], counts[2], counts[3]
    return ([tuple(pairs[i * 6:(i + 1) * 6]) for i in range(n_pairs)],
            [tuple(units[i * 5:(i + 1) * 5]) for i in range(n_units)],
            list(off[:n_ctas + 1]), n_pieces)
