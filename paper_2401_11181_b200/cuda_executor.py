"""CUDA executor: the scheduler's decisions executed on B200s via libtetri.

Each scheduler instance (p{i}, d{i}, c{i}) gets a device-side ``native.Instance``
(weights shared per device/model/seed, its own page-major KV pool and streams).
The executor keeps the *physical* side of the KV cache consistent with the
scheduler's page *counts* (PagedKvStore, pdsim/decode.py:41-95):

* prefill: a request's prompt pages are allocated from the prefill pool when
  its first slice is scheduled (pdsim/prefill.py:355-357) and freed when its
  KV handoff to the decode instance completes;
* handoff (pdsim/prefill.py:420-424): ``tk_kv_send`` copies the prompt pages
  page-by-page into pages of the destination pool (NVLink P2P across GPUs,
  a device copy when co-located).  Pages of a request that has arrived but is
  not yet admitted live in a receive staging area of the decode pool, outside
  ``mem_capacity_tokens`` (SURVEY.md §7 "KV residency");
* admission turns the staged pages into resident pages without a copy; next-
  token growth allocates pages (pdsim/decode.py:298-311); swap-out copies the
  victim's pages to pinned host memory and frees them (pdsim/decode.py:313-334);
  swap-in restores them into freshly allocated pages;
* a decode step feeds each running request its last token at position
  ``kv_tokens`` (prompt + generated) in ``running`` order
  (pdsim/decode.py:255-256) and keeps the greedy next tokens.

Length predictor: buckets come from the statistical PredictorModel on the
reference's "predictor" stream (decision parity; random-init weights carry no
signal), while the OPT-125M-class classifier runs on the prefill GPU for its
real cost -- concurrently on the predictor stream in ``parallel`` mode, before
the round's first chunk in ``sequential`` mode (pdsim/prefill.py:338-346).
"""

from __future__ import annotations

import time
from dataclasses import dataclass, field

from . import costs, native
from .engine import SimulationError
from .workload import Request, token_ids_for


@dataclass
class _Pool:
    """Physical page ids of one instance's KV pool."""

    n_pages: int
    free: list[int] = field(default_factory=list)

    def __post_init__(self):
        self.free = list(range(self.n_pages - 1, -1, -1))

    def take(self, n: int, who: str) -> list[int]:
        if n > len(self.free):
            raise SimulationError(f"{who}: physical KV pool exhausted ({n} pages wanted, "
                                  f"{len(self.free)} free of {self.n_pages})")
        return [self.free.pop() for _ in range(n)]

    def give(self, pages: list[int]) -> None:
        self.free.extend(reversed(pages))


def place_instance(iid: str, n_prefill: int, n_dev: int, overrides: dict | None = None) -> int:
    """CUDA ordinal of scheduler instance ``iid`` (p{i}, d{i}, c{i}).

    Prefill instances take the first ordinals, decode instances the next ones
    (2:6 on 8 GPUs -> p0,p1 on 0,1 and d0..d5 on 2..7), wrapping round-robin
    when there are fewer devices than instances (1 GPU: co-located).  An
    explicit ``devices`` map in the config wins.
    """
    if overrides and iid in overrides:
        return int(overrides[iid]) % n_dev
    kind, idx = iid[0], int(iid[1:])
    if kind in ("p", "c"):
        return idx % n_dev
    return (n_prefill + idx) % n_dev


class _Done:
    """A completion handle that is already complete (no device work)."""

    def done(self) -> bool:
        return True


class _Then:
    """Device handle plus a host callback run once when it completes."""

    def __init__(self, ev: native.Event, fn):
        self.ev, self.fn, self.fired = ev, fn, False

    def done(self) -> bool:
        if self.ev.done():
            if not self.fired:
                self.fired = True
                self.fn()
            return True
        return False

    def wait(self):
        self.ev.wait()
        return self.done()

    def done_time(self):
        return self.ev.done_time()


class CudaExecutor:
    """Executor protocol of executor.py on real devices."""

    def __init__(self, config, requests: list[Request] | None = None):
        native.load()
        self.config = config
        self.params = config.params
        mcfg = dict(config.model)
        self.shape = native.MODELS[mcfg.get("name", "opt-13b")]
        self.seed = int(mcfg.get("seed", 0))
        self.page_tokens = self.params.page_size
        n_dev = native.device_count()
        if n_dev < 1:
            raise native.NativeError("CudaExecutor needs at least one CUDA device")
        self.n_dev = n_dev
        self.devices = dict(config.devices)
        # pools (pages); defaults fit OPT-13B co-located on one 180 GB B200
        self.prefill_pages = int(mcfg.get("prefill_pages", 2048))
        self.staging_pages = int(mcfg.get("staging_pages", 512))
        self.max_batch = int(mcfg.get("max_decode_batch", 256))
        self.device_predictor = bool(mcfg.get("device_predictor", True))
        # handoff engine: "auto" (SM page-copy kernel on one device, copy engines
        # over NVLink across devices),
        # "sm", or "ce" (copy engines, leaves the SMs to the next chunk)
        self.send_engine = str(mcfg.get("kv_send_engine", "auto"))
        if self.send_engine not in native.SEND_ENGINES:
            raise ValueError(f"model.kv_send_engine must be one of {sorted(native.SEND_ENGINES)}")
        self.insts: dict[str, native.Instance] = {}
        self.pools: dict[str, _Pool] = {}
        self.tables: dict[str, dict[int, list[int]]] = {}   # inst -> req -> pages
        self.kv_home: dict[int, str] = {}                     # req -> instance holding its KV
        self.first_token: dict[int, int] = {}
        self.last_token: dict[int, int] = {}
        self.swap_host: dict[int, tuple[int, int]] = {}       # req -> (pinned ptr, pages)
        # receive staging (arrived, not yet admitted): pages held per decode instance,
        # bounded by staging_pages; beyond it the KV waits in pinned host memory
        self.staged: dict[str, int] = {}                      # inst -> staged pages
        self.staged_of: dict[int, int] = {}                   # req -> its staged pages
        self.host_staged: set[int] = set()                    # reqs staged in host memory
        self._streams: dict[int, dict] = {}                   # req -> streamed handoff state
        self.predictors: dict[int, native.Instance] = {}
        self.prompts: dict[int, list[int]] = {}
        self.stats = {"prefill_tokens": 0, "prefill_chunks": 0, "decode_steps": 0,
                      "decode_tokens": 0, "kv_bytes_sent": 0, "prefill_device_ns": 0,
                      "decode_device_ns": 0, "handoff_device_ns": 0, "predict_calls": 0,
                      "flips": 0, "flip_host_us": 0.0}
        self._req_by_id: dict[int, Request] = {r.id: r for r in (requests or [])}
        # every generated token per request (first token, then one per decode step);
        # kept when ``model.record_tokens`` is set (replay runs check them)
        self.token_log: dict[int, list[int]] | None = {} if mcfg.get("record_tokens") else None
        if mcfg.get("capacity_from_hbm"):
            self._size_capacity_from_hbm(float(mcfg.get("hbm_reserve_gb", 6.0)))

    def _size_capacity_from_hbm(self, reserve_gb: float) -> None:
        """Decode KV capacity (``mem_capacity_tokens``, pdsim/costs.py:46) from the
        free HBM of the decode GPUs: on each device
        that holds a decode instance, free memory minus the weights (once per
        device), the co-located prefill pools, each instance's receive staging
        and scratch, and a reserve, divided among its decode instances.  The
        smallest per-instance figure is every decode instance's capacity (the
        cost model has one).  run_experiment builds the executor first and hands
        the scheduler ``executor.params``."""
        import dataclasses
        cfg = self.config
        ids = ([f"p{i}" for i in range(cfg.n_prefill)] + [f"d{i}" for i in range(cfg.n_decode)])
        on: dict[int, list[str]] = {}
        for iid in ids:
            on.setdefault(self._device_of(iid), []).append(iid)
        pb = self.shape.kv_bytes_per_token * self.page_tokens
        weights = 2 * self.shape.params
        best = None
        for dev, here in on.items():
            n_dec = sum(1 for i in here if i[0] == "d")
            if not n_dec:
                continue
            free, _ = native.device_memory(dev)
            avail = free - weights - reserve_gb * 1e9
            avail -= sum(1 for i in here if i[0] == "p") * (self.prefill_pages * pb + 2e9)
            per = avail / n_dec - self.staging_pages * pb - 2e9
            pages = int(per // pb)
            best = pages if best is None else min(best, pages)
        if best is None:
            return
        if best < 64:
            raise native.NativeError(f"capacity_from_hbm: only {best} KV pages fit on the decode GPUs")
        tokens = best * self.page_tokens
        self.params = dataclasses.replace(self.params, mem_capacity_tokens=tokens)

    # -- lifecycle ---------------------------------------------------------------------
    def _device_of(self, iid: str) -> int:
        return place_instance(iid, self.config.n_prefill, self.n_dev, self.devices)

    device_of = _device_of

    def attach(self, inst) -> None:
        dev = self._device_of(inst.id)
        if inst.id in self.insts:
            # Instance flip (pdsim/control.py:408-482): the role changes, the device
            # state stays -- weights, KV pool, streams and page tables are reused
            # as they are (the pool was sized for both roles), so nothing is
            # reloaded or reallocated.  The pages still in flight of a drained
            # prefill instance come back to the same pool when their copies end.
            t0 = time.perf_counter()
            self._ensure_predictor(inst, dev)
            self.stats["flips"] += 1
            self.stats["flip_host_us"] += (time.perf_counter() - t0) * 1e6
            return
        flips = self.config.flip_policy.enabled
        if inst.role == "prefill" and not flips:
            pages, max_rows = self.prefill_pages, self.params.chunk_size
        elif inst.role == "decode" and not flips:
            pages, max_rows = self.params.capacity_pages + self.staging_pages, self.max_batch
        else:  # coupled (prefill + decode share one pool), or either role after a flip
            pages = max(self.params.capacity_pages + self.staging_pages,
                        self.prefill_pages if flips else 0)
            max_rows = max(self.params.chunk_size, self.max_batch)
        self.insts[inst.id] = native.Instance(self.shape, device=dev, seed=self.seed,
                                              kv_pages=pages, page_tokens=self.page_tokens,
                                              max_chunk=max_rows)
        self.pools[inst.id] = _Pool(pages)
        self.tables[inst.id] = {}
        self._ensure_predictor(inst, dev)

    def _ensure_predictor(self, inst, dev: int) -> None:
        if inst.role == "prefill" and self.device_predictor and dev not in self.predictors:
            self.predictors[dev] = native.Instance(native.PREDICTOR_125M, device=dev,
                                                   seed=self.seed + 1, kv_pages=16 * 32 + 8,
                                                   max_chunk=16 * 512)

    def detach(self, inst) -> None:
        pass  # device state is kept; the flipped id re-attaches with its new role

    def close(self) -> None:
        for i in list(self.insts.values()) + list(self.predictors.values()):
            i.close()
        for ptr, _ in self.swap_host.values():
            native.host_free(ptr)
        self.swap_host.clear()

    def _ids(self, req: Request) -> list[int]:
        ids = self.prompts.get(req.id)
        if ids is None:
            ids = self.prompts[req.id] = token_ids_for(req, self.shape.vocab, self.seed)
        return ids

    # -- prefill side -----------------------------------------------------------------------
    def predict_round(self, inst, batch, predictor) -> object:
        """Device classifier over the round's prompts (cost); buckets stay statistical."""
        dev = self._device_of(inst.id)
        pred = self.predictors.get(dev)
        if pred is None or not batch:
            return 0
        max_len = 512
        ids, lens = [], []
        for r in batch:
            toks = self._ids(r)[:max_len]
            ids += toks
            lens.append(len(toks))
        ev, _ = pred.predict(ids, lens, max_len)
        self.stats["predict_calls"] += 1
        if predictor.mode == "sequential":
            ev.wait()  # the round's first chunk starts after the predictor pass
        return 0

    def prefill_chunk(self, inst, chunk, starting: int, tax: bool, extra) -> object:
        dev_inst = self.insts[inst.id]
        pool = self.pools[inst.id]
        tables = self.tables[inst.id]
        ids, slices, bt = [], [], []
        emit_rids = []
        for rid, start, n in chunk.slices:
            req = inst.requests[rid]
            if start == 0:
                tables[rid] = pool.take(costs.pages_needed(self.params, req.prompt_len), inst.id)
                self.kv_home[rid] = inst.id
            ids += self._ids(req)[start:start + n]
            emit = int(start + n == req.prompt_len)
            slices.append((start, n, len(bt), len(tables[rid]), emit))
            bt += tables[rid]
            if emit:
                emit_rids.append((len(slices) - 1, rid))
        ev, out = dev_inst.prefill_chunk(ids, slices, bt)
        self.stats["prefill_tokens"] += len(ids)
        self.stats["prefill_chunks"] += 1

        def publish():
            for idx, rid in emit_rids:
                self._emit(rid, int(out[idx]), first=True)
            self.stats["prefill_device_ns"] += ev.elapsed_ns

        return _Then(ev, publish)

    def _emit(self, rid: int, tok: int, first: bool = False) -> None:
        if first:
            self.first_token[rid] = tok
        self.last_token[rid] = tok
        if self.token_log is not None:
            if first:
                self.token_log[rid] = [tok]
            else:
                self.token_log[rid].append(tok)

    def round_done(self, inst, requests) -> None:
        pass

    def kv_transfer(self, src_inst, req: Request, dst: str) -> object:
        src_id = self.kv_home.get(req.id) if src_inst is None else src_inst.id
        if src_id is None or req.id not in self.tables.get(src_id, {}):
            raise SimulationError(f"request {req.id}: no KV to transfer")
        src_pages = self.tables[src_id].pop(req.id)
        self.kv_home[req.id] = dst
        nbytes = len(src_pages) * self.insts[src_id].page_bytes
        if not self._stage_on_device(dst, req.id, len(src_pages)):
            # receive staging full (arrivals queue without bound in pdsim's decode
            # instance): park the KV in pinned host memory; admission restores it
            ptr = native.host_alloc(nbytes)
            ev = self.insts[src_id].swap_out(src_pages, ptr)
            self.swap_host[req.id] = (ptr, len(src_pages))
            self.host_staged.add(req.id)
            self.stats["kv_host_staged"] = self.stats.get("kv_host_staged", 0) + 1

            def release_src_host():
                self.pools[src_id].give(src_pages)

            return _Then(ev, release_src_host)
        dst_pages = self.pools[dst].take(len(src_pages), dst)  # receive staging
        self.tables[dst][req.id] = dst_pages
        ev = self.insts[src_id].kv_send(src_pages, self.insts[dst], dst_pages, self.send_engine)
        self.stats["kv_bytes_sent"] += nbytes

        def release_src():
            self.pools[src_id].give(src_pages)
            self.stats["handoff_device_ns"] += ev.elapsed_ns

        return _Then(ev, release_src)

    def kv_stream(self, src_inst, req: Request, dst: str, start: int, end: int,
                  final: bool) -> object:
        """Chunk-level KV streaming: copy the pages of prompt tokens [start, end)
        that are complete (a page straddling ``end`` goes with the next part) to
        pages reserved in ``dst``'s receive staging on the first part.  Parts run
        in order on the source's copy stream, each after the chunk that wrote it."""
        src_id = src_inst.id
        src_pages = self.tables[src_id][req.id]
        pb = self.insts[src_id].page_bytes
        st = self._streams.get(req.id)
        if st is None:
            st = self._streams[req.id] = {"sent": 0, "parts": []}
            if self._stage_on_device(dst, req.id, len(src_pages)):
                st["dst"] = self.pools[dst].take(len(src_pages), dst)
                self.tables[dst][req.id] = st["dst"]
            else:  # staging full: the parts collect in one pinned host buffer
                st["host"] = native.host_alloc(len(src_pages) * pb)
        hi = len(src_pages) if final else end // self.page_tokens
        lo = st["sent"]
        if "host" in st:
            ev = self.insts[src_id].swap_out(src_pages[lo:hi], st["host"] + lo * pb)
        else:
            ev = self.insts[src_id].kv_send(src_pages[lo:hi], self.insts[dst], st["dst"][lo:hi],
                                            self.send_engine)
        st["sent"] = max(lo, hi)
        nbytes = max(0, hi - lo) * pb
        self.stats["kv_bytes_sent"] += nbytes
        if not final:
            # keep the part's handle: the copy runs behind the next chunks
            st["parts"].append(ev)
            return ev
        del self._streams[req.id]
        self.tables[src_id].pop(req.id)
        self.kv_home[req.id] = dst
        if "host" in st:
            self.swap_host[req.id] = (st["host"], len(src_pages))
            self.host_staged.add(req.id)
            self.stats["kv_host_staged"] = self.stats.get("kv_host_staged", 0) + 1

        parts = st["parts"]

        def release_src():
            self.pools[src_id].give(src_pages)
            # every part's copy time, not only the final part's
            self.stats["handoff_device_ns"] += ev.elapsed_ns + sum(e.wait() for e in parts)

        return _Then(ev, release_src)

    # -- decode side ----------------------------------------------------------------------------
    def _stage_on_device(self, dst: str, rid: int, n: int) -> bool:
        """Reserve ``n`` receive-staging pages of ``dst`` for request ``rid``."""
        if self.staged.get(dst, 0) + n > self.staging_pages:
            return False
        self.staged[dst] = self.staged.get(dst, 0) + n
        self.staged_of[rid] = n
        return True

    def admit(self, inst, dreq) -> None:
        # staged pages become resident pages: the counts check happened in the store
        rid = dreq.req.id
        if rid in self.staged_of:
            self.staged[inst.id] -= self.staged_of.pop(rid)
        if rid in self.host_staged:  # KV parked in pinned host memory on arrival
            self.host_staged.discard(rid)
            self.swap_in(inst, dreq)
        have = self.tables[inst.id].get(dreq.req.id)
        need = costs.pages_needed(self.params, dreq.kv_tokens)
        if have is None:
            self.tables[inst.id][dreq.req.id] = self.pools[inst.id].take(need, inst.id)
        elif len(have) < need:
            have += self.pools[inst.id].take(need - len(have), inst.id)

    def grow(self, inst, dreq, pages: int) -> None:
        t = self.tables[inst.id][dreq.req.id]
        if pages > len(t):
            t += self.pools[inst.id].take(pages - len(t), inst.id)

    def release(self, inst, dreq) -> None:
        pages = self.tables[inst.id].pop(dreq.req.id, [])
        self.pools[inst.id].give(pages)
        self.kv_home.pop(dreq.req.id, None)

    def swap_out(self, inst, dreq) -> None:
        pages = self.tables[inst.id].pop(dreq.req.id)
        dev = self.insts[inst.id]
        ptr = native.host_alloc(len(pages) * dev.page_bytes)
        dev.swap_out(pages, ptr).wait()  # pages are reused right away by the grower
        self.swap_host[dreq.req.id] = (ptr, len(pages))
        self.pools[inst.id].give(pages)

    def swap_in(self, inst, dreq) -> None:
        ptr, n = self.swap_host.pop(dreq.req.id)
        pages = self.pools[inst.id].take(n, inst.id)
        self.insts[inst.id].swap_in(pages, ptr).wait()
        native.host_free(ptr)
        self.tables[inst.id][dreq.req.id] = pages

    def decode_step(self, inst, running, kv_tokens: int, swapped_out: int,
                    swapped_in: int) -> tuple[object, int]:
        p = inst.params
        modeled = costs.decode_iter_latency(p, len(running), kv_tokens) \
            + round(p.swap_penalty_us_per_page * (swapped_out + swapped_in))
        dev = self.insts[inst.id]
        tables = self.tables[inst.id]
        stride = max(len(tables[d.req.id]) for d in running)
        bt, last, ctx = [], [], []
        for d in running:
            t = tables[d.req.id]
            bt += t + [t[0]] * (stride - len(t))
            last.append(self.last_token.get(d.req.id, 0))
            ctx.append(d.kv_tokens)
        if len(running) > dev.max_chunk:
            raise SimulationError(f"{inst.id}: decode batch {len(running)} exceeds the device "
                                  f"batch capacity {dev.max_chunk}")
        ev, out = dev.decode_step(last, ctx, bt, stride)
        rids = [d.req.id for d in running]
        self.stats["decode_steps"] += 1
        self.stats["decode_tokens"] += len(rids)

        def publish():
            for i, rid in enumerate(rids):
                self._emit(rid, int(out[i]))
            self.stats["decode_device_ns"] += ev.elapsed_ns

        return _Then(ev, publish), modeled

    # -- coupled (vLLM-like) baseline: prefill and decode share one instance ------------
    def admit_prompt(self, inst, req: Request) -> None:
        self.tables[inst.id][req.id] = self.pools[inst.id].take(
            costs.pages_needed(self.params, req.prompt_len), inst.id)
        self.kv_home[req.id] = inst.id

    def mixed_step(self, inst, prefilling, running, prefill_tokens, kv_tokens, swapped_out,
                   swapped_in):
        """One coupled iteration (pdsim/coupled.py:82-101): the running batch decodes
        one token, then the admitted prompts are prefilled whole (in device chunks of
        the instance's row capacity); the iteration ends when both are done."""
        from .prefill import chunkify
        p = inst.params
        modeled = costs.mixed_iter_latency(p, prefill_tokens, len(running), kv_tokens,
                                           n_prefill=len(prefilling)) \
            + round(p.swap_penalty_us_per_page * (swapped_out + swapped_in))
        dev = self.insts[inst.id]
        tables = self.tables[inst.id]
        pending = []
        if running:
            stride = max(len(tables[d.req.id]) for d in running)
            bt, last, ctx = [], [], []
            for d in running:
                t = tables[d.req.id]
                bt += t + [t[0]] * (stride - len(t))
                last.append(self.last_token.get(d.req.id, 0))
                ctx.append(d.kv_tokens)
            ev, out = dev.decode_step(last, ctx, bt, stride)
            rids = [d.req.id for d in running]
            pending.append((ev, lambda out=out, rids=rids: [
                self._emit(r, int(out[i])) for i, r in enumerate(rids)]))
            self.stats["decode_steps"] += 1
            self.stats["decode_tokens"] += len(rids)
        by_id = {r.id: r for r in prefilling}
        for chunk in chunkify(list(prefilling), dev.max_chunk):
            ids, slices, bt, emit = [], [], [], []
            for rid, start, n in chunk.slices:
                req = by_id[rid]
                ids += self._ids(req)[start:start + n]
                e = int(start + n == req.prompt_len)
                slices.append((start, n, len(bt), len(tables[rid]), e))
                bt += tables[rid]
                if e:
                    emit.append((len(slices) - 1, rid))
            ev, out = dev.prefill_chunk(ids, slices, bt)
            pending.append((ev, lambda out=out, emit=emit: [
                self._emit(r, int(out[i]), first=True) for i, r in emit]))
            self.stats["prefill_tokens"] += len(ids)
            self.stats["prefill_chunks"] += 1
        if not pending:
            return _Done(), modeled
        last_ev = pending[-1][0]

        def publish():
            for ev, fn in pending:
                ev.wait()
                fn()

        return _Then(last_ev, publish), modeled

    # -- reporting ---------------------------------------------------------------------------------
    def summary_extras(self) -> dict:
        s = dict(self.stats)
        s["model"] = self.shape.name
        s["devices"] = {k: self._device_of(k) for k in self.insts}
        s["mem_capacity_tokens"] = self.params.mem_capacity_tokens
        if s["prefill_device_ns"]:
            s["prefill_tok_s_device"] = s["prefill_tokens"] / (s["prefill_device_ns"] / 1e9)
        if s["decode_device_ns"]:
            s["decode_tok_s_device"] = s["decode_tokens"] / (s["decode_device_ns"] / 1e9)
        if s["handoff_device_ns"]:
            s["handoff_gb_s"] = s["kv_bytes_sent"] / s["handoff_device_ns"]
        return s


class ReplayExecutor(CudaExecutor):
    """Replay mode (SURVEY.md section 7 mode 2; ``executor: "replay"``): the
    engine runs on pdsim's modeled clock, so every placement, chunk layout and
    batch is the reference's own decision (the SimExecutor latencies,
    pdsim/costs.py), while each decision is executed on the device -- every
    chunk, handoff, swap and decode step -- synchronously, before its modeled
    completion is scheduled.  The run therefore reproduces pdsim's decision trace
    exactly *and* produces the tokens those decisions generate on the GPU
    (``token_log``), which tests check against the fp32 oracle.  The device
    model only executes: the cost model keeps the reference's constants
    (kv_bytes_per_token, capacity), so any model shape can replay any config."""

    def __init__(self, config, requests=None):
        import dataclasses

        from .executor import SimExecutor
        mcfg = dict(config.model)
        mcfg.pop("capacity_from_hbm", None)
        mcfg.setdefault("record_tokens", True)
        super().__init__(dataclasses.replace(config, model=mcfg), requests)
        self.sim = SimExecutor(config.params)

    @staticmethod
    def _finish(handle) -> None:
        wait = getattr(handle, "wait", None)
        if wait is not None:
            wait()
        else:
            handle.done()

    def predict_round(self, inst, batch, predictor) -> int:
        super().predict_round(inst, batch, predictor)
        return self.sim.predict_round(inst, batch, predictor)

    def prefill_chunk(self, inst, chunk, starting: int, tax: bool, extra) -> int:
        self._finish(super().prefill_chunk(inst, chunk, starting, tax, extra))
        return self.sim.prefill_chunk(inst, chunk, starting, tax, extra)

    def kv_transfer(self, src_inst, req: Request, dst: str) -> int:
        self._finish(super().kv_transfer(src_inst, req, dst))
        return self.sim.kv_transfer(src_inst, req, dst)

    def kv_stream(self, src_inst, req: Request, dst: str, start: int, end: int,
                  final: bool) -> int:
        self._finish(super().kv_stream(src_inst, req, dst, start, end, final))
        return self.sim.kv_stream(src_inst, req, dst, start, end, final)

    def decode_step(self, inst, running, kv_tokens: int, swapped_out: int,
                    swapped_in: int) -> tuple[int, int]:
        handle, modeled = super().decode_step(inst, running, kv_tokens, swapped_out, swapped_in)
        self._finish(handle)
        return modeled, modeled

    def mixed_step(self, inst, prefilling, running, prefill_tokens, kv_tokens, swapped_out,
                   swapped_in) -> tuple[int, int]:
        handle, modeled = super().mixed_step(inst, prefilling, running, prefill_tokens,
                                             kv_tokens, swapped_out, swapped_in)
        self._finish(handle)
        return modeled, modeled
