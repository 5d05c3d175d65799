"""Executor seam between the host scheduler and the device.

Every place the reference calls a cost-model stand-in (SURVEY.md §8(b)
"Callers") now calls the instance's executor:

=====================  ===================================  ==========================
actor call site        reference stand-in                   executor method
=====================  ===================================  ==========================
prefill.py chunk loop  costs.chunk_cost (prefill.py:353)    prefill_chunk
prefill.py round       sequential_predictor_cost (:344)     predict_round
prefill.py send_kv     costs.transfer_latency (:422)        kv_transfer
control.py reroute     costs.transfer_latency (:341)        kv_transfer(src=None)
prefill.py chunk done  (new: chunk-level KV streaming)      kv_stream
decode.py boundary     decode_iter_latency (:256-258)       decode_step
coupled.py boundary    mixed_iter_latency (:90-93)          mixed_step
=====================  ===================================  ==========================

``SimExecutor`` returns the reference's integer latencies (decision parity).
The CUDA executor (cuda_executor.py) returns device completion handles.
"""

from __future__ import annotations

from . import costs
from .costs import CostModelParams


class SimExecutor:
    """Cost-model clock: reproduces pdsim timing exactly."""

    def __init__(self, params: CostModelParams):
        self.params = params

    # lifecycle hooks (no device state in sim mode)
    def attach(self, inst) -> None:
        pass

    def detach(self, inst) -> None:
        pass

    def admit(self, inst, dreq) -> None:
        pass

    def admit_prompt(self, inst, req) -> None:
        pass

    def grow(self, inst, dreq, pages: int) -> None:
        pass

    def release(self, inst, dreq) -> None:
        pass

    def swap_out(self, inst, dreq) -> None:
        pass

    def swap_in(self, inst, dreq) -> None:
        pass

    def round_done(self, inst, requests) -> None:
        pass

    # device work
    def predict_round(self, inst, batch, predictor) -> int:
        if predictor.mode == "sequential":
            return costs.sequential_predictor_cost(inst.params)
        return 0

    def prefill_chunk(self, inst, chunk, starting: int, tax: bool, extra: int) -> int:
        return costs.chunk_cost(inst.params, starting, tax) + extra

    def kv_transfer(self, src_inst, req, dst: str) -> int:
        return costs.transfer_latency(self.params, req.prompt_len)

    def kv_stream(self, src_inst, req, dst: str, start: int, end: int, final: bool) -> int:
        """One part of a streamed handoff: prompt tokens [start, end)."""
        return costs.transfer_latency(self.params, end - start)

    def decode_step(self, inst, running, kv_tokens: int, swapped_out: int,
                    swapped_in: int) -> tuple[int, int]:
        p = inst.params
        us = costs.decode_iter_latency(p, len(running), kv_tokens) \
            + round(p.swap_penalty_us_per_page * (swapped_out + swapped_in))
        return us, us

    def mixed_step(self, inst, prefilling, running, prefill_tokens: int, kv_tokens: int,
                   swapped_out: int, swapped_in: int) -> tuple[int, int]:
        p = inst.params
        us = costs.mixed_iter_latency(p, prefill_tokens, len(running), kv_tokens,
                                      n_prefill=len(prefilling)) \
            + round(p.swap_penalty_us_per_page * (swapped_out + swapped_in))
        return us, us
