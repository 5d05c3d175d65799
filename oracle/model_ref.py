"""fp32 CPU oracle of the device forward (TEST INFRASTRUCTURE ONLY).

Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline / reference
legs may import this module, and only as the checker or the timed CPU
baseline -- never as the product path.

What it restates
----------------
The reference (pdsim) has no numeric path: its chunk forward, decode step and
predictor are cost-model stand-ins (pdsim/costs.py:142-152, :104-109,
pdsim/prefill.py:99-109; SPEC.md:20 puts kernels out of scope).  The paper's
system ran OPT-13B / OPT-125M through vLLM and HuggingFace (PAPER.md:78,
:544-545, :593-594).  This oracle therefore restates the HuggingFace
semantics of those models, following transformers 5.5.0
(site-packages/transformers/models/opt/modeling_opt.py and
models/llama/modeling_llama.py):

* OPT: learned positions at index pos + 2 (modeling_opt.py:45-70), pre-LN
  blocks (do_layer_norm_before, :214-250), q scaled by head_dim**-0.5 after
  the bias (:128, :151), ReLU fc1/fc2 with biases (:198-199), final
  LayerNorm, LM head tied to embed_tokens without bias (:444, :451);
  sequence classification pools the last token and applies ``score`` without
  bias (:546, :590-603).
* Llama: RMSNorm, rotate-half RoPE, SwiGLU, no biases, untied lm_head.

and the chunked-prefill execution the device performs: prompts split into
the pdsim chunk layout (pdsim/prefill.py:140-165), each chunk's K/V written
into 16-token pages, each query attending causally to its request's pages.

Pinning: tests/test_oracle.py checks this module against transformers'
OPTForCausalLM / OPTForSequenceClassification / LlamaForCausalLM on the
same weights (the numeric parity is otherwise unpinned by the reference,
SURVEY.md §8(c)).
"""

from __future__ import annotations

from dataclasses import dataclass, field

import numpy as np
import torch

ARCH_OPT, ARCH_LLAMA = 0, 1


def bf16_bits_to_f32(bits: np.ndarray) -> torch.Tensor:
    """uint16 bf16 payload -> fp32 tensor (exact)."""
    b = np.ascontiguousarray(bits, dtype=np.uint16).astype(np.uint32) << 16
    return torch.from_numpy(b.view(np.float32).copy())


def f32_to_bf16_bits(t: torch.Tensor) -> np.ndarray:
    return t.to(torch.bfloat16).view(torch.int16).numpy().view(np.uint16)


@dataclass
class Shape:
    arch: int
    n_layers: int
    hidden: int
    n_heads: int
    ffn: int
    vocab: int
    max_positions: int = 2048
    n_labels: int = 0
    norm_eps: float = 1e-5
    rope_theta: float = 10000.0

    @property
    def head_dim(self) -> int:
        return self.hidden // self.n_heads


def weight_names(s: Shape) -> list[str]:
    """Tensor names in the device runtime's order (runtime.cu weight_specs)."""
    n = ["embed_tokens.weight"]
    if s.arch == ARCH_OPT:
        n.append("embed_positions.weight")
    for l in range(s.n_layers):
        p = f"layers.{l}."
        if s.arch == ARCH_OPT:
            n += [p + x for x in ("self_attn_layer_norm.weight", "self_attn_layer_norm.bias",
                                  "self_attn.qkv_proj.weight", "self_attn.qkv_proj.bias",
                                  "self_attn.out_proj.weight", "self_attn.out_proj.bias",
                                  "final_layer_norm.weight", "final_layer_norm.bias",
                                  "fc1.weight", "fc1.bias", "fc2.weight", "fc2.bias")]
        else:
            n += [p + x for x in ("input_layernorm.weight", "self_attn.qkv_proj.weight",
                                  "self_attn.o_proj.weight", "post_attention_layernorm.weight",
                                  "mlp.gate_up_proj.weight", "mlp.down_proj.weight")]
    n += (["final_layer_norm.weight", "final_layer_norm.bias"] if s.arch == ARCH_OPT
          else ["norm.weight"])
    if s.n_labels:
        n.append("score.weight")
    elif s.arch == ARCH_LLAMA:
        n.append("lm_head.weight")
    return n


def weight_shapes(s: Shape) -> dict[str, tuple[int, ...]]:
    h, f = s.hidden, s.ffn
    out: dict[str, tuple[int, ...]] = {"embed_tokens.weight": (s.vocab, h)}
    if s.arch == ARCH_OPT:
        out["embed_positions.weight"] = (s.max_positions + 2, h)
    for l in range(s.n_layers):
        p = f"layers.{l}."
        if s.arch == ARCH_OPT:
            out.update({p + "self_attn_layer_norm.weight": (h,), p + "self_attn_layer_norm.bias": (h,),
                        p + "self_attn.qkv_proj.weight": (3 * h, h), p + "self_attn.qkv_proj.bias": (3 * h,),
                        p + "self_attn.out_proj.weight": (h, h), p + "self_attn.out_proj.bias": (h,),
                        p + "final_layer_norm.weight": (h,), p + "final_layer_norm.bias": (h,),
                        p + "fc1.weight": (f, h), p + "fc1.bias": (f,),
                        p + "fc2.weight": (h, f), p + "fc2.bias": (h,)})
        else:
            out.update({p + "input_layernorm.weight": (h,), p + "self_attn.qkv_proj.weight": (3 * h, h),
                        p + "self_attn.o_proj.weight": (h, h),
                        p + "post_attention_layernorm.weight": (h,),
                        p + "mlp.gate_up_proj.weight": (2 * f, h),
                        p + "mlp.down_proj.weight": (h, f)})
    if s.arch == ARCH_OPT:
        out["final_layer_norm.weight"] = (h,)
        out["final_layer_norm.bias"] = (h,)
    else:
        out["norm.weight"] = (h,)
    if s.n_labels:
        out["score.weight"] = ((s.n_labels + 7) // 8 * 8, h)
    elif s.arch == ARCH_LLAMA:
        out["lm_head.weight"] = (s.vocab, h)
    return out


@dataclass
class PagedCache:
    """fp32 mirror of the device KV pool: pages[page][layer][kv][head][slot][dim]."""

    shape: Shape
    n_pages: int
    page_tokens: int = 16
    device: str = "cpu"
    pages: torch.Tensor = field(init=False)

    def __post_init__(self):
        s = self.shape
        self.pages = torch.zeros(self.n_pages, s.n_layers, 2, s.n_heads, self.page_tokens,
                                 s.head_dim, device=self.device)

    def write(self, layer: int, table: list[int], positions: torch.Tensor, k: torch.Tensor,
              v: torch.Tensor) -> None:
        pt = self.page_tokens
        pos = positions.to(self.device)
        page = torch.tensor(table, dtype=torch.long, device=self.device)[pos // pt]
        slot = pos % pt
        self.pages[page, layer, 0, :, slot] = k
        self.pages[page, layer, 1, :, slot] = v

    def read(self, layer: int, table: list[int], n: int) -> tuple[torch.Tensor, torch.Tensor]:
        idx = torch.tensor(table[: (n + self.page_tokens - 1) // self.page_tokens],
                           device=self.device)
        kv = self.pages[idx, layer]  # [np, 2, H, pt, D]
        k = kv[:, 0].permute(1, 0, 2, 3).reshape(self.shape.n_heads, -1, self.shape.head_dim)[:, :n]
        v = kv[:, 1].permute(1, 0, 2, 3).reshape(self.shape.n_heads, -1, self.shape.head_dim)[:, :n]
        return k, v


class OracleModel:
    """fp32 forward with the device's chunked, paged execution order."""

    def __init__(self, shape: Shape, weights: dict[str, torch.Tensor], device: str = "cpu"):
        self.s = shape
        self.device = device
        self.w = {k: v.float().to(device) for k, v in weights.items()}

    @classmethod
    def from_instance(cls, shape: Shape, inst, device: str = "cpu") -> "OracleModel":
        """Weights read back from a device instance.  ``device="cuda"`` runs the
        same fp32 arithmetic on the GPU (TF32 off) so the OPT-13B-width parity
        tests finish in seconds; it is still the checker, never the product."""
        if device != "cpu":
            torch.backends.cuda.matmul.allow_tf32 = False
            torch.backends.cudnn.allow_tf32 = False
        ws = weight_shapes(shape)
        return cls(shape, {n: bf16_bits_to_f32(inst.read_weight(n)).view(ws[n]) for n in ws},
                   device)

    # -- pieces ----------------------------------------------------------------
    def _norm(self, x, prefix):
        s = self.s
        if s.arch == ARCH_OPT:
            return torch.nn.functional.layer_norm(x, (s.hidden,), self.w[prefix + ".weight"],
                                                  self.w[prefix + ".bias"], s.norm_eps)
        var = x.pow(2).mean(-1, keepdim=True)
        return x * torch.rsqrt(var + s.norm_eps) * self.w[prefix + ".weight"]

    def _rope(self, x, pos):  # x [n, H, D]
        D = self.s.head_dim
        inv = self.s.rope_theta ** (-torch.arange(0, D, 2, dtype=torch.float32,
                                                  device=x.device) / D)
        ang = pos[:, None].float() * inv[None, :]
        cos, sin = torch.cat([ang.cos()] * 2, -1)[:, None], torch.cat([ang.sin()] * 2, -1)[:, None]
        x1, x2 = x[..., : D // 2], x[..., D // 2:]
        return x * cos + torch.cat([-x2, x1], -1) * sin

    def embed(self, ids: torch.Tensor, pos: torch.Tensor) -> torch.Tensor:
        x = self.w["embed_tokens.weight"][ids]
        if self.s.arch == ARCH_OPT:
            x = x + self.w["embed_positions.weight"][pos + 2]
        return x

    def layer(self, l: int, x: torch.Tensor, rows, cache: PagedCache) -> torch.Tensor:
        """rows: list of (table, positions tensor, row slice) per request in the batch."""
        s, w, p = self.s, self.w, f"layers.{l}."
        H, D, h = s.n_heads, s.head_dim, s.hidden
        opt = s.arch == ARCH_OPT
        xn = self._norm(x, p + ("self_attn_layer_norm" if opt else "input_layernorm"))
        qkv = xn @ w[p + "self_attn.qkv_proj.weight"].t()
        if opt:
            qkv = qkv + w[p + "self_attn.qkv_proj.bias"]
        q, k, v = qkv[:, :h].view(-1, H, D), qkv[:, h:2 * h].view(-1, H, D), qkv[:, 2 * h:].view(-1, H, D)
        attn = torch.empty_like(q)
        for table, pos, sl in rows:
            qi, ki = q[sl], k[sl]
            if not opt:
                qi, ki = self._rope(qi, pos), self._rope(ki, pos)
            cache.write(l, table, pos, ki, v[sl])
            n_ctx = int(pos[-1]) + 1
            K, V = cache.read(l, table, n_ctx)
            sc = torch.einsum("qhd,hkd->hqk", qi, K) * D ** -0.5
            mask = torch.arange(n_ctx, device=x.device)[None, :] > pos[:, None]
            sc = sc.masked_fill(mask[None], float("-inf"))
            attn[sl] = torch.einsum("hqk,hkd->qhd", torch.softmax(sc, -1), V)
        o = attn.reshape(-1, h) @ w[p + ("self_attn.out_proj.weight" if opt else "self_attn.o_proj.weight")].t()
        if opt:
            o = o + w[p + "self_attn.out_proj.bias"]
        x = x + o
        xn = self._norm(x, p + ("final_layer_norm" if opt else "post_attention_layernorm"))
        if opt:
            f = torch.relu(xn @ w[p + "fc1.weight"].t() + w[p + "fc1.bias"])
            f = f @ w[p + "fc2.weight"].t() + w[p + "fc2.bias"]
        else:
            gu = xn @ w[p + "mlp.gate_up_proj.weight"].t()
            g_, u = gu[:, :s.ffn], gu[:, s.ffn:]
            f = (torch.nn.functional.silu(g_) * u) @ w[p + "mlp.down_proj.weight"].t()
        return x + f

    def head(self, x: torch.Tensor) -> torch.Tensor:
        s = self.s
        xn = self._norm(x, "final_layer_norm" if s.arch == ARCH_OPT else "norm")
        if s.n_labels:
            return xn @ self.w["score.weight"][: s.n_labels].t()
        hw = self.w["embed_tokens.weight"] if s.arch == ARCH_OPT else self.w["lm_head.weight"]
        return xn @ hw.t()

    # -- the two device operations ---------------------------------------------------
    @torch.no_grad()
    def prefill_chunk(self, cache: PagedCache, token_ids, slices, block_tables) -> torch.Tensor:
        """Mirror of tk_prefill_chunk: slices (start, len, bt_off, n_pages, emit).

        Returns fp32 logits of the emitting slices' last tokens, in slice order.
        """
        dev = self.device
        ids = torch.tensor(token_ids, dtype=torch.long, device=dev)
        pos_all, rows, row = [], [], 0
        for start, n, bto, npg, _ in slices:
            pos = torch.arange(start, start + n, device=dev)
            pos_all.append(pos)
            rows.append((list(block_tables[bto:bto + npg]), pos, slice(row, row + n)))
            row += n
        x = self.embed(ids, torch.cat(pos_all))
        for l in range(self.s.n_layers):
            x = self.layer(l, x, rows, cache)
        last = [r[2].stop - 1 for r, s in zip(rows, slices) if s[4]]
        if not last:
            return torch.empty(0, self.s.vocab)
        return self.head(x[last])

    @torch.no_grad()
    def decode_step(self, cache: PagedCache, last_tokens, ctx_lens, tables) -> torch.Tensor:
        """Mirror of tk_decode_step; returns fp32 logits [B, V]."""
        ids = torch.tensor(last_tokens, dtype=torch.long, device=self.device)
        pos = torch.tensor(ctx_lens, dtype=torch.long, device=self.device)
        rows = [(tables[b], pos[b:b + 1], slice(b, b + 1)) for b in range(len(last_tokens))]
        x = self.embed(ids, pos)
        for l in range(self.s.n_layers):
            x = self.layer(l, x, rows, cache)
        return self.head(x)

    @torch.no_grad()
    def full_forward(self, token_ids: list[int]) -> torch.Tensor:
        """Whole-prompt logits [n, V] without paging (for the transformers pin)."""
        n = len(token_ids)
        pt = 16
        cache = PagedCache(self.s, (n + pt - 1) // pt, pt, device=self.device)
        table = list(range(cache.n_pages))
        ids = torch.tensor(token_ids, dtype=torch.long, device=self.device)
        pos = torch.arange(n, device=self.device)
        x = self.embed(ids, pos)
        for l in range(self.s.n_layers):
            x = self.layer(l, x, [(table, pos, slice(0, n))], cache)
        return self.head(x)


def random_weights(shape: Shape, seed: int = 0, std: float = 0.02) -> dict[str, torch.Tensor]:
    """bf16-representable random weights (norm weights 1, biases 0)."""
    g = torch.Generator().manual_seed(seed)
    out = {}
    for name, shp in weight_shapes(shape).items():
        if name.endswith("layernorm.weight") or name.endswith("layer_norm.weight") \
                or name == "norm.weight":
            t = torch.ones(shp)
        elif name.endswith(".bias"):
            t = torch.randn(shp, generator=g) * std
        else:
            t = torch.randn(shp, generator=g) * std
        out[name] = t.to(torch.bfloat16).float()
    return out
