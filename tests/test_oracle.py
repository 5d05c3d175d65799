"""Pin the fp32 oracle (oracle/model_ref.py) before trusting it.

The reference pins no numerics; the oracle restates the
HuggingFace models the paper served, so it is
checked here against transformers 5.5.0's own OPTForCausalLM,
OPTForSequenceClassification and LlamaForCausalLM on identical weights, and
its chunked/paged execution against its own whole-prompt forward.
"""

import pytest
import torch

from oracle.model_ref import (ARCH_LLAMA, ARCH_OPT, OracleModel, PagedCache, Shape,
                              random_weights)
from paper_2401_11181_b200.prefill import chunkify
from paper_2401_11181_b200.workload import Request

transformers = pytest.importorskip("transformers")

OPT_TINY = Shape(ARCH_OPT, n_layers=2, hidden=128, n_heads=4, ffn=256, vocab=512,
                 max_positions=600)
LLAMA_TINY = Shape(ARCH_LLAMA, n_layers=2, hidden=128, n_heads=4, ffn=192, vocab=512,
                   max_positions=600)


def _hf_opt(shape: Shape, w: dict, n_labels: int = 0):
    cfg = transformers.OPTConfig(
        vocab_size=shape.vocab, hidden_size=shape.hidden, num_hidden_layers=shape.n_layers,
        ffn_dim=shape.ffn, num_attention_heads=shape.n_heads,
        max_position_embeddings=shape.max_positions, do_layer_norm_before=True,
        word_embed_proj_dim=shape.hidden, activation_function="relu", dropout=0.0,
        attention_dropout=0.0, enable_bias=True, pad_token_id=1,
        num_labels=max(n_labels, 2))
    cls = transformers.OPTForSequenceClassification if n_labels else transformers.OPTForCausalLM
    model = cls(cfg).eval()
    h = shape.hidden
    sd = {"model.decoder.embed_tokens.weight": w["embed_tokens.weight"],
          "model.decoder.embed_positions.weight": w["embed_positions.weight"],
          "model.decoder.final_layer_norm.weight": w["final_layer_norm.weight"],
          "model.decoder.final_layer_norm.bias": w["final_layer_norm.bias"]}
    for l in range(shape.n_layers):
        src, dst = f"layers.{l}.", f"model.decoder.layers.{l}."
        qkv_w, qkv_b = w[src + "self_attn.qkv_proj.weight"], w[src + "self_attn.qkv_proj.bias"]
        for i, name in enumerate("qkv"):
            sd[dst + f"self_attn.{name}_proj.weight"] = qkv_w[i * h:(i + 1) * h]
            sd[dst + f"self_attn.{name}_proj.bias"] = qkv_b[i * h:(i + 1) * h]
        for name in ("self_attn.out_proj.weight", "self_attn.out_proj.bias",
                     "self_attn_layer_norm.weight", "self_attn_layer_norm.bias",
                     "final_layer_norm.weight", "final_layer_norm.bias", "fc1.weight",
                     "fc1.bias", "fc2.weight", "fc2.bias"):
            sd[dst + name] = w[src + name]
    if n_labels:
        sd["score.weight"] = w["score.weight"][:n_labels]
    else:
        sd["lm_head.weight"] = w["embed_tokens.weight"]
    missing, unexpected = model.load_state_dict(sd, strict=False)
    assert not unexpected and all("lm_head" in m for m in missing), (missing, unexpected)
    return model


def test_opt_oracle_matches_transformers():
    w = random_weights(OPT_TINY, seed=1, std=0.05)
    ora = OracleModel(OPT_TINY, w)
    hf = _hf_opt(OPT_TINY, w)
    ids = torch.randint(2, OPT_TINY.vocab, (1, 70), generator=torch.Generator().manual_seed(0))
    with torch.no_grad():
        ref = hf(input_ids=ids).logits[0]
    got = ora.full_forward(ids[0].tolist())
    assert torch.allclose(got, ref, atol=2e-4, rtol=1e-4), (got - ref).abs().max()


def test_opt_classifier_matches_transformers():
    shape = Shape(ARCH_OPT, 2, 128, 4, 256, 512, 600, n_labels=41)
    w = random_weights(shape, seed=2, std=0.05)
    ora = OracleModel(shape, w)
    hf = _hf_opt(shape, w, n_labels=41)
    ids = torch.randint(2, shape.vocab, (1, 33), generator=torch.Generator().manual_seed(3))
    with torch.no_grad():
        ref = hf(input_ids=ids).logits[0]
    got = ora.full_forward(ids[0].tolist())[-1]
    assert torch.allclose(got, ref, atol=2e-4, rtol=1e-4)


def test_llama_oracle_matches_transformers():
    s = LLAMA_TINY
    w = random_weights(s, seed=4, std=0.05)
    cfg = transformers.LlamaConfig(
        vocab_size=s.vocab, hidden_size=s.hidden, intermediate_size=s.ffn,
        num_hidden_layers=s.n_layers, num_attention_heads=s.n_heads,
        num_key_value_heads=s.n_heads, max_position_embeddings=s.max_positions,
        rms_norm_eps=s.norm_eps, rope_theta=s.rope_theta, tie_word_embeddings=False)
    hf = transformers.LlamaForCausalLM(cfg).eval()
    h, f = s.hidden, s.ffn
    sd = {"model.embed_tokens.weight": w["embed_tokens.weight"], "model.norm.weight": w["norm.weight"],
          "lm_head.weight": w["lm_head.weight"]}
    for l in range(s.n_layers):
        src, dst = f"layers.{l}.", f"model.layers.{l}."
        qkv = w[src + "self_attn.qkv_proj.weight"]
        for i, name in enumerate("qkv"):
            sd[dst + f"self_attn.{name}_proj.weight"] = qkv[i * h:(i + 1) * h]
        gu = w[src + "mlp.gate_up_proj.weight"]
        sd[dst + "mlp.gate_proj.weight"] = gu[:f]
        sd[dst + "mlp.up_proj.weight"] = gu[f:]
        sd[dst + "mlp.down_proj.weight"] = w[src + "mlp.down_proj.weight"]
        sd[dst + "self_attn.o_proj.weight"] = w[src + "self_attn.o_proj.weight"]
        sd[dst + "input_layernorm.weight"] = w[src + "input_layernorm.weight"]
        sd[dst + "post_attention_layernorm.weight"] = w[src + "post_attention_layernorm.weight"]
    hf.load_state_dict(sd)
    ids = torch.randint(0, s.vocab, (1, 50), generator=torch.Generator().manual_seed(5))
    with torch.no_grad():
        ref = hf(input_ids=ids).logits[0]
    got = OracleModel(s, w).full_forward(ids[0].tolist())
    assert torch.allclose(got, ref, atol=2e-4, rtol=1e-4), (got - ref).abs().max()


@pytest.mark.parametrize("shape", [OPT_TINY, LLAMA_TINY])
def test_chunked_paged_prefill_equals_whole_prompt(shape):
    """pdsim chunk layout (chunkify) over paged KV == unchunked forward."""
    w = random_weights(shape, seed=7, std=0.05)
    ora = OracleModel(shape, w)
    g = torch.Generator().manual_seed(9)
    lens = [18, 100, 300, 41]
    prompts = [torch.randint(2, shape.vocab, (n,), generator=g).tolist() for n in lens]
    reqs = [Request(id=i, arrival_us=0, prompt_len=n, true_decode_len=4) for i, n in enumerate(lens)]
    pt = 16
    tables, nxt = {}, 0
    for r in reqs:
        np_ = (r.prompt_len + pt) // pt + 1
        tables[r.id] = list(range(nxt, nxt + np_))
        nxt += np_
    cache = PagedCache(shape, nxt, pt)
    first = {}
    for chunk in chunkify(reqs, 128):
        ids, slices, bt = [], [], []
        for rid, start, n in chunk.slices:
            ids += prompts[rid][start:start + n]
            slices.append((start, n, len(bt), len(tables[rid]), int(start + n == lens[rid])))
            bt += tables[rid]
        logits = ora.prefill_chunk(cache, ids, slices, bt)
        emitting = [rid for (rid, s, n) in chunk.slices if s + n == lens[rid]]
        for rid, row in zip(emitting, logits):
            first[rid] = row
    for rid, toks in enumerate(prompts):
        ref = ora.full_forward(toks)[-1]
        assert torch.allclose(first[rid], ref, atol=1e-4, rtol=1e-4)
    # one decode step continues every request exactly
    last = [int(first[r].argmax()) for r in range(len(lens))]
    dec = ora.decode_step(cache, last, lens, [tables[r] for r in range(len(lens))])
    for rid, toks in enumerate(prompts):
        ref = ora.full_forward(toks + [last[rid]])[-1]
        assert torch.allclose(dec[rid], ref, atol=1e-4, rtol=1e-4)
