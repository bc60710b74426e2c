"""Load the shared seeded weights into transformers 5.5.0's Whisper modules so
the oracle can be pinned against an independent implementation (test helper;
third-party stand-in for the absent faster-whisper/CTranslate2)."""

from __future__ import annotations

import numpy as np
import torch


def hf_available() -> bool:
    try:
        import transformers  # noqa: F401
        from transformers import WhisperConfig  # noqa: F401
        return True
    except Exception:
        return False


def build_hf_whisper(dims, weights: dict[str, np.ndarray]):
    from transformers import WhisperConfig, WhisperForConditionalGeneration

    d = dims.d_model
    cfg = WhisperConfig(
        vocab_size=dims.vocab, num_mel_bins=dims.n_mels,
        encoder_layers=dims.enc_layers, decoder_layers=dims.dec_layers,
        encoder_attention_heads=dims.heads, decoder_attention_heads=dims.heads,
        encoder_ffn_dim=dims.ffn, decoder_ffn_dim=dims.ffn, d_model=d,
        max_source_positions=1500, max_target_positions=448,
        dropout=0.0, attention_dropout=0.0, activation_dropout=0.0,
        activation_function="gelu", scale_embedding=False,
        tie_word_embeddings=True)
    cfg._attn_implementation = "eager"
    m = WhisperForConditionalGeneration(cfg).eval()
    t = lambda a: torch.from_numpy(np.ascontiguousarray(a, dtype=np.float32))
    sd = {}
    e, dc = "model.encoder", "model.decoder"
    sd[f"{e}.conv1.weight"] = t(weights["enc.conv1.w"].transpose(0, 2, 1))
    sd[f"{e}.conv1.bias"] = t(weights["enc.conv1.b"])
    sd[f"{e}.conv2.weight"] = t(weights["enc.conv2.w"].transpose(0, 2, 1))
    sd[f"{e}.conv2.bias"] = t(weights["enc.conv2.b"])
    sd[f"{e}.embed_positions.weight"] = t(weights["enc.pos"])

    def attn(dst, src_qkv, has_self=True):
        w, b = weights[f"{src_qkv}.w"], weights[f"{src_qkv}.b"]
        sd[f"{dst}.q_proj.weight"] = t(w[:d]); sd[f"{dst}.q_proj.bias"] = t(b[:d])
        sd[f"{dst}.k_proj.weight"] = t(w[d:2 * d])
        sd[f"{dst}.v_proj.weight"] = t(w[2 * d:]); sd[f"{dst}.v_proj.bias"] = t(b[2 * d:])

    def lin(dst, src):
        sd[f"{dst}.weight"] = t(weights[f"{src}.w"])
        sd[f"{dst}.bias"] = t(weights[f"{src}.b"])

    def ln(dst, src):
        sd[f"{dst}.weight"] = t(weights[f"{src}.g"])
        sd[f"{dst}.bias"] = t(weights[f"{src}.b"])

    for i in range(dims.enc_layers):
        p, q = f"{e}.layers.{i}", f"enc.l{i}"
        attn(f"{p}.self_attn", f"{q}.qkv")
        lin(f"{p}.self_attn.out_proj", f"{q}.o")
        ln(f"{p}.self_attn_layer_norm", f"{q}.ln1")
        lin(f"{p}.fc1", f"{q}.fc1"); lin(f"{p}.fc2", f"{q}.fc2")
        ln(f"{p}.final_layer_norm", f"{q}.ln2")
    ln(f"{e}.layer_norm", "enc.ln")
    sd[f"{dc}.embed_tokens.weight"] = t(weights["dec.embed"])
    sd[f"{dc}.embed_positions.weight"] = t(weights["dec.pos"])
    xw, xb = weights["dec.xkv.w"], weights["dec.xkv.b"]
    for i in range(dims.dec_layers):
        p, q = f"{dc}.layers.{i}", f"dec.l{i}"
        attn(f"{p}.self_attn", f"{q}.qkv")
        lin(f"{p}.self_attn.out_proj", f"{q}.o")
        ln(f"{p}.self_attn_layer_norm", f"{q}.ln1")
        sd[f"{p}.encoder_attn.q_proj.weight"] = t(weights[f"{q}.xq.w"])
        sd[f"{p}.encoder_attn.q_proj.bias"] = t(weights[f"{q}.xq.b"])
        sd[f"{p}.encoder_attn.k_proj.weight"] = t(xw[i * 2 * d:i * 2 * d + d])
        sd[f"{p}.encoder_attn.v_proj.weight"] = t(xw[i * 2 * d + d:(i + 1) * 2 * d])
        sd[f"{p}.encoder_attn.v_proj.bias"] = t(xb[i * 2 * d + d:(i + 1) * 2 * d])
        lin(f"{p}.encoder_attn.out_proj", f"{q}.xo")
        ln(f"{p}.encoder_attn_layer_norm", f"{q}.ln2")
        lin(f"{p}.fc1", f"{q}.fc1"); lin(f"{p}.fc2", f"{q}.fc2")
        ln(f"{p}.final_layer_norm", f"{q}.ln3")
    ln(f"{dc}.layer_norm", "dec.ln")
    missing, unexpected = m.load_state_dict(sd, strict=False)
    missing = [k for k in missing if k != "proj_out.weight"]
    assert not missing and not unexpected, (missing, unexpected)
    m.tie_weights()
    return m


def hf_log_mel(samples_i16_list, n_mels: int) -> np.ndarray:
    """transformers' WhisperFeatureExtractor (torch path) on the
    pad_or_trim'ed float waveforms."""
    from transformers import WhisperFeatureExtractor
    fe = WhisperFeatureExtractor(feature_size=n_mels)
    wav = [np.asarray(s, np.int16).astype(np.float32) / 32768.0
           for s in samples_i16_list]
    out = fe(wav, sampling_rate=16000, return_tensors="np",
             padding="max_length", truncation=True)
    return out["input_features"]


def build_hf_wav2vec2(dims, weights):
    """transformers Wav2Vec2ForCTC (wav2vec2-base shape) loaded with the shared
    seeded weights; the positional conv's weight-norm is set so that its
    effective weight equals ours (g = ||W|| per tap, v = W)."""
    from transformers import Wav2Vec2Config, Wav2Vec2ForCTC
    cfg = Wav2Vec2Config(vocab_size=dims.vocab, hidden_size=dims.hidden,
                         num_hidden_layers=dims.layers, num_attention_heads=dims.heads,
                         intermediate_size=dims.ffn, hidden_act="gelu",
                         feat_extract_norm="group", feat_extract_activation="gelu",
                         conv_dim=list(dims.conv_dim), conv_kernel=list(dims.conv_kernel),
                         conv_stride=list(dims.conv_stride), conv_bias=False,
                         num_conv_pos_embeddings=dims.pos_conv_kernel,
                         num_conv_pos_embedding_groups=dims.pos_conv_groups,
                         do_stable_layer_norm=False, layer_norm_eps=dims.ln_eps,
                         hidden_dropout=0.0, attention_dropout=0.0, activation_dropout=0.0,
                         feat_proj_dropout=0.0, final_dropout=0.0, layerdrop=0.0,
                         apply_spec_augment=False, pad_token_id=dims.blank)
    cfg._attn_implementation = "eager"
    m = Wav2Vec2ForCTC(cfg).eval()
    t = lambda a: torch.from_numpy(np.ascontiguousarray(a, dtype=np.float32))
    sd = {}
    for i in range(len(dims.conv_dim)):
        sd[f"wav2vec2.feature_extractor.conv_layers.{i}.conv.weight"] = t(
            weights[f"fe.conv{i}.w"].transpose(0, 2, 1))
    sd["wav2vec2.feature_extractor.conv_layers.0.layer_norm.weight"] = t(weights["fe.gn.g"])
    sd["wav2vec2.feature_extractor.conv_layers.0.layer_norm.bias"] = t(weights["fe.gn.b"])
    sd["wav2vec2.feature_projection.layer_norm.weight"] = t(weights["fp.ln.g"])
    sd["wav2vec2.feature_projection.layer_norm.bias"] = t(weights["fp.ln.b"])
    sd["wav2vec2.feature_projection.projection.weight"] = t(weights["fp.proj.w"])
    sd["wav2vec2.feature_projection.projection.bias"] = t(weights["fp.proj.b"])
    g, cg, k = dims.pos_conv_groups, dims.hidden // dims.pos_conv_groups, dims.pos_conv_kernel
    W = weights["pos.w"].reshape(dims.hidden, k, cg).transpose(0, 2, 1)      # [out, in/g, k]
    conv = m.wav2vec2.encoder.pos_conv_embed.conv
    pre = "wav2vec2.encoder.pos_conv_embed.conv"
    if hasattr(conv, "parametrizations"):
        sd[f"{pre}.parametrizations.weight.original0"] = t(
            np.sqrt((W.astype(np.float64) ** 2).sum(axis=(0, 1), keepdims=True)))
        sd[f"{pre}.parametrizations.weight.original1"] = t(W)
    else:
        sd[f"{pre}.weight_g"] = t(np.sqrt((W.astype(np.float64) ** 2).sum(axis=(0, 1), keepdims=True)))
        sd[f"{pre}.weight_v"] = t(W)
    sd[f"{pre}.bias"] = t(weights["pos.b"])
    sd["wav2vec2.encoder.layer_norm.weight"] = t(weights["enc.ln.g"])
    sd["wav2vec2.encoder.layer_norm.bias"] = t(weights["enc.ln.b"])
    d = dims.hidden
    for i in range(dims.layers):
        p, q = f"wav2vec2.encoder.layers.{i}", f"l{i}"
        w, b = weights[f"{q}.qkv.w"], weights[f"{q}.qkv.b"]
        for j, nm in enumerate(("q_proj", "k_proj", "v_proj")):
            sd[f"{p}.attention.{nm}.weight"] = t(w[j * d:(j + 1) * d])
            sd[f"{p}.attention.{nm}.bias"] = t(b[j * d:(j + 1) * d])
        sd[f"{p}.attention.out_proj.weight"] = t(weights[f"{q}.o.w"])
        sd[f"{p}.attention.out_proj.bias"] = t(weights[f"{q}.o.b"])
        sd[f"{p}.layer_norm.weight"] = t(weights[f"{q}.ln1.g"])
        sd[f"{p}.layer_norm.bias"] = t(weights[f"{q}.ln1.b"])
        sd[f"{p}.feed_forward.intermediate_dense.weight"] = t(weights[f"{q}.fc1.w"])
        sd[f"{p}.feed_forward.intermediate_dense.bias"] = t(weights[f"{q}.fc1.b"])
        sd[f"{p}.feed_forward.output_dense.weight"] = t(weights[f"{q}.fc2.w"])
        sd[f"{p}.feed_forward.output_dense.bias"] = t(weights[f"{q}.fc2.b"])
        sd[f"{p}.final_layer_norm.weight"] = t(weights[f"{q}.ln2.g"])
        sd[f"{p}.final_layer_norm.bias"] = t(weights[f"{q}.ln2.b"])
    sd["lm_head.weight"] = t(weights["head.w"])
    sd["lm_head.bias"] = t(weights["head.b"])
    missing, unexpected = m.load_state_dict(sd, strict=False)
    missing = [k for k in missing if "masked_spec_embed" not in k]
    assert not missing and not unexpected, (missing, unexpected)
    return m
