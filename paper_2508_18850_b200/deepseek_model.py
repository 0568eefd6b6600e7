"""Greedy decode of a whole DeepSeek-V2-Lite-shaped model on the GPU
(BASELINE config #3 end to end; the paper reports DeepSeek TPOT).

One step = embedding gather of the current token -> ``n_layers`` x
``DeepSeekBlock`` (head-batched MLA engine + fused MoE, PDL-chained) -> final
RMSNorm + LM head + argmax (``cfb_lm_head_argmax``, which also writes the next
token on the device), captured as ONE CUDA graph and replayed step after step.

Semantics follow the reference's MLA dataflow: a layer's latent cache is an
input that the step attends together with the new token's latent row, and is
not appended to (``dataflows.py:393-397``) - so every replay costs exactly one
decode step at the given context.  Dims: the reference MLA preset (hidden
2048, 16 heads x 128, kv_lora_rank 512; ``cli.py:47-54``) with the
DeepSeek-V2-Lite MoE (64 experts, top-6, 2 shared, width 1408) in every layer,
27 layers and the 102,400-token vocabulary of DeepSeek-V2-Lite (its first
dense-FFN layer and the decoupled RoPE key are outside the reference's MLA).
The CPU restatement is ``oracle/deepseek_port.block`` per layer plus the LM
head of ``oracle/llama_port``.
"""

from __future__ import annotations

from dataclasses import dataclass

import numpy as np

from . import _native
from .deepseek import LITE, DeepSeekBlock, DeepSeekDims
from .layouts import row_tiles


@dataclass(frozen=True)
class DeepSeekModelDims:
    block: DeepSeekDims = LITE
    n_layers: int = 27
    vocab: int = 102400

    def step_bytes(self, seq_len: int) -> int:
        """Algorithmic HBM bytes of one step: every block + the embedding row
        + the final norm + the LM head (fp16)."""
        D = self.block.hidden
        return (self.n_layers * self.block.block_bytes(seq_len) + 2 * D + 2 * D
                + 2 * self.vocab * D)


LITE_MODEL = DeepSeekModelDims()


class DeepSeekDecoder:
    """Device-resident DeepSeek-shaped model: blocks, embedding, final norm and
    LM head; ``step`` / ``capture`` + ``replay`` decode one token each."""

    def __init__(self, mdims: DeepSeekModelDims, blocks: list, embed, final_norm, lm_head):
        import torch
        dev = _native.require_cuda()
        self.mdims, self.blocks = mdims, blocks
        D, V = mdims.block.hidden, mdims.vocab

        def h(a):
            if not isinstance(a, torch.Tensor):
                a = torch.from_numpy(np.ascontiguousarray(a, np.float32))
            return a.to(dev).half().contiguous()

        self.embed = h(embed)
        self.final_norm = h(final_norm)
        self.lm = row_tiles(h(lm_head))
        self.resid = torch.zeros(1, D, device=dev, dtype=torch.float32)
        self.token_buf = torch.zeros(1, device=dev, dtype=torch.int32)
        self.logits_buf = torch.zeros(1, V, device=dev, dtype=torch.float32)
        self.cand_val = torch.zeros(1024, device=dev, dtype=torch.float32)
        self.cand_idx = torch.zeros(1024, device=dev, dtype=torch.int32)
        self.ticket = torch.zeros(1, device=dev, dtype=torch.int32)
        self.stream = torch.cuda.Stream(device=dev)
        self.graph = None
        torch.cuda.synchronize()

    # ---------------------------------------------------------------- builders
    @classmethod
    def random(cls, mdims: DeepSeekModelDims, seq_len: int, seed: int = 0) -> "DeepSeekDecoder":
        """Random fp16 weights / latent caches drawn on the device (benchmarks)."""
        import torch
        dev = _native.require_cuda()
        blocks = [DeepSeekBlock.random(mdims.block, seq_len, seed=seed * 1000 + l)
                  for l in range(mdims.n_layers)]
        g = torch.Generator(device=dev)
        g.manual_seed(seed + 77)
        D, V = mdims.block.hidden, mdims.vocab
        embed = torch.randn(V, D, generator=g, device=dev)
        lm = torch.randn(V, D, generator=g, device=dev) * D ** -0.5
        return cls(mdims, blocks, embed, torch.ones(D, device=dev), lm)

    @classmethod
    def from_arrays(cls, mdims: DeepSeekModelDims, layers: list, embed, final_norm, lm_head):
        """``layers``: per layer (mla_arrays, moe_w, attn_norm, ffn_norm) in the
        ``DeepSeekBlock.from_arrays`` formats."""
        blocks = [DeepSeekBlock.from_arrays(mdims.block, m, w, ga, gf) for (m, w, ga, gf) in layers]
        return cls(mdims, blocks, embed, final_norm, lm_head)

    # ---------------------------------------------------------------- running
    def _enqueue(self, logits: bool) -> None:
        L = _native.lib()
        sp = self.stream.cuda_stream
        D, V = self.mdims.block.hidden, self.mdims.vocab
        _native.check(L.cfb_embed(2, self.embed.data_ptr(), self.token_buf.data_ptr(), self.resid.data_ptr(),
                                  1, D, sp))
        for b in self.blocks:
            b.launch(self.resid, pdl=True, stream=self.stream)
        a = _native.LmArgs(dtype=2, batch=1, hidden=D, vocab=V, grid=0, flags=_native.PDL,
                           eps=self.mdims.block.eps, resid=self.resid.data_ptr(),
                           norm_w=self.final_norm.data_ptr(), w=self.lm.data_ptr(),
                           logits=self.logits_buf.data_ptr() if logits else None,
                           cand_val=self.cand_val.data_ptr(), cand_idx=self.cand_idx.data_ptr(),
                           ticket=self.ticket.data_ptr(), token_out=self.token_buf.data_ptr(),
                           step_pos=None)
        _native.check(L.cfb_lm_head_argmax(a, sp))

    def set_token(self, token: int) -> None:
        import torch
        self.token_buf.fill_(int(token))
        torch.cuda.synchronize()

    def step(self, logits: bool = False) -> None:
        """One greedy step, eager: token -> model -> next token (on the device)."""
        self._enqueue(logits)

    def capture(self) -> None:
        import torch
        self.graph = torch.cuda.CUDAGraph()
        with torch.cuda.graph(self.graph, stream=self.stream):
            self._enqueue(False)

    def replay(self) -> None:
        import torch
        with torch.cuda.stream(self.stream):
            self.graph.replay()

    def token(self) -> int:
        self.stream.synchronize()
        return int(self.token_buf.item())

    def logits(self) -> np.ndarray:
        self.stream.synchronize()
        return self.logits_buf.cpu().numpy()[0]
