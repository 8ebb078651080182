"""NEXT(3): the attention of the sparsified tail of one generation step
across all layers, as the paper deploys SparVAR.

Per layer, at the decision scale S the model runs full attention; the target
scales S+1..K run block-sparse attention:

  Sink order (DESIGN.md READING 25): the S-level pattern is the Top-K alone and the map adds the
  sink at each target; sink_in_source=True ORs it in at S as well.
  CS4A layers (the first round(0.6 L), "substituted from the shallowest"):
      O_S, pattern = dense attention at S with the block masses read off its softmax and
                     selected (top-k / threshold)                (sparvar_dense_attn_mass;
                     fused=False: sparvar_dense_attn + sparvar_predict_pattern)
      O_cache = O_S - Softmax(Q_S K_inds^T) V_inds              (sparvar_cache_residual_from_dense)
      for k in S+1..K:
          lists_k = CSR(map S->k of the pattern)                 (sparvar_map_indices, _build_block_lists)
          O_k     = NN-upsample(O_cache) + Delta O_k             (sparvar_block_sparse_attn_cached)
  granularity="token" replaces the CS4A layers' block pattern by the paper's token-granular one
  (NEXT(2)): dense attention at S with its LSE, column sums over
  C-row query blocks, top-k tokens (alpha C_S) + sinks, token-level O_cache, and per target
  scale the token map, its lists and the cached token-list attention.
  CSLA layers (the rest):
      O_S     = dense attention at S
      for k in S+1..K:  O_k = block-sparse attention over the CSLA local mask of k
                        (sparvar_local_mask / _build_block_lists once per step: the mask is the
                         same for every layer and head)

Every step of the path is a kernel of libsparvar.so; this module only sequences the calls and
owns the per-step scratch (masks, lists, O_cache), allocated once and reused layer after layer.
"""
from __future__ import annotations

from typing import Dict, List, Sequence

import torch

import math

from . import (MAP_FOOTPRINT, SELECT_TOPK, block_sparse_attn, block_sparse_attn_cached,
               build_block_lists, cache_residual_from_dense, dense_attn, dense_attn_mass,
               dense_attn_mass_workspace, geometry, local_mask, map_indices, predict_pattern,
               token_cache_residual, token_colsum, token_map, token_select,
               token_sparse_attn_cached)


def layer_split(layers: int, cs4a_fraction: float = 0.6) -> int:
    """Number of CS4A layers (the shallowest ones), PAPER.md:990 ("6:4"), at least 0."""
    return max(0, min(layers, int(round(cs4a_fraction * layers))))


class SparsifiedStep:
    """Attention of scales S..K of one generation step for `layers` layers (see module doc).

    Inputs per layer l: q[l][k] (bh, N_k, D) bf16 for k in S..K, and the layer's K/V cache
    (bh, >= C_K, D) bf16.  Outputs out[l][k] (bh, N_k, D) bf16 (caller-allocated or created).
    """

    def __init__(self, sides: Sequence[int], decision: int, target: int, block: int, bh: int,
                 layers: int, head_dim: int = 128, cs4a_fraction: float = 0.6,
                 sink_scales: int = 5, windows=(7, 5, 3, 1, 1), select_mode=SELECT_TOPK,
                 topk: int = 5, threshold: float = 0.01, map_mode=MAP_FOOTPRINT,
                 fused: bool = True, granularity: str = "block", query_block: int = 192,
                 alpha: float = 0.2, sink_in_source: bool = False):
        if not 1 <= decision < target <= len(sides):
            raise ValueError("need 1 <= decision < target <= number of scales")
        self.sides, self.S, self.K, self.B, self.bh = list(sides), decision, target, block, bh
        self.layers, self.D = layers, head_dim
        self.n_cs4a = layer_split(layers, cs4a_fraction)
        self.sink, self.windows = sink_scales, tuple(windows)
        self.sink_S = sink_scales if sink_in_source else 0          # READING 25
        self.select_mode, self.topk, self.threshold, self.map_mode = select_mode, topk, threshold, map_mode
        self.targets = list(range(decision + 1, target + 1))
        dev = "cuda"
        gS = geometry(sides, decision, block)
        self.gS = gS
        self.src = torch.empty((bh, gS["G_q"], gS["W"]), dtype=torch.int32, device=dev)
        self.lists_S = self._lists(gS)
        self.o_cache = torch.empty((bh, gS["N"], head_dim), dtype=torch.bfloat16, device=dev)
        self.g = {k: geometry(sides, k, block) for k in self.targets}
        self.mapped = {k: torch.empty((bh, g["G_q"], g["W"]), dtype=torch.int32, device=dev)
                       for k, g in self.g.items()}
        self.local = {k: torch.empty((g["G_q"], g["W"]), dtype=torch.int32, device=dev)
                      for k, g in self.g.items()}
        self.lists_map = {k: self._lists(g) for k, g in self.g.items()}
        self.lists_csla = {k: self._lists(g) for k, g in self.g.items()}
        self.status = torch.zeros(1, dtype=torch.int32, device=dev)
        self.fused = fused
        self.ws = torch.empty(max(1, dense_attn_mass_workspace(sides, decision, block, bh)) if fused
                              else 1, dtype=torch.uint8, device=dev)
        if granularity not in ("block", "token"):
            raise ValueError("granularity is 'block' or 'token'")
        self.granularity, self.C = granularity, query_block
        if granularity == "token":
            C, n_S, c_S = query_block, sides[decision - 1] ** 2, sum(x * x for x in sides[:decision])
            self.k_tok = max(1, math.ceil(alpha * c_S))                    # READING 11
            self.tG_S = -(-n_S // C)
            self.lse = torch.empty((bh, n_S), dtype=torch.float32, device=dev)
            self.colsum = torch.empty((bh, self.tG_S, c_S), dtype=torch.float32, device=dev)
            self.tsel = torch.empty((bh, self.tG_S, -(-c_S // 32)), dtype=torch.int32, device=dev)
            self.tlists_S = self._tlists(self.tG_S, c_S)
            self.tG, self.tmap, self.tlists = {}, {}, {}
            for k in self.targets:
                n_k, c_k = sides[k - 1] ** 2, sum(x * x for x in sides[:k])
                self.tG[k] = -(-n_k // C)
                self.tmap[k] = torch.empty((bh, self.tG[k], -(-c_k // 32)), dtype=torch.int32,
                                           device=dev)
                self.tlists[k] = self._tlists(self.tG[k], c_k)

    def _lists(self, g):
        cap = self.bh * g["G_q"] * g["G_kv"]
        return (torch.empty(self.bh * g["G_q"] + 1, dtype=torch.int32, device="cuda"),
                torch.empty(cap, dtype=torch.int32, device="cuda"), cap)

    def _tlists(self, G, n_tokens):
        cap = self.bh * G * n_tokens
        return (torch.empty(self.bh * G + 1, dtype=torch.int32, device="cuda"),
                torch.empty(cap, dtype=torch.int32, device="cuda"), cap, G, n_tokens)

    def _token_cs4a(self, q, k_cache, v_cache, out, stream):
        S, C = self.S, self.C
        dense_attn(self.sides, S, q[S], k_cache, v_cache, o=out[S], lse=self.lse, stream=stream)
        token_colsum(self.sides, S, C, q[S], k_cache, self.lse, out=self.colsum, stream=stream)
        token_select(self.sides, S, C, self.sink_S, self.colsum, self.k_tok, out=self.tsel,
                     stream=stream)
        rpS, ciS, capS, G_S, nS = self.tlists_S
        build_block_lists(self.bh, G_S, nS, [(self.tsel, False)], capS, rpS, ciS, self.status,
                          stream=stream)
        token_cache_residual(self.sides, S, C, q[S], k_cache, v_cache, rpS, ciS, out[S],
                             o_cache=self.o_cache, stream=stream)
        for k in self.targets:
            token_map(self.sides, S, k, C, self.sink, self.tsel, self.map_mode, out=self.tmap[k],
                      stream=stream)
            rp, ci, cap, G, n = self.tlists[k]
            build_block_lists(self.bh, G, n, [(self.tmap[k], False)], cap, rp, ci, self.status,
                              stream=stream)
            token_sparse_attn_cached(self.sides, k, C, q[k], k_cache, v_cache, rp, ci,
                                     self.o_cache, S, o=out[k], stream=stream)

    def kind(self, layer: int) -> str:
        return "cs4a" if layer < self.n_cs4a else "csla"

    def alloc_outputs(self) -> List[Dict[int, torch.Tensor]]:
        return [{k: torch.empty((self.bh, self.sides[k - 1] ** 2, self.D), dtype=torch.bfloat16,
                                device="cuda") for k in [self.S] + self.targets}
                for _ in range(self.layers)]

    def csla_patterns(self, stream=None):
        """Local masks and their CSR lists for every target scale (once per step)."""
        for k in self.targets:
            g = self.g[k]
            local_mask(self.sides, k, self.B, self.sink, self.windows, out=self.local[k],
                       stream=stream)
            rp, ci, cap = self.lists_csla[k]
            build_block_lists(self.bh, g["G_q"], g["G_kv"], [(self.local[k], True)], cap, rp, ci,
                              self.status, stream=stream)

    def layer(self, l: int, q: Dict[int, torch.Tensor], k_cache, v_cache,
              out: Dict[int, torch.Tensor], stream=None):
        S, B = self.S, self.B
        if self.kind(l) == "cs4a" and self.granularity == "token":
            self._token_cs4a(q, k_cache, v_cache, out, stream)
        elif self.kind(l) == "cs4a":
            gS = self.gS
            if self.fused:
                dense_attn_mass(self.sides, S, B, self.sink_S, q[S], k_cache, v_cache,
                                self.select_mode, self.topk, self.threshold, o=out[S],
                                want_mass=False, mask_out=self.src, workspace=self.ws,
                                stream=stream)
            else:
                dense_attn(self.sides, S, q[S], k_cache, v_cache, o=out[S], stream=stream)
                predict_pattern(self.sides, S, B, self.sink_S, q[S], k_cache, self.select_mode,
                                self.topk, self.threshold, want_mass=False, mask_out=self.src,
                                stream=stream)
            rpS, ciS, capS = self.lists_S
            build_block_lists(self.bh, gS["G_q"], gS["G_kv"], [(self.src, False)], capS, rpS, ciS,
                              self.status, stream=stream)
            cache_residual_from_dense(self.sides, S, B, q[S], k_cache, v_cache, rpS, ciS, out[S],
                                      o_cache=self.o_cache, stream=stream)
            for k in self.targets:
                g = self.g[k]
                map_indices(self.sides, S, k, B, self.sink, self.src, self.map_mode,
                            out=self.mapped[k], stream=stream)
                rp, ci, cap = self.lists_map[k]
                build_block_lists(self.bh, g["G_q"], g["G_kv"], [(self.mapped[k], False)], cap, rp,
                                  ci, self.status, stream=stream)
                block_sparse_attn_cached(self.sides, k, B, q[k], k_cache, v_cache, rp, ci,
                                         self.o_cache, S, o=out[k], stream=stream)
        else:
            dense_attn(self.sides, S, q[S], k_cache, v_cache, o=out[S], stream=stream)
            for k in self.targets:
                rp, ci, _ = self.lists_csla[k]
                block_sparse_attn(self.sides, k, B, q[k], k_cache, v_cache, rp, ci, o=out[k],
                                  stream=stream)

    def run(self, qs: Sequence[Dict[int, torch.Tensor]], ks: Sequence[torch.Tensor],
            vs: Sequence[torch.Tensor], outs=None, stream=None):
        """The whole sparsified tail for all layers; returns outs[l][k]."""
        if outs is None:
            outs = self.alloc_outputs()
        self.csla_patterns(stream)
        for l in range(self.layers):
            self.layer(l, qs[l], ks[l], vs[l], outs[l], stream)
        return outs

    def run_dense(self, qs, ks, vs, outs, stream=None):
        """The same scales with dense attention everywhere: the step's denominator."""
        for l in range(self.layers):
            for k in [self.S] + self.targets:
                dense_attn(self.sides, k, qs[l][k], ks[l], vs[l], o=outs[l][k], stream=stream)
        return outs
