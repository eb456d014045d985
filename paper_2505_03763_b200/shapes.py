"""Model shapes the engine is benchmarked on (BASELINE.json configs): Llama-3-style
decoders with GQA, random-init weights generated on the device from the seed.
Field meanings follow sw_model_desc (include/splitwise.h)."""
from dataclasses import dataclass


@dataclass(frozen=True)
class Shape:
    n_layers: int
    d_model: int
    n_heads: int
    n_kv_heads: int
    head_dim: int
    ffn_dim: int
    vocab: int
    tied_embeddings: bool = False
    rope_theta: float = 500000.0
    norm_eps: float = 1e-5
    seed: int = 1


TINY = Shape(n_layers=2, d_model=256, n_heads=4, n_kv_heads=2, head_dim=64, ffn_dim=768, vocab=4096)
LLAMA_1B = Shape(n_layers=16, d_model=2048, n_heads=32, n_kv_heads=8, head_dim=64, ffn_dim=8192, vocab=128256,
                 tied_embeddings=True)
LLAMA_8B = Shape(n_layers=32, d_model=4096, n_heads=32, n_kv_heads=8, head_dim=128, ffn_dim=14336, vocab=128256)
