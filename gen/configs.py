"""Benchmark / parity configurations C1..C5 (BASELINE.json ``configs``) and the
integer cost profiles they use.

These are INPUT constants, not method arithmetic:
the paper gives no cost coefficients, so the profiles are assumptions chosen
to reproduce its qualitative rules: Discard below a
context threshold and Swap above it for long APIs, Preserve for
short APIs.  Tick = 1 microsecond, SH = 16, B = 16 tokens per block.

KV bytes per token (fp16, 2 * layers * hidden * 2 B): GPT-J 6B 28 x 4096 ->
458752 B (7 MiB per 16-token block); Vicuna 13B 40 x 5120 -> 819200 B
(12.5 MiB per block).  The same formula gives 2.25 GiB for GPT-3 175B at 512
tokens, the paper's "around 2.3 GB".
"""
from __future__ import annotations

KV_BYTES_PER_TOKEN = {
    "gptj": 2 * 28 * 4096 * 2,
    "vicuna": 2 * 40 * 5120 * 2,
    "gpt3": 2 * 96 * 12288 * 2,
}

PROFILES = {
    # tau: ticks per decode iteration; T_fwd(c) = (A1 c + A2 c^2) >> SH;
    # T_swap(c) = c ? (S0 + S1 c) >> SH : 0; c_other profiled batch context.
    "gptj": dict(tau=12_000, A1=100 << 16, A2=98, S0=12_000 << 16, S1=23 << 16, SH=16,
                 c_other=16_384, block_tokens=16, ticks_per_second=1e6),
    "vicuna": dict(tau=22_000, A1=200 << 16, A2=177, S0=22_000 << 16, S1=41 << 16, SH=16,
                   c_other=8_192, block_tokens=16, ticks_per_second=1e6),
}

# Table 2: API duration (mean, std) seconds and calls per request (mean, std).
API_CLASSES = {
    "math": dict(dur=(9e-5, 6e-5), num=(3.75, 1.3), resp=8),
    "qa": dict(dur=(0.69, 0.17), num=(2.52, 1.73), resp=64),
    "ve": dict(dur=(0.09, 0.014), num=(28.18, 15.2), resp=32),
    "chatbot": dict(dur=(28.6, 15.6), num=(4.45, 1.96), resp=128),
    "image": dict(dur=(20.03, 7.8), num=(6.91, 3.93), resp=16),
    "tts": dict(dur=(17.24, 7.6), num=(6.91, 3.93), resp=16),
    "toolbench": dict(dur=(1.72, 3.33), num=(2.45, 1.81), resp=96),
}
INFERCEPT_CLASSES = ["math", "qa", "ve", "chatbot", "image", "tts"]

# GiB of KV budget -> blocks of 16 tokens
def gib_to_blocks(gib: float, profile: str, B: int = 16) -> int:
    return int(gib * (1 << 30) // (KV_BYTES_PER_TOKEN[profile] * B))


CONFIGS = {
    # 16-request Single-API pool, GPT-J 6B KV footprint, 1 API type (Chatbot), 2 GB budget
    "C1": dict(name="C1", n=16, capacity=16, profile="gptj", classes=["chatbot"], multi_api=False,
               prompt=(256, 0.8, 16, 2048), kv_total=292, max_batch=16, starvation_threshold=100,
               score_bits=40, id_bits=23),
    # Single-API trace, 1800 requests, GPT-J 6B
    "C2": dict(name="C2", n=1800, capacity=2048, profile="gptj", classes=INFERCEPT_CLASSES,
               multi_api=False, prompt=(256, 0.8, 16, 2048), kv_total=3000, max_batch=256,
               starvation_threshold=100, score_bits=40, id_bits=23),
    # Multi-API trace, 1800 requests, Vicuna 13B, mixed P/D/S
    "C3": dict(name="C3", n=1800, capacity=2048, profile="vicuna", classes=INFERCEPT_CLASSES,
               multi_api=True, prompt=(256, 0.8, 16, 2048), kv_total=640, max_batch=256,
               starvation_threshold=100, score_bits=40, id_bits=23),
    # ToolBench-shaped multi-call trace, Vicuna 13B, 100k pool, starvation threshold
    "C4": dict(name="C4", n=100_000, capacity=131_072, profile="vicuna", classes=["toolbench"],
               multi_api=True, prompt=(1024, 0.8, 128, 4096), kv_total=10_000, max_batch=1024,
               starvation_threshold=100, score_bits=40, id_bits=23),
    # 1M-request pool (2^20 slots), GPT-J; per-shard budget 20000 blocks, max_batch 1024.
    # Key = 1 + 35 + 20 bits.
    "C5": dict(name="C5", n=1 << 20, capacity=1 << 20, profile="gptj", classes=INFERCEPT_CLASSES,
               multi_api=True, prompt=(256, 0.8, 16, 2048), kv_total=20_000, max_batch=1024,
               starvation_threshold=100, score_bits=35, id_bits=20),
}


def lib_config(cname: str, **over) -> dict:
    """The integer scheduler config (the lamps_config / oracle cfg fields) of a named config."""
    c = dict(CONFIGS[cname]); c.update(over)
    p = PROFILES[c["profile"]]
    d = dict(capacity=c["capacity"], block_tokens=p["block_tokens"], tau=p["tau"], A1=p["A1"],
             A2=p["A2"], S0=p["S0"], S1=p["S1"], SH=p["SH"], c_other=p["c_other"],
             ticks_per_second=p["ticks_per_second"],
             starvation_threshold=c["starvation_threshold"], max_batch=c["max_batch"],
             kv_capacity_blocks=max(c["kv_total"], 1 << 20), score_bits=c["score_bits"],
             id_bits=c["id_bits"], policy=c.get("policy", 0), score_interval=c.get("score_interval", 0))
    return d
