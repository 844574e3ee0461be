"""CPU oracle for the PIPO hot path — TEST INFRASTRUCTURE ONLY.

Only `tests/`, `__graft_entry__.smoke()` and `bench.py`'s `cpu_baseline` /
`--impl reference` legs may import anything in this package.  The product path
(`paper_2504_03664_b200`) never imports it and fails loudly when its CUDA
library is missing.  The oracle shares no code with the CUDA path; the only
common dependency is the seeded input generator `pipo_synth` (no method
arithmetic in it).

What it computes: pipelined offloading reaches *exactly the
plain result* faster — tiers, modes and timing do not change the math
(§3.1.1, Alg. 1) — so the oracle is the plain
OPT decoder forward with the paper's INT4 weight quantization (§2,
PAPER.md:305-309 §3.4, §4.1) and greedy decoding, written out in
float64 (the paper fixes no accumulation precision; its FP16 activations are the
GPU path's storage format, held to the 2e-2 tolerance of BASELINE.json).
The quantizer is an encoding, so it follows the step-by-step recipe in fp32 as
SURVEY.md §8(c) step 1 / SPEC.md:485-493 define it.

Modules:
  quant.py  — int4 group-64 symmetric quantize / pack / unpack / dequantize.
  opt.py    — OPT decoder forward (embed, pre-LN layers, LM head, greedy).
  llama.py  — LLaMA3.1 decoder forward (NEXT-4: GQA, RoPE llama3, RMSNorm, SwiGLU,
              untied LM head), pinned to transformers' LlamaForCausalLM.
  memory.py — PAPER.md §3.5 / App. B memory model (Eq. 1 planner inputs).
"""
