"""TEST INFRASTRUCTURE ONLY -- the checker, never the product.

Only ``tests/``, ``__graft_entry__.smoke()`` and ``bench.py``'s CPU-baseline leg
(``--impl reference`` / ``cpu_baseline``) may import this package.  The runtime
(``paper_2504_21411_b200``) never imports it and fails loudly without its CUDA
library.

Contents
  model_ref.py  -- single-device, unsharded plain-PyTorch GPT-2 / Llama-2 forward +
                   backward (loss and every parameter gradient), written from the
                   standard model definitions.  The reference repository has NO
                   forward/backward (SPEC.md:10 puts the runtime out of scope), so
                   runtime-numerics parity against the *reference* is UNPINNED; this
                   restatement is itself cross-checked against Hugging Face
                   ``transformers`` (LlamaForCausalLM / GPT2LMHeadModel) on shared
                   weights (tests/golden/make_model_golden.py, tests/test_oracle.py).
  The planner oracle is the reference planner itself, run in the build container
  to produce tests/golden/planner_golden.jsonl (parity pinned, byte-exact).
"""
