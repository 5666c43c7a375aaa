"""Prefill throughput: a 1024-token prompt of Qwen3-8B (36 layers) built on
the device by chunked prefill (C tokens per launch) vs the decode-step loop.

    python tools/prefill_bench.py [--chunk 64] [--tokens 1024]
"""
import argparse
import json
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import torch  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--chunk", type=int, default=64)
    ap.add_argument("--tokens", type=int, default=1024)
    ap.add_argument("--layers", type=int, default=36)
    args = ap.parse_args()
    from dataclasses import replace
    from paper_2604_15379_b200 import b200_from_probe, build_decoder_layer, model_preset
    from paper_2604_15379_b200.analytics import device_tiles
    from paper_2604_15379_b200.runtime import Megakernel, halves_topology, probe
    from paper_2604_15379_b200.weights import Qwen3Spec, Qwen3Weights
    topo = probe(0)
    if topo.num_dies != 2:
        topo = halves_topology(topo.num_sms)
    mach = b200_from_probe([topo.sms_per_die[i] for i in range(topo.num_dies)])
    model = replace(model_preset("qwen3-8b"), num_layers=args.layers)
    spec = Qwen3Spec.qwen3_8b(layers=args.layers)
    w = Qwen3Weights.random(spec, seed=0, device="cuda")
    t_max = args.tokens + 128

    def graph(B):
        return build_decoder_layer(model, mach, "chiplet", B,
                                   tile_overrides=device_tiles(model, mach, "chiplet", B),
                                   layers=args.layers)
    pages = -(-t_max // 64) + 2
    dec = Megakernel(graph(1), w, t_max=t_max, topo=topo, kv_pages=pages, keep_logits=False)
    pf = Megakernel(graph(args.chunk), w, t_max=t_max, topo=topo, prefill_for=dec, keep_logits=False)
    prompt = torch.randint(0, spec.vocab, (args.tokens,), generator=torch.Generator().manual_seed(1)).tolist()
    dec.prefill_chunked(0, prompt[:args.chunk], pf)          # warm-up
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    nxt = dec.prefill_chunked(0, prompt, pf)
    torch.cuda.synchronize()
    chunked = time.perf_counter() - t0
    n_loop = min(args.tokens, 128)                           # the decode loop, sampled
    dec.release_row(0)
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    for t in range(n_loop):
        dec.step([prompt[t]])
    torch.cuda.synchronize()
    loop = (time.perf_counter() - t0) / n_loop * args.tokens
    print(json.dumps({"prompt_tokens": args.tokens, "chunk": args.chunk, "layers": args.layers,
                      "chunked_prefill_s": round(chunked, 4),
                      "chunked_tok_per_s": round(args.tokens / chunked, 1),
                      "decode_loop_s_est": round(loop, 4),
                      "decode_loop_tok_per_s": round(args.tokens / loop, 1),
                      "speedup": round(loop / chunked, 2), "next_token": nxt}))


if __name__ == "__main__":
    main()
