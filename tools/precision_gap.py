"""Inherent bf16-vs-fp32 logit gap at depth (analysis tool, GPU box).

Runs the same token sequence through
  * transformers Qwen3ForCausalLM in fp32 (reference numerics),
  * transformers Qwen3ForCausalLM in bf16 (the reference model's own bf16 path),
  * the megakernel (bf16 storage, fp32 accumulate), decoding from position 0,
on hash-initialised Qwen3-8B-shaped weights with L layers, and prints the
normwise logit error max|a - b| / max|fp32| of each pair per position.  If
the megakernel's error against fp32 tracks HF-bf16's, the gap is the bf16
format's, not the kernel's.

    python tools/precision_gap.py --layers 36 --tokens 6
"""
import argparse
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import torch  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--layers", type=int, default=36)
    ap.add_argument("--tokens", type=int, default=6)
    ap.add_argument("--out", default="gpurun_out/precision_gap.json")
    args = ap.parse_args()
    from dataclasses import replace
    from oracle.gen_hf_golden import hf_model
    from paper_2604_15379_b200 import b200_from_probe, build_decoder_layer, model_preset
    from paper_2604_15379_b200.analytics import device_tiles
    from paper_2604_15379_b200.runtime import Megakernel, halves_topology, probe
    from paper_2604_15379_b200.weights import Qwen3Spec, Qwen3Weights

    spec = Qwen3Spec.qwen3_8b(layers=args.layers)
    w = Qwen3Weights.random(spec, seed=0, device="cuda")
    g = torch.Generator().manual_seed(1234)
    toks = torch.randint(0, spec.vocab, (1, args.tokens), generator=g)
    res = {}
    with torch.no_grad():
        m = hf_model(w, device="cuda")
        res["hf32"] = m(input_ids=toks.cuda()).logits[0].float().cpu()
        m = m.to(torch.bfloat16)
        res["hf16"] = m(input_ids=toks.cuda()).logits[0].float().cpu()
        del m
        torch.cuda.empty_cache()
    topo = probe(0)
    if topo.num_dies != 2:
        topo = halves_topology(topo.num_sms)
    mach = b200_from_probe([topo.sms_per_die[i] for i in range(topo.num_dies)])
    model = replace(model_preset("qwen3-8b"), num_layers=args.layers)
    gr = build_decoder_layer(model, mach, "chiplet", 1,
                             tile_overrides=device_tiles(model, mach, "chiplet", 1),
                             layers=args.layers)
    mk = Megakernel(gr, w, t_max=128, topo=topo)
    mk.set_positions([0])
    dev = []
    for t in range(args.tokens):
        mk.step(toks[:, t])
        dev.append(mk.logits().float().cpu()[0])
    res["dev"] = torch.stack(dev)
    mk.close()

    def err(a, b):
        return [((res[a][t] - res[b][t]).abs().max() / res[b][t].abs().max()).item()
                for t in range(args.tokens)]
    out = {"layers": args.layers,
           "dev_vs_hf32": err("dev", "hf32"), "hf16_vs_hf32": err("hf16", "hf32"),
           "dev_vs_hf16": err("dev", "hf16"),
           "greedy": {k: v.argmax(-1).tolist() for k, v in res.items()}}
    print(json.dumps(out))
    os.makedirs(os.path.dirname(args.out), exist_ok=True)
    json.dump(out, open(args.out, "w"), indent=1)


if __name__ == "__main__":
    main()
