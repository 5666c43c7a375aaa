"""Quick tcgen05-path check: mini Qwen3 (hidden 512, hd 128) at B>=16 vs the fp32 oracle."""
import os
import sys
import torch
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from oracle.qwen3_fp32 import Qwen3Fp32
from paper_2604_15379_b200 import build_decoder_layer, b200_from_probe
from paper_2604_15379_b200.machine import ModelConfig
from paper_2604_15379_b200.analytics import device_tiles
from paper_2604_15379_b200.runtime import Megakernel, probe, halves_topology
from paper_2604_15379_b200.weights import Qwen3Spec, Qwen3Weights

topo = probe(0)
if topo.num_dies != 2:
    topo = halves_topology(topo.num_sms)
mach = b200_from_probe([topo.sms_per_die[i] for i in range(2)])
m = ModelConfig(hidden_dim=512, ffn_dim=1024, num_layers=2, q_heads=4, kv_heads=2, dtype_bytes=2)
spec = Qwen3Spec(512, 1024, 2, 4, 2, 128, 1024)
w = Qwen3Weights.random(spec, seed=21)
for mode, sched in (("chiplet", "per_die"), ("standard", "flat")):
    for B in (16, 32):
        g = build_decoder_layer(m, mach, mode, B, tile_overrides=device_tiles(m, mach, mode, B), layers=2)
        mk = Megakernel(g, w, t_max=64, sched=sched, topo=topo, watchdog_s=3.0)
        ref = Qwen3Fp32(w, t_max=64, batch=B)
        toks = torch.arange(B) * 37 % 1024
        worst = 0.0
        try:
            for s in range(4):
                out = mk.step(toks).cpu()
                want = ref.step(toks)
                got = mk.logits().float().cpu()
                err = (got - want).abs().max().item() / want.abs().max().item()
                worst = max(worst, err)
                toks = want.argmax(-1)
            print(mode, B, "max rel err", worst, "argmax agree", (out == got.argmax(-1)).all().item(), flush=True)
        except Exception as e:
            print(mode, B, "FAILED", e, flush=True)
        mk.close()
