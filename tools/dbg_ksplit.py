"""Debug: mini-model decode with/without K-split, per-column logit errors."""
import sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from oracle.qwen3_fp32 import Qwen3Fp32
from paper_2604_15379_b200 import b200_from_probe, build_decoder_layer
from paper_2604_15379_b200.analytics import device_tiles
from paper_2604_15379_b200.machine import ModelConfig
from paper_2604_15379_b200.runtime import Megakernel, probe
from paper_2604_15379_b200.weights import Qwen3Spec, Qwen3Weights
from paper_2604_15379_b200 import _lib as L
import ctypes

B = int(sys.argv[1]) if len(sys.argv) > 1 else 1
topo = probe(0)
machine = b200_from_probe([topo.sms_per_die[i] for i in range(topo.num_dies)])
m = ModelConfig(hidden_dim=512, ffn_dim=1024, num_layers=2, q_heads=4, kv_heads=2, dtype_bytes=2)
spec = Qwen3Spec(512, 1024, 2, 4, 2, 128, 1024)
g = build_decoder_layer(m, machine, "chiplet", B, tile_overrides=device_tiles(m, machine, "chiplet", B), layers=2)
w = Qwen3Weights.random(spec, seed=32)
ref = Qwen3Fp32(w, t_max=40, batch=B)
toks = torch.arange(B) * 7 + 3
want = ref.step(toks)
for ks in (False, True):
    mk = Megakernel(g, w, t_max=40, topo=topo, ksplit=ks, watchdog_s=5.0)
    low = mk.lowered
    for i in range(len(low.tasks)):
        t = low.tasks[i]
        if t.op == L.OP_GEMM and t.level == 2:
            p = L.GemmParams.from_buffer_copy(low.params[t.param_off:t.param_off + ctypes.sizeof(L.GemmParams)])
            if p.ksplit or i < 3 or low.task_names[i].startswith("lm"):
                print(low.task_names[i], "ksplit", p.ksplit, "tile", (p.T_M, p.T_N, p.T_K), "M K N", (p.M, p.K, p.N), "ctr0", p.tile_ctr0)
    out = mk.step(toks)
    got = mk.logits().float().cpu()
    err = (got - want).abs()
    print("ksplit", ks, "max err", err.max().item(), "scale", want.abs().max().item())
    bad = (err > 0.05 * want.abs().max()).nonzero()
    print("bad entries", bad.shape[0], bad[:20].tolist())
    print("got[0,:8]", got[0, :8].tolist(), "want", want[0, :8].tolist())
    mk.close()
