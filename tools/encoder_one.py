"""One BERT-base encoder layer plan, run 3 times (for ncu launch lists)."""
import sys
sys.path.insert(0, __file__.rsplit("/tools/", 1)[0])
import torch  # noqa: E402
from paper_2210_12415_b200 import _abi, e2e  # noqa: E402
gen = torch.Generator(device="cuda")
gen.manual_seed(1)
g, gm, p = e2e.build_encoder(1, 64, flags=0, packed_qkv="packed" in sys.argv)
for k, x in e2e.make_encoder_inputs(g, gen).items():
    p.set_input_device(k, x)
for _ in range(3):
    p.run()
torch.cuda.synchronize()
for i in range(len(g.nodes)):
    print(i, p.node_kernel(i)[:100])
