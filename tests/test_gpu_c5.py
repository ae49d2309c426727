"""C5 (BASELINE.json configs[4]): ResNet-50 whose 16 3x3 convs are compressed
layers W ~ L + S running through the C-ABI library, every other layer dense
(§5.5, :343-387).  Logits vs the fp64 CPU reference network
(oracle/resnet_oracle.py, same seeded parameters), bf16 tolerance relL2 <= 2e-2.
"""
import numpy as np
import pytest
import torch

import workloads

pytestmark = pytest.mark.gpu


def test_c5_network_logits_vs_oracle():
    from oracle import resnet_oracle as R
    from paper_2006_06443_b200.resnet import build_compressed_resnet50
    n = 2
    model, comp = build_compressed_resnet50(batch_max=n)
    assert len(comp) == 16
    assert all(c.layer.sparse_engine[0] == 1 for c in comp.values())
    img = workloads.resnet50_images(n, seed=5)
    x = torch.from_numpy(img).to(torch.bfloat16).cuda().contiguous(memory_format=torch.channels_last)
    with torch.no_grad():
        y = model(x).float().cpu().numpy().astype(np.float64)
    ref = R.reference_logits(img)
    err = np.linalg.norm(y - ref) / np.linalg.norm(ref)
    assert err <= 2e-2, err


def test_c5_graph_replay_matches_eager():
    from paper_2006_06443_b200.resnet import build_compressed_resnet50
    n = 8
    model, _ = build_compressed_resnet50(batch_max=n)
    x = torch.from_numpy(workloads.resnet50_images(n, seed=6)).to(torch.bfloat16).cuda()
    x = x.contiguous(memory_format=torch.channels_last)
    s = torch.cuda.Stream()
    with torch.no_grad(), torch.cuda.stream(s):
        y0 = model(x)
        torch.cuda.synchronize()
        g = torch.cuda.CUDAGraph()
        with torch.cuda.graph(g, stream=s):
            y1 = model(x)
    g.replay()
    torch.cuda.synchronize()
    assert torch.equal(y0, y1)


@pytest.mark.parametrize("batch", [256, 32])
def test_c5_at_bench_batch_one_image_per_shard(batch):
    """The network as bench.py times it: handles sized for the bench's per-GPU batch
    (256 at 1 GPU, 32 at 8 -- the create-time autotuner may pick other plans for
    them), the whole forward captured in a CUDA graph and replayed.  The logits of
    one image per 32-image shard (varying position inside the shard) are checked
    against the fp64 reference network, image by image (bf16 bar relL2 <= 2e-2)."""
    from oracle import resnet_oracle as R
    from paper_2006_06443_b200.resnet import build_compressed_resnet50
    model, comp = build_compressed_resnet50(batch_max=batch)
    img = workloads.resnet50_images(batch, seed=9)
    x = torch.from_numpy(img).to(torch.bfloat16).cuda().contiguous(memory_format=torch.channels_last)
    s = torch.cuda.Stream()
    with torch.no_grad(), torch.cuda.stream(s):
        model(x)
        torch.cuda.synchronize()
        g = torch.cuda.CUDAGraph()
        with torch.cuda.graph(g, stream=s):
            logits = model(x)
    g.replay()
    g.replay()
    torch.cuda.synchronize()
    y = logits.float().cpu().numpy().astype(np.float64)
    idx = [32 * i + (11 * i + 3) % 32 for i in range(batch // 32)]
    ref = R.reference_logits(img[idx])
    for k, i in enumerate(idx):
        err = np.linalg.norm(y[i] - ref[k]) / np.linalg.norm(ref[k])
        assert err <= 2e-2, (i, err)
    for c in comp.values():
        c.close()
