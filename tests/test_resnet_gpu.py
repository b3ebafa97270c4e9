"""ResNet client layers on the tcgen05 engine vs torch fp32 on bf16-rounded operands (builder-defined
model: no reference ResNet exists).

NHWC implicit-GEMM convolutions (k = 1 / 3, stride 1 / 2, 4-D TMA boxes with out-of-bounds zero fill as
the padding): forward, data gradient (stride 1; stride 2 runs on the zero-upsampled gradient) and weight
gradient + SGD.  Tolerance: max-abs error <= 1e-2 x max |ref| (bf16 outputs, fp32 accumulation)."""

import pytest

pytestmark = pytest.mark.gpu

SHAPES = [  # (G, bp, H, cin, cout, k, s)
    (2, 4, 32, 64, 64, 3, 1),
    (1, 4, 32, 64, 128, 3, 2),
    (2, 8, 16, 128, 128, 3, 1),
    (1, 8, 16, 128, 256, 1, 2),
    (1, 16, 8, 256, 256, 3, 1),
    (2, 32, 4, 512, 512, 3, 1),
    (1, 32, 8, 256, 512, 3, 2),
]


def _w_layout(w):
    """torch [cout, cin, k, k] -> engine [k*k*cin][cout] (tap-major)."""
    co, ci, k, _ = w.shape
    return w.permute(2, 3, 1, 0).reshape(k * k * ci, co)


@pytest.mark.parametrize("G,bp,H,cin,cout,k,s", SHAPES)
def test_nhwc_conv_modes(G, bp, H, cin, cout, k, s):
    import torch
    import torch.nn.functional as F
    from paper_2305_15668_b200 import _abi
    torch.manual_seed(G * 100 + H + cin + k + s)
    dev = "cuda"
    n, Ho = G * bp, H // s
    bf = lambda t: t.to(torch.bfloat16).float()
    x = bf(torch.randn(n, cin, H, H))
    w = [bf(torch.randn(cout, cin, k, k) * (1.0 / (k * k * cin) ** 0.5)) for _ in range(G)]
    dy = bf(torch.randn(n, cout, Ho, Ho))
    sp = torch.cuda.current_stream().cuda_stream
    xd = x.permute(0, 2, 3, 1).contiguous().to(torch.bfloat16).to(dev)
    wd = torch.stack([_w_layout(t) for t in w]).to(torch.bfloat16).to(dev).contiguous()
    pad = k // 2
    # forward
    y = torch.zeros(n, Ho, Ho, cout, dtype=torch.bfloat16, device=dev)
    _abi.check(_abi.lib.fedhc_nhwc_conv(4, G, bp, H, H, cin, cout, k, s, xd.data_ptr(), None, wd.data_ptr(),
                                        y.data_ptr(), None, 0.0, sp))
    ref = torch.cat([F.conv2d(x[g * bp:(g + 1) * bp], w[g], stride=s, padding=pad) for g in range(G)])
    torch.cuda.synchronize()
    got = y.float().cpu().permute(0, 3, 1, 2)
    assert (got - ref).abs().max().item() <= 1e-2 * ref.abs().max().item()
    # data gradient: stride 1 directly; stride 2 through the zero-upsampled output gradient
    u = torch.zeros(n, cout, H, H)
    u[:, :, ::s, ::s] = dy
    ud = u.permute(0, 2, 3, 1).contiguous().to(torch.bfloat16).to(dev)
    dx = torch.zeros(n, H, H, cin, dtype=torch.bfloat16, device=dev)
    _abi.check(_abi.lib.fedhc_nhwc_conv(5, G, bp, H, H, cin, cout, k, 1, None, ud.data_ptr(), wd.data_ptr(),
                                        dx.data_ptr(), None, 0.0, sp))
    ref = torch.cat([torch.nn.grad.conv2d_input(x[g * bp:(g + 1) * bp].shape, w[g], dy[g * bp:(g + 1) * bp],
                                                stride=s, padding=pad) for g in range(G)])
    torch.cuda.synchronize()
    got = dx.float().cpu().permute(0, 3, 1, 2)
    assert (got - ref).abs().max().item() <= 1e-2 * ref.abs().max().item()
    # weight gradient + SGD (lr = 1, zero master): master = -grad
    dyd = dy.permute(0, 2, 3, 1).contiguous().to(torch.bfloat16).to(dev)
    master = torch.zeros(G, k * k * cin, cout, device=dev)
    _abi.check(_abi.lib.fedhc_nhwc_conv(6, G, bp, H, H, cin, cout, k, s, xd.data_ptr(), dyd.data_ptr(), None,
                                        master.data_ptr(), None, 1.0, sp))
    torch.cuda.synchronize()
    for g in range(G):
        gw = torch.nn.grad.conv2d_weight(x[g * bp:(g + 1) * bp], w[g].shape, dy[g * bp:(g + 1) * bp], stride=s,
                                         padding=pad)
        want = -_w_layout(gw)
        err = (master[g].cpu() - want).abs().max().item() / want.abs().max().item()
        assert err < 1e-3, (g, err)
