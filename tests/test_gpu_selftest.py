"""On-GPU validation of the PTX layer the tensor-core path is built on: tcgen05 smem/instruction
descriptors for all operand majorness combinations, and TMA 128B-swizzle placement. Compared with
plain PyTorch fp32 matmul / a numpy swizzle formula."""
import ctypes as C

import numpy as np
import pytest

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def torch_cuda():
    import torch
    assert torch.cuda.is_available()
    return torch


@pytest.mark.parametrize("a_mn,b_mn", [(0, 0), (0, 1), (1, 0), (1, 1)])
@pytest.mark.parametrize("N,K", [(64, 64), (128, 128), (256, 64), (48, 128)])
def test_umma_descriptors(torch_cuda, a_mn, b_mn, N, K):
    torch = torch_cuda
    from paper_1502_03409_b200 import lcae
    g = torch.Generator(device="cpu").manual_seed(N * 7 + K + 3 * a_mn + b_mn)
    A = torch.randn(128, K, generator=g).to(torch.bfloat16).cuda()
    B = torch.randn(K, N, generator=g).to(torch.bfloat16).cuda()
    D = torch.zeros(128, N, dtype=torch.float32, device="cuda")
    lcae.dev_check(lcae.devlib().lcae_dev_umma_selftest(a_mn, b_mn, N, K, 0, A.data_ptr(), B.data_ptr(), D.data_ptr()))
    ref = A.float() @ B.float()
    err = (D - ref).abs().max().item() / ref.abs().max().item()
    assert err < 1e-5, err


def _swizzled(tile):
    """numpy placement of a [rows][64] bf16 tile under the 128B swizzle (chunk ^= row % 8)."""
    rows = tile.shape[0]
    out = np.zeros((rows, 64), dtype=tile.dtype)
    for r in range(rows):
        for c in range(8):
            out[r, ((c ^ (r % 8)) * 8):((c ^ (r % 8)) * 8 + 8)] = tile[r, c * 8:c * 8 + 8]
    return out


def test_tma_swizzle_and_oob(torch_cuda):
    torch = torch_cuda
    from paper_1502_03409_b200 import lcae
    rows, cols = 40, 200
    src = torch.arange(rows * cols, dtype=torch.float32).reshape(rows, cols).to(torch.bfloat16).cuda()
    for (r0, c0, box) in ((0, 0, 16), (8, 64, 32), (30, 160, 16)):
        dump = torch.zeros(box * 128, dtype=torch.uint8, device="cuda")
        lcae.dev_check(lcae.devlib().lcae_dev_tma_selftest(src.data_ptr(), rows, cols, box, r0, c0, dump.data_ptr()))
        got = dump.cpu().view(torch.bfloat16).float().numpy().reshape(box, 64)
        full = np.zeros((box, 64), dtype=np.float32)
        s = src.float().cpu().numpy()
        rr = min(rows, r0 + box) - r0
        cc = min(cols, c0 + 64) - c0
        full[:rr, :cc] = s[r0:r0 + rr, c0:c0 + cc]          # out-of-bounds zero-filled
        np.testing.assert_array_equal(got, _swizzled(full))


def test_red_probe_reports(torch_cuda, capsys):
    """Throughput of global fp32 reductions (informs the dX overlap-add design)."""
    torch = torch_cuda
    from paper_1502_03409_b200 import lcae
    n = 1 << 24
    buf = torch.zeros(n, dtype=torch.float32, device="cuda")
    out = {}
    for mode in (0, 1, 2):
        ms = C.c_float()
        reps = 64
        lcae.dev_check(lcae.devlib().lcae_dev_red_probe(buf.data_ptr(), n, reps, mode, 148 * 16, C.byref(ms)))
        elems = 148 * 16 * 256 * reps * (4 if mode == 1 else 1)
        out[mode] = elems / (ms.value * 1e-3) / 1e9
    with capsys.disabled():
        print(f"\n[red probe] G elem/s: red.f32={out[0]:.1f} red.v4.f32={out[1]:.1f} ld+add+st={out[2]:.1f}")


@pytest.mark.gpu
def test_tmem_16x256b_thread_map():
    """tcgen05.ld.16x256b.x2: thread t holds rows t/4 and t/4 + 8 of the 16-lane block, columns 2(t%4), +1 of
    each 8-column half (the map ptx.cuh documents)."""
    from paper_1502_03409_b200 import lcae
    out = np.zeros((4, 2, 32, 8), dtype=np.uint32)
    lcae.devlib().lcae_dev_tmem_shape_selftest.argtypes = [C.c_void_p]
    lcae.dev_check(lcae.devlib().lcae_dev_tmem_shape_selftest(out.ctypes.data))
    for w in range(4):
        for h in range(2):
            for t in range(32):
                got = [(int(v) >> 8, int(v) & 255) for v in out[w, h, t]]
                r0 = 32 * w + 16 * h + t // 4
                c = 2 * (t % 4)
                want = [(r0, c), (r0, c + 1), (r0 + 8, c), (r0 + 8, c + 1),
                        (r0, c + 8), (r0, c + 9), (r0 + 8, c + 8), (r0 + 8, c + 9)]
                assert got == want, (w, h, t, got, want)
