"""The executor's device content digest (csrc/digest.cu):
the CUDA kernel against a numpy statement of its definition, on aligned,
unaligned, ragged and strided payloads, plus the content-addressing
properties the cache relies on."""

import numpy as np
import pytest
import torch

pytestmark = pytest.mark.gpu

M64 = (1 << 64) - 1
GOLDEN = 0x9E3779B97F4A7C15
SEED_A, SEED_B = 0x243F6A8885A308D3, 0x13198A2E03707344
TILE = 1024


def _u(x):
    return np.uint64(x & M64)


def mix_a(x):
    x = (x ^ (x >> np.uint64(30))) * _u(0xBF58476D1CE4E5B9)
    x = (x ^ (x >> np.uint64(27))) * _u(0x94D049BB133111EB)
    return x ^ (x >> np.uint64(31))


def mix_b(x):
    x = (x ^ (x >> np.uint64(27))) * _u(0x3C79AC492BA7B653)
    x = (x ^ (x >> np.uint64(33))) * _u(0x1C69B3F74AC4AE35)
    return x ^ (x >> np.uint64(27))


def digest_ref(rows_bytes: list[bytes]) -> bytes:
    """numpy restatement of digest_kernel's definition (see digest.cu)."""
    rb = len(rows_bytes[0])
    W = (rb + 7) // 8
    T = (W + TILE - 1) // TILE
    acc = np.zeros(4, dtype=np.uint64)
    with np.errstate(over="ignore"):
        for r, row in enumerate(rows_bytes):
            words = np.zeros(T * TILE, dtype=np.uint64)
            padded = row + b"\0" * (W * 8 - rb)
            words[:W] = np.frombuffer(padded, dtype="<u8")
            for t in range(T):
                lanes = np.arange(32, dtype=np.uint64)
                c = np.uint64(r * T + t) * np.uint64(32) + lanes
                a = mix_a(_u(SEED_A) ^ (c * _u(GOLDEN)))
                b = mix_b(_u(SEED_B) ^ (c * _u(GOLDEN)))
                for j in range(TILE // 32):
                    w = t * TILE + np.arange(32) + 32 * j
                    ok = w < W
                    v = words[w]
                    na = mix_a(a ^ v)
                    b = np.where(ok, (b ^ na) * _u(0xD6E8FEB86659FD93), b)
                    a = np.where(ok, na, a)
                acc[0] += mix_a(a + _u(0x5851F42D4C957F2D)).sum(dtype=np.uint64)
                acc[1] += mix_b(b + _u(0x14057B7EF767814F)).sum(dtype=np.uint64)
                acc[2] += mix_a(a ^ mix_b(b)).sum(dtype=np.uint64)
                acc[3] += mix_b(b ^ mix_a(a + _u(GOLDEN))).sum(dtype=np.uint64)
    return acc.view(np.int64).tobytes()


def _dev(buf: torch.Tensor, offset: int, rows: int, row_bytes: int, ld: int) -> bytes:
    from paper_2506_23364_b200 import _lib

    out = torch.zeros(4, dtype=torch.int64, device=buf.device)
    _lib.check(_lib.lib().wg_digest2d(buf.data_ptr() + offset, rows, row_bytes, ld, out.data_ptr(),
                                      _lib.stream_ptr()))
    return np.array(out.tolist(), dtype=np.int64).tobytes()


@pytest.mark.parametrize("rows,row_bytes,ld,offset", [
    (1, 8, 8, 0), (1, 1, 1, 0), (1, 8 * 1024, 8 * 1024, 0), (1, 8 * 2048 + 5, 0, 0),
    (3, 8 * 1024 * 2 + 5, 8 * 1024 * 2 + 8, 3), (5, 13, 16, 0), (4, 24 * 333, 24 * 400, 8),
    (2, 8 * 1500, 8 * 1500, 1), (7, 8 * 1024, 8 * 1100, 0),
])
def test_digest_matches_definition(rows, row_bytes, ld, offset):
    ld = ld or row_bytes
    n = offset + (rows - 1) * ld + row_bytes
    host = np.random.default_rng(rows * 7919 + row_bytes).integers(0, 256, size=n, dtype=np.uint8)
    buf = torch.from_numpy(host).cuda()
    rows_bytes = [host[offset + r * ld: offset + r * ld + row_bytes].tobytes() for r in range(rows)]
    assert _dev(buf, offset, rows, row_bytes, ld) == digest_ref(rows_bytes)


def test_digest_content_addressing():
    from paper_2506_23364_b200.workflow import device_digest

    g = torch.Generator().manual_seed(3)
    big = torch.rand(300, 517, generator=g, dtype=torch.float64).cuda()
    win = big[10:200, 33:450]
    # a strided window hashes like the same rows stored contiguously
    assert device_digest(win) == device_digest(win.contiguous())
    # position-sensitive: swapping two rows or two words changes the digest
    sw = win.contiguous().clone()
    sw[[0, 1]] = sw[[1, 0]]
    assert device_digest(sw) != device_digest(win.contiguous())
    sw = win.contiguous().clone()
    sw[5, 7], sw[5, 8] = sw[5, 8].clone(), sw[5, 7].clone()
    assert device_digest(sw) != device_digest(win.contiguous())
    # one flipped bit anywhere changes all four words
    base = device_digest(big)
    for (i, j) in [(0, 0), (299, 516), (150, 256)]:
        f = big.clone()
        f.view(torch.int64)[i, j] ^= 1
        d = device_digest(f)
        assert all(d[8 * k:8 * k + 8] != base[8 * k:8 * k + 8] for k in range(4))
    # deterministic across launches and a large payload (several tiles per row)
    x = torch.arange(1 << 22, dtype=torch.int64, device="cuda")
    assert device_digest(x) == device_digest(x.clone())


# -- staged host transfers (_device.upload / download above 64 MiB) ---------


@pytest.mark.parametrize("dtype,shape", [(torch.uint8, ((64 << 20) + 13,)), (torch.float64, (3001, 4099)),
                                         (torch.bool, ((200 << 20) + 7,)), (torch.int64, (9, 1 << 20, 1))])
def test_staged_transfers_round_trip(dtype, shape):
    from paper_2506_23364_b200 import _device

    g = torch.Generator(device="cuda").manual_seed(11)
    n = int(np.prod(shape))
    raw = torch.randint(0, 256, (n * torch.empty(0, dtype=dtype).element_size(),), dtype=torch.uint8,
                        device="cuda", generator=g)
    if dtype == torch.bool:
        raw = raw & 1
    t = raw.view(dtype).view(shape)
    t = t * 1 if dtype != torch.bool else t.clone()  # produced by a kernel just queued on the current stream
    h = _device.download(t)
    assert h.shape == tuple(shape) and h.flags.writeable
    want = t.cpu().numpy()
    assert np.array_equal(h.view(np.uint8), want.view(np.uint8))
    v = _device.host_view(t)
    assert not v.flags.writeable and np.array_equal(v.view(np.uint8), want.view(np.uint8))
    back = _device.upload(h)
    assert back.dtype == dtype and torch.equal(back.view(torch.uint8), t.view(torch.uint8))
    ro = np.frombuffer(h.tobytes(), dtype=h.dtype).reshape(h.shape)  # read-only source
    assert torch.equal(_device.upload(ro).view(torch.uint8), t.view(torch.uint8))
