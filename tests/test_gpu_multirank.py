"""Multi-rank row strips with the REAL CUDA band kernels.

tests/test_distributed.py checks the exchange / band bookkeeping on CPU with an
oracle band function.  Here two ranks (processes) each drive cuda:0 through
the product's own band entry points -- ``Transform.forward_rows`` /
``Transform.inverse_rows`` (b2dwt_forward_rows / b2dwt_inverse_rows) -- while
the halos travel between them over gloo, staged through host memory (one GPU:
the ranks never wait on each other's kernels, only on host messages).  The
strips must be bitwise equal to the single-GPU whole-image transform.

A second test runs the same decomposition over NCCL with device buffers when
the box has two or more GPUs (skipped on a single-GPU box).
"""

import os
import socket

import numpy as np
import pytest

pytestmark = pytest.mark.gpu

torch = pytest.importorskip("torch")
if not torch.cuda.is_available():  # pragma: no cover - CPU container
    pytest.skip("needs a CUDA device", allow_module_level=True)

import torch.distributed as dist  # noqa: E402
import torch.multiprocessing as mp  # noqa: E402

H, W = 1024, 768


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _image():
    return np.random.default_rng(21).random((H, W)).astype(np.float32)


def _gloo_worker(rank, world, port, levels, q):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        from paper_1705_08266_b200 import CDF97, Transform, build_scheme
        from paper_1705_08266_b200.distributed import RowStrips

        torch.cuda.set_device(0)
        tr = Transform(build_scheme("non-separable-split", CDF97), "single")
        img = _image()

        def band_forward(band, band_row0, height, r0, r1, out):
            got = tr.forward_rows(band.contiguous().cuda(), band_row0, height, r0, r1)
            for o, g in zip(out, got):
                o.copy_(g.cpu())

        strips = RowStrips(H, W, rank, world, tr.cone[:2], levels=levels)
        buf = strips.allocate(lambda s: torch.zeros(s, dtype=torch.float32))
        L = strips.layout(0)
        strips.owned(buf).copy_(torch.from_numpy(img[L.row0:L.row0 + L.rows]))
        ll, details = strips.dwt(band_forward, buf, lambda s: torch.zeros(s, dtype=torch.float32), overlap=True)

        want_ll, want_det = tr.dwt(torch.from_numpy(img).cuda(), levels)
        ok = True
        for lvl, (got, want) in enumerate(zip(details, want_det)):
            Ll = strips.layout(lvl)
            a, b = Ll.row0 // 2, (Ll.row0 + Ll.rows) // 2
            for g, wv in zip(got, want):
                ok &= torch.equal(g, wv[a:b].cpu())
        Ll = strips.layout(levels - 1)
        a, b = Ll.row0 // 2, (Ll.row0 + Ll.rows) // 2
        ok &= torch.equal(ll, want_ll[a:b].cpu())

        # inverse strips of level 0 (the inverse program's cone)
        inv = RowStrips(H, W, rank, world, tr.inv_plan.cone[:2], levels=1)
        q4 = tr.forward(torch.from_numpy(img).cuda())
        sb = inv.allocate_subbands(lambda s: torch.zeros(s, dtype=torch.float32))
        own = inv.owned_subbands(sb)
        L0 = inv.layout(0)
        for c in range(4):
            own[c].copy_(q4[c][L0.row0 // 2:(L0.row0 + L0.rows) // 2].cpu())

        def band_inverse(band, band_row0, height, r0, r1, out):
            out.copy_(tr.inverse_rows(tuple(b.contiguous().cuda() for b in band), band_row0, height, r0, r1).cpu())

        rec = torch.zeros((L0.rows, W), dtype=torch.float32)
        inv.inverse(band_inverse, sb, rec, overlap=True)
        full = tr.inverse(*q4)
        ok &= torch.equal(rec, full[L0.row0:L0.row0 + L0.rows].cpu())
        q.put((rank, bool(ok)))
    except Exception as exc:  # report instead of hanging the parent
        q.put((rank, repr(exc)))
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("levels", [1, 3])
def test_two_ranks_on_one_gpu_gloo_bitwise_equal_single_gpu(levels):
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_gloo_worker, args=(r, 2, port, levels, q)) for r in range(2)]
    for p in procs:
        p.start()
    results = dict(q.get(timeout=300) for _ in range(2))
    for p in procs:
        p.join(timeout=60)
    assert all(results[r] is True for r in range(2)), results


def _nccl_worker(rank, world, port, q):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    torch.cuda.set_device(rank)
    dist.init_process_group("nccl", rank=rank, world_size=world, device_id=torch.device("cuda", rank))
    try:
        from paper_1705_08266_b200 import CDF97, Transform, build_scheme
        from paper_1705_08266_b200.distributed import RowStrips

        tr = Transform(build_scheme("non-separable-split", CDF97), "single")
        img = _image()
        strips = RowStrips(H, W, rank, world, tr.cone[:2], levels=1)
        buf = strips.allocate(lambda s: torch.zeros(s, dtype=torch.float32, device="cuda"))
        L = strips.layout(0)
        strips.owned(buf).copy_(torch.from_numpy(img[L.row0:L.row0 + L.rows]))
        outs = tuple(torch.empty((L.rows // 2, W // 2), device="cuda") for _ in range(4))

        def band_forward(band, band_row0, height, r0, r1, out):
            tr.forward_rows(band, band_row0, height, r0, r1, out=out)

        strips.forward(band_forward, buf, outs, 0, None, overlap=True)
        full = tr.forward(torch.from_numpy(img).cuda())
        q0 = L.row0 // 2
        ok = all(torch.equal(o, f[q0:q0 + L.rows // 2]) for o, f in zip(outs, full))
        q.put((rank, bool(ok)))
    except Exception as exc:
        q.put((rank, repr(exc)))
    finally:
        dist.destroy_process_group()


@pytest.mark.skipif(torch.cuda.device_count() < 2, reason="needs two GPUs (NCCL halo exchange)")
def test_two_gpus_nccl_row_strips_bitwise_equal_single_gpu():
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_nccl_worker, args=(r, 2, port, q)) for r in range(2)]
    for p in procs:
        p.start()
    results = dict(q.get(timeout=300) for _ in range(2))
    for p in procs:
        p.join(timeout=60)
    assert all(results[r] is True for r in range(2)), results
