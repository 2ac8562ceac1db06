"""CPU tests of the boundary and the host-side logic (no GPU calls):

* libvreg_b200.so loads and exports every function include/*.h declares;
  the ctypes tables bind exactly those;
* the C config struct has the reference's RegistrationConfig layout;
* the slab / halo / reduction-fold protocol of the multi-GPU runtime, run
  as world_size-2 gloo process groups.
"""
import ctypes as C
import os
import re
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def header_functions():
    names = set()
    for h in ("vreg_cuda.h", "vreg_b200.h"):
        src = open(os.path.join(ROOT, "include", h)).read()
        src = re.sub(r"/\*.*?\*/", "", src, flags=re.S)
        names |= set(re.findall(r"\b(vreg_\w+)\s*\(", src))
    return names


def test_library_exports_every_declared_symbol():
    from paper_2008_12820_b200 import _lib
    import paper_2008_12820_b200.solver  # noqa: F401  (binds the solver table)
    L = _lib.lib()
    declared = header_functions()
    assert len(declared) > 60
    missing = [n for n in declared if not hasattr(L, n)]
    assert not missing, missing
    assert set(_lib.exported_symbols()) == declared


def test_status_codes_map_to_reference_exit_codes():
    from paper_2008_12820_b200 import _lib
    L = _lib.lib()
    # types.hpp:17-18: config/dimension/parameter -> 2, numerical -> 3, io -> 4
    assert [L.vreg_status_exit_code(s) for s in (0, 2, 3, 4, 5, 6, 7, 8)] == [0, 2, 3, 4, 2, 2, 2, 1]


def test_config_layout_matches_reference_config():
    from oracle import ref
    from paper_2008_12820_b200 import _lib
    from paper_2008_12820_b200.solver import Config, VregConfig
    # the reference's RegistrationConfig fields in order (optim.hpp:16-37),
    # then the B200 extensions (fp64 PCG iterates, H2 regularisation)
    names = [f[0] for f in VregConfig._fields_]
    assert names[:-2] == [f[0] for f in ref.VrefConfig._fields_]
    assert names[-2:] == ["pcg_fp64", "reg_order"]
    assert VregConfig.pcg_fp64.offset >= C.sizeof(ref.VrefConfig) - 4
    c = VregConfig()
    _lib.lib().vreg_config_default(C.byref(c))
    d = Config().to_c()
    for name, _ in VregConfig._fields_:
        assert getattr(c, name) == getattr(d, name), name


def test_bench_helpers():
    import bench
    assert bench.weak_grid(256, 1) == (256, 256, 256)
    assert bench.weak_grid(256, 2) == (512, 256, 256)
    assert bench.weak_grid(256, 8) == (512, 512, 512)
    assert bench.weak_grid(512, 8) == (1024, 1024, 1024)
    assert bench.bytes_per_voxel(4) == 552  # 88 + 116 nt
    assert bench.bytes_per_voxel_ours(4) == 500


def test_slab_layout():
    from paper_2008_12820_b200.dist import slab
    assert slab(256, 3, 4) == (64, 192)
    with pytest.raises(ValueError):
        slab(10, 0, 4)


# ---- world_size-2 gloo runs of the multi-GPU host protocol -------------------

def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, q):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    from paper_2008_12820_b200.dist import (fold_plane_partials, halo_exchange,
                                            plane_partials, slab)
    n1, n2, n3 = 12, 5, 7
    glob = torch.arange(n1 * n2 * n3, dtype=torch.float32).reshape(n1, n2, n3) * 0.37 + 1.0
    n1l, off = slab(n1, rank, world)
    local = glob[off:off + n1l].contiguous()
    out = {}
    for G in (1, 3, n1l):
        lo, hi = halo_exchange(local, G)
        idx_lo = [(off - G + t) % n1 for t in range(G)]
        idx_hi = [(off + n1l + t) % n1 for t in range(G)]
        out[G] = bool(torch.equal(lo, glob[idx_lo]) and torch.equal(hi, glob[idx_hi]))
    parts = plane_partials(local)
    allp = [torch.empty_like(parts) for _ in range(world)]
    dist.all_gather(allp, parts)
    folded = fold_plane_partials(torch.cat(allp))
    serial = fold_plane_partials(plane_partials(glob))
    q.put((rank, out, folded == serial))
    dist.destroy_process_group()


@pytest.mark.parametrize("world", [2, 3])
def test_halo_protocol_and_p_independent_fold_gloo(world):
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, q)) for r in range(world)]
    for p in procs:
        p.start()
    res = [q.get(timeout=120) for _ in procs]
    for p in procs:
        p.join(timeout=60)
    for rank, halos, fold_equal in res:
        assert all(halos.values()), (rank, halos)
        assert fold_equal


def test_volume_file_roundtrip_and_errors(tmp_path):
    """VolumeFile "VRG1": bitwise round trip for both
    scalar kinds and component counts; bad magic / truncated payload rejected."""
    from paper_2008_12820_b200 import VregError
    from paper_2008_12820_b200.volume import load_volume, save_volume
    rng = np.random.default_rng(7)
    for dt, shape in ((np.float32, (6, 5, 4)), (np.float64, (3, 6, 5, 4)),
                      (np.float32, (3, 2, 3, 4)), (np.float64, (4, 4, 4))):
        a = rng.standard_normal(shape).astype(dt)
        p = tmp_path / "v.vrg"
        save_volume(p, a)
        raw = p.read_bytes()
        assert raw[:4] == b"VRG1" and len(raw) == 18 + a.nbytes
        assert np.frombuffer(raw[4:16], "<u4").tolist() == list(shape[-3:])
        assert raw[16] == (0 if dt == np.float32 else 1) and raw[17] == (3 if len(shape) == 4 else 1)
        b = load_volume(p)
        assert b.dtype == a.dtype and b.shape == a.shape and b.tobytes() == a.tobytes()
    bad = tmp_path / "bad.vrg"
    bad.write_bytes(b"VRG2" + raw[4:])
    with pytest.raises(VregError) as e:
        load_volume(bad)
    assert e.value.kind == "io_error"
    bad.write_bytes(raw[:-4])
    with pytest.raises(VregError) as e:
        load_volume(bad)
    assert e.value.kind == "io_error"
    with pytest.raises(VregError) as e:
        load_volume(tmp_path / "missing.vrg")
    assert e.value.kind == "io_error"


def _halo_plan(n1l, G):
    from paper_2008_12820_b200 import _lib
    cap = 256
    d, c = (C.c_int * cap)(), (C.c_int * cap)()
    lo, hi = (C.c_longlong * cap)(), (C.c_longlong * cap)()
    n = _lib.lib().vreg_halo_chunks(n1l, G, cap, d, c, lo, hi)
    assert 0 < n <= cap
    return [(d[i], c[i], lo[i], hi[i]) for i in range(n)]


@pytest.mark.parametrize("p,n1l,G", [(2, 16, 3), (2, 16, 16), (2, 16, 23), (4, 8, 23),
                                     (3, 5, 14), (1, 8, 3), (4, 8, 40), (8, 2, 7)])
def test_wide_halo_plan(p, n1l, G):
    """Halo chunks of csrc/dist.cu (vreg_halo_chunks) for ghost widths up to
    and beyond the slab width: every rank's lo/hi ghosts hold the periodic
    neighbour planes, the reverse exchange folds ghost accumulators onto
    their owners, and the send/recv issue order (dist.cu halo_exchange /
    halo_reverse_send) matches per peer pair, as NCCL's in-order matching
    of same-peer messages needs."""
    chunks = _halo_plan(n1l, G)
    assert sum(c for _, c, _, _ in chunks) == G
    n1 = p * n1l
    for r in range(p):
        lo, hi = np.full(G, -1), np.full(G, -1)
        for d, c, l, h in chunks:
            a, b = (r - d) % p, (r + d) % p
            lo[l:l + c] = np.arange(a * n1l + n1l - c, a * n1l + n1l)
            hi[h:h + c] = np.arange(b * n1l, b * n1l + c)
        assert np.array_equal(lo, (r * n1l - G + np.arange(G)) % n1)
        assert np.array_equal(hi, (r * n1l + n1l + np.arange(G)) % n1)
    # reverse fold: extended accumulators [-G, n1l + G) per rank -> owners
    rng = np.random.default_rng(G)
    ext = rng.standard_normal((p, n1l + 2 * G))
    expect = np.zeros(n1)
    for r in range(p):
        np.add.at(expect, (r * n1l - G + np.arange(n1l + 2 * G)) % n1, ext[r])
    got = ext[:, G:G + n1l].copy()
    for r in range(p):
        for d, c, l, h in chunks:
            got[(r - d) % p, n1l - c:] += ext[r, l:l + c]          # lo chunk -> owner r-d
            got[(r + d) % p, :c] += ext[r, G + n1l + h:G + n1l + h + c]  # hi chunk -> owner r+d
    assert np.allclose(got.reshape(-1), expect)
    # issue order, forward and reverse (self transfers are local copies)
    for rev in (False, True):
        sends = {(a, b): [] for a in range(p) for b in range(p)}
        recvs = {(a, b): [] for a in range(p) for b in range(p)}
        for r in range(p):
            for d, c, _, _ in chunks:
                f, b = (r + d) % p, (r - d) % p
                pairs = [(b, f, "lo"), (f, b, "hi")] if rev else [(f, b, "lo"), (b, f, "hi")]
                for to, frm, tag in pairs:
                    if to == r:
                        continue
                    sends[(r, to)].append((tag, d, c))
                    recvs[(frm, r)].append((tag, d, c))
        for k in sends:
            assert sends[k] == recvs[k], (rev, k)
