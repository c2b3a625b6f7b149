"""CPU-side checks of the product library: it loads without a GPU, exports every
symbol include/marsit_b200.h declares, compiles schedules exactly like the
reference, and refuses to compute without a device (no CPU fallback)."""
import ctypes as C
import os
import re

import numpy as np
import pytest

import pyoracle as O
from conftest import ROOT, load_golden

import paper_2204_06787_b200 as mb
from paper_2204_06787_b200 import _native as N


def header_functions():
    src = open(os.path.join(ROOT, "include", "marsit_b200.h")).read()
    src = re.sub(r"/\*.*?\*/", "", src, flags=re.S)
    return sorted(set(re.findall(r"\b(marsit_[a-z0-9_]+)\s*\(", src)))


def test_library_exports_every_header_symbol():
    lib = C.CDLL(N.SO_PATH)
    names = header_functions()
    assert len(names) >= 20
    for name in names:
        assert hasattr(lib, name), name
    assert set(names) == set(N.SIGNATURES), set(names) ^ set(N.SIGNATURES)
    assert lib.marsit_abi_version() == 3


def test_schedules_match_reference_golden():
    for rec in load_golden("schedules"):
        s = (mb.build_ring_schedule(rec["a"]) if rec["topology"] == "ring"
             else mb.build_torus_schedule(rec["a"], rec["b"]))
        ph, st, rf, sg = s.tables()
        assert ph.tolist() == rec["phase"]
        assert st.tolist() == rec["send_to"]
        assert rf.tolist() == rec["recv_from"]
        assert sg.tolist() == rec["segment"]


def test_schedule_validation_errors():
    with pytest.raises(mb.ParameterError):
        mb.build_ring_schedule(1)
    with pytest.raises(mb.ParameterError):
        mb.build_torus_schedule(2, 1)
    # send/receive mismatch -> protocol_error (schedule.hpp:49-51)
    with pytest.raises(mb.ProtocolError):
        mb.Schedule.from_tables(2, 2, [0], [[1, 1]], [[1, 0]], [[0, 0]])
    with pytest.raises(mb.ProtocolError):
        mb.Schedule.from_tables(2, 2, [0], [[1, 0]], [[1, 0]], [[0, 5]])


def replay_plan(sched, signs, L, seed, rnd):
    """Owner-computes replay of the compiled plan with the oracle's merge:
    every segment's DAG in isolation, with each merge drawing from its
    receiver's stream and continuing it where offset_src says so."""
    W = sched.workers
    nw = O.words64(L)
    out = np.zeros((sched.segments, nw), np.uint64)
    counts = []
    for s in range(sched.segments):
        merges, final, fcount = sched.plan(s)
        nodes = {w: signs[w, s] for w in range(W)}
        used_after = {}
        for k, m in enumerate(merges):
            key = O.stream_key(seed, 5, m["receiver"], rnd, s)
            used0 = used_after[m["offset_src"]] if m["offset_src"] >= 0 else 0
            res, used = O.merge_signs(nodes[m["recv_node"]], m["c_recv"],
                                      nodes[m["local_node"]], m["c_local"], L, key, used0)
            nodes[W + k] = res
            used_after[k] = used
        out[s] = nodes[final]
        counts.append(fcount)
    return out, counts


def test_compiled_plan_replays_allreduce_sign_golden():
    for rec in load_golden("allreduce"):
        sched = (mb.build_ring_schedule(rec["a"]) if rec["topology"] == "ring"
                 else mb.build_torus_schedule(rec["a"], rec["b"]))
        L = rec["seg_len"]
        nw = O.words64(L)
        signs = np.array([int(x, 16) for x in rec["signs"]], np.uint64).reshape(
            sched.workers, sched.segments, nw)
        got, counts = replay_plan(sched, signs, L, rec["seed"], rec["round"])
        state = np.array([int(x, 16) for x in rec["state"]], np.uint64).reshape(
            sched.workers, sched.segments, nw)
        assert np.array_equal(got, state[0])
        assert counts == rec["counts"][:sched.segments]


def test_plan_structure_torus_chain():
    # SURVEY §3.3 chain_dump for torus 2x4, segment 0:
    # 0->1, 4->5, 1->2, 5->6, 2->3, 6->7, 3->7 (4+4, continuing receiver 7's stream)
    sched = mb.build_torus_schedule(2, 4)
    merges, final, count = sched.plan(0)
    assert [m["receiver"] for m in merges] == [1, 5, 2, 6, 3, 7, 7]
    assert [(m["c_recv"], m["c_local"]) for m in merges][-1] == (4, 4)
    assert merges[-1]["offset_src"] == 5 and merges[-1]["stage"] == 1
    assert count == 8 and final == 8 + 6
    ring = mb.build_ring_schedule(4)
    merges, final, count = ring.plan(0)
    assert [m["receiver"] for m in merges] == [1, 2, 3]
    assert all(m["offset_src"] == -1 and m["stage"] == 0 for m in merges)


def test_no_cpu_fallback_without_device():
    torch = pytest.importorskip("torch")
    if torch.cuda.is_available():
        pytest.skip("a device is present")
    with pytest.raises(mb.CudaError):
        mb.Context(1000, mb.build_ring_schedule(4))


REF_INC = "/root/reference/proj/include"


@pytest.mark.skipif(not os.path.isdir(REF_INC), reason="reference headers absent")
def test_dropin_shim_compiles_against_reference_headers():
    """include/marsit_b200/drop_in.hpp builds inside the reference's own type
    system (marsit::MarsitRoundResult etc.) and links the C-ABI library."""
    import subprocess
    r = subprocess.run(["make", "-s", "-C", os.path.join(ROOT, "tools"), "dropin"],
                       capture_output=True, text=True)
    assert r.returncode == 0, r.stdout + r.stderr
    assert os.path.exists(os.path.join(ROOT, "build", "dropin_parity"))


def test_dropin_binary_fails_loudly_without_gpu():
    import subprocess
    exe = os.path.join(ROOT, "build", "dropin_parity")
    if not os.path.exists(exe):
        pytest.skip("dropin_parity not built here")
    torch = pytest.importorskip("torch")
    if torch.cuda.is_available():
        pytest.skip("a device is present")
    r = subprocess.run([exe], capture_output=True, text=True, timeout=60)
    assert r.returncode != 0 and "no CUDA device" in r.stdout


def test_plain_c_program_builds_and_fails_loudly_without_gpu():
    """tools/sign_round_c.c uses the C-ABI from plain C (gcc -std=c11, no C++
    or torch in the translation unit); without a device it must stop with
    the library's no-CPU-path error."""
    import subprocess
    r = subprocess.run(["make", "-s", "-C", os.path.join(ROOT, "tools"), "sign_round_c"],
                       capture_output=True, text=True)
    assert r.returncode == 0, r.stdout + r.stderr
    exe = os.path.join(ROOT, "build", "sign_round_c")
    assert os.path.exists(exe)
    torch = pytest.importorskip("torch")
    if torch.cuda.is_available():
        pytest.skip("a device is present (the GPU suite runs it)")
    r = subprocess.run([exe], capture_output=True, text=True, timeout=60)
    assert r.returncode != 0 and "no CUDA device" in r.stderr
