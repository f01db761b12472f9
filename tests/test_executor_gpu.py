"""Executor API semantics on the GPU, mirroring the reference's test_executor.py cases."""

import numpy as np
import pytest

from conftest import plan_from_doc

pytestmark = pytest.mark.gpu


def _plan(grid_docs, name):
    return plan_from_doc(next(d for d in grid_docs if d["name"] == name)["plan"])


def test_ghz3_final_state_and_stats(grid_docs):
    # test_executor.py:29-47
    from paper_2509_14098_b200 import gather, run_plan

    res = run_plan(_plan(grid_docs, "ghz3-2"))
    dense = gather(res.state)
    exp = np.zeros(8, dtype=complex)
    exp[0] = exp[7] = 2 ** -0.5
    np.testing.assert_allclose(dense, exp, atol=1e-12)
    assert res.stats.task_counts == {"Alloc": 1, "ApplyFused": 2, "Pack": 1, "Exchange": 1,
                                     "Unpack": 1, "Free": 1}
    (e,) = res.stats.exchanges
    assert e["messages"] == 2 and e["amps"] // e["messages"] == 2 and e["bytes"] == 16 * e["amps"]


def test_initial_state_and_drift(grid_docs):
    # test_executor.py:104-117
    from paper_2509_14098_b200 import NonUnitaryDrift, gather, run_plan

    plan = _plan(grid_docs, "x0-2")
    init = np.zeros(4, dtype=complex)
    init[1] = 1.0
    dense = gather(run_plan(plan, initial=init).state)
    np.testing.assert_allclose(dense, np.eye(4)[3], atol=1e-12)
    with pytest.raises(NonUnitaryDrift):
        run_plan(plan, initial=np.full(4, 0.9, dtype=complex))


def test_protocol_errors(grid_docs):
    # test_executor.py:146-175
    from paper_2509_14098_b200 import PlanInvalid, run_plan
    from paper_2509_14098_b200.plan import ExecutionPlan, Task

    plan = _plan(grid_docs, "ghz3-2")
    t = list(plan.tasks)
    t[1], t[5] = t[5], t[1]
    with pytest.raises(PlanInvalid):
        run_plan(ExecutionPlan(plan.d, plan.g, plan.layout_phases, t))
    extra = Task(len(plan.tasks), "Alloc", (len(plan.tasks) - 1,), plan.tasks[0].payload)
    with pytest.raises(PlanInvalid):
        run_plan(ExecutionPlan(plan.d, plan.g, plan.layout_phases, list(plan.tasks) + [extra]))
    nopack = [x for x in plan.tasks if x.kind != "Pack"]
    nopack = [Task(i, x.kind, (i - 1,) if i else (), x.payload) for i, x in enumerate(nopack)]
    with pytest.raises(PlanInvalid):
        run_plan(ExecutionPlan(plan.d, plan.g, plan.layout_phases, nopack))
    # stale passthrough mark
    bad = [Task(x.id, x.kind, x.deps, dict(x.payload)) for x in plan.tasks]
    g0 = dict(bad[1].payload["gates"][0])
    g0["passthrough"] = not g0["passthrough"]
    bad[1].payload["gates"] = [g0] + bad[1].payload["gates"][1:]
    with pytest.raises(PlanInvalid):
        run_plan(ExecutionPlan(plan.d, plan.g, plan.layout_phases, bad))


def test_scatter_gather_compare(grid_docs):
    # test_executor.py:66-101
    from paper_2509_14098_b200 import DimensionMismatch, compare, gather, scatter

    plan = _plan(grid_docs, "ghz3-2")
    rng = np.random.default_rng(5)
    v = rng.normal(size=8) + 1j * rng.normal(size=8)
    v /= np.linalg.norm(v)
    for ph in (0, 1):
        np.testing.assert_allclose(gather(scatter(v, plan, ph)), v, atol=1e-15)
    w = np.exp(1j * 1.234) * v
    assert compare(v, w) < 1e-12 and compare(v, v) == 0.0
    a = np.zeros(4, dtype=complex)
    a[0] = 1
    b = np.zeros(4, dtype=complex)
    b[1] = 1
    assert compare(a, b) > 0.9
    with pytest.raises(DimensionMismatch):
        scatter(np.zeros(4, dtype=complex), plan)
    with pytest.raises(DimensionMismatch):
        compare(a, np.zeros(8, dtype=complex))


def test_histograms(grid_docs):
    # test_executor.py:128-143 + bit-identity with the reference sampler
    from paper_2509_14098_b200 import run_plan, sample

    plan = _plan(grid_docs, "ghz3-2")
    r1 = run_plan(plan, shots=200, seed=9)
    r2 = run_plan(plan, shots=200, seed=9)
    assert r1.histogram == r2.histogram and sum(r1.histogram.values()) == 200
    assert set(r1.histogram) <= {"000", "111"}
    d = np.zeros(4, dtype=complex)
    d[2] = 1
    assert sample(d, 50, seed=1) == {"10": 50}


def test_oracle_simulate_and_size_guard(grid_docs, grid_states):
    from paper_2509_14098_b200 import TooLarge, compare, oracle_simulate

    class Op:
        def __init__(self, kind, params, qubits):
            from paper_2509_14098_b200 import gates
            self.gate = gates.gate(kind, tuple(params))
            self.qubits = tuple(qubits)

    class Circ:
        def __init__(self, d, ops):
            self.num_qubits, self.ops = d, ops

    n = 0
    for doc in grid_docs:
        if doc["name"] + "::dense" not in grid_states or doc["plan"]["d"] > 10 or n > 40:
            continue
        ops = [Op(g["kind"], g["params"], g["qubits"]) for t in doc["plan"]["tasks"]
               if t["kind"] == "ApplyFused" for g in t["payload"]["gates"]]
        v = oracle_simulate(Circ(doc["plan"]["d"], ops))
        assert compare(v, grid_states[doc["name"] + "::dense"]) < 1e-10, doc["name"]
        n += 1
    with pytest.raises(TooLarge):
        oracle_simulate(Circ(15, []))


def test_kernel_plugin_matches_numpy():
    # test_kernels.py:33-81: GPU plugin vs the numpy twin, random unitaries/diagonals
    from oracle.oracle import _NumpyKernels
    from paper_2509_14098_b200 import kernels

    rng = np.random.default_rng(3)
    for _ in range(40):
        L = int(rng.integers(1, 9))
        ranks = 1 << int(rng.integers(0, 3))
        p = int(rng.integers(1, min(L, 4) + 1))
        bits = [int(b) for b in rng.permutation(L)[:p]]
        m = rng.normal(size=(1 << p, 1 << p)) + 1j * rng.normal(size=(1 << p, 1 << p))
        u, _ = np.linalg.qr(m)
        a = rng.normal(size=(ranks, 1 << L)) + 1j * rng.normal(size=(ranks, 1 << L))
        b = a.copy()
        _NumpyKernels.apply_gate(a, u, bits)
        kernels.apply_gate(b, u, bits)
        np.testing.assert_allclose(a, b, atol=1e-12)
        dg = np.exp(1j * rng.uniform(-3, 3, size=1 << p))
        _NumpyKernels.apply_diagonal(a, dg, bits)
        kernels.apply_diagonal(b, dg, bits)
        np.testing.assert_allclose(a, b, atol=1e-12)
    with pytest.raises(ValueError):
        kernels.core_apply_gate(np.zeros((1, 4), complex), np.eye(4, dtype=complex), [0])
    big = np.zeros((1, 1 << 8), complex)
    big[0, 0] = 1
    kernels.apply_gate(big, np.linalg.qr(rng.normal(size=(128, 128)))[0].astype(complex), list(range(7)))
    assert abs(np.linalg.norm(big) - 1) < 1e-10


def test_async_out_download_and_pipelining():
    """run_plan(out=...) copies the final blocks on a copy stream: the result
    matches the device state, back-to-back runs with initial/out buffers
    pipeline correctly, and a wrongly shaped out is rejected."""
    from pathlib import Path

    import torch

    from paper_2509_14098_b200 import DimensionMismatch, gather, plan as planmod, run_plan

    plan = planmod.load(str(Path(__file__).resolve().parent.parent / "plans" / "qft20_h18-12.json.gz"))
    L = plan.d - plan.g
    rows = 1 << plan.g
    out = torch.empty((rows, 1 << L), dtype=torch.complex128).pin_memory()
    ref = run_plan(plan)
    want = ref.state.blocks.cpu()
    res = run_plan(plan, out=out).wait()
    assert torch.equal(out, want)
    # pipelined: each run uploads a different basis state and downloads its QFT
    outs, runs = [], []
    for x in (3, 77, 1000):
        init = torch.zeros(1 << plan.d, dtype=torch.complex128)
        init[x] = 1.0
        o = torch.empty((rows, 1 << L), dtype=torch.complex128).pin_memory()
        runs.append(run_plan(plan, initial=init, out=o))
        outs.append((x, o))
    for r, (x, o) in zip(runs, outs):
        r.wait()
        dense = gather(r.state)
        y = np.arange(1 << plan.d)
        exp = np.exp(-2j * np.pi * ((x * y) % (1 << plan.d)) / (1 << plan.d)) / 2 ** (plan.d / 2)
        assert np.max(np.abs(dense - exp)) < 1e-12
        assert torch.equal(o, r.state.blocks.cpu())
    with pytest.raises(DimensionMismatch):
        run_plan(plan, out=torch.empty(7, dtype=torch.complex128))
    del res


def test_deferred_finish_pipelining_and_drift():
    """run_plan(wait=False): results and stats complete at wait(); a drifted
    initial state raises NonUnitaryDrift from wait()."""
    from pathlib import Path

    import torch

    from paper_2509_14098_b200 import NonUnitaryDrift, plan as planmod, run_plan

    plan = planmod.load(str(Path(__file__).resolve().parent.parent / "plans" / "qft20_h18-12.json.gz"))
    rows, L = 1 << plan.g, plan.d - plan.g
    want = run_plan(plan).state.blocks.cpu()
    outs = [torch.empty((rows, 1 << L), dtype=torch.complex128).pin_memory() for _ in range(3)]
    runs = [run_plan(plan, out=o, wait=False) for o in outs]
    for r, o in zip(runs, outs):
        r.wait()
        assert torch.equal(o, want)
        assert r.stats.compute_seconds > 0
    bad = np.full(1 << plan.d, 0.5, dtype=complex)
    r = run_plan(plan, initial=bad, wait=False)
    with pytest.raises(NonUnitaryDrift):
        r.wait()
    with pytest.raises(ValueError):
        run_plan(plan, shots=10, wait=False)


def test_compare_propagates_nan():
    """numpy's argmax/max return NaN for a NaN amplitude, so the reference's
    compare() is NaN (and `compare(...) < tol` fails); the device reduction
    must not drop it (fmax would)."""
    import math

    from oracle import oracle as orc
    from paper_2509_14098_b200 import compare

    rng = np.random.default_rng(5)
    a = rng.normal(size=4096) + 1j * rng.normal(size=4096)
    for pos in (0, 1234, 4095):
        b = a.copy()
        b[pos] = complex(float("nan"), 0.0)
        assert math.isnan(orc.compare(a, b))
        assert math.isnan(compare(a, b)), pos
        assert math.isnan(compare(b, a)), pos
    assert compare(a, a) == 0.0


@pytest.mark.parametrize("nbits", [10, 11, 12, 13, 17, 22])
def test_layout_kernels_match_numpy(nbits):
    """svb_bitperm (tiled when a tile of <= 10 bits covers the low source
    and destination bits) and in-place svb_bitswap against numpy index math."""
    import torch

    from paper_2509_14098_b200 import _native

    lib = _native.load()
    rng = np.random.default_rng(nbits)
    n = 1 << nbits
    x = rng.normal(size=n) + 1j * rng.normal(size=n)
    src = torch.from_numpy(x).cuda()
    st = torch.cuda.current_stream().cuda_stream
    f = np.arange(n)
    for trial in range(6):
        perm = list(rng.permutation(nbits)) if trial else list(range(nbits - 1, -1, -1))
        dst = torch.empty_like(src)
        arr, p32 = _native.i32_array(perm)
        _native.check(lib.svb_bitperm(src.data_ptr(), dst.data_ptr(), nbits, p32, st), "svb_bitperm")
        p = np.zeros_like(f)
        for k in range(nbits):
            p |= ((f >> k) & 1) << perm[k]
        want = np.empty_like(x)
        want[p] = x
        assert np.array_equal(dst.cpu().numpy(), want), (nbits, perm)
    for trial in range(6):
        m = int(rng.integers(1, 4))
        bits = rng.permutation(nbits)[:2 * m]
        u = np.asarray(bits[:m], dtype=np.int32)
        w = np.asarray(bits[m:], dtype=np.int32)
        buf = src.clone()
        _native.check(lib.svb_bitswap(buf.data_ptr(), nbits, u.ctypes.data_as(_native._pi32),
                                      w.ctypes.data_as(_native._pi32), m, st), "svb_bitswap")
        p = f.copy()
        for a, b in zip(u, w):
            ba, bb = (f >> a) & 1, (f >> b) & 1
            p = (p & ~((1 << a) | (1 << b))) | (bb << a) | (ba << b)
        want = np.empty_like(x)
        want[p] = x
        assert np.array_equal(buf.cpu().numpy(), want), (nbits, u, w)


def test_gather_scatter_round_trip_30_qubits():
    """Bit-exact storage -> basis -> storage round trip of a 2^30-amplitude
    state in a reversed layout (the layout kernels at full size)."""
    import torch

    from paper_2509_14098_b200 import gather_device, scatter
    from paper_2509_14098_b200.executor import DistState
    from paper_2509_14098_b200.plan import ExecutionPlan

    d = 30
    layout = list(range(d - 1, -1, -1))
    plan = ExecutionPlan(d, 0, [layout], [])
    gen = torch.Generator(device="cuda").manual_seed(3)
    dense = torch.randn(1 << d, dtype=torch.complex128, device="cuda", generator=gen)
    st = scatter(dense, plan)
    back = gather_device(DistState(blocks=st.blocks, phase=0, d=d, g=0, layouts=[layout]))
    assert torch.equal(back, dense)
    # reversal: storage index f holds basis index reverse(f)
    f = torch.tensor([0, 1, 2, 12345, (1 << d) - 2], device="cuda")
    rev = torch.zeros_like(f)
    for k in range(d):
        rev |= ((f >> k) & 1) << (d - 1 - k)
    assert torch.equal(st.blocks.view(-1)[f], dense[rev])


def test_chunked_gather_matches_device_gather(grid_docs, monkeypatch):
    """The chunked host assembly (used for sharded and very large states)
    equals the device bit permutation, for every layout phase shape."""
    from paper_2509_14098_b200 import executor, gather_device, run_plan

    monkeypatch.setattr(executor, "GATHER_CHUNK_BITS", 3)
    n = 0
    for doc in grid_docs[::9]:
        plan = plan_from_doc(doc["plan"])
        if plan.d < 4:
            continue
        st = run_plan(plan).state
        want = gather_device(st).cpu().numpy()
        assert np.array_equal(executor._gather_chunked(st, None), want), doc["name"]
        n += 1
    assert n > 20
