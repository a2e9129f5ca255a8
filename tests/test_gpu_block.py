"""The per-block boundary (xlf_block_prepare / xlf_block_run), the successor
of run_fused_block (fused_exec.hpp:35-37, fused_exec.cpp:30-311):

* every fused block of the reference partition, fed the oracle's own values of
  its producer inputs (multi-input merge blocks included), stores tensors equal
  to the oracle's -- bit for bit in fp32_exact, within the tolerance in
  bf16 / TF32;
* a reference TilingPlan's geometry (plan_tiling text) drives the kernel's
  tile; a plan for another block is refused (validation), a geometry B200
  cannot hold is refused (infeasible);
* caller-owned NHWC buffers: the two expands of a fire block write straight
  into one caller concat buffer at their channel offsets;
* concurrent xlf_block_run calls from two threads on two streams."""
import threading

import numpy as np
import pytest

import paper_2007_06000_b200 as X
from oracle import oracle as O
from tests.conftest import graph_text

pytestmark = pytest.mark.gpu

TOL = {"fp32_exact": 0.0, "fp32": 1e-5, "tf32": 1e-3, "bf16": 1e-2}


def _oracle_values(name, batch):
    text = graph_text(name)
    og = O.load_graph(text)
    w = O.seeded_weights(og, 42)
    x = O.seeded_batch(og, 42, batch)
    vals = O.run_batch(og, x, w, [l.name for l in og.layers])
    vals[og.inputs[0][0]] = x
    return X.Graph(text), og, O.flat_weights(og, w), vals


@pytest.mark.parametrize("prec", ["fp32_exact", "bf16", "tf32"])
@pytest.mark.parametrize("name", ["a1", "a2", "b1", "c1", "residual", "inc3a", "squeezenet11"])
def test_every_reference_block(name, prec):
    import torch
    g, og, w, vals = _oracle_values(name, 2)
    blocks = [b for b in X.detect_fusion_blocks(g) if b.fused()]
    assert blocks
    for b in blocks:
        values = {k: torch.from_numpy(np.ascontiguousarray(v)).cuda() for k, v in vals.items()}
        for n in list(values):
            if n in b.members:
                del values[n]
        fits = [s for s in X.device_plan(g, "reference", 2, prec)["steps"] if s["id"] == b.id]
        if not fits:  # the B200 planner splits this block at this precision (a1 in TF32: 192-channel fp32 staging)
            with pytest.raises(X.XlfError) as ei:
                X.run_fused_block(g, b, values, w, precision=prec)
            assert ei.value.kind == "infeasible"
            continue
        written = X.run_fused_block(g, b, values, w, precision=prec)
        assert written
        for n in written:
            got = values[n].cpu().numpy()
            if prec == "fp32_exact":
                assert np.array_equal(got, vals[n]), (name, b.id, n)
            else:
                assert O.normwise(got, vals[n]) <= TOL[prec], (name, b.id, n, O.normwise(got, vals[n]))


def test_merge_block_reads_two_inputs():
    g = X.Graph(graph_text("residual"))
    merges = [b for b in X.detect_fusion_blocks(g) if b.mode == "merge"]
    assert merges
    blk = X.Block(g, merges[0], X.seeded_weights(g, 42), "fp32_exact")
    assert len(blk.inputs) >= 1 and blk.info["mode"] == "merge"


@pytest.mark.parametrize("prec", ["fp32_exact", "bf16"])
def test_plan_geometry_drives_the_kernel(prec):
    import torch
    g, og, w, vals = _oracle_values("b1", 1)
    b = [b for b in X.detect_fusion_blocks(g) if b.fused()][0]
    out_h, out_w = g.shape_of(b.consumer_stage[0])[1:]
    for th, tw in ((11, 11), (5, 9)):
        plan = X.plan_tiling(g, b.id, (th, tw), (-(-out_h // th), -(-out_w // tw)), "b200")
        blk = X.Block(g, b, w, prec, plan=plan)
        assert blk.info["plan_tile"] == [th, tw] and blk.info["tile_source"].startswith("plan")
        # the kernel runs the plan's tile or an exact sub-tile of it
        kt = blk.info["tile"]
        assert th % kt[0] == 0 and tw % kt[1] == 0, kt
        if prec == "fp32_exact":
            assert kt == [th, tw]
        x = torch.from_numpy(vals[blk.inputs[0]]).cuda()
        outs = {o: torch.empty((1,) + tuple(g.shape_of(o)), device="cuda") for o in blk.outputs}
        blk.run([X.Block.ref(x)], [X.Block.ref(outs[o]) for o in blk.outputs], 1)
        for o in blk.outputs:
            got = outs[o].cpu().numpy()
            assert (np.array_equal(got, vals[o]) if prec == "fp32_exact" else O.normwise(got, vals[o]) <= TOL[prec]), (th, tw, o)
    # a geometry that does not cover the output, another block's plan, an infeasible tile
    with pytest.raises(X.XlfError) as ei:
        X.Block(g, b, w, prec, plan=X.plan_tiling(g, b.id, (11, 11), (1, 1), "b200"))
    assert ei.value.kind == "validation"
    sq = X.Graph(graph_text("squeezenet11"))
    sb = [x for x in X.detect_fusion_blocks(sq) if x.fused()]
    foreign = X.plan_tiling(sq, sb[1].id, (9, 9), (7, 7), "b200")
    with pytest.raises(X.XlfError) as ei:
        X.Block(sq, sb[0], X.seeded_weights(sq, 42), prec, plan=foreign)
    assert ei.value.kind == "validation"
    # a plan tile too big for one CTA runs as exact sub-tiles of it
    fire2 = sb[0]
    h2, w2 = sq.shape_of(fire2.consumer_stage[0])[1:]
    blk = X.Block(sq, fire2, X.seeded_weights(sq, 42), prec, plan=X.plan_tiling(sq, fire2.id, (h2, w2), (1, 1), "b200"))
    kt = blk.info["tile"]
    assert blk.info["plan_tile"] == [h2, w2] and kt != [h2, w2] and h2 % kt[0] == 0 and w2 % kt[1] == 0


def _nhwc(t, cstride, dtype):
    import torch
    n, c, h, w = t.shape
    out = torch.zeros((n, h, w, cstride), dtype=dtype, device="cuda")
    out[..., :c] = t.permute(0, 2, 3, 1).to(dtype)
    return out


@pytest.mark.parametrize("prec", ["fp32_exact", "bf16", "tf32"])
def test_nhwc_caller_buffers_with_concat_offsets(prec):
    """fire: squeeze -> expand1 | expand3; both expands store into ONE caller
    buffer at channel offsets 0 and 64 (= the concat, no copy kernel)."""
    import torch
    g, og, w, vals = _oracle_values("b1", 2)
    b = [b for b in X.detect_fusion_blocks(g) if b.fused()][0]
    blk = X.Block(g, b, w, prec, max_batch=2)
    dt = torch.bfloat16 if prec == "bf16" else torch.float32
    assert blk.info["element_bytes"] == (2 if prec == "bf16" else 4)
    x = torch.from_numpy(vals[blk.inputs[0]]).cuda()
    xin = _nhwc(x, x.shape[1], dt)
    e1, e3 = blk.outputs  # stored_tensors order: the consumers
    c1, c3 = g.shape_of(e1)[0], g.shape_of(e3)[0]
    h, wd = g.shape_of(e1)[1:]
    cat = torch.full((2, h, wd, c1 + c3 + 16), float("nan"), dtype=dt, device="cuda")
    blk.run([X.Block.ref(xin, "nhwc")], [X.Block.ref(cat, "nhwc", coff=0), X.Block.ref(cat, "nhwc", coff=c1)], 2)
    torch.cuda.synchronize()
    got = cat[..., :c1 + c3].float().permute(0, 3, 1, 2).cpu().numpy()
    ref = np.concatenate([vals[e1], vals[e3]], axis=1)
    if prec == "fp32_exact":
        assert np.array_equal(got, ref)
    else:
        assert O.normwise(got, ref) <= TOL[prec]
    assert torch.isnan(cat[..., c1 + c3:].float()).all(), "wrote past the two slices"
    # misaligned offset / pitch are refused
    with pytest.raises(X.XlfError):
        blk.run([X.Block.ref(xin, "nhwc")], [X.Block.ref(cat, "nhwc", coff=3), X.Block.ref(cat, "nhwc", coff=c1)], 2)


def test_concurrent_runs_on_two_streams():
    import torch
    g, og, w, vals = _oracle_values("b1", 4)
    b = [b for b in X.detect_fusion_blocks(g) if b.fused()][0]
    blk = X.Block(g, b, w, "fp32_exact", max_batch=4)
    x = torch.from_numpy(vals[blk.inputs[0]]).cuda()
    res, errs = {}, []

    def work(k):
        try:
            s = torch.cuda.Stream()
            outs = {o: torch.empty((4,) + tuple(g.shape_of(o)), device="cuda") for o in blk.outputs}
            with torch.cuda.stream(s):
                for _ in range(20):
                    blk.run([X.Block.ref(x)], [X.Block.ref(outs[o]) for o in blk.outputs], 4, stream=s)
            s.synchronize()
            res[k] = outs
        except Exception as e:  # noqa: BLE001
            errs.append(e)

    ts = [threading.Thread(target=work, args=(k,)) for k in range(2)]
    for t in ts:
        t.start()
    for t in ts:
        t.join()
    assert not errs, errs
    for k in range(2):
        for o in blk.outputs:
            assert np.array_equal(res[k][o].cpu().numpy(), vals[o])
