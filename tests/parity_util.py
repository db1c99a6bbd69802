"""Shared helpers for the GPU-vs-oracle parity tests (tests only)."""
from __future__ import annotations

import dataclasses

import numpy as np

INT_FIELDS = ("queries", "hit_tokens", "input_tokens", "probes", "inserted_blocks", "evictions",
              "rlt_draws", "rlt_resets", "rlt_fallbacks", "max_pending", "decision_digest", "status")
FP_FIELDS = ("sum_latency_ms", "sum_ttft_ms", "max_latency_ms", "makespan_ms",
             "last_completion_ms", "sum_load_ms")
# north_star: decisions and counts bit-exact; latency/TTFT/makespan aggregates within 1e-12 rel.
# Both sides evaluate the same fp64 expressions in the same order without contraction, so the
# test demands bit equality and reports the relative error if that ever fails.
FP_RTOL = 1e-12


def to_oracle_policy(oracle, pol):
    d = dataclasses.asdict(pol)
    return oracle.OraclePolicy(**d)


def run_oracle(oracle, tr, W, B, pols, keys, truth, ring, record, victims_cap, bins=0):
    cfg = oracle.OracleConfig(W=W, capacity_blocks=B, alpha_cached_ms=truth[0],
                              alpha_miss_ms=truth[1], out_ms_per_token=truth[2],
                              pending_ring=ring, latency_hist_bins=bins)
    outs = []
    for k, pol in zip(keys, pols):
        r = oracle.run(cfg, tr, to_oracle_policy(oracle, pol), int(k), record=record,
                       victims_cap=victims_cap)
        assert r.rc == 0, r.rc
        outs.append(r)
    return outs


def run_gpu(kvr, traces, W, B, pols, keys, truth, ring, record, victims_cap, force_tier=0,
            trial_trace=None, bins=0, next_use=False):
    from paper_2601_18999_b200.kvr import DeviceTrace, Simulator, policies_array
    dts = [DeviceTrace(t) for t in traces]
    if next_use:   # offline OPT trials need the next-use index
        dts = [d.with_next_use() for d in dts]
    sim = Simulator(W, B, alpha_cached_ms=truth[0], alpha_miss_ms=truth[1],
                    out_ms_per_token=truth[2], pending_ring=ring,
                    record_trials=len(keys) if record else 0, force_tier=force_tier,
                    latency_hist_bins=bins)
    out = sim.run(dts, np.asarray(keys, np.uint64), policies_array(pols),
                  trial_trace=trial_trace, victims_cap=victims_cap * len(keys) if record else 0)
    return out, dts, sim


# the batching engine sums latency / TTFT per worker and adds the partial sums in
# worker order (kvr_batch.cu); the oracle sums them in query order (the plain
# definition).  The north star bounds those aggregates at 1e-12 relative.
BATCH_SUM_FIELDS = ("sum_latency_ms", "sum_ttft_ms")
REL_TOL = 1e-12


def assert_result_equal(g, o, ctx="", rel_fields=()):
    for f in INT_FIELDS:
        assert int(g[f]) == int(o[f]), f"{ctx} field {f}: gpu {int(g[f])} oracle {int(o[f])}"
    for f in FP_FIELDS:
        gv, ov = float(g[f]), float(o[f])
        rel = abs(gv - ov) / max(abs(ov), 1e-300)
        if f in rel_fields:
            assert gv == ov or rel <= REL_TOL, f"{ctx} field {f}: gpu {gv!r} oracle {ov!r} rel {rel:.3e}"
        else:
            assert gv == ov, f"{ctx} field {f}: gpu {gv!r} oracle {ov!r} rel {rel:.3e}"


def assert_records_equal(grec, orec, n, ctx=""):
    for fld in ("worker", "hit_tokens", "n_victims", "victim_offset"):
        a, b = grec[fld][:n], orec[fld][:n]
        if not np.array_equal(a, b):
            j = int(np.nonzero(a != b)[0][0])
            raise AssertionError(f"{ctx} record {fld} differs first at query {j}: "
                                 f"gpu {a[j]} oracle {b[j]}")
    for fld in ("ttft_ms", "latency_ms", "score"):
        a, b = grec[fld][:n], orec[fld][:n]
        if not np.array_equal(a, b, equal_nan=True):   # NaN payloads differ CPU vs GPU
            j = int(np.nonzero(a != b)[0][0])
            raise AssertionError(f"{ctx} record {fld} differs first at query {j}: "
                                 f"gpu {a[j]!r} oracle {b[j]!r}")


def compare(oracle, kvr, tr, W, B, pols, keys, truth=(0.0, 1.0, 20.0), ring=256, record=True,
            victims_cap=None, force_tier=0, bins=0, next_use=False):
    n = tr.n_queries
    if victims_cap is None:
        victims_cap = max(1, tr.total_blocks)
    out, _, _ = run_gpu(kvr, [tr], W, B, pols, keys, truth, ring, record, victims_cap,
                        force_tier=force_tier, bins=bins, next_use=next_use)
    orc = run_oracle(oracle, tr, W, B, pols, keys, truth, ring, record, victims_cap, bins=bins)
    for t, o in enumerate(orc):
        ctx = f"trial {t} key {keys[t]} pol {pols[t]}"
        g = out.results[t]
        if o.result["status"] == 1 or int(g["status"]) == 1:   # ring overflow: stop point only
            assert int(g["status"]) == o.result["status"] and int(g["queries"]) == o.result["queries"], ctx
            continue
        assert_result_equal(g, o.result, ctx)
        if record:
            assert_records_equal(out.records[t], o.records, n, ctx)
            nv = int(o.result["evictions"])
            gv = out.victims[t * victims_cap: t * victims_cap + min(nv, victims_cap)]
            assert np.array_equal(gv, o.victims[: min(nv, victims_cap)]), ctx + " victims"
        if bins:
            assert np.array_equal(out.hist[t], o.hist), ctx + " hist"
    return out, orc


# ------------------------------------------------------------ continuous batching
def compare_batched(oracle, kvr, tr, W, B, beta, pols, keys, truth=(0.0, 1.0, 20.0), ring=256,
                    record=True, victims_cap=None, force_tier=0, bins=0):
    """GPU batching kernel (kvr_batch.cu) vs the oracle's batching engine (A30-A36).
    Trials with a nonzero status compare the status only (counters unspecified)."""
    from paper_2601_18999_b200.kvr import DeviceTrace, Simulator, policies_array
    n = tr.n_queries
    if victims_cap is None:
        victims_cap = W * max(1, tr.total_blocks)
    sim = Simulator(W, B, alpha_cached_ms=truth[0], alpha_miss_ms=truth[1],
                    out_ms_per_token=truth[2], pending_ring=ring,
                    record_trials=len(keys) if record else 0, force_tier=force_tier,
                    latency_hist_bins=bins, batch_slots=beta)
    out = sim.run(DeviceTrace(tr), np.asarray(keys, np.uint64), policies_array(pols),
                  victims_cap=victims_cap * len(keys) if record else 0)
    cfg = oracle.OracleConfig(W=W, capacity_blocks=B, alpha_cached_ms=truth[0],
                              alpha_miss_ms=truth[1], out_ms_per_token=truth[2],
                              pending_ring=ring, latency_hist_bins=bins, batch_slots=beta)
    orc = []
    for t, (k, pol) in enumerate(zip(keys, pols)):
        o = oracle.run(cfg, tr, to_oracle_policy(oracle, pol), int(k), record=record,
                       victims_cap=victims_cap)
        assert o.rc == 0, o.rc
        orc.append(o)
        ctx = f"batched beta={beta} trial {t} key {k} pol {pol}"
        g = out.results[t]
        if o.result["status"] not in (0, 2) or int(g["status"]) not in (0, 2):
            assert int(g["status"]) == o.result["status"], ctx
            continue
        assert_result_equal(g, o.result, ctx, rel_fields=BATCH_SUM_FIELDS)
        if record:
            assert_records_equal(out.records[t], o.records, n, ctx)
            gv = out.victims[t * victims_cap:(t + 1) * victims_cap]
            for j in range(n):
                off, nv = int(o.records[j]["victim_offset"]), int(o.records[j]["n_victims"])
                hi = min(off + nv, (int(o.records[j]["worker"]) + 1) * (victims_cap // W))
                if hi > off:
                    assert np.array_equal(gv[off:hi], o.victims[off:hi]), f"{ctx} victims q{j}"
        if bins:
            assert np.array_equal(out.hist[t], o.hist), ctx + " hist"
    return out, orc
