"""Walker-sharded Dirichlet map vs one device at C3 shapes (5e3 / 1e5 / 1e6
walkers per observation), emulated groups of 2 and 8 members on device 0,
concurrent (SMC_GROUP_SERIAL=0) and serialised (=1).  Prints the largest
mean / SE / exit-time differences and any count mismatch; all must be 0.
(The serialised runs exposed the staging race fixed in round 2.)

    python tools/bvp_shard_check.py
"""
import os, sys
sys.path[:0] = ['.', 'tests']
os.environ["SMC_GROUP_EXCHANGE"] = "emulated"
import paper_1808_10580_b200 as S, specs
base = S.default_context(0)
for n in [5000, 100000, 1000000]:
    spec = specs.c3_spec(n_particles=n)
    ref = S.observe_bvp(spec, 606, ctx=base)
    for serial in ["0", "1"]:
        os.environ["SMC_GROUP_SERIAL"] = serial
        for w in [2, 8]:
            ctx = S.Context(devices=[0] * w)
            got = S.observe_bvp(spec, 606, ctx=ctx)
            dm = max(abs(a.mean - b.mean) for a, b in zip(got, ref))
            ds = max(abs(a.std_error - b.std_error) for a, b in zip(got, ref))
            dn = [(a.n_particles, b.n_particles, a.n_failed, b.n_failed) for a, b in zip(got, ref) if a.n_particles != b.n_particles or a.n_failed != b.n_failed]
            da = max(abs(a.aux_mean - b.aux_mean) for a, b in zip(got, ref))
            print(n, "serial", serial, "W", w, "dmean", dm, "dse", ds, "daux", da, "counts", dn[:3], flush=True)
            del ctx
