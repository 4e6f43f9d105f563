import sys; sys.path[:0] = ['.', 'tests']
import paper_1808_10580_b200 as S, specs
ctx = S.default_context(0)
spec = specs.c3_spec()
e = S.observe_bvp(spec, 606, ctx=ctx)
print("steps", ctx.stats().particle_steps, "obs0", e[0].mean, e[0].aux_mean)
