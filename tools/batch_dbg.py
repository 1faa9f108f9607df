import sys, numpy as np
sys.path.insert(0, ".")
import paper_1805_06604_b200 as E
def prob(m, n, r, s):
    rng = np.random.default_rng(s)
    return rng.random((m, r)) @ rng.random((r, n)), rng.random((m, r)), rng.random((r, n))
cfg = E.algorithm_config("e-ahals-hp3"); cfg.max_outer_iterations = 6
case = sys.argv[1]
if case == "a": probs = [prob(500, 2100, 100, i) for i in range(3)]
elif case == "b": probs = [prob(300, 260, 20, i) for i in range(3)]
elif case == "c": probs = [prob(500, 2100, 100, 1), prob(300, 260, 20, 2)]
elif case == "d": probs = [prob(500, 2100, 100, i) for i in range(2)]
elif case == "e": probs = [prob(2100, 500, 100, i) for i in range(2)]
try:
    out = E.run_batch(probs, cfg, streams=4)
    print(case, "ok", [o.column("error")[-1] for o in out])
except Exception as ex:
    print(case, "FAIL", ex)
