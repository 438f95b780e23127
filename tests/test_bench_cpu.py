"""bench.py host logic that needs no GPU: the per-strategy table covers exactly
the 14 codes Principle 1 allows (Table 1), and every one of them
plans on the bench's own launch configuration at the 2x4 split of BASELINE
configs[1] with the footprint fields the OOM check reads."""
import bench
from oracle import strategy as S
from paper_2310_06003_b200 import paro
from paro_synth import llama_param_sizes


def test_strategy_list_is_table1():
    assert sorted(bench.STRATEGIES) == sorted(S.paro_strategies())
    assert len(set(bench.STRATEGIES)) == 14


def test_every_code_plans_with_bench_options_at_2x4():
    args = bench.parse(["--gpus", "8"])
    assert args.strategy_steps > 0
    ctx = paro.Context(8, bench.default_group(8))
    sizes = llama_param_sizes(args.model)
    for code in bench.STRATEGIES:
        pl = paro.Plan(ctx, code, sizes, **bench.plan_kwargs(args, None))
        i = pl.info()
        pl.close()
        foot = (i["grad_buffer_bytes"] + i["mem_p_bytes"] + (i["mem_g_bytes"] if i["g_numel"] > 0 else 0)
                + i["mem_os_bytes"] + i["workspace_bytes"])
        assert 0 < foot < 180e9, (code, foot)          # all 14 fit a B200 at 2x4
        assert i["psi"] == 6738415616
    ctx.close()
