"""bench.py's roofline model names every kernel of the covariance step (the
launch list of profiles/r08b_launches_cov_step.txt), so a renamed kernel
cannot silently drop out of the bench line's `roofline.all_kernels`."""
import importlib.util
from pathlib import Path

ROOT = Path(__file__).resolve().parent.parent


def _bench():
    spec = importlib.util.spec_from_file_location("bench_mod", ROOT / "bench.py")
    mod = importlib.util.module_from_spec(spec)
    spec.loader.exec_module(mod)
    return mod


STEP_KERNELS = {  # shared design (the bench workload)
    "k_oz_syrk", "k_oz_slice", "k_oz_colmax", "k_tphase2v", "k_pass_cols", "k_solve_sep_tri", "k_center_mirror",
}


def test_model_covers_the_step_kernels():
    b = _bench()
    model = b.kernel_model(64 * 64, 2000, True)
    missing = STEP_KERNELS - set(model)
    assert not missing, missing
    for name, (bound, work) in model.items():
        assert bound in ("hbm", "tensor", "int8"), name
        assert work > 0, name


def test_model_general_design_has_the_mass_path():
    b = _bench()
    model = b.kernel_model(64 * 64, 2000, False)
    for k in ("k_oz_syrk", "k_tphase2v", "k_pass_cols", "k_solve_tri", "k_center_mirror"):
        assert k in model, k


def test_launch_list_kernels_are_modelled():
    """Every kernel with a measurable share in the committed launch list of
    one covariance step has a model entry."""
    b = _bench()
    model = b.kernel_model(64 * 64, 2000, True)
    lst = (ROOT / "profiles" / "r08b_launches_cov_step.txt").read_text().splitlines()
    names = []
    for line in lst[1:]:
        parts = line.split()
        if not parts or parts[0] == "total":
            continue
        base = parts[0].split("::")[-1].split("<")[0]
        share = float(parts[-1])
        if share >= 0.02:
            names.append(base)
    assert names
    assert set(names) <= set(model), set(names) - set(model)
