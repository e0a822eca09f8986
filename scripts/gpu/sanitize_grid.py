import sys, os
sys.path[:0] = [os.getcwd(), os.path.join(os.getcwd(), "src"), os.path.join(os.getcwd(), "tests")]
from conftest import load_case
from gpu_helpers import run_device
prob, cfg, out = load_case("tests/golden/lm_ba_all_visible.npz")
cfg["max_iters"] = 3
d = run_device([prob], cfg, "f64", kernel="grid")[0]
print(d["costs"])
