import sys, json, dataclasses
sys.path.insert(0, '.'); sys.path.insert(0, 'tests')
import bench
from oracle import interp_np as O
from paper_1905_02241_b200.ir import MechIR
from paper_1905_02241_b200.runner import CudaRunner, simulate
from paper_1905_02241_b200.metrics import parity
for st in ("K_Pst", "NaTs2_t", "Ca_HVA", "SKv3_1", "Ih", "hh_subset"):
    ir = MechIR.load(f'fixtures/ir/{st}.json')
    n = 8192
    ref = O.simulate(ir, O.init(ir, n, 7), 1000)
    opts = dataclasses.replace(bench.options_for(st), divc_approx=True)
    gpu = simulate(ir, O.init(ir, n, 7), 1000, runner=CudaRunner(ir, options=opts))
    dev, where = parity(ir, ref, gpu)
    print(json.dumps({"stem": st, "divc_approx": True, "dev": dev, "where": where}), flush=True)
