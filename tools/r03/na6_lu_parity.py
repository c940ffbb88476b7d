import sys, json, dataclasses
sys.path.insert(0, '.'); sys.path.insert(0, 'tests')
import bench
from oracle import interp_np as O
from paper_1905_02241_b200.ir import MechIR
from paper_1905_02241_b200.runner import CudaRunner, simulate
from paper_1905_02241_b200.metrics import parity
ir = MechIR.load('fixtures/ir/na6.json')
n = 8192
ref = O.simulate(ir, O.init(ir, n, 7), 1000)
for la in (0, 1, 2, 3):
    opts = dataclasses.replace(bench.options_for('na6'), lu_approx=la)
    gpu = simulate(ir, O.init(ir, n, 7), 1000, runner=CudaRunner(ir, options=opts))
    dev, where = parity(ir, ref, gpu)
    print(json.dumps({"lu_approx": la, "dev": dev, "where": where, "iters_equal": gpu.newton_iters == ref.newton_iters}), flush=True)
