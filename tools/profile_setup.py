"""A short config-2 run for ncu captures of the plan builds and the
stochastic weigh pass: one deterministic and one stochastic
reconstruct_channel call of 3 iterations (public API)."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import torch  # noqa: E402

from tests.fullsize_common import device_loop  # noqa: E402
from workloads import CONFIGS, device_scene  # noqa: E402

torch.cuda.set_device(0)
sc = device_scene(*CONFIGS[2])
device_loop(sc, 3, "plan", record=False)
device_loop(sc, 3, "plan", record=False, deterministic=False)
torch.cuda.synchronize()
print("ok")
