import sys; sys.path.insert(0, '.')
from paper_2603_15202_b200 import workloads as W
from paper_2603_15202_b200.trace import generate_synthetic_device, generate_synthetic_packed
import numpy as np
spec = W.chat_spec(3000, 48.0, 0)
a = generate_synthetic_device(spec); b = generate_synthetic_packed(spec)
print(len(a), all(np.array_equal(getattr(a,c).view('u8'), getattr(b,c).view('u8')) for c in ('arrival_s','blocks','blk_off','out_tokens','class_key')))
