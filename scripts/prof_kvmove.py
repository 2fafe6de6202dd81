"""One staged evict + restore of 2048 scattered Llama-3-8B blocks (for an ncu
capture of the KV movers: k_kv_stage and the copy-engine DMAs)."""
import os, sys
sys.path.insert(0, os.getcwd())
import numpy as np
from paper_2604_26963_b200.engine import MarsEngine
from paper_2604_26963_b200.kvstore import LLAMA3_8B_BLOCK_BYTES, LLAMA3_8B_LAYERS, KvBlockManager
eng = MarsEngine(max_rows=64, max_queue=1)
kv = KvBlockManager(eng, 8192, max_blocks_per_row=16, block_bytes=LLAMA3_8B_BLOCK_BYTES,
                    layers=LLAMA3_8B_LAYERS, host_blocks=2048)
ids = np.random.default_rng(3).choice(8192, size=2048, replace=False).astype(np.uint32)
for _ in range(2):
    kv.evict(ids, 0, 2)
    kv.restore(ids, 0, 2)
print("ok")
