"""cProfile of detect_pattern on the 32768^2 stand-in (host-side phases)."""
import cProfile, os, pstats, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import paper_2105_01170_b200 as bt
from paper_2105_01170_b200 import configs

patg, blocks = configs.gather_standin()
a = bt.struct_assemble(patg, torch.from_numpy(blocks).cuda())
bt.detect_pattern(a, patg.m, patg.n)
torch.cuda.synchronize()
pr = cProfile.Profile()
pr.enable()
bt.detect_pattern(a, patg.m, patg.n)
torch.cuda.synchronize()
pr.disable()
pstats.Stats(pr).sort_stats("cumtime").print_stats(25)
