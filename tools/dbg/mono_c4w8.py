"""c4w8 monodomain reference only (for ncu launch lists; debugging aid)."""
import sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
import kfp_inputs as ki
from paper_1306_4596_b200 import Problem
run = ki.scaled(ki.config("c4w8"), nt=20, t_final=0.01 / 500 * 20)
with Problem(ki.make_problem(run)) as pb:
    pb.monodomain(copy=False)
