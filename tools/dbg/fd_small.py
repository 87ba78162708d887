"""Small IMEX FD solve (debugging aid)."""
import sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
import kfp_inputs as ki
from paper_1306_4596_b200 import kfp
run = ki.config("c0")
with kfp.Problem(ki.make_problem(run)) as pb:
    print(pb.monodomain()[5, :4])
