"""cProfile of a few c2 outer steps (host-side overhead hunt; development aid)."""
import cProfile, os, pstats, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
sys.argv = [sys.argv[0]]
exec(open(os.path.join(os.path.dirname(os.path.abspath(__file__)), "prof_solve_timeline.py")).read().split("run(2)")[0])
run(2)
pr = cProfile.Profile()
pr.enable()
run(4)
pr.disable()
st = pstats.Stats(pr)
st.sort_stats("tottime").print_stats(25)
