"""cProfile of the facade producer loop (HBM store, 4 host-sync consumers)."""
import cProfile
import os
import pstats
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

if __name__ == "__main__":
    import tools.facade_rate as fr

    pr = cProfile.Profile()
    pr.enable()
    sys.argv = ["x", "1500", "host"]
    fr.main()
    pr.disable()
    pstats.Stats(pr).sort_stats("tottime").print_stats(30)
