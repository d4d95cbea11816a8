"""Diagnose a hang of the single-GPU local-group DP test: run one world=W
scenario with periodic Python stack dumps of every thread."""
import faulthandler
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "tests"))


def main():
    world = int(sys.argv[1]) if len(sys.argv) > 1 else 4
    faulthandler.dump_traceback_later(4, repeat=True, file=sys.stderr)
    import test_gpu_local as T
    T.test_local_dp_rounds(world)
    faulthandler.cancel_dump_traceback_later()
    print("OK world", world, flush=True)


if __name__ == "__main__":
    main()
