"""Run a script with a faulthandler stack dump after 40 s (hang diagnosis under torchrun):
    python -m torch.distributed.run ... tools/trace_run.py bench.py <args>"""
import faulthandler, runpy, sys
faulthandler.dump_traceback_later(40, exit=True)
sys.argv = sys.argv[1:]
runpy.run_path(sys.argv[0], run_name="__main__")
