"""Shows the race the binding's cudaStreamLegacy mapping removes: with torch's default stream passed as
0 ("no stream": the library's own unordered stream), a device-pointer call that follows unsynchronised
torch work reads stale inputs.  Runs tests/test_gpu_streams.py's ordering test under the old mapping.
    python tools/stream_race_demo.py"""
import importlib.util
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
from paper_2202_12674_b200 import binding as B  # noqa: E402

spec = importlib.util.spec_from_file_location("tgs", os.path.join(ROOT, "tests", "test_gpu_streams.py"))
T = importlib.util.module_from_spec(spec)
spec.loader.exec_module(T)
B.CUDA_STREAM_LEGACY = 0  # the old behaviour
try:
    T.test_device_pointer_call_is_ordered_after_torch_default_stream()
    print("old mapping: PASSED (race not observed)")
except AssertionError as e:
    print("old mapping: FAILED as expected, relative error", str(e)[:80])
