"""smoke() with a traceback dump if it hangs (GPU debugging aid)."""
import faulthandler
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
faulthandler.dump_traceback_later(int(sys.argv[1]) if len(sys.argv) > 1 else 120, exit=True)
import __graft_entry__ as g  # noqa: E402

g.smoke()
print("smoke returned", flush=True)
