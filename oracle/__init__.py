"""Float64 CPU oracle (TEST INFRASTRUCTURE ONLY -- see oracle/cascade.py header)."""
from .cascade import *  # noqa: F401,F403
