"""plansim-b200: B200-native evaluate-all-plans engine for APEX-style plan search.

Drop-in for plansim::search (/root/reference/proj/src/simulator.cpp:242-296);
see DESIGN.md and include/psg.h.
"""
from .errors import DataError, InfeasibleError, PlanSearchError  # noqa: F401
from .inputs import Cluster, Config, Plans, Store, Trace  # noqa: F401
