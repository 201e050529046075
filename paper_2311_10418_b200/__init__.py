"""B200-native DynaPipe micro-batch planner.

The ctypes binding lives in ``paper_2311_10418_b200.capi`` and is imported on
demand so that ``build`` can run before the shared library exists.
"""
