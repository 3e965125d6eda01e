"""Import the unmodified reference package compiled into oracle/_ref/ (by
oracle/build_ref.sh) -- test infrastructure: the reference itself as the
checker.  Returns None when the build is absent."""

import os
import sys

REF = os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "oracle", "_ref")


def reference():
    if not os.path.isdir(os.path.join(REF, "refusion")):
        return None
    if REF not in sys.path:
        sys.path.insert(0, REF)
    os.environ.setdefault("REFUSION_BACKEND", "compiled")
    import refusion.geometry as G
    import refusion.keyframe_fusion as KF
    import refusion.volume as V

    return {"G": G, "KF": KF, "V": V}
