"""Golden fixtures for the "ref" route on 3D nested Kuhn chains (the route of
BASELINE configs[2], at a size the reference runs in seconds).

    python tests/golden/make_ref3d.py

Runs the UNMODIFIED reference (/root/reference/pkg/src) on chains built by
``kuhn.kuhn_chain`` (refine()-style vertex numbering)
and stores inputs + outputs like make_golden.py.
"""
import os
import sys

HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, HERE)

from make_golden import kuhn, run_case  # noqa: E402


def main():
    # configs[2]'s coefficient field and shift on the chain 2 -> 4 -> 8
    s, meshes, rmaps = kuhn.config_chain("c3", 8, 2)
    run_case("kuhn8_c3ref", s, "ref", meshes, rmaps, full=False)
    # the 1e6 checkerboard (configs[1]'s field) on the same chain
    s, meshes, rmaps = kuhn.config_chain("c2", 8, 2)
    run_case("kuhn8_c2ref", s, "ref", meshes, rmaps, full=False)


if __name__ == "__main__" and not (len(sys.argv) > 1 and sys.argv[1] == "more"):
    main()


def more_fields():
    """configs[3] (64 seeded inclusions, beta 1e-4) and configs[4] (8^3
    checkerboard 1 / 1e6) coefficient fields on the n = 8 cube, "alg" route."""
    run_case("kuhn8_c4", kuhn.config_system("c4", n=8), "alg", full=False)
    run_case("kuhn8_c5", kuhn.config_system("c5", n=8), "alg", full=False)


if __name__ == "__main__" and len(sys.argv) > 1 and sys.argv[1] == "more":
    more_fields()
