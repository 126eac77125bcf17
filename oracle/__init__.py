"""CPU ORACLE -- TEST INFRASTRUCTURE ONLY.

Clean-room, Eigen-free restatement of the reference's correction-step path
(/root/reference/proj). Loaded only by tests/, __graft_entry__.smoke() (as the
checker) and bench.py's cpu_baseline / --impl reference legs. The product
package never imports it.

Parity pin: the reference cannot be built in this image (Eigen3, doctest and
CLI11 are absent) and ships no golden vectors, so this
oracle is pinned by restated versions of the reference's own known-answer and
identity tests (tests/test_oracle_pins.py) -- not by reference outputs.
"""
from .binding import (OBlocks, OMesh, OOperator, Oracle, OracleError, dorfler_mark, gen_eig, keast, lib,  # noqa: F401
                      solve_bordered)
