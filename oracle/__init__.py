"""CPU oracle of the reference path -- test infrastructure only (see cpu.py)."""
