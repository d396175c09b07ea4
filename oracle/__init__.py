"""CPU oracle of the reference planner path - test infrastructure only (see oracle.c)."""
