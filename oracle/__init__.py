"""TEST INFRASTRUCTURE ONLY: CPU oracle for the LDG path (see ldg_oracle.py)."""
