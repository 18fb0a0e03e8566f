"""CPU oracle — TEST INFRASTRUCTURE ONLY (see castfem_oracle.c header)."""
