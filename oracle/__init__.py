"""TEST INFRASTRUCTURE ONLY — the CPU parity oracle (see oracle/svt_oracle.hpp)."""
