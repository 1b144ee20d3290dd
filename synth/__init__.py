"""Seeded synthetic road networks and trips.

This package is the ONLY code shared between the oracle tests and the CUDA
path: it builds inputs (lane-graph CSR + trip lists) and holds none of the
method's arithmetic (no IDM, MOBIL, signal or ordering logic).
"""
from .networks import (save_scenario, load_scenario, rcb_partition, NetBuilder, Scenario, ring, grid, city, tiled_city, pressure_junction, batch,
                       default_params, default_profiles, TURN_STRAIGHT,
                       TURN_LEFT, TURN_RIGHT, KIND_NORMAL, KIND_DYNAMIC,
                       KIND_TIDAL, POLICY_NONE, POLICY_FIXED, POLICY_MANUAL, POLICY_MAXP)
from .states import random_state

__all__ = ["save_scenario", "load_scenario", "rcb_partition", "NetBuilder", "Scenario", "ring", "grid", "city", "tiled_city",
           "default_params", "default_profiles", "random_state",
           "TURN_STRAIGHT", "TURN_LEFT", "TURN_RIGHT", "KIND_NORMAL",
           "KIND_DYNAMIC", "KIND_TIDAL", "POLICY_NONE", "POLICY_FIXED",
           "POLICY_MANUAL", "POLICY_MAXP"]
