"""B200-native batched AC power flow (drop-in for the `acpflow` batched-solve path).

Public names mirror the reference package's ``acpflow/__init__.py`` for the
hot path: loaders, model builders, scenario generation, the batch driver and
the two solvers, whose solves run on sm_100a kernels through libacpf.so
(``include/acpf.h``). See DESIGN.md.
"""

from .network import (AdmittanceMatrix, BranchRecord, BusKind, BusPartition, BusRecord,
                      CaseParseError, TransmissionNetwork, build_ybus, network_from_json,
                      network_to_json, parse_matpower_case, partition_buses)
from .distribution import (DistributionScenario, FixedPointOptions, FixedPointResult, LoadSpec,
                           SchemaError, SingularYbusError, ThreePhaseNetwork, VoltageFloorError,
                           ZBusModel, base_distribution_scenario, batch_zbus_solve,
                           build_three_phase_ybus, build_zbus_model, current_injection,
                           distribution_to_json, fixed_point_residual, kirchhoff_residual,
                           parse_distribution_json, read_reference_voltages, reduce_zbus,
                           zbus_iterate)
from .transmission import (GmresOptions, GpuNewtonSolver, NewtonOptions, NewtonResult, PolarState,
                           TransmissionModel, TransmissionScenario, base_scenario,
                           batch_newton_solve, branch_flows, build_transmission_model,
                           calc_injections, dense_jacobian, flat_start, mismatch, newton_solve)
from .batch import (BatchReport, ScenarioSpec, apply_multipliers, distribution_base,
                    generate_load_multipliers, make_scenario_arrays, make_scenarios,
                    report_to_csv, report_to_dict, run_batch, transmission_base)

__version__ = "0.1.0"
