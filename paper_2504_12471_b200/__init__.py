"""B200-native D2FT hot path: scheduler, compaction and the subnet-skipping
fine-tuning step on sm_100a, behind the C-ABI in include/d2ft_b200.h."""
from ._lib import Error  # noqa: F401
from .scheduler import (  # noqa: F401
    BudgetSpec, Capacities, CostModel, CostTables, DpResult, ScalerConfig, ScalerResult, ScheduleTable,
    ScoreTable, Scheduler, brute_force_schedule, build_cost_tables, capacities_from_budget, check_shared_budget, compact, dp_search,
    knapsack_schedule, merge_selections, row_cost_units, scaler_schedule, schedule_objective)
