"""B200-native batched evaluation of candidate device mappings for DNN task
graphs (the data-parallel hot path of DiviML, arXiv 2308.00127).

The public surface mirrors the reference package ``hetsched``: data model
(``core``), decoder and heuristics (``heuristics``), lower bound
(``bounds``) and the split heuristic's module solver (``splitting``). The
compute runs in hand-written sm_100a CUDA kernels behind the C ABI of
``include/hetsched_b200.h`` (``libhetsched_b200.so``); there is no CPU
fallback.
"""
from .core import (Device, DnnGraph, GraphError, HardwareSystem,
                   LatencyTable, Schedule, ScheduledBatch, ScheduleError,
                   TaskNode, bfs_topological_order, load_graph, load_hardware,
                   load_instance, load_latency, load_schedule, save_graph,
                   save_hardware, save_latency, save_schedule,
                   transitive_closure)
from .heuristics import (MappingGenome, argmin_batch, best_device, decode,
                         fitness, fitness_batch, fitness_batch_packed,
                         genome_from_map, greedy, met, pack_genes, pack_genes3,
                         one_plus_one_ea, random_search, simulated_annealing,
                         simulated_annealing_multi, one_plus_one_ea_multi,
                         specialize, throughput)
from .bounds import (BoundReport, critical_path_bound, critical_path_bounds,
                     dep_subgraph, lower_bound, pre_subgraph)
from .splitting import (ModuleDecomposition, ModuleSolver,
                        find_bridges_and_articulation_points,
                        gpu_module_solver, k_edge_components, milp_split)
from .batched import (batched_genes_from_schedule, batched_options,
                      decode_batched, fitness_batched, random_search_batched)
from .validate import validate_schedule, validate_schedules
from .modularity import (decomposition_modularity, modularity,
                         modularity_batch, modularity_split)

__version__ = "0.1.0"
