// Level-batched netlist runner (replaces hvp::netlist::Evaluator<TfheBackend>,
// engine.hpp:107-405, engine.cpp:113-148).  Included by vsp_capi.cu after the launch
// helpers.
//
// The reference list-schedules individual cells onto host threads (engine.hpp:263-351).
// Every cell's output is a deterministic function of its inputs, so evaluating the
// DAG one ASAP level at a time (Dag::level, netlist.cpp:387-406) yields bit-identical
// values; each level's gates become ONE batched gate-bootstrap launch sequence, and
// the memory ports of the level run the batched CMUX-memory pipeline.  The value
// table, DFF state and the RAM image stay resident in HBM across cycles.
//
// With a communicator attached (vsp_attach_comm) every rank runs the same runner on its
// own GPU: each level's gates are sharded across the ranks and all-gathered
// (hom_gate_level_dev, multi.cuh); memory ports run replicated (identical deterministic
// results on every rank), so the DFF latch stays rank-local.
#pragma once

namespace vsp {

// hvp::netlist::CellKind order (netlist.hpp:12-28)
enum CellKindDev : int {
    cAnd = 0, cAndNot, cMux, cNand, cNor, cNot, cOr, cOrNot, cXnor, cXor,
    cDff, cRom, cRam, cConst0, cConst1
};

__global__ void gather_tlwe_kernel(const int* __restrict__ nets, int count,
                                   const uint32_t* __restrict__ values, uint32_t* __restrict__ out,
                                   int n)
{
    const int c = blockIdx.x;
    if (c >= count)
        return;
    const int net = nets[c];
    for (int k = threadIdx.x; k <= n; k += blockDim.x)
        out[(size_t)c * (n + 1) + k] = net >= 0 ? values[(size_t)net * (n + 1) + k] : 0u;
}

__global__ void scatter_tlwe_kernel(const int* __restrict__ nets, int count,
                                    const uint32_t* __restrict__ src, uint32_t* __restrict__ values,
                                    int n)
{
    const int c = blockIdx.x;
    if (c >= count)
        return;
    const int net = nets[c];
    if (net < 0)
        return;
    for (int k = threadIdx.x; k <= n; k += blockDim.x)
        values[(size_t)net * (n + 1) + k] = src[(size_t)c * (n + 1) + k];
}

}  // namespace vsp

struct vsp_netlist {
    vsp_ctx* ctx = nullptr;
    std::string name;  // Netlist::name (snapshots record it with netlistHash)
    int nets = 0;
    std::vector<int> kind, id, in_off, in_nets, out_off, out_nets;
    // DAG (buildDag, netlist.cpp:348-432)
    std::vector<int> dag_cells, level, height, dff_cells;
    std::vector<int> launch_level;  // per DAG node: the level it is evaluated in (build_dag)
    std::vector<int> level_tasks;   // blind-rotation tasks of each launch level's gates
    // per launch level: the gates' input nets [G][3] then output nets [G], device resident
    // (uploaded once), so a level reads and writes the value table in place
    DevBuf lvl_nets;
    std::vector<size_t> lvl_off;
    std::vector<std::vector<int32_t>> lvl_kinds;
    // the cycle as a CUDA graph (one GPU): captured after an eager warm-up cycle at the
    // same buffer / option generations, replayed while they hold
    cudaGraphExec_t gexec = nullptr;
    uint64_t g_buf = ~0ull, g_opt = ~0ull, ready_buf = ~0ull, ready_opt = ~0ull;
    uint64_t g_launches = 0, g_counters[5] = {0, 0, 0, 0, 0};
    PinnedArena arena;
    std::vector<int> node_of_cell;
    int rom_cell = -1, ram_cell = -1, gmax = 0, depth = 0;
    // per level: gate cells (kinds 0..9) and memory ports
    std::vector<std::vector<int>> level_gates, level_mem;
    std::vector<int> const_cells;
    // device state
    DevBuf values, dff, gin, gout, nets_buf, inputs_store;
    std::vector<int> input_nets;     // nets driven by module inputs (setInput targets)
    std::vector<uint8_t> is_input;   // net -> is module input
    std::vector<int> dff_q, dff_d;   // per DFF: output net (Q), input net (D)
    bool table_valid = false;
    uint64_t cycle = 0;
    // the largest narrow level's CTAs with two tasks per SM (ram_overlap partition)
    int max_level_ctas = 0;
    // memory ports
    DevBuf ram, rom;
    uint32_t ram_v = 0, ram_w = 0, rom_depth = 0, rom_nluts = 0;
    bool has_ram = false, has_rom = false;
};

namespace {

[[noreturn]] void nl_fail(const std::string& m) { throw std::runtime_error("netlist: " + m); }

const char* cell_kind_name(int k)  // cellKindName (netlist.cpp:47-80)
{
    static const char* names[] = {"AND", "ANDNOT", "MUX", "NAND", "NOR", "NOT", "OR", "ORNOT",
                                  "XNOR", "XOR", "DFF", "ROM", "RAM", "CONST0", "CONST1"};
    return k >= 0 && k <= cConst1 ? names[k] : "?";
}

// validateNetlist (netlist.cpp:265-345) on the flat C-ABI arrays, with the reference's
// messages.  The flat form also has to enforce what the reference's JSON schema gives
// for free (netlist.cpp:106-199): known kinds, one output per gate / DFF / constant.
void validate_netlist(const vsp_netlist* nl)
{
    const int C = (int)nl->kind.size();
    const int nets = nl->nets;
    std::unordered_set<int> ids;
    for (int i = 0; i < C; i++) {
        if (nl->kind[i] < 0 || nl->kind[i] > cConst1)
            throw std::invalid_argument("netlist: unknown cell kind");
        if (!ids.insert(nl->id[i]).second)
            nl_fail("duplicate cell id " + std::to_string(nl->id[i]));
    }
    std::vector<int> driver(nets, -1);  // -2 module input, else cell index
    for (int b : nl->input_nets) {
        if (b < 0 || b >= nets)
            nl_fail("input port 'in' references bad net " + std::to_string(b));
        if (driver[b] != -1)
            nl_fail("multiple drivers on net " + std::to_string(b));
        driver[b] = -2;
    }
    int roms = 0, rams = 0;
    for (int i = 0; i < C; i++) {
        const int k = nl->kind[i];
        const int nin = nl->in_off[i + 1] - nl->in_off[i];
        const int nout = nl->out_off[i + 1] - nl->out_off[i];
        const std::string who = "cell " + std::to_string(nl->id[i]) + " (" + cell_kind_name(k) + ")";
        int arity = 2;
        if (k == cNot || k == cDff)
            arity = 1;
        else if (k == cMux)
            arity = 3;
        else if (k == cConst0 || k == cConst1)
            arity = 0;
        else if (k == cRom || k == cRam)
            arity = nin;
        if (nin != arity)
            nl_fail(who + " has wrong input count");
        if (k == cRom) {
            roms++;
            if (nout != 32)
                nl_fail("ROM port must have 32 rdata bits");
            if (nin == 0)
                nl_fail("ROM port needs address bits");
        }
        else if (k == cRam) {
            rams++;
            if (nout == 0 || nin < nout + 2)
                nl_fail("RAM port pin widths are inconsistent");
        }
        else if (nout != 1) {
            nl_fail(who + " must drive exactly one net");
        }
        for (int q = nl->out_off[i]; q < nl->out_off[i + 1]; q++) {
            const int b = nl->out_nets[q];
            if (b < 0 || b >= nets)
                nl_fail("cell " + std::to_string(nl->id[i]) + " drives bad net " + std::to_string(b));
            if (driver[b] != -1)
                nl_fail("multiple drivers on net " + std::to_string(b) + " (cell " +
                        std::to_string(nl->id[i]) + ")");
            driver[b] = i;
        }
    }
    for (int i = 0; i < C; i++)
        for (int q = nl->in_off[i]; q < nl->in_off[i + 1]; q++) {
            const int b = nl->in_nets[q];
            if (b < 0 || b >= nets || driver[b] == -1)
                nl_fail("dangling input net " + std::to_string(b) + " on cell " +
                        std::to_string(nl->id[i]));
        }
    if (roms > 1 || rams > 1)
        nl_fail("at most one ROM port and one RAM port are supported");
}

// sms: SMs of the device the levels launch on (one latency wave = sms tasks).
void build_dag(vsp_netlist* nl, int sms)
{
    const int C = (int)nl->kind.size();
    nl->node_of_cell.assign(C, -1);
    for (int i = 0; i < C; i++) {
        if (nl->kind[i] == cDff) {
            nl->dff_cells.push_back(i);
            continue;
        }
        if (nl->kind[i] == cRom)
            nl->rom_cell = i;
        if (nl->kind[i] == cRam)
            nl->ram_cell = i;
        nl->node_of_cell[i] = (int)nl->dag_cells.size();
        nl->dag_cells.push_back(i);
    }
    std::vector<int> producer(nl->nets, -1);
    for (int i = 0; i < C; i++)
        if (nl->node_of_cell[i] >= 0)
            for (int k = nl->out_off[i]; k < nl->out_off[i + 1]; k++)
                producer[nl->out_nets[k]] = nl->node_of_cell[i];
    const int n = (int)nl->dag_cells.size();
    std::vector<std::vector<int>> consumers(n);
    std::vector<int> indeg(n, 0);
    for (int node = 0; node < n; node++) {
        const int c = nl->dag_cells[node];
        for (int k = nl->in_off[c]; k < nl->in_off[c + 1]; k++) {
            const int p = producer[nl->in_nets[k]];
            if (p >= 0) {
                consumers[p].push_back(node);
                indeg[node]++;
            }
        }
    }
    // Kahn's algorithm; level = longest path from the sources
    nl->level.assign(n, 0);
    std::vector<int> q, topo;
    for (int i = 0; i < n; i++)
        if (indeg[i] == 0)
            q.push_back(i);
    for (size_t h = 0; h < q.size(); h++) {
        const int node = q[h];
        topo.push_back(node);
        for (int cns : consumers[node]) {
            nl->level[cns] = std::max(nl->level[cns], nl->level[node] + 1);
            if (--indeg[cns] == 0)
                q.push_back(cns);
        }
    }
    if ((int)topo.size() != n) {
        for (int i = 0; i < n; i++)
            if (indeg[i] > 0)
                nl_fail("combinational cycle through cell " + std::to_string(nl->id[nl->dag_cells[i]]));
    }
    nl->height.assign(n, 0);
    for (auto it = topo.rbegin(); it != topo.rend(); ++it)
        for (int cns : consumers[*it])
            nl->height[*it] = std::max(nl->height[*it], nl->height[cns] + 1);
    int maxLevel = -1;
    std::vector<int> width;
    for (int i = 0; i < n; i++) {
        maxLevel = std::max(maxLevel, nl->level[i]);
        if ((int)width.size() <= nl->level[i])
            width.resize(nl->level[i] + 1, 0);
        width[nl->level[i]]++;
    }
    nl->gmax = 0;
    for (int w : width)
        nl->gmax = std::max(nl->gmax, w);
    nl->depth = maxLevel + 1;
    // Launch schedule: the ASAP levels (nl->level, the reference's buildDag) with gates that
    // have slack moved one level later when their level holds more blind-rotation tasks
    // than one wave of the latency kernel (one task per SM): a 149-task level costs two
    // 630-step waves, 148 tasks one.  A gate moves from L to L + 1 only if every consumer
    // sits at L + 2 or later (DFF inputs and module outputs are read after the cycle), so
    // each gate still sees the same input ciphertexts and computes the same output words.
    std::vector<int> slev(nl->level);
    {
        auto tasks_of = [&](int node) {
            const int k = nl->kind[nl->dag_cells[node]];
            return k == cMux ? 2 : (k == cNot || k > cXor) ? 0 : 1;
        };
        std::vector<std::vector<int>> at(std::max(nl->depth, 0));
        for (int node = 0; node < n; node++)
            if (nl->kind[nl->dag_cells[node]] <= cXor)
                at[slev[node]].push_back(node);
        // Only when the level can get down to one wave, and without pushing the next level
        // out of the latency kernel's two-wave range; the next level then sheds its own
        // excess the same way (the last level keeps what it receives).
        const int cap = sms;
        auto level_tasks = [&](int L) {
            int T = 0;
            for (int node : at[L])
                T += tasks_of(node);
            return T;
        };
        for (int L = 0; L + 1 < nl->depth; L++) {
            int T = level_tasks(L);
            if (T <= cap || T > 2 * cap)
                continue;
            auto movable = [&](int node) {
                if (tasks_of(node) == 0)
                    return false;
                for (int cns : consumers[node])
                    if (slev[cns] < L + 2)
                        return false;
                return true;
            };
            int M = 0;
            for (int node : at[L])
                M += movable(node) ? tasks_of(node) : 0;
            int Tn = level_tasks(L + 1);
            if (T - M > cap || Tn + (T - cap) > 2 * cap)
                continue;
            std::vector<int> keep;
            for (int node : at[L]) {
                if (T > cap && movable(node)) {
                    slev[node] = L + 1;
                    at[L + 1].push_back(node);
                    T -= tasks_of(node);
                }
                else {
                    keep.push_back(node);
                }
            }
            at[L].swap(keep);
        }
    }
    nl->launch_level = slev;
    nl->level_gates.assign(std::max(nl->depth, 0), {});
    nl->level_mem.assign(std::max(nl->depth, 0), {});
    for (int node = 0; node < n; node++) {
        const int c = nl->dag_cells[node];
        const int k = nl->kind[c];
        if (k <= cXor)
            nl->level_gates[slev[node]].push_back(c);
        else if (k == cRom || k == cRam)
            nl->level_mem[nl->level[node]].push_back(c);
        else
            nl->const_cells.push_back(c);
    }
    nl->max_level_ctas = 0;
    nl->level_tasks.clear();
    for (const auto& lg : nl->level_gates) {
        int tasks = 0;
        for (int cell : lg)
            tasks += nl->kind[cell] == cMux ? 2 : nl->kind[cell] == cNot ? 0 : 1;
        nl->level_tasks.push_back(tasks);
        const int ctas = tasks <= 2 * sms ? (tasks > 64 ? (tasks + 1) / 2 : tasks) : sms;
        nl->max_level_ctas = std::max(nl->max_level_ctas, ctas);
    }
}

// tlweTrivial (ops.cpp:212-217): a = 0, b = +-mu
std::vector<uint32_t> trivial_tlwe(uint32_t n, bool m)
{
    std::vector<uint32_t> t(n + 1, 0);
    t[n] = m ? kMu32 : 0u - kMu32;
    return t;
}

void upload_ints(vsp_ctx* c, DevBuf& buf, const std::vector<int>& v, cudaStream_t st)
{
    int* d = buf.as<int>(std::max<size_t>(v.size(), 1));
    h2d(c, d, v.data(), v.size() * sizeof(int), st);
}

// A ROM port and a RAM port in the same level: their address circuit bootstraps (v_rom + v
// TLWEs -> TRGSWs) run as ONE batched launch sequence -- the level-2 blind rotations of
// both ports side by side on the SMs -- then the two ports proceed as in the per-cell
// path.  The ports are independent, so the results equal the per-port order.
void run_mem_pair(vsp_netlist* nl, const std::vector<int>& cells, uint32_t* vals, cudaStream_t st)
{
    vsp_ctx* c = nl->ctx;
    const size_t n1 = c->p.n + 1;
    const int rom = nl->kind[cells[0]] == cRom ? cells[0] : cells[1];
    const int ram = rom == cells[0] ? cells[1] : cells[0];
    std::vector<int> ins(nl->in_nets.begin() + nl->in_off[rom], nl->in_nets.begin() + nl->in_off[rom + 1]);
    const int vrom = (int)ins.size();
    ins.insert(ins.end(), nl->in_nets.begin() + nl->in_off[ram], nl->in_nets.begin() + nl->in_off[ram + 1]);
    std::vector<int> outs(nl->out_nets.begin() + nl->out_off[rom], nl->out_nets.begin() + nl->out_off[rom + 1]);
    const int nrom_out = (int)outs.size();
    outs.insert(outs.end(), nl->out_nets.begin() + nl->out_off[ram], nl->out_nets.begin() + nl->out_off[ram + 1]);
    const int w = (int)outs.size() - nrom_out;
    const int v = (int)ins.size() - vrom - w - 1;
    if (v != (int)nl->ram_v || w != (int)nl->ram_w)
        throw std::invalid_argument("ramCycle: address width mismatch");
    upload_ints(c, nl->nets_buf, ins, st);
    uint32_t* gin = nl->gin.as<uint32_t>(ins.size() * n1);
    uint32_t* gout = nl->gout.as<uint32_t>(outs.size() * n1);
    gather_tlwe_kernel<<<(unsigned)ins.size(), 128, 0, st>>>(nl->nets_buf.as<int>(0), (int)ins.size(),
                                                              vals, gin, (int)c->p.n);
    c->launches++;
    const uint32_t* g = gin + (size_t)vrom * n1;  // RAM: addr[v], wdata[w], wflag
    mem_pair_dev(c, nl->rom.as<uint32_t>(0), (int)nl->rom_nluts, nl->rom_depth, gin, vrom, gout,
                 nl->ram.as<uint32_t>(0), v, w, g, g + (size_t)(v + w) * n1, g + (size_t)v * n1,
                 gout + (size_t)nrom_out * n1, st);
    upload_ints(c, nl->nets_buf, outs, st);
    scatter_tlwe_kernel<<<(unsigned)outs.size(), 128, 0, st>>>(nl->nets_buf.as<int>(0), (int)outs.size(),
                                                                gout, vals, (int)c->p.n);
    c->launches++;
    VSP_CUDA_CHECK(cudaGetLastError());
}

// ram_overlap: SMs left to the deferred write bars beside the widest narrow level (two
// tasks per SM) and a margin for the levels' key-switch / gather kernels; 0 = no overlap.
int write_ctas(const vsp_netlist* nl)
{
    const vsp_ctx* c = nl->ctx;
    if (!c->ram_overlap || nl->ram_cell < 0 || !c->p.fft || sharded(c))
        return 0;
    const int k = c->sms - nl->max_level_ctas - 2;
    return k >= 16 ? k : 0;
}

void run_cycle_body(vsp_netlist* nl, cudaStream_t st);

void run_cycle(vsp_netlist* nl, cudaStream_t st)
{
    vsp_ctx* c = nl->ctx;
    const int k = write_ctas(nl);
    if (!k) {
        run_cycle_body(nl, st);
        return;
    }
    struct Restore {  // options hold for this cycle only, also on an exception
        vsp_ctx* c;
        int lat;
        ~Restore()
        {
            c->lat_tasks = lat;
            c->defer_write_now = false;
            c->w_ctas = 0;
        }
    } restore{c, c->lat_tasks};
    c->lat_tasks = 2;
    c->w_ctas = k;
    c->defer_write_now = true;
    run_cycle_body(nl, st);
}

void run_cycle_body(vsp_netlist* nl, cudaStream_t st)
{
    vsp_ctx* c = nl->ctx;
    const uint32_t n = c->p.n;
    const size_t n1 = n + 1;
    uint32_t* vals = nl->values.as<uint32_t>((size_t)nl->nets * n1);
    // sources: module inputs and DFF outputs (engine.hpp:271-274)
    if (!nl->input_nets.empty()) {
        upload_ints(c, nl->nets_buf, nl->input_nets, st);
        scatter_tlwe_kernel<<<(unsigned)nl->input_nets.size(), 128, 0, st>>>(
            nl->nets_buf.as<int>(0), (int)nl->input_nets.size(), nl->inputs_store.as<uint32_t>(0),
            vals, (int)n);
        c->launches++;
    }
    if (!nl->dff_q.empty()) {
        upload_ints(c, nl->nets_buf, nl->dff_q, st);
        scatter_tlwe_kernel<<<(unsigned)nl->dff_q.size(), 128, 0, st>>>(
            nl->nets_buf.as<int>(0), (int)nl->dff_q.size(), nl->dff.as<uint32_t>(0), vals, (int)n);
        c->launches++;
    }
    VSP_CUDA_CHECK(cudaGetLastError());
    // write-bar backfill: idle latency-wave slots of levels L.. (one GPU, FFT path,
    // write unit inline); levels without blind rotations launch nothing and take none
    c->bar_total = c->bar_done = 0;
    struct BarReset {  // no deferred write bar outlives the cycle (also on an exception)
        vsp_ctx* c;
        ~BarReset() { c->bar_total = c->bar_done = c->bar_cap = 0; }
    } bar_reset{c};
    const bool backfill = c->backfill && c->p.fft && !sharded(c) && !c->defer_write_now;
    auto spare_from = [&](int L) {
        int cap = 0;
        for (int l = L; l < nl->depth; l++)
            if (nl->level_tasks[l] >= 1 && nl->level_tasks[l] < c->sms)
                cap += c->sms - nl->level_tasks[l];
        return cap;
    };
    struct BarCap {  // bar_cap is open only while a RAM port of this cycle runs
        vsp_ctx* c;
        ~BarCap() { c->bar_cap = 0; }
    };
    // Each level: its memory ports first, then its gates (same ASAP level, so neither
    // reads the other's outputs): the level's gate launch can then take deferred write
    // bars of its own RAM port.
    auto run_mem = [&](int L) {
        BarCap bar_guard{c};
        if (backfill && !nl->level_mem[L].empty())
            c->bar_cap = spare_from(L);
        if (nl->level_mem[L].size() == 2 && nl->has_rom && nl->has_ram) {
            run_mem_pair(nl, nl->level_mem[L], vals, st);
            return;
        }
        for (int cell : nl->level_mem[L]) {
            std::vector<int> ins(nl->in_nets.begin() + nl->in_off[cell],
                                 nl->in_nets.begin() + nl->in_off[cell + 1]);
            std::vector<int> outs(nl->out_nets.begin() + nl->out_off[cell],
                                  nl->out_nets.begin() + nl->out_off[cell + 1]);
            upload_ints(c, nl->nets_buf, ins, st);
            uint32_t* gin = nl->gin.as<uint32_t>(ins.size() * n1);
            uint32_t* gout = nl->gout.as<uint32_t>(outs.size() * n1);
            gather_tlwe_kernel<<<(unsigned)ins.size(), 128, 0, st>>>(nl->nets_buf.as<int>(0),
                                                                      (int)ins.size(), vals, gin,
                                                                      (int)n);
            c->launches++;
            if (nl->kind[cell] == cRom) {  // engine.hpp:361-366
                if (!nl->has_rom)
                    throw std::runtime_error("ROM image not bound");
                rom_read_dev(c, nl->rom.as<uint32_t>(0), (int)nl->rom_nluts, nl->rom_depth, gin,
                             (int)ins.size(), gout, st);
            }
            else {  // engine.hpp:367-376: addr[v], wdata[w], wflag
                if (!nl->has_ram)
                    throw std::runtime_error("RAM image not bound");
                const int w = (int)outs.size();
                const int v = (int)ins.size() - w - 1;
                if (v != (int)nl->ram_v || w != (int)nl->ram_w)
                    throw std::invalid_argument("ramCycle: address width mismatch");
                ram_cycle_dev(c, nl->ram.as<uint32_t>(0), v, w, gin, gin + (size_t)(v + w) * n1,
                              gin + (size_t)v * n1, gout, st);
            }
            upload_ints(c, nl->nets_buf, outs, st);
            scatter_tlwe_kernel<<<(unsigned)outs.size(), 128, 0, st>>>(
                nl->nets_buf.as<int>(0), (int)outs.size(), gout, vals, (int)n);
            c->launches++;
            VSP_CUDA_CHECK(cudaGetLastError());
        }
    };
    if (nl->lvl_off.empty()) {
        // static per netlist: every level's input / output nets and kinds
        std::vector<int> all;
        nl->lvl_kinds.assign(nl->depth, {});
        for (int L = 0; L < nl->depth; L++) {
            const auto& gates = nl->level_gates[L];
            nl->lvl_off.push_back(all.size());
            const size_t base = all.size();
            all.resize(base + gates.size() * 4, -1);
            for (size_t g = 0; g < gates.size(); g++) {
                const int cell = gates[g];
                nl->lvl_kinds[L].push_back(nl->kind[cell]);
                for (int k = nl->in_off[cell], q = 0; k < nl->in_off[cell + 1]; k++, q++)
                    all[base + g * 3 + q] = nl->in_nets[k];
                all[base + gates.size() * 3 + g] = nl->out_nets[nl->out_off[cell]];
            }
        }
        int* d = nl->lvl_nets.as<int>(std::max<size_t>(all.size(), 1));
        if (!all.empty())
            VSP_CUDA_CHECK(cudaMemcpyAsync(d, all.data(), all.size() * sizeof(int),
                                           cudaMemcpyHostToDevice, st));
        VSP_CUDA_CHECK(cudaStreamSynchronize(st));  // `all` is pageable and goes out of scope
    }
    auto run_gates = [&](int L) {
        const auto& gates = nl->level_gates[L];
        if (!gates.empty() && !sharded(c)) {
            // one GPU: the level reads its inputs from and writes its outputs into the value
            // table by net index (no gather / scatter kernels)
            const size_t G = gates.size();
            const int* d = nl->lvl_nets.as<int>(0) + nl->lvl_off[L];
            const LevelIdx lx{vals, d, d + 3 * G};
            hom_gate_dev(c, nl->lvl_kinds[L].data(), nullptr, nullptr, G, st, nullptr, &lx);
            VSP_CUDA_CHECK(cudaGetLastError());
        }
        else if (!gates.empty()) {
            const int G = (int)gates.size();
            std::vector<int> gnets((size_t)G * 3, -1), onets(G);
            std::vector<int32_t> kinds(G);
            for (int g = 0; g < G; g++) {
                const int cell = gates[g];
                kinds[g] = nl->kind[cell];  // CellKind 0..9 == GateKind 0..9
                for (int k = nl->in_off[cell], s = 0; k < nl->in_off[cell + 1]; k++, s++)
                    gnets[(size_t)g * 3 + s] = nl->in_nets[k];
                onets[g] = nl->out_nets[nl->out_off[cell]];
            }
            upload_ints(c, nl->nets_buf, gnets, st);
            uint32_t* gin = nl->gin.as<uint32_t>((size_t)G * 3 * n1);
            uint32_t* gout = nl->gout.as<uint32_t>((size_t)G * n1);
            gather_tlwe_kernel<<<G * 3, 128, 0, st>>>(nl->nets_buf.as<int>(0), G * 3, vals, gin,
                                                      (int)n);
            c->launches++;
            hom_gate_level_dev(c, kinds.data(), gin, gout, (size_t)G, st);  // sharded when world > 1
            upload_ints(c, nl->nets_buf, onets, st);
            scatter_tlwe_kernel<<<G, 128, 0, st>>>(nl->nets_buf.as<int>(0), G, gout, vals, (int)n);
            c->launches++;
            VSP_CUDA_CHECK(cudaGetLastError());
        }
    };
    for (int L = 0; L < nl->depth; L++) {
        run_mem(L);
        run_gates(L);
    }
    bar_flush(c, st);  // deferred write bars no later level took
    nl->table_valid = true;
    // synchronous DFF latch (engine.hpp:341-345): sample every D, then update all Qs
    if (!nl->dff_d.empty()) {
        upload_ints(c, nl->nets_buf, nl->dff_d, st);
        gather_tlwe_kernel<<<(unsigned)nl->dff_d.size(), 128, 0, st>>>(
            nl->nets_buf.as<int>(0), (int)nl->dff_d.size(), vals, nl->dff.as<uint32_t>(0), (int)n);
        c->launches++;
        VSP_CUDA_CHECK(cudaGetLastError());
    }
}

}  // namespace
