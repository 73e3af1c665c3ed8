// nccl_min.h — NCCL types for the dlopen'ed API (symbols resolved at run time).
#pragma once
#include <nccl.h>
